/* Declaration-only CBLAS header for building the reference library against
 * the OpenBLAS 0.3.15 that ships inside the image (opencv wheel). The image
 * has no system cblas.h; these are the standard CBLAS prototypes for the four
 * routines the reference calls (src/gemm.cpp:55,63,70,79). TEST
 * INFRASTRUCTURE ONLY — used by oracle/Makefile, never by the product. */
#ifndef MUMODE_ORACLE_CBLAS_SHIM_H
#define MUMODE_ORACLE_CBLAS_SHIM_H
#ifdef __cplusplus
extern "C" {
#endif
typedef enum { CblasRowMajor = 101, CblasColMajor = 102 } CBLAS_ORDER;
typedef enum { CblasNoTrans = 111, CblasTrans = 112, CblasConjTrans = 113 } CBLAS_TRANSPOSE;
typedef enum { CblasUpper = 121, CblasLower = 122 } CBLAS_UPLO;
typedef enum { CblasNonUnit = 131, CblasUnit = 132 } CBLAS_DIAG;
typedef enum { CblasLeft = 141, CblasRight = 142 } CBLAS_SIDE;

void cblas_dgemm(CBLAS_ORDER, CBLAS_TRANSPOSE, CBLAS_TRANSPOSE, int m, int n, int k,
                 double alpha, const double* a, int lda, const double* b, int ldb,
                 double beta, double* c, int ldc);
void cblas_zgemm(CBLAS_ORDER, CBLAS_TRANSPOSE, CBLAS_TRANSPOSE, int m, int n, int k,
                 const void* alpha, const void* a, int lda, const void* b, int ldb,
                 const void* beta, void* c, int ldc);
void cblas_dtrsm(CBLAS_ORDER, CBLAS_SIDE, CBLAS_UPLO, CBLAS_TRANSPOSE, CBLAS_DIAG, int m,
                 int n, double alpha, const double* a, int lda, double* b, int ldb);
void cblas_ztrsm(CBLAS_ORDER, CBLAS_SIDE, CBLAS_UPLO, CBLAS_TRANSPOSE, CBLAS_DIAG, int m,
                 int n, const void* alpha, const void* a, int lda, void* b, int ldb);
#ifdef __cplusplus
}
#endif
#endif
