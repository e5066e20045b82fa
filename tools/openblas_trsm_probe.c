// Probe: the triangular-solve order of OpenBLAS cblas_dtrsm (the arithmetic of the
// reference lu_solve, lu.hpp:52-69) against the restatement used by the host
// expm (paper_2112_11238_b200/csrc/host_util.cpp). Prints the number of
// differing elements per case (0 = bitwise). Build and run:
//   OB=/opt/prime-rl/.venv/lib/python3.12/site-packages/opencv_python_headless.libs
//   gcc -O2 -DUSEFMA -ffp-contract=off tools/openblas_trsm_probe.c -o /tmp/tp \
//       -L$OB -l:libopenblasp-r0-59ffcd50.3.15.so -lm
//   LD_LIBRARY_PATH=$OB OPENBLAS_CORETYPE=SKYLAKEX /tmp/tp 200 200
// (without -DUSEFMA the in-block updates are multiply-then-subtract: not bitwise)
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <string.h>
void cblas_dtrsm(int,int,int,int,int,int,int,double,const double*,int,double*,int);
static double rnd(){return (double)rand()/RAND_MAX*2-1;}
#ifndef USEFMA
#define SUB(c,x,a) ((c) - (x)*(a))
#else
#define SUB(c,x,a) fma(-(x),(a),(c))
#endif
#define UM 16
// forward, lower, unit: rows in blocks of UM (remainder blocks 8,4,2,1 after), GEMM update then in-block solve
__attribute__((target("avx2,fma"))) void fwd(int n,int nrhs,const double*L,double*X){
  for(int j=0;j<nrhs;j++){double*x=X+(size_t)j*n;
    int r0=0; int sizes[64],ns=0; int full=n/UM; for(int b=0;b<full;b++)sizes[ns++]=UM; for(int i=UM/2;i>0;i>>=1) if(n&i) sizes[ns++]=i;
    for(int b=0;b<ns;b++){int bs=sizes[b];
      for(int r=r0;r<r0+bs;r++){ if(r0>0){double acc=0; for(int k=0;k<r0;k++) acc=fma(L[r+(size_t)k*n],x[k],acc); x[r]=x[r]-acc;} }
      for(int i=r0;i<r0+bs;i++){ double bb=x[i]*1.0; x[i]=bb; for(int k=i+1;k<r0+bs;k++) x[k]=SUB(x[k],bb,L[k+(size_t)i*n]); }
      r0+=bs; } } }
// backward, upper, non-unit: remainder block at the bottom first (sizes 1,2,4,8 from the bottom), then UM blocks upward
__attribute__((target("avx2,fma"))) void bwd(int n,int nrhs,const double*U,double*X){
  for(int j=0;j<nrhs;j++){double*x=X+(size_t)j*n;
    int starts[64],lens[64],nb=0; int top=n;
    for(int i=1;i<UM;i*=2) if(n&i){ int s=(n&~(i-1))-i; starts[nb]=s; lens[nb]=i; nb++; }
    int full=n/UM; int s=(n&~(UM-1))-UM; for(int b=0;b<full;b++){starts[nb]=s;lens[nb]=UM;nb++; s-=UM;}
    for(int b=0;b<nb;b++){int r0=starts[b],bs=lens[b]; int kk=r0+bs;
      if(kk<n) for(int r=r0;r<r0+bs;r++){double acc=0; for(int k=kk;k<n;k++) acc=fma(U[r+(size_t)k*n],x[k],acc); x[r]=x[r]-acc;}
      for(int i=r0+bs-1;i>=r0;i--){ double inv=1.0/U[i+(size_t)i*n]; double bb=x[i]*inv; x[i]=bb; for(int k=r0;k<i;k++) x[k]=SUB(x[k],bb,U[k+(size_t)i*n]); }
    } } }
int main(int argc,char**argv){int n=argc>1?atoi(argv[1]):200,m=argc>2?atoi(argv[2]):200; size_t nn=(size_t)n*n;
 double*A=malloc(8*nn),*B=malloc(8*n*m),*X1=malloc(8*n*m),*X2=malloc(8*n*m);
 for(size_t i=0;i<nn;i++)A[i]=rnd(); for(int i=0;i<n;i++)A[i+(size_t)i*n]+=n*0.1; for(size_t i=0;i<(size_t)n*m;i++)B[i]=rnd();
 memcpy(X1,B,8*n*m); memcpy(X2,B,8*n*m);
 cblas_dtrsm(102,141,122,111,132,n,m,1.0,A,n,X1,n); fwd(n,m,A,X2);
 int d=0; for(size_t i=0;i<(size_t)n*m;i++) d+=X1[i]!=X2[i]; printf("fwd n=%d diffs=%d\n",n,d);
 memcpy(X1,B,8*n*m); memcpy(X2,B,8*n*m);
 cblas_dtrsm(102,141,121,111,131,n,m,1.0,A,n,X1,n); bwd(n,m,A,X2);
 d=0; for(size_t i=0;i<(size_t)n*m;i++) d+=X1[i]!=X2[i]; printf("bwd n=%d diffs=%d\n",n,d);}
