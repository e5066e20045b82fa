// Host preprocessing for the mu-mode engine: the seeded input generator and
// the matrix exponential used to build exponential-integrator factors.
// Neither is on the timed hot path.
#include <algorithm>
#include <cmath>
#include <complex>
#include <limits>
#include <numeric>
#include <cstdint>
#include <cstring>
#include <new>
#include <random>
#include <string>
#include <vector>

#include "../../include/mumode_gpu.h"

namespace mumode_gpu {
void set_error(const std::string& msg);
}

// ------------------------------------------------------------------ rng
// The reference draws every benchmark/test input from std::mt19937_64 with a
// FRESH std::normal_distribution<double> per tensor or matrix
// (tools/mumode_cli.cpp:94-121, tests/acceptance.cpp:41-66); libstdc++'s
// polar method caches its second sample inside the distribution object, so
// the call structure matters. These entry points reproduce it exactly by
// using the same libstdc++ engine and distribution.
struct mumode_rng_s {
  std::mt19937_64 eng;
};

extern "C" int mumode_rng_create(mumode_rng_t* r, uint64_t seed) {
  if (!r) return MUMODE_ERR_ARGUMENT;
  *r = new (std::nothrow) mumode_rng_s{std::mt19937_64(seed)};
  return *r ? MUMODE_OK : MUMODE_ERR_OOM;
}

extern "C" int mumode_rng_destroy(mumode_rng_t r) {
  delete r;
  return MUMODE_OK;
}

extern "C" int mumode_rng_normal(mumode_rng_t r, double* out, int64_t n, int complex_) {
  if (!r || (n > 0 && !out)) return MUMODE_ERR_ARGUMENT;
  std::normal_distribution<double> dist;
  const int64_t count = complex_ ? 2 * n : n;
  for (int64_t k = 0; k < count; ++k) out[k] = dist(r->eng);
  return MUMODE_OK;
}

extern "C" int mumode_rng_u64(mumode_rng_t r, uint64_t* out, int64_t n) {
  if (!r || (n > 0 && !out)) return MUMODE_ERR_ARGUMENT;
  for (int64_t k = 0; k < n; ++k) out[k] = r->eng();
  return MUMODE_OK;
}

// ------------------------------------------------------------------ expm
// Scaling and squaring with diagonal Pade approximants of degree 3,5,7,9,13
// (N. J. Higham, "The scaling and squaring method for the matrix exponential
// revisited", SIAM J. Matrix Anal. Appl. 26(4), 2005, Algorithm 2.3): pick the
// lowest degree whose theta bound covers ||A||_1, otherwise scale by 2^-s to
// reach theta_13, evaluate r_13 = (V-U)^{-1}(V+U) and square s times.
namespace {

using Mat = std::vector<double>;  // column-major n x n

// C = A B with every element one k-ordered fused-multiply-add chain from 0:
// the arithmetic of the reference's la::gemm (cblas_dgemm, src/gemm.cpp:53-66)
// on OpenBLAS's x86 kernels, so products round like the reference's.
__attribute__((target("avx2,fma"))) void matmul(const Mat& A, const Mat& B, Mat& C, int64_t n) {
  std::fill(C.begin(), C.end(), 0.0);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t k = 0; k < n; ++k) {
      const double b = B[k + j * n];
      const double* a = &A[k * n];
      double* c = &C[j * n];
      for (int64_t i = 0; i < n; ++i) c[i] = std::fma(a[i], b, c[i]);
    }
}

double norm1(const Mat& A, int64_t n) {
  double best = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += std::fabs(A[i + j * n]);
    best = std::max(best, s);
  }
  return best;
}

// Triangular solves in the arithmetic of the reference's lu_solve
// (lu.hpp:52-69: two cblas_dtrsm calls, src/gemm.cpp:68-74) on OpenBLAS's
// x86 kernels (trsm drivers with 16-row blocks, DGEMM_UNROLL_M = 16): a row
// block first subtracts ONE k-ordered FMA chain over the rows solved before it
// (the GEMM kernel, alpha = -1), then solves inside the block with FMA
// updates; the backward sweep multiplies by the reciprocal diagonal and takes
// the sub-16 remainder block at the bottom first. Verified bitwise against
// cblas_dtrsm of OpenBLAS 0.3.15 (SkylakeX) for n <= 384 (one k-panel).
constexpr int kTrsmBlock = 16;

__attribute__((target("avx2,fma"))) void trsm_lower_unit(const Mat& Q, double* x, int64_t n) {
  std::vector<int64_t> blocks;
  for (int64_t b = 0; b < n / kTrsmBlock; ++b) blocks.push_back(kTrsmBlock);
  for (int i = kTrsmBlock / 2; i > 0; i >>= 1)
    if (n & i) blocks.push_back(i);
  int64_t r0 = 0;
  for (const int64_t bs : blocks) {
    if (r0 > 0)
      for (int64_t r = r0; r < r0 + bs; ++r) {
        double acc = 0.0;
        for (int64_t k = 0; k < r0; ++k) acc = std::fma(Q[r + k * n], x[k], acc);
        x[r] = x[r] - acc;
      }
    for (int64_t i = r0; i < r0 + bs; ++i)
      for (int64_t k = i + 1; k < r0 + bs; ++k) x[k] = std::fma(-x[i], Q[k + i * n], x[k]);
    r0 += bs;
  }
}

__attribute__((target("avx2,fma"))) void trsm_upper(const Mat& Q, const std::vector<double>& inv_diag, double* x,
                                                    int64_t n) {
  std::vector<std::pair<int64_t, int64_t>> blocks;  // (first row, rows), in solve order
  for (int i = 1; i < kTrsmBlock; i *= 2)
    if (n & i) blocks.emplace_back((n & ~int64_t(i - 1)) - i, i);
  for (int64_t s = (n & ~int64_t(kTrsmBlock - 1)) - kTrsmBlock; s >= 0; s -= kTrsmBlock) blocks.emplace_back(s, kTrsmBlock);
  for (const auto& [r0, bs] : blocks) {
    const int64_t kk = r0 + bs;
    if (kk < n)
      for (int64_t r = r0; r < kk; ++r) {
        double acc = 0.0;
        for (int64_t k = kk; k < n; ++k) acc = std::fma(Q[r + k * n], x[k], acc);
        x[r] = x[r] - acc;
      }
    for (int64_t i = kk - 1; i >= r0; --i) {
      const double xi = x[i] * inv_diag[static_cast<size_t>(i)];
      x[i] = xi;
      for (int64_t k = r0; k < i; ++k) x[k] = std::fma(-xi, Q[k + i * n], x[k]);
    }
  }
}

// Solve Q X = P in place (P overwritten by X): LU with partial pivoting as
// lu_factor (lu.hpp:23-47, plain multiply-subtract updates, reciprocal pivot),
// row swaps, then the two triangular solves above. Returns false on an
// exactly singular pivot.
bool solve(Mat Q, Mat& P, int64_t n) {
  std::vector<int64_t> piv(static_cast<size_t>(n));
  for (int64_t k = 0; k < n; ++k) {
    int64_t p = k;
    double best = std::fabs(Q[k + k * n]);
    for (int64_t i = k + 1; i < n; ++i)
      if (std::fabs(Q[i + k * n]) > best) best = std::fabs(Q[i + k * n]), p = i;
    if (best == 0.0) return false;
    piv[static_cast<size_t>(k)] = p;
    if (p != k)
      for (int64_t j = 0; j < n; ++j) std::swap(Q[k + j * n], Q[p + j * n]);
    const double inv_pivot = 1.0 / Q[k + k * n];
    for (int64_t i = k + 1; i < n; ++i) {
      const double f = Q[i + k * n] * inv_pivot;
      Q[i + k * n] = f;
      for (int64_t j = k + 1; j < n; ++j) Q[i + j * n] -= f * Q[k + j * n];
    }
  }
  std::vector<double> inv_diag(static_cast<size_t>(n));
  for (int64_t k = 0; k < n; ++k) inv_diag[static_cast<size_t>(k)] = 1.0 / Q[k + k * n];
  for (int64_t c = 0; c < n; ++c) {
    double* x = &P[c * n];
    for (int64_t k = 0; k < n; ++k) {
      const int64_t p = piv[static_cast<size_t>(k)];
      if (p != k) std::swap(x[k], x[p]);
    }
    trsm_lower_unit(Q, x, n);
    trsm_upper(Q, inv_diag, x, n);
  }
  return true;
}

}  // namespace

extern "C" int mumode_expm_f64(int64_t n, const double* Ain, double* E) {
  if (n < 1 || !Ain || !E) {
    mumode_gpu::set_error("expm: matrix must be non-empty");
    return MUMODE_ERR_ARGUMENT;
  }
  const size_t nn = static_cast<size_t>(n * n);
  for (size_t k = 0; k < nn; ++k)
    if (!std::isfinite(Ain[k])) {
      mumode_gpu::set_error("expm: input has non-finite entries");
      return MUMODE_ERR_ARGUMENT;
    }
  // Pade coefficients b_0..b_m (Higham 2005, Table 2.3 / eq. (2.11)).
  static const double b3[] = {120, 60, 12, 1};
  static const double b5[] = {30240, 15120, 3360, 420, 30, 1};
  static const double b7[] = {17297280, 8648640, 1995840, 277200, 25200, 1512, 56, 1};
  static const double b9[] = {17643225600.0, 8821612800.0, 2075673600.0, 302702400.0,
                              30270240.0,    2162160.0,    110880.0,     3960.0,
                              90.0,          1.0};
  static const double b13[] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                               1187353796428800.0,  129060195264000.0,   10559470521600.0,
                               670442572800.0,      33522128640.0,       1323241920.0,
                               40840800.0,          960960.0,            16380.0,
                               182.0,               1.0};
  static const double theta[] = {1.495585217958292e-2, 2.539398330063230e-1,
                                 9.504178996162932e-1, 2.097847961257068e0,
                                 5.371920351148152e0};
  Mat A(Ain, Ain + nn), I(nn, 0.0), U(nn), V(nn), tmp(nn);
  for (int64_t i = 0; i < n; ++i) I[i + i * n] = 1.0;
  const double nrm = norm1(A, n);
  auto axpy = [&](Mat& Y, double a, const Mat& X) {
    for (size_t k = 0; k < nn; ++k) Y[k] += a * X[k];
  };
  int s = 0;
  const double* b = nullptr;
  int deg = 13;
  if (nrm <= theta[0]) b = b3, deg = 3;
  else if (nrm <= theta[1]) b = b5, deg = 5;
  else if (nrm <= theta[2]) b = b7, deg = 7;
  else if (nrm <= theta[3]) b = b9, deg = 9;
  if (deg < 13) {
    std::vector<Mat> even{I};  // I, A^2, A^4, ...
    Mat A2(nn);
    matmul(A, A, A2, n);
    even.push_back(A2);
    for (int k = 2; 2 * k < deg + 1; ++k) {
      Mat next(nn);
      matmul(even.back(), A2, next, n);
      even.push_back(next);
    }
    Mat Us(nn, 0.0);
    std::fill(V.begin(), V.end(), 0.0);
    for (int k = 0; 2 * k + 1 <= deg; ++k) axpy(Us, b[2 * k + 1], even[static_cast<size_t>(k)]);
    for (int k = 0; 2 * k <= deg - 1; ++k) axpy(V, b[2 * k], even[static_cast<size_t>(k)]);
    matmul(A, Us, U, n);
  } else {
    if (nrm > theta[4]) s = static_cast<int>(std::ceil(std::log2(nrm / theta[4])));
    const double sc = std::ldexp(1.0, -s);
    for (auto& v : A) v *= sc;
    Mat A2(nn), A4(nn), A6(nn), W(nn, 0.0), Us(nn);
    matmul(A, A, A2, n);
    matmul(A2, A2, A4, n);
    matmul(A2, A4, A6, n);
    axpy(W, b13[13], A6);
    axpy(W, b13[11], A4);
    axpy(W, b13[9], A2);
    matmul(A6, W, Us, n);
    axpy(Us, b13[7], A6);
    axpy(Us, b13[5], A4);
    axpy(Us, b13[3], A2);
    axpy(Us, b13[1], I);
    matmul(A, Us, U, n);
    Mat W2(nn, 0.0);
    axpy(W2, b13[12], A6);
    axpy(W2, b13[10], A4);
    axpy(W2, b13[8], A2);
    matmul(A6, W2, V, n);
    axpy(V, b13[6], A6);
    axpy(V, b13[4], A4);
    axpy(V, b13[2], A2);
    axpy(V, b13[0], I);
  }
  Mat P(nn), Q(nn);
  for (size_t k = 0; k < nn; ++k) P[k] = V[k] + U[k], Q[k] = V[k] - U[k];
  if (!solve(Q, P, n)) {
    mumode_gpu::set_error("expm: singular Pade denominator");
    return MUMODE_ERR_NUMERICAL;
  }
  for (int k = 0; k < s; ++k) {
    matmul(P, P, tmp, n);
    std::swap(P, tmp);
  }
  std::memcpy(E, P.data(), sizeof(double) * nn);
  return MUMODE_OK;
}

// ------------------------------------------------------------------ inverse
// Per-mode inverse for the inverse Tucker operator (ops::itucker,
// tucker.hpp:187-204): LU with partial pivoting (the FactorizedStack role,
// lu.hpp:23-47), then n solves against the identity. A zero pivot reports the
// reference's NumericalError text.
extern "C" int mumode_inverse_f64(int64_t n, const double* P, double* Pinv) {
  if (n < 1 || !P || !Pinv) {
    mumode_gpu::set_error("inverse: matrix must be non-empty");
    return MUMODE_ERR_ARGUMENT;
  }
  const size_t nn = static_cast<size_t>(n * n);
  Mat Q(P, P + nn), X(nn, 0.0);
  for (int64_t i = 0; i < n; ++i) X[static_cast<size_t>(i + i * n)] = 1.0;
  if (!solve(Q, X, n)) {
    mumode_gpu::set_error("lu_factor: singular pivot");
    return MUMODE_ERR_NUMERICAL;
  }
  std::memcpy(Pinv, X.data(), sizeof(double) * nn);
  return MUMODE_OK;
}

// ------------------------------------------------------------------ LU factors
// la::lu_factor (lu.hpp:23-47) restated on the same types: partial pivoting on
// |M(i,k)| (std::abs, complex modulus for complex), a reciprocal pivot
// T{1}/M(k,k), multipliers M(i,k)*inv_pivot and plain multiply-subtract
// updates (this file is compiled without FMA contraction, like the reference),
// so lu and piv are bitwise the reference's FactorizedStack factors.
namespace {
template <class T>
int lu_factor_impl(int64_t n, const T* A, T* lu, int64_t* piv) {
  if (n < 1 || !A || !lu || !piv) {
    mumode_gpu::set_error("lu_factor: matrix must be non-empty");
    return MUMODE_ERR_ARGUMENT;
  }
  std::copy(A, A + n * n, lu);
  auto M = [&](int64_t i, int64_t j) -> T& { return lu[i + j * n]; };
  for (int64_t k = 0; k < n; ++k) {
    int64_t p = k;
    double best = std::abs(M(k, k));
    for (int64_t i = k + 1; i < n; ++i)
      if (std::abs(M(i, k)) > best) {
        best = std::abs(M(i, k));
        p = i;
      }
    if (best == 0.0) {
      mumode_gpu::set_error("lu_factor: singular pivot");
      return MUMODE_ERR_NUMERICAL;
    }
    piv[k] = p;
    if (p != k)
      for (int64_t j = 0; j < n; ++j) std::swap(M(k, j), M(p, j));
    const T inv_pivot = T{1} / M(k, k);
    for (int64_t i = k + 1; i < n; ++i) {
      const T m = M(i, k) * inv_pivot;
      M(i, k) = m;
      for (int64_t j = k + 1; j < n; ++j) M(i, j) -= m * M(k, j);
    }
  }
  return MUMODE_OK;
}
}  // namespace

extern "C" int mumode_lu_factor_f64(int64_t n, const double* P, double* lu, int64_t* piv) {
  return lu_factor_impl<double>(n, P, lu, piv);
}

extern "C" int mumode_lu_factor_c128(int64_t n, const double* P, double* lu, int64_t* piv) {
  using C = std::complex<double>;
  return lu_factor_impl<C>(n, reinterpret_cast<const C*>(P), reinterpret_cast<C*>(lu), piv);
}

// ------------------------------------------------------------------ IMEX direct solver factors
// extract_tridiag (src/imex.cpp:28-48): the symmetric tridiagonal part of a
// factor M, rejecting entries off the three diagonals and asymmetric
// off-diagonals with the reference's ArgumentError texts.
extern "C" int mumode_extract_tridiag_f64(int64_t n, const double* M, double* diag, double* offdiag) {
  if (n < 1 || !M || !diag || (n > 1 && !offdiag)) {
    mumode_gpu::set_error("symtridiag_eig: empty matrix");
    return MUMODE_ERR_ARGUMENT;
  }
  double scale = 0.0;
  for (int64_t k = 0; k < n * n; ++k) scale = std::max(scale, std::abs(M[k]));
  for (int64_t i = 0; i < n; ++i) {
    diag[i] = M[i + i * n];
    for (int64_t j = 0; j < n; ++j)
      if (std::abs(i - j) > 1 && M[i + j * n] != 0.0) {
        mumode_gpu::set_error("imex direct backend: factor is not tridiagonal");
        return MUMODE_ERR_ARGUMENT;
      }
    if (i + 1 < n) {
      const double up = M[i + (i + 1) * n], lo = M[(i + 1) + i * n];
      if (std::abs(up - lo) > 1e-12 * scale) {
        mumode_gpu::set_error("imex direct backend: factor is not symmetric");
        return MUMODE_ERR_ARGUMENT;
      }
      offdiag[i] = 0.5 * (up + lo);
    }
  }
  return MUMODE_OK;
}

// la::symtridiag_eig with EigMode::FullVectors (src/tridiag.cpp:12-90):
// implicit-shift QL with Wilkinson shifts (cap 50 iterations per eigenvalue),
// rotations accumulated into the identity, eigenpairs sorted ascending.
// Same operations in the same order on the same types, so values and vectors
// are bitwise the reference's. vectors: m x m column-major, eigenvector j in
// column j.
extern "C" int mumode_symtridiag_eig_f64(int64_t m, const double* diag, const double* offdiag, double* values,
                                         double* vectors) {
  if (m < 1 || !diag || !values || !vectors || (m > 1 && !offdiag)) {
    mumode_gpu::set_error("symtridiag_eig: empty matrix");
    return MUMODE_ERR_ARGUMENT;
  }
  std::vector<double> d(diag, diag + m);
  std::vector<double> e(offdiag ? offdiag : diag, offdiag ? offdiag + (m - 1) : diag);
  e.push_back(0.0);
  std::vector<double> zs(static_cast<size_t>(m * m), 0.0);
  auto z = [&](int64_t i, int64_t j) -> double& { return zs[static_cast<size_t>(i + j * m)]; };
  for (int64_t i = 0; i < m; ++i) z(i, i) = 1.0;
  const double eps = std::numeric_limits<double>::epsilon();
  for (int64_t l = 0; l < m; ++l) {
    int iter = 0;
    int64_t mm;
    do {
      for (mm = l; mm < m - 1; ++mm) {
        const double dd = std::abs(d[mm]) + std::abs(d[mm + 1]);
        if (std::abs(e[mm]) <= eps * dd) break;
      }
      if (mm != l) {
        if (iter++ == 50) {
          mumode_gpu::set_error("symtridiag_eig: QL iteration did not converge");
          return MUMODE_ERR_NUMERICAL;
        }
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = d[mm] - d[l] + e[l] / (g + std::copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int64_t i;
        for (i = mm; i-- > l;) {
          double f = s * e[i];
          const double b = c * e[i];
          r = std::hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[mm] = 0.0;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          for (int64_t k = 0; k < m; ++k) {
            f = z(k, i + 1);
            z(k, i + 1) = s * z(k, i) + c * f;
            z(k, i) = c * z(k, i) - s * f;
          }
        }
        if (r == 0.0 && i + 1 > l) continue;
        d[l] -= p;
        e[l] = g;
        e[mm] = 0.0;
      }
    } while (mm != l);
  }
  std::vector<int64_t> order(static_cast<size_t>(m));
  std::iota(order.begin(), order.end(), int64_t{0});
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return d[a] < d[b]; });
  for (int64_t j = 0; j < m; ++j) {
    values[j] = d[static_cast<size_t>(order[static_cast<size_t>(j)])];
    for (int64_t k = 0; k < m; ++k) vectors[k + j * m] = z(k, order[static_cast<size_t>(j)]);
  }
  return MUMODE_OK;
}
