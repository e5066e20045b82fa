// Generic mu-mode product kernel: any extents, any alignment, real or complex,
// forward or adjoint factor. SIMT fp64 FMA, operands staged through shared
// memory. This is the path for shapes the TMA/DMMA kernel cannot describe
// (odd extents, unaligned bases, tiny modes); it computes
//     S(a, i, c) = sum_{k ascending} op(L)(i, k) * T(a, k, c)
// with a over modes < mu (stride 1), c over modes > mu -- the index form of
// core::mode_product (proj/include/mumode/mode_product.hpp:64-77) without the
// permute/ipermute pair of mode_product.hpp:73-76.
#pragma once
#include "common.cuh"

namespace mumode_gpu {

struct GenericArgs {
  const double* T;  // (A, K, C) column-major
  const double* L;  // op(L)(i, k) = L[i*sLi + k*sLk] (complex: in units of complex)
  double* S;        // (A, N, C)
  int64_t A, K, N, C;
  int64_t sLi, sLk;
  int conj;  // complex only: conjugate L entries (cttucker)
  int accumulate;  // S += result (kronsumv)
};

constexpr int kGenFibers = 64;  // fibers (a, c) per CTA
constexpr int kGenRows = 32;    // output rows i per CTA
constexpr int kGenK = 16;       // k chunk staged per iteration
constexpr int kGenThreads = 256;

// Each thread owns one fiber and kGenRows/4 = 8 output rows.
template <bool CPLX>
__global__ void __launch_bounds__(kGenThreads)
    modeprod_generic_kernel(GenericArgs g) {
  using V = typename std::conditional<CPLX, double2, double>::type;
  __shared__ V Ts[kGenK][kGenFibers];
  __shared__ V Ls[kGenK][kGenRows];

  const int tid = threadIdx.x;
  const int64_t f0 = static_cast<int64_t>(blockIdx.x) * kGenFibers;
  const int64_t i0 = static_cast<int64_t>(blockIdx.y) * kGenRows;
  const int64_t nfib = g.A * g.C;
  const int fl = tid % kGenFibers;
  const int ig = tid / kGenFibers;  // 0..3

  const V* T = reinterpret_cast<const V*>(g.T);
  const V* L = reinterpret_cast<const V*>(g.L);
  V* S = reinterpret_cast<V*>(g.S);

  // complex: four real chains (rr, ii, ri, ir) combined at the end, as
  // OpenBLAS's zgemm kernels do (re = rr - ii, im = ri + ir)
  V acc[kGenRows / 4], acc2[kGenRows / 4];
#pragma unroll
  for (int j = 0; j < kGenRows / 4; ++j) {
    if constexpr (CPLX) acc[j] = acc2[j] = make_double2(0.0, 0.0);
    else acc[j] = acc2[j] = 0.0;
  }

  for (int64_t k0 = 0; k0 < g.K; k0 += kGenK) {
    // stage T(a, k, c) for kGenFibers fibers x kGenK k's (coalesced along a)
    for (int e = tid; e < kGenK * kGenFibers; e += kGenThreads) {
      const int kk = e / kGenFibers, ff = e % kGenFibers;
      const int64_t f = f0 + ff, k = k0 + kk;
      V v;
      if constexpr (CPLX) v = make_double2(0.0, 0.0);
      else v = 0.0;
      if (f < nfib && k < g.K) {
        const int64_t a = f % g.A, c = f / g.A;
        v = T[a + k * g.A + c * g.A * g.K];
      }
      Ts[kk][ff] = v;
    }
    for (int e = tid; e < kGenK * kGenRows; e += kGenThreads) {
      const int kk = e / kGenRows, ii = e % kGenRows;
      const int64_t i = i0 + ii, k = k0 + kk;
      V v;
      if constexpr (CPLX) v = make_double2(0.0, 0.0);
      else v = 0.0;
      if (i < g.N && k < g.K) {
        v = L[i * g.sLi + k * g.sLk];
        if constexpr (CPLX) {
          if (g.conj) v.y = -v.y;
        }
      }
      Ls[kk][ii] = v;
    }
    __syncthreads();
    const int kmax = static_cast<int>((g.K - k0) < kGenK ? (g.K - k0) : kGenK);
    for (int kk = 0; kk < kmax; ++kk) {
      const V t = Ts[kk][fl];
#pragma unroll
      for (int j = 0; j < kGenRows / 4; ++j) {
        const V l = Ls[kk][ig + 4 * j];
        if constexpr (CPLX) {
          acc[j].x = fma(l.x, t.x, acc[j].x);    // rr
          acc2[j].x = fma(l.y, t.y, acc2[j].x);  // ii
          acc[j].y = fma(l.x, t.y, acc[j].y);    // ri
          acc2[j].y = fma(l.y, t.x, acc2[j].y);  // ir
        } else {
          acc[j] = fma(l, t, acc[j]);
        }
      }
    }
    __syncthreads();
  }

  if constexpr (CPLX) {
#pragma unroll
    for (int j = 0; j < kGenRows / 4; ++j) acc[j] = make_double2(acc[j].x - acc2[j].x, acc[j].y + acc2[j].y);
  }
  const int64_t f = f0 + fl;
  if (f < nfib) {
    const int64_t a = f % g.A, c = f / g.A;
#pragma unroll
    for (int j = 0; j < kGenRows / 4; ++j) {
      const int64_t i = i0 + ig + 4 * j;
      if (i < g.N) {
        V* dst = &S[a + i * g.A + c * g.A * g.N];
        if (g.accumulate) {
          if constexpr (CPLX) *dst = make_double2(dst->x + acc[j].x, dst->y + acc[j].y);
          else *dst = *dst + acc[j];
        } else {
          *dst = acc[j];
        }
      }
    }
  }
}

}  // namespace mumode_gpu
