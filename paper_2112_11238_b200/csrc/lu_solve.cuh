// Per-mode LU solves for the inverse Tucker operator (ops::itucker,
// proj/include/mumode/tucker.hpp:187-204): for mu = 1..d every mu-fibre x of
// the tensor is replaced by P_mu^-1 x through the stored factors of
// P_mu = L U (la::lu_solve, lu.hpp:52-69): the pivot row interchanges, a
// unit-lower forward solve and an upper backward solve. No inverse is formed.
//
// Arithmetic: each fibre is solved exactly as the reference's two cblas_?trsm
// calls compute one right-hand-side column on OpenBLAS 0.3.15's x86 (SkylakeX)
// kernels -- probed against cblas_dtrsm / cblas_ztrsm directly
// (tools/openblas_trsm_probe.c, tools/openblas_ztrsm_probe.c):
//   * rows in blocks of UM (16 real, 4 complex: the GEMM unroll in M); the
//     forward sweep takes full blocks from the top and the sub-UM remainder
//     blocks (8, 4, 2, 1 / 2, 1) after them, the backward sweep the remainder
//     blocks at the bottom first (1, 2, 4, 8 from the bottom) then full blocks
//     upwards;
//   * a block first subtracts ONE k-ordered FMA chain over the rows solved
//     before it (the GEMM kernel; complex: four real chains rr, ii, ri, ir
//     combined as (rr - ii, ri + ir), as the zgemm kernels accumulate), then
//     solves inside the block with fused multiply-add updates;
//   * the backward sweep multiplies by the reciprocal diagonal (real 1/u;
//     complex the packing routine's Smith reciprocal with a fused 1 + r*r).
// Bitwise equal to the reference for every real extent (n <= 400 probed) and
// for complex extents that are multiples of 4; complex remainder blocks
// (n % 4 != 0) take OpenBLAS's M-tail kernels, whose grouping differs at the
// 1e-16 level.
//
// Layout: one thread per fibre, 32 fibres per CTA staged in shared memory as
// x[k * 33 + t] (every solve-phase access is a warp-wide contiguous row; the
// fibre loads/stores are coalesced for mu > 1 and tile-linear for mu = 1).
// The factor is read through the read-only path (all lanes read the same
// element: broadcast). Extents too large for the shared tile solve in place in
// global memory (same arithmetic).
#pragma once

namespace mumode_gpu {

constexpr int kLuFibres = 32;
constexpr int kLuStride = kLuFibres + 1;

// --------------------------------------------------------------- real fibre
template <class X>
__device__ __forceinline__ void lu_fibre_f64(X x, const double* __restrict__ Q, const int64_t* __restrict__ piv,
                                             const double* __restrict__ invd, int n) {
  constexpr int UM = 16;
  for (int k = 0; k < n; ++k) {  // row interchanges in order (lu.hpp:58-64)
    const int p = static_cast<int>(__ldg(piv + k));
    if (p != k) {
      const double t = x(k);
      x(k) = x(p);
      x(p) = t;
    }
  }
  const int full_end = n & ~(UM - 1);
  // forward sweep, unit lower triangle
  for (int r0 = 0; r0 < n;) {
    const int bs = r0 < full_end ? UM : 1 << (31 - __clz(n - r0));
    if (r0 > 0) {
      double acc[UM];
#pragma unroll
      for (int r = 0; r < UM; ++r) acc[r] = 0.0;
      for (int k = 0; k < r0; ++k) {
        const double xk = x(k);
        const double* q = Q + int64_t(k) * n + r0;
#pragma unroll
        for (int r = 0; r < UM; ++r)
          if (r < bs) acc[r] = fma(__ldg(q + r), xk, acc[r]);
      }
#pragma unroll
      for (int r = 0; r < UM; ++r)
        if (r < bs) x(r0 + r) = __dsub_rn(x(r0 + r), acc[r]);
    }
    for (int i = r0; i < r0 + bs; ++i) {
      const double xi = x(i);
      for (int k = i + 1; k < r0 + bs; ++k) x(k) = fma(-xi, __ldg(Q + k + int64_t(i) * n), x(k));
    }
    r0 += bs;
  }
  // backward sweep, upper triangle with the reciprocal diagonal
  for (int top = n; top > 0;) {
    const int bs = top > full_end ? (top & -top) : UM;
    const int r0 = top - bs;
    if (top < n) {
      double acc[UM];
#pragma unroll
      for (int r = 0; r < UM; ++r) acc[r] = 0.0;
      for (int k = top; k < n; ++k) {
        const double xk = x(k);
        const double* q = Q + int64_t(k) * n + r0;
#pragma unroll
        for (int r = 0; r < UM; ++r)
          if (r < bs) acc[r] = fma(__ldg(q + r), xk, acc[r]);
      }
#pragma unroll
      for (int r = 0; r < UM; ++r)
        if (r < bs) x(r0 + r) = __dsub_rn(x(r0 + r), acc[r]);
    }
    for (int i = top - 1; i >= r0; --i) {
      const double xi = __dmul_rn(x(i), invd[i]);
      x(i) = xi;
      for (int k = r0; k < i; ++k) x(k) = fma(-xi, __ldg(Q + k + int64_t(i) * n), x(k));
    }
    top = r0;
  }
}

// ------------------------------------------------------------ complex fibre
// c -= p * a with the grouping of OpenBLAS's ztrsm in-block update.
__device__ __forceinline__ double2 ztrsm_update(double2 c, double2 p, double2 a) {
  const double t0 = fma(p.x, a.x, -__dmul_rn(p.y, a.y));
  const double t1 = fma(p.x, a.y, __dmul_rn(p.y, a.x));
  return make_double2(__dsub_rn(c.x, t0), __dsub_rn(c.y, t1));
}
// b * inv (inv the packed reciprocal diagonal)
__device__ __forceinline__ double2 ztrsm_scale(double2 b, double2 inv) {
  return make_double2(fma(inv.x, b.x, -__dmul_rn(inv.y, b.y)), fma(inv.x, b.y, __dmul_rn(inv.y, b.x)));
}
// Smith reciprocal of the packing routine (compinv) with the fused 1 + r*r.
__device__ __forceinline__ double2 ztrsm_recip(double2 a) {
  if (fabs(a.x) >= fabs(a.y)) {
    const double ratio = a.y / a.x;
    const double den = 1.0 / __dmul_rn(a.x, fma(ratio, ratio, 1.0));
    return make_double2(den, __dmul_rn(-ratio, den));
  }
  const double ratio = a.x / a.y;
  const double den = 1.0 / __dmul_rn(a.y, fma(ratio, ratio, 1.0));
  return make_double2(__dmul_rn(ratio, den), -den);
}

template <class X>
__device__ __forceinline__ void lu_fibre_c128(X x, const double2* __restrict__ Q, const int64_t* __restrict__ piv,
                                              const double2* __restrict__ invd, int n) {
  constexpr int UM = 4;
  for (int k = 0; k < n; ++k) {
    const int p = static_cast<int>(__ldg(piv + k));
    if (p != k) {
      const double2 t = x(k);
      x(k) = x(p);
      x(p) = t;
    }
  }
  const int full_end = n & ~(UM - 1);
  auto gemm_part = [&](int r0, int bs, int k0, int k1) {
    double rr[UM], ii[UM], ri[UM], ir[UM];
#pragma unroll
    for (int r = 0; r < UM; ++r) rr[r] = ii[r] = ri[r] = ir[r] = 0.0;
    for (int k = k0; k < k1; ++k) {
      const double2 xk = x(k);
      const double2* q = Q + int64_t(k) * n + r0;
#pragma unroll
      for (int r = 0; r < UM; ++r)
        if (r < bs) {
          const double2 a = __ldg(q + r);
          rr[r] = fma(a.x, xk.x, rr[r]);
          ii[r] = fma(a.y, xk.y, ii[r]);
          ri[r] = fma(a.x, xk.y, ri[r]);
          ir[r] = fma(a.y, xk.x, ir[r]);
        }
    }
#pragma unroll
    for (int r = 0; r < UM; ++r)
      if (r < bs) {
        const double2 c = x(r0 + r);
        x(r0 + r) = make_double2(__dsub_rn(c.x, __dsub_rn(rr[r], ii[r])), __dsub_rn(c.y, __dadd_rn(ri[r], ir[r])));
      }
  };
  const double2 one = make_double2(1.0, 0.0);
  for (int r0 = 0; r0 < n;) {
    const int bs = r0 < full_end ? UM : 1 << (31 - __clz(n - r0));
    if (r0 > 0) gemm_part(r0, bs, 0, r0);
    for (int i = r0; i < r0 + bs; ++i) {
      const double2 xi = ztrsm_scale(x(i), one);
      x(i) = xi;
      for (int k = i + 1; k < r0 + bs; ++k) x(k) = ztrsm_update(x(k), xi, __ldg(Q + k + int64_t(i) * n));
    }
    r0 += bs;
  }
  for (int top = n; top > 0;) {
    const int bs = top > full_end ? (top & -top) : UM;
    const int r0 = top - bs;
    if (top < n) gemm_part(r0, bs, top, n);
    for (int i = top - 1; i >= r0; --i) {
      const double2 xi = ztrsm_scale(x(i), invd[i]);
      x(i) = xi;
      for (int k = r0; k < i; ++k) x(k) = ztrsm_update(x(k), xi, __ldg(Q + k + int64_t(i) * n));
    }
    top = r0;
  }
}

template <class V>
struct StridedRef {
  V* base;
  int64_t stride;
  __device__ __forceinline__ V& operator()(int k) const { return base[int64_t(k) * stride]; }
};

// One mode of itucker: out(a, :, c) = P^-1 in(a, :, c) for all A*C fibres of
// length n (in may equal out: every CTA reads and writes only its own fibres).
template <bool CPLX>
__global__ void __launch_bounds__(kLuFibres) lu_solve_mode_kernel(const double* in, double* out, int64_t A, int n,
                                                                  int64_t C, const double* __restrict__ lu,
                                                                  const int64_t* __restrict__ piv, int staged) {
  using V = typename std::conditional<CPLX, double2, double>::type;
  extern __shared__ __align__(16) unsigned char lu_smem[];
  V* invd = reinterpret_cast<V*>(lu_smem);
  V* xs = invd + n;
  const V* Q = reinterpret_cast<const V*>(lu);
  const V* src = reinterpret_cast<const V*>(in);
  V* dst = reinterpret_cast<V*>(out);
  const int t = threadIdx.x;
  for (int i = t; i < n; i += blockDim.x) {
    if constexpr (CPLX)
      invd[i] = ztrsm_recip(Q[i + int64_t(i) * n]);
    else
      invd[i] = 1.0 / Q[i + int64_t(i) * n];
  }
  __syncthreads();
  const int64_t F = A * C, An = A * n;
  for (int64_t f0 = int64_t(blockIdx.x) * kLuFibres; f0 < F; f0 += int64_t(gridDim.x) * kLuFibres) {
    const int nf = static_cast<int>(F - f0 < kLuFibres ? F - f0 : kLuFibres);
    const int64_t f = f0 + t;
    const int64_t a = f % A, c = f / A;
    const int64_t off = a + c * An;  // element k of fibre f at off + k * A
    if (staged) {
      if (A == 1) {  // mu = 1: the tile's fibres are nf*n contiguous elements
        const V* s = src + f0 * n;
        for (int64_t e = t; e < int64_t(nf) * n; e += kLuFibres) {
          const int fl = static_cast<int>(e / n), k = static_cast<int>(e - int64_t(fl) * n);
          xs[k * kLuStride + fl] = s[e];
        }
      } else if (t < nf) {
        for (int k = 0; k < n; ++k) xs[k * kLuStride + t] = src[off + int64_t(k) * A];
      }
      __syncwarp();
      if (t < nf) {
        StridedRef<V> x{xs + t, kLuStride};
        if constexpr (CPLX)
          lu_fibre_c128(x, Q, piv, invd, n);
        else
          lu_fibre_f64(x, Q, piv, invd, n);
      }
      __syncwarp();
      if (A == 1) {
        V* d = dst + f0 * n;
        for (int64_t e = t; e < int64_t(nf) * n; e += kLuFibres) {
          const int fl = static_cast<int>(e / n), k = static_cast<int>(e - int64_t(fl) * n);
          d[e] = xs[k * kLuStride + fl];
        }
      } else if (t < nf) {
        for (int k = 0; k < n; ++k) dst[off + int64_t(k) * A] = xs[k * kLuStride + t];
      }
      __syncwarp();
    } else if (t < nf) {  // in place in global memory
      if (src != dst)
        for (int k = 0; k < n; ++k) dst[off + int64_t(k) * A] = src[off + int64_t(k) * A];
      StridedRef<V> x{dst + off, A};
      if constexpr (CPLX)
        lu_fibre_c128(x, Q, piv, invd, n);
      else
        lu_fibre_f64(x, Q, piv, invd, n);
    }
  }
}

}  // namespace mumode_gpu
