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
// Layout: 32 fibres per CTA staged in shared memory as x[k * 33 + fibre]
// (loads / stores coalesced along a for mu > 1 and tile-linear for mu = 1),
// each fibre solved by a group of UM lanes (below). Extents too large for the
// shared tile are solved in global memory (same arithmetic).
#pragma once

namespace mumode_gpu {

constexpr int kLuFibres = 32;
constexpr int kLuStride = kLuFibres + 4;  // 36 doubles: = 8 mod 32 words, conflict-free DMMA B fragments

// Cooperative layout: a fibre is solved by UM lanes (16 real, 4 complex), lane
// l owning row r0 + l of the current block. The GEMM part of a block is then
// UM independent k-ordered chains (one per lane, x[k] broadcast from shared
// memory, the factor's block rows read coalesced), and the in-block solve
// passes each finished x_i to the lanes below it by a shuffle -- the same
// operations in the same order per element as the serial restatement
// (host_util.cpp, tools/openblas_trsm_probe.c), on UM lanes at once.
// Row interchanges are applied while staging: x(k) = in(perm[k]), perm being
// the sequential swaps of piv applied to an index array (lu_perm_kernel).

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

template <class V>
__device__ __forceinline__ V shfl_v(V v, int src, int width) {
  if constexpr (sizeof(V) == 16) {
    return make_double2(__shfl_sync(0xffffffffu, v.x, src, width), __shfl_sync(0xffffffffu, v.y, src, width));
  } else {
    return __shfl_sync(0xffffffffu, v, src, width);
  }
}

// The lane's row of the factor through Qrow(k) = Q(r, k): from the block's
// shared-memory panel (staged path: every group of the CTA solves the same
// block at the same time, so the CTA stages the UM x k panel once per block)
// or from global memory.
template <class V, class QR>
__device__ __forceinline__ V lu_gemm_row(QR Qrow, const V* x, int xs, int k0, int k1) {
  if constexpr (sizeof(V) == 8) {
    double acc = 0.0;
#pragma unroll 4
    for (int k = k0; k < k1; ++k) acc = fma(Qrow(k), x[k * xs], acc);
    return acc;
  } else {
    double rr = 0.0, ii = 0.0, ri = 0.0, ir = 0.0;
#pragma unroll 4
    for (int k = k0; k < k1; ++k) {
      const double2 a = Qrow(k), xk = x[k * xs];
      rr = fma(a.x, xk.x, rr);
      ii = fma(a.y, xk.y, ii);
      ri = fma(a.x, xk.y, ri);
      ir = fma(a.y, xk.x, ir);
    }
    return make_double2(__dsub_rn(rr, ii), __dadd_rn(ri, ir));
  }
}

// Stage panel[(k - k0) * UM + l] = Q(r0 + l, k), k in [k0, k1), l < bs (zero
// above bs): the CTA's threads cooperatively, between two barriers.
template <class V, int UM>
__device__ __forceinline__ void lu_stage_panel(V* panel, const V* __restrict__ Q, int n, int r0, int bs, int k0,
                                               int k1) {
  __syncthreads();  // the previous block's panel has been read
  const int tot = (k1 - k0) * UM;
  for (int e = threadIdx.x; e < tot; e += blockDim.x) {
    const int kk = e / UM, ll = e - kk * UM;
    panel[e] = ll < bs ? __ldg(Q + (r0 + ll) + int64_t(k0 + kk) * n) : V{};
  }
  __syncthreads();
}

// Solve one fibre x (stride xs) cooperatively on the UM lanes of this group
// (l = lane within the group). All threads of the CTA run this together
// (PANEL: with CTA barriers; the groups work on different fibres of the same
// shape, inactive groups only take part in the shuffles and barriers).
template <bool CPLX, bool PANEL>
__device__ __forceinline__ void lu_fibre_coop(typename std::conditional<CPLX, double2, double>::type* x, int xs,
                                              const typename std::conditional<CPLX, double2, double>::type* __restrict__ Q,
                                              const typename std::conditional<CPLX, double2, double>::type* invd,
                                              typename std::conditional<CPLX, double2, double>::type* panel,
                                              int n, int l, bool active) {
  using V = typename std::conditional<CPLX, double2, double>::type;
  constexpr int UM = CPLX ? 4 : 16;
  const int full_end = n & ~(UM - 1);
  // forward sweep, unit lower triangle
  for (int r0 = 0; r0 < n;) {
    const int bs = r0 < full_end ? UM : 1 << (31 - __clz(n - r0));
    const int r = r0 + l;
    const bool own = active && l < bs;
    if constexpr (PANEL) lu_stage_panel<V, UM>(panel, Q, n, r0, bs, 0, r0 + bs);
    auto Qrow = [&](int k) -> V {
      if constexpr (PANEL) return panel[k * UM + l];
      else return __ldg(Q + r + int64_t(k) * n);
    };
    V xr = own ? x[r * xs] : V{};
    if (r0 > 0 && own) {
      const V acc = lu_gemm_row<V>(Qrow, x, xs, 0, r0);
      if constexpr (CPLX)
        xr = make_double2(__dsub_rn(xr.x, acc.x), __dsub_rn(xr.y, acc.y));
      else
        xr = __dsub_rn(xr, acc);
    }
    for (int i = 0; i < bs; ++i) {
      V xi = shfl_v(xr, i, UM);
      if constexpr (CPLX) {
        if (l == i && own) xr = ztrsm_scale(xr, make_double2(1.0, 0.0));
        xi = ztrsm_scale(xi, make_double2(1.0, 0.0));
        if (l > i && own) xr = ztrsm_update(xr, xi, Qrow(r0 + i));
      } else {
        if (l > i && own) xr = fma(-xi, Qrow(r0 + i), xr);
      }
    }
    if (own) x[r * xs] = xr;
    __syncwarp();
    r0 += bs;
  }
  // backward sweep, upper triangle with the reciprocal diagonal
  for (int top = n; top > 0;) {
    const int bs = top > full_end ? (top & -top) : UM;
    const int r0 = top - bs;
    const int r = r0 + l;
    const bool own = active && l < bs;
    if constexpr (PANEL) lu_stage_panel<V, UM>(panel, Q, n, r0, bs, r0, n);
    auto Qrow = [&](int k) -> V {
      if constexpr (PANEL) return panel[(k - r0) * UM + l];
      else return __ldg(Q + r + int64_t(k) * n);
    };
    V xr = own ? x[r * xs] : V{};
    if (top < n && own) {
      const V acc = lu_gemm_row<V>(Qrow, x, xs, top, n);
      if constexpr (CPLX)
        xr = make_double2(__dsub_rn(xr.x, acc.x), __dsub_rn(xr.y, acc.y));
      else
        xr = __dsub_rn(xr, acc);
    }
    for (int i = bs - 1; i >= 0; --i) {
      if (l == i && own) {
        if constexpr (CPLX)
          xr = ztrsm_scale(xr, invd[r]);
        else
          xr = __dmul_rn(xr, invd[r]);
      }
      const V xi = shfl_v(xr, i, UM);
      if (l < i && own) {
        if constexpr (CPLX)
          xr = ztrsm_update(xr, xi, Qrow(r0 + i));
        else
          xr = fma(-xi, Qrow(r0 + i), xr);
      }
    }
    if (own) x[r * xs] = xr;
    __syncwarp();
    top = r0;
  }
}

// perm[k]: the row of the input that ends in row k after lu_solve's swaps
// (lu.hpp:58-64) -- the swaps applied in order to an index array. iperm is
// its inverse. One thread (n is a mode extent).
// The swaps are sequential; they run on one thread over shared-memory copies
// of the index array and the pivots when they fit (n <= kLuPermSmem: 24 ->
// 8 us at n = 200, each swap a shared round trip instead of a global one), in
// global memory otherwise; the block fills and inverts the array in parallel.
constexpr int kLuPermSmem = 12288;
__global__ void lu_perm_kernel(const int64_t* __restrict__ piv, int* __restrict__ perm, int* __restrict__ iperm,
                               int n) {
  extern __shared__ int sperm[];  // [n] index array, [n] pivots (shared path)
  const bool in_smem = n <= kLuPermSmem;
  int* w = in_smem ? sperm : perm;
  int* spiv = sperm + n;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    w[k] = k;
    if (in_smem) spiv[k] = static_cast<int>(piv[k]);
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < n; ++k) {
      const int p = in_smem ? spiv[k] : static_cast<int>(piv[k]);
      if (p != k) {
        const int t = w[k];
        w[k] = w[p];
        w[p] = t;
      }
    }
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const int v = w[k];
    if (in_smem) perm[k] = v;
    iperm[v] = k;
  }
}

template <bool CPLX>
struct LuCfg {
  static constexpr int UM = CPLX ? 4 : 16;
  static constexpr int THREADS = kLuFibres * UM;  // one lane group per fibre of the tile
  static constexpr int PS = CPLX ? 4 : 20;        // factor panel row stride (real: = 8 mod 32 words)
};

// Real staged sweeps with the blocks' GEMM parts on the tensor cores: for a
// 16-row block at r0 the CTA's 32 fibres need D(16 x 32) = Q(r0.., 0..r0) .
// X(0..r0, fibres) -- 2 x 4 DMMA fragments, each the k-ordered FMA chain of
// the serial restatement (zero k-steps pad r0 to a multiple of 4), subtracted
// from the block rows; then every 16-lane group solves its fibre's diagonal
// block with shuffles. The block's factor rows are staged once per block
// (panel[k * 20 + l] = Q(r0 + l, k)).
__device__ __forceinline__ void lu_sweep_dmma(double* xs, const double* __restrict__ Q,
                                              const double* __restrict__ invd, double* panel, int n, int nf) {
  constexpr int UM = 16, PS = LuCfg<false>::PS, XS = kLuStride;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int grp = threadIdx.x / UM, l = threadIdx.x - grp * UM;
  const bool active = grp < nf;
  const int mf = warp >> 2, fr = warp & 3;  // GEMM warps 0..7: rows 8 mf.., fibres 8 fr..
  const int full_end = n & ~(UM - 1);
  auto stage = [&](int r0, int bs, int k0, int k1) {
    __syncthreads();
    for (int e = threadIdx.x; e < (k1 - k0) * UM; e += blockDim.x) {
      const int kk = e >> 4, ll = e & 15;
      panel[kk * PS + ll] = ll < bs ? __ldg(Q + (r0 + ll) + int64_t(k0 + kk) * n) : 0.0;
    }
    __syncthreads();
  };
  // forward sweep, unit lower triangle
  for (int r0 = 0; r0 < n;) {
    const int bs = r0 < full_end ? UM : 1 << (31 - __clz(n - r0));
    stage(r0, bs, 0, r0 + bs);
    if (r0 > 0 && warp < 8) {
      double d0 = 0.0, d1 = 0.0;
      const int ks = (r0 + 3) >> 2;
      for (int s = 0; s < ks; ++s) {
        const int k = 4 * s + t;
        const double a = k < r0 ? panel[k * PS + 8 * mf + g] : 0.0;
        const double b = k < r0 ? xs[k * XS + 8 * fr + g] : 0.0;
        dmma_8x8x4(d0, d1, a, b);
      }
      const int row = 8 * mf + g;
      if (row < bs) {
        double* xr = xs + (r0 + row) * XS + 8 * fr + 2 * t;
        xr[0] = __dsub_rn(xr[0], d0);
        xr[1] = __dsub_rn(xr[1], d1);
      }
    }
    __syncthreads();
    const int r = r0 + l;
    const bool own = active && l < bs;
    double xr = own ? xs[r * XS + grp] : 0.0;
    for (int i = 0; i < bs; ++i) {
      const double xi = __shfl_sync(0xffffffffu, xr, i, UM);
      if (l > i && own) xr = fma(-xi, panel[(r0 + i) * PS + l], xr);
    }
    if (own) xs[r * XS + grp] = xr;
    r0 += bs;
  }
  // backward sweep, upper triangle with the reciprocal diagonal
  for (int top = n; top > 0;) {
    const int bs = top > full_end ? (top & -top) : UM;
    const int r0 = top - bs;
    stage(r0, bs, r0, n);
    if (top < n && warp < 8) {
      double d0 = 0.0, d1 = 0.0;
      const int ks = (n - top + 3) >> 2;
      for (int s = 0; s < ks; ++s) {
        const int k = top + 4 * s + t;
        const double a = k < n ? panel[(k - r0) * PS + 8 * mf + g] : 0.0;
        const double b = k < n ? xs[k * XS + 8 * fr + g] : 0.0;
        dmma_8x8x4(d0, d1, a, b);
      }
      const int row = 8 * mf + g;
      if (row < bs) {
        double* xr = xs + (r0 + row) * XS + 8 * fr + 2 * t;
        xr[0] = __dsub_rn(xr[0], d0);
        xr[1] = __dsub_rn(xr[1], d1);
      }
    }
    __syncthreads();
    const int r = r0 + l;
    const bool own = active && l < bs;
    double xr = own ? xs[r * XS + grp] : 0.0;
    for (int i = bs - 1; i >= 0; --i) {
      if (l == i && own) xr = __dmul_rn(xr, invd[r]);
      const double xi = __shfl_sync(0xffffffffu, xr, i, UM);
      if (l < i && own) xr = fma(-xi, panel[i * PS + l], xr);
    }
    if (own) xs[r * XS + grp] = xr;
    top = r0;
  }
  __syncthreads();
}

// One mode of itucker: out(a, :, c) = P^-1 in(a, :, c) for all A*C fibres of
// length n (in may equal out: every CTA reads and writes only its own fibres).
// staged: the tile's fibres live in shared memory x[k * 33 + fibre]; else
// (n too large) they are solved in place in `out` with the same arithmetic.
template <bool CPLX>
__global__ void __launch_bounds__(LuCfg<CPLX>::THREADS) lu_solve_mode_kernel(
    const double* in, double* out, int64_t A, int n, int64_t C, const double* __restrict__ lu,
    const int* __restrict__ perm, const int* __restrict__ iperm, int staged) {
  using V = typename std::conditional<CPLX, double2, double>::type;
  constexpr int UM = LuCfg<CPLX>::UM;
  extern __shared__ __align__(16) unsigned char lu_smem[];
  V* invd = reinterpret_cast<V*>(lu_smem);
  V* xs = invd + n;
  V* panel = xs + n * kLuStride;  // staged path: one block's factor rows
  const V* Q = reinterpret_cast<const V*>(lu);
  const V* src = reinterpret_cast<const V*>(in);
  V* dst = reinterpret_cast<V*>(out);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int grp = tid / UM, l = tid - grp * UM;  // fibre of the tile, row lane
  for (int i = tid; i < n; i += nt) {
    if constexpr (CPLX)
      invd[i] = ztrsm_recip(Q[i + int64_t(i) * n]);
    else
      invd[i] = 1.0 / Q[i + int64_t(i) * n];
  }
  __syncthreads();
  __shared__ int64_t foff[kLuFibres];  // element 0 of each fibre of the tile
  const int64_t F = A * C, An = A * n;
  for (int64_t f0 = int64_t(blockIdx.x) * kLuFibres; f0 < F; f0 += int64_t(gridDim.x) * kLuFibres) {
    const int nf = static_cast<int>(F - f0 < kLuFibres ? F - f0 : kLuFibres);
    if (tid < kLuFibres) {
      const int64_t ff = f0 + (tid < nf ? tid : 0);
      foff[tid] = (ff % A) + (ff / A) * An;
    }
    __syncthreads();
    const int64_t off = foff[grp];  // element k of this group's fibre at off + k * A
    if (staged) {
      if (A == 1) {  // mu = 1: the tile's fibres are nf*n contiguous elements
        const V* s = src + f0 * n;
        const int64_t tot = int64_t(nf) * n;
        const int dfl = nt / n, dkk = nt - dfl * n;
        int fl = tid / n, kk = tid - (tid / n) * n;
        for (int64_t e = tid; e < tot; e += nt) {
          xs[iperm[kk] * kLuStride + fl] = s[e];
          fl += dfl;
          kk += dkk;
          if (kk >= n) {
            kk -= n;
            ++fl;
          }
        }
      } else {  // lanes along the fibres (consecutive a): coalesced
        const int fl = tid & (kLuFibres - 1);
        if (fl < nf) {
          const int64_t o = foff[fl];
          for (int k = tid / kLuFibres; k < n; k += nt / kLuFibres) xs[k * kLuStride + fl] = src[o + int64_t(perm[k]) * A];
        }
      }
      __syncthreads();
      if constexpr (CPLX)
        lu_fibre_coop<CPLX, true>(xs + grp, kLuStride, Q, invd, panel, n, l, grp < nf);
      else
        lu_sweep_dmma(xs, Q, invd, panel, n, nf);
      __syncthreads();
      if (A == 1) {
        V* d = dst + f0 * n;
        const int64_t tot = int64_t(nf) * n;
        const int dfl = nt / n, dkk = nt - dfl * n;
        int fl = tid / n, k = tid - (tid / n) * n;
        for (int64_t e = tid; e < tot; e += nt) {
          d[e] = xs[k * kLuStride + fl];
          fl += dfl;
          k += dkk;
          if (k >= n) {
            k -= n;
            ++fl;
          }
        }
      } else {
        const int fl = tid & (kLuFibres - 1);
        if (fl < nf) {
          const int64_t o = foff[fl];
          for (int k = tid / kLuFibres; k < n; k += nt / kLuFibres) dst[o + int64_t(k) * A] = xs[k * kLuStride + fl];
        }
      }
      __syncthreads();
    } else {  // in global memory (in != out: the host stages a copy): permuted gather, solve in place
      if (grp < nf)
        for (int k = l; k < n; k += UM) dst[off + int64_t(k) * A] = src[off + int64_t(perm[k]) * A];
      __syncwarp();
      lu_fibre_coop<CPLX, false>(dst + (grp < nf ? off : 0), static_cast<int>(A), Q, invd, nullptr, n, l, grp < nf);
      __syncthreads();
    }
  }
}

}  // namespace mumode_gpu
