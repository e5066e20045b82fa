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
// Bitwise equal to the reference for every real extent up to 384 (beyond, the
// library splits each trsm update at GEMM_Q = 384 columns: ~1e-16 apart) and
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
// its inverse. One block per mode (all modes of an itucker in one launch);
// the swaps are sequential: one thread walks them over shared-memory copies
// of the index array and the pivots when they fit (n <= kLuPermSmem: 24 ->
// 8 us at n = 200, each swap a shared round trip instead of a global one), in
// global memory otherwise; the block fills and inverts the array in parallel.
constexpr int kLuPermSmem = 6144;  // 2 n ints <= 48 KB of dynamic shared memory
struct LuPermBatch {
  const int64_t* piv[32];
  int n[32];
  int off[32];  // perm of mode b at base + off[b], iperm at base + off[b] + n[b]
};
__global__ void lu_perm_kernel(const LuPermBatch pb, int* __restrict__ base) {
  extern __shared__ int sperm[];  // [n] index array, [n] pivots (shared path)
  const int n = pb.n[blockIdx.x];
  const int64_t* __restrict__ piv = pb.piv[blockIdx.x];
  int* perm = base + pb.off[blockIdx.x];
  int* iperm = perm + n;
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

// Tile staging: the tile's nf fibres into / out of shared memory as
// xs[k * (NF + 4) + fibre], rows permuted on the way in (x(k) = in(perm[k])).
template <class V, int NF = kLuFibres>
__device__ __forceinline__ void lu_tile_load(V* xs, const V* src, const int64_t* foff, const int* __restrict__ perm,
                                             const int* __restrict__ iperm, int64_t A, int n, int64_t f0, int nf) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (A == 1) {  // mu = 1: the tile's fibres are nf*n contiguous elements
    const V* s = src + f0 * n;
    const int64_t tot = int64_t(nf) * n;
    const int dfl = nt / n, dkk = nt - dfl * n;
    int fl = tid / n, kk = tid - (tid / n) * n;
    for (int64_t e = tid; e < tot; e += nt) {
      xs[iperm[kk] * (NF + 4) + fl] = s[e];
      fl += dfl;
      kk += dkk;
      if (kk >= n) {
        kk -= n;
        ++fl;
      }
    }
  } else {  // lanes along the fibres (consecutive a): coalesced
    const int fl = tid % NF;
    if (fl < nf) {
      const int64_t o = foff[fl];
      for (int k = tid / NF; k < n; k += nt / NF) xs[k * (NF + 4) + fl] = src[o + int64_t(perm[k]) * A];
    }
  }
}
template <class V, int NF = kLuFibres>
__device__ __forceinline__ void lu_tile_store(const V* xs, V* dst, const int64_t* foff, int64_t A, int n, int64_t f0,
                                              int nf) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (A == 1) {
    V* d = dst + f0 * n;
    const int64_t tot = int64_t(nf) * n;
    const int dfl = nt / n, dkk = nt - dfl * n;
    int fl = tid / n, k = tid - (tid / n) * n;
    for (int64_t e = tid; e < tot; e += nt) {
      d[e] = xs[k * (NF + 4) + fl];
      fl += dfl;
      k += dkk;
      if (k >= n) {
        k -= n;
        ++fl;
      }
    }
  } else {
    const int fl = tid % NF;
    if (fl < nf) {
      const int64_t o = foff[fl];
      for (int k = tid / NF; k < n; k += nt / NF) dst[o + int64_t(k) * A] = xs[k * (NF + 4) + fl];
    }
  }
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
      lu_tile_load<V>(xs, src, foff, perm, iperm, A, n, f0, nf);
      __syncthreads();
      if constexpr (CPLX)
        lu_fibre_coop<CPLX, true>(xs + grp, kLuStride, Q, invd, panel, n, l, grp < nf);
      else
        lu_sweep_dmma(xs, Q, invd, panel, n, nf);
      __syncthreads();
      lu_tile_store<V>(xs, dst, foff, A, n, f0, nf);
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

// ---------------------------------------------------------------------------
// Real staged sweeps, second form (n <= kLuRlMaxN): the same arithmetic with
// the dependent work taken off the critical path.
//
//  * Forward sweep RIGHT-LOOKING: row r's GEMM chain is acc = sum over
//    k = 0..r0-1 ascending, and the blocks are solved in ascending order, so
//    the chain can be fed block by block as the x_k become known: after block
//    j is solved, every row below it takes the 16 k's of block j (4 DMMAs per
//    8 x 8 fragment) into an accumulator that stays in registers (the warp's
//    row fragments mq + RG i of its 8 fibres, indexed from the bottom so the
//    live ones are a prefix). Each element sees exactly the FMA sequence of
//    the left-looking form (zero k-steps are exact no-ops), so the result is
//    bit for bit the same -- but the per-block critical path is the in-block
//    solve plus 4 DMMAs instead of a chain over all solved rows, and the
//    update is many independent chains on every warp. A dependent DMMA issues
//    ~90 cycles after its predecessor (measured with clock64 per phase), so
//    the fragments advance together k-step by k-step; and a predicated-off
//    DMMA still takes its slot in the fp64 pipe (ncu: 38 % pipe-active for
//    22 % of useful DMMAs), so the unrolled loops leave by uniform branches.
//  * Backward sweep left-looking as before (a row's chain starts with the x's
//    of the block solved just before it, so it cannot start earlier): one
//    chain per warp, ~90 cycles per k-step of 4.
//  * Diagonal blocks: four lanes per fibre (lu_*_diag_quad), ~80 cycles per
//    row instead of 16 warps of shuffle steps.
//  * Both sweeps: the next block's factor panel (forward: the 16 columns of
//    block j below its diagonal; backward: the block's 16 rows right of the
//    diagonal) arrives in the other of two buffers while the current block is
//    worked on -- by 8-byte cp.async issued under the DMMA phases, or (BULK:
//    even n > 128, 64- / 32-fibre tiles) by one bulk copy per column / row completing on an
//    mbarrier, the backward rows read from a transposed copy of the factor.
//  * NF = 64 or 96 fibres per CTA (16 / 24 warps, one CTA per SM from n = 129):
//    every phase is latency-bound, so throughput is fibres in flight per SM;
//    the host picks 96 when it saves enough waves (a 96-fibre tile takes
//    ~1.4x a 64-fibre tile's time).
// Panel buffers: 16 x PST doubles, PST >= roundup8(n), = 4 mod 8 (conflict-free A
// fragments); forward pan[kk * PST + (row - r0)], backward
// pan[l * PST + (k - r0)].
// Measured (tools/itucker_time.py, n^3, L2 flushed): 128: 0.330 -> 0.236 ms,
// 200: 1.35 -> 0.96, 256: 4.04 -> 2.02, 300: 7.74 -> 4.76, 400: 19.9 -> 11.5.
constexpr int kLuRlMaxN = 408;

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void lu_bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Qt(k, r) = Q(r, k): the backward panels' rows become contiguous (bulk copies)
__global__ void lu_transpose_kernel(const double* __restrict__ Q, double* __restrict__ Qt, int n) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y)
    if (bx + threadIdx.x < n && by + j < n) tile[j][threadIdx.x] = Q[(bx + threadIdx.x) + int64_t(by + j) * n];
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y)
    if (by + threadIdx.x < n && bx + j < n) Qt[(by + threadIdx.x) + int64_t(bx + j) * n] = tile[threadIdx.x][j];
}
__device__ __forceinline__ void cp_async_commit_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// >= the rows of the last 8-row fragment (its rows beyond n are read, never used), = 4 mod 8 doubles
__host__ __device__ inline int lu_rl_pst(int n) { return ((n + 7) & ~7) + 4; }

// Diagonal-block solves of the remainder blocks (8 / 4 / 2 / 1 rows), one lane
// per fibre (x = the fibre's BS block rows, stride XS = NF + 4): the same
// per-element update order as trsm's in-block solve (row l takes the finished
// x_i in ascending / descending i). Full 16-row blocks take the quad form below.
template <int BS, int XS>
__device__ __forceinline__ void lu_fwd_diag(double* x, const double* pj, int PST) {
  double v[BS];
#pragma unroll
  for (int l = 0; l < BS; ++l) v[l] = x[l * XS];
#pragma unroll
  for (int i = 0; i + 1 < BS; ++i)
#pragma unroll
    for (int l = i + 1; l < BS; ++l) v[l] = fma(-v[i], pj[i * PST + l], v[l]);
#pragma unroll
  for (int l = 1; l < BS; ++l) x[l * XS] = v[l];
}
template <int BS, int XS>
__device__ __forceinline__ void lu_bwd_diag(double* x, const double* pj, int PST, const double* invd) {
  double v[BS];
#pragma unroll
  for (int l = 0; l < BS; ++l) v[l] = x[l * XS];
#pragma unroll
  for (int i = BS - 1; i >= 0; --i) {
    v[i] = __dmul_rn(v[i], invd[i]);
#pragma unroll
    for (int l = 0; l < i; ++l) v[l] = fma(-v[i], pj[l * PST + i], v[l]);
  }
#pragma unroll
  for (int l = 0; l < BS; ++l) x[l * XS] = v[l];
}

// Full 16-row diagonal blocks: four lanes per fibre (warps 0..3, eight fibres
// each), lane q owning rows q, q + 4, q + 8, q + 12. Step i broadcasts the
// finished x_i inside the quad and every lane updates its rows beyond i -- the
// same per-row update order again; the factor loads do not depend on the
// chain, so a step costs one shuffle plus one FMA of latency (the one-lane
// form pays a shared-memory load per FMA, the 16-lane form 16 warps of
// instructions per step).
template <int XS>
__device__ __forceinline__ void lu_fwd_diag_quad(double* xs, const double* pj, int PST, int r0, int warp, int lane) {
  const int q = lane & 3, f = 8 * warp + (lane >> 2);
  double* x = xs + (r0 + q) * XS + f;
  const double* pq = pj + q;
  double v[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) v[m] = x[4 * m * XS];
#pragma unroll
  for (int i = 0; i < 15; ++i) {
    const int qi = i & 3, mi = i >> 2;
    const double xi = __shfl_sync(0xffffffffu, v[mi], qi, 4);
#pragma unroll
    for (int m = mi; m < 4; ++m) {
      const double u = fma(-xi, pq[i * PST + 4 * m], v[m]);
      v[m] = (m > mi || q > qi) ? u : v[m];
    }
  }
#pragma unroll
  for (int m = 0; m < 4; ++m) x[4 * m * XS] = v[m];
}
template <int XS>
__device__ __forceinline__ void lu_bwd_diag_quad(double* xs, const double* pj, int PST, const double* invd, int r0,
                                                 int warp, int lane) {
  const int q = lane & 3, f = 8 * warp + (lane >> 2);
  double* x = xs + (r0 + q) * XS + f;
  const double* pq = pj + q * PST;
  double v[4], dinv[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    v[m] = x[4 * m * XS];
    dinv[m] = invd[r0 + q + 4 * m];
  }
#pragma unroll
  for (int i = 15; i >= 0; --i) {
    const int qi = i & 3, mi = i >> 2;
    v[mi] = q == qi ? __dmul_rn(v[mi], dinv[mi]) : v[mi];
    const double xi = __shfl_sync(0xffffffffu, v[mi], qi, 4);
#pragma unroll
    for (int m = 0; m <= mi; ++m) {
      const double u = fma(-xi, pq[4 * m * PST + i], v[m]);
      v[m] = (m < mi || q < qi) ? u : v[m];
    }
  }
#pragma unroll
  for (int m = 0; m < 4; ++m) x[4 * m * XS] = v[m];
}

template <int NF, int NW, int MAXI, bool BULK>
__device__ __forceinline__ void lu_sweep_rl(double* xs, const double* __restrict__ Q, const double* __restrict__ Qt,
                                            const double* __restrict__ invd, double* pan, int n, uint64_t* pbar,
                                            uint32_t& st) {
  constexpr int UM = 16, XS = NF + 4, FRW = NF / 8, RG = NW / FRW;  // fibre fragments, row groups of the warps
  const int PST = lu_rl_pst(n), PSZ = 16 * PST;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int mq = warp / FRW, fr = warp % FRW;
  const int full_end = n & ~(UM - 1);
  auto fwd_bs = [&](int r0) { return r0 < full_end ? UM : 1 << (31 - __clz(n - r0)); };
  auto bwd_bs = [&](int top) { return top > full_end ? (top & -top) : UM; };
  // forward panel of the block at r0: Q(r0.., r0 + kk), kk < bs -- warp kk copies column kk
  constexpr int CW = NW;  // every warp copies its share of the next panel at the start of the DMMA phases
  const int cw = warp;
  // BULK (even n, Qt given): panels by bulk copies, one per column (forward) / row (backward, from the
  // transposed factor), issued by the last warp and completing on the buffer's mbarrier; the
  // step counter st picks the buffer (st & 1) and its phase parity ((st >> 1) & 1). Otherwise:
  // 8-byte cp.async by every warp at the start of the DMMA phases.
  constexpr bool bulk = BULK;
  auto issue_bulk = [&](int b, const double* src, int bs, int len) {  // bs pieces of len doubles, source pitch n
    if (warp == NW - 1) {
      if (lane == 0) mbar_arrive_expect_tx(pbar + b, uint32_t(bs) * uint32_t(len) * 8u);
      __syncwarp();
      if (lane < bs) lu_bulk_load(pan + b * PSZ + lane * PST, src + int64_t(lane) * n, uint32_t(len) * 8u, pbar + b);
    }
  };
  auto panel_wait = [&]() {
    if (bulk) mbar_wait(pbar + (st & 1), (st >> 1) & 1);
    else cp_async_commit_wait_all();
  };
  auto issue_fwd = [&](double* pb, int r0, int bs) {
    for (int kk = cw; kk < bs; kk += CW) {
      const double* q = Q + r0 + int64_t(r0 + kk) * n;
      double* d = pb + kk * PST;
      for (int rr = lane; rr < n - r0; rr += 32) cp_async8(d + rr, q + rr);
    }
  };
  // backward panel of the block at r0: Q(r0 + ll, r0..n-1), ll < bs
  auto issue_bwd = [&](double* pb, int r0, int bs) {
    const int ll = lane & 15;
    if (ll < bs) {
      const double* q = Q + (r0 + ll) + int64_t(r0) * n;
      double* d = pb + ll * PST;
      for (int kk = 2 * cw + (lane >> 4); kk < n - r0; kk += 2 * CW) cp_async8(d + kk, q + int64_t(kk) * n);
    }
  };

  const int ihi = (n - 8 * mq + 8 * RG - 1) / (8 * RG);  // this warp's row fragments: mq + RG i, i < ihi
  double acc[MAXI][2];  // acc[ip]: fragment i = ihi - 1 - ip (indexed from the bottom, see the update)
#pragma unroll
  for (int i = 0; i < MAXI; ++i) acc[i][0] = acc[i][1] = 0.0;
  int buf = st & 1;
  if (bulk) issue_bulk(buf, Q, fwd_bs(0), n);
  else issue_fwd(pan + buf * PSZ, 0, fwd_bs(0));
  // forward sweep, unit lower triangle
  for (int r0 = 0; r0 < n;) {
    const int bs = fwd_bs(r0), rn = r0 + bs;
    double* pj = pan + buf * PSZ;
    if (r0 > 0) {
      // a block spans at most two row fragments, owned by different row groups: the warp's only
      // candidate is its topmost fragment with rows >= r0
      const int il = (r0 - 8 - 8 * mq + 8 * RG) / (8 * RG), ipf = ihi - 1 - il;
      const int row = 8 * (mq + RG * il) + g;
      if (ipf >= 0 && row >= r0 && row < rn) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int ip = 0; ip < MAXI; ++ip) {
          a0 = ip == ipf ? acc[ip][0] : a0;
          a1 = ip == ipf ? acc[ip][1] : a1;
        }
        double* xr = xs + row * XS + 8 * fr + 2 * t;
        xr[0] = __dsub_rn(xr[0], a0);
        xr[1] = __dsub_rn(xr[1], a1);
      }
    }
    panel_wait();
    __syncthreads();  // panel j and the flushed rows are visible; the other buffer is free
    if (bulk) {
      if (rn < n) issue_bulk(buf ^ 1, Q + rn + int64_t(rn) * n, fwd_bs(rn), n - rn);
      else issue_bulk(buf ^ 1, Qt + (n - bwd_bs(n)) + int64_t(n - bwd_bs(n)) * n, bwd_bs(n), bwd_bs(n));
    }
    if (bs == UM) {
      if (warp < FRW) lu_fwd_diag_quad<XS>(xs, pj, PST, r0, warp, lane);
    } else if (32 * warp + lane < NF) {  // remainder blocks: one lane per fibre
      double* x = xs + r0 * XS + 32 * warp + lane;
      switch (bs) {
        case 8: lu_fwd_diag<8, XS>(x, pj, PST); break;
        case 4: lu_fwd_diag<4, XS>(x, pj, PST); break;
        case 2: lu_fwd_diag<2, XS>(x, pj, PST); break;
        default: break;
      }
    }
    __syncthreads();
    // cp.async panels: the next one (its buffer was last read before the barrier above), under the DMMA phase
    if (!bulk) {
      if (rn < n) issue_fwd(pan + (buf ^ 1) * PSZ, rn, fwd_bs(rn));
      else issue_bwd(pan + (buf ^ 1) * PSZ, n - bwd_bs(n), bwd_bs(n));
    }
    if (rn < n) {
      if (bs == UM) {  // full block: fragments are entirely above or below it, no k padding
        double b[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) b[s] = xs[(r0 + 4 * s + t) * XS + 8 * fr + g];
        // k-step outer, fragments inner: a DMMA's result is ~90 cycles away, so the warp's
        // fragments advance together as independent chains (rows >= n of the last fragment are
        // never flushed; a fragment above the block only accumulates into dead registers)
        // The accumulators are indexed from the bottom (acc[ip]: the warp's ip-th fragment from
        // the last one), so the live ones are ip < cnt and the unrolled loops leave by a uniform
        // branch -- a predicated-off DMMA still takes its slot in the fp64 pipe.
        const int cnt = ihi - (rn - 8 * mq + 8 * RG - 1) / (8 * RG);
        const double* pa = pj + (8 * (mq + RG * (ihi - 1)) + g - r0) + t * PST;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          constexpr int CH = 4;  // A fragments loaded CH at a time (registers)
#pragma unroll
          for (int c = 0; c < MAXI; c += CH) {
            if (c >= cnt) break;
            double a[CH];
#pragma unroll
            for (int u = 0; u < CH; ++u)
              if (c + u < MAXI && c + u < cnt) a[u] = pa[-8 * RG * (c + u) + 4 * s * PST];
#pragma unroll
            for (int u = 0; u < CH; ++u) {
              if (c + u >= MAXI || c + u >= cnt) break;
              dmma_8x8x4(acc[c + u][0], acc[c + u][1], a[u], b[s]);
            }
          }
        }
      } else {
        const int ks = (bs + 3) >> 2;
        double b[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const int k = 4 * s + t;
          b[s] = (s < ks && k < bs) ? xs[(r0 + k) * XS + 8 * fr + g] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < MAXI; ++i) {
          const int rb = 8 * (mq + RG * (ihi - 1 - i));
          if (i < ihi && rb + 8 > rn) {  // the fragment has rows below block j
            const int row = rb + g;
            const bool rv = row >= rn && row < n;
            const double* pa = pj + (row - r0);
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              if (s < ks) {
                const int k = 4 * s + t;
                const double a = (rv && k < bs) ? pa[k * PST] : 0.0;
                dmma_8x8x4(acc[i][0], acc[i][1], a, b[s]);
              }
            }
          }
        }
      }
    }
    r0 = rn;
    buf ^= 1;
    ++st;
  }
  // backward sweep, upper triangle with the reciprocal diagonal
  for (int top = n; top > 0;) {
    const int bs = bwd_bs(top), r0 = top - bs;
    double* pj = pan + buf * PSZ;
    panel_wait();
    __syncthreads();  // panel j and the previous block's x are visible; the other buffer is free
    if (r0 > 0) {
      const int nb = bwd_bs(r0), nr = r0 - nb;
      if (bulk) issue_bulk(buf ^ 1, Qt + nr + int64_t(nr) * n, nb, n - nr);
      else issue_bwd(pan + (buf ^ 1) * PSZ, nr, nb);
    }
    if (top < n && mq < 2) {
      double d0 = 0.0, d1 = 0.0;
      const int ks = (n - top + 3) >> 2;
      const double* pa = pj + (8 * mq + g) * PST + (top - r0) + t;
      const double* pb = xs + (top + t) * XS + 8 * fr + g;
      int s = 0;
      for (; s + 4 <= ks - 1; s += 4) {  // full k-steps, four loads ahead of the chain
        double a4[4], b4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a4[u] = pa[4 * (s + u)];
          b4[u] = pb[4 * (s + u) * XS];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma_8x8x4(d0, d1, a4[u], b4[u]);
      }
      for (; s < ks; ++s) {
        const bool kv = top + 4 * s + t < n;
        const double a = kv ? pa[4 * s] : 0.0;
        const double b = kv ? pb[4 * s * XS] : 0.0;
        dmma_8x8x4(d0, d1, a, b);
      }
      const int row = 8 * mq + g;
      if (row < bs) {
        double* xr = xs + (r0 + row) * XS + 8 * fr + 2 * t;
        xr[0] = __dsub_rn(xr[0], d0);
        xr[1] = __dsub_rn(xr[1], d1);
      }
    }
    __syncthreads();
    if (bs == UM) {
      if (warp < FRW) lu_bwd_diag_quad<XS>(xs, pj, PST, invd, r0, warp, lane);
    } else if (32 * warp + lane < NF) {  // remainder blocks: one lane per fibre
      double* x = xs + r0 * XS + 32 * warp + lane;
      switch (bs) {
        case 8: lu_bwd_diag<8, XS>(x, pj, PST, invd + r0); break;
        case 4: lu_bwd_diag<4, XS>(x, pj, PST, invd + r0); break;
        case 2: lu_bwd_diag<2, XS>(x, pj, PST, invd + r0); break;
        default: lu_bwd_diag<1, XS>(x, pj, PST, invd + r0); break;
      }
    }
    top = r0;
    buf ^= 1;
    ++st;
  }
  __syncthreads();
}

// One real mode of itucker through lu_sweep_rl (staged tiles, n <= kLuRlMaxN).
// Shared memory: invd[n], xs[n * (NF + 4)], two panel buffers of 16 * PST. NF fibres per CTA on NW warps (NW / (NF / 8)
// row groups): 64 on 16 (or 96 on 24 up to n = 208) while the tile fits, 48 on 12 up to 328, else 32 on 16 -- the host
// chooses (itucker_dev); BULK: panels by bulk copies, lut = the transposed factor.
template <int NF, int NW, int MAXI, int MINB, bool BULK>
__global__ void __launch_bounds__(32 * NW, MINB) lu_solve_rl_kernel(
    const double* in, double* out, int64_t A, int n, int64_t C, const double* __restrict__ lu,
    const double* __restrict__ lut, const int* __restrict__ perm, const int* __restrict__ iperm) {
  extern __shared__ __align__(16) unsigned char lu_smem[];
  double* invd = reinterpret_cast<double*>(lu_smem);
  double* xs = invd + n;
  double* pan = xs + (n + (n & 1)) * (NF + 4);  // 16-byte aligned for the bulk copies
  __shared__ __align__(8) uint64_t pbar[2];
  if (threadIdx.x == 0) {
    mbar_init(pbar, 1);
    mbar_init(pbar + 1, 1);
    fence_barrier_init();
  }
  uint32_t st = 0;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < n; i += nt) invd[i] = 1.0 / lu[i + int64_t(i) * n];
  __shared__ int64_t foff[NF];
  const int64_t F = A * C, An = A * n;
  for (int64_t f0 = int64_t(blockIdx.x) * NF; f0 < F; f0 += int64_t(gridDim.x) * NF) {
    const int nf = static_cast<int>(F - f0 < NF ? F - f0 : NF);
    if (tid < NF) {
      const int64_t ff = f0 + (tid < nf ? tid : 0);
      foff[tid] = (ff % A) + (ff / A) * An;
    }
    __syncthreads();
    lu_tile_load<double, NF>(xs, in, foff, perm, iperm, A, n, f0, nf);
    __syncthreads();
    lu_sweep_rl<NF, NW, MAXI, BULK>(xs, lu, lut, invd, pan, n, pbar, st);
    lu_tile_store<double, NF>(xs, out, foff, A, n, f0, nf);
    __syncthreads();
  }
}

inline size_t lu_rl_smem(int n, int nf) {
  return sizeof(double) * (size_t(n) + size_t(n + (n & 1)) * (nf + 4) + 2 * 16 * size_t(lu_rl_pst(n)));
}

}  // namespace mumode_gpu
