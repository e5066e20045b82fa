// Real fp64 mu-mode product for shapes the TMA path cannot describe (TMA
// needs 16-byte-multiple strides and bases; an odd leading extent gives
// 8-byte ones). Same contraction, fragment maps and DMMA loop as
// tma_dmma.cuh, but operands travel global -> registers -> shared memory with
// plain coalesced 8-byte loads, software-swizzled into the XK / KX layouts
// (so fragment reads stay bank-conflict-free), double-buffered: the loads
// for k-block kb+1 are in flight while k-block kb computes. The epilogue uses
// 8-byte stores (no alignment assumptions). Not persistent: one CTA per tile,
// several CTAs per SM.
#pragma once
#include "common.cuh"

namespace mumode_gpu {

struct LdgArgs {
  const double* T;
  const double* L;
  double* S;
  int64_t A, K, N, C;  // job: S(a, i, c) = sum_k op(L)(i, k) T(a, k, c), i < N
  int64_t sLi, sLk;    // op(L)(i, k) = L[i*sLi + k*sLk]
  int64_t Mlim;        // valid rows: N (mode 1) or A
  int64_t ntot;        // valid columns: C (mode 1) or N
  int AB;              // M fragments per batch (mu > 1)
  int64_t mfrags;
  int mt, nt;
  int accumulate;      // S += result
};

// byte offset inside a 512-B-aligned sub-tile with the 64B swizzle
__device__ __forceinline__ uint32_t sw64(uint32_t a) { return a ^ (((a >> 7) & 3u) << 4); }

template <bool QK, int BM, int BN, int BK, int WM, int WN>
__global__ void __launch_bounds__(WM * WN * 32)
    modeprod_ldg_kernel(const LdgArgs g) {
  constexpr int THREADS = WM * WN * 32;
  constexpr int WTM = BM / WM, WTN = BN / WN, FM = WTM / 8, FN = WTN / 8;
  constexpr int P_EL = BM * BK, Q_EL = BN * BK;
  constexpr int P_PER = P_EL / THREADS, Q_PER = Q_EL / THREADS;
  constexpr int STAGE = (P_EL + Q_EL) * 8;
  static_assert(P_EL % THREADS == 0 && Q_EL % THREADS == 0, "even load split");
  static_assert(BK % 8 == 0, "k blocks of 8");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int mtile, ntile;
  if constexpr (QK) {
    mtile = static_cast<int>(blockIdx.x % g.mt);
    ntile = static_cast<int>(blockIdx.x / g.mt);
  } else {
    ntile = static_cast<int>(blockIdx.x % g.nt);
    mtile = static_cast<int>(blockIdx.x / g.nt);
  }
  const int64_t n0 = int64_t(ntile) * BN;

  // Per-thread P rows (fixed across k-blocks): element e = tid + j*THREADS,
  // r = e % BM (rows fastest: coalesced along a / i), kk = e / BM.
  int64_t p_base[P_PER];
  bool p_ok[P_PER];
#pragma unroll
  for (int j = 0; j < P_PER; ++j) {
    const int e = tid + j * THREADS, r = e % BM;
    const int64_t q = int64_t(mtile) * (BM / 8) + r / 8;
    if constexpr (QK) {
      const int64_t row = 8 * q + (r & 7);
      p_ok[j] = row < g.Mlim;
      p_base[j] = row * g.sLi;
    } else {
      const int64_t c = q / g.AB, a = 8 * (q - c * g.AB) + (r & 7);
      p_ok[j] = q < g.mfrags && a < g.A;
      p_base[j] = a + c * g.A * g.K;
    }
  }
  auto p_addr = [&](int j, int64_t k) -> int64_t {
    return QK ? p_base[j] + k * g.sLk : p_base[j] + k * g.A;
  };
  // Q elements: mode 1 (T, K-contiguous) k fastest; otherwise (L rows) n fastest
  auto q_coord = [&](int j, int& n, int& kk) {
    const int e = tid + j * THREADS;
    if constexpr (QK) {
      kk = e % BK;
      n = e / BK;
    } else {
      n = e % BN;
      kk = e / BN;
    }
  };

  double pr[P_PER], qr[Q_PER];
  const int KT = static_cast<int>((g.K + BK - 1) / BK);
  auto load = [&](int kb) {
    const int64_t k0 = int64_t(kb) * BK;
#pragma unroll
    for (int j = 0; j < P_PER; ++j) {
      const int e = tid + j * THREADS, kk = e / BM;
      const int64_t k = k0 + kk;
      const double* src = QK ? g.L : g.T;
      pr[j] = (p_ok[j] && k < g.K) ? __ldg(src + p_addr(j, k)) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < Q_PER; ++j) {
      int n, kk;
      q_coord(j, n, kk);
      const int64_t k = k0 + kk, nn = n0 + n;
      double v = 0.0;
      if (k < g.K && nn < g.ntot) v = QK ? __ldg(g.T + k + nn * g.K) : __ldg(g.L + nn * g.sLi + k * g.sLk);
      qr[j] = v;
    }
  };
  auto store = [&](int buf) {
    uint8_t* sP = smem + buf * STAGE;
    uint8_t* sQ = sP + P_EL * 8;
#pragma unroll
    for (int j = 0; j < P_PER; ++j) {
      const int e = tid + j * THREADS, r = e % BM, kk = e / BM;
      const uint32_t off = (r / 8) * (BK * 64) + sw64(static_cast<uint32_t>(kk * 64 + (r & 7) * 8));
      *reinterpret_cast<double*>(sP + off) = pr[j];
    }
#pragma unroll
    for (int j = 0; j < Q_PER; ++j) {
      int n, kk;
      q_coord(j, n, kk);
      uint32_t off;
      if constexpr (QK)  // KX: [k-block][n][8 k]
        off = (kk / 8) * (BN * 64) + sw64(static_cast<uint32_t>(n * 64 + (kk & 7) * 8));
      else               // XK: [n-block][k][8 n]
        off = (n / 8) * (BK * 64) + sw64(static_cast<uint32_t>(kk * 64 + (n & 7) * 8));
      *reinterpret_cast<double*>(sQ + off) = qr[j];
    }
  };

  const int g8 = lane >> 2, t = lane & 3;
  const int wm = warp % WM, wn = warp / WM;
  const int mw = wm * WTM, nw = wn * WTN;
  const int jg = 2 * ((g8 >> 1) & 1) + (g8 >> 2);
  const uint32_t J0 = static_cast<uint32_t>(jg ^ (t >> 1)) << 4;
  const uint32_t xk_off = static_cast<uint32_t>(t * 64 + (g8 & 1) * 8);
  const uint32_t kx_off = static_cast<uint32_t>(xmap8(g8) * 64 + (t & 1) * 8);

  double acc[FM][FN][2];
#pragma unroll
  for (int fm = 0; fm < FM; ++fm)
#pragma unroll
    for (int fn = 0; fn < FN; ++fn) acc[fm][fn][0] = acc[fm][fn][1] = 0.0;

  load(0);
  store(0);
  __syncthreads();
  for (int kb = 0; kb < KT; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < KT) load(kb + 1);  // in flight during this k-block's math
    const uint8_t* sP = smem + buf * STAGE;
    const uint8_t* sQ = sP + P_EL * 8;
#pragma unroll
    for (int s = 0; s < BK / 4; ++s) {
      const uint32_t Js = J0 ^ (32u * static_cast<uint32_t>(s & 1));
      double pf[FM], qf[FN];
#pragma unroll
      for (int fm = 0; fm < FM; ++fm)
        pf[fm] = *reinterpret_cast<const double*>(sP + ((mw >> 3) + fm) * (BK * 64) + (4 * s) * 64 + xk_off + Js);
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) {
        if constexpr (QK)
          qf[fn] = *reinterpret_cast<const double*>(sQ + (s >> 1) * (BN * 64) + (nw + 8 * fn) * 64 + kx_off + Js);
        else
          qf[fn] = *reinterpret_cast<const double*>(sQ + ((nw >> 3) + fn) * (BK * 64) + (4 * s) * 64 + xk_off + Js);
      }
#pragma unroll
      for (int fm = 0; fm < FM; ++fm)
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) dmma_8x8x4(acc[fm][fn][0], acc[fm][fn][1], qf[fn], pf[fm]);
    }
    if (kb + 1 < KT) store(buf ^ 1);
    __syncthreads();
  }

  // epilogue: 8-byte stores, any alignment
  const int mp = xmap8(2 * t);
#pragma unroll
  for (int fm = 0; fm < FM; ++fm) {
    const int64_t q = int64_t(mtile) * (BM / 8) + (mw >> 3) + fm;
    int64_t c = 0, row0;
    if constexpr (QK) {
      row0 = 8 * q + mp;
    } else {
      if (q >= g.mfrags) continue;
      c = q / g.AB;
      row0 = 8 * (q - c * g.AB) + mp;
    }
#pragma unroll
    for (int fn = 0; fn < FN; ++fn) {
      const int64_t n = n0 + nw + 8 * fn + xmap8(g8);
      if (n >= g.ntot) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t row = row0 + h;
        if (row >= g.Mlim) continue;
        double* dst = QK ? g.S + row + n * g.N : g.S + row + n * g.A + c * g.A * g.N;
        *dst = g.accumulate ? *dst + acc[fm][fn][h] : acc[fm][fn][h];
      }
    }
  }
}

}  // namespace mumode_gpu
