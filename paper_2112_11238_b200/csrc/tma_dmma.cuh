// Persistent, warp-specialised mu-mode product kernel for sm_100a:
// TMA (cp.async.bulk.tensor, 128B swizzle) stages operand slabs into a
// multi-stage shared-memory ring guarded by mbarriers; eight consumer warps
// run fp64 tensor-core MMAs (mma.sync m8n8k4 -> SASS DMMA.8x8x4: the only
// fp64 tensor-core path on sm_100a, tcgen05 has no f64 kind) and store
// straight from registers.
//
// Every mu-mode product is cast as D(M x N) [+ batch] = P(M x K) * Q(K x N)
// with D and P contiguous along M (column-major):
//   mu == 1 : P = L (n x m), Q = T viewed m x prod(m_2..m_d) (K-contiguous),
//             D = S (n x prod(..)), no batch            -> QK = true
//   mu  > 1 : P = T_c (A x m, A = prod_{k<mu} m_k), Q = L^T (N-contiguous),
//             D = S_c (A x n), batch c over modes > mu  -> QK = false
// so interior modes are contracted in place: the permute -> GEMM -> ipermute
// of the reference (mode_product.hpp:73-76, tucker.hpp:96-107) never happens.
//
// Shared-memory layout: operands arrive as 16-double (128 B) wide boxes with
// the TMA 128B swizzle (16-B chunk j of 128-B row r stored at chunk j ^ (r&7)).
// A k-step's four k rows are taken in the order {0,4,1,5} / {2,6,3,7} of each
// 8-row group, which makes every fragment load hit each bank exactly twice
// (two wavefronts for 256 B: conflict-free) in all three operand layouts.
#pragma once
#include "common.cuh"

namespace mumode_gpu {

struct TmaParams {
  double* D;
  int64_t ldD;      // column stride of D (elements)
  int64_t bstride;  // batch stride of D (elements)
  int M, N, K;
  int mt, nt;       // tile counts along M and N
  int64_t tiles;    // mt * nt * batches
};

template <int BM_, int BN_, int BK_, int STAGES_, int WM_, int WN_>
struct TmaCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, STAGES = STAGES_, WM = WM_, WN = WN_;
  static constexpr int MMA_WARPS = WM * WN;
  // MMA warps + one producer warpgroup (setmaxnreg works per warpgroup; the
  // 4 x 32 x 168 producer-group registers are what the MMA warps grow into).
  static constexpr int THREADS = (MMA_WARPS + 4) * 32;
  static_assert(MMA_WARPS % 4 == 0, "MMA warps must form whole warpgroups");
  static constexpr int WTM = BM / WM, WTN = BN / WN;  // warp tile
  static constexpr int FM = WTM / 8, FN = WTN / 8;    // fragments per warp
  static constexpr int P_BYTES = BM * BK * 8, Q_BYTES = BN * BK * 8;
  static constexpr int STAGE_BYTES = P_BYTES + Q_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 2 * STAGES * 8;
  static_assert(BM % 16 == 0 && BN % 16 == 0 && BK % 16 == 0, "16-double TMA boxes");
  static_assert(WTM % 16 == 0 && WTN % 16 == 0, "warp tile must cover whole 16-wide boxes");
  static_assert(BN <= 256 && BK <= 256, "TMA box extent limit");
};

// Physical k row (within a stage) of k-step s for lane quad index t.
__device__ __forceinline__ int krow_of(int s, int t) {
  return 8 * (s >> 1) + 2 * (s & 1) + (t >> 1) + 4 * (t & 1);
}

template <class Cfg, bool QK>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    modeprod_tma_kernel(const __grid_constant__ CUtensorMap mapP,
                        const __grid_constant__ CUtensorMap mapQ, const TmaParams p) {
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr int FM = Cfg::FM, FN = Cfg::FN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KT = (p.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], Cfg::MMA_WARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp >= Cfg::MMA_WARPS) {
    // ------------------------------------------------------------ producer
    // 12 warps at launch cap every thread at 168 registers; the producer
    // warpgroup drops to 40 so the two MMA warpgroups can grow to 232.
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == Cfg::MMA_WARPS && lane == 0) {
      tma_prefetch_desc(&mapP);
      tma_prefetch_desc(&mapQ);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
        const int mtile = static_cast<int>(tile % p.mt);
        const int64_t rest = tile / p.mt;
        const int ntile = static_cast<int>(rest % p.nt);
        const int batch = static_cast<int>(rest / p.nt);
        const int m0 = mtile * BM, n0 = ntile * BN;
        for (int kb = 0; kb < KT; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sP = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sQ = sP + Cfg::P_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
          const int k0 = kb * BK;
#pragma unroll
          for (int b = 0; b < BM / 16; ++b) {
            if constexpr (QK)
              tma_load_2d(sP + b * BK * 128, &mapP, &full_bar[stage], m0 + 16 * b, k0);
            else
              tma_load_3d(sP + b * BK * 128, &mapP, &full_bar[stage], m0 + 16 * b, k0, batch);
          }
          if constexpr (QK) {
#pragma unroll
            for (int b = 0; b < BK / 16; ++b)
              tma_load_2d(sQ + b * BN * 128, &mapQ, &full_bar[stage], k0 + 16 * b, n0);
          } else {
#pragma unroll
            for (int b = 0; b < BN / 16; ++b)
              tma_load_2d(sQ + b * BK * 128, &mapQ, &full_bar[stage], n0 + 16 * b, k0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % Cfg::WM, wn = warp / Cfg::WM;
  const int mw = wm * Cfg::WTM, nw = wn * Cfg::WTN;

  // Per-fragment byte offsets that do not depend on the k-step.
  // P sub-tile (16 m) b: rows k (128 B each); chunk index = (m%16)>>1.
  uint32_t p_off[FM];
  int p_ch[FM];
#pragma unroll
  for (int fm = 0; fm < FM; ++fm) {
    const int m = mw + fm * 8 + g;
    p_off[fm] = (m >> 4) * (BK * 128) + ((m & 1) << 3);
    p_ch[fm] = (m & 15) >> 1;
  }
  uint32_t q_off[FN];
  int q_ch[FN];
#pragma unroll
  for (int fn = 0; fn < FN; ++fn) {
    const int n = nw + fn * 8 + g;
    if constexpr (QK) {
      q_off[fn] = n * 128;  // row n of each 16-k sub-tile
      q_ch[fn] = n & 7;     // swizzle key of row n
    } else {
      q_off[fn] = (n >> 4) * (BK * 128) + ((n & 1) << 3);
      q_ch[fn] = (n & 15) >> 1;
    }
  }

  int stage = 0;
  uint32_t phase = 0;
  for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
    const int mtile = static_cast<int>(tile % p.mt);
    const int64_t rest = tile / p.mt;
    const int ntile = static_cast<int>(rest % p.nt);
    const int64_t batch = rest / p.nt;

    double acc[FM][FN][2];
#pragma unroll
    for (int fm = 0; fm < FM; ++fm)
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) acc[fm][fn][0] = acc[fm][fn][1] = 0.0;

    for (int kb = 0; kb < KT; ++kb) {
      mbar_wait(&full_bar[stage], phase);
      const uint8_t* sP = smem + stage * Cfg::STAGE_BYTES;
      const uint8_t* sQ = sP + Cfg::P_BYTES;
#pragma unroll
      for (int s = 0; s < BK / 4; ++s) {
        const int kr = krow_of(s, t);  // 0..BK-1
        const int kx = kr & 7;
        double pf[FM], qf[FN];
#pragma unroll
        for (int fm = 0; fm < FM; ++fm)
          pf[fm] = *reinterpret_cast<const double*>(sP + p_off[fm] + kr * 128 +
                                                    ((p_ch[fm] ^ kx) << 4));
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) {
          if constexpr (QK) {
            const int kk = kr & 15;
            qf[fn] = *reinterpret_cast<const double*>(
                sQ + (kr >> 4) * (BN * 128) + q_off[fn] + ((((kk >> 1) ^ q_ch[fn])) << 4) +
                ((kk & 1) << 3));
          } else {
            qf[fn] = *reinterpret_cast<const double*>(sQ + q_off[fn] + kr * 128 +
                                                      ((q_ch[fn] ^ kx) << 4));
          }
        }
#pragma unroll
        for (int fm = 0; fm < FM; ++fm)
#pragma unroll
          for (int fn = 0; fn < FN; ++fn) dmma_8x8x4(acc[fm][fn][0], acc[fm][fn][1], qf[fn], pf[fm]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[stage]);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }

    // epilogue: D(m, m+1 ; n) from registers, 16-B stores along M
    double* Db = p.D + batch * p.bstride;
    const int mbase = mtile * BM + mw + 2 * t;
    const int nbase = ntile * BN + nw + g;
#pragma unroll
    for (int fn = 0; fn < FN; ++fn) {
      const int n = nbase + fn * 8;
      if (n >= p.N) continue;
      double* col = Db + static_cast<int64_t>(n) * p.ldD;
#pragma unroll
      for (int fm = 0; fm < FM; ++fm) {
        const int m = mbase + fm * 8;
        if (m < p.M) stg_f64x2(col + m, acc[fm][fn][0], acc[fm][fn][1]);
      }
    }
  }
}

}  // namespace mumode_gpu
