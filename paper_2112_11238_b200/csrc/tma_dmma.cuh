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
// Fragment-to-element maps (below) keep every 64-bit fragment load
// conflict-free (two wavefronts per warp) in all three operand layouts.
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

// Fragment -> element maps (lane = 4*g + t). 64-bit shared loads are served
// per half-warp, so each half-warp's 16 addresses must land on 16 distinct
// 8-byte bank slots. With k-step s reading k rows 4s + t:
//   x-contiguous operands ([k][x] 128B-swizzled rows: P, and Q when QK=false)
//     fragment pair half h, column g  ->  x = 16*blk + 4h + xmap(g)
//     xmap(g) = (g&1) + 8((g>>1)&1) + 2(g>>2)     {0,1,8,9,2,3,10,11}
//   k-contiguous Q ([n][k] rows, QK=true)
//     fragment pair half h, row g     ->  n = 16*blk + 2g + h
// Both are bijections onto the 16-wide box and conflict-free for every s, h;
// xmap(2t), xmap(2t)+1 stay adjacent so the epilogue keeps 16-byte stores.
__device__ __forceinline__ int xmap(int g) { return (g & 1) + 8 * ((g >> 1) & 1) + 2 * (g >> 2); }

template <class Cfg, bool QK>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    modeprod_tma_kernel(const __grid_constant__ CUtensorMap mapP,
                        const __grid_constant__ CUtensorMap mapQ, const TmaParams p) {
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr int FM = Cfg::FM, FN = Cfg::FN;
  static_assert(FM % 2 == 0 && FN % 2 == 0, "fragments come in 16-wide pairs");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment for the 128B-swizzle atoms, by pointer arithmetic so the
  // compiler keeps the shared address space (LDS, not generic LD).
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
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

  // tile -> (mtile, ntile, batch); the operand tile shared by consecutive
  // CTAs is the big tensor (Q = T for mode 1: m fastest; P = T_c otherwise:
  // n fastest), so T streams from HBM once and repeats hit L2.
  auto decode = [&](int64_t tile, int& mt, int& nt, int64_t& b) {
    if constexpr (QK) {
      mt = static_cast<int>(tile % p.mt);
      const int64_t r = tile / p.mt;
      nt = static_cast<int>(r % p.nt);
      b = r / p.nt;
    } else {
      nt = static_cast<int>(tile % p.nt);
      const int64_t r = tile / p.nt;
      mt = static_cast<int>(r % p.mt);
      b = r / p.mt;
    }
  };

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
        int mtile, ntile;
        int64_t batch;
        decode(tile, mtile, ntile, batch);
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
              tma_load_3d(sP + b * BK * 128, &mapP, &full_bar[stage], m0 + 16 * b, k0,
                          static_cast<int32_t>(batch));
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

  // Per-thread byte offsets inside a stage. x-contiguous operand, element
  // (x = 16*blk + 4h + xmap(g), k = 4s + t): blk*BK*128 + k*128 + chunk*16 + (g&1)*8
  // with chunk = (j ^ (k&7)), j = 4((g>>1)&1) + (g>>2) + 2h, so
  // chunk*16 = ((j0 ^ t) << 4) ^ (2h << 4) ^ ((4(s&1)) << 4).
  const uint32_t jx = static_cast<uint32_t>((4 * ((g >> 1) & 1) + (g >> 2)) ^ t) << 4;
  const uint32_t xoff = static_cast<uint32_t>(t * 128 + (g & 1) * 8);
  // k-contiguous Q, element (n = 16*blk + 2g + h, k = 4s + t):
  // n*128 + (((2s + (t>>1)) ^ (n&7)) << 4) + (t&1)*8.
  const uint32_t jq = static_cast<uint32_t>(((t >> 1) ^ ((2 * g) & 7))) << 4;
  const uint32_t qoff = static_cast<uint32_t>(2 * g * 128 + (t & 1) * 8);

  int stage = 0;
  uint32_t phase = 0;
  for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
    int mtile, ntile;
    int64_t batch;
    decode(tile, mtile, ntile, batch);

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
        double pf[FM], qf[FN];
#pragma unroll
        for (int fm = 0; fm < FM; ++fm) {
          const int blk = (mw >> 4) + (fm >> 1), h = fm & 1;
          const uint32_t ch = jx ^ (static_cast<uint32_t>(2 * h) << 4) ^
                              (static_cast<uint32_t>(4 * (s & 1)) << 4);
          pf[fm] = *reinterpret_cast<const double*>(sP + blk * (BK * 128) + (4 * s) * 128 + xoff + ch);
        }
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) {
          const int blk = (nw >> 4) + (fn >> 1), h = fn & 1;
          if constexpr (QK) {
            const int kb16 = (4 * s) >> 4, s4 = s & 3;
            const uint32_t ch = jq ^ (static_cast<uint32_t>((2 * s4) ^ h) << 4);
            qf[fn] = *reinterpret_cast<const double*>(sQ + kb16 * (BN * 128) + (16 * blk + h) * 128 +
                                                      qoff + ch);
          } else {
            const uint32_t ch = jx ^ (static_cast<uint32_t>(2 * h) << 4) ^
                                (static_cast<uint32_t>(4 * (s & 1)) << 4);
            qf[fn] = *reinterpret_cast<const double*>(sQ + blk * (BK * 128) + (4 * s) * 128 + xoff + ch);
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

    // epilogue: D(m, m+1 ; n) straight from registers, 16-byte stores along M
    double* Db = p.D + batch * p.bstride;
    const int mrow = mtile * BM + mw + 8 * (t & 1) + 2 * (t >> 1);
#pragma unroll
    for (int fn = 0; fn < FN; ++fn) {
      const int blk = (nw >> 4) + (fn >> 1), h = fn & 1;
      const int n = ntile * BN + 16 * blk + (QK ? (2 * g + h) : (4 * h + xmap(g)));
      if (n >= p.N) continue;
      double* col = Db + static_cast<int64_t>(n) * p.ldD;
#pragma unroll
      for (int fm = 0; fm < FM; ++fm) {
        const int m = mrow + 16 * (fm >> 1) + 4 * (fm & 1);
        if (m < p.M) stg_f64x2(col + m, acc[fm][fn][0], acc[fm][fn][1]);
      }
    }
  }
}

}  // namespace mumode_gpu
