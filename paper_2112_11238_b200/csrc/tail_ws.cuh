// Strided fused two-mode pass, streamed: the tail pass of tail.cuh (32-wide a
// tiles, 256-B rows for TMA loads and stores) without the resident
// intermediate.
//
// tail_pair_kernel keeps the whole mode-mu result of a tile (Y, 147 KB for
// MU = 24) in shared memory, which leaves a 3-deep load ring, and separates
// the two modes by CTA-wide barriers (ncu on C5 pass 3: DMMA pipe 76 %
// active; stage-data waits ~10 % and phase barriers ~9 % of stall samples).
// Here mode mu+1 accumulates in registers as the b2 stages arrive, so only
// a few stages of the intermediate exist at a time (NYS buffers), and the
// two modes run on separate warp groups:
//
//   producer warpgroup : TMA ring of stages {16 a, 2, MU b1, 4 b2, 1} (as tail)
//   group A (1 wg)     : mode mu on stage z: X -> Ys[z % NYS] (tail's maps)
//   group B (2 wgs)    : mode mu+1: acc(i, j, a) += L2(j, b2) Ys(i, b2, a)
//                        over the tile's MU/4 stages; each warp owns MU/8
//                        i's (MU/8 x 4 x NF accumulator fragments); at the
//                        end of a tile it stages one i at a time (MU rows of
//                        256 B, TMA-box layout) and TMA-stores it.
//
// Ys handoffs are named barriers (ids 2 + yb "stage full": A arrives, B
// syncs; 2 + NYS + yb "stage free": B arrives, A syncs; the first / last NYS
// stages of a CTA skip the free handshake). The k-order of every output's
// DMMA chain (b1 for mode mu, b2 = stage by stage for mode mu+1) is the
// tail kernel's, so results are bitwise equal to it. Stage buffer rows and
// swizzle = tail's Y slot rows (only b2 & 3 and i & 1 enter the swizzle), so
// every fragment load and store stays bank-conflict-free.
#pragma once
#include "common.cuh"
#include "tail.cuh"

namespace mumode_gpu {

template <int MU>
struct TailWsCfg {
  static constexpr int NF = MU / 8;
  static constexpr int KS = MU / 4;
  static constexpr int KB = 4;           // b2 values per stage
  static constexpr int NST = MU / KB;    // stages per tile
  static constexpr int WB = 8;           // mode mu+1 warps (2 warpgroups)
  static constexpr int WA = 4;           // mode mu warps (1 warpgroup)
  static constexpr int THREADS = (WB + WA + 4) * 32;
  static constexpr int IPW = MU / WB;    // i's per group-B warp
  static constexpr int UPA = 4 * KB / WA;  // mode-mu units per group-A warp per stage
  static constexpr int GA = 2;           // group-A units advanced together
  static constexpr int X_BYTES = 32 * MU * KB * 8;
  static constexpr int YS_BYTES = MU * 1024;   // MU slots of 4 b2 rows x 256 B
  static constexpr int STG_BYTES = MU * 256;   // one i: MU j-rows x 256 B
  // stage buffers between the groups: C5 pass 3 643 (2) / 614 (3) / 607 (4)
  // / 653 us (5: the load ring drops to 2 stages)
  static constexpr int NYS = 4;
  static constexpr int FIXED = NYS * YS_BYTES + WB * STG_BYTES + 1024 + 256;
  static constexpr int NBUF_RAW = (227 * 1024 - FIXED) / X_BYTES;
  static constexpr int NBUF = NBUF_RAW > 6 ? 6 : NBUF_RAW;
  static constexpr int SMEM_BYTES = NBUF * X_BYTES + FIXED;
  // setmaxnreg split of the 128-per-thread launch allocation
  static constexpr int LAUNCH_REGS = 65536 / THREADS;
  static constexpr int P_REGS = 24, A_REGS = 104, B_REGS = 192;
  static_assert(128 * P_REGS + 128 * A_REGS + WB * 32 * B_REGS <= LAUNCH_REGS * THREADS, "setmaxnreg budget");
  static_assert(A_REGS <= LAUNCH_REGS && B_REGS >= LAUNCH_REGS, "dec / inc directions");
  static_assert(MU % 8 == 0 && MU <= 24 && MU % WB == 0, "square modes of 8..24");
  static_assert(UPA % GA == 0, "group-A unit batches");
  static_assert(NBUF >= 2, "shared memory for a 2-deep ring");
  static_assert(X_BYTES % 1024 == 0 && YS_BYTES % 1024 == 0 && STG_BYTES % 1024 == 0, "128B-swizzle atoms");
};

// stage-buffer element (slot i, b2 & 3, h, a16): tail_y_off's row and swizzle
__device__ __forceinline__ uint32_t ys_off(int i, int b2l, int h, int a16) {
  const uint32_t ch = (static_cast<uint32_t>(a16 >> 1) ^ ((2u * b2l) ^ (2u * h + 4u * (i & 1)))) & 7u;
  return static_cast<uint32_t>(i * 1024 + (2 * b2l + h) * 128) + ch * 16 + (a16 & 1) * 8;
}

template <int MU>
__global__ void __launch_bounds__(TailWsCfg<MU>::THREADS, 1)
    tail_ws_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapS,
                   const TailParams p) {
  using Cfg = TailWsCfg<MU>;
  constexpr int NYS = Cfg::NYS;
  constexpr int NF = Cfg::NF, KS = Cfg::KS, NST = Cfg::NST, NBUF = Cfg::NBUF;
  constexpr int WA = Cfg::WA, WB = Cfg::WB, GA = Cfg::GA;
  constexpr int PAIR = (WA + WB) * 32;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* Xs = smem;
  uint8_t* Ys = Xs + NBUF * Cfg::X_BYTES;
  uint8_t* Stg = Ys + NYS * Cfg::YS_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(Stg + WB * Cfg::STG_BYTES);
  uint64_t* empty_bar = full_bar + NBUF;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(&full_bar[b], 1);
      mbar_init(&empty_bar[b], WA);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();  // before any global access (factors included)

  const int64_t ntiles = (p.tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;  // tiles of this CTA
  const int64_t nst = ntiles * NST;                                           // stages of this CTA

  if (warp >= WB + WA) {
    // ------------------------------------------------------- producer warpgroup
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(Cfg::P_REGS) : "memory");
    if (warp == WB + WA && lane == 0) {
      tma_prefetch_desc(&mapX);
      int buf = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
        const int64_t c = tile / p.ablks, ab = tile - c * p.ablks;
        for (int st = 0; st < NST; ++st) {
          mbar_wait(&empty_bar[buf], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[buf], Cfg::X_BYTES);
          tma_load_5d(Xs + buf * Cfg::X_BYTES, &mapX, &full_bar[buf], 0, static_cast<int32_t>(2 * ab), 0,
                      Cfg::KB * st, static_cast<int32_t>(c));
          if (++buf == NBUF) {
            buf = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  const int g = lane >> 2, t = lane & 3;
  if (warp >= WB) {
    // ------------------------------------------------ group A: mode mu, X -> Ys
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(Cfg::A_REGS) : "memory");
    const int wa = warp - WB;
    double l1[NF][KS];
#pragma unroll
    for (int nf = 0; nf < NF; ++nf)
#pragma unroll
      for (int s = 0; s < KS; ++s) l1[nf][s] = p.L1[(8 * nf + g) + (4 * s + t) * MU];
    // B-fragment column of this lane: (a16, h) = (4f + (g&1) + 2(g>>2), (g>>1)&1)
    const int xa = (g & 1) + 2 * (g >> 2), xh = (g >> 1) & 1;
    int buf = 0;
    uint32_t phase = 0;
    for (int64_t z = 0; z < nst; ++z) {
      const int yb = static_cast<int>(z % NYS);
      mbar_wait(&full_bar[buf], phase);
      if (z >= NYS) named_barrier_sync(2 + NYS + yb, PAIR);  // Ys[yb] consumed by group B
      const uint8_t* X = Xs + buf * Cfg::X_BYTES;
      uint8_t* Y = Ys + yb * Cfg::YS_BYTES;
#pragma unroll
      for (int bt = 0; bt < Cfg::UPA / GA; ++bt) {
        double acc[GA][NF][2];
#pragma unroll
        for (int uu = 0; uu < GA; ++uu)
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) acc[uu][nf][0] = acc[uu][nf][1] = 0.0;
#pragma unroll
        for (int s = 0; s < KS; ++s)
#pragma unroll
          for (int uu = 0; uu < GA; ++uu) {
            const int u = wa + WA * (bt * GA + uu);
            const int b2l = u >> 2, f = u & 3;
            const uint32_t row = static_cast<uint32_t>((b2l * MU + 4 * s + t) * 2 + xh);
            const double xf = *reinterpret_cast<const double*>(X + sw128_off(row, 4 * f + xa));
#pragma unroll
            for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[uu][nf][0], acc[uu][nf][1], l1[nf][s], xf);
          }
        // D[g -> i = 8nf + g][cols 2t, 2t+1 -> a16 = 4f + 2(t>>1) + {0,1}, h = t&1]
#pragma unroll
        for (int uu = 0; uu < GA; ++uu) {
          const int u = wa + WA * (bt * GA + uu);
          const int b2l = u >> 2, f = u & 3;
#pragma unroll
          for (int nf = 0; nf < NF; ++nf)
            *reinterpret_cast<double2*>(Y + ys_off(8 * nf + g, b2l, t & 1, 4 * f + 2 * (t >> 1))) =
                make_double2(acc[uu][nf][0], acc[uu][nf][1]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[buf]);  // X[buf] may be refilled
      named_barrier_arrive(2 + yb, PAIR);            // Ys[yb] complete
      if (++buf == NBUF) {
        buf = 0;
        phase ^= 1;
      }
    }
    return;
  }

  // ------------------------------------- group B: mode mu+1, Ys -> registers -> HBM
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(Cfg::B_REGS) : "memory");
  constexpr int IPW = Cfg::IPW;
  uint8_t* slot = Stg + warp * Cfg::STG_BYTES;
  const double* l2col = p.L2 + (tail_sig(g)) + t * MU;  // L2(8nf + sig(g), 4st + t)
  int64_t z = 0;
  for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
    const int64_t c = tile / p.ablks, ab = tile - c * p.ablks;
    double acc[IPW][4][NF][2];
#pragma unroll
    for (int ii = 0; ii < IPW; ++ii)
#pragma unroll
      for (int F = 0; F < 4; ++F)
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) acc[ii][F][nf][0] = acc[ii][F][nf][1] = 0.0;
#pragma unroll 1
    for (int st = 0; st < NST; ++st, ++z) {
      double l2f[NF];
#pragma unroll
      for (int nf = 0; nf < NF; ++nf) l2f[nf] = __ldg(l2col + 8 * nf + 4 * st * MU);
      const int yb = static_cast<int>(z % NYS);
      named_barrier_sync(2 + yb, PAIR);  // Ys[yb] complete
      const uint8_t* Y = Ys + yb * Cfg::YS_BYTES;
#pragma unroll
      for (int ii = 0; ii < IPW; ++ii) {
        const int i = warp + WB * ii;
#pragma unroll
        for (int F = 0; F < 4; ++F) {
          const int h = F >> 1, m4 = F & 1;
          const double yf = *reinterpret_cast<const double*>(Y + ys_off(i, t, h, 8 * m4 + g));
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[ii][F][nf][0], acc[ii][F][nf][1], l2f[nf], yf);
        }
      }
      // every Ys value of this stage has been consumed by a DMMA
      if (z + NYS < nst) named_barrier_arrive_after_reads(2 + NYS + yb, PAIR);
    }
    // epilogue: one i at a time through this warp's staging slot (TMA-box
    // layout {16 a, 2 h, 1, MU j}: row 2j + h), then one TMA store
#pragma unroll
    for (int ii = 0; ii < IPW; ++ii) {
      if (lane == 0) bulk_wait_read_all();  // the slot's previous store has read it
      __syncwarp();
#pragma unroll
      for (int F = 0; F < 4; ++F)
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) {
          const int h = F >> 1, m4 = F & 1;
          const uint32_t row = static_cast<uint32_t>(2 * (8 * nf + tail_sig(g)) + h);
          *reinterpret_cast<double2*>(slot + sw128_off(row, 8 * m4 + 2 * t)) =
              make_double2(acc[ii][F][nf][0], acc[ii][F][nf][1]);
        }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tma_store_5d(&mapS, slot, 0, static_cast<int32_t>(2 * ab), warp + WB * ii, 0, static_cast<int32_t>(c));
        bulk_commit();
      }
    }
  }
  if (lane == 0) bulk_wait_all();
}

}  // namespace mumode_gpu
