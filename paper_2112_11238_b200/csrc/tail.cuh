// Fused two-mode pass for small square modes whose leading extent A is large
// (the last pass of config C5, 24^6: modes 5-6 over A = 24^4).
//
// Why a separate kernel: each (b1, b2) row of the tile lies A*8 B (2.65 MB
// for C5) from the next, so every row is a new 2-MB page. Measured on B200
// (tools/tma_pattern_probe.cu), the rate of such page-crossing row requests is
// fixed: 64-B rows cap a read at 2.4 TB/s, 128-B rows at 4.8 TB/s, 256-B rows
// reach 6.2 TB/s (= contiguous). Stores behave the same (8 rows x 64 B per
// warp store: 2.8 TB/s; 256-B rows or TMA stores: 6.0 TB/s). The pair kernel
// in fused.cuh moves 64-B rows (8 a's per tile). This kernel moves 256-B rows:
//
//   tile     = 32 consecutive a's x all (b1, b2) for one c.
//   load     = the tile streamed in MU/KB stages of KB b2-values, each ONE 5-D
//              TMA box {16 a, 2, MU b1, KB b2, 1} (128B swizzle; every b1 row
//              is one 256-B run) into a ring of NBUF stages.
//   mode mu  = contract b1 per stage: D(i, a) = L1 (registers) x X fragments;
//              results go to Y, resident for the whole tile (MU^2 x 32
//              doubles: 147 KB for MU = 24), one 1-KB-aligned "slot" per i.
//   mode mu+1= contract b2 from Y: each warp owns slots i, reads all of slot
//              i, then overwrites the slot with the finished outputs
//              S(a, i, :) in TMA-box layout and one lane issues a TMA store
//              {16, 2, 1, MU, 1} (MU rows of 256 B).
//
// Fragment maps (bank-conflict-free for all four shared-memory access
// patterns; checked exhaustively for MU = 8, 16, 24):
//   mode mu columns   n -> (a16, h) = (4f + (n&1) + 2(n>>2), (n>>1)&1)
//   mode mu+1 columns n -> (a16, h) = (8 m4 + n, h)  with F = (h, m4)
//   mode mu+1 rows    g -> j = 8 nf + sig(g), sig swaps bits 0 and 1 of g
//   Y slot i          row 2 b2 + h, 16-B chunk (a16>>1) ^ (2(b2&3) ^ (2h + 4(i&1)))
// where a = 16 h + a16 inside the 32-wide tile.
#pragma once
#include "common.cuh"

namespace mumode_gpu {

template <int MU>
struct TailCfg {
  static constexpr int NF = MU / 8;
  static constexpr int KS = MU / 4;
  static constexpr int KB = 4;                    // b2 values per stage
  static constexpr int NST = MU / KB;             // stages per tile
  static constexpr int WARPS = 8;                 // consumer warps
  static constexpr int THREADS = (WARPS + 1) * 32;
  static constexpr int SLOT = MU * 256;           // one i: MU rows (b2 / j) x 256 B
  static constexpr int Y_BYTES = MU * SLOT;
  static constexpr int X_BYTES = 32 * MU * KB * 8;
  static constexpr int AVAIL = 227 * 1024 - 1024 - 256 - Y_BYTES;
  static constexpr int NBUF_RAW = AVAIL / X_BYTES;
  static constexpr int NBUF = NBUF_RAW > 6 ? 6 : NBUF_RAW;
  static constexpr int SMEM_BYTES = Y_BYTES + NBUF * X_BYTES + 1024 + 256;
  static_assert(MU % 8 == 0 && MU <= 24, "square modes of 8..24");
  static_assert(NBUF >= 2, "shared memory for a 2-deep ring");
  static_assert(SLOT % 1024 == 0 && X_BYTES % 1024 == 0, "128B-swizzle atoms");
};

struct TailParams {
  const double* L1;
  const double* L2;
  int64_t ablks;  // A / 32
  int64_t tiles;  // ablks * C
};

__device__ __forceinline__ int tail_sig(int g) { return ((g & 1) << 1) | ((g >> 1) & 1) | (g & 4); }

// TMA 128B swizzle inside a 1024-B-aligned region: 16-B chunk ^= 128-B row & 7
__device__ __forceinline__ uint32_t sw128_off(uint32_t row, uint32_t a16) {
  return row * 128 + ((((a16 >> 1) ^ row) & 7u) << 4) + (a16 & 1) * 8;
}

template <int MU>
__device__ __forceinline__ uint32_t tail_y_off(int i, int b2, int h, int a16) {
  const uint32_t ch = (static_cast<uint32_t>(a16 >> 1) ^ ((2u * (b2 & 3)) ^ (2u * h + 4u * (i & 1)))) & 7u;
  return static_cast<uint32_t>(i * TailCfg<MU>::SLOT + (2 * b2 + h) * 128) + ch * 16 + (a16 & 1) * 8;
}

template <int MU>
__global__ void __launch_bounds__(TailCfg<MU>::THREADS, 1)
    tail_pair_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapS,
                     const TailParams p) {
  using Cfg = TailCfg<MU>;
  constexpr int NF = Cfg::NF, KS = Cfg::KS, KB = Cfg::KB, NST = Cfg::NST, NBUF = Cfg::NBUF;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* Y = smem;
  uint8_t* Xs = smem + Cfg::Y_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(Xs + NBUF * Cfg::X_BYTES);
  uint64_t* empty_bar = full_bar + NBUF;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(&full_bar[b], 1);
      mbar_init(&empty_bar[b], Cfg::WARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();  // before any global access (factors included)

  if (warp == Cfg::WARPS) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      tma_prefetch_desc(&mapX);
      int buf = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
        const int64_t c = tile / p.ablks, ab = tile - c * p.ablks;
        for (int st = 0; st < NST; ++st) {
          mbar_wait(&empty_bar[buf], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[buf], Cfg::X_BYTES);
          tma_load_5d(Xs + buf * Cfg::X_BYTES, &mapX, &full_bar[buf], 0, static_cast<int32_t>(2 * ab), 0,
                      KB * st, static_cast<int32_t>(c));
          if (++buf == NBUF) {
            buf = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int g = lane >> 2, t = lane & 3;
  // A-operand fragments A[g][t] of both factors, resident for the whole
  // kernel (mode mu+1 rows permuted by sig)
  double l1[NF][KS], l2[NF][KS];
#pragma unroll
  for (int nf = 0; nf < NF; ++nf)
#pragma unroll
    for (int s = 0; s < KS; ++s) {
      l1[nf][s] = p.L1[(8 * nf + g) + (4 * s + t) * MU];
      l2[nf][s] = p.L2[(8 * nf + tail_sig(g)) + (4 * s + t) * MU];
    }
  // mode-mu B-fragment column of this lane: (a16, h) = (4f + (g&1) + 2(g>>2), (g>>1)&1)
  const int xa = (g & 1) + 2 * (g >> 2), xh = (g >> 1) & 1;

  int buf = 0;
  uint32_t phase = 0;
  for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
    const int64_t c = tile / p.ablks, ab = tile - c * p.ablks;
    // ---- mode mu: stream stages, X -> Y
    for (int st = 0; st < NST; ++st) {
      mbar_wait(&full_bar[buf], phase);
      const uint8_t* X = Xs + buf * Cfg::X_BYTES;
#pragma unroll
      for (int uu = 0; uu < (4 * KB) / Cfg::WARPS; ++uu) {
        const int u = warp + Cfg::WARPS * uu;
        const int b2l = u >> 2, f = u & 3;
        double acc[NF][2];
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) acc[nf][0] = acc[nf][1] = 0.0;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          const uint32_t row = static_cast<uint32_t>((b2l * MU + 4 * s + t) * 2 + xh);
          const double xf = *reinterpret_cast<const double*>(X + sw128_off(row, 4 * f + xa));
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[nf][0], acc[nf][1], l1[nf][s], xf);
        }
        // D[g -> i = 8nf + g][cols 2t, 2t+1 -> a16 = 4f + 2(t>>1) + {0,1}, h = t&1]
        const int b2 = KB * st + b2l;
#pragma unroll
        for (int nf = 0; nf < NF; ++nf)
          *reinterpret_cast<double2*>(Y + tail_y_off<MU>(8 * nf + g, b2, t & 1, 4 * f + 2 * (t >> 1))) =
              make_double2(acc[nf][0], acc[nf][1]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[buf]);
      if (++buf == NBUF) {
        buf = 0;
        phase ^= 1;
      }
    }
    named_barrier_sync(1, Cfg::WARPS * 32);  // Y complete

    // ---- mode mu+1: Y slot i -> outputs S(a, i, :) staged in place -> TMA store
#pragma unroll 1
    for (int i = warp; i < MU; i += Cfg::WARPS) {
      double acc[4][NF][2];
#pragma unroll
      for (int F = 0; F < 4; ++F)
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) acc[F][nf][0] = acc[F][nf][1] = 0.0;
#pragma unroll
      for (int s = 0; s < KS; ++s)
#pragma unroll
        for (int F = 0; F < 4; ++F) {
          const int h = F >> 1, m4 = F & 1;
          const double yf = *reinterpret_cast<const double*>(Y + tail_y_off<MU>(i, 4 * s + t, h, 8 * m4 + g));
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[F][nf][0], acc[F][nf][1], l2[nf][s], yf);
        }
      __syncwarp();  // every lane has read slot i
      uint8_t* slot = Y + i * Cfg::SLOT;
#pragma unroll
      for (int F = 0; F < 4; ++F)
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) {
          const int h = F >> 1, m4 = F & 1;
          const uint32_t row = static_cast<uint32_t>(2 * (8 * nf + tail_sig(g)) + h);
          *reinterpret_cast<double2*>(slot + sw128_off(row, 8 * m4 + 2 * t)) =
              make_double2(acc[F][nf][0], acc[F][nf][1]);
        }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tma_store_5d(&mapS, slot, 0, static_cast<int32_t>(2 * ab), i, 0, static_cast<int32_t>(c));
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait_read_all();     // slots readable again
    named_barrier_sync(1, Cfg::WARPS * 32);  // Y free for the next tile
  }
  if (lane == 0) bulk_wait_all();
}

}  // namespace mumode_gpu
