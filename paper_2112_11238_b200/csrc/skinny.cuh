// Mode products with small extents (K = m_mu <= 32, N = n_mu <= 32): the
// products of high-order tensors with small modes (the paper's d = 6, n = 12..20
// Tucker benchmarks; any single mode product of a 24^6 tensor).
//
// Such a product does 2N flop per 16 B moved: HBM-bound. The tile kernels of
// tma_dmma.cuh stage it as 8-row (64-B) boxes of a large M tile and reach
// 1.4-3.9 TB/s on 12^6..24^6. Here every tile is small and moves 256-B rows:
//
//   mu > 1: tile = TC boxes of 32 consecutive a's x all K: ONE 5-D TMA box
//           {16 a, 2, P k, 1 | TC a-blocks, TC | 1 c} of the view
//           {16, 2, K, A/32, C} (128B swizzle, every k row one 256-B run) in,
//           D(n, a) = L(n, k) X(k, a) on DMMA, the 32 x N result staged in
//           TMA-box layout and written by ONE TMA store of the same shape.
//   mu = 1: tile = 32 TC consecutive fibres c (contiguous): box {P k, 32 TC}
//           in (no swizzle), D'(c, n) = X(c, k) L(n, k)^T, the result
//           (contiguous) out by one TMA store {P n, 32 TC c}.
//
// P = K and N rounded up to a multiple of 8 (8..32). Elements k >= K are
// zero-filled by TMA (box beyond the tensor extent), factor entries with
// k >= K or n >= N are zero in registers, and the TMA store clips n >= N and
// a >= A, so any K, N <= 32 work (mu = 1 needs even K and N: 16-B strides).
// The k-order of every output's DMMA chain is ascending k, as in the tile
// kernels.
//
// Warp-per-tile: the W consumer warps each own a ring of R stages and one
// staging buffer; the producer lane deals tiles round-robin to the warps, so
// no two consumer warps ever synchronise with each other.
#pragma once
#include "common.cuh"
#include "tail.cuh"

namespace mumode_gpu {

// TA = a's (mu > 1) or fibres (mu = 1) per box: 32, or 16 for mu > 1 when A
// is not a multiple of 16 (then the 4-D {16, A/16, ...} view does not exist;
// 128-B rows of a 3-D {A, K, C} view instead). A tile is TC such boxes along
// c (mu = 1: TC x 32 consecutive fibres) so that every stage moves >= 8 KB:
// with 2-4 KB stages the per-tile hand-offs, not HBM, set the pace
// (14^6 / 18^6 modes 3-4 at 2.1-2.9 TB/s).
template <int P, int TA = 32>
struct SkinnyCfg {
  static constexpr int NF = P / 8;  // 8-wide output fragments
  static constexpr int KS = P / 4;  // k-steps
  static constexpr int FA = TA / 8; // 8-wide a fragments
  static constexpr int W = 8;       // consumer warps
  static constexpr int THREADS = (W + 1) * 32;
  static constexpr int BOX_DOUBLES = TA * P;                                  // one box
  static constexpr int TC = BOX_DOUBLES >= 1024 ? 1 : 1024 / BOX_DOUBLES;      // boxes per tile
  static constexpr int TILE_BYTES = TC * BOX_DOUBLES * 8;  // one stage (and one staged result)
  static constexpr int R_RAW = (227 * 1024 - 1024 - 256) / (W * TILE_BYTES) - 1;
  static constexpr int R = R_RAW > 4 ? 4 : R_RAW;  // stages per warp
  static constexpr int SMEM_BYTES = W * (R + 1) * TILE_BYTES + 1024 + 2 * W * R * 8 + 64;
  static_assert(P % 8 == 0 && P >= 8 && P <= 32, "P in 8..32");
  static_assert(TA == 32 || TA == 16, "32- or 16-wide tiles");
  static_assert(R >= 2, "shared memory for 2 stages per warp");
  static_assert((BOX_DOUBLES * 8) % 1024 == 0, "128B-swizzle atoms per box");
};

struct SkinnyParams {
  const double* L;
  int64_t sLi, sLk;  // op(L)(n, k) = L[n * sLi + k * sLk]
  int K, N;
  int64_t ablks;     // mu > 1: ceil(A / TA)
  int64_t tiles;
  int A, TC;         // skinny_slab_kernel: a-extent (<= 32) and c-slabs per tile
  int a_major;       // skinny_kernel, 32-a boxes: a tile's TC boxes run along a (few c's)
};

// 16-wide a tiles: fragment column n of a-fragment f -> a = 4f + (n&1) +
// 8((n>>1)&1) + 2(n>>2), so the 8 (k, a-pair) chunks a half-warp loads hit 8
// distinct 16-B bank groups of the 128B-swizzled k rows.
__device__ __forceinline__ int skinny_col16(int f, int n) { return 4 * f + (n & 1) + 8 * ((n >> 1) & 1) + 2 * (n >> 2); }

// ACC: S += result (the kronsumv term accumulation, tucker.hpp:222-231): each
// warp TMA-loads its output tile of S into the staging buffer while it
// computes, and adds before the TMA store (old + term, the reference's order).
template <int P, bool MODE1, int TA = 32, bool ACC = false>
__global__ void __launch_bounds__(SkinnyCfg<P, TA>::THREADS, 1)
    skinny_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapS,
                  const SkinnyParams p) {
  using Cfg = SkinnyCfg<P, TA>;
  constexpr int NF = Cfg::NF, KS = Cfg::KS, FA = Cfg::FA, W = Cfg::W, R = Cfg::R, TC = Cfg::TC;
  constexpr int BOXB = Cfg::BOX_DOUBLES * 8;
  static_assert(!MODE1 || TA == 32, "mode 1 uses 32-fibre boxes");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* Xs = smem;                                   // [warp][stage]
  uint8_t* Stg = smem + W * R * Cfg::TILE_BYTES;        // [warp]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(Stg + W * Cfg::TILE_BYTES);
  uint64_t* empty_bar = full_bar + W * R;
  uint64_t* acc_bar = empty_bar + W * R;  // ACC: per warp, the S tile load
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  static_assert(!(ACC && MODE1), "accumulating mode-1 products take the tile kernels");

  if (threadIdx.x == 0) {
    for (int b = 0; b < W * R; ++b) {
      mbar_init(&full_bar[b], 1);
      mbar_init(&empty_bar[b], 1);
    }
    for (int w = 0; w < W; ++w) mbar_init(&acc_bar[w], 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();  // before any global access (factor included)

  // tile -> box coordinates: mu = 1 fibre offset; mu > 1 (a-block, c) of the
  // tile's first box; its TC boxes run along c, or along a when a_major
  auto coords = [&](int64_t tile, int32_t& ca, int32_t& cc0) {
    if constexpr (MODE1) {
      ca = 0;
      cc0 = static_cast<int32_t>(tile * 32 * TC);
    } else {
      const int64_t cb = tile / p.ablks, ab = tile - cb * p.ablks;
      const bool am = (TA == 32) && p.a_major;
      ca = static_cast<int32_t>(am ? ab * TC : ab);
      cc0 = static_cast<int32_t>(am ? cb : cb * TC);
    }
  };

  if (warp == W) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      tma_prefetch_desc(&mapX);
      int64_t k = 0;
      for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x, ++k) {
        const int w = static_cast<int>(k % W);
        const int64_t q = k / W;  // this warp's tile count so far
        const int slot = static_cast<int>(q % R);
        const uint32_t phase = static_cast<uint32_t>((q / R) & 1);
        const int b = w * R + slot;
        mbar_wait(&empty_bar[b], phase ^ 1);
        mbar_arrive_expect_tx(&full_bar[b], Cfg::TILE_BYTES);
        uint8_t* dst = Xs + b * Cfg::TILE_BYTES;
        int32_t ca, cc0;
        coords(tile, ca, cc0);
        if constexpr (MODE1)
          tma_load_2d(dst, &mapX, &full_bar[b], 0, cc0);
        else if constexpr (TA == 32)
          tma_load_5d(dst, &mapX, &full_bar[b], 0, 0, 0, ca, cc0);
        else
          tma_load_3d(dst, &mapX, &full_bar[b], 16 * ca, 0, cc0);
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int g = lane >> 2, t = lane & 3;
  // factor fragments op(L)(n, k), zero outside N x K:
  //   mu > 1: A operand A[g][t] = L(8nf + g, 4s + t)
  //   mu = 1: B operand B[t][g] = L(8nf + g, 4s + t)  (D' = X L^T)
  double lf[NF][KS];
#pragma unroll
  for (int nf = 0; nf < NF; ++nf)
#pragma unroll
    for (int s = 0; s < KS; ++s) {
      const int n = 8 * nf + g, kk = 4 * s + t;
      lf[nf][s] = (n < p.N && kk < p.K) ? __ldg(p.L + n * p.sLi + kk * p.sLk) : 0.0;
    }
  const int xa = (g & 1) + 2 * (g >> 2), xh = (g >> 1) & 1;  // tail's B-fragment column map
  uint8_t* slot_out = Stg + warp * Cfg::TILE_BYTES;
  int64_t q = 0;
  for (int64_t tile = blockIdx.x + static_cast<int64_t>(warp) * gridDim.x; tile < p.tiles;
       tile += static_cast<int64_t>(W) * gridDim.x, ++q) {
    const int b = warp * R + static_cast<int>(q % R);
    mbar_wait(&full_bar[b], static_cast<uint32_t>((q / R) & 1));
    if (lane == 0) bulk_wait_read_all();  // the staging buffer's previous store has read it
    if constexpr (ACC) {
      if (lane == 0) {  // the current S tile into the staging buffer (same box as the store)
        int32_t ca, cc0;
        coords(tile, ca, cc0);
        mbar_arrive_expect_tx(&acc_bar[warp], Cfg::TILE_BYTES);
        if constexpr (TA == 32)
          tma_load_5d(slot_out, &mapS, &acc_bar[warp], 0, 0, 0, ca, cc0);
        else
          tma_load_3d(slot_out, &mapS, &acc_bar[warp], 16 * ca, 0, cc0);
      }
    }
    __syncwarp();
#pragma unroll 1
    for (int cc = 0; cc < TC; ++cc) {
      const uint8_t* X = Xs + b * Cfg::TILE_BYTES + cc * BOXB;
      uint8_t* D = slot_out + cc * BOXB;
      double acc[NF][FA][2];
#pragma unroll
      for (int nf = 0; nf < NF; ++nf)
#pragma unroll
        for (int f = 0; f < FA; ++f) acc[nf][f][0] = acc[nf][f][1] = 0.0;
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        double xf[FA];
#pragma unroll
        for (int f = 0; f < FA; ++f) {
          if constexpr (MODE1) {
            // A operand X(c = 8f + g, k = 4s + t), rows of P doubles
            xf[f] = *reinterpret_cast<const double*>(X + ((8 * f + g) * P + 4 * s + t) * 8);
          } else if constexpr (TA == 32) {
            // B operand X(k = 4s + t, a16 = 4f + xa, h = xh): row 2k + h, 128B swizzle
            xf[f] = *reinterpret_cast<const double*>(X + sw128_off(static_cast<uint32_t>(2 * (4 * s + t) + xh),
                                                                   static_cast<uint32_t>(4 * f + xa)));
          } else {
            // B operand X(k = 4s + t, a = skinny_col16(f, g)): row k, 128B swizzle
            xf[f] = *reinterpret_cast<const double*>(X + sw128_off(static_cast<uint32_t>(4 * s + t),
                                                                   static_cast<uint32_t>(skinny_col16(f, g))));
          }
        }
#pragma unroll
        for (int nf = 0; nf < NF; ++nf)
#pragma unroll
          for (int f = 0; f < FA; ++f) {
            if constexpr (MODE1)
              dmma_8x8x4(acc[nf][f][0], acc[nf][f][1], xf[f], lf[nf][s]);
            else
              dmma_8x8x4(acc[nf][f][0], acc[nf][f][1], lf[nf][s], xf[f]);
          }
      }
#pragma unroll
      for (int nf = 0; nf < NF; ++nf)
#pragma unroll
        for (int f = 0; f < FA; ++f) {
          uint32_t off;
          if constexpr (MODE1) {
            // D'[g -> c = 8f + g][n = 8nf + 2t + {0,1}]: rows of P doubles
            off = static_cast<uint32_t>(((8 * f + g) * P + 8 * nf + 2 * t) * 8);
          } else if constexpr (TA == 16) {
            // D[g -> n = 8nf + g][a = skinny_col16(f, 2t + {0,1})]: box row n
            off = sw128_off(static_cast<uint32_t>(8 * nf + g), static_cast<uint32_t>(skinny_col16(f, 2 * t)));
          } else {
            // D[g -> n = 8nf + g][a16 = 4f + 2(t>>1) + {0,1}, h = t&1]: box row 2n + h
            off = sw128_off(static_cast<uint32_t>(2 * (8 * nf + g) + (t & 1)),
                            static_cast<uint32_t>(4 * f + 2 * (t >> 1)));
          }
          if constexpr (ACC) {
            if (cc == 0 && nf == 0 && f == 0) mbar_wait(&acc_bar[warp], static_cast<uint32_t>(q & 1));
            const double2 o = *reinterpret_cast<const double2*>(D + off);
            *reinterpret_cast<double2*>(D + off) = make_double2(o.x + acc[nf][f][0], o.y + acc[nf][f][1]);
          } else {
            *reinterpret_cast<double2*>(D + off) = make_double2(acc[nf][f][0], acc[nf][f][1]);
          }
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[b]);  // the stage may be refilled
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      int32_t ca, cc0;
      coords(tile, ca, cc0);
      if constexpr (MODE1)
        tma_store_2d(&mapS, slot_out, 0, cc0);
      else if constexpr (TA == 32)
        tma_store_5d(&mapS, slot_out, 0, 0, 0, ca, cc0);
      else
        tma_store_3d(&mapS, slot_out, 16 * ca, 0, cc0);
      bulk_commit();
    }
  }
  if (lane == 0) bulk_wait_all();
}

// mu > 1 with a small leading extent A (even, <= 32; e.g. mode 2 of a
// 20^6 tensor, A = 20): a 32-a tile would be mostly padding, so a tile is TC
// whole c-slabs instead -- ONE 3-D box {A, P k, TC c} (no swizzle, a
// contiguous run of TC * A * K doubles; k >= K zero-filled) -- and the result
// leaves as ONE contiguous box {A, P n, TC c} (n >= N and c >= C clipped).
// Same warp-per-tile pipeline as skinny_kernel; per slab c the warp computes
// D_c(n, a) = L(n, k) X_c(k, a) with a-fragments of 8 consecutive a's.
template <int P, bool ACC = false>
__global__ void __launch_bounds__(SkinnyCfg<P>::THREADS, 1)
    skinny_slab_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapS,
                       const SkinnyParams p) {
  using Cfg = SkinnyCfg<P>;
  constexpr int NF = Cfg::NF, KS = Cfg::KS, W = Cfg::W, R = Cfg::R;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* Xs = smem;
  uint8_t* Stg = smem + W * R * Cfg::TILE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(Stg + W * Cfg::TILE_BYTES);
  uint64_t* empty_bar = full_bar + W * R;
  uint64_t* acc_bar = empty_bar + W * R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t tile_bytes = static_cast<uint32_t>(p.TC * P * p.A * 8);

  if (threadIdx.x == 0) {
    for (int b = 0; b < W * R; ++b) {
      mbar_init(&full_bar[b], 1);
      mbar_init(&empty_bar[b], 1);
    }
    for (int w = 0; w < W; ++w) mbar_init(&acc_bar[w], 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();

  if (warp == W) {
    if (lane == 0) {
      tma_prefetch_desc(&mapX);
      int64_t k = 0;
      for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x, ++k) {
        const int64_t q = k / W;
        const int b = static_cast<int>(k % W) * R + static_cast<int>(q % R);
        mbar_wait(&empty_bar[b], static_cast<uint32_t>((q / R) & 1) ^ 1);
        mbar_arrive_expect_tx(&full_bar[b], tile_bytes);
        tma_load_3d(Xs + b * Cfg::TILE_BYTES, &mapX, &full_bar[b], 0, 0, static_cast<int32_t>(tile * p.TC));
      }
    }
    return;
  }

  const int g = lane >> 2, t = lane & 3;
  double lf[NF][KS];
#pragma unroll
  for (int nf = 0; nf < NF; ++nf)
#pragma unroll
    for (int s = 0; s < KS; ++s) {
      const int n = 8 * nf + g, kk = 4 * s + t;
      lf[nf][s] = (n < p.N && kk < p.K) ? __ldg(p.L + n * p.sLi + kk * p.sLk) : 0.0;
    }
  const int A = p.A, AF = (A + 7) / 8;
  uint8_t* slot_out = Stg + warp * Cfg::TILE_BYTES;
  int64_t q = 0;
  for (int64_t tile = blockIdx.x + static_cast<int64_t>(warp) * gridDim.x; tile < p.tiles;
       tile += static_cast<int64_t>(W) * gridDim.x, ++q) {
    const int b = warp * R + static_cast<int>(q % R);
    mbar_wait(&full_bar[b], static_cast<uint32_t>((q / R) & 1));
    const double* X = reinterpret_cast<const double*>(Xs + b * Cfg::TILE_BYTES);
    if (lane == 0) bulk_wait_read_all();  // the staging buffer's previous store has read it
    if constexpr (ACC) {
      if (lane == 0) {
        mbar_arrive_expect_tx(&acc_bar[warp], tile_bytes);
        tma_load_3d(slot_out, &mapS, &acc_bar[warp], 0, 0, static_cast<int32_t>(tile * p.TC));
      }
      mbar_wait(&acc_bar[warp], static_cast<uint32_t>(q & 1));
    }
    __syncwarp();
    double* D = reinterpret_cast<double*>(slot_out);
    for (int cc = 0; cc < p.TC; ++cc) {
#pragma unroll
      for (int af = 0; af < 4; ++af) {
        if (af < AF) {
          double acc[NF][2];
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) acc[nf][0] = acc[nf][1] = 0.0;
#pragma unroll
          for (int s = 0; s < KS; ++s) {
            // B operand X_c(k = 4s + t, a = 8af + g) (a >= A: a neighbour's
            // value, only feeding output columns that are not stored)
            const double xf = X[(cc * P + 4 * s + t) * A + 8 * af + g];
#pragma unroll
            for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[nf][0], acc[nf][1], lf[nf][s], xf);
          }
          const int a = 8 * af + 2 * t;
          if (a < A) {
#pragma unroll
            for (int nf = 0; nf < NF; ++nf) {
              double2* o = reinterpret_cast<double2*>(D + (cc * P + 8 * nf + g) * A + a);
              if constexpr (ACC) {
                const double2 v = *o;
                *o = make_double2(v.x + acc[nf][0], v.y + acc[nf][1]);
              } else {
                *o = make_double2(acc[nf][0], acc[nf][1]);
              }
            }
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[b]);  // the stage may be refilled
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      tma_store_3d(&mapS, slot_out, 0, 0, static_cast<int32_t>(tile * p.TC));
      bulk_commit();
    }
  }
  if (lane == 0) bulk_wait_all();
}

}  // namespace mumode_gpu
