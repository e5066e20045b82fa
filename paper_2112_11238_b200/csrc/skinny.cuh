// Mode products with small extents (K = m_mu <= 32, N = n_mu <= 32): the
// products of high-order tensors with small modes (the paper's d = 6, n = 12..20
// Tucker benchmarks; any single mode product of a 24^6 tensor).
//
// Such a product does 2N flop per 16 B moved: HBM-bound. The tile kernels of
// tma_dmma.cuh stage it as 8-row (64-B) boxes of a large M tile and reach
// 1.4-3.9 TB/s on 12^6..24^6. Here every tile is small and moves 256-B rows:
//
//   mu > 1: tile = 32 consecutive a's x all K x one c. ONE 4-D TMA box
//           {16 a, 2, P k, 1} (128B swizzle, every k row one 256-B run) in,
//           D(n, a) = L(n, k) X(k, a) on DMMA, the 32 x N result staged in
//           TMA-box layout and written by ONE TMA store {16, 2, P n, 1}.
//   mu = 1: tile = 32 consecutive fibres c (contiguous 32 K doubles): box
//           {P k, 32 c} in (no swizzle), D'(c, n) = X(c, k) L(n, k)^T, the
//           32 x N result (contiguous) out by one TMA store {P n, 32 c}.
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

// TA = a's (mu > 1) or fibres (mu = 1) per tile: 32, or 16 for mu > 1 when
// A is not a multiple of 16 (then the 4-D {16, A/16, ...} view does not
// exist; 128-B rows of a 3-D {A, K, C} view instead -- such A are small, so
// the rows of a tile lie close together).
template <int P, int TA = 32>
struct SkinnyCfg {
  static constexpr int NF = P / 8;  // 8-wide output fragments
  static constexpr int KS = P / 4;  // k-steps
  static constexpr int FA = TA / 8; // 8-wide a fragments
  static constexpr int W = 8;       // consumer warps
  static constexpr int THREADS = (W + 1) * 32;
  static constexpr int TILE_BYTES = TA * P * 8;  // one stage (and one staged result)
  static constexpr int R_RAW = (227 * 1024 - 1024 - 256) / (W * TILE_BYTES) - 1;
  static constexpr int R = R_RAW > 4 ? 4 : R_RAW;  // stages per warp
  static constexpr int SMEM_BYTES = W * (R + 1) * TILE_BYTES + 1024 + 2 * W * R * 8 + 64;
  static_assert(P % 8 == 0 && P >= 8 && P <= 32, "P in 8..32");
  static_assert(TA == 32 || TA == 16, "32- or 16-wide tiles");
  static_assert(R >= 2, "shared memory for 2 stages per warp");
  static_assert(TILE_BYTES % 1024 == 0, "128B-swizzle atoms");
};

struct SkinnyParams {
  const double* L;
  int64_t sLi, sLk;  // op(L)(n, k) = L[n * sLi + k * sLk]
  int K, N;
  int64_t ablks;     // mu > 1: ceil(A / TA)
  int64_t tiles;
};

// 16-wide a tiles: fragment column n of a-fragment f -> a = 4f + (n&1) +
// 8((n>>1)&1) + 2(n>>2), so the 8 (k, a-pair) chunks a half-warp loads hit 8
// distinct 16-B bank groups of the 128B-swizzled k rows.
__device__ __forceinline__ int skinny_col16(int f, int n) { return 4 * f + (n & 1) + 8 * ((n >> 1) & 1) + 2 * (n >> 2); }

template <int P, bool MODE1, int TA = 32>
__global__ void __launch_bounds__(SkinnyCfg<P, TA>::THREADS, 1)
    skinny_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapS,
                  const SkinnyParams p) {
  using Cfg = SkinnyCfg<P, TA>;
  constexpr int NF = Cfg::NF, KS = Cfg::KS, FA = Cfg::FA, W = Cfg::W, R = Cfg::R;
  static_assert(!MODE1 || TA == 32, "mode 1 uses 32-fibre tiles");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* Xs = smem;                                   // [warp][stage]
  uint8_t* Stg = smem + W * R * Cfg::TILE_BYTES;        // [warp]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(Stg + W * Cfg::TILE_BYTES);
  uint64_t* empty_bar = full_bar + W * R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int b = 0; b < W * R; ++b) {
      mbar_init(&full_bar[b], 1);
      mbar_init(&empty_bar[b], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();  // before any global access (factor included)

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
        if constexpr (MODE1) {
          tma_load_2d(dst, &mapX, &full_bar[b], 0, static_cast<int32_t>(32 * tile));
        } else if constexpr (TA == 32) {
          const int64_t c = tile / p.ablks, ab = tile - c * p.ablks;
          tma_load_4d(dst, &mapX, &full_bar[b], 0, static_cast<int32_t>(2 * ab), 0, static_cast<int32_t>(c));
        } else {
          const int64_t c = tile / p.ablks, ab = tile - c * p.ablks;
          tma_load_3d(dst, &mapX, &full_bar[b], static_cast<int32_t>(16 * ab), 0, static_cast<int32_t>(c));
        }
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
    const uint8_t* X = Xs + b * Cfg::TILE_BYTES;
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
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&empty_bar[b]);  // the stage may be refilled
      bulk_wait_read_all();        // the staging buffer's previous store has read it
    }
    __syncwarp();
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
        *reinterpret_cast<double2*>(slot_out + off) = make_double2(acc[nf][f][0], acc[nf][f][1]);
      }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      if constexpr (MODE1) {
        tma_store_2d(&mapS, slot_out, 0, static_cast<int32_t>(32 * tile));
      } else if constexpr (TA == 32) {
        const int64_t c = tile / p.ablks, ab = tile - c * p.ablks;
        tma_store_4d(&mapS, slot_out, 0, static_cast<int32_t>(2 * ab), 0, static_cast<int32_t>(c));
      } else {
        const int64_t c = tile / p.ablks, ab = tile - c * p.ablks;
        tma_store_3d(&mapS, slot_out, static_cast<int32_t>(16 * ab), 0, static_cast<int32_t>(c));
      }
      bulk_commit();
    }
  }
  if (lane == 0) bulk_wait_all();
}

}  // namespace mumode_gpu
