// Fused two-mode Tucker pass for small square modes (config C5: 24^6).
//
// With m = n = 24 a single mu-mode product does 48 flop per 16 B moved
// (3 flop/B, below the fp64 ridge of ~5.7), so six separate products are
// HBM-bound at <= 53 % of the roofline. This kernel applies two
// adjacent modes (mu, mu+1) per pass with the intermediate kept on chip:
// three HBM passes instead of six for an order-6 tensor.
//
//   FIRST == false (mu >= 2, A = prod_{k<mu} m_k, A % 8 == 0):
//     tile = 8 consecutive a's x all (b1, b2) for one c: ONE 4-D TMA box
//     {8, MU, MU, 1} -> smem [b2][b1][8a] (64B swizzle); mode mu contracts b1,
//     mode mu+1 contracts b2.
//   FIRST == true  (mu == 1, K-contiguous): tile = 8 consecutive c's x all
//     (j1, j2): ONE 3-D TMA box {8 k, 8*MU fibres, MU/8} -> smem
//     [k-block][fibre (j2,c)][8 k]; mode 1 contracts j1, mode 2 contracts j2.
//
// Both factor matrices live in registers for the whole kernel (DMMA
// fragments, (MU/8)*(MU/4) doubles each), so shared memory only carries the
// tensor. The mode-mu result goes to a padded shared buffer Y (one pad row
// per 64-B-row slab, software 64B swizzle) whose 16-byte writes and fragment
// reads are both bank-optimal; mode mu+1 reads Y and stores the final values
// straight to HBM as 16-byte stores. The tensor tile ring is 2-4 deep (as deep
// as shared memory allows): the producer warp keeps several TMA boxes in
// flight so HBM latency (each box row of the last pass of 24^6 lies 2.65 MB
// from the next) is covered while earlier tiles compute and store.
#pragma once
#include "common.cuh"

namespace mumode_gpu {

// RA = a's per tile for FIRST == false (8 or 16: 16 halves the number of
// scattered 64-B box rows per byte when the a-stride is large).
template <int MU, bool FIRST, int RA = 8>
struct FusedCfg {
  static constexpr int NF = MU / 8;   // 8-wide output fragments per mode
  static constexpr int KS = MU / 4;   // k-steps per contraction
  static constexpr int AH = FIRST ? 1 : RA / 8;  // 8-a halves per tile
  static constexpr int UNITS = MU * AH;          // units per mode (UNITS / WARPS per warp)
  // consumer warps: 12 where the units split evenly (MU = 24: pass 1 of C5
  // 600 -> 580 us, pass 2 649 -> 614 us), else 8; one producer warp. (A
  // 4-warp producer group donating registers via setmaxnreg was slower.)
  static constexpr int WARPS = (UNITS % 12 == 0) ? 12 : 8;
  static constexpr int THREADS = (WARPS + 1) * 32;
  static constexpr int X_BYTES = 8 * AH * MU * MU * 8;
  static constexpr int Y_ROWS = (FIRST ? 8 * NF : AH * MU) * (MU + 1);
  static constexpr int Y_BYTES = Y_ROWS * 64;
  // tensor-tile ring depth: enough bytes in flight per SM to cover HBM latency
  // (Little's law: ~90 KB at ~2 us), within the 227 KB shared-memory limit
  static constexpr int NBUF = (4 * X_BYTES + Y_BYTES + 2048 <= 227 * 1024) ? 4
                              : (3 * X_BYTES + Y_BYTES + 2048 <= 227 * 1024) ? 3 : 2;
  static constexpr int SMEM_BYTES = NBUF * X_BYTES + Y_BYTES + 1024 + 128;
  static_assert(MU % 8 == 0 && MU >= 8 && MU <= 32, "square modes of 8..32");
  static_assert(RA == 8 || RA == 16, "8 or 16 a's per tile");
};

struct FusedParams {
  double* S;
  const double* L1;  // mode mu factor, MU x MU column-major
  const double* L2;  // mode mu+1 factor
  int64_t A;         // prod of extents before mu (1 when FIRST)
  int64_t C;         // prod of extents after mu+1
  int64_t tiles;
};

// Y element (row r, x) -> byte offset: 64-B rows, 16-B chunk (x>>1) ^ ((r>>1)&3)
__device__ __forceinline__ uint32_t y_off(int r, int x) {
  return static_cast<uint32_t>(r * 64 + ((((x >> 1) ^ ((r >> 1) & 3))) << 4) + (x & 1) * 8);
}

template <int MU, bool FIRST, int RA>
__global__ void __launch_bounds__(FusedCfg<MU, FIRST, RA>::THREADS, 1)
    fused_pair_kernel(const __grid_constant__ CUtensorMap mapX, const FusedParams p) {
  using Cfg = FusedCfg<MU, FIRST, RA>;
  constexpr int AH = Cfg::AH;
  constexpr int NF = Cfg::NF, KS = Cfg::KS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int NBUF = Cfg::NBUF;
  uint8_t* Y = smem + NBUF * Cfg::X_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(Y + Cfg::Y_BYTES);
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
      const int64_t ablks = FIRST ? 1 : p.A / RA;
      for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
        mbar_wait(&empty_bar[buf], phase ^ 1);
        mbar_arrive_expect_tx(&full_bar[buf], Cfg::X_BYTES);
        uint8_t* dst = smem + buf * Cfg::X_BYTES;
        if constexpr (FIRST) {
          tma_load_3d(dst, &mapX, &full_bar[buf], 0, static_cast<int32_t>(tile * 8 * MU), 0);
        } else {
          const int64_t c = tile / ablks, ab = tile - c * ablks;
#pragma unroll
          for (int hh = 0; hh < AH; ++hh)
            tma_load_4d(dst + hh * (MU * MU * 64), &mapX, &full_bar[buf], static_cast<int32_t>(RA * ab + 8 * hh), 0,
                        0, static_cast<int32_t>(c));
        }
        if (++buf == NBUF) {
          buf = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int g = lane >> 2, t = lane & 3;
  const int jg = 2 * ((g >> 1) & 1) + (g >> 2);
  const uint32_t J0 = static_cast<uint32_t>(jg ^ (t >> 1)) << 4;
  const uint32_t xk_off = static_cast<uint32_t>(t * 64 + (g & 1) * 8);
  const uint32_t kx_off = static_cast<uint32_t>(xmap8(g) * 64 + (t & 1) * 8);

  // factor fragments, resident for the whole kernel.
  //   FIRST mode 1: L1 is the B operand  B[t][g] = L1(8nf + xmap8(g), 4s + t)
  //   otherwise:    L  is the A operand  A[g][t] = L (8nf + g,        4s + t)
  double l1[NF][KS], l2[NF][KS];
#pragma unroll
  for (int nf = 0; nf < NF; ++nf)
#pragma unroll
    for (int s = 0; s < KS; ++s) {
      const int row1 = FIRST ? 8 * nf + xmap8(g) : 8 * nf + g;
      l1[nf][s] = p.L1[row1 + (4 * s + t) * MU];
      l2[nf][s] = p.L2[(8 * nf + g) + (4 * s + t) * MU];
    }

  int buf = 0;
  uint32_t phase = 0;
  const int64_t ablks = FIRST ? 1 : p.A / RA;
  for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
    mbar_wait(&full_bar[buf], phase);
    const uint8_t* X = smem + buf * Cfg::X_BYTES;

    // ---- mode mu: X -> Y. For FIRST a warp's UPW (3) units advance together
    // (9 independent accumulator chains hide the DMMA latency: pass 1 of C5
    // 619 -> 602 us); with 16-wide a tiles (6 units) that costs more than it
    // hides, so the others go one unit at a time.
    constexpr int GROUP = FIRST ? Cfg::UNITS / Cfg::WARPS : 1;
#pragma unroll
    for (int grp = 0; grp < (Cfg::UNITS / Cfg::WARPS) / GROUP; ++grp) {
      constexpr int UPW = GROUP;
      double acc[UPW][NF][2];
#pragma unroll
      for (int uu = 0; uu < UPW; ++uu)
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) acc[uu][nf][0] = acc[uu][nf][1] = 0.0;
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        const uint32_t Js = J0 ^ (32u * static_cast<uint32_t>(s & 1));
#pragma unroll
        for (int uu = 0; uu < UPW; ++uu) {
          const int u = warp + Cfg::WARPS * (grp * GROUP + uu);  // FIRST: fibre fragment; else (a-half, b2)
          if constexpr (FIRST) {
            // A = X^T fragment (fibres 8u + xmap8(g), k = 4s + t), KX layout
            const double xf = *reinterpret_cast<const double*>(X + (s >> 1) * (8 * MU * 64) + (8 * u) * 64 +
                                                               kx_off + Js);
#pragma unroll
            for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[uu][nf][0], acc[uu][nf][1], xf, l1[nf][s]);
          } else {
            // B = X fragment (k = b1 = 4s + t, a = xmap8(g)) in slab (a-half, b2) = u, XK layout
            const double xf = *reinterpret_cast<const double*>(X + u * (MU * 64) + (4 * s) * 64 + xk_off + Js);
#pragma unroll
            for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[uu][nf][0], acc[uu][nf][1], l1[nf][s], xf);
          }
        }
      }
#pragma unroll
      for (int uu = 0; uu < UPW; ++uu) {
        const int u = warp + Cfg::WARPS * (grp * GROUP + uu);
        if constexpr (FIRST) {
          // D[g <-> fibre f = 8u + xmap8(g)][i pair = 8nf + xmap8(2t)] -> Y row (cl, nf, j2)
          const int f = 8 * u + xmap8(g);
          const int j2 = f % MU, cl = f / MU;
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) {
            const int r = (cl * NF + nf) * (MU + 1) + j2;
            *reinterpret_cast<double2*>(Y + y_off(r, xmap8(2 * t))) = make_double2(acc[uu][nf][0], acc[uu][nf][1]);
          }
        } else {
          // D[g <-> i = 8nf + g][a pair = xmap8(2t)] -> Y row (a-half, i, b2)
          const int ah = u / MU, b2 = u % MU;
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) {
            const int r = (ah * MU + 8 * nf + g) * (MU + 1) + b2;
            *reinterpret_cast<double2*>(Y + y_off(r, xmap8(2 * t))) = make_double2(acc[uu][nf][0], acc[uu][nf][1]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[buf]);  // X[buf] may be refilled
    named_barrier_sync(1, Cfg::WARPS * 32);         // Y complete

    // ---- mode mu+1: Y -> HBM
    int64_t c_base = 0, a_base = 0;
    if constexpr (FIRST) {
      c_base = tile * 8;
    } else {
      c_base = tile / ablks;
      a_base = RA * (tile - c_base * ablks);
    }
    // one unit at a time here: advancing FIRST's three units together
    // bunches their 16-B store bursts (pass 1 of C5 602 -> 688 us)
    constexpr int GROUP2 = 1;
#pragma unroll
    for (int grp = 0; grp < (Cfg::UNITS / Cfg::WARPS) / GROUP2; ++grp) {
      constexpr int UPW = GROUP2;
      double acc[UPW][NF][2];
#pragma unroll
      for (int uu = 0; uu < UPW; ++uu)
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) acc[uu][nf][0] = acc[uu][nf][1] = 0.0;
#pragma unroll
      for (int s = 0; s < KS; ++s)
#pragma unroll
        for (int uu = 0; uu < UPW; ++uu) {
          const int u = warp + Cfg::WARPS * (grp * GROUP2 + uu);  // FIRST: (cl, ib) = (u / NF, u % NF); else (a-half, i)
          const double yf = *reinterpret_cast<const double*>(Y + y_off(u * (MU + 1) + 4 * s + t, xmap8(g)));
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[uu][nf][0], acc[uu][nf][1], l2[nf][s], yf);
        }
      const int x = xmap8(2 * t);  // output pair along the contiguous index
#pragma unroll
      for (int uu = 0; uu < UPW; ++uu) {
        const int u = warp + Cfg::WARPS * (grp * GROUP2 + uu);
        if constexpr (FIRST) {
          const int cl = u / NF, ib = u % NF;
          const int64_t c = c_base + cl;
          if (c < p.C) {
#pragma unroll
            for (int nf = 0; nf < NF; ++nf) {
              const int j = 8 * nf + g;
              stg_f64x2(p.S + (8 * ib + x) + static_cast<int64_t>(MU) * (j + static_cast<int64_t>(MU) * c),
                        acc[uu][nf][0], acc[uu][nf][1]);
            }
          }
        } else {
          const int ah = u / MU, i = u % MU;
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) {
            const int j = 8 * nf + g;
            stg_f64x2(p.S + a_base + 8 * ah + x +
                          p.A * (i + static_cast<int64_t>(MU) * (j + static_cast<int64_t>(MU) * c_base)),
                      acc[uu][nf][0], acc[uu][nf][1]);
          }
        }
      }
    }
    named_barrier_sync(1, Cfg::WARPS * 32);  // Y free for the next tile
    if (++buf == NBUF) {
      buf = 0;
      phase ^= 1;
    }
  }
}

}  // namespace mumode_gpu
