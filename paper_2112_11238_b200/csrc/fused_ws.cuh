// Warp-specialised first fused two-mode pass (modes 1 and 2; same
// contraction, tiles, Y layout and fragment maps as fused_pair_kernel<MU,
// true> in fused.cuh).
//
// fused_pair_kernel runs both modes of a tile on all consumer warps, split by
// two CTA-wide barriers per tile (Y complete, Y free): every tile the DMMA
// pipe drains at each barrier (ncu on C5 pass 1: DMMA pipe 87 % of active
// cycles). Here two warp groups run the two modes concurrently on
// consecutive tiles through a double-buffered Y:
//
//   group 0 (GW warps): mode 1   X ring -> Y[k & 1]   (waits: X full, Y free)
//   group 1 (GW warps): mode 2   Y[k & 1] -> HBM        (waits: Y full)
//
// Y handoffs are named barriers (bar.arrive by the writer group, bar.sync by
// the reader group; ids 2 + yb "Y full", 2 + NY + yb "Y free"). bar.arrive
// orders prior shared WRITES only, so group 1 frees Y[yb] after a shared
// store that depends on every value it loaded from it (loads complete,
// DMMAs may follow); freeing it only after the global stores cost 545 ->
// 590 us on C5 pass 1, a fence 557 -> 586 us. Group 0 skips the "Y free"
// wait for its first two tiles and group 1 skips the "Y free" arrival for its
// last two, so every barrier instance completes. Each group holds only its
// own factor's fragments. Measured on C5 (24^6) pass 1: 581 -> 564 us, DMMA
// pipe 87 % -> 89 % of active cycles (ncu). For the strided middle pass the
// same split with 8-a tiles was slower than fused_pair_kernel's 16-a tiles
// (two Y buffers leave no room for 16-a tiles), so it is not used there.
#pragma once
#include "common.cuh"
#include "fused.cuh"

namespace mumode_gpu {

template <int MU, int NY_ = 2>
struct FusedWsCfg {
  using Base = FusedCfg<MU, true, 8>;
  static constexpr int NF = MU / 8;
  static constexpr int KS = MU / 4;
  static constexpr int UNITS = MU;                  // units per mode per tile
  static constexpr int GW = (MU % 6 == 0) ? 6 : 4;  // warps per mode group
  static constexpr int UPW = UNITS / GW;            // units per warp
  static constexpr int THREADS = (2 * GW + 1) * 32;
  static constexpr int X_BYTES = Base::X_BYTES;
  static constexpr int Y_BYTES = Base::Y_BYTES;
  // Y buffers between the groups (C5 pass 1: 2 -> 545 us with a 4-deep ring,
  // 3 -> 551 us with a 3-deep ring)
  static constexpr int NY = NY_;
  static constexpr int NBUF = (4 * X_BYTES + NY * Y_BYTES + 2048 + GW * 256 <= 227 * 1024) ? 4
                              : (3 * X_BYTES + NY * Y_BYTES + 2048 + GW * 256 <= 227 * 1024) ? 3 : 2;
  static constexpr int SMEM_BYTES = NBUF * X_BYTES + NY * Y_BYTES + 1024 + 128 + GW * 32 * 8;
  static_assert(MU == 8 || MU == 16 || MU == 24, "square modes of 8, 16, 24");
  static_assert(UNITS % GW == 0, "units split evenly over a group");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory");
};

// GA = mode-1 units a warp advances together (independent accumulator chains)
template <int MU, int GA, int NY>
__global__ void __launch_bounds__(FusedWsCfg<MU, NY>::THREADS, 1)
    fused_ws_kernel(const __grid_constant__ CUtensorMap mapX, const FusedParams p) {
  using Cfg = FusedWsCfg<MU, NY>;
  constexpr int NF = Cfg::NF, KS = Cfg::KS, GW = Cfg::GW, UPW = Cfg::UPW, NBUF = Cfg::NBUF;
  constexpr int PAIR = 2 * GW * 32;  // threads of both groups
  static_assert(UPW % GA == 0, "group-0 unit batches");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* Ybase = smem + NBUF * Cfg::X_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(Ybase + NY * Cfg::Y_BYTES);
  uint64_t* empty_bar = full_bar + NBUF;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // per group-1 warp: 32 words the "Y free" dependency stores go to
  uint64_t* scratch = empty_bar + NBUF + 32 * (warp % Cfg::GW);

  if (threadIdx.x == 0) {
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(&full_bar[b], 1);
      mbar_init(&empty_bar[b], GW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();  // before any global access (factors included)

  if (warp == 2 * GW) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      tma_prefetch_desc(&mapX);
      int buf = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
        mbar_wait(&empty_bar[buf], phase ^ 1);
        mbar_arrive_expect_tx(&full_bar[buf], Cfg::X_BYTES);
        tma_load_3d(smem + buf * Cfg::X_BYTES, &mapX, &full_bar[buf], 0, static_cast<int32_t>(tile * 8 * MU), 0);
        if (++buf == NBUF) {
          buf = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }

  const int grp = warp / GW, w = warp - grp * GW;
  const int g = lane >> 2, t = lane & 3;
  const int64_t ntiles = (p.tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;  // tiles of this CTA

  if (grp == 0) {
    // ----------------------------------------------------- mode 1: X -> Y
    const int jg = 2 * ((g >> 1) & 1) + (g >> 2);
    const uint32_t J0 = static_cast<uint32_t>(jg ^ (t >> 1)) << 4;
    const uint32_t kx_off = static_cast<uint32_t>(xmap8(g) * 64 + (t & 1) * 8);
    double l1[NF][KS];
#pragma unroll
    for (int nf = 0; nf < NF; ++nf)
#pragma unroll
      for (int s = 0; s < KS; ++s) l1[nf][s] = p.L1[(8 * nf + xmap8(g)) + (4 * s + t) * MU];  // B operand

    int buf = 0;
    uint32_t phase = 0;
    for (int64_t k = 0; k < ntiles; ++k) {
      const int yb = static_cast<int>(k % NY);
      uint8_t* Y = Ybase + yb * Cfg::Y_BYTES;
      mbar_wait(&full_bar[buf], phase);
      if (k >= NY) named_barrier_sync(2 + NY + yb, PAIR);  // Y[yb] read by group 1
      const uint8_t* X = smem + buf * Cfg::X_BYTES;
#pragma unroll
      for (int bt = 0; bt < UPW / GA; ++bt) {
        double acc[GA][NF][2];
#pragma unroll
        for (int uu = 0; uu < GA; ++uu)
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) acc[uu][nf][0] = acc[uu][nf][1] = 0.0;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          const uint32_t Js = J0 ^ (32u * static_cast<uint32_t>(s & 1));
#pragma unroll
          for (int uu = 0; uu < GA; ++uu) {
            const int u = w + GW * (bt * GA + uu);  // fibre fragment
            // A = X^T fragment (fibres 8u + xmap8(g), k = 4s + t), KX layout
            const double xf =
                *reinterpret_cast<const double*>(X + (s >> 1) * (8 * MU * 64) + (8 * u) * 64 + kx_off + Js);
#pragma unroll
            for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[uu][nf][0], acc[uu][nf][1], xf, l1[nf][s]);
          }
        }
#pragma unroll
        for (int uu = 0; uu < GA; ++uu) {
          const int u = w + GW * (bt * GA + uu);
          // D[g <-> fibre f = 8u + xmap8(g)][i pair = 8nf + xmap8(2t)] -> Y row (cl, nf, j2)
          const int f = 8 * u + xmap8(g);
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) {
            const int r = ((f / MU) * NF + nf) * (MU + 1) + f % MU;
            *reinterpret_cast<double2*>(Y + y_off(r, xmap8(2 * t))) = make_double2(acc[uu][nf][0], acc[uu][nf][1]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[buf]);  // X[buf] may be refilled
      named_barrier_arrive(2 + yb, PAIR);            // Y[yb] complete
      if (++buf == NBUF) {
        buf = 0;
        phase ^= 1;
      }
    }
    return;
  }

  // ------------------------------------------------------- mode 2: Y -> HBM
  double l2[NF][KS];
#pragma unroll
  for (int nf = 0; nf < NF; ++nf)
#pragma unroll
    for (int s = 0; s < KS; ++s) l2[nf][s] = p.L2[(8 * nf + g) + (4 * s + t) * MU];
  const int x = xmap8(2 * t);  // output pair along the contiguous index
  for (int64_t k = 0; k < ntiles; ++k) {
    const int64_t c_base = (blockIdx.x + k * gridDim.x) * 8;
    const int yb = static_cast<int>(k % NY);
    const uint8_t* Y = Ybase + yb * Cfg::Y_BYTES;
    named_barrier_sync(2 + yb, PAIR);  // Y[yb] complete
#pragma unroll
    for (int q = 0; q < UPW; ++q) {
      const int u = w + GW * q;  // (cl, ib) = (u / NF, u % NF)
      double yf[KS];
#pragma unroll
      for (int s = 0; s < KS; ++s)
        yf[s] = *reinterpret_cast<const double*>(Y + y_off(u * (MU + 1) + 4 * s + t, xmap8(g)));
      if (q == UPW - 1 && k + NY < ntiles) {
        // free Y[yb] as soon as the last unit's loads are complete: a shared
        // store that depends on every loaded value (bar.arrive keeps it
        // before the arrive; ptxas cannot sink it like a DMMA)
        uint64_t dep = 0;
#pragma unroll
        for (int s = 0; s < KS; ++s) dep ^= static_cast<uint64_t>(__double_as_longlong(yf[s]));
        *reinterpret_cast<volatile uint64_t*>(scratch + lane) = dep;
        named_barrier_arrive(2 + NY + yb, PAIR);
      }
      double acc[NF][2];
#pragma unroll
      for (int nf = 0; nf < NF; ++nf) acc[nf][0] = acc[nf][1] = 0.0;
#pragma unroll
      for (int s = 0; s < KS; ++s)
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[nf][0], acc[nf][1], l2[nf][s], yf[s]);
      const int cl = u / NF, ib = u % NF;
      const int64_t c = c_base + cl;
      if (c < p.C) {
#pragma unroll
        for (int nf = 0; nf < NF; ++nf)
          stg_f64x2(p.S + (8 * ib + x) + static_cast<int64_t>(MU) * ((8 * nf + g) + static_cast<int64_t>(MU) * c),
                    acc[nf][0], acc[nf][1]);
      }
    }
  }
}

}  // namespace mumode_gpu
