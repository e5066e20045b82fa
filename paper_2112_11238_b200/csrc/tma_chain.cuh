// Persistent chain kernel: all modes of one Tucker application in ONE launch.
//
// Each mode of a Tucker chain is a separate persistent launch otherwise; every
// launch pays a ramp (first TMA loads) and a last-wave tail (tiles % SMs), and
// ncu shows 92-95 % DMMA-active inside the kernels but only 84-91 % of the
// elapsed time (C3: 200^3). Here the CTAs walk one global item list -- mode
// 1's tiles, then mode 2's, ... -- so a CTA that finishes its share of mode mu
// immediately starts mode mu+1 tiles whose inputs are ready.
//
// Readiness is tracked per consumer M-tile: the host (chain.cuh) maps every
// producer tile's output region to the consumer M-tiles that read it; after a
// producer tile's epilogue the MMA warps only bar.arrive (they never wait),
// and a publisher warp of the producer group bar.syncs, fences and increments
// the listed counters with relaxed reductions over its lanes; the consumer's TMA lane spins (ld.acquire.gpu, nanosleep, trap
// after 2^26 polls) until its M-tile counter reaches the host-computed target,
// then fences the async proxy and issues the loads. Items are processed in
// increasing global order by every CTA and depend only on earlier items, so
// the smallest unfinished item is always ready (no deadlock with a persistent
// grid of at most one CTA per SM).
//
// The smem ring, its barriers and the (stage, phase) counters continue across
// modes; mode 1 (QK) uses tile config CfgA, the other modes CfgB (same
// thread count, ring geometry and register split).
#pragma once
#include "tma_dmma.cuh"

namespace mumode_gpu {

constexpr int kChainMaxModes = 8;
constexpr int kChainPubSlots = 4;  // publisher hand-off ring depth
constexpr int kChainExtraSmem = 2 * kChainPubSlots * 8;

struct ChainMaps {
  CUtensorMap P[kChainMaxModes];
  CUtensorMap Q[kChainMaxModes];
};

struct ChainPhase {
  TmaParams p;
  int64_t base;            // first global item of this mode
  int n_major;             // tile order for mu > 1: 1 = N-tile slowest
  int* wait_ctr;           // mu > 1: one counter per M-tile (device)
  const int* wait_target;  // ... and its target
  const int* sig_off;      // mu < last: CSR offsets per tile into sig_idx
  const int* sig_idx;      // counter indices of the next mode (its wait_ctr)
  int* sig_ctr;            // = next mode's wait_ctr
};

struct ChainParams {
  int nphases;
  int64_t total;
  ChainPhase ph[kChainMaxModes];
};

__device__ __forceinline__ void chain_wait(const int* ctr, int target) {
  uint32_t polls = 0;
  int v;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory");
    if (v >= target) break;
    __nanosleep(32);
    if (++polls == (1u << 26)) __trap();
  }
  // the producers wrote through the generic proxy; our loads are TMA
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

// after a fence: the reductions themselves need no release semantics
__device__ __forceinline__ void chain_signal(int* ctr) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;\n" ::"l"(ctr) : "memory");
}

template <class CfgA, class CfgB>
__global__ void __launch_bounds__(CfgB::THREADS, 1)
    tucker_chain_kernel(const __grid_constant__ ChainMaps maps, const __grid_constant__ ChainParams cp) {
  static_assert(CfgA::THREADS == CfgB::THREADS && CfgA::STAGES == CfgB::STAGES &&
                    CfgA::STAGE_BYTES == CfgB::STAGE_BYTES && CfgA::MMA_WARPS == CfgB::MMA_WARPS &&
                    CfgA::E == CfgB::E && CfgA::LAUNCH_REGS == CfgB::LAUNCH_REGS,
                "chain configs must share the CTA shape and the ring");
  using Cfg = CfgB;
  // the producer group runs the TMA lane AND the publisher loop here: more
  // registers than the single-mode kernel gives it (24)
  constexpr int PREGS = 40;
  constexpr int CREGS_RAW = ((Cfg::LAUNCH_REGS * Cfg::THREADS - 4 * 32 * PREGS) / (Cfg::MMA_WARPS * 32)) / 8 * 8;
  constexpr int CREGS = CREGS_RAW > 232 ? 232 : CREGS_RAW;
  static_assert(CREGS >= Cfg::LAUNCH_REGS, "setmaxnreg.inc must not shrink");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + Cfg::STAGES;
  // publisher hand-off ring: the MMA warps report a finished producer tile in
  // slot j % NB (pub_full), the publisher frees the slot after signalling
  // (pub_empty). Flow-controlled: with named barriers the MMA warps could
  // lap the publisher on short tiles (K = 24..32) and corrupt the barrier
  // count -- a deadlock that ended in the watchdog trap (32^5, policy 11).
  constexpr int NB = kChainPubSlots;
  uint64_t* pub_full = empty_bar + Cfg::STAGES;
  uint64_t* pub_empty = pub_full + NB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], Cfg::MMA_WARPS);
    }
    for (int s = 0; s < NB; ++s) {
      mbar_init(&pub_full[s], Cfg::MMA_WARPS);
      mbar_init(&pub_empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  // No programmatic dependent launch here: the CTAs wait on each other's
  // tiles, so all of them must become resident. An early-launched successor
  // grid could take the SMs of CTAs not yet scheduled and spin in its own
  // griddepcontrol.wait until this grid ends -- a deadlock (seen as the
  // watchdog trap in a long test session). Launched as a plain kernel, it
  // starts after its predecessor and releases its successor only at exit.

  // item -> (mode, tile, M-tile, N-tile); items only increase per CTA
  auto locate = [&](int64_t item, int& ph, int& mt, int& nt) {
    while (ph + 1 < cp.nphases && item >= cp.ph[ph + 1].base) ++ph;
    const ChainPhase& P = cp.ph[ph];
    const int64_t tile = item - P.base;
    if (ph == 0) {  // QK: m fastest
      mt = static_cast<int>(tile % P.p.mt);
      nt = static_cast<int>(tile / P.p.mt);
    } else if (P.n_major) {
      mt = static_cast<int>(tile % P.p.mt);
      nt = static_cast<int>(tile / P.p.mt);
    } else {
      nt = static_cast<int>(tile % P.p.nt);
      mt = static_cast<int>(tile / P.p.nt);
    }
  };
  int stage = 0;
  uint32_t phase = 0;
  if (warp >= Cfg::MMA_WARPS) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PREGS) : "memory");
    if (warp == Cfg::MMA_WARPS + 1) {
      // publisher: after the MMA warps' arrival for a producer tile (its
      // epilogue stores issued), fence and increment the listed counters;
      // the MMA warps never wait for this
      int ph = 0;
      int64_t j = 0;
      for (int64_t item = blockIdx.x; item < cp.total; item += gridDim.x, ++j) {
        while (ph + 1 < cp.nphases && item >= cp.ph[ph + 1].base) ++ph;
        if (ph + 1 == cp.nphases) break;
        const ChainPhase& P = cp.ph[ph];
        const int slot = static_cast<int>(j % NB);
        mbar_wait(&pub_full[slot], static_cast<uint32_t>((j / NB) & 1));
        __threadfence();
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        const int64_t tile = item - P.base;
        for (int k = P.sig_off[tile] + lane; k < P.sig_off[tile + 1]; k += 32) chain_signal(P.sig_ctr + P.sig_idx[k]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&pub_empty[slot]);
      }
    }
    if (warp == Cfg::MMA_WARPS && lane == 0) {
      int ph = 0;
      for (int64_t item = blockIdx.x; item < cp.total; item += gridDim.x) {
        int mt, nt;
        locate(item, ph, mt, nt);
        const ChainPhase& P = cp.ph[ph];
        if (ph == 0) {
          tma_produce_tile<CfgA, true>(&maps.P[0], &maps.Q[0], P.p, mt, nt, smem, full_bar, empty_bar, stage,
                                       phase);
        } else {
          chain_wait(P.wait_ctr + mt, P.wait_target[mt]);
          tma_produce_tile<CfgB, false>(&maps.P[ph], &maps.Q[ph], P.p, mt, nt, smem, full_bar, empty_bar, stage,
                                        phase);
        }
      }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CREGS) : "memory");
  const FragOffsets foA = tma_frag_offsets<CfgA>(warp, lane);
  const FragOffsets foB = tma_frag_offsets<CfgB>(warp, lane);
  int ph = 0;
  int64_t j = 0;
  for (int64_t item = blockIdx.x; item < cp.total; item += gridDim.x, ++j) {
    int mt, nt;
    locate(item, ph, mt, nt);
    const ChainPhase& P = cp.ph[ph];
    if (ph == 0)
      tma_consume_tile<CfgA, true, 0>(P.p, mt, nt, smem, full_bar, empty_bar, stage, phase, foA, lane);
    else
      tma_consume_tile<CfgB, false, 0>(P.p, mt, nt, smem, full_bar, empty_bar, stage, phase, foB, lane);
    if (ph + 1 < cp.nphases) {  // the tile's stores are issued: hand it to the publisher
      const int slot = static_cast<int>(j % NB);
      mbar_wait(&pub_empty[slot], static_cast<uint32_t>((j / NB) & 1) ^ 1);  // the slot's last use is published
      asm volatile("fence.acq_rel.cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&pub_full[slot]);
    }
  }
}

}  // namespace mumode_gpu
