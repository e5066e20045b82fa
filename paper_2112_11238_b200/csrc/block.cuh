// K9 — in-place block passes for small square extents (the paper's d = 6
// sizes n = 12..20): up to THREE consecutive modes of a Tucker chain per HBM
// pass, with the whole block of the tensor those modes touch resident in
// shared memory and every mode applied to it in place.
//
//   pass over modes (mu .. mu+KM-1), view X(a, i_1 .. i_KM, c):
//   * R = 1 (mu = 1, "cube"): a block is CB consecutive c's of the
//     contiguous e_1 x .. x e_KM cube (18^3 = 46.7 KB, 20^3 = 64 KB);
//   * R > 1 (mu > 1): a block is R consecutive a's (256-B rows for R = 32)
//     times the e_1 x .. x e_KM modes, for one c.
//
// A cube is copied into a shared-memory slot by 1-D bulk copies
// (cp.async.bulk, one per contiguous global row; rows that are contiguous in
// both places are merged, so an unpadded cube is ONE copy); a 32-a block by
// four copy warps in 16-byte cp.async chunks (row-by-row bulk copies were 4x
// slower there: one TMA request per 256-B row) -- both into a PADDED
// layout chosen on the host for conflict-free fragment access. Mode j of the
// block is a GEMM with M = the block's rows for that mode (every index
// combination except i_j), N = n_j and K = m_j = n_j (square), so in place is
// safe: a warp owns 8 rows, loads every k of them before its DMMAs and stores
// n_j outputs back into the same rows. The rows of each mode are grouped 8
// per m-tile by a host table (u16 offsets in the slot) so that the four rows
// of every half-warp hit 16 distinct 8-byte bank slots; K is padded to a
// multiple of 4 with zero A values (predicated loads) and N to multiples of 8
// with zero factor entries, so every output is the k-ordered DMMA chain over
// the true k's plus exact zero terms: bitwise the per-mode kernels' results.
//
//   warps 0..15 : G groups of 16/G warps; block i goes to group i % G, which
//                 runs its modes separated by a group named barrier (several
//                 groups keep the DMMA pipe busy through each other's
//                 barrier tails)
//   warp 16     : cubes: producer -- bulk loads into an NB-deep ring of slots
//                 (full[] mbarriers, complete_tx), bulk stores of finished
//                 blocks (done[] mbarriers, one arrival per compute warp),
//                 slot reuse after the store has read it
//   warps 16..19: 32-a blocks: copy warps -- cp.async chunks in (arrivals
//                 on full[] via cp.async.mbarrier.arrive.noinc), LDS + STG
//                 out, storing block i and loading block i + NB in one walk
#pragma once
#include <algorithm>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace mumode_gpu {

constexpr int BLK_MAX_NB = 6;
constexpr int BLK_WARPS = 16;
constexpr int BLK_CWARPS = 4;  // copy warps (R > 1: cp.async rows; R = 1: one bulk-copy warp)
constexpr int BLK_THREADS = (BLK_WARPS + BLK_CWARPS) * 32;
constexpr uint16_t BLK_NOROW = 0xFFFF;

struct BlkSeg {
  int64_t goff;   // doubles, relative to the block origin
  uint32_t soff;  // doubles, relative to the slot
  uint32_t len;   // doubles (R > 1: the row length R, clipped at A)
  uint32_t unit;  // R = 1: the c (unit) of the block this row belongs to
  uint32_t pad_;
};

struct BlockParams {
  const double* X;
  double* S;
  const double* L[3];  // e_j x e_j, column-major, ld = e_j
  const uint16_t* tab;  // row tables of all modes
  const BlkSeg* seg;
  int64_t A, C;         // view extents around the block modes
  int64_t E;            // e_1 * .. * e_KM
  int64_t nblocks;
  int R, CB;            // R > 1: a's per block; R = 1: c's per block
  int KM, NB, G;
  int e[3], s[3];       // extents, slot strides of the modes
  int mt[3], tab_off[3];
  int ntab, nseg;
  int slot_dbl;
  int ls_off, tab_soff, bar_off;  // shared-memory layout (bytes)
};

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}

template <int P4, int NF>
__global__ void __launch_bounds__(BLK_THREADS, 1) block_kernel(const BlockParams p) {
  constexpr int KS = P4 / 4, NP = 8 * NF;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  double* slots = reinterpret_cast<double*>(smem_raw);
  double* Ls = reinterpret_cast<double*>(smem_raw + p.ls_off);
  uint16_t* tab = reinterpret_cast<uint16_t*>(smem_raw + p.tab_soff);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + p.bar_off);
  uint64_t* done = full + BLK_MAX_NB;
  volatile int64_t* tag = reinterpret_cast<volatile int64_t*>(done + BLK_MAX_NB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NB = p.NB, G = p.G, W = BLK_WARPS / G;
  // Block i goes to group i % G and slot i % NB (phase i / NB of that slot's
  // barriers). Groups share slots, so a group may reach block i while the
  // slot still holds block i - NB (its load not even issued): a parity wait
  // would then alias phase i / NB - 2. The producer tags the slot with the
  // block id before loading it; a group first waits for the tag, after which
  // the slot's barrier is exactly in phase i / NB.
  auto slot_of = [&](int64_t i) { return static_cast<int>(i % NB); };

  if (threadIdx.x == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], p.R > 1 ? BLK_CWARPS * 32 : 1);
      mbar_init(&done[b], W);
      tag[b] = -1;
    }
    fence_barrier_init();
  }
  pdl_launch_dependents();
  pdl_wait();  // before any global access (factors and tables included)
  // factors, zero-padded to NP x P4, and the row tables
  for (int i = threadIdx.x; i < p.KM * NP * P4; i += blockDim.x) {
    const int j = i / (NP * P4), r = i - j * (NP * P4);
    const int row = r % NP, col = r / NP, e = p.e[j];
    Ls[i] = (row < e && col < e) ? p.L[j][row + e * col] : 0.0;
  }
  for (int i = threadIdx.x; i < p.ntab; i += blockDim.x) tab[i] = p.tab[i];
  __syncthreads();

  const int64_t n = (p.nblocks - blockIdx.x + gridDim.x - 1) / gridDim.x;  // blocks of this CTA

  if (warp >= BLK_WARPS && p.R > 1) {
    // ---------------------------------------------- copy warps, R > 1 rows
    // Row rho of a block (rho = i_1 + e_1 i_2 + e_1 e_2 i_3) is R contiguous
    // doubles at global a0 + A (E c + rho) and slot offset sum_j i_j s_j.
    // 16-byte cp.async chunks in (completion counted on full[] by
    // cp.async.mbarrier.arrive.noinc), 16-byte LDS + STG out. Row-by-row
    // bulk copies measured 4x slower here (one TMA request per 256-B row).
    const int ct = threadIdx.x - BLK_WARPS * 32;  // 0..127
    const int cpr = p.R >> 1;                      // chunks per row (divides 128: R in {2, 4, .., 32})
    const int q = ct % cpr, rstep = (BLK_CWARPS * 32) / cpr;
    const int64_t nab = (p.A + p.R - 1) / p.R;
    const int E = static_cast<int>(p.E);
    const int e0 = p.e[0], e1 = p.KM > 1 ? p.e[1] : 1;
    const int s0 = p.s[0], s1 = p.s[1], s2 = p.s[2];
    auto locate = [&](int64_t i, int64_t& origin, int& w) {
      const int64_t blk = blockIdx.x + i * gridDim.x;
      const int64_t c = blk / nab, a0 = (blk - c * nab) * p.R;
      origin = a0 + p.A * p.E * c;
      w = static_cast<int>(p.R < p.A - a0 ? int64_t(p.R) : p.A - a0);
    };
    // rows rho = ct / cpr + k * rstep, walked incrementally (no divisions in
    // the loop: 64-bit index math per chunk made these warps the bottleneck)
    auto for_rows = [&](auto&& body) {
      int rho = ct / cpr;
      int i0 = rho % e0, r1 = rho / e0;
      int i1 = r1 % e1, i2 = r1 / e1;
      for (; rho < E; rho += rstep) {
        body(rho, i0 * s0 + i1 * s1 + i2 * s2);
        i0 += rstep;
        while (i0 >= e0) {
          i0 -= e0;
          if (++i1 == e1) {
            i1 = 0;
            ++i2;
          }
        }
      }
    };
    auto load = [&](int64_t i) {
      const int slot = slot_of(i);
      int64_t origin;
      int w;
      locate(i, origin, w);
      double* base = slots + static_cast<int64_t>(slot) * p.slot_dbl + 2 * q;
      const double* src = p.X + origin + 2 * q;
      if (ct == 0) tag[slot] = i;
      if (2 * q < w)
        for_rows([&](int rho, int soff) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(base + soff)), "l"(src + p.A * rho)
                       : "memory");
        });
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&full[slot])) : "memory");
    };
    auto store = [&](int64_t i) {
      const int slot = slot_of(i);
      int64_t origin;
      int w;
      locate(i, origin, w);
      const double* base = slots + static_cast<int64_t>(slot) * p.slot_dbl + 2 * q;
      double* dst = p.S + origin + 2 * q;
      if (2 * q < w)
        for_rows([&](int rho, int soff) {
          const double2 v = *reinterpret_cast<const double2*>(base + soff);
          stg_f64x2(dst + p.A * rho, v.x, v.y);
        });
    };
    const int64_t pre = int64_t(NB) < n ? int64_t(NB) : n;
    for (int64_t i = 0; i < pre; ++i) load(i);
    // store block i and load block i + NB into the same slot in one walk:
    // every thread loads exactly the 16-byte chunks it stored, right after
    // storing each (its LDS has returned before the STG issues), so no
    // barrier separates the two streams
    auto store_load = [&](int64_t i, int64_t i2) {
      const int slot = slot_of(i);
      int64_t o1, o2;
      int w1, w2;
      locate(i, o1, w1);
      locate(i2, o2, w2);
      double* base = slots + static_cast<int64_t>(slot) * p.slot_dbl + 2 * q;
      double* dst = p.S + o1 + 2 * q;
      const double* src = p.X + o2 + 2 * q;
      const bool st = 2 * q < w1, ld = 2 * q < w2;
      if (ct == 0) tag[slot] = i2;
      for_rows([&](int rho, int soff) {
        if (st) {
          const double2 v = *reinterpret_cast<const double2*>(base + soff);
          stg_f64x2(dst + p.A * rho, v.x, v.y);
        }
        if (ld)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(base + soff)), "l"(src + p.A * rho)
                       : "memory");
      });
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&full[slot])) : "memory");
    };
    for (int64_t i = 0; i < n; ++i) {
      const int slot = slot_of(i);
      mbar_wait(&done[slot], static_cast<uint32_t>((i / NB) & 1));
      if (i + NB < n) store_load(i, i + NB);
      else store(i);
    }
    return;
  }
  if (warp > BLK_WARPS) return;
  if (warp == BLK_WARPS) {
    // ------------------------------------------------------------ producer
    const int64_t nab = (p.A + p.R - 1) / p.R;
    auto locate = [&](int64_t i, int64_t& origin, int& w, int& nvalid) {
      const int64_t blk = blockIdx.x + i * gridDim.x;
      if (p.R > 1) {
        const int64_t c = blk / nab, ab = blk - c * nab;
        const int64_t a0 = ab * p.R;
        origin = a0 + p.A * p.E * c;
        w = static_cast<int>((p.R < p.A - a0 ? int64_t(p.R) : p.A - a0));
        nvalid = 0;
      } else {
        const int64_t c0 = blk * p.CB;
        origin = c0 * p.E;
        w = 0;
        nvalid = static_cast<int>((int64_t(p.CB) < p.C - c0 ? int64_t(p.CB) : p.C - c0));
      }
    };
    auto issue_load = [&](int64_t i) {
      const int slot = slot_of(i);
      int64_t origin;
      int w, nvalid;
      locate(i, origin, w, nvalid);
      const uint32_t bytes = p.R > 1 ? static_cast<uint32_t>(p.nseg) * w * 8u
                                     : static_cast<uint32_t>(nvalid * p.E * 8);
      if (lane == 0) {
        tag[slot] = i;
        mbar_arrive_expect_tx(&full[slot], bytes);
      }
      __syncwarp();
      double* base = slots + static_cast<int64_t>(slot) * p.slot_dbl;
      for (int k = lane; k < p.nseg; k += 32) {
        const BlkSeg sg = p.seg[k];
        if (p.R == 1 && static_cast<int>(sg.unit) >= nvalid) continue;
        const uint32_t len = p.R > 1 ? static_cast<uint32_t>(w) : sg.len;
        bulk_load(base + sg.soff, p.X + origin + sg.goff, len * 8u, &full[slot]);
      }
    };
    auto issue_store = [&](int64_t i) {
      const int slot = slot_of(i);
      int64_t origin;
      int w, nvalid;
      locate(i, origin, w, nvalid);
      const double* base = slots + static_cast<int64_t>(slot) * p.slot_dbl;
      for (int k = lane; k < p.nseg; k += 32) {
        const BlkSeg sg = p.seg[k];
        if (p.R == 1 && static_cast<int>(sg.unit) >= nvalid) continue;
        const uint32_t len = p.R > 1 ? static_cast<uint32_t>(w) : sg.len;
        bulk_store(p.S + origin + sg.goff, base + sg.soff, len * 8u);
      }
      bulk_commit();
    };
    const int64_t pre = int64_t(NB) < n ? int64_t(NB) : n;
    for (int64_t i = 0; i < pre; ++i) issue_load(i);
    for (int64_t i = 0; i < n; ++i) {
      const int slot = slot_of(i);
      mbar_wait(&done[slot], static_cast<uint32_t>((i / NB) & 1));
      issue_store(i);
      if (i + NB < n) {
        bulk_wait_read_all();  // this lane's stores have read the slot
        __syncwarp();          // ... and every other lane's
        issue_load(i + NB);
      }
    }
    bulk_wait_all();
    return;
  }

  // -------------------------------------------------------------- compute
  const int gid = warp / W, w = warp - gid * W;
  const int g = lane >> 2, t = lane & 3;
  for (int64_t i = gid; i < n; i += G) {
    const int slot = slot_of(i);
    if (tag[slot] != i) {
      uint32_t polls = 0;
      while (tag[slot] != i)
        if (++polls == (1u << 28)) __trap();
    }
    mbar_wait(&full[slot], static_cast<uint32_t>((i / NB) & 1));
    double* Xs = slots + static_cast<int64_t>(slot) * p.slot_dbl;
    for (int j = 0; j < p.KM; ++j) {
      const int e = p.e[j], s = p.s[j];
      const double* Lj = Ls + j * NP * P4;
      double bf[KS][NF];
#pragma unroll
      for (int k = 0; k < KS; ++k)
#pragma unroll
        for (int f = 0; f < NF; ++f) bf[k][f] = Lj[(g + 8 * f) + NP * (t + 4 * k)];
      const uint16_t* tj = tab + p.tab_off[j];
      const int mtn = p.mt[j];
      for (int mt = w; mt < mtn; mt += W) {
        const uint32_t b = tj[mt * 8 + g];
        const bool rv = b != BLK_NOROW;
        double a[KS];
#pragma unroll
        for (int k = 0; k < KS; ++k) {
          const int kk = t + 4 * k;
          a[k] = (rv && kk < e) ? Xs[b + s * kk] : 0.0;
        }
        double acc[NF][2];
#pragma unroll
        for (int f = 0; f < NF; ++f) acc[f][0] = acc[f][1] = 0.0;
#pragma unroll
        for (int k = 0; k < KS; ++k)
#pragma unroll
          for (int f = 0; f < NF; ++f) dmma_8x8x4(acc[f][0], acc[f][1], a[k], bf[k][f]);
        if (rv) {
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            const int j0 = 2 * t + 8 * f;
            if (j0 < e) Xs[b + s * j0] = acc[f][0];
            if (j0 + 1 < e) Xs[b + s * (j0 + 1)] = acc[f][1];
          }
        }
      }
      if (j + 1 < p.KM) named_barrier_sync(1 + gid, W * 32);
    }
    fence_proxy_async();  // this thread's shared stores -> the bulk store (async proxy)
    __syncwarp();
    if (lane == 0) mbar_arrive(&done[slot]);
  }
}

// ------------------------------------------------------------------ host plan
// Layout search and row tables for one (A, e_1..e_KM, C, R, CB) block pass.
struct BlockLayout {
  int R = 0, CB = 1, KM = 0;
  int e[3] = {0, 0, 0};
  int s[3] = {0, 0, 0};
  int slot_dbl = 0;
  int mt[3] = {0, 0, 0}, tab_off[3] = {0, 0, 0};
  std::vector<uint16_t> tab;
  std::vector<BlkSeg> seg;
  int64_t cost = 0;  // shared-memory wavefronts per block (fragment loads + stores)
};

// wavefronts of one 64-bit shared access by 16 lanes (addresses in doubles):
// distinct 128-B lines per 8-byte bank slot, maximised over the slots
static int blk_wavefronts(const int64_t* addr, int nlanes) {
  int worst = 0;
  for (int i = 0; i < nlanes; ++i) {
    if (addr[i] < 0) continue;
    int cnt = 0;
    for (int k = 0; k < nlanes; ++k) {
      if (addr[k] < 0 || (addr[k] & 15) != (addr[i] & 15)) continue;
      bool first = true;  // count each distinct line once
      for (int q = 0; q < k; ++q)
        if (addr[q] >= 0 && (addr[q] & 15) == (addr[i] & 15) && (addr[q] >> 4) == (addr[k] >> 4)) first = false;
      cnt += first;
    }
    worst = std::max(worst, cnt);
  }
  return worst;
}

// group the rows of one mode 8 per m-tile, 4 per half-warp, so that each
// half-warp's fragment loads (row base + s*t, t = 0..3) hit distinct slots
static void blk_group_rows(const std::vector<int64_t>& rows, int s, std::vector<int64_t>& out) {
  const int64_t nr = static_cast<int64_t>(rows.size());
  std::vector<char> used(nr, 0);
  auto mask_of = [&](int64_t b) {
    uint32_t m = 0;
    for (int t = 0; t < 4; ++t) m |= 1u << ((b + int64_t(s) * t) & 15);
    return m;
  };
  int64_t cursor = 0, placed = 0;
  out.clear();
  while (placed < nr) {
    uint32_t hw_mask = 0;
    for (int pick = 0; pick < 4; ++pick) {
      while (cursor < nr && used[cursor]) ++cursor;
      if (cursor >= nr) {
        out.push_back(-1);
        continue;
      }
      int64_t chosen = -1;
      for (int64_t q = cursor, seen = 0; q < nr && seen < 96; ++q) {
        if (used[q]) continue;
        ++seen;
        const uint32_t m = mask_of(rows[q]);
        if (__builtin_popcount(m) == 4 && !(m & hw_mask)) {
          chosen = q;
          break;
        }
      }
      if (chosen < 0) chosen = cursor;
      used[chosen] = 1;
      ++placed;
      hw_mask |= mask_of(rows[chosen]);
      out.push_back(rows[chosen]);
    }
  }
  while (out.size() % 8) out.push_back(-1);
}

static int64_t blk_mode_cost(const std::vector<int64_t>& grp, int s, int e) {
  const int KS = (e + 3) / 4, NFr = (e + 7) / 8;
  int64_t cost = 0;
  int64_t addr[16];
  for (size_t m0 = 0; m0 < grp.size(); m0 += 8)
    for (int hw = 0; hw < 2; ++hw) {
      const int64_t* r = &grp[m0 + 4 * hw];
      for (int k = 0; k < KS; ++k) {
        for (int g = 0; g < 4; ++g)
          for (int t = 0; t < 4; ++t) addr[4 * g + t] = (r[g] < 0 || t + 4 * k >= e) ? -1 : r[g] + int64_t(s) * (t + 4 * k);
        cost += blk_wavefronts(addr, 16);
      }
      for (int f = 0; f < NFr; ++f)
        for (int dl = 0; dl < 2; ++dl) {
          for (int g = 0; g < 4; ++g)
            for (int t = 0; t < 4; ++t) {
              const int jj = 2 * t + dl + 8 * f;
              addr[4 * g + t] = (r[g] < 0 || jj >= e) ? -1 : r[g] + int64_t(s) * jj;
            }
          cost += blk_wavefronts(addr, 16);
        }
    }
  return cost;
}

// Build the layout with the lowest fragment-access cost whose slot fits
// `max_slot_dbl`. Block dims (innermost first): R > 1: [R, e_1..e_KM];
// R = 1: [e_1..e_KM, CB]. Pads: the row pitch (innermost) by 0/2/4/6, the
// next two dims by 0..3.
static bool blk_plan_layout(int64_t A, const int* e, int KM, int R, int CB, int64_t max_slot_dbl, BlockLayout& best) {
  std::vector<int64_t> ext;
  if (R > 1) ext.push_back(R);
  for (int j = 0; j < KM; ++j) ext.push_back(e[j]);
  if (R == 1 && CB > 1) ext.push_back(CB);
  const int nd = static_cast<int>(ext.size());
  const int mode0 = (R > 1) ? 1 : 0;  // dim index of block mode 0
  if (ext[0] & 1) return false;       // 16-byte rows
  bool found = false;
  std::vector<int64_t> best_st;
  std::vector<int64_t> rows, grp;
  for (int p0 = 0; p0 <= 6; p0 += 2)
    for (int p1 = 0; p1 <= (nd > 2 ? 3 : 0); ++p1)
      for (int p2 = 0; p2 <= (nd > 3 ? 3 : 0); ++p2) {
        const int pad[4] = {p0, nd > 2 ? p1 : 0, nd > 3 ? p2 : 0, 0};
        std::vector<int64_t> st(nd);
        st[0] = 1;
        for (int d = 1; d < nd; ++d) st[d] = st[d - 1] * (ext[d - 1] + (d - 1 < 4 ? pad[d - 1] : 0));
        int64_t slot = st[nd - 1] * ext[nd - 1];
        slot = (slot + 15) / 16 * 16;
        if (slot > max_slot_dbl || slot > 65000) continue;
        BlockLayout L;
        L.R = R;
        L.CB = CB;
        L.KM = KM;
        L.slot_dbl = static_cast<int>(slot);
        int64_t cost = 0;
        for (int j = 0; j < KM; ++j) {
          const int dj = mode0 + j;
          L.e[j] = e[j];
          L.s[j] = static_cast<int>(st[dj]);
          rows.clear();
          // every index combination of the other dims, innermost fastest
          std::vector<int64_t> idx(nd, 0);
          for (;;) {
            int64_t b = 0;
            for (int d = 0; d < nd; ++d) b += idx[d] * st[d];
            rows.push_back(b);
            int d = 0;
            for (; d < nd; ++d) {
              if (d == dj) continue;
              if (++idx[d] < ext[d]) break;
              idx[d] = 0;
            }
            if (d == nd) break;
          }
          blk_group_rows(rows, L.s[j], grp);
          cost += blk_mode_cost(grp, L.s[j], e[j]);
          L.tab_off[j] = static_cast<int>(L.tab.size());
          L.mt[j] = static_cast<int>(grp.size() / 8);
          for (int64_t v : grp) L.tab.push_back(v < 0 ? BLK_NOROW : static_cast<uint16_t>(v));
        }
        L.cost = cost;
        if (!found || cost < best.cost || (cost == best.cost && L.slot_dbl < best.slot_dbl)) {
          best = std::move(L);
          best_st = st;
          found = true;
        }
      }
  if (!found) return false;
  // copy segments: one per contiguous global row (dim 0), merged where
  // consecutive rows are contiguous in both global memory and the slot
  std::vector<int64_t> gst(nd);
  gst[0] = 1;
  for (int d = 1; d < nd; ++d) {
    if (R > 1) gst[d] = gst[d - 1] * (d == 1 ? A : ext[d - 1]);
    else gst[d] = gst[d - 1] * ext[d - 1];
  }
  best.seg.clear();
  std::vector<int64_t> idx(nd, 0);
  for (;;) {
    BlkSeg sg{};
    for (int d = 1; d < nd; ++d) {
      sg.goff += idx[d] * gst[d];
      sg.soff += static_cast<uint32_t>(idx[d] * best_st[d]);
    }
    sg.len = static_cast<uint32_t>(ext[0]);
    sg.unit = (R == 1 && CB > 1) ? static_cast<uint32_t>(idx[nd - 1]) : 0u;
    if (R == 1 && !best.seg.empty()) {
      BlkSeg& b = best.seg.back();
      if (b.unit == sg.unit && b.goff + b.len == sg.goff && b.soff + b.len == sg.soff) {
        b.len += sg.len;
        sg.len = 0;
      }
    }
    if (sg.len) best.seg.push_back(sg);
    int d = 1;
    for (; d < nd; ++d) {
      if (++idx[d] < ext[d]) break;
      idx[d] = 0;
    }
    if (d >= nd) break;
  }
  return true;
}

}  // namespace mumode_gpu
