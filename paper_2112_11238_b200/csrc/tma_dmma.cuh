// Persistent, warp-specialised mu-mode product kernel for sm_100a:
// TMA (cp.async.bulk.tensor) stages operand slabs into a multi-stage
// shared-memory ring guarded by mbarriers (one elected lane of a 4-warp
// producer group issues the boxes); the MMA warps (Cfg::MMA_WARPS, 16 for the
// main configurations; registers rebalanced with setmaxnreg) run fp64
// tensor-core MMAs (mma.sync m8n8k4 -> SASS DMMA.8x8x4: the only fp64
// tensor-core path on sm_100a, tcgen05 has no f64 kind) and store straight
// from registers (or scatter / accumulate / divide, see EPI). Real fp64 and
// complex128 share the pipeline. Launched with programmatic dependent launch.
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
// Tiles have 8-element granularity in M, N and K (8-element-wide TMA boxes),
// so extents like 200 (config C3) or 192 (C4) tile without padding, and for
// mu > 1 the M dimension runs over a list of 8-row fragments (a-block, c) so
// batches never pad either.
#pragma once
#include "common.cuh"

namespace mumode_gpu {

// Scatter epilogue (EPI 2): the output is the (rows x w) matrix of a slab's
// last local mode; row rho belongs to rank q with a_off[q] <= rho < a_off[q+1]
// and lands at dst[q][(rho - a_off[q]) + (a_off[q+1] - a_off[q]) * (col0 + c)]
// -- the rank's received (A_q x m_d) matrix, written in place over NVLink
// peer pointers (csrc/slab_dist.cuh) instead of pack + exchange.
constexpr int kScatterMaxRanks = 64;
struct ScatterParams {
  int P;
  int64_t col0;
  int64_t a_off[kScatterMaxRanks + 1];
  double* dst[kScatterMaxRanks];
};

// owner rank of row rho (binary search over P + 1 offsets)
__device__ __forceinline__ int scatter_owner(const ScatterParams* sp, int64_t rho) {
  int lo = 0, hi = sp->P - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(&sp->a_off[mid]) <= rho) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ void scatter_store(const ScatterParams* sp, int64_t rho, int64_t col, double v0,
                                              double v1) {
  const int64_t gcol = sp->col0 + col;
  const int q = scatter_owner(sp, rho);
  const int64_t lo = __ldg(&sp->a_off[q]), hi = __ldg(&sp->a_off[q + 1]);
  double* d0 = sp->dst[q] + (rho - lo) + (hi - lo) * gcol;
  if (rho + 1 < hi) {  // both rows on rank q
    if ((reinterpret_cast<uintptr_t>(d0) & 15u) == 0) {
      stg_f64x2(d0, v0, v1);
    } else {
      d0[0] = v0;
      d0[1] = v1;
    }
  } else {  // the pair straddles two ranks
    d0[0] = v0;
    const int q1 = scatter_owner(sp, rho + 1);
    const int64_t lo1 = __ldg(&sp->a_off[q1]), hi1 = __ldg(&sp->a_off[q1 + 1]);
    sp->dst[q1][(rho + 1 - lo1) + (hi1 - lo1) * gcol] = v1;
  }
}

// complex element (re, im) of row rho, column col (rows and offsets count
// complex elements; dst points at interleaved doubles)
__device__ __forceinline__ void scatter_store_c(const ScatterParams* sp, int64_t rho, int64_t col, double re,
                                                double im) {
  const int q = scatter_owner(sp, rho);
  const int64_t lo = __ldg(&sp->a_off[q]), hi = __ldg(&sp->a_off[q + 1]);
  stg_f64x2(sp->dst[q] + 2 * ((rho - lo) + (hi - lo) * (sp->col0 + col)), re, im);
}

struct TmaParams {
  const ScatterParams* scat;  // EPI 2 only (device memory)
  const double* div_front;    // EPI 3: D(a, n) /= (div_front[a] + div_last[n])
  const double* div_last;
  double* D;
  int64_t ldD;      // stride of D between consecutive n (elements)
  int64_t bstride;  // stride of D between batches c (elements)
  int Mlim;         // valid rows per batch: A (mu > 1) or n_out (mu == 1)
  int N, K;
  int AB;           // 8-row M fragments per batch = ceil(Mlim / 8)
  int64_t mfrags;   // M fragments over all batches = AB * batches
  int mt, nt;       // tile counts along the M-fragment list and along N
  int64_t tiles;    // mt * nt
  // Blocked views: the whole operand tile is ONE TMA box per stage
  //   P blocked: mode 1 {8e, K, n/8} box {8e, BK, BM/8};
  //              mode >1 {8e, K, A/8, C} box {8e, BK, BM/8, 1} (tiles never straddle c)
  //   Q blocked: mode 1 {8e, C, K/8} box {8e, BN, BK/8}; mode >1 {8e, K, n/8} box {8e, BK, BN/8}
  // (e = doubles per element). Otherwise one box per 8-element block.
  int p_blocked, q_blocked;
};

// E = doubles per element (1: fp64, 2: complex128). A staged row of 8
// elements is 64 B (fp64, 64B swizzle) or 128 B (complex, 128B swizzle).
template <int BM_, int BN_, int BK_, int STAGES_, int WM_, int WN_, int E_ = 1>
struct TmaCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, STAGES = STAGES_, WM = WM_, WN = WN_, E = E_;
  static constexpr int ROW = 64 * E;  // bytes of one staged 8-element row
  static constexpr int MMA_WARPS = WM * WN;
  // MMA warps + one producer warpgroup (setmaxnreg works per warpgroup; the
  // producer group's registers are what the MMA warps grow into).
  static constexpr int THREADS = (MMA_WARPS + 4) * 32;
  // Register split after setmaxnreg. setmaxnreg.inc draws from the CTA's LAUNCH
  // allocation (per-thread limit of the launch bounds x THREADS), not the whole
  // register file -- asking for more blocks forever. The producer warpgroup
  // keeps 24; the MMA warps share the rest (multiple of 8, <= 232).
  static constexpr int LAUNCH_REGS = (65536 / THREADS) / 8 * 8 > 255 ? 248 : (65536 / THREADS) / 8 * 8;
  static constexpr int POOL = LAUNCH_REGS * THREADS;
  static constexpr int PRODUCER_REGS = 24;
  static constexpr int CONSUMER_REGS_RAW = ((POOL - 4 * 32 * PRODUCER_REGS) / (MMA_WARPS * 32)) / 8 * 8;
  static constexpr int CONSUMER_REGS = CONSUMER_REGS_RAW > 232 ? 232 : CONSUMER_REGS_RAW;
  static_assert(4 * 32 * PRODUCER_REGS + MMA_WARPS * 32 * CONSUMER_REGS <= POOL, "setmaxnreg budget");
  static_assert(CONSUMER_REGS >= LAUNCH_REGS, "setmaxnreg.inc must not shrink");
  static constexpr int WTM = BM / WM, WTN = BN / WN;  // warp tile
  static constexpr int FM = WTM / 8, FN = WTN / 8;    // 8-wide fragments per warp
  static constexpr int P_BYTES = BM * BK * 8 * E, Q_BYTES = BN * BK * 8 * E;
  static constexpr int STAGE_BYTES = P_BYTES + Q_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 2 * STAGES * 8;
  static_assert(E == 1 || E == 2, "fp64 or complex128");
  static_assert(MMA_WARPS % 4 == 0, "MMA warps must form whole warpgroups");
  static_assert(BM % 8 == 0 && BN % 8 == 0 && BK % 8 == 0, "8-element TMA boxes");
  static_assert(WTM % 8 == 0 && WTN % 8 == 0, "warp tiles are whole 8-wide fragments");
  static_assert(BN <= 256 && BK <= 256 && BM / 8 <= 256, "TMA box extent limit");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory per CTA");
};

// ---------------------------------------------------------------- fragments
// lane = 4g + t. A fragment covers 8 elements x = 8*blk + map(g) of its
// operand's free dimension; k-step s reads the k rows 4s + t. DMMA ownership:
// A[g][t] (Q side, rows n), B[t][g] (P side, cols m), D[g][2t], D[g][2t+1].
//
// fp64 (64B swizzle: 16-B chunk c of a 64-B row at byte a -> c ^ ((a>>7)&3)).
// 64-bit shared loads are serviced per half-warp; xmap8 puts each half-warp's
// 16 loads on 16 distinct 8-byte bank slots in both layouts, every s:
//   XK ([x-block][k][8]):  blk*BK*64 + 4s*64 + t*64 + (g&1)*8 + J_s
//   KX ([k-block][x][8]):  (s>>1)*BX*64 + (8blk + xmap8(g))*64 + (t&1)*8 + J_s
//   J_s = ((jg ^ (t>>1)) << 4) ^ (32(s&1)),  jg = 2((g>>1)&1) + (g>>2)
// xmap8(2t), xmap8(2t)+1 are adjacent -> 16-B epilogue stores.
//
// complex128 (128B swizzle: chunk c of a 128-B row -> c ^ ((a>>7)&7)); one
// 16-B chunk = one element, read with LDS.128 (re, im), serviced per quarter
// warp; xmapc puts each quarter-warp on 8 distinct chunks in both layouts:
//   XK:  blk*BK*128 + 4s*128 + t*128 + Jc_s
//   KX:  (s>>1)*BX*128 + (8blk + xmapc(g))*128 + Jc_s
//   Jc_s = ((xmapc(g) ^ t) << 4) ^ (64(s&1))
// (all maps checked exhaustively against the swizzle and bank models).
// (xmap8 / xmapc live in common.cuh)

// QK == true  (mu == 1): P = L (XK), Q = T (KX)
// QK == false (mu  > 1): P = T (XK, fragment list over (a-block, c)), Q = L (XK)
// One output tile of the mode product, producer side: the elected lane
// issues the tile's K-stages into the ring (stage / phase persist across
// tiles and, in the chain kernel, across modes).
template <class Cfg, bool QK>
__device__ __forceinline__ void tma_produce_tile(const CUtensorMap* mapP, const CUtensorMap* mapQ, const TmaParams& p,
                                                 int mtile, int ntile, uint8_t* smem, uint64_t* full_bar,
                                                 uint64_t* empty_bar, int& stage, uint32_t& phase) {
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES, E = Cfg::E, ROW = Cfg::ROW;
  const int KT = (p.K + BK - 1) / BK;
  const int n0 = ntile * BN;
  // first M fragment of the tile -> (batch c0, a-block ab0); later
  // fragments advance incrementally (no per-stage divisions)
  const uint32_t q0 = static_cast<uint32_t>(mtile) * (BM / 8);
  const uint32_t qlast = static_cast<uint32_t>(p.mfrags - 1);
  uint32_t c0 = 0, ab0 = q0;
  if constexpr (!QK) {
    c0 = q0 / static_cast<uint32_t>(p.AB);
    ab0 = q0 - c0 * static_cast<uint32_t>(p.AB);
  }
  for (int kb = 0; kb < KT; ++kb) {
    mbar_wait(&empty_bar[stage], phase ^ 1);
    uint8_t* sP = smem + stage * Cfg::STAGE_BYTES;
    uint8_t* sQ = sP + Cfg::P_BYTES;
    mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
    const int k0 = kb * BK;
    if (p.p_blocked) {
      if constexpr (QK)
        tma_load_3d(sP, mapP, &full_bar[stage], 0, k0, static_cast<int32_t>(q0));
      else
        tma_load_4d(sP, mapP, &full_bar[stage], 0, k0, static_cast<int32_t>(ab0),
                    static_cast<int32_t>(c0));
    } else {
      uint32_t c = c0, ab = ab0;
#pragma unroll 1
      for (int f = 0; f < BM / 8; ++f) {
        // fragments past the end re-load the last valid one (masked later)
        if constexpr (QK) {
          const uint32_t q = (q0 + f <= qlast) ? (q0 + f) : qlast;
          tma_load_2d(sP + f * BK * ROW, mapP, &full_bar[stage], static_cast<int32_t>(8 * E * q), k0);
        } else {
          if (q0 + f > qlast) {
            c = qlast / static_cast<uint32_t>(p.AB);
            ab = qlast - c * static_cast<uint32_t>(p.AB);
          }
          tma_load_3d(sP + f * BK * ROW, mapP, &full_bar[stage], static_cast<int32_t>(8 * E * ab), k0,
                      static_cast<int32_t>(c));
          if (++ab == static_cast<uint32_t>(p.AB)) {
            ab = 0;
            ++c;
          }
        }
      }
    }
    if (p.q_blocked) {
      if constexpr (QK)
        tma_load_3d(sQ, mapQ, &full_bar[stage], 0, n0, k0 / 8);
      else
        tma_load_3d(sQ, mapQ, &full_bar[stage], 0, k0, n0 / 8);
    } else if constexpr (QK) {
#pragma unroll 1
      for (int b = 0; b < BK / 8; ++b)
        tma_load_2d(sQ + b * BN * ROW, mapQ, &full_bar[stage], E * (k0 + 8 * b), n0);
    } else {
#pragma unroll 1
      for (int b = 0; b < BN / 8; ++b)
        tma_load_2d(sQ + b * BK * ROW, mapQ, &full_bar[stage], E * (n0 + 8 * b), k0);
    }
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1;
    }
  }
}

// Thread-constant parts of the fragment addresses (see the maps above).
struct FragOffsets {
  int g, t, mw, nw;
  uint32_t J0, xk_off, kx_off;
};

template <class Cfg>
__device__ __forceinline__ FragOffsets tma_frag_offsets(int warp, int lane) {
  FragOffsets o;
  o.g = lane >> 2;
  o.t = lane & 3;
  o.mw = (warp % Cfg::WM) * Cfg::WTM;
  o.nw = (warp / Cfg::WM) * Cfg::WTN;
  if constexpr (Cfg::E == 2) {
    o.J0 = static_cast<uint32_t>(xmapc(o.g) ^ o.t) << 4;
    o.xk_off = static_cast<uint32_t>(o.t * 128);
    o.kx_off = static_cast<uint32_t>(xmapc(o.g) * 128);
  } else {
    const int jg = 2 * ((o.g >> 1) & 1) + (o.g >> 2);
    o.J0 = static_cast<uint32_t>(jg ^ (o.t >> 1)) << 4;
    o.xk_off = static_cast<uint32_t>(o.t * 64 + (o.g & 1) * 8);
    o.kx_off = static_cast<uint32_t>(xmap8(o.g) * 64 + (o.t & 1) * 8);
  }
  return o;
}

// One output tile, MMA-warp side: consume the tile's K-stages from the ring
// (DMMA), then the epilogue (EPI) straight from registers.
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// (before_epilogue runs between the main loop and the epilogue: the chain
// kernel publishes the previous tile there)
template <class Cfg, bool QK, int EPI, class Hook = NoHook>
__device__ __forceinline__ void tma_consume_tile(const TmaParams& p, int mtile, int ntile, const uint8_t* smem,
                                                 uint64_t* full_bar, uint64_t* empty_bar, int& stage,
                                                 uint32_t& phase, const FragOffsets& fo, int lane,
                                                 const Hook& before_epilogue = Hook()) {
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr int FM = Cfg::FM, FN = Cfg::FN, E = Cfg::E, ROW = Cfg::ROW;
  constexpr bool CPLX = (E == 2);
  constexpr bool ACC = (EPI == 1);
  constexpr uint32_t JFLIP = CPLX ? 64u : 32u;  // XOR applied on odd k-steps
  const int KT = (p.K + BK - 1) / BK;
  const int g = fo.g, t = fo.t, mw = fo.mw, nw = fo.nw;
  const uint32_t J0 = fo.J0, xk_off = fo.xk_off, kx_off = fo.kx_off;
  // real: acc[fm][fn][0..1]. complex: four real chains, as OpenBLAS's zgemm
  // kernels keep them -- [0..1] sum qr*pr, [2..3] sum qi*pi, [4..5] sum qr*pi,
  // [6..7] sum qi*pr -- combined once in the epilogue (re = rr - ii,
  // im = ri + ir), so complex results round like the reference's cblas_zgemm
  constexpr int NACC = CPLX ? 8 : 2;
  double acc[FM][FN][NACC];
#pragma unroll
  for (int fm = 0; fm < FM; ++fm)
#pragma unroll
    for (int fn = 0; fn < FN; ++fn)
#pragma unroll
      for (int r = 0; r < NACC; ++r) acc[fm][fn][r] = 0.0;

  if constexpr (ACC) {
    // kronsumv: the epilogue adds into D. Its reads would start a DRAM round trip after the last
    // DMMA with the whole CTA waiting; prefetch the lines into L2 now, under the main loop.
#pragma unroll
    for (int fm = 0; fm < FM; ++fm) {
      const uint32_t q = static_cast<uint32_t>(mtile) * (BM / 8) + (mw >> 3) + fm;
      if (q >= static_cast<uint32_t>(p.mfrags)) continue;
      uint32_t c = 0, ab = q;
      if constexpr (!QK) {
        c = q / static_cast<uint32_t>(p.AB);
        ab = q - c * static_cast<uint32_t>(p.AB);
      }
      const int m = 8 * static_cast<int>(ab) + (CPLX ? t : xmap8(2 * t));
      if (m >= p.Mlim) continue;
      const double* base = p.D + E * (static_cast<int64_t>(c) * p.bstride + m);
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) {
        const int n = ntile * BN + nw + 8 * fn + (CPLX ? xmapc(g) : xmap8(g));
        if (n >= p.N) continue;
        const double* a = base + E * static_cast<int64_t>(n) * p.ldD;
        asm volatile("prefetch.global.L2 [%0];\n" ::"l"(a));
        if constexpr (CPLX) {
          if (m + 4 < p.Mlim) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(a + 8));
        }
      }
    }
  }
  for (int kb = 0; kb < KT; ++kb) {
    mbar_wait(&full_bar[stage], phase);
    const uint8_t* sP = smem + stage * Cfg::STAGE_BYTES;
    const uint8_t* sQ = sP + Cfg::P_BYTES;
#pragma unroll
    for (int s = 0; s < BK / 4; ++s) {
      const uint32_t Js = J0 ^ (JFLIP * static_cast<uint32_t>(s & 1));
      if constexpr (!CPLX) {
        double pf[FM], qf[FN];
#pragma unroll
        for (int fm = 0; fm < FM; ++fm)
          pf[fm] = *reinterpret_cast<const double*>(sP + ((mw >> 3) + fm) * (BK * ROW) + (4 * s) * ROW +
                                                    xk_off + Js);
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) {
          if constexpr (QK)
            qf[fn] = *reinterpret_cast<const double*>(sQ + (s >> 1) * (BN * ROW) + (nw + 8 * fn) * ROW +
                                                      kx_off + Js);
          else
            qf[fn] = *reinterpret_cast<const double*>(sQ + ((nw >> 3) + fn) * (BK * ROW) + (4 * s) * ROW +
                                                      xk_off + Js);
        }
#pragma unroll
        for (int fm = 0; fm < FM; ++fm)
#pragma unroll
          for (int fn = 0; fn < FN; ++fn) dmma_8x8x4(acc[fm][fn][0], acc[fm][fn][1], qf[fn], pf[fm]);
      } else {
        double2 pf[FM], qf[FN];
#pragma unroll
        for (int fm = 0; fm < FM; ++fm)
          pf[fm] = *reinterpret_cast<const double2*>(sP + ((mw >> 3) + fm) * (BK * ROW) + (4 * s) * ROW +
                                                     xk_off + Js);
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) {
          if constexpr (QK)
            qf[fn] = *reinterpret_cast<const double2*>(sQ + (s >> 1) * (BN * ROW) + (nw + 8 * fn) * ROW +
                                                       kx_off + Js);
          else
            qf[fn] = *reinterpret_cast<const double2*>(sQ + ((nw >> 3) + fn) * (BK * ROW) + (4 * s) * ROW +
                                                       xk_off + Js);
        }
        // complex MAC as four real DMMAs into four separate chains
#pragma unroll
        for (int fn = 0; fn < FN; ++fn)
#pragma unroll
          for (int fm = 0; fm < FM; ++fm) {
            dmma_8x8x4(acc[fm][fn][0], acc[fm][fn][1], qf[fn].x, pf[fm].x);
            dmma_8x8x4(acc[fm][fn][2], acc[fm][fn][3], qf[fn].y, pf[fm].y);
            dmma_8x8x4(acc[fm][fn][4], acc[fm][fn][5], qf[fn].x, pf[fm].y);
            dmma_8x8x4(acc[fm][fn][6], acc[fm][fn][7], qf[fn].y, pf[fm].x);
          }
      }
    }
    // The stage's shared-memory reads must be complete before it is released:
    // ptxas sinks the last k-step's DMMAs past the arrive and leaves their
    // LDS in flight, and the producer's next TMA write then races them (seen
    // as an intermittently wrong 8x8 output fragment of the complex 96x32
    // config, ~1 run in 5). fence.acq_rel.cta waits for the warp's
    // outstanding shared loads.
    asm volatile("fence.acq_rel.cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[stage]);
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1;
    }
  }

  before_epilogue();
  // epilogue straight from registers
#pragma unroll
  for (int fm = 0; fm < FM; ++fm) {
    const uint32_t q = static_cast<uint32_t>(mtile) * (BM / 8) + (mw >> 3) + fm;
    if (q >= static_cast<uint32_t>(p.mfrags)) continue;
    uint32_t c = 0, ab = q;
    if constexpr (!QK) {
      c = q / static_cast<uint32_t>(p.AB);
      ab = q - c * static_cast<uint32_t>(p.AB);
    }
    if constexpr (!CPLX) {
      // D(m, m+1 ; n): one 16-byte store along M
      const int m = 8 * static_cast<int>(ab) + xmap8(2 * t);
      if (m >= p.Mlim) continue;
      double* base = p.D + static_cast<int64_t>(c) * p.bstride + m;
      if constexpr (ACC) {
        // all of the row's reads first: a read after the previous column's store may alias it for the
        // compiler, which made FN serial memory round trips per tile (200^3 term: 132 -> 104 us)
        double2 o[FN];
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) {
          const int n = ntile * BN + nw + 8 * fn + xmap8(g);
          if (n < p.N) o[fn] = *reinterpret_cast<const double2*>(base + static_cast<int64_t>(n) * p.ldD);
        }
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) {
          const int n = ntile * BN + nw + 8 * fn + xmap8(g);
          if (n < p.N)
            stg_f64x2(base + static_cast<int64_t>(n) * p.ldD, o[fn].x + acc[fm][fn][0], o[fn].y + acc[fm][fn][1]);
        }
        continue;
      }
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) {
        const int n = ntile * BN + nw + 8 * fn + xmap8(g);
        if (n >= p.N) continue;
        if constexpr (EPI == 2) {
          // row of the (rows x w) matrix and its column (m even, Mlim even)
          if constexpr (QK)
            scatter_store(p.scat, m, n, acc[fm][fn][0], acc[fm][fn][1]);
          else
            scatter_store(p.scat, m + static_cast<int64_t>(n) * p.ldD, c, acc[fm][fn][0], acc[fm][fn][1]);
          continue;
        }
        double* dst = base + static_cast<int64_t>(n) * p.ldD;
        if constexpr (EPI == 3) {
          // the last mode: rows m, m+1 index the modes before it (batch 0)
          const double2 fr = __ldg(reinterpret_cast<const double2*>(p.div_front + m));  // read-only: not reloaded after the stores
          const double ln = __ldg(p.div_last + n);
          stg_f64x2(dst, acc[fm][fn][0] / (fr.x + ln), acc[fm][fn][1] / (fr.y + ln));
          continue;
        }
        stg_f64x2(dst, acc[fm][fn][0], acc[fm][fn][1]);
      }
    } else {
      // D(m) and D(m+4) (xmapc(2t) = t, xmapc(2t+1) = t+4): two 16-byte stores
      const int m = 8 * static_cast<int>(ab) + t;
      double* base = p.D + 2 * (static_cast<int64_t>(c) * p.bstride + m);
      double2 oa[ACC ? FN : 1], ob[ACC ? FN : 1];  // accumulate: the reads of all columns first (see above)
      if constexpr (ACC) {
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) {
          const int n = ntile * BN + nw + 8 * fn + xmapc(g);
          if (n >= p.N) continue;
          const double* col = base + 2 * static_cast<int64_t>(n) * p.ldD;
          if (m < p.Mlim) oa[fn] = *reinterpret_cast<const double2*>(col);
          if (m + 4 < p.Mlim) ob[fn] = *reinterpret_cast<const double2*>(col + 8);
        }
      }
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) {
        const int n = ntile * BN + nw + 8 * fn + xmapc(g);
        if (n >= p.N) continue;
        double* col = base + 2 * static_cast<int64_t>(n) * p.ldD;
        double r0 = acc[fm][fn][0] - acc[fm][fn][2], r1 = acc[fm][fn][1] - acc[fm][fn][3];
        double i0 = acc[fm][fn][4] + acc[fm][fn][6], i1 = acc[fm][fn][5] + acc[fm][fn][7];
        if constexpr (EPI == 2) {
          // one complex element per 16-byte store: rows m and m + 4
          const int64_t rho0 = QK ? m : m + static_cast<int64_t>(n) * p.ldD;
          const int64_t colx = QK ? n : static_cast<int64_t>(c);
          if (m < p.Mlim) scatter_store_c(p.scat, rho0, colx, r0, i0);
          if (m + 4 < p.Mlim) scatter_store_c(p.scat, rho0 + 4, colx, r1, i1);
          continue;
        }
        if constexpr (ACC) {
          if (m < p.Mlim) r0 += oa[fn].x, i0 += oa[fn].y;
          if (m + 4 < p.Mlim) r1 += ob[fn].x, i1 += ob[fn].y;
        }
        if (m < p.Mlim) stg_f64x2(col, r0, i0);
        if (m + 4 < p.Mlim) stg_f64x2(col + 8, r1, i1);
      }
    }
  }
}

// EPI: 0 = store; 1 = D += result (kronsumv term accumulation,
// tucker.hpp:222-231); 2 = scatter to the owning ranks; 3 = divide by the
// eigenvalue Kronecker sum (the direct solver's pointwise step,
// imex.cpp:70-80; last mode, real). A compile-time switch -- a runtime branch
// in the epilogue costs ~2 % on C2.
template <class Cfg, bool QK, int EPI = 0>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    modeprod_tma_kernel(const __grid_constant__ CUtensorMap mapP,
                        const __grid_constant__ CUtensorMap mapQ, const TmaParams p) {
  static_assert(EPI != 3 || Cfg::E == 1, "the divide epilogue is real-only");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment by pointer arithmetic so the compiler keeps the shared
  // address space (LDS, not generic LD).
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + Cfg::STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], Cfg::MMA_WARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();
  // the successor may launch (its CTAs take SMs as ours exit); nothing below
  // reads or writes global memory before the predecessor grid is complete
  pdl_launch_dependents();
  pdl_wait();

  // Tile order: the CTAs that share the big tensor's slab run together (mode
  // 1: T is Q, so m fastest; otherwise T is P, so n fastest) -> T streams
  // from HBM once, repeats hit L2.
  auto decode = [&](int64_t tile, int& mt, int& nt) {
    if constexpr (QK) {
      mt = static_cast<int>(tile % p.mt);
      nt = static_cast<int>(tile / p.mt);
    } else {
      nt = static_cast<int>(tile % p.nt);
      mt = static_cast<int>(tile / p.nt);
    }
  };
  int stage = 0;
  uint32_t phase = 0;
  if (warp >= Cfg::MMA_WARPS) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(Cfg::PRODUCER_REGS) : "memory");
    if (warp == Cfg::MMA_WARPS && lane == 0) {
      tma_prefetch_desc(&mapP);
      tma_prefetch_desc(&mapQ);
      for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
        int mtile, ntile;
        decode(tile, mtile, ntile);
        tma_produce_tile<Cfg, QK>(&mapP, &mapQ, p, mtile, ntile, smem, full_bar, empty_bar, stage, phase);
      }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(Cfg::CONSUMER_REGS) : "memory");
  const FragOffsets fo = tma_frag_offsets<Cfg>(warp, lane);
  for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
    int mtile, ntile;
    decode(tile, mtile, ntile);
    tma_consume_tile<Cfg, QK, EPI>(p, mtile, ntile, smem, full_bar, empty_bar, stage, phase, fo, lane);
  }
}

}  // namespace mumode_gpu
