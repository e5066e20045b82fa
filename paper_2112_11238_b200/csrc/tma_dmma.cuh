// Persistent, warp-specialised mu-mode product kernel for sm_100a:
// TMA (cp.async.bulk.tensor, 64B swizzle) stages operand slabs into a
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
// Tiles have 8-element granularity in M, N and K (8-wide TMA boxes), so
// extents like 200 (config C3) tile without padding.
#pragma once
#include "common.cuh"

namespace mumode_gpu {

struct TmaParams {
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
  //   P blocked: mode 1 {8, K, n/8} box {8, BK, BM/8};
  //              mode >1 {8, K, A/8, C} box {8, BK, BM/8, 1} (tiles never straddle c)
  //   Q blocked: mode 1 {8, C, K/8} box {8, BN, BK/8}; mode >1 {8, K, n/8} box {8, BK, BN/8}
  int p_blocked, q_blocked;
};

template <int BM_, int BN_, int BK_, int STAGES_, int WM_, int WN_>
struct TmaCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, STAGES = STAGES_, WM = WM_, WN = WN_;
  static constexpr int MMA_WARPS = WM * WN;
  // MMA warps + one producer warpgroup (setmaxnreg works per warpgroup; the
  // producer group's registers are what the MMA warps grow into).
  static constexpr int THREADS = (MMA_WARPS + 4) * 32;
  static constexpr int WTM = BM / WM, WTN = BN / WN;  // warp tile
  static constexpr int FM = WTM / 8, FN = WTN / 8;    // 8-wide fragments per warp
  static constexpr int P_BYTES = BM * BK * 8, Q_BYTES = BN * BK * 8;
  static constexpr int STAGE_BYTES = P_BYTES + Q_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 2 * STAGES * 8;
  static_assert(MMA_WARPS % 4 == 0, "MMA warps must form whole warpgroups");
  static_assert(BM % 8 == 0 && BN % 8 == 0 && BK % 8 == 0, "8-wide TMA boxes");
  static_assert(WTM % 8 == 0 && WTN % 8 == 0, "warp tiles are whole 8-wide fragments");
  static_assert(BN <= 256 && BK <= 256, "TMA box extent limit");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory per CTA");
};

// Fragment -> element map (lane = 4g + t). Every operand tile is staged as
// 8-element-wide TMA boxes with the 64B swizzle (16-B chunk c of a 64-B row at
// smem byte address a moves to c ^ ((a >> 7) & 3)). A fragment covers the 8
// elements x = 8*blk + xmap8(g) of its operand's free dimension; k-step s reads
// the k rows 4s + t. 64-bit shared loads are serviced per half-warp; with this
// map each half-warp's 16 loads hit 16 distinct 8-byte bank slots in BOTH smem
// layouts below, for every s (checked exhaustively). xmap8(2t), xmap8(2t)+1 are
// adjacent, so the epilogue keeps 16-byte stores.
//   XK layout (operand contiguous along x; [x-block][k][8]):
//     byte = blk*BK*64 + 4s*64 + t*64 + (g&1)*8 + J_s
//   KX layout (operand contiguous along k; [k-block][x][8]):
//     byte = (s>>1)*BX*64 + (8*blk + xmap8(g))*64 + (t&1)*8 + J_s
//   J_s = ((jg ^ (t>>1)) << 4) ^ (32*(s&1)),  jg = 2((g>>1)&1) + (g>>2)
__device__ __forceinline__ int xmap8(int g) { return (g & 1) + 4 * ((g >> 1) & 1) + 2 * (g >> 2); }

// QK == true  (mu == 1): P = L  (XK, 2-D map {n_out, K}), Q = T (KX, 2-D map {K, C})
// QK == false (mu  > 1): P = T  (XK, 3-D map {A, K, C}; M runs over a list of
//                         8-row fragments (a-block, c) so batches never pad),
//                        Q = L  (XK, 2-D map {n_out, K})
template <class Cfg, bool QK>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    modeprod_tma_kernel(const __grid_constant__ CUtensorMap mapP,
                        const __grid_constant__ CUtensorMap mapQ, const TmaParams p) {
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr int FM = Cfg::FM, FN = Cfg::FN;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment by pointer arithmetic so the compiler keeps the shared
  // address space (LDS, not generic LD).
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

  if (warp >= Cfg::MMA_WARPS) {
    // ------------------------------------------------------------ producer
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == Cfg::MMA_WARPS && lane == 0) {
      tma_prefetch_desc(&mapP);
      tma_prefetch_desc(&mapQ);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
        int mtile, ntile;
        decode(tile, mtile, ntile);
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
              tma_load_3d(sP, &mapP, &full_bar[stage], 0, k0, static_cast<int32_t>(q0));
            else
              tma_load_4d(sP, &mapP, &full_bar[stage], 0, k0, static_cast<int32_t>(ab0), static_cast<int32_t>(c0));
          } else {
            uint32_t c = c0, ab = ab0;
#pragma unroll 1
            for (int f = 0; f < BM / 8; ++f) {
              // fragments past the end re-load the last valid one (masked later)
              if constexpr (QK) {
                const uint32_t q = (q0 + f <= qlast) ? (q0 + f) : qlast;
                tma_load_2d(sP + f * BK * 64, &mapP, &full_bar[stage], static_cast<int32_t>(8 * q), k0);
              } else {
                if (q0 + f > qlast) {
                  c = qlast / static_cast<uint32_t>(p.AB);
                  ab = qlast - c * static_cast<uint32_t>(p.AB);
                }
                tma_load_3d(sP + f * BK * 64, &mapP, &full_bar[stage], static_cast<int32_t>(8 * ab), k0,
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
              tma_load_3d(sQ, &mapQ, &full_bar[stage], 0, n0, k0 / 8);
            else
              tma_load_3d(sQ, &mapQ, &full_bar[stage], 0, k0, n0 / 8);
          } else if constexpr (QK) {
#pragma unroll 1
            for (int b = 0; b < BK / 8; ++b)
              tma_load_2d(sQ + b * BN * 64, &mapQ, &full_bar[stage], k0 + 8 * b, n0);
          } else {
#pragma unroll 1
            for (int b = 0; b < BN / 8; ++b)
              tma_load_2d(sQ + b * BK * 64, &mapQ, &full_bar[stage], n0 + 8 * b, k0);
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
  const int jg = 2 * ((g >> 1) & 1) + (g >> 2);
  const uint32_t J0 = static_cast<uint32_t>(jg ^ (t >> 1)) << 4;
  const uint32_t xk_off = static_cast<uint32_t>(t * 64 + (g & 1) * 8);
  const uint32_t kx_off = static_cast<uint32_t>(xmap8(g) * 64 + (t & 1) * 8);

  int stage = 0;
  uint32_t phase = 0;
  for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
    int mtile, ntile;
    decode(tile, mtile, ntile);

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
        const uint32_t Js = J0 ^ static_cast<uint32_t>(32 * (s & 1));
        double pf[FM], qf[FN];
#pragma unroll
        for (int fm = 0; fm < FM; ++fm)
          pf[fm] = *reinterpret_cast<const double*>(sP + ((mw >> 3) + fm) * (BK * 64) + (4 * s) * 64 +
                                                    xk_off + Js);
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) {
          if constexpr (QK)
            qf[fn] = *reinterpret_cast<const double*>(sQ + (s >> 1) * (BN * 64) + (nw + 8 * fn) * 64 +
                                                      kx_off + Js);
          else
            qf[fn] = *reinterpret_cast<const double*>(sQ + ((nw >> 3) + fn) * (BK * 64) + (4 * s) * 64 +
                                                      xk_off + Js);
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
    const int mpair = xmap8(2 * t);
#pragma unroll
    for (int fm = 0; fm < FM; ++fm) {
      const uint32_t q = static_cast<uint32_t>(mtile) * (BM / 8) + (mw >> 3) + fm;
      if (q >= static_cast<uint32_t>(p.mfrags)) continue;
      uint32_t c = 0, ab = q;
      if constexpr (!QK) {
        c = q / static_cast<uint32_t>(p.AB);
        ab = q - c * static_cast<uint32_t>(p.AB);
      }
      const int m = 8 * static_cast<int>(ab) + mpair;
      if (m >= p.Mlim) continue;
      double* base = p.D + static_cast<int64_t>(c) * p.bstride + m;
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) {
        const int n = ntile * BN + nw + 8 * fn + xmap8(g);
        if (n < p.N) stg_f64x2(base + static_cast<int64_t>(n) * p.ldD, acc[fm][fn][0], acc[fm][fn][1]);
      }
    }
  }
}

}  // namespace mumode_gpu
