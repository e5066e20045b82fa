// Fused two-mode passes for SMALL extents that are not multiples of 8
// (the paper's d = 6 sizes, n = 12..20, e.g. 18^6 and 20^6): modes (mu,
// mu+1) of a tile in one HBM pass, so a d-mode Tucker reads and writes the
// tensor ceil(d/2) times instead of d times.
//
// The fused_ws / tail_ws kernels are specialised to square extents of 8, 16
// and 24 (their TMA boxes and swizzled fragment maps assume them); these
// kernels take any extents <= 24 at run time:
//   * operands are staged with cp.async (16-byte chunks, zero-filled beyond
//     the tensor) into PADDED shared rows chosen for conflict-free DMMA
//     fragment access instead of TMA swizzle: X rows of 36 doubles (72 words
//     = 8 mod 32: the four k-rows of a B fragment hit disjoint banks),
//     intermediate / output rows of 40 doubles (80 words = 16 mod 32: the two
//     rows of a 128-bit fragment store do) and intermediate k-blocks whose
//     stride is 8 mod 32 words;
//   * the contraction K is padded to a multiple of 4 (P4) and the outputs to
//     multiples of 8 (NF fragments) with zero factor entries, so every DMMA
//     chain is the k-ordered FMA chain over the true k's followed by exact
//     zero terms: results are bitwise those of the per-mode kernels.
//
// spair_kernel (mu >= 2, A even): the streamed tail scheme of tail_ws.cuh --
//   producer warpgroup : cp.async ring of stages X(32 a, K1, 4 k2) per tile
//   group A (4 warps)  : mode mu on each stage -> Ys[k2l][i1][a]
//   group B (8 warps)  : mode mu+1: acc(i1, i2, a) += L2(i2, k2) Ys(k2, i1, a)
//                        stage by stage in registers; at the end of a tile
//                        each warp stages its i1 slices and writes 256-B rows.
// spair1_kernel (mu = 1): every c is independent for both modes, so a stage
//   is a block of CB whole c-slabs: group A runs mode 1, group B mode 2 on
//   the intermediate and writes the contiguous output slabs.
#pragma once
#include "common.cuh"

namespace mumode_gpu {

struct SpairParams {
  const double* X;
  double* S;
  const double* L1;  // N1 x K1, ld N1
  const double* L2;  // N2 x K2, ld N2
  int64_t A, C;
  int K1, N1, K2, N2;
  int64_t ablks, tiles;
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int P4, int NF>
struct SpairCfg {
  static constexpr int KS = P4 / 4;  // k-steps of mode mu
  static constexpr int NP = 8 * NF;  // padded output rows
  // k2 values per stage: 8 where shared memory allows (half the stage
  // hand-offs per unit of work; the output is staged in the tile's last
  // intermediate buffer), else 4 with separate output slots
  static constexpr int KB = 4;  // 8 (one more k4-step per hand-off, 2-deep load ring) measured slower
  static constexpr bool EPI_IN_YS = (KB == 8);
  static constexpr int KQ = KB / 4;     // mode mu+1 k-steps per stage
  static constexpr int UPW = KB / 2;    // mode mu units per group-A warp per stage
  static constexpr int WB = 8, WA = 8;  // 2 + 2 warps per sub-partition; A also issues the loads
  static constexpr int THREADS = (WB + WA) * 32;
  static constexpr int RSX = 36, RSY = 40;
  static constexpr int X_DBL = KB * P4 * RSX;
  static constexpr int YB_DBL = NP * RSY + 4;  // k2l block stride: 8 mod 32 words
  static constexpr int YS_DBL = KB * YB_DBL;
  static constexpr int SLOT_DBL = NP * RSY;
  static constexpr int NYS = EPI_IN_YS ? 2 : 3;
  static constexpr int FIXED = (NYS * YS_DBL + (EPI_IN_YS ? 0 : WB * SLOT_DBL)) * 8 + 1024;
  static constexpr int NBUF_RAW = (227 * 1024 - FIXED) / (X_DBL * 8);
  static constexpr int NBUF = NBUF_RAW > 6 ? 6 : NBUF_RAW;
  static constexpr int SMEM_BYTES = NBUF * X_DBL * 8 + FIXED;
  // setmaxnreg split of the 128-per-thread launch allocation; every
  // sub-partition holds two warps of each group (16384 registers each)
  static constexpr int LAUNCH_REGS = 65536 / THREADS;
  static constexpr int A_REGS = 80, B_REGS = 176;
  static_assert(2 * A_REGS + 2 * B_REGS <= 4 * LAUNCH_REGS, "setmaxnreg budget per sub-partition");
  static_assert(A_REGS <= LAUNCH_REGS && B_REGS >= LAUNCH_REGS, "dec / inc directions");
  static_assert(NBUF >= 2, "shared memory for a 2-deep ring");
  static_assert(!EPI_IN_YS || WB * SLOT_DBL <= YS_DBL, "output staging fits an intermediate buffer");
  static_assert(P4 % 4 == 0 && P4 <= 24 && NF <= 3, "extents up to 24");
};

template <int P4, int NF>
__global__ void __launch_bounds__(SpairCfg<P4, NF>::THREADS, 1) spair_kernel(const SpairParams p) {
  using Cfg = SpairCfg<P4, NF>;
  constexpr int KS = Cfg::KS, NBUF = Cfg::NBUF, NYS = Cfg::NYS, RSX = Cfg::RSX, RSY = Cfg::RSY;
  constexpr int WA = Cfg::WA, WB = Cfg::WB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  double* Xs = reinterpret_cast<double*>(smem_raw);
  double* Ys = Xs + NBUF * Cfg::X_DBL;
  double* Slots = Ys + NYS * Cfg::YS_DBL;  // (KB = 4 only)
  // stage hand-offs between the groups: mbarriers (one arrival per warp)
  uint64_t* yfull = reinterpret_cast<uint64_t*>(Slots + (Cfg::EPI_IN_YS ? 0 : WB * Cfg::SLOT_DBL));
  uint64_t* yfree = yfull + NYS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K1 = p.K1, N1 = p.N1, K2 = p.K2, N2 = p.N2;
  const int64_t A = p.A;
  const int nst = (K2 + Cfg::KB - 1) / Cfg::KB;  // stages per tile

  // rows k1 in [K1, P4) of every X buffer stay zero (never copied into)
  for (int b = 0; b < NBUF; ++b)
    for (int e = threadIdx.x; e < Cfg::KB * (P4 - K1) * RSX; e += blockDim.x) {
      const int r = e / RSX, col = e - r * RSX;
      const int k2l = r / (P4 - K1), k1 = K1 + (r - k2l * (P4 - K1));
      Xs[b * Cfg::X_DBL + (k2l * P4 + k1) * RSX + col] = 0.0;
    }
  if (threadIdx.x == 0) {
    for (int b = 0; b < NYS; ++b) {
      mbar_init(&yfull[b], WA);
      mbar_init(&yfree[b], WB);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();  // before any global access (factors included)

  const int64_t ntiles = (p.tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int64_t nz = ntiles * nst;  // stages of this CTA

  const int g = lane >> 2, t = lane & 3;
  if (warp >= WB) {
    // ------------------------------------------ group A: mode mu, X -> Ys
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(Cfg::A_REGS) : "memory");
    const int wa = warp - WB;
    const int f = wa & 3, kh = wa >> 2;  // a fragment; stage k2 values kh, kh + 2, ...
    // the group's 256 threads also stage X: thread at = wa * 32 + lane copies
    // 16-B chunk j = at & 15 of rows r = at / 16 + 16 i, i.e. (k2l, k1)
    // advanced without divisions
    const int at = wa * 32 + lane, j = at & 15, r0 = at >> 4;
    const int rows = Cfg::KB * K1;
    const int64_t AK1 = A * K1;
    // the issue stream walks (tile, stage) in order: incremental state, no
    // 64-bit divisions on the critical path
    int64_t it_tile = blockIdx.x, it_c = blockIdx.x / p.ablks, it_ab = blockIdx.x - (blockIdx.x / p.ablks) * p.ablks;
    int it_st = 0, it_buf = 0;
    const int k2l0 = r0 / K1, k10 = r0 - k2l0 * K1;
    auto issue = [&]() {  // cp.async of the next stage into buffer it_buf
      const int64_t a = 32 * it_ab + 2 * j;
      const bool a_ok = a < A;
      double* X = Xs + it_buf * Cfg::X_DBL;
      const int64_t base = a + AK1 * (Cfg::KB * it_st + static_cast<int64_t>(K2) * it_c);
      int k2l = k2l0, k1 = k10;
      for (int r = r0; r < rows; r += 16) {
        const bool ok = a_ok && Cfg::KB * it_st + k2l < K2;
        cp_async16(X + (k2l * P4 + k1) * RSX + 2 * j, ok ? p.X + base + A * k1 + AK1 * k2l : p.X, ok);
        k1 += 16;
        while (k1 >= K1) {
          k1 -= K1;
          ++k2l;
        }
      }
      if (++it_buf == NBUF) it_buf = 0;
      if (++it_st == nst) {
        it_st = 0;
        it_tile += gridDim.x;
        it_ab += gridDim.x;
        while (it_ab >= p.ablks) {
          it_ab -= p.ablks;
          ++it_c;
        }
      }
    };
    double l1[NF][KS];
#pragma unroll
    for (int nf = 0; nf < NF; ++nf)
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        const int i = 8 * nf + g, k = 4 * s + t;
        l1[nf][s] = (i < N1 && k < K1) ? p.L1[i + static_cast<int64_t>(N1) * k] : 0.0;
      }
    // multistage cp.async pipeline (one commit group per stage, NBUF - 1
    // stages in flight): per stage, wait for this thread's copies of stage z,
    // then one group-A barrier makes every thread's copies visible and
    // certifies that stage z-1's buffer is free for stage z + NBUF - 1
    for (int zz = 0; zz < NBUF - 1; ++zz) {
      if (zz < nz) issue();
      cp_async_commit();
    }
    int yb = 0, buf = 0;
    for (int64_t z = 0; z < nz; ++z) {
      cp_async_wait<NBUF - 2>();
      named_barrier_sync(1, WA * 32);
      if (z + NBUF - 1 < nz) issue();
      cp_async_commit();
      if (z >= NYS) mbar_wait(&yfree[yb], static_cast<uint32_t>((z / NYS - 1) & 1));  // Ys[yb] consumed by group B
      const double* X = Xs + buf * Cfg::X_DBL;
      double* Y = Ys + yb * Cfg::YS_DBL;
#pragma unroll
      for (int ub = 0; ub < Cfg::UPW; ub += 2) {
        double acc[2][NF][2];  // two units: independent chains
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) acc[u][nf][0] = acc[u][nf][1] = 0.0;
#pragma unroll
        for (int s = 0; s < KS; ++s)
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int k2l = kh + 2 * (ub + u);
            const double xf = X[(k2l * P4 + 4 * s + t) * RSX + 8 * f + g];
#pragma unroll
            for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[u][nf][0], acc[u][nf][1], l1[nf][s], xf);
          }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int k2l = kh + 2 * (ub + u);
#pragma unroll
          for (int nf = 0; nf < NF; ++nf)
            *reinterpret_cast<double2*>(Y + k2l * Cfg::YB_DBL + (8 * nf + g) * RSY + 8 * f + 2 * t) =
                make_double2(acc[u][nf][0], acc[u][nf][1]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&yfull[yb]);  // Ys[yb] complete (release after the warp's stores)
      if (++yb == NYS) yb = 0;
      if (++buf == NBUF) buf = 0;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    return;
  }

  // ----------------------------- group B: mode mu+1, Ys -> registers -> HBM
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(Cfg::B_REGS) : "memory");
  constexpr int KQ = Cfg::KQ;
  int64_t z = 0;
  int yb = 0;
  int64_t c = blockIdx.x / p.ablks, ab = blockIdx.x - (blockIdx.x / p.ablks) * p.ablks;
  for (int64_t tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
    const int64_t a0 = 32 * ab;
    double acc[NF][4][NF][2];  // [i1 slice][a fragment][i2 fragment]
#pragma unroll
    for (int ii = 0; ii < NF; ++ii)
#pragma unroll
      for (int F = 0; F < 4; ++F)
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) acc[ii][F][nf][0] = acc[ii][F][nf][1] = 0.0;
    int yb_last = 0;
    bool free_last = false;
#pragma unroll 1
    for (int st = 0; st < nst; ++st, ++z) {
      double l2f[KQ][NF];
#pragma unroll
      for (int q = 0; q < KQ; ++q)
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) {
          const int i = 8 * nf + g, k = Cfg::KB * st + 4 * q + t;
          l2f[q][nf] = (i < N2 && k < K2) ? __ldg(p.L2 + i + static_cast<int64_t>(N2) * k) : 0.0;
        }
      mbar_wait(&yfull[yb], static_cast<uint32_t>((z / NYS) & 1));  // Ys[yb] complete
      const double* Y = Ys + yb * Cfg::YS_DBL;
#pragma unroll
      for (int q = 0; q < KQ; ++q)
#pragma unroll
        for (int ii = 0; ii < NF; ++ii) {
          const int i1 = warp + WB * ii;
          if (i1 < N1) {
#pragma unroll
            for (int F = 0; F < 4; ++F) {
              const double yf = Y[(4 * q + t) * Cfg::YB_DBL + i1 * RSY + 8 * F + g];
#pragma unroll
              for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[ii][F][nf][0], acc[ii][F][nf][1], l2f[q][nf], yf);
            }
          }
        }
      const bool release = z + NYS < nz;
      if (Cfg::EPI_IN_YS && st == nst - 1) {
        yb_last = yb;  // freed after the epilogue has staged through it
        free_last = release;
      } else if (release) {
        asm volatile("fence.acq_rel.cta;\n" ::: "memory");  // this thread's Ys loads are complete
        __syncwarp();
        if (lane == 0) mbar_arrive(&yfree[yb]);
      }
      if (++yb == NYS) yb = 0;
    }
    // epilogue: per i1 slice, stage (i2, a) in this warp's slot, then 256-B rows
    double* slot;
    if constexpr (Cfg::EPI_IN_YS) {
      named_barrier_sync(2 + 2 * NYS, WB * 32);  // every B warp has read the last stage
      slot = Ys + yb_last * Cfg::YS_DBL + warp * Cfg::SLOT_DBL;
    } else {
      slot = Slots + warp * Cfg::SLOT_DBL;
    }
#pragma unroll
    for (int ii = 0; ii < NF; ++ii) {
      const int i1 = warp + WB * ii;
      if (i1 >= N1) continue;
#pragma unroll
      for (int F = 0; F < 4; ++F)
#pragma unroll
        for (int nf = 0; nf < NF; ++nf)
          *reinterpret_cast<double2*>(slot + (8 * nf + g) * RSY + 8 * F + 2 * t) =
              make_double2(acc[ii][F][nf][0], acc[ii][F][nf][1]);
      __syncwarp();
      const int col = 2 * (lane & 15);
      const int64_t a = a0 + col;
      for (int i2 = lane >> 4; i2 < N2; i2 += 2) {
        const double2 v = *reinterpret_cast<const double2*>(slot + i2 * RSY + col);
        if (a < A)
          stg_f64x2(p.S + a + A * (i1 + static_cast<int64_t>(N1) * (i2 + static_cast<int64_t>(N2) * c)), v.x, v.y);
      }
      __syncwarp();
    }
    if (Cfg::EPI_IN_YS && free_last) {
      asm volatile("fence.acq_rel.cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&yfree[yb_last]);
    }
    ab += gridDim.x;
    while (ab >= p.ablks) {
      ab -= p.ablks;
      ++c;
    }
  }
}

// ------------------------------------------------------------------ mu = 1
// X(k1, k2, c), S(i1, i2, c): a stage is CB = 8 whole c-slabs (CB*K1*K2
// contiguous doubles in, CB*N1*N2 out). Shared rows: X [c][k2][k1] with
// RX = 4 mod 8 doubles (B fragments k1 x col, conflict-free), the
// intermediate [c][i1][k2] with the same row rule (mode 2's B fragments k2
// x i1), output slots [c][i2][i1] with RO1 = 8 mod 16 doubles (conflict-free
// 128-bit fragment stores), copied out as contiguous slabs. RO1 = RO.
template <int P4, int NF>
struct Spair1Cfg {
  static constexpr int KS = P4 / 4;
  static constexpr int NP = 8 * NF;
  static constexpr int CB = 8;
  static constexpr int WB = 8, WA = 8;  // A also issues the loads
  static constexpr int THREADS = (WB + WA) * 32;
  static constexpr int RX = (P4 + 3) / 8 * 8 + 4;  // = 4 mod 8 (row stride 8 or 24 mod 32 words), >= P4
  static constexpr int RO = (NP <= 24) ? 24 : 40;  // = 8 mod 16, >= NP
  static constexpr int X_DBL = CB * P4 * RX;       // rows (c, k2) for k2 < P4
  static constexpr int Y_DBL = CB * NP * RX;       // rows (c, i1), k2 along the row
  static constexpr int SLOT_DBL = NP * RO;
  static constexpr int NYS = (P4 <= 20) ? 3 : 2;
  static constexpr int FIXED = (NYS * Y_DBL + WB * SLOT_DBL) * 8 + 1024;
  static constexpr int NBUF_RAW = (227 * 1024 - FIXED) / (X_DBL * 8);
  static constexpr int NBUF = NBUF_RAW > 6 ? 6 : NBUF_RAW;
  static constexpr int SMEM_BYTES = NBUF * X_DBL * 8 + FIXED;
  static_assert(NBUF >= 2, "shared memory for a 2-deep ring");
  static_assert(P4 % 4 == 0 && P4 <= 24 && NF <= 3, "extents up to 24");
};

template <int P4, int NF>
__global__ void __launch_bounds__(Spair1Cfg<P4, NF>::THREADS, 1) spair1_kernel(const SpairParams p) {
  using Cfg = Spair1Cfg<P4, NF>;
  constexpr int KS = Cfg::KS, NBUF = Cfg::NBUF, NYS = Cfg::NYS, RX = Cfg::RX, RO = Cfg::RO, NP = Cfg::NP;
  constexpr int WA = Cfg::WA, WB = Cfg::WB, CB = Cfg::CB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  double* Xs = reinterpret_cast<double*>(smem_raw);
  double* Ys = Xs + NBUF * Cfg::X_DBL;
  double* Slots = Ys + NYS * Cfg::Y_DBL;
  uint64_t* yfull = reinterpret_cast<uint64_t*>(Slots + WB * Cfg::SLOT_DBL);  // hand-offs, one arrival per warp
  uint64_t* yfree = yfull + NYS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K1 = p.K1, N1 = p.N1, K2 = p.K2, N2 = p.N2;
  const int64_t C = p.C;
  const int64_t nstage = (C + CB - 1) / CB;

  // k1 columns in [K1, RX) of every X row and k2 columns in [K2, RX) of every
  // intermediate row stay zero (the padded k-steps read them)
  for (int b = 0; b < NBUF; ++b)
    for (int e = threadIdx.x; e < CB * P4 * RX; e += blockDim.x)
      if (e % RX >= K1) Xs[b * Cfg::X_DBL + e] = 0.0;
  for (int b = 0; b < NYS; ++b)
    for (int e = threadIdx.x; e < CB * NP * RX; e += blockDim.x)
      if (e % RX >= K2) Ys[b * Cfg::Y_DBL + e] = 0.0;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NYS; ++b) {
      mbar_init(&yfull[b], WA);
      mbar_init(&yfree[b], WB);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();

  const int64_t nz = (nstage - blockIdx.x + gridDim.x - 1) / gridDim.x;  // stages of this CTA

  const int g = lane >> 2, t = lane & 3;
  if (warp >= WB) {
    // --------------------------- group A: mode 1, columns (c, k2) of X -> Y
    const int wa = warp - WB;
    double l1[NF][KS];
#pragma unroll
    for (int nf = 0; nf < NF; ++nf)
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        const int i = 8 * nf + g, k = 4 * s + t;
        l1[nf][s] = (i < N1 && k < K1) ? p.L1[i + static_cast<int64_t>(N1) * k] : 0.0;
      }
    const int nfr = K2;  // column fragments: CB * K2 / 8
    // the group's 256 threads also stage X: chunk e = at + 256 i of a stage
    // is (row r, chunk j) of hk 16-B chunks per (c, k2) row
    const int at = wa * 32 + lane;
    const int hk = K1 / 2;
    const int nch = CB * K2 * hk;
    const int r_init = at / hk, j_init = at - r_init * hk;
    const int cl_init = r_init / K2, k2_init = r_init - cl_init * K2;
    const int dr = (WA * 32) / hk, dj = WA * 32 - dr * hk;
    auto issue = [&](int64_t zz) {
      const int64_t st = blockIdx.x + zz * gridDim.x;
      double* X = Xs + (zz % NBUF) * Cfg::X_DBL;
      const int64_t c0 = st * CB;
      const double* src0 = p.X + static_cast<int64_t>(K1) * K2 * c0;
      int r = r_init, j = j_init, cl = cl_init, k2 = k2_init;  // r = cl * K2 + k2
      for (int e = at; e < nch; e += WA * 32) {
        const bool ok = c0 + cl < C;
        cp_async16(X + (cl * P4 + k2) * RX + 2 * j, ok ? src0 + static_cast<int64_t>(K1) * r + 2 * j : p.X, ok);
        int step = dr;
        j += dj;
        if (j >= hk) {
          j -= hk;
          ++step;
        }
        r += step;
        k2 += step;
        while (k2 >= K2) {
          k2 -= K2;
          ++cl;
        }
      }
    };
    for (int64_t zz = 0; zz < NBUF - 1; ++zz) {  // multistage pipeline as in spair_kernel
      if (zz < nz) issue(zz);
      cp_async_commit();
    }
    for (int64_t z = 0; z < nz; ++z) {
      const int yb = static_cast<int>(z % NYS);
      const int buf = static_cast<int>(z % NBUF);
      cp_async_wait<NBUF - 2>();
      named_barrier_sync(1, WA * 32);
      if (z + NBUF - 1 < nz) issue(z + NBUF - 1);
      cp_async_commit();
      if (z >= NYS) mbar_wait(&yfree[yb], static_cast<uint32_t>((z / NYS - 1) & 1));
      const double* X = Xs + buf * Cfg::X_DBL;
      double* Y = Ys + yb * Cfg::Y_DBL;
      for (int f0 = wa; f0 < nfr; f0 += 2 * WA) {  // two column fragments: independent chains
        const bool two = f0 + WA < nfr;
        double acc[2][NF][2];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) acc[u][nf][0] = acc[u][nf][1] = 0.0;
        const double* xr[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int col = 8 * (f0 + (two ? u * WA : 0)) + g;  // (c, k2) = (col / K2, col % K2)
          const int ccl = col / K2, ck2 = col - ccl * K2;
          xr[u] = X + (ccl * P4 + ck2) * RX + t;
        }
#pragma unroll
        for (int s = 0; s < KS; ++s)
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const double xf = xr[u][4 * s];
#pragma unroll
            for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[u][nf][0], acc[u][nf][1], l1[nf][s], xf);
          }
        // D(i1 = 8nf + g, cols 8f + 2t, +1) -> Y[(c, i1)][k2]
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (u == 1 && !two) break;
          const int f = f0 + u * WA;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int cc = 8 * f + 2 * t + h;
            const int ycl = cc / K2, yk2 = cc - ycl * K2;
#pragma unroll
            for (int nf = 0; nf < NF; ++nf) Y[(ycl * NP + 8 * nf + g) * RX + yk2] = acc[u][nf][h];
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&yfull[yb]);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    return;
  }

  // --------------------- group B: mode 2 on slab c = warp, out -> HBM
  double l2[NF][KS];
#pragma unroll
  for (int nf = 0; nf < NF; ++nf)
#pragma unroll
    for (int s = 0; s < KS; ++s) {
      const int i = 8 * nf + g, k = 4 * s + t;
      l2[nf][s] = (i < N2 && k < K2) ? p.L2[i + static_cast<int64_t>(N2) * k] : 0.0;
    }
  double* slot = Slots + warp * Cfg::SLOT_DBL;
  const int nout = N1 * N2;
  int64_t z = 0;
  for (int64_t st = blockIdx.x; st < nstage; st += gridDim.x, ++z) {
    const int yb = static_cast<int>(z % NYS);
    mbar_wait(&yfull[yb], static_cast<uint32_t>((z / NYS) & 1));
    const double* Y = Ys + yb * Cfg::Y_DBL + warp * NP * RX;  // this warp's slab
    double acc[NF][NF][2];  // [i1 fragment][i2 fragment]
#pragma unroll
    for (int f = 0; f < NF; ++f)
#pragma unroll
      for (int nf = 0; nf < NF; ++nf) acc[f][nf][0] = acc[f][nf][1] = 0.0;
#pragma unroll
    for (int s = 0; s < KS; ++s)
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const double yf = Y[(8 * f + g) * RX + 4 * s + t];
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[f][nf][0], acc[f][nf][1], l2[nf][s], yf);
      }
    if (z + NYS < nz) {
      asm volatile("fence.acq_rel.cta;\n" ::: "memory");  // this thread's Y loads are complete
      __syncwarp();
      if (lane == 0) mbar_arrive(&yfree[yb]);
    }
    // D(i2 = 8nf + g, i1 = 8f + 2t, +1) -> slot[i2][i1], then the contiguous slab
#pragma unroll
    for (int f = 0; f < NF; ++f)
#pragma unroll
      for (int nf = 0; nf < NF; ++nf)
        *reinterpret_cast<double2*>(slot + (8 * nf + g) * RO + 8 * f + 2 * t) = make_double2(acc[f][nf][0], acc[f][nf][1]);
    __syncwarp();
    const int64_t c = st * CB + warp;
    if (c < C) {
      double* dst = p.S + static_cast<int64_t>(nout) * c;
      for (int e = lane; e < nout; e += 32) {
        const int i2 = e / N1, i1 = e - i2 * N1;
        dst[e] = slot[i2 * RO + i1];
      }
    }
    __syncwarp();
  }
}

}  // namespace mumode_gpu
