// One mu-mode product on device buffers: the job description, TMA
// legality, the tile-configuration cost model and the launchers of every
// kernel path (TMA/DMMA, LDG-staged DMMA, SIMT), and run_job, which picks the
// path. Included by mumode_gpu.cu after the handle / error definitions (not
// a standalone header).
#pragma once

namespace mumode_gpu {

// ------------------------------------------------------------------ one product
// S(a, i, c) = sum_k op(L)(i, k) T(a, k, c); op(L)(i,k) = L[i*sLi + k*sLk].
struct ModeJob {
  const double* T;
  const double* L;
  double* S;
  int64_t A, K, N, C;
  int64_t sLi, sLk;
  bool cplx;
  bool conj;
  bool accumulate = false;  // S += T x_mu op(L)
  const ScatterParams* scat = nullptr;  // device table: scatter the (rows x C) result to ranks (S unused)
  const double* div_front = nullptr;    // last mode: S(a, n) /= (div_front[a] + div_last[n])
  const double* div_last = nullptr;
};

// Compiled tile configurations (BM, BN, BK, stages, warps along M, along N).
using CfgBig = TmaCfg<128, 128, 16, 6, 4, 4>;  // 16 MMA warps, 32x32 warp tiles, 6-stage ring (C2-class shapes)
using CfgTM = TmaCfg<128, 40, 40, 3, 16, 1>;   // T-side M, small L-side N (n = 40k)
using CfgLM = TmaCfg<40, 128, 40, 3, 1, 16>;   // small L-side M, T-side N (mode 1, n = 40k)
using CfgMid = TmaCfg<64, 128, 32, 4, 2, 4>;   // 32x32 warp tiles
using CfgSmall = TmaCfg<32, 32, 32, 2, 2, 4>;  // 16x8 warp tiles: spreads small products over SMs
using CfgTM48 = TmaCfg<128, 48, 48, 3, 16, 1>;  // n = 48k (the paper's 144 / 288 / 336) and 324 (7 x 48)
using CfgLM48 = TmaCfg<48, 128, 48, 3, 1, 16>;
using CfgTM56 = TmaCfg<128, 56, 32, 4, 16, 1>;  // n = 56k (112, 168, 224, 280, 336) and 208 / 216 (4 x 56)
using CfgLM56 = TmaCfg<56, 128, 32, 4, 1, 16>;
// complex128 (E = 2): 4 real DMMAs per complex MAC, 16-B elements
// (four accumulator chains per complex output: warp tiles hold 32 outputs)
using CfgCa = TmaCfg<64, 64, 16, 6, 2, 4, 2>;  // 8 MMA warps, 32x16 complex warp tiles
using CfgCb = TmaCfg<128, 32, 16, 5, 4, 2, 2>;  // 8 MMA warps, 32x16
using CfgCc = TmaCfg<96, 32, 16, 4, 4, 4, 2>;   // 24x8 warp tiles, fine-grained
using CfgCd = TmaCfg<192, 16, 16, 4, 8, 1, 2>;

static bool aligned16(const void* p) { return aligned16_ptr(p); }

// Can the TMA/DMMA kernel describe this job? (16-byte strides and bases,
// forward layout of L, real, even M, sizes within int32 coordinates.)
static bool tma_ok(const ModeJob& j) {
  if (j.conj) return false;
  if (j.cplx) {  // 16-byte elements: every stride is 16-B aligned
    if (j.sLi != 1 || !aligned16(j.T) || !aligned16(j.L) || !aligned16(j.S)) return false;
    const int64_t lim = int64_t(1) << 30;
    return j.N < lim && j.K < lim && j.C < lim && j.A < lim && (j.A + 7) / 8 * j.C < lim;
  }
  if (j.sLi != 1) return false;  // L must be used forward: op(L) = L, ld = N
  if (!aligned16(j.T) || !aligned16(j.L) || !aligned16(j.S)) return false;
  if (j.sLk % 2) return false;
  const int64_t lim = int64_t(1) << 31;
  if (j.N >= lim || j.K >= lim || j.C >= lim || j.A >= lim) return false;
  if (j.A == 1) {  // mode 1: M = N_out, Q = T (K x C)
    if (j.N % 2 || j.K % 2) return false;
  } else {
    if (j.A % 2) return false;
    if ((j.A + 7) / 8 * j.C >= lim) return false;
  }
  return true;
}

static bool tma_worthwhile(const ModeJob& j) {
  const int64_t M = (j.A == 1) ? j.N : j.A;
  return M >= 16 && j.K >= 16 && ((j.A == 1) ? j.C : j.N) >= 16;
}

struct TileChoice {
  int cfg;  // 0 Big, 1 TM, 2 LM, 3 Mid
  double cost;
};

// Wave-quantised padded work: waves * (BM * BN * K_padded) / efficiency.
template <class Cfg>
static double tile_cost(int64_t mfrags, int64_t N, int64_t K, int sms, double eff) {
  const int64_t mt = (mfrags + Cfg::BM / 8 - 1) / (Cfg::BM / 8);
  const int64_t nt = (N + Cfg::BN - 1) / Cfg::BN;
  const int64_t tiles = mt * nt;
  const int64_t waves = (tiles + sms - 1) / sms;
  const int64_t kp = (K + Cfg::BK - 1) / Cfg::BK * Cfg::BK;
  return double(waves) * double(Cfg::BM) * double(Cfg::BN) * double(kp) / eff;
}

static int choose_cfg(const ModeJob& j, int sms) {
  const bool mode1 = (j.A == 1);
  const int64_t mfrags = mode1 ? (j.N + 7) / 8 : (j.A + 7) / 8 * j.C;
  const int64_t N = mode1 ? j.C : j.N;
  if (j.cplx) {
    const double c[4] = {tile_cost<CfgCa>(mfrags, N, j.K, sms, 1.00),
                         tile_cost<CfgCb>(mfrags, N, j.K, sms, 1.00),
                         tile_cost<CfgCc>(mfrags, N, j.K, sms, 0.97),
                         tile_cost<CfgCd>(mfrags, N, j.K, sms, 0.96)};
    int best = 0;
    for (int i = 1; i < 4; ++i)
      if (c[i] < c[best]) best = i;
    return 4 + best;
  }
  // relative per-tile efficiency of the narrow-N (40/48/56) and narrow-M
  // families against the 128x128 tiles: 0.96 -> 0.99 measured better at
  // 384^3 (34.9 -> 35.7 TF/s), 456^3 (31.1 -> 32.5), 464^3 (32.1 -> 33.7), no
  // size slower (tools/auto_sweep.py 176..512, 200^3 and 256^3 unchanged)
  constexpr double tm_eff = 0.99;
  const double c0 = tile_cost<CfgBig>(mfrags, N, j.K, sms, 1.00);
  const double c1 = tile_cost<CfgTM>(mfrags, N, j.K, sms, tm_eff);
  const double c2 = tile_cost<CfgLM>(mfrags, N, j.K, sms, tm_eff);
  const double c3 = tile_cost<CfgMid>(mfrags, N, j.K, sms, 0.97);
  // small tiles reuse operands poorly; they win only when they save waves
  // (products of a few tiles: C1's 100 x 100 modes take 16 CTAs, not 3).
  // tools/small_sweep.py, GPU time per Tucker without / with it: 100^2
  // 15.8 -> 8.0 us, 256^2 27.6 -> 8.8, 512^2 47.6 -> 26.4, 48^3 18.8 -> 8.3,
  // 64^3 19.4 -> 11.1, >= 80^3 unchanged (efficiency 0.4-0.6 choose alike,
  // 0.25 gives up 512^2 and 64^3)
  const double c8 = tile_cost<CfgSmall>(mfrags, N, j.K, sms, 0.5);
  const double c9 = tile_cost<CfgTM48>(mfrags, N, j.K, sms, tm_eff);
  const double c10 = tile_cost<CfgLM48>(mfrags, N, j.K, sms, tm_eff);
  const double c11 = tile_cost<CfgTM56>(mfrags, N, j.K, sms, tm_eff);
  const double c12 = tile_cost<CfgLM56>(mfrags, N, j.K, sms, tm_eff);
  int best = 0;
  double bc = c0;
  if (c1 < bc) best = 1, bc = c1;
  if (c2 < bc) best = 2, bc = c2;
  if (c3 < bc) best = 3, bc = c3;
  if (c8 < bc) best = 8, bc = c8;
  if (c9 < bc * 0.995) best = 9, bc = c9;  // the 48-wide tiles only where they save work
  if (c10 < bc * 0.995) best = 10, bc = c10;
  if (c11 < bc * 0.995) best = 11, bc = c11;
  if (c12 < bc * 0.995) best = 12, bc = c12;
  return best;
}

// Tensor maps and kernel parameters of one mode product for tile config Cfg
// (shared by the single-mode launch and the chain kernel).
template <class Cfg>
static int tma_setup(mumode_handle_s* h, const ModeJob& j, const CUtensorMap** mpo, const CUtensorMap** mqo,
                     TmaParams& p) {
  const CUtensorMap* mp = nullptr;
  const CUtensorMap* mq = nullptr;
  p = TmaParams{};
  p.D = j.S;
  const bool mode1 = (j.A == 1);
  constexpr uint32_t BM8 = Cfg::BM / 8, BN8 = Cfg::BN / 8, BK8 = Cfg::BK / 8;
  // all map dims/strides in doubles: e doubles per element, 8e per box row
  constexpr uint64_t e = Cfg::E;
  constexpr uint32_t box0 = 8 * Cfg::E;
  constexpr bool sw = (Cfg::E == 2);
  if (mode1) {
    // P = L (n_out x K, ld = sLk), Q = T (K x C, K contiguous)
    p.p_blocked = (j.N % 8 == 0);
    if (p.p_blocked) {
      uint64_t d[3] = {box0, uint64_t(j.K), uint64_t(j.N / 8)}, st[2] = {e * uint64_t(j.sLk), 8 * e};
      uint32_t b[3] = {box0, Cfg::BK, BM8};
      MM_TRY(get_map(h, j.L, 3, d, st, b, &mp, sw));
    } else {
      uint64_t d[2] = {e * uint64_t(j.N), uint64_t(j.K)}, st[1] = {e * uint64_t(j.sLk)};
      uint32_t b[2] = {box0, Cfg::BK};
      MM_TRY(get_map(h, j.L, 2, d, st, b, &mp, sw));
    }
    p.q_blocked = (j.K % 8 == 0);
    if (p.q_blocked) {
      uint64_t d[3] = {box0, uint64_t(j.C), uint64_t(j.K / 8)}, st[2] = {e * uint64_t(j.K), 8 * e};
      uint32_t b[3] = {box0, Cfg::BN, BK8};
      MM_TRY(get_map(h, j.T, 3, d, st, b, &mq, sw));
    } else {
      uint64_t d[2] = {e * uint64_t(j.K), uint64_t(j.C)}, st[1] = {e * uint64_t(j.K)};
      uint32_t b[2] = {box0, Cfg::BN};
      MM_TRY(get_map(h, j.T, 2, d, st, b, &mq, sw));
    }
    p.Mlim = int(j.N);
    p.N = int(j.C);
    p.ldD = j.N;
    p.bstride = 0;
    p.AB = int((j.N + 7) / 8);
    p.mfrags = p.AB;
  } else {
    // P = T (A x K x C, A contiguous), Q = L (n_out x K, ld = sLk)
    const int64_t AB = (j.A + 7) / 8;
    p.p_blocked = (j.A % 8 == 0) && (AB % BM8 == 0);
    if (p.p_blocked) {
      uint64_t d[4] = {box0, uint64_t(j.K), uint64_t(AB), uint64_t(j.C)};
      uint64_t st[3] = {e * uint64_t(j.A), 8 * e, e * uint64_t(j.A * j.K)};
      uint32_t b[4] = {box0, Cfg::BK, BM8, 1};
      MM_TRY(get_map(h, j.T, 4, d, st, b, &mp, sw));
    } else {
      uint64_t d[3] = {e * uint64_t(j.A), uint64_t(j.K), uint64_t(j.C)};
      uint64_t st[2] = {e * uint64_t(j.A), e * uint64_t(j.A * j.K)};
      uint32_t b[3] = {box0, Cfg::BK, 1};
      MM_TRY(get_map(h, j.T, 3, d, st, b, &mp, sw));
    }
    p.q_blocked = (j.N % 8 == 0);
    if (p.q_blocked) {
      uint64_t d[3] = {box0, uint64_t(j.K), uint64_t(j.N / 8)}, st[2] = {e * uint64_t(j.sLk), 8 * e};
      uint32_t b[3] = {box0, Cfg::BK, BN8};
      MM_TRY(get_map(h, j.L, 3, d, st, b, &mq, sw));
    } else {
      uint64_t d[2] = {e * uint64_t(j.N), uint64_t(j.K)}, st[1] = {e * uint64_t(j.sLk)};
      uint32_t b[2] = {box0, Cfg::BK};
      MM_TRY(get_map(h, j.L, 2, d, st, b, &mq, sw));
    }
    p.Mlim = int(j.A);
    p.N = int(j.N);
    p.ldD = j.A;
    p.bstride = j.A * j.N;
    p.AB = int(AB);
    p.mfrags = AB * j.C;
  }
  p.K = int(j.K);
  p.mt = int((p.mfrags + Cfg::BM / 8 - 1) / (Cfg::BM / 8));
  p.nt = (p.N + Cfg::BN - 1) / Cfg::BN;
  p.tiles = int64_t(p.mt) * p.nt;
  p.scat = j.scat;
  p.div_front = j.div_front;
  p.div_last = j.div_last;
  *mpo = mp;
  *mqo = mq;
  return MUMODE_OK;
}

template <class Cfg>
static int launch_tma(mumode_handle_s* h, const ModeJob& j) {
  const CUtensorMap* mp = nullptr;
  const CUtensorMap* mq = nullptr;
  TmaParams p;
  MM_TRY(tma_setup<Cfg>(h, j, &mp, &mq, p));
  const bool mode1 = (j.A == 1);
  const int grid = static_cast<int>(std::min<int64_t>(p.tiles, persistent_sms(h)));
  if (j.div_front) {
    if constexpr (Cfg::E == 1) {
      if (mode1 || j.C != 1) return fail(MUMODE_ERR_ARGUMENT, "divide epilogue: last mode of order >= 2 only");
      auto k = modeprod_tma_kernel<Cfg, false, 3>;
      MM_TRY(smem_opt_in(k, Cfg::SMEM_BYTES));
      MM_TRY(launch_pdl(k, grid, Cfg::THREADS, Cfg::SMEM_BYTES, h->stream, *mp, *mq, p));
    } else {
      return fail(MUMODE_ERR_ARGUMENT, "divide epilogue is real-only");
    }
  } else if (j.scat) {
    auto k = mode1 ? modeprod_tma_kernel<Cfg, true, 2> : modeprod_tma_kernel<Cfg, false, 2>;
    MM_TRY(smem_opt_in(k, Cfg::SMEM_BYTES));
    MM_TRY(launch_pdl(k, grid, Cfg::THREADS, Cfg::SMEM_BYTES, h->stream, *mp, *mq, p));
  } else if (mode1) {
    auto k = modeprod_tma_kernel<Cfg, true>;
    MM_TRY(smem_opt_in(k, Cfg::SMEM_BYTES));
    MM_TRY(launch_pdl(k, grid, Cfg::THREADS, Cfg::SMEM_BYTES, h->stream, *mp, *mq, p));
  } else if (j.accumulate) {
    auto k = modeprod_tma_kernel<Cfg, false, 1>;
    MM_TRY(smem_opt_in(k, Cfg::SMEM_BYTES));
    MM_TRY(launch_pdl(k, grid, Cfg::THREADS, Cfg::SMEM_BYTES, h->stream, *mp, *mq, p));
  } else {
    auto k = modeprod_tma_kernel<Cfg, false>;
    MM_TRY(smem_opt_in(k, Cfg::SMEM_BYTES));
    MM_TRY(launch_pdl(k, grid, Cfg::THREADS, Cfg::SMEM_BYTES, h->stream, *mp, *mq, p));
  }
  MM_CUDA(cudaGetLastError());
  h->launches++;
  return MUMODE_OK;
}

static int launch_tma_auto(mumode_handle_s* h, const ModeJob& j) {
  const int forced = (h->policy >= 3 && h->policy <= 6) ? h->policy - 3 : -1;
  int cfg = choose_cfg(j, h->num_sms);
  if (forced >= 0) cfg = j.cplx ? 4 + forced : forced;
  if (!j.cplx && h->policy >= 18 && h->policy <= 21) cfg = h->policy - 9;  // 48- / 56-wide tiles forced (tests)
  switch (cfg) {
    case 11: return launch_tma<CfgTM56>(h, j);
    case 12: return launch_tma<CfgLM56>(h, j);
    case 9: return launch_tma<CfgTM48>(h, j);
    case 10: return launch_tma<CfgLM48>(h, j);
    case 1: return launch_tma<CfgTM>(h, j);
    case 2: return launch_tma<CfgLM>(h, j);
    case 3: return launch_tma<CfgMid>(h, j);
    case 4: return launch_tma<CfgCa>(h, j);
    case 5: return launch_tma<CfgCb>(h, j);
    case 6: return launch_tma<CfgCc>(h, j);
    case 7: return launch_tma<CfgCd>(h, j);
    case 8: return launch_tma<CfgSmall>(h, j);
    default: return launch_tma<CfgBig>(h, j);
  }
}

static int launch_generic(mumode_handle_s* h, const ModeJob& j) {
  GenericArgs g{j.T, j.L, j.S, j.A, j.K, j.N, j.C, j.sLi, j.sLk, j.conj ? 1 : 0, j.accumulate ? 1 : 0};
  const int64_t nfib = j.A * j.C;
  dim3 grid(static_cast<unsigned>((nfib + kGenFibers - 1) / kGenFibers),
            static_cast<unsigned>((j.N + kGenRows - 1) / kGenRows));
  if (grid.y > 65535) return fail(MUMODE_ERR_SIZE, "mode product output extent too large");
  if (j.cplx)
    modeprod_generic_kernel<true><<<grid, kGenThreads, 0, h->stream>>>(g);
  else
    modeprod_generic_kernel<false><<<grid, kGenThreads, 0, h->stream>>>(g);
  MM_CUDA(cudaGetLastError());
  h->launches++;
  return MUMODE_OK;
}

// LDG-staged DMMA kernel for real shapes the TMA path cannot describe.
constexpr int kLdgBM = 64, kLdgBN = 64, kLdgBK = 16, kLdgWM = 2, kLdgWN = 2;

static int launch_ldg(mumode_handle_s* h, const ModeJob& j) {
  LdgArgs g{};
  g.T = j.T;
  g.L = j.L;
  g.S = j.S;
  g.A = j.A;
  g.K = j.K;
  g.N = j.N;
  g.C = j.C;
  g.sLi = j.sLi;
  g.sLk = j.sLk;
  g.accumulate = j.accumulate ? 1 : 0;
  const bool mode1 = (j.A == 1);
  if (mode1) {
    g.Mlim = j.N;
    g.ntot = j.C;
    g.AB = int((j.N + 7) / 8);
    g.mfrags = g.AB;
  } else {
    g.Mlim = j.A;
    g.ntot = j.N;
    g.AB = int((j.A + 7) / 8);
    g.mfrags = int64_t(g.AB) * j.C;
  }
  g.mt = int((g.mfrags + kLdgBM / 8 - 1) / (kLdgBM / 8));
  g.nt = int((g.ntot + kLdgBN - 1) / kLdgBN);
  const int64_t tiles = int64_t(g.mt) * g.nt;
  if (tiles >= (int64_t(1) << 31)) return fail(MUMODE_ERR_SIZE, "mode product too large for one launch");
  constexpr int smem = 2 * (kLdgBM + kLdgBN) * kLdgBK * 8 + 1024;
  if (mode1) {
    auto k = modeprod_ldg_kernel<true, kLdgBM, kLdgBN, kLdgBK, kLdgWM, kLdgWN>;
    MM_TRY(smem_opt_in(k, smem));
    k<<<static_cast<unsigned>(tiles), kLdgWM * kLdgWN * 32, smem, h->stream>>>(g);
  } else {
    auto k = modeprod_ldg_kernel<false, kLdgBM, kLdgBN, kLdgBK, kLdgWM, kLdgWN>;
    MM_TRY(smem_opt_in(k, smem));
    k<<<static_cast<unsigned>(tiles), kLdgWM * kLdgWN * 32, smem, h->stream>>>(g);
  }
  MM_CUDA(cudaGetLastError());
  h->launches++;
  return MUMODE_OK;
}

static bool ldg_worthwhile(const ModeJob& j) {
  const int64_t M = (j.A == 1) ? j.N : j.A;
  return M >= 16 && j.K >= 8 && ((j.A == 1) ? j.C : j.N) >= 16;
}

// ------------------------------------------------------------ skinny products
// Small-extent real products (skinny.cuh): HBM-bound, 32-wide tiles with
// 256-B rows. Policy 13 disables the path (auto otherwise).
static bool skinny_ok(const mumode_handle_s* h, const ModeJob& j) {
  if (j.cplx || j.conj || j.scat || j.div_front || (j.accumulate && j.A == 1)) return false;
  if (!(h->policy == 0 || h->policy == 7 || h->policy == 9 || h->policy == 10 || h->policy == 12 || h->policy == 14 ||
        h->policy == 15 || h->policy == 16 || h->policy == 17))
    return false;
  if (j.K > 32 || j.N > 32 || !aligned16(j.T) || !aligned16(j.S)) return false;
  if (j.A == 1) {
    // TMA box coordinates are int32: fibre offsets up to C + 32 TC
    if ((j.K & 1) || (j.N & 1) || j.C >= (int64_t(1) << 31) - 1024) return false;
    return j.C >= int64_t(64) * h->num_sms;  // enough 32-fibre tiles to fill the SMs
  }
  if (j.A % 2 != 0 || j.A >= (int64_t(1) << 31) - 1024 || j.C >= (int64_t(1) << 31) - 1024) return false;
  // 16-a tiles (A not a multiple of 16) pay off from A ~ 64 (18^6 modes 3/4,
  // A = 324 / 5832: 300 -> 193 us); for A = 12..24 they waste up to a third
  // of every box, so A <= 32 takes whole c-slabs (skinny_slab_kernel)
  if (j.A % 16 != 0 && j.A < 64) {
    if (j.A > 32) return false;
    const int P = int((std::max(j.K, j.N) + 7) / 8 * 8);
    const int64_t tc = std::max<int64_t>(1, std::min<int64_t>(256, (32 * P) / (P * j.A)));
    return (j.C + tc - 1) / tc >= int64_t(2) * h->num_sms;
  }
  return ((j.A + 31) / 32) * j.C >= int64_t(2) * h->num_sms;
}

template <int P, int TA>
static int launch_skinny_p(mumode_handle_s* h, const ModeJob& j) {
  using Cfg = SkinnyCfg<P, TA>;
  constexpr uint32_t TC = Cfg::TC;
  const CUtensorMap *mx = nullptr, *ms = nullptr;
  SkinnyParams p{j.L, j.sLi, j.sLk, int(j.K), int(j.N), 0, 0, int(j.A), int(TC), 0};
  const bool mode1 = (j.A == 1);
  if (TA == 16) {
    // A even, not a multiple of 16: 3-D view {A, K, C}, boxes {16 a, P, TC c}
    uint64_t dx[3] = {uint64_t(j.A), uint64_t(j.K), uint64_t(j.C)}, sx[2] = {uint64_t(j.A), uint64_t(j.A * j.K)};
    uint64_t ds[3] = {uint64_t(j.A), uint64_t(j.N), uint64_t(j.C)}, ss[2] = {uint64_t(j.A), uint64_t(j.A * j.N)};
    uint32_t b[3] = {16, P, TC};
    MM_TRY(get_map(h, j.T, 3, dx, sx, b, &mx, 1));
    MM_TRY(get_map(h, j.S, 3, ds, ss, b, &ms, 1));
    p.ablks = (j.A + 15) / 16;
    p.tiles = p.ablks * ((j.C + TC - 1) / TC);
  } else if (mode1) {
    // boxes {P k, 32 TC fibres}
    uint64_t dx[2] = {uint64_t(j.K), uint64_t(j.C)}, sx[1] = {uint64_t(j.K)};
    uint64_t ds[2] = {uint64_t(j.N), uint64_t(j.C)}, ss[1] = {uint64_t(j.N)};
    uint32_t b[2] = {P, 32 * TC};
    MM_TRY(get_map(h, j.T, 2, dx, sx, b, &mx, 2));
    MM_TRY(get_map(h, j.S, 2, ds, ss, b, &ms, 2));
    p.tiles = (j.C + 32 * TC - 1) / (32 * TC);
  } else {
    // 5-D view {16, 2, K, A/32, C} (a-block as its own dimension): a tile's TC
    // boxes run along c, or along the a-blocks when C < TC (e.g. the last
    // mode, C = 1)
    const int64_t nab = j.A / 32;
    p.a_major = (j.C < int64_t(TC)) ? 1 : 0;
    uint64_t dx[5] = {16, 2, uint64_t(j.K), uint64_t(nab), uint64_t(j.C)};
    uint64_t sx[4] = {16, uint64_t(j.A), 32, uint64_t(j.A * j.K)};
    uint64_t ds[5] = {16, 2, uint64_t(j.N), uint64_t(nab), uint64_t(j.C)};
    uint64_t ss[4] = {16, uint64_t(j.A), 32, uint64_t(j.A * j.N)};
    uint32_t b[5] = {16, 2, P, p.a_major ? TC : 1u, p.a_major ? 1u : TC};
    MM_TRY(get_map(h, j.T, 5, dx, sx, b, &mx, 1));
    MM_TRY(get_map(h, j.S, 5, ds, ss, b, &ms, 1));
    if (p.a_major) {
      p.ablks = (nab + TC - 1) / TC;
      p.tiles = p.ablks * j.C;
    } else {
      p.ablks = nab;
      p.tiles = nab * ((j.C + TC - 1) / TC);
    }
  }
  const int grid = static_cast<int>(std::min<int64_t>(p.tiles, persistent_sms(h)));
  auto k = TA == 16 ? (j.accumulate ? skinny_kernel<P, false, 16, true> : skinny_kernel<P, false, 16>)
                    : (mode1 ? skinny_kernel<P, true>
                             : (j.accumulate ? skinny_kernel<P, false, 32, true> : skinny_kernel<P, false>));
  MM_TRY(smem_opt_in(k, Cfg::SMEM_BYTES));
  MM_TRY(launch_pdl(k, grid, Cfg::THREADS, Cfg::SMEM_BYTES, h->stream, *mx, *ms, p));
  MM_CUDA(cudaGetLastError());
  h->launches++;
  return MUMODE_OK;
}

template <int P>
static int launch_skinny_slab_p(mumode_handle_s* h, const ModeJob& j) {
  using Cfg = SkinnyCfg<P>;
  const CUtensorMap *mx = nullptr, *ms = nullptr;
  SkinnyParams p{j.L, j.sLi, j.sLk, int(j.K), int(j.N), 0, 0, int(j.A), 0, 0};
  // c-slabs per tile: as many as fit one stage (32 P doubles)
  p.TC = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(256, (32 * P) / (P * j.A))));
  uint64_t dx[3] = {uint64_t(j.A), uint64_t(j.K), uint64_t(j.C)}, sx[2] = {uint64_t(j.A), uint64_t(j.A * j.K)};
  uint64_t ds[3] = {uint64_t(j.A), uint64_t(j.N), uint64_t(j.C)}, ss[2] = {uint64_t(j.A), uint64_t(j.A * j.N)};
  uint32_t b[3] = {uint32_t(j.A), P, uint32_t(p.TC)};
  MM_TRY(get_map(h, j.T, 3, dx, sx, b, &mx, 2));
  MM_TRY(get_map(h, j.S, 3, ds, ss, b, &ms, 2));
  p.tiles = (j.C + p.TC - 1) / p.TC;
  const int grid = static_cast<int>(std::min<int64_t>(p.tiles, persistent_sms(h)));
  auto k = j.accumulate ? skinny_slab_kernel<P, true> : skinny_slab_kernel<P>;
  MM_TRY(smem_opt_in(k, Cfg::SMEM_BYTES));
  MM_TRY(launch_pdl(k, grid, Cfg::THREADS, Cfg::SMEM_BYTES, h->stream, *mx, *ms, p));
  MM_CUDA(cudaGetLastError());
  h->launches++;
  return MUMODE_OK;
}

template <int TA>
static int launch_skinny_ta(mumode_handle_s* h, const ModeJob& j) {
  const int64_t e = std::max(j.K, j.N);
  if (e <= 8) return launch_skinny_p<8, TA>(h, j);
  if (e <= 16) return launch_skinny_p<16, TA>(h, j);
  if (e <= 24) return launch_skinny_p<24, TA>(h, j);
  return launch_skinny_p<32, TA>(h, j);
}

static int launch_skinny(mumode_handle_s* h, const ModeJob& j) {
  if (j.A != 1 && j.A % 16 != 0 && j.A <= 32) {
    const int64_t e = std::max(j.K, j.N);
    if (e <= 8) return launch_skinny_slab_p<8>(h, j);
    if (e <= 16) return launch_skinny_slab_p<16>(h, j);
    if (e <= 24) return launch_skinny_slab_p<24>(h, j);
    return launch_skinny_slab_p<32>(h, j);
  }
  return (j.A != 1 && j.A % 32 != 0) ? launch_skinny_ta<16>(h, j) : launch_skinny_ta<32>(h, j);
}

static int run_job(mumode_handle_s* h, const ModeJob& j0) {
  ModeJob j = j0;
  // A real mu > 1 product whose factor has an odd leading dimension (odd n_mu)
  // is TMA-describable once the factor's N used rows are re-laid with an even
  // ld >= N (a tiny copy; the tensor strides are what they are). Only those
  // rows are read: j.L may be a row block of a larger factor.
  if (!j.cplx && !j.conj && j.A != 1 && j.sLi == 1 && (j.sLk & 1) && h->policy != 1 && h->policy != 8) {
    ModeJob jp = j;
    jp.sLk = (j.N + 1) & ~int64_t(1);
    jp.L = reinterpret_cast<const double*>(uintptr_t(256));  // the staged copy is 256-B aligned
    if (tma_ok(jp) && tma_worthwhile(jp)) {
      MM_TRY(h->lstage.ensure(size_t(jp.sLk * j.K) * sizeof(double)));
      auto* Lp = static_cast<double*>(h->lstage.p);
      pad2d_kernel<<<pad_grid(jp.sLk, j.K, h->num_sms), 256, 0, h->stream>>>(j.L, j.N, j.K, j.sLk, Lp, jp.sLk,
                                                                              j.K);
      MM_CUDA(cudaGetLastError());
      h->launches++;
      jp.L = Lp;
      j = jp;
    }
  }
  if (j.div_front) {
    // the direct solver's division in the last mode's epilogue, else a pass
    if (!j.cplx && !j.accumulate && j.A > 1 && j.C == 1 && tma_ok(j) && h->policy != 1 && h->policy != 8 &&
        (h->policy >= 2 || tma_worthwhile(j)))
      return launch_tma_auto(h, j);
    ModeJob jt = j;
    jt.div_front = jt.div_last = nullptr;
    MM_TRY(run_job(h, jt));
    const int64_t A = j.A, N = j.N;
    const int gx = static_cast<int>(std::min<int64_t>((A + 255) / 256, 64));
    const int gy = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(N, int64_t(h->num_sms) * 16 / gx)));
    eigsum_divide_kernel<<<dim3(gx, gy), 256, 0, h->stream>>>(j.S, j.div_front, j.div_last, A, N);
    MM_CUDA(cudaGetLastError());
    h->launches++;
    return MUMODE_OK;
  }
  if (j.scat) {
    // fused exchange: the TMA kernel's epilogue scatters to the ranks; any
    // other path computes the (rows x C) result and scatter-copies it
    if (!j.accumulate && tma_ok(j) && h->policy != 1 && h->policy != 8 && (h->policy >= 2 || tma_worthwhile(j)))
      return launch_tma_auto(h, j);
    ModeJob jt = j;
    jt.scat = nullptr;
    const int el = j.cplx ? 2 : 1;
    const int64_t rows = (j.A == 1) ? j.N : j.A * j.N, cols = j.C;
    MM_TRY(h->scat_tmp.ensure(size_t(rows * cols * el) * sizeof(double)));
    jt.S = static_cast<double*>(h->scat_tmp.p);
    MM_TRY(run_job(h, jt));
    const unsigned gy = static_cast<unsigned>(std::min<int64_t>(8, (rows * el + 255) / 256));
    scatter_copy_kernel<<<dim3(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(cols * 64, int64_t(h->num_sms) * 8))), gy),
                          256, 0, h->stream>>>(static_cast<const double*>(h->scat_tmp.p), rows, cols, el, j.scat);
    MM_CUDA(cudaGetLastError());
    h->launches++;
    return MUMODE_OK;
  }
  if (skinny_ok(h, j)) return launch_skinny(h, j);
  // accumulating products: real mu > 1 have a TMA instantiation; others generic
  const bool can_tma = tma_ok(j) && !(j.accumulate && j.A == 1);
  if (h->policy == 8 && !j.cplx) return launch_ldg(h, j);
  if (h->policy == 1) return launch_generic(h, j);
  if (!can_tma) return (!j.cplx && ldg_worthwhile(j)) ? launch_ldg(h, j) : launch_generic(h, j);
  if ((h->policy >= 2 && h->policy <= 6) || tma_worthwhile(j)) return launch_tma_auto(h, j);
  return launch_generic(h, j);
}

}  // namespace mumode_gpu
