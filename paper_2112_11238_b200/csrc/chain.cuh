// Tucker chains on device buffers: the fused two-mode passes (fused.cuh,
// tail.cuh) and tucker_dev, which runs modes mu_lo..mu_hi of a chain
// (odd-extent padding, fused pairs, per-mode jobs, scatter / divide
// epilogues of the last mode). Included by mumode_gpu.cu after dispatch.cuh.
#pragma once

namespace mumode_gpu {

// ------------------------------------------------------------------ fused pairs
template <int MU, bool FIRST, int RA>
static int launch_fused(mumode_handle_s* h, const double* T, double* S, const double* L1,
                        const double* L2, int64_t A, int64_t C) {
  using Cfg = FusedCfg<MU, FIRST, RA>;
  const CUtensorMap* mp = nullptr;
  FusedParams p{S, L1, L2, A, C, 0};
  if (FIRST) {
    uint64_t d[3] = {8, uint64_t(MU) * uint64_t(C), uint64_t(MU / 8)}, st[2] = {uint64_t(MU), 8};
    uint32_t b[3] = {8, 8 * MU, MU / 8};
    MM_TRY(get_map(h, T, 3, d, st, b, &mp));
    p.tiles = (C + 7) / 8;
  } else {
    uint64_t d[4] = {uint64_t(A), uint64_t(MU), uint64_t(MU), uint64_t(C)};
    uint64_t st[3] = {uint64_t(A), uint64_t(A) * MU, uint64_t(A) * MU * MU};
    uint32_t b[4] = {8, MU, MU, 1};
    MM_TRY(get_map(h, T, 4, d, st, b, &mp));
    p.tiles = (A / RA) * C;
  }
  const int grid = static_cast<int>(std::min<int64_t>(p.tiles, persistent_sms(h)));
  auto k = fused_pair_kernel<MU, FIRST, RA>;
  MM_TRY(smem_opt_in(k, Cfg::SMEM_BYTES));
  MM_TRY(launch_pdl(k, grid, Cfg::THREADS, Cfg::SMEM_BYTES, h->stream, *mp, p));
  MM_CUDA(cudaGetLastError());
  h->launches++;
  return MUMODE_OK;
}

// Warp-specialised first pass (fused_ws.cuh): modes 1 and 2.
template <int MU, int NY = 2>
static int launch_fused_ws(mumode_handle_s* h, const double* T, double* S, const double* L1,
                           const double* L2, int64_t C) {
  using Cfg = FusedWsCfg<MU, NY>;
  const CUtensorMap* mp = nullptr;
  FusedParams p{S, L1, L2, 1, C, (C + 7) / 8};
  uint64_t d[3] = {8, uint64_t(MU) * uint64_t(C), uint64_t(MU / 8)}, st[2] = {uint64_t(MU), 8};
  uint32_t b[3] = {8, 8 * MU, MU / 8};
  MM_TRY(get_map(h, T, 3, d, st, b, &mp));
  const int grid = static_cast<int>(std::min<int64_t>(p.tiles, persistent_sms(h)));
  auto k = fused_ws_kernel<MU, 2, NY>;
  MM_TRY(smem_opt_in(k, Cfg::SMEM_BYTES));
  MM_TRY(launch_pdl(k, grid, Cfg::THREADS, Cfg::SMEM_BYTES, h->stream, *mp, p));
  MM_CUDA(cudaGetLastError());
  h->launches++;
  return MUMODE_OK;
}

// Strided-pair pass with 32-wide a tiles (tail.cuh): 256-B rows for loads and
// stores instead of 64-B ones.
template <int MU>
static int launch_tail(mumode_handle_s* h, const double* T, double* S, const double* L1,
                       const double* L2, int64_t A, int64_t C) {
  using Cfg = TailCfg<MU>;
  const CUtensorMap *mx = nullptr, *ms = nullptr;
  uint64_t d[5] = {16, uint64_t(A / 16), uint64_t(MU), uint64_t(MU), uint64_t(C)};
  uint64_t st[4] = {16, uint64_t(A), uint64_t(A) * MU, uint64_t(A) * MU * MU};
  uint32_t bx[5] = {16, 2, MU, Cfg::KB, 1}, bs[5] = {16, 2, 1, MU, 1};
  MM_TRY(get_map(h, T, 5, d, st, bx, &mx, true));
  MM_TRY(get_map(h, S, 5, d, st, bs, &ms, true));
  TailParams p{L1, L2, A / 32, (A / 32) * C};
  const int grid = static_cast<int>(std::min<int64_t>(p.tiles, persistent_sms(h)));
  auto k = tail_pair_kernel<MU>;
  MM_TRY(smem_opt_in(k, Cfg::SMEM_BYTES));
  MM_TRY(launch_pdl(k, grid, Cfg::THREADS, Cfg::SMEM_BYTES, h->stream, *mx, *ms, p));
  MM_CUDA(cudaGetLastError());
  h->launches++;
  return MUMODE_OK;
}

template <int MU>
static int launch_tail_ws(mumode_handle_s* h, const double* T, double* S, const double* L1,
                          const double* L2, int64_t A, int64_t C) {
  using Cfg = TailWsCfg<MU>;
  const CUtensorMap *mx = nullptr, *ms = nullptr;
  uint64_t d[5] = {16, uint64_t(A / 16), uint64_t(MU), uint64_t(MU), uint64_t(C)};
  uint64_t st[4] = {16, uint64_t(A), uint64_t(A) * MU, uint64_t(A) * MU * MU};
  uint32_t bx[5] = {16, 2, MU, Cfg::KB, 1}, bs[5] = {16, 2, 1, MU, 1};
  MM_TRY(get_map(h, T, 5, d, st, bx, &mx, true));
  MM_TRY(get_map(h, S, 5, d, st, bs, &ms, true));
  TailParams p{L1, L2, A / 32, (A / 32) * C};
  const int grid = static_cast<int>(std::min<int64_t>(p.tiles, persistent_sms(h)));
  auto k = tail_ws_kernel<MU>;
  MM_TRY(smem_opt_in(k, Cfg::SMEM_BYTES));
  MM_TRY(launch_pdl(k, grid, Cfg::THREADS, Cfg::SMEM_BYTES, h->stream, *mx, *ms, p));
  MM_CUDA(cudaGetLastError());
  h->launches++;
  return MUMODE_OK;
}

// The tail kernels pay off once the a-stride makes every tile row a new page
// (and for MU = 8 at any A: 8^8 middle passes 60-80 -> 51 us). Policy 9
// forces the tail path wherever the shape allows, 10 disables it, 12 runs the
// kernels without warp specialisation (fused_pair_kernel for the first pass,
// tail_pair_kernel for the tail).
static constexpr int64_t kTailMinA = 16384;

template <int MU>
static int launch_fused_mu(mumode_handle_s* h, bool first, const double* T, double* S,
                           const double* L1, const double* L2, int64_t A, int64_t C) {
  const bool legacy = h->policy == 12;
  if constexpr (MU <= 24) {
    if (first && !legacy) return launch_fused_ws<MU>(h, T, S, L1, L2, C);
  }
  if (first) return launch_fused<MU, true, 8>(h, T, S, L1, L2, A, C);
  if constexpr (MU <= 24) {
    if (A % 32 == 0 && h->policy != 10 && (h->policy == 9 || A >= kTailMinA || (MU == 8 && !legacy)))
      return legacy ? launch_tail<MU>(h, T, S, L1, L2, A, C) : launch_tail_ws<MU>(h, T, S, L1, L2, A, C);
    // the streamed tail kernel also wins at smaller A once there are enough
    // 32-a tiles to fill the SMs (C5 pass 2, A = 576: 614 -> 604 us)
    if (A % 32 == 0 && h->policy != 10 && !legacy && (A / 32) * C >= 8 * persistent_sms(h))
      return launch_tail_ws<MU>(h, T, S, L1, L2, A, C);
  }
  // 16 a's per tile when shared memory allows it and A tiles evenly
  constexpr bool wide_fits = FusedCfg<MU, false, 16>::SMEM_BYTES <= 227 * 1024 &&
                             FusedCfg<MU, false, 16>::NBUF >= 2;
  if (wide_fits && A % 16 == 0 && A <= 4096) return launch_fused<MU, false, (wide_fits ? 16 : 8)>(h, T, S, L1, L2, A, C);
  return launch_fused<MU, false, 8>(h, T, S, L1, L2, A, C);
}

// Fused two-mode passes apply to real, forward chains whose modes are all
// square with one small extent MU in {8, 16, 24, 32} (e.g. config C5, 24^6):
// there each single product is HBM-bound and pairing halves the HBM passes.
static int fused_extent(int d, const int64_t* m, const int64_t* n, bool cplx, bool adjoint,
                        int policy, int mu_lo, int mu_hi, const double* T, const double* S,
                        const double* const* L) {
  if (cplx || adjoint || !(policy == 0 || policy == 7 || policy == 9 || policy == 10 || policy == 12 || policy == 13 || policy == 17) || mu_hi - mu_lo < 1)
    return 0;
  const int64_t MU = m[0];
  if (MU != 8 && MU != 16 && MU != 24 && MU != 32) return 0;
  for (int k = 0; k < d; ++k)
    if (m[k] != MU || n[k] != MU) return 0;
  if (!aligned16_ptr(T) || !aligned16_ptr(S)) return 0;
  for (int k = mu_lo - 1; k < mu_hi; ++k)
    if (!aligned16_ptr(L[k])) return 0;
  int64_t total = 1;
  for (int k = 0; k < d; ++k) total *= MU;
  if (total / MU >= (int64_t(1) << 31)) return 0;
  // a first pass of a few 8-c tiles of 32 MU^3 flop each leaves the GPU
  // idle: unfused small-tile products win there for MU >= 24 (32^3 11.7 ->
  // 6.2 us, 24^3 6.6 -> 6.3 us; 16^3 is faster fused, 4.4 vs 6.2 us), while
  // 4-D and larger keep the fused passes (24^4 11.1 us fused vs 17.1 unfused)
  if (MU >= 24 && (total / (MU * MU) + 7) / 8 < 16) return 0;
  return static_cast<int>(MU);
}

// ------------------------------------------------------------------ small-extent pairs
// Fused two-mode passes for extents <= 24 that the MU kernels do not cover
// (spair.cuh): auto paths (policy 0/7/9/10/12) use them where they measured
// faster than two skinny passes (largest extent 17..20: 20^6 1.10 -> 0.98 ms,
// 18^6 0.68 -> 0.64 ms; tools/small_pairs_sweep.py); 15 forces them wherever
// eligible (tests), 14 disables them.
static bool spair_policy(int policy) {
  return policy == 0 || policy == 7 || policy == 9 || policy == 10 || policy == 12 || policy == 15 || policy == 16 ||
         policy == 17;
}

template <int P4, int NF>
static int launch_spair_p(mumode_handle_s* h, const SpairParams& p0, bool mode1) {
  SpairParams p = p0;
  if (mode1) {
    using Cfg = Spair1Cfg<P4, NF>;
    const int64_t stages = (p.C + Cfg::CB - 1) / Cfg::CB;
    auto k = spair1_kernel<P4, NF>;
    MM_TRY(smem_opt_in(k, Cfg::SMEM_BYTES));
    const int grid = static_cast<int>(std::min<int64_t>(stages, persistent_sms(h)));
    MM_TRY(launch_pdl(k, grid, Cfg::THREADS, Cfg::SMEM_BYTES, h->stream, p));
  } else {
    using Cfg = SpairCfg<P4, NF>;
    p.ablks = (p.A + 31) / 32;
    p.tiles = p.ablks * p.C;
    auto k = spair_kernel<P4, NF>;
    MM_TRY(smem_opt_in(k, Cfg::SMEM_BYTES));
    const int grid = static_cast<int>(std::min<int64_t>(p.tiles, persistent_sms(h)));
    MM_TRY(launch_pdl(k, grid, Cfg::THREADS, Cfg::SMEM_BYTES, h->stream, p));
  }
  MM_CUDA(cudaGetLastError());
  h->launches++;
  return MUMODE_OK;
}

// Can modes (mu, mu+1) of the current extents run as one small-extent pass?
static int spair_size(const int64_t* ext, const int64_t* n, int d, int mu, bool forced) {
  const int64_t K1 = ext[mu - 1], N1 = n[mu - 1], K2 = ext[mu], N2 = n[mu];
  const int64_t e = std::max(std::max(K1, K2), std::max(N1, N2));
  if (e > 24 || std::min(std::min(K1, K2), std::min(N1, N2)) < 2) return 0;
  if (!forced && (e < 17 || e > 20)) return 0;
  const int64_t A = prod(ext, 0, mu - 1);
  if (mu == 1 ? (K1 & 1) : (A & 1)) return 0;  // 16-byte cp.async chunks
  return static_cast<int>((e + 3) / 4 * 4);
}

static int launch_spair(mumode_handle_s* h, const int64_t* ext, const int64_t* n, int d, int mu, const double* T,
                        const double* L1, const double* L2, double* S) {
  SpairParams p{};
  p.X = T;
  p.S = S;
  p.L1 = L1;
  p.L2 = L2;
  p.A = prod(ext, 0, mu - 1);
  p.C = prod(ext, mu + 1, d);
  p.K1 = static_cast<int>(ext[mu - 1]);
  p.N1 = static_cast<int>(n[mu - 1]);
  p.K2 = static_cast<int>(ext[mu]);
  p.N2 = static_cast<int>(n[mu]);
  const bool mode1 = (mu == 1);
  switch (spair_size(ext, n, d, mu, true)) {
    case 4:
    case 8: return launch_spair_p<8, 1>(h, p, mode1);
    case 12: return launch_spair_p<12, 2>(h, p, mode1);
    case 16: return launch_spair_p<16, 2>(h, p, mode1);
    case 20: return launch_spair_p<20, 3>(h, p, mode1);
    case 24: return launch_spair_p<24, 3>(h, p, mode1);
    default: return fail(MUMODE_ERR_ARGUMENT, "small-extent pair: unsupported extents");
  }
}

// Chains of small extents: any real forward chain whose modes are all <= 24
// and large enough to fill the GPU (>= 2^20 elements throughout).
static bool spair_chain_ok(mumode_handle_s* h, int d, const int64_t* m, const int64_t* n, bool cplx, bool adjoint,
                           int mu_lo, int mu_hi, const double* T, const double* S, const double* const* L) {
  if (cplx || adjoint || !spair_policy(h->policy) || mu_hi - mu_lo < 1) return false;
  if (!aligned16_ptr(T) || !aligned16_ptr(S)) return false;
  for (int k = mu_lo - 1; k < mu_hi; ++k)
    if (m[k] > 24 || n[k] > 24 || !L[k]) return false;
  return std::min(prod(m, 0, d), prod(n, 0, d)) >= (int64_t(1) << 20);
}

// ------------------------------------------------------------------ block passes
// In-place block passes (block.cuh): modes (mu .. mu+KM-1), all square with
// extents <= 24, of a view (A, e_1..e_KM, C). R = 1 for mu = 1 (cubes of
// CB consecutive c's), else R = 32 a's per block. The plan (layout search,
// row tables, copy segments) is built once per shape and cached on the handle.
static int block_plan(mumode_handle_s* h, int64_t A, const int* e, int KM, int64_t C, BlockPlan** out) {
  *out = nullptr;
  if (A > 1 && (A & 1)) return MUMODE_OK;
  int emax = 0;
  int64_t E = 1;
  for (int j = 0; j < KM; ++j) {
    if (e[j] < 2 || e[j] > 24) return MUMODE_OK;
    emax = std::max(emax, e[j]);
    E *= e[j];
  }
  if (A == 1 && (e[0] & 1)) return MUMODE_OK;
  const std::vector<int64_t> key{A, C, KM, e[0], KM > 1 ? e[1] : 0, KM > 2 ? e[2] : 0};
  auto it = h->blocks.find(key);
  if (it != h->blocks.end()) {
    *out = it->second.get();  // null: not eligible (cached)
    return MUMODE_OK;
  }
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  MM_CUDA(cudaStreamIsCapturing(h->stream, &cap));
  if (cap != cudaStreamCaptureStatusNone) return MUMODE_OK;  // plans are built outside graph capture
  const int P4 = (emax + 3) / 4 * 4, NF = (emax + 7) / 8;
  auto plan = std::make_unique<BlockPlan>();
  plan->P4 = P4 <= 8 ? 8 : (P4 <= 12 ? 12 : (P4 <= 16 ? 16 : (P4 <= 20 ? 20 : 24)));
  plan->NF = NF;
  const int ls_bytes = KM * (8 * NF) * plan->P4 * 8;
  // R > 1: the widest row (32 a's = 256 B, the DRAM-friendly width) whose
  // padded slot still gives a conflict-free layout; R = 1: CB whole cubes
  BlockLayout lay;
  bool ok = false;
  int CB = 1;
  if (A == 1) CB = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(C, 49152 / (E * 8))));
  int rcand[3] = {32, 16, 8};  // chunks per row must divide the 128 copy threads
  if (const char* r = getenv("MUMODE_BLOCK_R")) rcand[0] = rcand[1] = rcand[2] = std::max(2, atoi(r) / 2 * 2);
  for (int ri = 0; ri < (A == 1 ? 1 : 3) && !ok; ++ri) {
    const int R = (A == 1) ? 1 : rcand[ri];
    int64_t rows = 0;  // table bound: rows of every mode, padded to m-tiles
    for (int j = 0; j < KM; ++j) rows += (R * CB * E / e[j] + 15) / 8 * 8;
    const int fixed = ls_bytes + static_cast<int>(rows) * 2 + 3 * BLK_MAX_NB * 8 + 256;
    const int budget = 227 * 1024 - fixed;
    for (int nbmin = 3; nbmin >= 2 && !ok; --nbmin) {
      ok = blk_plan_layout(A, e, KM, R, CB, budget / nbmin / 8, lay);
      if (ok && R > 1 && ri < 2) {  // accept a narrower row only to avoid bank conflicts
        int64_t ideal = 0;
        for (int j = 0; j < KM; ++j) ideal += int64_t(lay.mt[j]) * 2 * ((e[j] + 3) / 4 + 2 * ((e[j] + 7) / 8));
        if (lay.cost > ideal * 3 / 2) ok = false;
      }
    }
  }
  const int budget = 227 * 1024 - (ls_bytes + static_cast<int>(lay.tab.size()) * 2 + 3 * BLK_MAX_NB * 8 + 256);
  const int R = lay.R;
  if (ok) {
    const int slot_bytes = lay.slot_dbl * 8;
    plan->NB = std::min(BLK_MAX_NB, budget / slot_bytes);
    // groups per CTA (tools/block_sweep.py, tools/block_cfg_runs.sh): 18^3 cubes 226 -> 212 us
    // with 4 groups of 4 warps (NB 4), 20^3 352 us with 2 groups (NB 3; 4: 367)
    plan->G = plan->NB >= 4 ? 4 : (plan->NB >= 2 ? 2 : 1);
    if (const char* g = getenv("MUMODE_BLOCK_G")) plan->G = std::max(1, std::min(4, atoi(g)));
    if (const char* nb = getenv("MUMODE_BLOCK_NB")) plan->NB = std::max(2, std::min(plan->NB, atoi(nb)));
    if (plan->G == 3) plan->G = 2;  // 16 warps split in 1, 2 or 4 groups
    plan->ls_off = plan->NB * slot_bytes;
    plan->tab_soff = plan->ls_off + ls_bytes;
    plan->bar_off = (plan->tab_soff + static_cast<int>(lay.tab.size()) * 2 + 15) / 16 * 16;
    plan->smem = plan->bar_off + 3 * BLK_MAX_NB * 8;  // full, done, tags
    plan->nblocks = (R > 1) ? ((A + R - 1) / R) * C : (C + CB - 1) / CB;
    MM_TRY(plan->tab.ensure(lay.tab.size() * sizeof(uint16_t)));
    MM_TRY(plan->seg.ensure(lay.seg.size() * sizeof(BlkSeg)));
    MM_CUDA(cudaMemcpy(plan->tab.p, lay.tab.data(), lay.tab.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
    MM_CUDA(cudaMemcpy(plan->seg.p, lay.seg.data(), lay.seg.size() * sizeof(BlkSeg), cudaMemcpyHostToDevice));
    if (getenv("MUMODE_BLOCK_DEBUG")) {
      int64_t ideal = 0;
      for (int j = 0; j < KM; ++j) ideal += int64_t(lay.mt[j]) * 2 * ((e[j] + 3) / 4 + 2 * ((e[j] + 7) / 8));
      fprintf(stderr, "mumode block plan: A=%lld e=(%d,%d,%d) C=%lld R=%d CB=%d slot=%d dbl NB=%d G=%d s=(%d,%d,%d) "
              "mt=(%d,%d,%d) segs=%zu cost=%lld ideal=%lld smem=%d\n",
              (long long)A, e[0], KM > 1 ? e[1] : 0, KM > 2 ? e[2] : 0, (long long)C, R, CB, lay.slot_dbl, plan->NB,
              plan->G, lay.s[0], lay.s[1], lay.s[2], lay.mt[0], lay.mt[1], lay.mt[2], lay.seg.size(),
              (long long)lay.cost, (long long)ideal, plan->smem);
    }
    plan->lay = std::move(lay);
    *out = plan.get();
    h->blocks[key] = std::move(plan);
  } else {
    h->blocks[key] = nullptr;
  }
  return MUMODE_OK;
}

template <int P4, int NF>
static int launch_block_p(mumode_handle_s* h, const BlockParams& p, int smem) {
  auto k = block_kernel<P4, NF>;
  MM_TRY(smem_opt_in(k, smem));
  const int grid = static_cast<int>(std::min<int64_t>(p.nblocks, persistent_sms(h)));
  MM_TRY(launch_pdl(k, grid, BLK_THREADS, smem, h->stream, p));
  MM_CUDA(cudaGetLastError());
  h->launches++;
  return MUMODE_OK;
}

static int launch_block(mumode_handle_s* h, BlockPlan* bp, const double* T, double* S, const double* const* Lm,
                        int64_t A, int64_t C) {
  const BlockLayout& lay = bp->lay;
  BlockParams p{};
  p.X = T;
  p.S = S;
  p.tab = static_cast<const uint16_t*>(bp->tab.p);
  p.seg = static_cast<const BlkSeg*>(bp->seg.p);
  p.A = A;
  p.C = C;
  p.E = 1;
  for (int j = 0; j < lay.KM; ++j) {
    p.L[j] = Lm[j];
    p.e[j] = lay.e[j];
    p.s[j] = lay.s[j];
    p.mt[j] = lay.mt[j];
    p.tab_off[j] = lay.tab_off[j];
    p.E *= lay.e[j];
  }
  p.nblocks = bp->nblocks;
  p.R = lay.R;
  p.CB = lay.CB;
  p.KM = lay.KM;
  p.NB = bp->NB;
  p.G = bp->G;
  p.ntab = static_cast<int>(lay.tab.size());
  p.nseg = static_cast<int>(lay.seg.size());
  p.slot_dbl = lay.slot_dbl;
  p.ls_off = bp->ls_off;
  p.tab_soff = bp->tab_soff;
  p.bar_off = bp->bar_off;
  switch (bp->P4 * 4 + bp->NF) {
    case 8 * 4 + 1: return launch_block_p<8, 1>(h, p, bp->smem);
    case 12 * 4 + 2: return launch_block_p<12, 2>(h, p, bp->smem);
    case 16 * 4 + 2: return launch_block_p<16, 2>(h, p, bp->smem);
    case 20 * 4 + 3: return launch_block_p<20, 3>(h, p, bp->smem);
    case 24 * 4 + 3: return launch_block_p<24, 3>(h, p, bp->smem);
    default: return fail(MUMODE_ERR_ARGUMENT, "block pass: unsupported extent class");
  }
}

// Block passes for a chain: every mode square, <= 24, real, forward. Auto
// (policy 0) uses them where measured faster; 16 forces, 17 disables.
static bool block_policy(int policy) { return policy == 0 || policy == 16; }

static bool block_chain_ok(mumode_handle_s* h, int d, const int64_t* m, const int64_t* n, bool cplx, bool adjoint,
                           int mu_lo, int mu_hi, const double* T, const double* S, const double* const* L) {
  if (cplx || adjoint || !block_policy(h->policy) || mu_hi - mu_lo < 1) return false;
  if (!aligned16_ptr(T) || !aligned16_ptr(S)) return false;
  for (int k = mu_lo - 1; k < mu_hi; ++k)
    if (m[k] != n[k] || m[k] > 24 || !L[k]) return false;
  if (h->policy == 16) return true;
  // auto: cube passes (modes 1-3 in place) beat two skinny / pair passes for
  // the paper's d = 6 sizes (18^6 0.650 -> 0.546 ms, 20^6 1.000 -> 0.863,
  // 14^6 128 -> 112 us, 12^6 64 -> 57 us); extents that are multiples of 8
  // take the MU kernels before this point
  return d - mu_lo + 1 >= 4 && mu_lo == 1 && std::min(prod(m, 0, d), prod(n, 0, d)) >= (int64_t(1) << 20);
}

// One mode product on device buffers: T with extents m (d modes), op(L)
// n_mu x m_mu given by (L, sLi, sLk, conj).
static int mode_product_dev(mumode_handle_s* h, int d, const int64_t* m, int mu, int64_t n_mu,
                            const double* T, const double* L, int64_t sLi, int64_t sLk,
                            bool cplx, bool conj, double* S, bool accumulate = false,
                            const ScatterParams* scat = nullptr, const double* div_front = nullptr,
                            const double* div_last = nullptr) {
  ModeJob j;
  j.accumulate = accumulate;
  j.scat = scat;
  j.div_front = div_front;
  j.div_last = div_last;
  j.T = T;
  j.L = L;
  j.S = S;
  j.A = prod(m, 0, mu - 1);
  j.K = m[mu - 1];
  j.C = prod(m, mu, d);
  j.N = n_mu;
  j.sLi = sLi;
  j.sLk = sLk;
  j.cplx = cplx;
  j.conj = conj;
  return run_job(h, j);
}

// ------------------------------------------------------------------ chain kernel
// middle modes run N-tile slowest (their consumers' inputs complete
// progressively: measured better than n-fastest, 2.1 % on C2, 4.3 % at 200^3)
#define CHAIN_N_MAJOR 1
// Tile decode shared by the host tables and the kernel (tma_chain.cuh):
// mode 1 m-fastest; middle modes N-tile slowest (their consumers' inputs then
// complete progressively); the last mode n-fastest.
static void chain_decode(const TmaParams& p, int k, int nmodes, int64_t tile, int& mt, int& nt) {
  if (k == 0 || (CHAIN_N_MAJOR && k + 1 < nmodes)) {
    mt = static_cast<int>(tile % p.mt);
    nt = static_cast<int>(tile / p.mt);
  } else {
    nt = static_cast<int>(tile % p.nt);
    mt = static_cast<int>(tile / p.nt);
  }
}

// For every producer tile of mode k, the consumer (mode k+1) M-tiles whose
// input rows it writes; targets = how many producer tiles each consumer
// M-tile waits for.
static bool chain_boundary(const ModeJob& jp, const TmaParams& pp, int bm_p, int bn_p, const ModeJob& jc,
                           const TmaParams& pc, int bm_c, int k, int nmodes, std::vector<int>& target,
                           std::vector<int>& sig_off, std::vector<int>& sig_idx) {
  const int64_t A_c = jp.A * jp.N, K_c = jc.K, AB_c = (A_c + 7) / 8, FB_c = bm_c / 8;
  target.assign(static_cast<size_t>(pc.mt), 0);
  sig_off.assign(1, 0);
  sig_idx.clear();
  std::vector<int> cur;
  for (int64_t t = 0; t < pp.tiles; ++t) {
    int mt, nt;
    chain_decode(pp, k, nmodes, t, mt, nt);
    cur.clear();
    if (k == 0) {  // QK: rows i (= consumer a), columns = (k_c + K_c * c)
      const int64_t i0 = int64_t(mt) * bm_p, i1 = std::min<int64_t>(i0 + bm_p, pp.Mlim);
      const int64_t c0 = int64_t(nt) * bn_p, c1 = std::min<int64_t>(c0 + bn_p, pp.N);
      for (int64_t c = c0 / K_c; c <= (c1 - 1) / K_c; ++c) {
        const int64_t qlo = i0 / 8 + AB_c * c, qhi = (i1 - 1) / 8 + AB_c * c;
        for (int64_t m = qlo / FB_c; m <= qhi / FB_c; ++m) cur.push_back(static_cast<int>(m));
      }
    } else {  // fragments (alpha, c') x outputs i: consumer a = a' + A_p i, c = c' / K_c
      const int64_t A_p = jp.A, AB_p = (A_p + 7) / 8;
      const int64_t q0 = int64_t(mt) * (bm_p / 8), q1 = std::min<int64_t>(q0 + bm_p / 8, pp.mfrags);
      const int64_t i0 = int64_t(nt) * bn_p, i1 = std::min<int64_t>(i0 + bn_p, pp.N);
      int last = -1;
      for (int64_t q = q0; q < q1; ++q) {
        const int64_t alpha = q % AB_p, cp_ = q / AB_p, c = cp_ / K_c;
        const int64_t alo = 8 * alpha, ahi = std::min<int64_t>(8 * alpha + 8, A_p) - 1;
        for (int64_t i = i0; i < i1; ++i) {
          const int64_t blo = (alo + A_p * i) / 8, bhi = (ahi + A_p * i) / 8;
          for (int64_t b = blo; b <= bhi; ++b) {
            const int m = static_cast<int>((b + AB_c * c) / FB_c);
            if (m != last) cur.push_back(m), last = m;
          }
        }
      }
    }
    std::sort(cur.begin(), cur.end());
    cur.erase(std::unique(cur.begin(), cur.end()), cur.end());
    for (int m : cur) {
      if (m < 0 || m >= pc.mt) return false;  // never expected; the caller runs the modes one by one
      sig_idx.push_back(m);
      ++target[static_cast<size_t>(m)];
    }
    sig_off.push_back(static_cast<int>(sig_idx.size()));
  }
  return true;
}

template <class CfgA, class CfgB>
static int launch_chain(mumode_handle_s* h, const std::vector<ModeJob>& jobs, int cfg_a, int cfg_b) {
  const int d = static_cast<int>(jobs.size());
  ChainMaps maps;
  ChainParams cp{};
  cp.nphases = d;
  std::vector<TmaParams> ps(static_cast<size_t>(d));
  for (int k = 0; k < d; ++k) {
    const CUtensorMap *mp = nullptr, *mq = nullptr;
    if (k == 0)
      MM_TRY(tma_setup<CfgA>(h, jobs[0], &mp, &mq, ps[0]));
    else
      MM_TRY(tma_setup<CfgB>(h, jobs[static_cast<size_t>(k)], &mp, &mq, ps[static_cast<size_t>(k)]));
    maps.P[k] = *mp;
    maps.Q[k] = *mq;
  }
  // dependency tables: built once per shape and config pair
  std::vector<int64_t> key{d, jobs[0].cplx ? 1 : 0, cfg_a, cfg_b};
  for (const auto& j : jobs) key.insert(key.end(), {j.A, j.K, j.N, j.C});
  auto it = h->chains.find(key);
  if (it == h->chains.end()) {
    auto plan = std::make_unique<ChainPlan>();
    std::vector<int> all;
    size_t ctr = 0;
    plan->target_off.assign(d, -1);
    plan->sigoff_off.assign(d, -1);
    plan->sigidx_off.assign(d, -1);
    plan->ctr_off.assign(d, -1);
    for (int k = 0; k + 1 < d; ++k) {
      std::vector<int> target, sig_off, sig_idx;
      if (!chain_boundary(jobs[k], ps[k], k == 0 ? CfgA::BM : CfgB::BM, k == 0 ? CfgA::BN : CfgB::BN,
                          jobs[k + 1], ps[k + 1], CfgB::BM, k, d, target, sig_off, sig_idx))
        return -1;  // a producer tile maps outside the consumer's M-tiles: run per mode
      plan->target_off[k + 1] = static_cast<int64_t>(all.size());
      all.insert(all.end(), target.begin(), target.end());
      plan->sigoff_off[k] = static_cast<int64_t>(all.size());
      all.insert(all.end(), sig_off.begin(), sig_off.end());
      plan->sigidx_off[k] = static_cast<int64_t>(all.size());
      all.insert(all.end(), sig_idx.begin(), sig_idx.end());
      plan->ctr_off[k + 1] = static_cast<int64_t>(ctr);
      ctr += target.size();
    }
    MM_TRY(plan->tables.ensure(std::max<size_t>(all.size(), 1) * sizeof(int)));
    MM_CUDA(cudaMemcpy(plan->tables.p, all.data(), all.size() * sizeof(int), cudaMemcpyHostToDevice));
    MM_TRY(plan->counters.ensure(std::max<size_t>(ctr, 1) * sizeof(int)));
    plan->counter_ints = ctr;
    it = h->chains.emplace(key, std::move(plan)).first;
  }
  const ChainPlan& pl = *it->second;
  auto* tab = static_cast<const int*>(pl.tables.p);
  auto* ctr = static_cast<int*>(pl.counters.p);
  int64_t base = 0;
  for (int k = 0; k < d; ++k) {
    ChainPhase& P = cp.ph[k];
    P.p = ps[static_cast<size_t>(k)];
    P.base = base;
    P.n_major = (CHAIN_N_MAJOR && k > 0 && k + 1 < d) ? 1 : 0;
    base += P.p.tiles;
    if (k > 0) {
      P.wait_ctr = ctr + pl.ctr_off[k];
      P.wait_target = tab + pl.target_off[k];
    }
    if (k + 1 < d) {
      P.sig_off = tab + pl.sigoff_off[k];
      P.sig_idx = tab + pl.sigidx_off[k];
      P.sig_ctr = ctr + pl.ctr_off[k + 1];
    }
  }
  cp.total = base;
  if (pl.counter_ints) MM_CUDA(cudaMemsetAsync(pl.counters.p, 0, pl.counter_ints * sizeof(int), h->stream));
  const int grid = static_cast<int>(std::min<int64_t>(cp.total, persistent_sms(h)));
  auto kern = tucker_chain_kernel<CfgA, CfgB>;
  MM_TRY(smem_opt_in(kern, CfgB::SMEM_BYTES + kChainExtraSmem));
  kern<<<grid, CfgB::THREADS, CfgB::SMEM_BYTES + kChainExtraSmem, h->stream>>>(maps, cp);  // no PDL (tma_chain.cuh)
  MM_CUDA(cudaGetLastError());
  h->launches++;
  return MUMODE_OK;
}

// The whole chain as one persistent launch when every mode is a plain TMA
// product (no fused pairs / epilogue variants) and the per-mode tile configs
// form an instantiated pair. Sets `done` when it ran.
static int try_chain(mumode_handle_s* h, const std::vector<ModeJob>& jobs, bool& done) {
  done = false;
  const int d = static_cast<int>(jobs.size());
  if (d < 2 || d > kChainMaxModes) return MUMODE_OK;
  for (const auto& j : jobs)
    if (j.accumulate || j.scat || j.div_front || !tma_ok(j) || !tma_worthwhile(j)) return MUMODE_OK;
  const int a = choose_cfg(jobs[0], h->num_sms);
  int b = -1;
  for (int k = 1; k < d; ++k) {
    const int c = choose_cfg(jobs[static_cast<size_t>(k)], h->num_sms);
    if (b >= 0 && c != b) return MUMODE_OK;
    b = c;
  }
  // instantiated pairs (same CTA shape and ring): 0 Big, 1 TM, 2 LM (real)
  int rc = -1;
  if (a == 0 && b == 0) rc = launch_chain<CfgBig, CfgBig>(h, jobs, a, b);
  else if (a == 2 && b == 1) rc = launch_chain<CfgLM, CfgTM>(h, jobs, a, b);
  else if (a == 1 && b == 1) rc = launch_chain<CfgTM, CfgTM>(h, jobs, a, b);
  if (rc < 0) return MUMODE_OK;
  MM_TRY(rc);
  done = true;
  return MUMODE_OK;
}

// ------------------------------------------------------------------ tucker chain
// Modes 1..d in order (tucker.hpp:84-110). Lmat[mu] points at the stored
// matrix; forward: op(L) = L (n x m, ld n); adjoint: op(L) = L^H (L is m x n).
// Real adjoint and complex adjoint use the generic kernel's strided/conj
// access, or a materialised op(L) when the TMA path applies.
static int tucker_dev(mumode_handle_s* h, int d, const int64_t* m, const int64_t* n,
                      const double* T, const double* const* L, double* S, bool adjoint,
                      bool cplx, int mu_lo = 1, int mu_hi = 0, const ScatterParams* scat = nullptr,
                      const double* div_front = nullptr, const double* div_last = nullptr) {
  if (mu_hi == 0) mu_hi = d;
  const int el = cplx ? 2 : 1;
  const int nmodes = mu_hi - mu_lo + 1;
  if (scat) {
    // the range's last mode scatters its (rows x cols) result to the ranks
    // (fused exchange, csrc/slab_dist.cuh); the modes before it run as usual
    if (adjoint) return fail(MUMODE_ERR_ARGUMENT, "scatter: forward chains only");
    std::vector<int64_t> ext(m, m + d);
    const double* src = T;
    if (nmodes > 1) {
      for (int k = mu_lo - 1; k < mu_hi - 1; ++k) ext[k] = n[k];
      MM_TRY(h->scat_mid.ensure(size_t(prod(ext.data(), 0, d) * el) * sizeof(double)));
      auto* mid = static_cast<double*>(h->scat_mid.p);
      MM_TRY(tucker_dev(h, d, m, n, T, L, mid, false, cplx, mu_lo, mu_hi - 1));
      src = mid;
    }
    return mode_product_dev(h, d, ext.data(), mu_hi, n[mu_hi - 1], src, L[mu_hi - 1], 1, n[mu_hi - 1], cplx,
                            false, nullptr, false, scat);
  }
  // An odd real leading extent gives 8-byte strides, which TMA cannot
  // describe (every stride is a multiple of the mode-1 extent). A whole
  // chain then runs on a copy whose mode 1 is padded by one zero row (and
  // mode-1 factor by a zero column / row): zero k-terms leave the FMA chains
  // unchanged, the pad row of the output is dropped. Two copy passes buy the
  // TMA/DMMA kernels for every mode.
  if (!cplx && !adjoint && !div_front && mu_lo == 1 && mu_hi == d && d >= 2 && h->policy == 0 && ((m[0] | n[0]) & 1) &&
      aligned16_ptr(T) && aligned16_ptr(S)) {
    // measured (tools/odd_sweep.py): the padded chain wins from ~223^3 up
    // (255^3: 26.5 -> 28.7 TF/s); below ~208 the LDG-staged kernel's smaller
    // tiles quantise better
    bool big = true;
    for (int k = 0; k < d; ++k) big = big && m[k] >= 208 && n[k] >= 208;
    const int64_t numel_in = prod(m, 0, d), numel_out = prod(n, 0, d);
    if (big && std::max(numel_in, numel_out) >= (int64_t(1) << 20)) {
      std::vector<int64_t> mp(m, m + d), np(n, n + d);
      mp[0] += m[0] & 1;
      np[0] += n[0] & 1;
      const int64_t rest_in = numel_in / m[0], rest_out = numel_out / n[0];
      const bool ok = (mp[0] == m[0] || h->pad_in.ensure(size_t(mp[0] * rest_in) * sizeof(double)) == MUMODE_OK) &&
                      h->lpad.ensure(size_t(np[0] * mp[0]) * sizeof(double)) == MUMODE_OK &&
                      (np[0] == n[0] || h->pad_out.ensure(size_t(np[0] * rest_out) * sizeof(double)) == MUMODE_OK);
      if (ok) {
        const double* Tp = T;
        auto* Lp = static_cast<double*>(h->lpad.p);
        double* Sp = np[0] == n[0] ? S : static_cast<double*>(h->pad_out.p);
        if (mp[0] != m[0]) {
          auto* Tpad = static_cast<double*>(h->pad_in.p);
          pad2d_kernel<<<pad_grid(mp[0], rest_in, h->num_sms), 256, 0, h->stream>>>(T, m[0], rest_in, m[0], Tpad, mp[0],
                                                                                    rest_in);
          h->launches++;
          Tp = Tpad;
        }
        pad2d_kernel<<<pad_grid(np[0], mp[0], h->num_sms), 256, 0, h->stream>>>(L[0], n[0], m[0], n[0], Lp, np[0], mp[0]);
        MM_CUDA(cudaGetLastError());
        h->launches++;
        std::vector<const double*> Lpad(L, L + d);
        Lpad[0] = Lp;
        MM_TRY(tucker_dev(h, d, mp.data(), np.data(), Tp, Lpad.data(), Sp, false, false));
        if (Sp != S) {
          pad2d_kernel<<<pad_grid(n[0], rest_out, h->num_sms), 256, 0, h->stream>>>(Sp, np[0], rest_out, np[0], S, n[0],
                                                                                 rest_out);
          MM_CUDA(cudaGetLastError());
          h->launches++;
        }
        return MUMODE_OK;
      }
      g_err.clear();  // not enough memory for the padded copies: run unpadded
    }
  }
  // workspace: largest intermediate
  std::vector<int64_t> ext(m, m + d);
  size_t maxel = 0;
  for (int mu = mu_lo - 1; mu < mu_hi - 1; ++mu) {
    ext[mu] = n[mu];
    maxel = std::max(maxel, size_t(prod(ext.data(), 0, d)));
  }
  if (nmodes > 1) {
    MM_TRY(h->ws[0].ensure(maxel * el * sizeof(double)));
    if (nmodes > 2) MM_TRY(h->ws[1].ensure(maxel * el * sizeof(double)));
  }
  // materialise op(L) = L^T / L^H when adjoint (tiny: n x m per mode)
  std::vector<const double*> Lop(d);
  if (adjoint) {
    size_t tot = 0;
    for (int mu = mu_lo - 1; mu < mu_hi; ++mu) tot += size_t(m[mu] * n[mu]) * el + 2;
    MM_TRY(h->lbuf.ensure(tot * sizeof(double) + 256));
    double* dst = static_cast<double*>(h->lbuf.p);
    for (int mu = mu_lo - 1; mu < mu_hi; ++mu) {
      const int64_t rows = m[mu], cols = n[mu];  // stored L is m x n
      transpose_conj_kernel<<<grid_for(rows * cols, h->num_sms), 256, 0, h->stream>>>(
          L[mu], dst, rows, cols, cplx ? 1 : 0, 1);
      MM_CUDA(cudaGetLastError());
      h->launches++;
      Lop[mu] = dst;
      dst += ((rows * cols * el + 1) / 2) * 2;  // keep 16-B alignment
    }
  } else {
    for (int mu = 0; mu < d; ++mu) Lop[mu] = L[mu];
  }
  ext.assign(m, m + d);
  const double* src = T;
  const int MU = fused_extent(d, m, n, cplx, adjoint, h->policy, mu_lo, mu_hi, T, S, L);
  if (MU) {
    // pairs (mu, mu+1) as fused passes; an odd last mode runs alone below
    int pass = 0, mu = mu_lo;
    for (; mu + 1 <= mu_hi; mu += 2, ++pass) {
      double* dst = (mu + 1 == mu_hi) ? S : static_cast<double*>(h->ws[pass % 2].p);
      const int64_t A = prod(ext.data(), 0, mu - 1), C = prod(ext.data(), mu + 1, d);
      int rc;
      switch (MU) {
        case 8: rc = launch_fused_mu<8>(h, mu == 1, src, dst, L[mu - 1], L[mu], A, C); break;
        case 16: rc = launch_fused_mu<16>(h, mu == 1, src, dst, L[mu - 1], L[mu], A, C); break;
        case 24: rc = launch_fused_mu<24>(h, mu == 1, src, dst, L[mu - 1], L[mu], A, C); break;
        default: rc = launch_fused_mu<32>(h, mu == 1, src, dst, L[mu - 1], L[mu], A, C); break;
      }
      MM_TRY(rc);
      src = dst;
    }
    if (mu == mu_hi) {
      MM_TRY(mode_product_dev(h, d, ext.data(), mu, n[mu - 1], src, L[mu - 1], 1, n[mu - 1], false, false, S,
                              false, nullptr, div_front, div_last));
    } else if (div_front) {  // the last pass was a fused pair: divide in a pass of its own
      const int64_t A = prod(n, 0, d - 1), N = n[d - 1];
      const int gx = static_cast<int>(std::min<int64_t>((A + 255) / 256, 64));
      const int gy = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(N, int64_t(h->num_sms) * 16 / gx)));
      eigsum_divide_kernel<<<dim3(gx, gy), 256, 0, h->stream>>>(S, div_front, div_last, A, N);
      MM_CUDA(cudaGetLastError());
      h->launches++;
    }
    return MUMODE_OK;
  }
  if (!div_front && block_chain_ok(h, d, m, n, cplx, adjoint, mu_lo, mu_hi, T, S, L)) {
    // groups of up to three modes as in-place block passes where a plan
    // exists (largest group first), single products (skinny kernels) otherwise
    int pass = 0, mu = mu_lo;
    while (mu <= mu_hi) {
      const int64_t A = prod(ext.data(), 0, mu - 1);
      BlockPlan* bp = nullptr;
      int km = std::min(3, mu_hi - mu + 1);
      // mu = 1: cubes of modes 1-3; mu > 1: blocks of 32 a's (256-B rows) x
      // the modes (an 18^2 pair is 86 KB: two slots, fed by the copy warps'
      // fused store/load walk). Auto takes cubes with >= 3 slots (22^3 fits
      // two: 22^5 0.099 -> 0.104 ms) and 32-a pairs where the spair kernel
      // would run (largest extent 17..20: 18^6 modes 4-5 185 vs 213 us, 20^6
      // 319 vs 332 us; at 12^6 / 14^6 two skinny passes are faster)
      const bool force = h->policy == 16;
      const bool spair_here = mu < mu_hi && spair_size(ext.data(), n, d, mu, false) != 0;
      for (; km >= 2; --km) {
        if (!force && (A == 1 ? km != 3 : (km != 2 || !spair_here))) continue;
        int e3[3] = {0, 0, 0};
        for (int j = 0; j < km; ++j) e3[j] = static_cast<int>(ext[mu - 1 + j]);
        MM_TRY(block_plan(h, A, e3, km, prod(ext.data(), mu - 1 + km, d), &bp));
        if (bp && !force && A == 1 && bp->NB < 3) bp = nullptr;
        if (bp) break;
      }
      const bool pair = !bp && mu < mu_hi && spair_size(ext.data(), n, d, mu, false) != 0;
      const int step = bp ? km : (pair ? 2 : 1);
      double* dst = (mu + step - 1 == mu_hi) ? S : static_cast<double*>(h->ws[pass % 2].p);
      if (bp) {
        MM_TRY(launch_block(h, bp, src, dst, L + (mu - 1), A, prod(ext.data(), mu - 1 + km, d)));
      } else if (pair) {
        MM_TRY(launch_spair(h, ext.data(), n, d, mu, src, L[mu - 1], L[mu], dst));
      } else {
        MM_TRY(mode_product_dev(h, d, ext.data(), mu, n[mu - 1], src, L[mu - 1], 1, n[mu - 1], false, false, dst));
      }
      src = dst;
      mu += step;
      ++pass;
    }
    return MUMODE_OK;
  }
  if (!div_front && spair_chain_ok(h, d, m, n, cplx, adjoint, mu_lo, mu_hi, T, S, L)) {
    // pairs (mu, mu+1) as small-extent fused passes where eligible, single
    // products (skinny kernels) otherwise
    int pass = 0, mu = mu_lo;
    while (mu <= mu_hi) {
      const bool last_single = (mu == mu_hi);
      const bool pair = !last_single && spair_size(ext.data(), n, d, mu, h->policy == 15) != 0;
      const int step = pair ? 2 : 1;
      double* dst = (mu + step - 1 == mu_hi) ? S : static_cast<double*>(h->ws[pass % 2].p);
      if (pair) {
        MM_TRY(launch_spair(h, ext.data(), n, d, mu, src, L[mu - 1], L[mu], dst));
        ext[mu - 1] = n[mu - 1];
        ext[mu] = n[mu];
      } else {
        MM_TRY(mode_product_dev(h, d, ext.data(), mu, n[mu - 1], src, L[mu - 1], 1, n[mu - 1], false, false, dst));
        ext[mu - 1] = n[mu - 1];
      }
      src = dst;
      mu += step;
      ++pass;
    }
    return MUMODE_OK;
  }
  if (h->policy == 11 && !div_front && nmodes >= 2) {
    // one persistent launch for the whole chain (tma_chain.cuh)
    std::vector<ModeJob> jobs;
    std::vector<int64_t> e2(ext);
    const double* src2 = src;
    for (int mu = mu_lo; mu <= mu_hi; ++mu) {
      ModeJob j;
      j.T = src2;
      j.L = Lop[mu - 1];
      j.S = (mu == mu_hi) ? S : static_cast<double*>(h->ws[(mu - mu_lo) % 2].p);
      j.A = prod(e2.data(), 0, mu - 1);
      j.K = e2[mu - 1];
      j.C = prod(e2.data(), mu, d);
      j.N = n[mu - 1];
      j.sLi = 1;
      j.sLk = n[mu - 1];
      j.cplx = cplx;
      j.conj = false;
      jobs.push_back(j);
      e2[mu - 1] = n[mu - 1];
      src2 = j.S;
    }
    // the chain kernel's first mode must be a QK (mode 1) product
    if (mu_lo == 1) {
      bool done = false;
      MM_TRY(try_chain(h, jobs, done));
      if (done) return MUMODE_OK;
    }
  }
  for (int mu = mu_lo; mu <= mu_hi; ++mu) {
    double* dst = (mu == mu_hi) ? S : static_cast<double*>(h->ws[(mu - mu_lo) % 2].p);
    const bool last = (mu == mu_hi);
    MM_TRY(mode_product_dev(h, d, ext.data(), mu, n[mu - 1], src, Lop[mu - 1], 1, n[mu - 1],
                            cplx, false, dst, false, nullptr, last ? div_front : nullptr,
                            last ? div_last : nullptr));
    ext[mu - 1] = n[mu - 1];
    src = dst;
  }
  return MUMODE_OK;
}

// [a, a + na) and [b, b + nb) (doubles) overlap?
static bool overlaps(const double* a, int64_t na, const double* b, int64_t nb) {
  return a < b + nb && b < a + na;
}

static int check_no_alias(const double* T, int64_t nt, const double* S, int64_t ns, const char* who) {
  if (overlaps(T, nt, S, ns))
    return fail(MUMODE_ERR_ARGUMENT, std::string(who) + ": output overlaps the input (results are new tensors)");
  return MUMODE_OK;
}

static int check_stack(int d, const int64_t* m, const int64_t* n, const double* T,
                       const double* const* L, const void* S, const char* who) {
  MM_TRY(check_shape(d, m, who));
  if (!T || !L || !S || !n) return fail(MUMODE_ERR_ARGUMENT, std::string(who) + ": null pointer");
  for (int k = 0; k < d; ++k) {
    if (n[k] < 1) return fail(MUMODE_ERR_ARGUMENT, "matrix dimensions must be positive");
    if (!L[k])
      return fail(MUMODE_ERR_ARGUMENT,
                  std::string(who) + ": null matrix for mode " + std::to_string(k + 1));
  }
  return MUMODE_OK;
}

}  // namespace mumode_gpu
