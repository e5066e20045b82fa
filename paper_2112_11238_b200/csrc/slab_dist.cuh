// Slab-partitioned Tucker across GPUs behind the C-ABI:
// mumode_comm_* and mumode_dist_tucker_{f64,c128}. Included by mumode_gpu.cu
// (shares its static helpers); the algorithm is the one in
// paper_2112_11238_b200/dist.py:
//
//   rank r holds the last-mode slab T[..., c_r]. For each of `chunks`
//   sub-slabs (column runs of the slab):
//     compute stream: modes 1..d-1 (tucker_dev; TMA/DMMA or fused kernels)
//                     -> Y_j (A x w), packed by destination row block;
//     comm stream:    one NCCL group of sends (block q -> rank q) and
//                     receives (every rank's chunk j lands in its final,
//                     contiguous columns of Z = (A_r x m_d)), own block by a
//                     device copy;
//   so the exchange of chunk j overlaps the contraction of chunk j+1. Then
//   mode d on Z -> S_r (A_r x n_d), rows A_r of the flattened result.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): inside a process that
// already loaded NCCL (e.g. through torch) the same library is reused, and the
// engine has no link-time NCCL dependency. nccl.h supplies the types only.
#pragma once
#include <dlfcn.h>
#include <chrono>
#include <thread>
#include <nccl.h>

namespace mumode_gpu {

struct NcclApi {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclGetVersion) get_version = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  // optional (failure detection): present in every NCCL >= 2.4
  decltype(&ncclCommGetAsyncError) get_async_error = nullptr;
  decltype(&ncclCommAbort) comm_abort = nullptr;
};

static NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      const char* e = dlerror();
      a.why = std::string("NCCL library not found: ") + (e ? e : "dlopen failed");
      return a;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(lib, name));
      if (!fn) all = false;
    };
    sym(a.get_unique_id, "ncclGetUniqueId");
    sym(a.comm_init_rank, "ncclCommInitRank");
    sym(a.comm_destroy, "ncclCommDestroy");
    sym(a.group_start, "ncclGroupStart");
    sym(a.group_end, "ncclGroupEnd");
    sym(a.send, "ncclSend");
    sym(a.recv, "ncclRecv");
    sym(a.error_string, "ncclGetErrorString");
    sym(a.get_version, "ncclGetVersion");
    sym(a.all_gather, "ncclAllGather");
    a.ok = all;
    a.get_async_error = reinterpret_cast<decltype(&ncclCommGetAsyncError)>(dlsym(lib, "ncclCommGetAsyncError"));
    a.comm_abort = reinterpret_cast<decltype(&ncclCommAbort)>(dlsym(lib, "ncclCommAbort"));
    if (!all) a.why = "NCCL library lacks the point-to-point API";
    return a;
  }();
  return api;
}

#define MM_NCCL(call)                                                                        \
  do {                                                                                       \
    ncclResult_t r_ = (call);                                                                \
    if (r_ != ncclSuccess)                                                                   \
      return fail(MUMODE_ERR_NCCL, std::string("NCCL: ") + nccl_api().error_string(r_) +   \
                                       " (" #call ")");                                      \
  } while (0)

static void even_splits(int64_t total, int parts, int64_t* off) {
  const int64_t base = total / parts, extra = total % parts;
  off[0] = 0;
  for (int q = 0; q < parts; ++q) off[q + 1] = off[q] + base + (q < extra ? 1 : 0);
}

// The partition of one application (dist.py SlabPlan): last-mode slabs c_off,
// output row blocks a_off over A = prod_{k<d} n_k.
static int slab_plan(int P, int d, const int64_t* m, const int64_t* n, int64_t* c_off, int64_t* a_off) {
  if (P < 1 || P > kMaxRanks) return fail(MUMODE_ERR_ARGUMENT, "slab plan: 1..64 ranks");
  if (d < 2) return fail(MUMODE_ERR_SIZE, "slab partitioning needs an order >= 2 tensor");
  MM_TRY(check_shape(d, m, "slab plan"));
  for (int k = 0; k < d; ++k)
    if (n[k] < 1) return fail(MUMODE_ERR_ARGUMENT, "matrix dimensions must be positive");
  if (m[d - 1] < P)
    return fail(MUMODE_ERR_SIZE, "last mode extent " + std::to_string(m[d - 1]) + " < " + std::to_string(P) +
                                     " ranks");
  even_splits(m[d - 1], P, c_off);
  even_splits(prod(n, 0, d - 1), P, a_off);
  return MUMODE_OK;
}

// The complete per-rank schedule of one slab-partitioned application, built
// on the host (and exposed as mumode_dist_plan so the multi-rank logic is
// verified on CPU: tests/test_dist.py simulates every rank executing it).
struct DistChunk {
  int64_t col0;      // first slab column of the sub-slab
  int64_t w;         // its width (0: this rank has no sub-slab j)
  int64_t send_off;  // doubles: where the packed sub-slab sits in the send buffer
};
struct DistOp {
  int64_t chunk, kind, peer;  // kind 0 = send, 1 = receive, 2 = own block (device copy)
  int64_t buf_off;            // send buffer offset (send, copy source)
  int64_t z_off;              // Z offset (receive, copy destination)
  int64_t count;              // doubles
};
struct DistPlan {
  int64_t c_off[kMaxRanks + 1], a_off[kMaxRanks + 1];
  int64_t rows_in = 0, A = 0, A_r = 0, m_d = 0, n_d = 0, wmax = 0, send_elems = 0, z_elems = 0;
  std::vector<DistChunk> ch;
  std::vector<DistOp> ops;  // grouped by chunk; within a chunk: copy, sends (q order), receives (s order)
};

static int dist_plan(int P, int r, int d, const int64_t* m, const int64_t* n, int chunks, int el, DistPlan& pl) {
  if (r < 0 || r >= P) return fail(MUMODE_ERR_ARGUMENT, "dist plan: bad rank");
  if (chunks < 0) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: chunks must be >= 0 (0 = auto)");
  MM_TRY(slab_plan(P, d, m, n, pl.c_off, pl.a_off));
  pl.rows_in = prod(m, 0, d - 1);
  pl.A = prod(n, 0, d - 1);
  pl.A_r = pl.a_off[r + 1] - pl.a_off[r];
  pl.m_d = m[d - 1];
  pl.n_d = n[d - 1];
  // auto: split a slab only while every sub-slab keeps >= 4M elements, so the
  // per-chunk kernels still fill the GPU (at most 4 sub-slabs); the same on
  // every rank (smallest slab)
  if (chunks == 0) {
    const int64_t c_min = pl.c_off[1] - pl.c_off[0] - ((m[d - 1] % P) ? 1 : 0);
    chunks = static_cast<int>(
        std::max<int64_t>(1, std::min<int64_t>(4, pl.rows_in * std::max<int64_t>(c_min, 1) / (int64_t(1) << 22))));
  }
  // every rank's sub-slab split (all ranks derive all of them, so the posted
  // sends and receives match)
  int nch = 0;
  std::vector<std::vector<int64_t>> sub(P);
  for (int s = 0; s < P; ++s) {
    const int64_t cs = pl.c_off[s + 1] - pl.c_off[s];
    const int k = static_cast<int>(std::min<int64_t>(chunks, cs));
    sub[s].assign(k + 1, 0);
    even_splits(cs, k, sub[s].data());
    nch = std::max(nch, k);
  }
  auto width = [&](int s, int j) -> int64_t {
    return j + 1 < static_cast<int>(sub[s].size()) ? sub[s][j + 1] - sub[s][j] : 0;
  };
  const int64_t A = pl.A, A_r = pl.A_r;
  pl.ch.clear();
  pl.ops.clear();
  pl.wmax = 0;
  for (int j = 0; j < nch; ++j) {
    const int64_t w = width(r, j);
    const int64_t c0 = w > 0 ? sub[r][j] : 0;
    pl.ch.push_back({c0, w, A * c0 * el});
    pl.wmax = std::max(pl.wmax, w);
    const int64_t sbase = A * c0 * el;
    if (w > 0 && A_r > 0)  // own row block: straight into its final columns
      pl.ops.push_back({j, 2, r, sbase + pl.a_off[r] * w * el, A_r * (pl.c_off[r] + c0) * el, A_r * w * el});
    if (w > 0)
      for (int q = 0; q < P; ++q) {
        const int64_t rows = pl.a_off[q + 1] - pl.a_off[q];
        if (q == r || rows == 0) continue;
        pl.ops.push_back({j, 0, q, sbase + pl.a_off[q] * w * el, 0, rows * w * el});
      }
    for (int s = 0; s < P; ++s) {
      const int64_t ws = width(s, j);
      if (s == r || ws == 0 || A_r == 0) continue;
      pl.ops.push_back({j, 1, s, 0, A_r * (pl.c_off[s] + sub[s][j]) * el, A_r * ws * el});
    }
  }
  pl.send_elems = A * (pl.c_off[r + 1] - pl.c_off[r]) * el;
  pl.z_elems = A_r * pl.m_d * el;
  return MUMODE_OK;
}

// Return exchange after an application: rank r's output rows (A_r x n_d,
// column-major, the rows buffer R) become the last-mode slabs of the output
// tensor for the next application (A x c'_r). Rank r sends R's columns of
// slab q (contiguous: A_r x c'_q) to q and receives (A_s x c'_r) from every s
// into a staging buffer laid out like the pack ([s][A_s x c'_r]), which
// slab_pack_kernel<true> (the unpack) turns into the slab. ops: buf_off into R, z_off into the
// staging buffer.
static int return_plan(int P, int r, int d, const int64_t* n, std::vector<DistOp>& ops, int64_t* c_off,
                       int64_t* a_off, int el) {
  if (r < 0 || r >= P) return fail(MUMODE_ERR_ARGUMENT, "dist plan: bad rank");
  MM_TRY(slab_plan(P, d, n, n, c_off, a_off));
  ops.clear();
  const int64_t A_r = a_off[r + 1] - a_off[r], c_r = c_off[r + 1] - c_off[r];
  if (A_r > 0) ops.push_back({0, 2, r, A_r * c_off[r] * el, a_off[r] * c_r * el, A_r * c_r * el});
  for (int q = 0; q < P; ++q) {
    const int64_t c_q = c_off[q + 1] - c_off[q];
    if (q == r || A_r == 0 || c_q == 0) continue;
    ops.push_back({0, 0, q, A_r * c_off[q] * el, 0, A_r * c_q * el});
  }
  for (int s = 0; s < P; ++s) {
    const int64_t A_s = a_off[s + 1] - a_off[s];
    if (s == r || A_s == 0) continue;
    ops.push_back({0, 1, s, 0, a_off[s] * c_r * el, A_s * c_r * el});
  }
  return MUMODE_OK;
}

}  // namespace mumode_gpu

struct mumode_comm_s {
  ncclComm_t comm = nullptr;
  bool owned = false;
  bool local = false;  // no NCCL: peer-store exchange with caller-exchanged IPC handles
  int nranks = 1, rank = 0, device = 0;
  cudaStream_t stream = nullptr;          // exchange stream
  std::vector<cudaEvent_t> events;        // per-chunk "packed" + start/done
  mumode_gpu::DevBuf y, send, z;          // chunk intermediate, packed slab, received (A_r x m_d)
  mumode_gpu::DevBuf rows, stage, spare;  // expint: output rows, return staging, slab ping-pong
  cudaEvent_t ret_in = nullptr, ret_out = nullptr;  // expint: return exchange
  // exchange 1 (peer stores): double-buffered Z and epoch flags, mapped into
  // every peer with CUDA IPC; the scatter table for the epilogue
  int exchange = 0;
  int overlap_sms = 16;                    // SMs left to NCCL while sub-slabs overlap the exchange
  int64_t epoch = 0;
  mumode_gpu::DevBuf pz[2], flags, handles, scat;
  mumode_gpu::DevBuf scat_tabs;            // NCCL path: per-chunk scatter tables (pack-free send buffer)
  size_t mapped_bytes = 0;                 // Z size the peer mappings were made for
  std::vector<double*> peer_z[2];          // [parity][rank] (own rank: local pointer)
  std::vector<int64_t*> peer_flags;        // [rank] flag array of that rank
};

namespace mumode_gpu {

static int comm_finish(mumode_comm_s* c, mumode_comm_t* out) {
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    if (c->owned && c->comm) nccl_api().comm_destroy(c->comm);
    delete c;
    return fail(MUMODE_ERR_CUDA, "comm stream creation failed");
  }
  *out = c;
  return MUMODE_OK;
}

static int comm_events(mumode_comm_s* c, size_t want) {
  while (c->events.size() < want) {
    cudaEvent_t e;
    MM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->events.push_back(e);
  }
  return MUMODE_OK;
}

// ---- exchange 1: peer stores over NVLink (CUDA IPC mappings)
// Signal: every earlier write of this stream (the scatter kernel's peer
// stores) is ordered before the flags by a system-scope fence, then each peer
// q gets flags_q[r] = epoch (release, system scope).
__global__ void p2p_signal_kernel(int64_t* const* __restrict__ peer_flags, int P, int r, int64_t epoch) {
  asm volatile("fence.sc.sys;\n" ::: "memory");
  for (int q = threadIdx.x; q < P; q += blockDim.x)
    asm volatile("st.release.sys.global.b64 [%0], %1;\n" ::"l"(peer_flags[q] + r), "l"(epoch) : "memory");
}
// Wait until every rank's flag in the local array reached epoch (acquire,
// system scope). Watchdog: a peer that has not signalled within 10 s of
// global time traps the kernel, so a lost peer surfaces as a launch failure
// instead of a hung GPU.
__global__ void p2p_wait_kernel(const int64_t* __restrict__ flags, int P, int64_t epoch) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t0));
  for (int s = threadIdx.x; s < P; s += blockDim.x) {
    int64_t v;
    for (uint32_t polls = 1;; ++polls) {
      asm volatile("ld.acquire.sys.global.b64 %0, [%1];\n" : "=l"(v) : "l"(flags + s) : "memory");
      if (v >= epoch) break;
      if ((polls & 1023u) == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
        if (t - t0 > 10000000000ull) __trap();
      }
    }
  }
  __syncthreads();
  asm volatile("fence.sc.sys;\n" ::: "memory");
}

// Peer mappings of the double-buffered Z and the epoch flags. export: make
// sure the local buffers hold `zbytes` and write their three CUDA-IPC handles
// (Z[0], Z[1], flags); import: open every other rank's handles (P x 3, rank
// order). p2p_map does both around an NCCL all-gather (a collective: every
// rank calls it with the same size in the same dist_tucker call); a comm
// without NCCL (mumode_comm_create_local) gets the handles from its caller.
constexpr size_t kIpcHandleBytes = sizeof(cudaIpcMemHandle_t);

static void p2p_unmap(mumode_comm_s* cm) {
  const int r = cm->rank;
  for (int b = 0; b < 2; ++b)
    for (int q = 0; q < static_cast<int>(cm->peer_z[b].size()); ++q)
      if (q != r && cm->peer_z[b][q]) cudaIpcCloseMemHandle(cm->peer_z[b][q]);
  for (int q = 0; q < static_cast<int>(cm->peer_flags.size()); ++q)
    if (q != r && cm->peer_flags[q]) cudaIpcCloseMemHandle(cm->peer_flags[q]);
  for (int b = 0; b < 2; ++b) cm->peer_z[b].clear();
  cm->peer_flags.clear();
  cm->mapped_bytes = 0;
}

static int p2p_export(mumode_comm_s* cm, size_t zbytes, void* out3) {
  p2p_unmap(cm);
  MM_TRY(cm->pz[0].ensure(zbytes));
  MM_TRY(cm->pz[1].ensure(zbytes));
  if (!cm->flags.p) {
    MM_TRY(cm->flags.ensure(sizeof(int64_t) * kMaxRanks));
    MM_CUDA(cudaMemset(cm->flags.p, 0, sizeof(int64_t) * kMaxRanks));
  }
  auto* h3 = static_cast<cudaIpcMemHandle_t*>(out3);
  MM_CUDA(cudaIpcGetMemHandle(&h3[0], cm->pz[0].p));
  MM_CUDA(cudaIpcGetMemHandle(&h3[1], cm->pz[1].p));
  MM_CUDA(cudaIpcGetMemHandle(&h3[2], cm->flags.p));
  return MUMODE_OK;
}

static int p2p_import(mumode_comm_s* cm, size_t zbytes, const void* all3P) {
  const int P = cm->nranks, r = cm->rank;
  const auto* all = static_cast<const cudaIpcMemHandle_t*>(all3P);
  for (int b = 0; b < 2; ++b) cm->peer_z[b].assign(P, nullptr);
  cm->peer_flags.assign(P, nullptr);
  for (int q = 0; q < P; ++q) {
    if (q == r) {
      cm->peer_z[0][q] = static_cast<double*>(cm->pz[0].p);
      cm->peer_z[1][q] = static_cast<double*>(cm->pz[1].p);
      cm->peer_flags[q] = static_cast<int64_t*>(cm->flags.p);
      continue;
    }
    void* ptr = nullptr;
    for (int b = 0; b < 2; ++b) {
      MM_CUDA(cudaIpcOpenMemHandle(&ptr, all[3 * q + b], cudaIpcMemLazyEnablePeerAccess));
      cm->peer_z[b][q] = static_cast<double*>(ptr);
    }
    MM_CUDA(cudaIpcOpenMemHandle(&ptr, all[3 * q + 2], cudaIpcMemLazyEnablePeerAccess));
    cm->peer_flags[q] = static_cast<int64_t*>(ptr);
  }
  cm->mapped_bytes = zbytes;
  return MUMODE_OK;
}

static int p2p_map(mumode_comm_s* cm, size_t zbytes) {
  const int P = cm->nranks;
  constexpr size_t HB = kIpcHandleBytes;
  std::vector<cudaIpcMemHandle_t> mine(3);
  MM_TRY(p2p_export(cm, zbytes, mine.data()));
  MM_TRY(cm->handles.ensure(3 * HB * (P + 1)));
  auto* dh = static_cast<uint8_t*>(cm->handles.p);
  MM_CUDA(cudaMemcpy(dh, mine.data(), 3 * HB, cudaMemcpyHostToDevice));
  auto& api = nccl_api();
  MM_NCCL(api.all_gather(dh, dh + 3 * HB, 3 * HB, ncclUint8, cm->comm, cm->stream));
  MM_CUDA(cudaStreamSynchronize(cm->stream));
  std::vector<cudaIpcMemHandle_t> all(3 * P);
  MM_CUDA(cudaMemcpy(all.data(), dh + 3 * HB, 3 * HB * P, cudaMemcpyDeviceToHost));
  return p2p_import(cm, zbytes, all.data());
}

// Bytes of one Z buffer of the peer-store exchange for this shape (the
// largest rank's received matrix, so every rank maps equal sizes).
static size_t p2p_zbytes(const DistPlan& pl, int P, int el) {
  size_t want = 0;
  for (int q = 0; q < P; ++q)
    want = std::max(want, size_t((pl.a_off[q + 1] - pl.a_off[q]) * pl.m_d * el) * sizeof(double));
  return std::max(want, size_t(8));
}

// One application with the exchange fused into the last local mode's
// epilogue: the TMA kernel stores every row pair straight into the owning
// rank's Z (peer pointers), then signal / wait, then mode d on the local Z.
//
// phase 0: the whole application. phase 1: local modes + peer stores +
// signal, then return; phase 2: wait for every rank's signal of the current
// epoch + mode d. A caller that runs phase 2 only after every rank finished
// phase 1 (host barrier) never has a kernel waiting on another process --
// the form in which the handshake can be exercised with several processes
// on ONE GPU (tests/test_dist_ipc.py).
static int dist_tucker_p2p(mumode_handle_s* h, mumode_comm_s* cm, int d, const int64_t* m, const int64_t* n,
                           const double* T, const double* const* L, double* S, const DistPlan& pl, bool cplx,
                           int phase) {
  const int P = cm->nranks, r = cm->rank;
  const int el = cplx ? 2 : 1;
  const size_t want = p2p_zbytes(pl, P, el);
  if (phase != 2) {
    // all ranks see the same shapes, so they remap in the same call
    if (P > 1 && want > cm->mapped_bytes) {
      if (!cm->comm)
        return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: peer buffers not mapped for this shape (" +
                                             std::to_string(want) +
                                             " bytes): exchange handles with mumode_comm_ipc_export/import");
      MM_TRY(p2p_map(cm, want));
    }
    if (P == 1) {
      MM_TRY(cm->pz[0].ensure(want));
      MM_TRY(cm->pz[1].ensure(want));
      for (int b = 0; b < 2; ++b) cm->peer_z[b].assign(1, static_cast<double*>(cm->pz[b].p));
    }
    const int par = static_cast<int>(++cm->epoch & 1);
    ScatterParams sp{};
    sp.P = P;
    sp.col0 = pl.c_off[r];
    for (int q = 0; q <= P; ++q) sp.a_off[q] = pl.a_off[q];
    for (int q = 0; q < P; ++q) sp.dst[q] = cm->peer_z[par][q];
    MM_TRY(cm->scat.ensure(sizeof(ScatterParams) + sizeof(int64_t*) * kMaxRanks));
    auto* dsp = static_cast<ScatterParams*>(cm->scat.p);
    auto** dflags = reinterpret_cast<int64_t**>(static_cast<uint8_t*>(cm->scat.p) + sizeof(ScatterParams));
    MM_CUDA(cudaMemcpyAsync(dsp, &sp, sizeof(sp), cudaMemcpyHostToDevice, h->stream));
    if (P > 1)
      MM_CUDA(cudaMemcpyAsync(dflags, cm->peer_flags.data(), sizeof(int64_t*) * P, cudaMemcpyHostToDevice,
                              h->stream));
    // the local slab: m_1 x ... x m_{d-1} x c_r (the global m_d is the sum)
    std::vector<int64_t> ext(m, m + d);
    ext[d - 1] = pl.c_off[r + 1] - pl.c_off[r];
    MM_TRY(tucker_dev(h, d, ext.data(), n, T, L, nullptr, false, cplx, 1, d - 1, dsp));
    if (P > 1) {
      p2p_signal_kernel<<<1, 64, 0, h->stream>>>(dflags, P, r, cm->epoch);
      MM_CUDA(cudaGetLastError());
      h->launches++;
    }
    if (phase == 1) return MUMODE_OK;
  } else if (cm->epoch == 0 || (P > 1 && cm->mapped_bytes < want)) {
    return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: phase 2 without a phase 1 for this shape");
  }
  const int par = static_cast<int>(cm->epoch & 1);
  if (P > 1 && phase == 2) {
    // split phases: the caller promised every rank finished phase 1; check
    // it on the host so the wait below never has to wait on another process
    std::vector<int64_t> fl(static_cast<size_t>(P));
    MM_CUDA(cudaStreamSynchronize(h->stream));
    MM_CUDA(cudaMemcpy(fl.data(), cm->flags.p, sizeof(int64_t) * P, cudaMemcpyDeviceToHost));
    for (int q = 0; q < P; ++q)
      if (fl[static_cast<size_t>(q)] < cm->epoch)
        return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: phase 2 before rank " + std::to_string(q) +
                                             " completed phase 1 of epoch " + std::to_string(cm->epoch));
  }
  if (P > 1) {
    p2p_wait_kernel<<<1, 64, 0, h->stream>>>(static_cast<const int64_t*>(cm->flags.p), P, cm->epoch);
    MM_CUDA(cudaGetLastError());
    h->launches++;
  }
  if (pl.A_r == 0) return MUMODE_OK;
  const int64_t zext[2] = {pl.A_r, pl.m_d};
  return mode_product_dev(h, 2, zext, 2, pl.n_d, cm->peer_z[par][r], L[d - 1], 1, pl.n_d, cplx, false, S);
}

// No pack pass: each sub-slab's last local mode stores its rows through the
// scatter epilogue (EPI 2) straight into the packed send layout -- row block
// q of chunk j is the contiguous (A_q x w) matrix at send_off + a_off[q] * w
// -- and its own row block straight into its final columns of Z. One
// scatter table per chunk, uploaded once per call (stream-ordered).
static int upload_scatter_tables(mumode_handle_s* h, DevBuf& buf, const DistPlan& pl, int P, int r, double* send,
                                 double* Z, int el) {
  const int nch = static_cast<int>(pl.ch.size());
  std::vector<ScatterParams> tabs(static_cast<size_t>(std::max(nch, 1)));
  for (int j = 0; j < nch; ++j) {
    const DistChunk& c = pl.ch[j];
    ScatterParams& sp = tabs[static_cast<size_t>(j)];
    sp = ScatterParams{};
    sp.P = P;
    sp.col0 = 0;
    for (int q = 0; q <= P; ++q) sp.a_off[q] = pl.a_off[q];
    for (int q = 0; q < P; ++q) {
      const bool empty = pl.a_off[q + 1] == pl.a_off[q] || c.w == 0;
      sp.dst[q] = empty ? nullptr
                        : (q == r ? Z + pl.A_r * (pl.c_off[r] + c.col0) * el
                                  : send + c.send_off + pl.a_off[q] * c.w * el);
    }
  }
  MM_TRY(buf.ensure(sizeof(ScatterParams) * tabs.size()));
  MM_CUDA(cudaMemcpyAsync(buf.p, tabs.data(), sizeof(ScatterParams) * tabs.size(), cudaMemcpyHostToDevice,
                          h->stream));
  return MUMODE_OK;
}

static int dist_tucker(mumode_handle_s* h, mumode_comm_s* cm, int d, const int64_t* m, const int64_t* n,
                       const double* T, const double* const* L, double* S, int chunks, bool cplx, int phase = 0) {
  const int P = cm->nranks, r = cm->rank;
  if (cm->device != h->device) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: handle and comm on different devices");
  if (!T || !L || !S) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: null pointer");
  for (int k = 0; k < d; ++k)
    if (!L[k]) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: null matrix for mode " + std::to_string(k + 1));
  const int el = cplx ? 2 : 1;
  DistPlan pl;
  MM_TRY(dist_plan(P, r, d, m, n, chunks, el, pl));
  if (phase != 0 && cm->exchange != 1)
    return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: phases apply to the peer-store exchange only");
  if (cm->exchange == 1) return dist_tucker_p2p(h, cm, d, m, n, T, L, S, pl, cplx, phase);
  if (P == 1 && chunks <= 1) {
    // one rank: no exchange, and its output rows (A x n_d) ARE the whole
    // result: the plain chain (fused passes included). Explicit chunks > 1
    // still take the general path (exercised by the tests).
    return tucker_dev(h, d, m, n, T, L, S, false, cplx);
  }
  const int64_t A_r = pl.A_r, m_d = pl.m_d, n_d = pl.n_d;
  const int nch = static_cast<int>(pl.ch.size());
  MM_TRY(cm->send.ensure(size_t(std::max<int64_t>(pl.send_elems, 1)) * sizeof(double)));
  MM_TRY(cm->z.ensure(size_t(std::max<int64_t>(pl.z_elems, 1)) * sizeof(double)));
  MM_TRY(comm_events(cm, size_t(nch) + 2));
  auto* send = static_cast<double*>(cm->send.p);
  auto* Z = static_cast<double*>(cm->z.p);
  MM_TRY(upload_scatter_tables(h, cm->scat_tabs, pl, P, r, send, Z, el));
  auto* dtabs = static_cast<ScatterParams*>(cm->scat_tabs.p);

  // Z (and send) may still be read by the previous call's work on h->stream
  MM_CUDA(cudaEventRecord(cm->events[nch], h->stream));
  MM_CUDA(cudaStreamWaitEvent(cm->stream, cm->events[nch], 0));
  std::vector<int64_t> ext(m, m + d);
  size_t op = 0;
  // overlapped exchange: leave SMs to NCCL's kernels while the sub-slabs run
  struct Reserve {
    mumode_handle_s* h;
    int prev;
    ~Reserve() { h->sm_reserve = prev; }
  } reserve{h, h->sm_reserve};
  if (P > 1 && nch > 1) h->sm_reserve = std::min(cm->overlap_sms, h->num_sms - 1);
  for (int j = 0; j < nch; ++j) {
    const DistChunk& c = pl.ch[j];
    if (c.w > 0) {
      ext[d - 1] = c.w;
      MM_TRY(tucker_dev(h, d, ext.data(), n, T + pl.rows_in * c.col0 * el, L, nullptr, false, cplx, 1, d - 1,
                        dtabs + j));
      MM_CUDA(cudaEventRecord(cm->events[j], h->stream));
      MM_CUDA(cudaStreamWaitEvent(cm->stream, cm->events[j], 0));
    }
    const size_t first = op;
    while (op < pl.ops.size() && pl.ops[op].chunk == j) ++op;
    // (the plan's own-block copy, kind 2, is done by the scatter epilogue)
    if (P > 1) {
      auto& api = nccl_api();
      MM_NCCL(api.group_start());
      for (size_t k = first; k < op; ++k) {
        const DistOp& o = pl.ops[k];
        if (o.kind == 0)
          MM_NCCL(api.send(send + o.buf_off, size_t(o.count), ncclFloat64, static_cast<int>(o.peer), cm->comm,
                           cm->stream));
        else if (o.kind == 1)
          MM_NCCL(api.recv(Z + o.z_off, size_t(o.count), ncclFloat64, static_cast<int>(o.peer), cm->comm,
                           cm->stream));
      }
      MM_NCCL(api.group_end());
    }
  }
  h->sm_reserve = reserve.prev;  // the last mode runs after the exchange: all SMs
  MM_CUDA(cudaEventRecord(cm->events[nch + 1], cm->stream));
  MM_CUDA(cudaStreamWaitEvent(h->stream, cm->events[nch + 1], 0));
  if (A_r == 0) return MUMODE_OK;
  const int64_t zext[2] = {A_r, m_d};
  return mode_product_dev(h, 2, zext, 2, n_d, Z, L[d - 1], 1, n_d, cplx, false, S);
}

// Wait for the handle's and the comm's queued work with failure detection:
// polls the streams and ncclCommGetAsyncError; an NCCL error, or no progress
// within timeout_ms, aborts the communicator (ncclCommAbort) and fails with
// MUMODE_ERR_NCCL instead of hanging on a lost peer.
static int comm_poll(mumode_handle_s* h, mumode_comm_s* cm, int64_t timeout_ms) {
  auto& api = nccl_api();
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t a = cudaStreamQuery(h->stream);
    const cudaError_t b = cm->stream ? cudaStreamQuery(cm->stream) : cudaSuccess;
    if (a != cudaSuccess && a != cudaErrorNotReady) {
      cudaGetLastError();
      return fail(MUMODE_ERR_CUDA, std::string("CUDA error while waiting: ") + cudaGetErrorString(a));
    }
    if (b != cudaSuccess && b != cudaErrorNotReady) {
      cudaGetLastError();
      return fail(MUMODE_ERR_CUDA, std::string("CUDA error while waiting: ") + cudaGetErrorString(b));
    }
    if (a == cudaSuccess && b == cudaSuccess) return MUMODE_OK;
    if (cm->comm && api.get_async_error) {
      ncclResult_t st = ncclSuccess;
      api.get_async_error(cm->comm, &st);
      if (st != ncclSuccess && st != ncclInProgress) {
        if (api.comm_abort && cm->owned) {
          api.comm_abort(cm->comm);
          cm->comm = nullptr;
        }
        return fail(MUMODE_ERR_NCCL, std::string("NCCL asynchronous error: ") + api.error_string(st));
      }
    }
    const auto ms =
        std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
    if (timeout_ms > 0 && ms > timeout_ms) {
      if (cm->comm && api.comm_abort && cm->owned) {
        api.comm_abort(cm->comm);
        cm->comm = nullptr;
      }
      return fail(MUMODE_ERR_NCCL, "timed out after " + std::to_string(ms) +
                                       " ms waiting for the exchange (a peer is lost or stalled); communicator "
                                       "aborted");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

// Copies and one NCCL group of a schedule on the exchange stream.
static int run_ops(mumode_comm_s* cm, const DistOp* ops, size_t nops, const double* src, double* dst) {
  for (size_t k = 0; k < nops; ++k)
    if (ops[k].kind == 2)
      MM_CUDA(cudaMemcpyAsync(dst + ops[k].z_off, src + ops[k].buf_off, size_t(ops[k].count) * sizeof(double),
                              cudaMemcpyDeviceToDevice, cm->stream));
  if (cm->nranks == 1) return MUMODE_OK;
  auto& api = nccl_api();
  MM_NCCL(api.group_start());
  for (size_t k = 0; k < nops; ++k) {
    const DistOp& o = ops[k];
    if (o.kind == 0)
      MM_NCCL(api.send(src + o.buf_off, size_t(o.count), ncclFloat64, static_cast<int>(o.peer), cm->comm, cm->stream));
    else if (o.kind == 1)
      MM_NCCL(api.recv(dst + o.z_off, size_t(o.count), ncclFloat64, static_cast<int>(o.peer), cm->comm, cm->stream));
  }
  MM_NCCL(api.group_end());
  return MUMODE_OK;
}

// steps x (slab-partitioned Tucker with E, return exchange, unpack): the
// exponential-integrator step (evolution.cpp:70-82) across ranks; modes in the
// reference order every step. u0 / u: this rank's last-mode slabs.
static int dist_expint(mumode_handle_s* h, mumode_comm_s* cm, int d, const int64_t* m, const double* const* E,
                       const double* u0, double* u, int steps) {
  const int P = cm->nranks, r = cm->rank;
  if (cm->device != h->device) return fail(MUMODE_ERR_ARGUMENT, "dist_expint: handle and comm on different devices");
  if (steps < 0) return fail(MUMODE_ERR_ARGUMENT, "expint: steps must be non-negative");
  if (!u0 || !u || !E) return fail(MUMODE_ERR_ARGUMENT, "dist_expint: null pointer");
  int64_t c_off[kMaxRanks + 1], a_off[kMaxRanks + 1];
  std::vector<DistOp> ops;
  MM_TRY(return_plan(P, r, d, m, ops, c_off, a_off, 1));
  const int64_t A = prod(m, 0, d - 1), c_r = c_off[r + 1] - c_off[r], A_r = a_off[r + 1] - a_off[r];
  const size_t slab_bytes = size_t(A * c_r) * sizeof(double);
  if (steps == 0) {
    if (u != u0) MM_CUDA(cudaMemcpyAsync(u, u0, slab_bytes, cudaMemcpyDeviceToDevice, h->stream));
    return MUMODE_OK;
  }
  MM_TRY(cm->spare.ensure(std::max<size_t>(slab_bytes, 8)));
  if (P > 1) {
    MM_TRY(cm->rows.ensure(std::max<size_t>(size_t(A_r * m[d - 1]) * sizeof(double), 8)));
    MM_TRY(cm->stage.ensure(std::max<size_t>(slab_bytes, 8)));
  }
  if (!cm->ret_in) MM_CUDA(cudaEventCreateWithFlags(&cm->ret_in, cudaEventDisableTiming));
  if (!cm->ret_out) MM_CUDA(cudaEventCreateWithFlags(&cm->ret_out, cudaEventDisableTiming));
  cudaEvent_t ev_in = cm->ret_in, ev_out = cm->ret_out;
  auto* spare = static_cast<double*>(cm->spare.p);
  PackOffsets off{};
  for (int q = 0; q <= P; ++q) off.a[q] = a_off[q];
  const double* cur = u0;
  for (int s = 0; s < steps; ++s) {
    double* dst = ((steps - 1 - s) % 2 == 0) ? u : spare;
    if (dst == cur) dst = (dst == u) ? spare : u;
    if (P == 1) {  // the output rows ARE the slab
      MM_TRY(dist_tucker(h, cm, d, m, m, cur, E, dst, 0, false));
    } else {
      auto* R = static_cast<double*>(cm->rows.p);
      auto* stage = static_cast<double*>(cm->stage.p);
      MM_TRY(dist_tucker(h, cm, d, m, m, cur, E, R, 0, false));
      MM_CUDA(cudaEventRecord(ev_in, h->stream));
      MM_CUDA(cudaStreamWaitEvent(cm->stream, ev_in, 0));
      MM_TRY(run_ops(cm, ops.data(), ops.size(), R, stage));
      MM_CUDA(cudaEventRecord(ev_out, cm->stream));
      MM_CUDA(cudaStreamWaitEvent(h->stream, ev_out, 0));
      slab_pack_kernel<true><<<pack_grid(A, c_r, P, h->num_sms), 256, 0, h->stream>>>(stage, dst, A, c_r, P, off);
      MM_CUDA(cudaGetLastError());
      h->launches++;
    }
    cur = dst;
  }
  if (cur != u) MM_CUDA(cudaMemcpyAsync(u, cur, slab_bytes, cudaMemcpyDeviceToDevice, h->stream));
  return MUMODE_OK;
}

}  // namespace mumode_gpu

extern "C" {

int mumode_comm_unique_id(void* id_out) {
  using namespace mumode_gpu;
  if (!id_out) return fail(MUMODE_ERR_ARGUMENT, "null id buffer");
  auto& api = nccl_api();
  if (!api.ok) return fail(MUMODE_ERR_NCCL, api.why);
  ncclUniqueId id;
  MM_NCCL(api.get_unique_id(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return MUMODE_OK;
}

int mumode_comm_create(mumode_comm_t* out, int device, const void* id, int nranks, int rank) {
  using namespace mumode_gpu;
  if (!out || !id) return fail(MUMODE_ERR_ARGUMENT, "comm_create: null pointer");
  *out = nullptr;
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks)
    return fail(MUMODE_ERR_ARGUMENT, "comm_create: bad rank / size");
  auto& api = nccl_api();
  if (!api.ok) return fail(MUMODE_ERR_NCCL, api.why);
  MM_DEVICE(device);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  auto* c = new mumode_comm_s();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  c->owned = true;
  ncclResult_t res = api.comm_init_rank(&c->comm, nranks, uid, rank);
  if (res != ncclSuccess) {
    delete c;
    return fail(MUMODE_ERR_NCCL, std::string("NCCL: ") + api.error_string(res) + " (ncclCommInitRank)");
  }
  return comm_finish(c, out);
}

int mumode_comm_wrap(mumode_comm_t* out, int device, void* nccl_comm, int nranks, int rank) {
  using namespace mumode_gpu;
  if (!out || (!nccl_comm && nranks > 1)) return fail(MUMODE_ERR_ARGUMENT, "comm_wrap: null pointer");
  *out = nullptr;
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks)
    return fail(MUMODE_ERR_ARGUMENT, "comm_wrap: bad rank / size");
  if (nranks > 1 && !nccl_api().ok) return fail(MUMODE_ERR_NCCL, nccl_api().why);
  MM_DEVICE(device);
  auto* c = new mumode_comm_s();
  c->comm = static_cast<ncclComm_t>(nccl_comm);
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  c->owned = false;
  return comm_finish(c, out);
}

int mumode_comm_destroy(mumode_comm_t c) {
  if (!c) return MUMODE_OK;
  mumode_gpu::DeviceGuard guard(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto e : c->events) cudaEventDestroy(e);
  mumode_gpu::p2p_unmap(c);
  if (c->ret_in) cudaEventDestroy(c->ret_in);
  if (c->ret_out) cudaEventDestroy(c->ret_out);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->owned && c->comm) mumode_gpu::nccl_api().comm_destroy(c->comm);
  delete c;
  return MUMODE_OK;
}

int mumode_comm_set_overlap_sms(mumode_comm_t c, int sms) {
  using namespace mumode_gpu;
  if (!c) return fail(MUMODE_ERR_ARGUMENT, "null comm");
  if (sms < 0 || sms > 128) return fail(MUMODE_ERR_ARGUMENT, "overlap SMs: 0..128");
  c->overlap_sms = sms;
  return MUMODE_OK;
}

int mumode_comm_set_exchange(mumode_comm_t c, int mode) {
  using namespace mumode_gpu;
  if (!c) return fail(MUMODE_ERR_ARGUMENT, "null comm");
  if (mode != 0 && mode != 1) return fail(MUMODE_ERR_ARGUMENT, "exchange: 0 = NCCL send/recv, 1 = peer stores");
  if (mode == 1 && c->nranks > 1 && !c->local && (!c->comm || !nccl_api().ok))
    return fail(MUMODE_ERR_NCCL, "peer-store exchange needs an NCCL communicator to map the peers");
  if (mode == 0 && c->local && c->nranks > 1)
    return fail(MUMODE_ERR_ARGUMENT, "a comm without NCCL exchanges by peer stores only");
  c->exchange = mode;
  return MUMODE_OK;
}

int mumode_slab_plan(int nranks, int d, const int64_t* m, const int64_t* n, int64_t* c_off, int64_t* a_off) {
  using namespace mumode_gpu;
  if (!m || !n || !c_off || !a_off) return fail(MUMODE_ERR_ARGUMENT, "slab plan: null pointer");
  return slab_plan(nranks, d, m, n, c_off, a_off);
}

int mumode_dist_plan(int nranks, int rank, int d, const int64_t* m, const int64_t* n, int chunks, int cplx,
                     int64_t* chunk_tab, int max_chunks, int* n_chunks, int64_t* op_tab, int max_ops, int* n_ops) {
  using namespace mumode_gpu;
  if (!m || !n || !n_chunks || !n_ops) return fail(MUMODE_ERR_ARGUMENT, "dist plan: null pointer");
  DistPlan pl;
  MM_TRY(dist_plan(nranks, rank, d, m, n, chunks, cplx ? 2 : 1, pl));
  *n_chunks = static_cast<int>(pl.ch.size());
  *n_ops = static_cast<int>(pl.ops.size());
  if (*n_chunks > max_chunks || *n_ops > max_ops || (max_chunks > 0 && !chunk_tab) || (max_ops > 0 && !op_tab))
    return fail(MUMODE_ERR_ARGUMENT, "dist plan: tables too small (sizes returned in n_chunks / n_ops)");
  for (size_t j = 0; j < pl.ch.size(); ++j) {
    chunk_tab[3 * j] = pl.ch[j].col0;
    chunk_tab[3 * j + 1] = pl.ch[j].w;
    chunk_tab[3 * j + 2] = pl.ch[j].send_off;
  }
  for (size_t k = 0; k < pl.ops.size(); ++k) {
    const DistOp& o = pl.ops[k];
    const int64_t row[6] = {o.chunk, o.kind, o.peer, o.buf_off, o.z_off, o.count};
    std::memcpy(op_tab + 6 * k, row, sizeof(row));
  }
  return MUMODE_OK;
}

int mumode_dist_return_plan(int nranks, int rank, int d, const int64_t* n, int64_t* op_tab, int max_ops,
                            int* n_ops) {
  using namespace mumode_gpu;
  if (!n || !n_ops) return fail(MUMODE_ERR_ARGUMENT, "dist plan: null pointer");
  int64_t c_off[kMaxRanks + 1], a_off[kMaxRanks + 1];
  std::vector<DistOp> ops;
  MM_TRY(return_plan(nranks, rank, d, n, ops, c_off, a_off, 1));
  *n_ops = static_cast<int>(ops.size());
  if (*n_ops > max_ops || (max_ops > 0 && !op_tab))
    return fail(MUMODE_ERR_ARGUMENT, "dist plan: tables too small (size returned in n_ops)");
  for (size_t k = 0; k < ops.size(); ++k) {
    const int64_t row[6] = {ops[k].chunk, ops[k].kind, ops[k].peer, ops[k].buf_off, ops[k].z_off, ops[k].count};
    std::memcpy(op_tab + 6 * k, row, sizeof(row));
  }
  return MUMODE_OK;
}

int mumode_dist_expint_f64(mumode_handle_t h, mumode_comm_t c, int d, const int64_t* m, const double* const* E,
                           const double* u0, double* u, int steps) {
  using namespace mumode_gpu;
  if (!h || !c) return fail(MUMODE_ERR_ARGUMENT, "dist_expint: null handle / comm");
  if (!m) return fail(MUMODE_ERR_ARGUMENT, "dist_expint: null extents");
  MM_DEVICE(h->device);
  return dist_expint(h, c, d, m, E, u0, u, steps);
}

int mumode_dist_tucker_f64(mumode_handle_t h, mumode_comm_t c, int d, const int64_t* m, const int64_t* n,
                           const double* T, const double* const* L, double* S, int chunks) {
  using namespace mumode_gpu;
  if (!h || !c) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: null handle / comm");
  if (!m || !n) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: null extents");
  MM_DEVICE(h->device);
  return dist_tucker(h, c, d, m, n, T, L, S, chunks, false);
}

int mumode_dist_tucker_c128(mumode_handle_t h, mumode_comm_t c, int d, const int64_t* m, const int64_t* n,
                            const double* T, const double* const* L, double* S, int chunks) {
  using namespace mumode_gpu;
  if (!h || !c) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: null handle / comm");
  if (!m || !n) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: null extents");
  MM_DEVICE(h->device);
  return dist_tucker(h, c, d, m, n, T, L, S, chunks, true);
}

int mumode_comm_create_local(mumode_comm_t* out, int device, int nranks, int rank) {
  using namespace mumode_gpu;
  if (!out) return fail(MUMODE_ERR_ARGUMENT, "comm_create_local: null pointer");
  *out = nullptr;
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks)
    return fail(MUMODE_ERR_ARGUMENT, "comm_create_local: bad rank / size");
  MM_DEVICE(device);
  auto* c = new mumode_comm_s();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  c->local = true;
  c->exchange = 1;
  return comm_finish(c, out);
}

int mumode_comm_ipc_export(mumode_comm_t c, int d, const int64_t* m, const int64_t* n, int cplx, void* handles) {
  using namespace mumode_gpu;
  if (!c || !m || !n || !handles) return fail(MUMODE_ERR_ARGUMENT, "comm_ipc_export: null pointer");
  MM_DEVICE(c->device);
  DistPlan pl;
  MM_TRY(dist_plan(c->nranks, c->rank, d, m, n, 1, cplx ? 2 : 1, pl));
  return p2p_export(c, p2p_zbytes(pl, c->nranks, cplx ? 2 : 1), handles);
}

int mumode_comm_ipc_import(mumode_comm_t c, int d, const int64_t* m, const int64_t* n, int cplx,
                           const void* all_handles) {
  using namespace mumode_gpu;
  if (!c || !m || !n || !all_handles) return fail(MUMODE_ERR_ARGUMENT, "comm_ipc_import: null pointer");
  MM_DEVICE(c->device);
  DistPlan pl;
  MM_TRY(dist_plan(c->nranks, c->rank, d, m, n, 1, cplx ? 2 : 1, pl));
  const size_t zbytes = p2p_zbytes(pl, c->nranks, cplx ? 2 : 1);
  if (c->pz[0].bytes < zbytes || !c->flags.p)
    return fail(MUMODE_ERR_ARGUMENT, "comm_ipc_import: export this shape first");
  return p2p_import(c, zbytes, all_handles);
}

int mumode_comm_ipc_handle_bytes(void) { return static_cast<int>(3 * mumode_gpu::kIpcHandleBytes); }

int mumode_dist_tucker_phase_f64(mumode_handle_t h, mumode_comm_t c, int d, const int64_t* m, const int64_t* n,
                                 const double* T, const double* const* L, double* S, int phase) {
  using namespace mumode_gpu;
  if (!h || !c) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: null handle / comm");
  if (!m || !n) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: null extents");
  if (phase < 0 || phase > 2) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: phase 0, 1 or 2");
  MM_DEVICE(h->device);
  return dist_tucker(h, c, d, m, n, T, L, S, 1, false, phase);
}

int mumode_dist_tucker_phase_c128(mumode_handle_t h, mumode_comm_t c, int d, const int64_t* m, const int64_t* n,
                                  const double* T, const double* const* L, double* S, int phase) {
  using namespace mumode_gpu;
  if (!h || !c) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: null handle / comm");
  if (!m || !n) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: null extents");
  if (phase < 0 || phase > 2) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: phase 0, 1 or 2");
  MM_DEVICE(h->device);
  return dist_tucker(h, c, d, m, n, T, L, S, 1, true, phase);
}

int mumode_comm_poll(mumode_handle_t h, mumode_comm_t c, int64_t timeout_ms) {
  using namespace mumode_gpu;
  if (!h || !c) return fail(MUMODE_ERR_ARGUMENT, "comm_poll: null handle / comm");
  MM_DEVICE(h->device);
  return comm_poll(h, c, timeout_ms);
}

int mumode_dist_local_f64(mumode_handle_t h, int nranks, int rank, int d, const int64_t* m, const int64_t* n,
                          const double* T, const double* const* L, double* send, double* Z, int chunks) {
  using namespace mumode_gpu;
  if (!h || !m || !n || !T || !L || !send || !Z) return fail(MUMODE_ERR_ARGUMENT, "dist_local: null pointer");
  MM_DEVICE(h->device);
  DistPlan pl;
  MM_TRY(dist_plan(nranks, rank, d, m, n, chunks, 1, pl));
  MM_TRY(h->scat_params.ensure(sizeof(ScatterParams)));  // keep the handle's single table intact
  static thread_local DevBuf tabs;
  MM_TRY(upload_scatter_tables(h, tabs, pl, nranks, rank, send, Z, 1));
  std::vector<int64_t> ext(m, m + d);
  for (size_t j = 0; j < pl.ch.size(); ++j) {
    const DistChunk& c = pl.ch[j];
    if (c.w == 0) continue;
    ext[d - 1] = c.w;
    MM_TRY(tucker_dev(h, d, ext.data(), n, T + pl.rows_in * c.col0, L, nullptr, false, false, 1, d - 1,
                      static_cast<const ScatterParams*>(tabs.p) + j));
  }
  return MUMODE_OK;
}

}  // extern "C"


