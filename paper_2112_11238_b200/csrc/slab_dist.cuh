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
    a.ok = all;
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

}  // namespace mumode_gpu

struct mumode_comm_s {
  ncclComm_t comm = nullptr;
  bool owned = false;
  int nranks = 1, rank = 0, device = 0;
  cudaStream_t stream = nullptr;          // exchange stream
  std::vector<cudaEvent_t> events;        // per-chunk "packed" + start/done
  mumode_gpu::DevBuf y, send, z;          // chunk intermediate, packed slab, received (A_r x m_d)
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

static int dist_tucker(mumode_handle_s* h, mumode_comm_s* cm, int d, const int64_t* m, const int64_t* n,
                       const double* T, const double* const* L, double* S, int chunks, bool cplx) {
  const int P = cm->nranks, r = cm->rank;
  if (cm->device != h->device) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: handle and comm on different devices");
  if (chunks < 0) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: chunks must be >= 0 (0 = auto)");
  int64_t c_off[kMaxRanks + 1], a_off[kMaxRanks + 1];
  MM_TRY(slab_plan(P, d, m, n, c_off, a_off));
  if (!T || !L || !S) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: null pointer");
  for (int k = 0; k < d; ++k)
    if (!L[k]) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: null matrix for mode " + std::to_string(k + 1));
  const int el = cplx ? 2 : 1;
  const int64_t rows_in = prod(m, 0, d - 1);       // slab rows per last-mode column
  const int64_t A = prod(n, 0, d - 1);             // rows after modes 1..d-1
  const int64_t A_r = a_off[r + 1] - a_off[r];
  const int64_t m_d = m[d - 1], n_d = n[d - 1];
  if (P == 1 && chunks <= 1) {
    // one rank: no exchange; modes 1..d-1 straight into Z, then mode d
    // (explicit chunks > 1 still take the general path: exercised by tests)
    MM_TRY(cm->z.ensure(size_t(std::max<int64_t>(A * m_d * el, 1)) * sizeof(double)));
    auto* Z = static_cast<double*>(cm->z.p);
    MM_TRY(tucker_dev(h, d, m, n, T, L, Z, false, cplx, 1, d - 1));
    const int64_t zext[2] = {A, m_d};
    return mode_product_dev(h, 2, zext, 2, n_d, Z, L[d - 1], 1, n_d, cplx, false, S);
  }
  // auto: split a slab only while every sub-slab keeps >= 4M elements, so the
  // per-chunk kernels still fill the GPU (at most 4 sub-slabs)
  if (chunks == 0) {
    const int64_t c_min = c_off[1] - c_off[0] - ((m[d - 1] % P) ? 1 : 0);
    chunks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(4, rows_in * std::max<int64_t>(c_min, 1) / (int64_t(1) << 22))));
  }
  // every rank's sub-slab split (all ranks derive all of them, so the posted
  // sends and receives match)
  int nch = 0;
  std::vector<std::vector<int64_t>> sub(P);
  for (int s = 0; s < P; ++s) {
    const int64_t cs = c_off[s + 1] - c_off[s];
    const int k = static_cast<int>(std::min<int64_t>(chunks, cs));
    sub[s].assign(k + 1, 0);
    even_splits(cs, k, sub[s].data());
    nch = std::max(nch, k);
  }
  auto width = [&](int s, int j) -> int64_t {
    return j + 1 < static_cast<int>(sub[s].size()) ? sub[s][j + 1] - sub[s][j] : 0;
  };
  int64_t wmax = 0;
  for (int j = 0; j < nch; ++j) wmax = std::max(wmax, width(r, j));
  const int64_t c_r = c_off[r + 1] - c_off[r];
  MM_TRY(cm->y.ensure(size_t(std::max<int64_t>(A * wmax * el, 1)) * sizeof(double)));
  MM_TRY(cm->send.ensure(size_t(std::max<int64_t>(A * c_r * el, 1)) * sizeof(double)));
  MM_TRY(cm->z.ensure(size_t(std::max<int64_t>(A_r * m_d * el, 1)) * sizeof(double)));
  MM_TRY(comm_events(cm, size_t(nch) + 2));
  auto* Y = static_cast<double*>(cm->y.p);
  auto* send = static_cast<double*>(cm->send.p);
  auto* Z = static_cast<double*>(cm->z.p);
  const ncclDataType_t f64 = ncclFloat64;

  // Z (and send) may still be read by the previous call's work on h->stream
  MM_CUDA(cudaEventRecord(cm->events[nch], h->stream));
  MM_CUDA(cudaStreamWaitEvent(cm->stream, cm->events[nch], 0));
  std::vector<int64_t> ext(m, m + d);
  PackOffsets off{};
  for (int q = 0; q <= P; ++q) off.a[q] = a_off[q] * el;
  for (int j = 0; j < nch; ++j) {
    const int64_t w = width(r, j);
    double* sj = send + A * sub[r][std::min<size_t>(j, sub[r].size() - 1)] * el;
    if (w > 0) {
      ext[d - 1] = w;
      const double* Tj = T + rows_in * sub[r][j] * el;
      MM_TRY(tucker_dev(h, d, ext.data(), n, Tj, L, Y, false, cplx, 1, d - 1));
      slab_pack_kernel<<<grid_for(A * el * w, h->num_sms), 256, 0, h->stream>>>(Y, sj, A * el, w, P, off);
      MM_CUDA(cudaGetLastError());
      h->launches++;
      MM_CUDA(cudaEventRecord(cm->events[j], h->stream));
      MM_CUDA(cudaStreamWaitEvent(cm->stream, cm->events[j], 0));
      // own row block: straight into its final columns
      const int64_t col0 = c_off[r] + sub[r][j];
      if (A_r > 0)
        MM_CUDA(cudaMemcpyAsync(Z + A_r * col0 * el, sj + a_off[r] * w * el, size_t(A_r * w * el) * sizeof(double),
                                cudaMemcpyDeviceToDevice, cm->stream));
    }
    if (P > 1) {
      auto& api = nccl_api();
      MM_NCCL(api.group_start());
      if (w > 0)
        for (int q = 0; q < P; ++q) {
          const int64_t rows = a_off[q + 1] - a_off[q];
          if (q == r || rows == 0) continue;
          MM_NCCL(api.send(sj + a_off[q] * w * el, size_t(rows * w * el), f64, q, cm->comm, cm->stream));
        }
      for (int s = 0; s < P; ++s) {
        const int64_t ws = width(s, j);
        if (s == r || ws == 0 || A_r == 0) continue;
        const int64_t col0 = c_off[s] + sub[s][j];
        MM_NCCL(api.recv(Z + A_r * col0 * el, size_t(A_r * ws * el), f64, s, cm->comm, cm->stream));
      }
      MM_NCCL(api.group_end());
    }
  }
  MM_CUDA(cudaEventRecord(cm->events[nch + 1], cm->stream));
  MM_CUDA(cudaStreamWaitEvent(h->stream, cm->events[nch + 1], 0));
  if (A_r == 0) return MUMODE_OK;
  const int64_t zext[2] = {A_r, m_d};
  return mode_product_dev(h, 2, zext, 2, n_d, Z, L[d - 1], 1, n_d, cplx, false, S);
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
  MM_CUDA(cudaSetDevice(device));
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
  MM_CUDA(cudaSetDevice(device));
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
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto e : c->events) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->owned && c->comm) mumode_gpu::nccl_api().comm_destroy(c->comm);
  delete c;
  return MUMODE_OK;
}

int mumode_slab_plan(int nranks, int d, const int64_t* m, const int64_t* n, int64_t* c_off, int64_t* a_off) {
  using namespace mumode_gpu;
  if (!m || !n || !c_off || !a_off) return fail(MUMODE_ERR_ARGUMENT, "slab plan: null pointer");
  return slab_plan(nranks, d, m, n, c_off, a_off);
}

int mumode_dist_tucker_f64(mumode_handle_t h, mumode_comm_t c, int d, const int64_t* m, const int64_t* n,
                           const double* T, const double* const* L, double* S, int chunks) {
  using namespace mumode_gpu;
  if (!h || !c) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: null handle / comm");
  if (!m || !n) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: null extents");
  MM_CUDA(cudaSetDevice(h->device));
  return dist_tucker(h, c, d, m, n, T, L, S, chunks, false);
}

int mumode_dist_tucker_c128(mumode_handle_t h, mumode_comm_t c, int d, const int64_t* m, const int64_t* n,
                            const double* T, const double* const* L, double* S, int chunks) {
  using namespace mumode_gpu;
  if (!h || !c) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: null handle / comm");
  if (!m || !n) return fail(MUMODE_ERR_ARGUMENT, "dist_tucker: null extents");
  MM_CUDA(cudaSetDevice(h->device));
  return dist_tucker(h, c, d, m, n, T, L, S, chunks, true);
}

}  // extern "C"
