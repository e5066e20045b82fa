// C-ABI implementation of the B200 mu-mode product / Tucker engine
// (include/mumode_gpu.h). Host orchestration only: argument checks with the
// reference's error contract, workspace + TMA-descriptor ownership, kernel
// selection, the Tucker chain, the exponential-integrator graph, and the
// host-buffer drop-in entry points. All arithmetic runs in the CUDA kernels of
// generic.cuh / tma_dmma.cuh / elementwise kernels below; there is no CPU
// compute path.
#include <cudaTypedefs.h>

#include <cstdio>
#include <algorithm>
#include <atomic>
#include <cstring>
#include <type_traits>
#include <map>
#include <unordered_map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/mumode_gpu.h"
#include "common.cuh"
#include "generic.cuh"
#include "tma_dmma.cuh"
#include "fused.cuh"
#include "fused_ws.cuh"
#include "tail.cuh"
#include "tail_ws.cuh"
#include "skinny.cuh"
#include "tma_chain.cuh"
#include "ldg_dmma.cuh"
#include "lu_solve.cuh"
#include "spair.cuh"
#include "block.cuh"
#include "kron12.cuh"

namespace mumode_gpu {

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

#define MM_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      set_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call); \
      return MUMODE_ERR_CUDA;                                                          \
    }                                                                                  \
  } while (0)

#define MM_TRY(expr)          \
  do {                        \
    int rc_ = (expr);         \
    if (rc_ != MUMODE_OK) return rc_; \
  } while (0)

static int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

// ------------------------------------------------------------------ handle
// Bumped whenever any workspace buffer is (re)allocated: captured CUDA graphs
// hold raw workspace pointers and by-value TMA descriptors, so a graph
// captured before a reallocation must not be replayed after it.
static std::atomic<uint64_t> g_workspace_gen{0};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t want) {
    if (want <= bytes) return MUMODE_OK;
    g_workspace_gen.fetch_add(1, std::memory_order_relaxed);
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (cudaMalloc(&p, want) != cudaSuccess) {
      cudaGetLastError();
      return fail(MUMODE_ERR_OOM, "device allocation of " + std::to_string(want) + " bytes failed");
    }
    bytes = want;
    return MUMODE_OK;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

using MapKey = std::vector<uint64_t>;  // base, rank, swizzle, dims, strides, box
struct MapKeyHash {
  size_t operator()(const MapKey& k) const noexcept {
    uint64_t h = 1469598103934665603ull;
    for (uint64_t v : k) h = (h ^ v) * 1099511628211ull;
    return static_cast<size_t>(h);
  }
};

// Dependency tables of the chain kernel for one shape and config pair
// (tma_chain.cuh): per mode boundary, the consumer M-tile counters' targets
// and the CSR list of counters each producer tile increments.
struct ChainPlan {
  DevBuf tables;    // int32 targets / sig_off / sig_idx of every boundary
  DevBuf counters;  // int32, zeroed per launch
  size_t counter_ints = 0;
  std::vector<int64_t> target_off, sigoff_off, sigidx_off, ctr_off;  // per mode, in ints
};

// In-place block pass (block.cuh) for one shape: the host layout and its
// device copies (row tables, copy segments), never reallocated.
struct BlockPlan {
  BlockLayout lay;
  DevBuf tab, seg;
  int NB = 0, G = 1, smem = 0, P4 = 0, NF = 0;
  int ls_off = 0, tab_soff = 0, bar_off = 0;
  int64_t nblocks = 0;
};

struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  int64_t nodes = 0;
  uint64_t gen = 0;  // g_workspace_gen at capture
};

// Make the handle's device current for the scope of one entry point and
// restore the caller's device on exit (as torch's DeviceGuard does).
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int device) {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      cudaGetLastError();
      prev = -1;
    }
    if (prev != device) err = cudaSetDevice(device);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

#define MM_DEVICE(dev)                                                                         \
  ::mumode_gpu::DeviceGuard device_guard_(dev);                                                \
  do {                                                                                         \
    if (device_guard_.err != cudaSuccess) {                                                    \
      cudaGetLastError();                                                                      \
      return fail(MUMODE_ERR_CUDA, std::string("cudaSetDevice failed: ") +                     \
                                       cudaGetErrorString(device_guard_.err));                 \
    }                                                                                          \
  } while (0)

}  // namespace mumode_gpu

struct mumode_handle_s {
  int device = 0;
  int num_sms = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int policy = 0;
  int aux_policy = 0;  // 23..26: itucker / kronsumv kernel choices; every other decision stays auto
  int sm_reserve = 0;           // SMs left free by the persistent kernels (dist exchange overlap)
  int64_t launches = 0;
  mumode_gpu::DevBuf ws[3];     // Tucker ping-pong intermediates + expint buffer
  mumode_gpu::DevBuf pad_in, pad_out, lpad;  // odd-leading-extent chains run on an even-padded copy
  mumode_gpu::DevBuf lstage;    // a factor with an odd leading dimension, re-laid with an even one
  mumode_gpu::DevBuf scat_params, scat_tmp, scat_mid;  // scatter table; fallback output; chain intermediate
  mumode_gpu::DevBuf lbuf;      // materialised op(L) for adjoint / promotion
  mumode_gpu::DevBuf lperm;     // itucker: per-mode row permutations of the pivots
  mumode_gpu::DevBuf host_in, host_out, host_mats, host_mid;  // host drop-in staging
  mumode_gpu::DevBuf slot_in[2], slot_out[2], slot_mats[2];   // pipelined host calls, double-buffered
  int64_t host_calls = 0;
  cudaStream_t copy_in = nullptr, copy_out = nullptr;         // host drop-in copy engines
  std::vector<cudaEvent_t> events;                            // pipeline events (reused)
  std::unordered_map<mumode_gpu::MapKey, CUtensorMap, mumode_gpu::MapKeyHash> maps;
  std::map<std::vector<uint64_t>, mumode_gpu::GraphEntry> graphs;
  std::map<std::vector<int64_t>, std::unique_ptr<mumode_gpu::ChainPlan>> chains;  // per shape + configs
  std::map<std::vector<int64_t>, std::unique_ptr<mumode_gpu::BlockPlan>> blocks;  // per block-pass shape
};

namespace mumode_gpu {

// CTAs of a persistent kernel: one per SM, minus the SMs reserved so NCCL's
// kernels can run beside the compute during an overlapped exchange.
static int persistent_sms(const mumode_handle_s* h) { return std::max(1, h->num_sms - h->sm_reserve); }

// Launch with programmatic stream serialization (PDL): the kernel may start
// while its predecessor in the stream drains; it calls griddepcontrol.wait
// before its first global access.
template <class K, class... Args>
static int launch_pdl(K kernel, int grid, int threads, int smem, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(static_cast<unsigned>(threads));
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MM_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
  static const bool debug_sync = getenv("MUMODE_DEBUG_SYNC") != nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (debug_sync) cudaStreamIsCapturing(stream, &cap);
  if (debug_sync && cap == cudaStreamCaptureStatusNone) {  // diagnostics: name the launch that faults
    const cudaError_t e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) {
      const char* name = nullptr;
      cudaFuncGetName(&name, reinterpret_cast<const void*>(kernel));
      fprintf(stderr, "mumode: kernel %s (grid %d, block %d, smem %d) failed: %s\n", name ? name : "?", grid,
              threads, smem, cudaGetErrorString(e));
      return fail(MUMODE_ERR_CUDA, std::string("kernel failed: ") + (name ? name : "?"));
    }
  }
  return MUMODE_OK;
}

// Opt a kernel instance into its dynamic shared memory once per (device,
// kernel): function attributes belong to the device's context, so a second
// GPU in the same process needs its own opt-in.
template <class K>
static int smem_opt_in(K kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  MM_CUDA(cudaGetDevice(&dev));
  const std::pair<int, const void*> key{dev, reinterpret_cast<const void*>(kernel)};
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return MUMODE_OK;
  MM_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done[key] = bytes;
  return MUMODE_OK;
}

// ------------------------------------------------------------------ TMA maps
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// fp64-typed tiled map (dims/strides in doubles); 64B swizzle for 8-double
// boxes (real), 128B swizzle for 16-double boxes (8 complex). dims/strides in elements (dim0 contiguous).
static int get_map(mumode_handle_s* h, const void* base, int rank, const uint64_t* dims,
                   const uint64_t* strides_el, const uint32_t* box, const CUtensorMap** out,
                   int swz = 0) {  // 0: 64B swizzle, 1 (true): 128B, 2: none
  MapKey key{reinterpret_cast<uint64_t>(base), uint64_t(rank), uint64_t(swz)};
  for (int r = 0; r < rank; ++r) key.push_back(dims[r]);
  for (int r = 0; r + 1 < rank; ++r) key.push_back(strides_el[r]);
  for (int r = 0; r < rank; ++r) key.push_back(box[r]);
  auto it = h->maps.find(key);
  if (it != h->maps.end()) {
    *out = &it->second;
    return MUMODE_OK;
  }
  auto fn = encode_fn();
  if (!fn) return fail(MUMODE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  CUtensorMap map;
  cuuint64_t gdim[5];
  cuuint64_t gstride[4];
  cuuint32_t bdim[5], estride[5];
  for (int r = 0; r < rank; ++r) {
    gdim[r] = dims[r];
    bdim[r] = box[r];
    estride[r] = 1;
  }
  for (int r = 0; r + 1 < rank; ++r) gstride[r] = strides_el[r] * sizeof(double);
  CUresult res = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void*>(base), gdim,
                    gstride, bdim, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swz == 1 ? CU_TENSOR_MAP_SWIZZLE_128B
                             : (swz == 2 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_64B),
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (res != CUDA_SUCCESS)
    return fail(MUMODE_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(res) + ")");
  auto ins = h->maps.emplace(key, map);
  *out = &ins.first->second;
  return MUMODE_OK;
}

// ------------------------------------------------------------------ small kernels
__global__ void transpose_conj_kernel(const double* __restrict__ L, double* __restrict__ out,
                                      int64_t rows, int64_t cols, int cplx, int conj) {
  // out (cols x rows) = L^T (or L^H), column-major.
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % cols, j = e / cols;  // out(i, j) = L(j, i)
    const int64_t src = j + i * rows;
    if (cplx) {
      out[2 * e] = L[2 * src];
      out[2 * e + 1] = conj ? -L[2 * src + 1] : L[2 * src + 1];
    } else {
      out[e] = L[src];
    }
  }
}

__global__ void real_to_complex_kernel(const double* __restrict__ x, double* __restrict__ z,
                                       int64_t n) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    z[2 * e] = x[e];
    z[2 * e + 1] = 0.0;
  }
}


// Slab-transpose pack: Y (A x C, column-major) -> send buffer holding, for
// each destination q, the row block Y[a_off[q] : a_off[q+1], 0:C] as a
// contiguous column-major (|A_q| x C) matrix, blocks in q order. One CTA per
// (column, destination) pair copies one contiguous run to one contiguous run
// (no per-element index arithmetic: the kernel runs at copy bandwidth).
// UNPACK = true is the inverse (send layout -> Y).
constexpr int kMaxRanks = 64;
struct PackOffsets {
  int64_t a[kMaxRanks + 1];
};
template <bool UNPACK>
__global__ void __launch_bounds__(256) slab_pack_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                        int64_t A, int64_t C, int P, PackOffsets off) {
  constexpr int64_t SEG = 4096;  // doubles per CTA work item (long runs are split over CTAs)
  const int64_t pairs = C * P;
  for (int64_t pr = blockIdx.x; pr < pairs; pr += gridDim.x) {
    const int64_t c = pr / P;
    const int q = static_cast<int>(pr - c * P);
    const int64_t lo = off.a[q], rows = off.a[q + 1] - lo;
    const int64_t y0 = lo + c * A, s0 = lo * C + c * rows;
    for (int64_t seg = blockIdx.y * SEG; seg < rows; seg += int64_t(gridDim.y) * SEG) {
      const int64_t len = rows - seg < SEG ? rows - seg : SEG;
      const double* src = in + (UNPACK ? s0 : y0) + seg;
      double* dst = out + (UNPACK ? y0 : s0) + seg;
      if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15u) == 0) {
        const int64_t n2 = len / 2;
        for (int64_t i = threadIdx.x; i < n2; i += blockDim.x)
          reinterpret_cast<double2*>(dst)[i] = reinterpret_cast<const double2*>(src)[i];
        if ((len & 1) && threadIdx.x == 0) dst[len - 1] = src[len - 1];
      } else {
        for (int64_t i = threadIdx.x; i < len; i += blockDim.x) dst[i] = src[i];
      }
    }
  }
}

// Fallback of the scatter epilogue: Y (A x C, el doubles per element) ->
// dst[q] rows (A_q x ...) at column col0 + c, one contiguous run per
// (column, rank).
__global__ void __launch_bounds__(256) scatter_copy_kernel(const double* __restrict__ Y, int64_t A, int64_t C, int el,
                                                           const ScatterParams* __restrict__ sp) {
  const int P = sp->P;
  for (int64_t pr = blockIdx.x; pr < C * P; pr += gridDim.x) {
    const int64_t c = pr / P;
    const int q = static_cast<int>(pr - c * P);
    const int64_t lo = sp->a_off[q] * el, rows = (sp->a_off[q + 1] - sp->a_off[q]) * el;
    const double* src = Y + c * A * el + lo;
    double* dst = sp->dst[q] + rows * (sp->col0 + c);
    for (int64_t i = blockIdx.y * int64_t(blockDim.x) + threadIdx.x; i < rows; i += int64_t(gridDim.y) * blockDim.x)
      dst[i] = src[i];
  }
}

// w(a, n) /= (esum_front[a] + ev_last[n]) for the direct Kronecker-sum solve;
// denominators summed in the reference's order (imex.cpp:70-77). One CTA row
// per column n (no per-element division).
__global__ void __launch_bounds__(256) eigsum_divide_kernel(double* __restrict__ w, const double* __restrict__ esum_front,
                                                            const double* __restrict__ ev_last, int64_t A, int64_t N) {
  for (int64_t n = blockIdx.y; n < N; n += gridDim.y) {
    const double en = ev_last[n];
    double* col = w + n * A;
    for (int64_t a = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; a < A; a += int64_t(gridDim.x) * blockDim.x)
      col[a] /= (esum_front[a] + en);
  }
}

// (column, destination) pairs on x, 4096-double segments of long runs on y
// dst (rd x cd) = src (rs x cs, leading dimension src_ld >= rs) zero-extended
// / cropped, column-major.
__global__ void __launch_bounds__(256) pad2d_kernel(const double* __restrict__ src, int64_t rs, int64_t cs,
                                                    int64_t src_ld, double* __restrict__ dst, int64_t rd,
                                                    int64_t cd) {
  for (int64_t c = blockIdx.y; c < cd; c += gridDim.y)
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < rd; r += int64_t(gridDim.x) * blockDim.x)
      dst[r + c * rd] = (r < rs && c < cs) ? src[r + c * src_ld] : 0.0;
}

static dim3 pad_grid(int64_t rows, int64_t cols, int sms) {
  const int64_t gx = std::min<int64_t>((rows + 255) / 256, 8);
  const int64_t gy = std::max<int64_t>(1, std::min<int64_t>(cols, int64_t(sms) * 16 / gx));
  return dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
}

static dim3 pack_grid(int64_t A, int64_t C, int P, int sms) {
  const int64_t pairs = C * P, cap = int64_t(sms) * 16;
  const int64_t segs = std::min<int64_t>((A / P + 4095) / 4096 + 1, 64);
  const int64_t gx = std::max<int64_t>(1, std::min(pairs, std::max<int64_t>(cap / segs, 1)));
  return dim3(static_cast<unsigned>(gx), static_cast<unsigned>(segs));
}

static int grid_for(int64_t n, int sms) {
  int64_t b = (n + 255) / 256;
  int64_t cap = int64_t(sms) * 8;
  return static_cast<int>(b < cap ? (b > 0 ? b : 1) : cap);
}

// ------------------------------------------------------------------ checks
static int check_shape(int d, const int64_t* m, const char* who) {
  if (d < 1) return fail(MUMODE_ERR_ARGUMENT, "tensor order must be >= 1");
  if (d > 32) return fail(MUMODE_ERR_ARGUMENT, std::string(who) + ": tensor order above 32");
  for (int k = 0; k < d; ++k)
    if (m[k] < 1) return fail(MUMODE_ERR_ARGUMENT, "tensor extents must be positive");
  return MUMODE_OK;
}

static bool aligned16_ptr(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

static int64_t prod(const int64_t* m, int lo, int hi) {
  int64_t p = 1;
  for (int k = lo; k < hi; ++k) p *= m[k];
  return p;
}

}  // namespace mumode_gpu

#include "dispatch.cuh"
#include "chain.cuh"


using namespace mumode_gpu;

// ====================================================================== C-ABI
extern "C" {

const char* mumode_last_error(void) { return g_err.c_str(); }
const char* mumode_version(void) { return "mumode-b200 0.1 (sm_100a)"; }

int mumode_handle_create(mumode_handle_t* out, int device) {
  if (!out) return fail(MUMODE_ERR_ARGUMENT, "null handle pointer");
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(MUMODE_ERR_CUDA, "no CUDA device available: the mu-mode engine has no CPU path");
  }
  if (device < 0 || device >= ndev) return fail(MUMODE_ERR_ARGUMENT, "bad device index");
  MM_DEVICE(device);
  int major = 0;
  MM_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  if (major != 10)
    return fail(MUMODE_ERR_CUDA, "this build targets sm_100a (B200); device has compute major " +
                                     std::to_string(major));
  auto* h = new mumode_handle_s();
  h->device = device;
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete h;
    return fail(MUMODE_ERR_CUDA, "stream creation failed");
  }
  h->stream = h->own_stream;
  *out = h;
  return MUMODE_OK;
}

int mumode_handle_destroy(mumode_handle_t h) {
  if (!h) return MUMODE_OK;
  DeviceGuard guard(h->device);
  cudaStreamSynchronize(h->stream);
  for (auto& kv : h->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  for (auto e : h->events) cudaEventDestroy(e);
  if (h->copy_in) cudaStreamDestroy(h->copy_in);
  if (h->copy_out) cudaStreamDestroy(h->copy_out);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  delete h;
  return MUMODE_OK;
}

int mumode_set_stream(mumode_handle_t h, void* stream) {
  if (!h) return fail(MUMODE_ERR_ARGUMENT, "null handle");
  // The caller's stream exactly (NULL = the legacy default stream, which is
  // what torch's default stream reports), so work is ordered with theirs.
  h->stream = static_cast<cudaStream_t>(stream);
  return MUMODE_OK;
}

void* mumode_get_stream(mumode_handle_t h) { return h ? static_cast<void*>(h->stream) : nullptr; }

int64_t mumode_launch_count(mumode_handle_t h) { return h ? h->launches : -1; }

int mumode_set_kernel_policy(mumode_handle_t h, int policy) {
  if (!h || policy < 0 || policy > 26) return fail(MUMODE_ERR_ARGUMENT, "bad kernel policy");
  // 3..6 force real tile configuration 0..3 / complex configuration 0..3
  h->policy = policy >= 23 ? 0 : policy;
  h->aux_policy = policy >= 23 ? policy : 0;
  return MUMODE_OK;
}

static int mode_product_entry(mumode_handle_t h, int d, const int64_t* m, int mu, int64_t n_mu,
                              const double* T, const double* L, double* S, bool cplx) {
  if (!h) return fail(MUMODE_ERR_ARGUMENT, "null handle");
  MM_TRY(check_shape(d, m, "mode_product"));
  if (mu < 1 || mu > d)
    return fail(MUMODE_ERR_ARGUMENT, "mode index " + std::to_string(mu) + " out of range 1.." +
                                         std::to_string(d));
  if (n_mu < 1) return fail(MUMODE_ERR_ARGUMENT, "matrix dimensions must be positive");
  if (!T || !L || !S) return fail(MUMODE_ERR_ARGUMENT, "mode_product: null pointer");
  {
    const int el = cplx ? 2 : 1;
    std::vector<int64_t> out(m, m + d);
    out[mu - 1] = n_mu;
    MM_TRY(check_no_alias(T, prod(m, 0, d) * el, S, prod(out.data(), 0, d) * el, "mode_product"));
  }
  MM_DEVICE(h->device);
  return mode_product_dev(h, d, m, mu, n_mu, T, L, 1, n_mu, cplx, false, S);
}

int mumode_mode_product_f64(mumode_handle_t h, int d, const int64_t* m, int mu, int64_t n_mu,
                            const double* T, const double* L, double* S) {
  return mode_product_entry(h, d, m, mu, n_mu, T, L, S, false);
}
int mumode_mode_product_c128(mumode_handle_t h, int d, const int64_t* m, int mu, int64_t n_mu,
                             const double* T, const double* L, double* S) {
  return mode_product_entry(h, d, m, mu, n_mu, T, L, S, true);
}

static int tucker_entry(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                        const double* T, const double* const* L, double* S, int adjoint,
                        bool cplx) {
  if (!h) return fail(MUMODE_ERR_ARGUMENT, "null handle");
  MM_TRY(check_stack(d, m, n, T, L, S, adjoint ? "cttucker" : "tucker"));
  if (d == 1) {  // d >= 2 reads T only in mode 1 and writes S only in mode d
    const int el = cplx ? 2 : 1;
    MM_TRY(check_no_alias(T, prod(m, 0, d) * el, S, prod(n, 0, d) * el, "tucker"));
  }
  MM_DEVICE(h->device);
  return tucker_dev(h, d, m, n, T, L, S, adjoint != 0, cplx);
}

int mumode_tucker_f64(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                      const double* T, const double* const* L, double* S, int adjoint) {
  return tucker_entry(h, d, m, n, T, L, S, adjoint, false);
}
int mumode_tucker_c128(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                       const double* T, const double* const* L, double* S, int adjoint) {
  return tucker_entry(h, d, m, n, T, L, S, adjoint, true);
}

int mumode_tucker_range_f64(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                            const double* T, const double* const* L, double* S, int mu_lo,
                            int mu_hi) {
  if (!h) return fail(MUMODE_ERR_ARGUMENT, "null handle");
  MM_TRY(check_shape(d, m, "tucker_range"));
  if (mu_lo < 1 || mu_hi > d || mu_lo > mu_hi)
    return fail(MUMODE_ERR_ARGUMENT, "tucker_range: bad mode range");
  if (!T || !L || !S || !n) return fail(MUMODE_ERR_ARGUMENT, "tucker_range: null pointer");
  for (int k = mu_lo - 1; k < mu_hi; ++k)
    if (!L[k] || n[k] < 1) return fail(MUMODE_ERR_ARGUMENT, "tucker_range: bad matrix for mode " + std::to_string(k + 1));
  MM_DEVICE(h->device);
  return tucker_dev(h, d, m, n, T, L, S, false, false, mu_lo, mu_hi);
}

static int tucker_range_scatter(mumode_handle_t h, int d, const int64_t* m, const int64_t* n, const double* T,
                                const double* const* L, int mu_lo, int mu_hi, int P, const int64_t* a_off,
                                int64_t col0, double* const* dst, bool cplx) {
  if (!h) return fail(MUMODE_ERR_ARGUMENT, "null handle");
  MM_TRY(check_shape(d, m, "tucker_range_scatter"));
  if (mu_lo < 1 || mu_hi > d || mu_lo > mu_hi)
    return fail(MUMODE_ERR_ARGUMENT, "tucker_range_scatter: bad mode range");
  if (!T || !L || !n || !a_off || !dst) return fail(MUMODE_ERR_ARGUMENT, "tucker_range_scatter: null pointer");
  if (P < 1 || P > kScatterMaxRanks) return fail(MUMODE_ERR_ARGUMENT, "tucker_range_scatter: 1..64 ranks");
  for (int k = mu_lo - 1; k < mu_hi; ++k)
    if (!L[k] || n[k] < 1)
      return fail(MUMODE_ERR_ARGUMENT, "tucker_range_scatter: bad matrix for mode " + std::to_string(k + 1));
  // rows of the scattered matrix: every extent up to mode mu_hi (outputs
  // for modes in the range), columns: the extents after it
  int64_t rows = 1;
  for (int k = 0; k < mu_hi; ++k) rows *= (k >= mu_lo - 1) ? n[k] : m[k];
  if (a_off[0] != 0 || a_off[P] != rows)
    return fail(MUMODE_ERR_SIZE, "tucker_range_scatter: row offsets must cover the result's rows");
  for (int q = 0; q < P; ++q) {
    if (a_off[q + 1] < a_off[q]) return fail(MUMODE_ERR_ARGUMENT, "tucker_range_scatter: offsets must ascend");
    if (!dst[q] && a_off[q + 1] > a_off[q]) return fail(MUMODE_ERR_ARGUMENT, "tucker_range_scatter: null destination");
  }
  MM_DEVICE(h->device);
  ScatterParams sp{};
  sp.P = P;
  sp.col0 = col0;
  for (int q = 0; q <= P; ++q) sp.a_off[q] = a_off[q];
  for (int q = 0; q < P; ++q) sp.dst[q] = dst[q];
  MM_TRY(h->scat_params.ensure(sizeof(ScatterParams)));
  auto* dsp = static_cast<ScatterParams*>(h->scat_params.p);
  MM_CUDA(cudaMemcpyAsync(dsp, &sp, sizeof(sp), cudaMemcpyHostToDevice, h->stream));
  return tucker_dev(h, d, m, n, T, L, nullptr, false, cplx, mu_lo, mu_hi, dsp);
}

int mumode_tucker_range_scatter_f64(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                                    const double* T, const double* const* L, int mu_lo, int mu_hi, int P,
                                    const int64_t* a_off, int64_t col0, double* const* dst) {
  return tucker_range_scatter(h, d, m, n, T, L, mu_lo, mu_hi, P, a_off, col0, dst, false);
}

int mumode_tucker_range_scatter_c128(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                                     const double* T, const double* const* L, int mu_lo, int mu_hi, int P,
                                     const int64_t* a_off, int64_t col0, double* const* dst) {
  return tucker_range_scatter(h, d, m, n, T, L, mu_lo, mu_hi, P, a_off, col0, dst, true);
}

int mumode_slab_pack_f64(mumode_handle_t h, int64_t A, int64_t C, int P, const int64_t* a_off,
                         const double* Y, double* send) {
  if (!h || !a_off || !Y || !send) return fail(MUMODE_ERR_ARGUMENT, "slab_pack: null pointer");
  if (P < 1 || P > kMaxRanks) return fail(MUMODE_ERR_ARGUMENT, "slab_pack: 1..64 ranks");
  if (a_off[0] != 0 || a_off[P] != A) return fail(MUMODE_ERR_SIZE, "slab_pack: row offsets must cover 0..A");
  PackOffsets off{};
  for (int q = 0; q <= P; ++q) off.a[q] = a_off[q];
  MM_DEVICE(h->device);
  slab_pack_kernel<false><<<pack_grid(A, C, P, h->num_sms), 256, 0, h->stream>>>(Y, send, A, C, P, off);
  MM_CUDA(cudaGetLastError());
  h->launches++;
  return MUMODE_OK;
}

int mumode_slab_unpack_f64(mumode_handle_t h, int64_t A, int64_t C, int P, const int64_t* a_off,
                           const double* send, double* Y) {
  if (!h || !a_off || !Y || !send) return fail(MUMODE_ERR_ARGUMENT, "slab_unpack: null pointer");
  if (P < 1 || P > kMaxRanks) return fail(MUMODE_ERR_ARGUMENT, "slab_unpack: 1..64 ranks");
  if (a_off[0] != 0 || a_off[P] != A) return fail(MUMODE_ERR_SIZE, "slab_unpack: row offsets must cover 0..A");
  PackOffsets off{};
  for (int q = 0; q <= P; ++q) off.a[q] = a_off[q];
  MM_DEVICE(h->device);
  slab_pack_kernel<true><<<pack_grid(A, C, P, h->num_sms), 256, 0, h->stream>>>(send, Y, A, C, P, off);
  MM_CUDA(cudaGetLastError());
  h->launches++;
  return MUMODE_OK;
}

int mumode_kronsum_solve_f64(mumode_handle_t h, int d, const int64_t* m, const double* const* Q,
                             const double* const* Qt, const double* const* evals, const double* b,
                             double* x) {
  if (!h) return fail(MUMODE_ERR_ARGUMENT, "null handle");
  MM_TRY(check_stack(d, m, m, b, Q, x, "kronsum_solve"));
  if (!Qt || !evals) return fail(MUMODE_ERR_ARGUMENT, "kronsum_solve: null pointer");
  for (int k = 0; k < d; ++k)
    if (!Qt[k] || !evals[k])
      return fail(MUMODE_ERR_ARGUMENT, "kronsum_solve: null data for mode " + std::to_string(k + 1));
  MM_DEVICE(h->device);
  const int64_t numel = prod(m, 0, d);
  const int64_t A = prod(m, 0, d - 1), N = m[d - 1];
  // eigenvalue sums over modes 1..d-1, built mode by mode: esum(a) =
  // ((0 + ev_1) + ev_2) + ... in the reference's summation order (imex.cpp:73-75)
  std::vector<double> esum(static_cast<size_t>(A + N));
  esum[0] = 0.0;
  int64_t len = 1;
  for (int k = 0; k < d - 1; ++k) {
    for (int64_t jk = m[k] - 1; jk >= 0; --jk)  // in place, high blocks first
      for (int64_t a = 0; a < len; ++a) esum[static_cast<size_t>(a + len * jk)] = esum[static_cast<size_t>(a)] + evals[k][jk];
    len *= m[k];
  }
  // a zero denominator esum[a] + ev_last[n] (the reference throws on it,
  // imex.cpp:76-77) exists iff ev_last[n] == -esum[a] exactly (IEEE: x + y
  // rounds to 0 only when y == -x): binary search in the sorted ev_last
  std::vector<double> last(evals[d - 1], evals[d - 1] + N);
  std::sort(last.begin(), last.end());
  for (int64_t a = 0; a < A; ++a)
    if (std::binary_search(last.begin(), last.end(), -esum[static_cast<size_t>(a)]))
      return fail(MUMODE_ERR_NUMERICAL, "imex direct backend: singular implicit operator");
  for (int64_t n = 0; n < N; ++n) esum[static_cast<size_t>(A + n)] = evals[d - 1][n];
  MM_TRY(h->ws[2].ensure(size_t(numel) * sizeof(double)));
  MM_TRY(h->lbuf.ensure(esum.size() * sizeof(double)));
  double* w = static_cast<double*>(h->ws[2].p);
  double* dsum = static_cast<double*>(h->lbuf.p);
  // pageable source: the call returns once esum is staged, so it may go
  MM_CUDA(cudaMemcpyAsync(dsum, esum.data(), esum.size() * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  // w = b x {Q^T}, divided by the eigenvalue sums in the last mode's epilogue
  MM_TRY(tucker_dev(h, d, m, m, b, Qt, w, false, false, 1, d, nullptr, dsum, dsum + A));
  return tucker_dev(h, d, m, m, w, Q, x, false, false);
}

int mumode_tucker_promote(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                          const double* T, const double* const* L, double* S, int adjoint) {
  if (!h) return fail(MUMODE_ERR_ARGUMENT, "null handle");
  MM_TRY(check_stack(d, m, n, T, L, S, adjoint ? "cttucker" : "tucker"));
  MM_DEVICE(h->device);
  const int64_t numel = prod(m, 0, d);
  MM_TRY(h->ws[2].ensure(size_t(numel) * 2 * sizeof(double)));
  double* z = static_cast<double*>(h->ws[2].p);
  real_to_complex_kernel<<<grid_for(numel, h->num_sms), 256, 0, h->stream>>>(T, z, numel);
  MM_CUDA(cudaGetLastError());
  h->launches++;
  return tucker_dev(h, d, m, n, z, L, S, adjoint != 0, true);
}

static int kronsumv_entry(mumode_handle_t h, int d, const int64_t* m, const double* V, const double* const* A,
                          double* W, bool cplx) {
  if (!h) return fail(MUMODE_ERR_ARGUMENT, "null handle");
  MM_TRY(check_stack(d, m, m, V, A, W, "kronsumv"));
  const int el = cplx ? 2 : 1;
  MM_TRY(check_no_alias(V, prod(m, 0, d) * el, W, prod(m, 0, d) * el, "kronsumv"));
  MM_DEVICE(h->device);
  // W = V x_1 A_1, then W += V x_mu A_mu for mu = 2..d in the products'
  // epilogues (the reference's acc += term order, tucker.hpp:222-231): no
  // term buffer and no separate accumulation pass over W.
  int first = 2;
  // small square modes 1 and 2 (even extents 10..24): both terms in one pass over V (kron12.cuh)
  if (!cplx && d >= 3 && m[0] == m[1] && m[0] >= 10 && m[0] <= 24 && m[0] % 2 == 0 && prod(m, 2, d) >= 2048 &&
      aligned16_ptr(V) && aligned16_ptr(W) && h->aux_policy != 26) {
    const int n = static_cast<int>(m[0]), nb = (n + 7) / 8;
    const int64_t nsl = prod(m, 2, d);
    const size_t smem = kron12_smem(nb);
    const int grid = static_cast<int>(std::min<int64_t>((nsl + kKron12Warps - 1) / kKron12Warps, h->num_sms));
    auto launch = [&](auto kern) -> int {
      MM_TRY(smem_opt_in(kern, static_cast<int>(smem)));
      kern<<<grid, 32 * kKron12Warps, smem, h->stream>>>(V, A[0], A[1], W, nsl, n);
      return MUMODE_OK;
    };
    if (n == 16) MM_TRY(launch(kron12_kernel<2, true>));
    else if (n == 24) MM_TRY(launch(kron12_kernel<3, true>));
    else if (nb == 2) MM_TRY(launch(kron12_kernel<2, false>));
    else MM_TRY(launch(kron12_kernel<3, false>));
    MM_CUDA(cudaGetLastError());
    h->launches++;
    first = 3;
  } else {
    MM_TRY(mode_product_dev(h, d, m, 1, m[0], V, A[0], 1, m[0], cplx, false, W));
  }
  for (int mu = first; mu <= d; ++mu)
    MM_TRY(mode_product_dev(h, d, m, mu, m[mu - 1], V, A[mu - 1], 1, m[mu - 1], cplx, false, W, true));
  return MUMODE_OK;
}

int mumode_kronsumv_f64(mumode_handle_t h, int d, const int64_t* m, const double* V, const double* const* A,
                        double* W) {
  return kronsumv_entry(h, d, m, V, A, W, false);
}
int mumode_kronsumv_c128(mumode_handle_t h, int d, const int64_t* m, const double* V, const double* const* A,
                         double* W) {
  return kronsumv_entry(h, d, m, V, A, W, true);
}

// ops::itucker (tucker.hpp:187-204): per mode, every mu-fibre solved with the
// stored LU factors of P_mu (lu_solve_mode_kernel). Mode 1 reads T, later
// modes work in place on S (a CTA only touches its own fibres), so T may
// alias S and no workspace is needed.
static int itucker_dev(mumode_handle_t h, int d, const int64_t* m, const double* T, const double* const* LU,
                       const int64_t* const* piv, double* S, bool cplx) {
  const size_t vb = cplx ? 16 : 8;
  constexpr size_t kMaxSmem = 227 * 1024;
  int64_t nsum = 0;
  for (int k = 0; k < d; ++k) nsum += m[k];
  // per-mode row permutations, then one transposed factor (real extents up to kLuRlMaxN: the
  // backward panels of lu_sweep_rl are rows of the factor)
  int64_t nt_max = 0;
  for (int k = 0; k < d; ++k)
    if (!cplx && m[k] <= kLuRlMaxN) nt_max = std::max(nt_max, m[k]);
  const size_t perm_bytes = (size_t(2 * nsum) * sizeof(int) + 255) & ~size_t(255);
  MM_TRY(h->lperm.ensure(perm_bytes + size_t(nt_max * nt_max) * sizeof(double)));
  int* perm = static_cast<int*>(h->lperm.p);
  double* lut_buf = reinterpret_cast<double*>(static_cast<char*>(h->lperm.p) + perm_bytes);
  {  // every mode's permutation in one launch (one block per mode)
    LuPermBatch pb{};
    int64_t off = 0, nsm = 0;
    for (int k = 0; k < d; ++k) {
      if (m[k] > (int64_t(1) << 30)) return fail(MUMODE_ERR_ARGUMENT, "itucker: extent too large");
      pb.piv[k] = piv[k];
      pb.n[k] = static_cast<int>(m[k]);
      pb.off[k] = static_cast<int>(off);
      off += 2 * m[k];
      if (m[k] <= kLuPermSmem) nsm = std::max(nsm, m[k]);
    }
    if (off > (int64_t(1) << 31) - 1) return fail(MUMODE_ERR_ARGUMENT, "itucker: extents too large");
    lu_perm_kernel<<<d, 256, 2 * static_cast<size_t>(nsm) * sizeof(int), h->stream>>>(pb, perm);
    MM_CUDA(cudaGetLastError());
    h->launches++;
  }
  for (int mu = 1; mu <= d; ++mu) {
    const int64_t n = m[mu - 1], A = prod(m, 0, mu - 1), C = prod(m, mu, d);
    if (n > (int64_t(1) << 30)) return fail(MUMODE_ERR_ARGUMENT, "itucker: extent too large");
    const size_t ps = cplx ? LuCfg<true>::PS : LuCfg<false>::PS;
    size_t smem = vb * size_t(n) * (1 + kLuStride + ps);  // invd, fibre tile, factor panel
    int staged = 1;
    const double* src = mu == 1 ? T : S;
    if (smem > kMaxSmem) {
      staged = 0;
      smem = vb * size_t(n);
      if (smem > kMaxSmem)
        return fail(MUMODE_ERR_ARGUMENT, "itucker: extent of mode " + std::to_string(mu) + " is too large");
      if (src == S) {  // the global-memory path gathers from a separate copy
        const size_t bytes = size_t(prod(m, 0, d)) * vb;
        MM_TRY(h->ws[2].ensure(bytes));
        MM_CUDA(cudaMemcpyAsync(h->ws[2].p, S, bytes, cudaMemcpyDeviceToDevice, h->stream));
        src = static_cast<const double*>(h->ws[2].p);
      }
    }
    const int64_t tiles = (A * C + kLuFibres - 1) / kLuFibres;
    const int grid = static_cast<int>(std::min<int64_t>(tiles, int64_t(h->num_sms) * 32));
    if (!cplx && n <= kLuRlMaxN && h->aux_policy != 23) {
      // real extents up to 408: right-looking forward sweep, prefetched panels (lu_sweep_rl)
      const int ni = static_cast<int>(n);
      // 64-fibre tiles (16 warps, one CTA per SM from n = 129) or, up to 208, 96-fibre tiles (24 warps),
      // which take ~1.4x a 64-fibre tile's time: chosen by wave count
      const int64_t sms = h->num_sms, F = A * C;
      const int64_t w64 = ((F + 63) / 64 + sms - 1) / sms, w96 = ((F + 95) / 96 + sms - 1) / sms;
      const bool nf96 = n > 128 && n <= 208 && h->aux_policy != 24 && 14 * w96 < 10 * w64;
      // even extents above 128 with a 16-byte aligned factor: panels by bulk copies (backward ones from
      // a transposed copy of the factor). Measured: 208^3 1.15 -> 1.09 ms, 256^3 2.16 -> 2.06, 300^3
      // 5.41 -> 4.93; no gain with the 96-fibre tiles (their cp.async issue hides under the DMMA phases) or
      // up to 128, where the transpose launch costs more than it saves. Policy 25 forbids the bulk path.
      const double* lut = nullptr;
      if (n > 128 && !nf96 && n % 2 == 0 && reinterpret_cast<uintptr_t>(LU[mu - 1]) % 16 == 0 && h->aux_policy != 25) {
        const unsigned tb = static_cast<unsigned>((n + 31) / 32);
        lu_transpose_kernel<<<dim3(tb, tb), dim3(32, 8), 0, h->stream>>>(LU[mu - 1], lut_buf, ni);
        MM_CUDA(cudaGetLastError());
        h->launches++;
        lut = lut_buf;
      }
      auto launch = [&](auto kern, int nf, int nw) -> int {
        const size_t rsmem = lu_rl_smem(ni, nf);
        MM_TRY(smem_opt_in(kern, static_cast<int>(rsmem)));
        const int64_t tiles = (A * C + nf - 1) / nf;
        const int grid = static_cast<int>(std::min<int64_t>(tiles, int64_t(h->num_sms) * 32));
        kern<<<grid, 32 * nw, rsmem, h->stream>>>(src, S, A, ni, C, LU[mu - 1], lut, perm, perm + n);
        return MUMODE_OK;
      };
      // 64 fibres per CTA while the tile fits in shared memory (n <= 280), else 48 / 32; 32 also when
      // the 32-fibre tiles fit in one wave (few fibres: every tile is one serial chain of steps, so more,
      // smaller tiles finish sooner: 200 x 200 x 10 0.206 -> 0.168 ms)
      if (n > 128 && (F + 31) / 32 <= sms && F > 32 && h->aux_policy != 24) {
        if (lut) MM_TRY(launch(lu_solve_rl_kernel<32, 16, 13, 1, true>, 32, 16));
        else MM_TRY(launch(lu_solve_rl_kernel<32, 16, 13, 1, false>, 32, 16));
      } else if (n <= 64) MM_TRY(launch(lu_solve_rl_kernel<64, 16, 4, 2, false>, 64, 16));
      else if (n <= 128) MM_TRY(launch(lu_solve_rl_kernel<64, 16, 8, 2, false>, 64, 16));
      else if (nf96) MM_TRY(launch(lu_solve_rl_kernel<96, 24, 13, 1, false>, 96, 24));
      else if (n <= 208) {
        if (lut) MM_TRY(launch(lu_solve_rl_kernel<64, 16, 13, 1, true>, 64, 16));
        else MM_TRY(launch(lu_solve_rl_kernel<64, 16, 13, 1, false>, 64, 16));
      } else if (n <= 280) {
        if (lut) MM_TRY(launch(lu_solve_rl_kernel<64, 16, 18, 1, true>, 64, 16));
        else MM_TRY(launch(lu_solve_rl_kernel<64, 16, 18, 1, false>, 64, 16));
      } else if (n <= 328 && h->aux_policy != 24) {  // 48 fibres (12 warps) still fit beside the panels
        if (lut) MM_TRY(launch(lu_solve_rl_kernel<48, 12, 21, 1, true>, 48, 12));
        else MM_TRY(launch(lu_solve_rl_kernel<48, 12, 21, 1, false>, 48, 12));
      } else {
        if (lut) MM_TRY(launch(lu_solve_rl_kernel<32, 16, 13, 1, true>, 32, 16));
        else MM_TRY(launch(lu_solve_rl_kernel<32, 16, 13, 1, false>, 32, 16));
      }
    } else {
      auto kern = cplx ? lu_solve_mode_kernel<true> : lu_solve_mode_kernel<false>;
      const int threads = cplx ? LuCfg<true>::THREADS : LuCfg<false>::THREADS;
      MM_TRY(smem_opt_in(kern, static_cast<int>(smem)));
      kern<<<grid, threads, smem, h->stream>>>(src, S, A, static_cast<int>(n), C, LU[mu - 1], perm, perm + n, staged);
    }
    MM_CUDA(cudaGetLastError());
    h->launches++;
    perm += 2 * n;
  }
  return MUMODE_OK;
}

static int itucker_entry(mumode_handle_t h, int d, const int64_t* m, const double* T, const double* const* LU,
                         const int64_t* const* piv, double* S, bool cplx) {
  if (!h) return fail(MUMODE_ERR_ARGUMENT, "null handle");
  MM_TRY(check_shape(d, m, "itucker"));
  if (!T || !S || !LU || !piv) return fail(MUMODE_ERR_ARGUMENT, "itucker: null pointer");
  for (int k = 0; k < d; ++k)
    if (!LU[k] || !piv[k]) return fail(MUMODE_ERR_ARGUMENT, "itucker: null factor for mode " + std::to_string(k + 1));
  MM_DEVICE(h->device);
  return itucker_dev(h, d, m, T, LU, piv, S, cplx);
}

int mumode_itucker_f64(mumode_handle_t h, int d, const int64_t* m, const double* T, const double* const* LU,
                       const int64_t* const* piv, double* S) {
  return itucker_entry(h, d, m, T, LU, piv, S, false);
}
int mumode_itucker_c128(mumode_handle_t h, int d, const int64_t* m, const double* T, const double* const* LU,
                        const int64_t* const* piv, double* S) {
  return itucker_entry(h, d, m, T, LU, piv, S, true);
}

int mumode_expint_f64(mumode_handle_t h, int d, const int64_t* m, const double* const* E,
                      const double* u0, double* u_out, int steps) {
  if (!h) return fail(MUMODE_ERR_ARGUMENT, "null handle");
  MM_TRY(check_stack(d, m, m, u0, E, u_out, "expint"));
  if (steps < 0) return fail(MUMODE_ERR_ARGUMENT, "expint: steps must be non-negative");
  MM_DEVICE(h->device);
  const int64_t numel = prod(m, 0, d);
  const size_t bytes = size_t(numel) * sizeof(double);
  if (steps == 0) {
    if (u_out != u0) MM_CUDA(cudaMemcpyAsync(u_out, u0, bytes, cudaMemcpyDeviceToDevice, h->stream));
    return MUMODE_OK;
  }
  MM_TRY(h->ws[2].ensure(bytes));
  double* spare = static_cast<double*>(h->ws[2].p);
  // Graph key: shape, pointers, steps.
  std::vector<uint64_t> key{uint64_t(d), uint64_t(steps), reinterpret_cast<uint64_t>(u0),
                            reinterpret_cast<uint64_t>(u_out), uint64_t(h->policy)};
  for (int k = 0; k < d; ++k) {
    key.push_back(uint64_t(m[k]));
    key.push_back(reinterpret_cast<uint64_t>(E[k]));
  }
  auto body = [&]() -> int {
    const double* cur = u0;
    for (int s = 0; s < steps; ++s) {
      // end in u_out; never read and write the same buffer within one step
      double* dst = ((steps - 1 - s) % 2 == 0) ? u_out : spare;
      if (dst == cur) dst = (dst == u_out) ? spare : u_out;
      MM_TRY(tucker_dev(h, d, m, m, cur, E, dst, false, false));
      cur = dst;
    }
    if (cur != u_out)
      MM_CUDA(cudaMemcpyAsync(u_out, cur, bytes, cudaMemcpyDeviceToDevice, h->stream));
    return MUMODE_OK;
  };
  auto it = h->graphs.find(key);
  if (it != h->graphs.end() && it->second.gen != g_workspace_gen.load(std::memory_order_relaxed)) {
    // a workspace the graph was captured on has been reallocated since
    if (it->second.exec) cudaGraphExecDestroy(it->second.exec);
    h->graphs.erase(it);
    it = h->graphs.end();
  }
  if (it == h->graphs.end()) {
    // First call: run eagerly (allocates workspace, encodes TMA maps), then
    // capture the identical launch sequence for later calls.
    MM_TRY(body());
    GraphEntry ge;
    cudaGraph_t graph = nullptr;
    // Capture on the handle's own stream (the legacy stream cannot be
    // captured); nothing executes during capture. Replays go to h->stream.
    cudaStream_t user = h->stream;
    h->stream = h->own_stream;
    if (cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      h->stream = user;
      cudaGetLastError();
      return fail(MUMODE_ERR_CUDA, "graph capture could not begin");
    }
    const int64_t l0 = h->launches;
    int rc = body();
    cudaError_t ce = cudaStreamEndCapture(h->stream, &graph);
    h->stream = user;
    if (rc != MUMODE_OK) return rc;
    if (ce != cudaSuccess) return fail(MUMODE_ERR_CUDA, "graph capture failed");
    ge.nodes = h->launches - l0;
    h->launches = l0;  // captured, not executed
    ge.gen = g_workspace_gen.load(std::memory_order_relaxed);
    MM_CUDA(cudaGraphInstantiate(&ge.exec, graph, 0));
    cudaGraphDestroy(graph);
    h->graphs.emplace(key, ge);
    return MUMODE_OK;
  }
  MM_CUDA(cudaGraphLaunch(it->second.exec, h->stream));
  h->launches += it->second.nodes;
  return MUMODE_OK;
}

// ---------------------------------------------------------------- host drop-in
static int stage_in(mumode_handle_t h, const double* src, size_t bytes, mumode_gpu::DevBuf& buf,
                    size_t offset) {
  MM_CUDA(cudaMemcpyAsync(static_cast<char*>(buf.p) + offset, src, bytes, cudaMemcpyHostToDevice,
                          h->stream));
  return MUMODE_OK;
}

// Upload T and the d matrices (sizes el*Lsz[k] doubles) into staging; returns
// device pointers.
static int upload(mumode_handle_t h, const double* T, size_t t_el, int d, const double* const* L,
                  const int64_t* Lsz, const double** dT, std::vector<const double*>& dL) {
  size_t mat_bytes = 0;
  for (int k = 0; k < d; ++k) mat_bytes += ((size_t(Lsz[k]) * sizeof(double) + 255) / 256) * 256;
  MM_TRY(h->host_in.ensure(t_el * sizeof(double)));
  MM_TRY(h->host_mats.ensure(mat_bytes + 256));
  MM_TRY(stage_in(h, T, t_el * sizeof(double), h->host_in, 0));
  *dT = static_cast<const double*>(h->host_in.p);
  size_t off = 0;
  dL.resize(d);
  for (int k = 0; k < d; ++k) {
    MM_TRY(stage_in(h, L[k], size_t(Lsz[k]) * sizeof(double), h->host_mats, off));
    dL[k] = reinterpret_cast<const double*>(static_cast<char*>(h->host_mats.p) + off);
    off += ((size_t(Lsz[k]) * sizeof(double) + 255) / 256) * 256;
  }
  return MUMODE_OK;
}

static int download(mumode_handle_t h, double* S, size_t el) {
  MM_CUDA(cudaMemcpyAsync(S, h->host_out.p, el * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  MM_CUDA(cudaStreamSynchronize(h->stream));
  return MUMODE_OK;
}

// Pipelined host drop-in for real forward Tucker chains (d >= 2): the input
// streams in as last-mode slabs on a copy stream while modes 1..d-1 run on
// each arrived slab (the slabs of the intermediate are contiguous), then the
// last mode runs in row blocks of L_d whose outputs (contiguous last-mode
// slabs of S) stream back on a second copy stream. H2D and D2H stay serial
// (every output needs all of the input) but the compute hides under them.
static int ensure_pipeline(mumode_handle_t h, size_t nev) {
  if (!h->copy_in) MM_CUDA(cudaStreamCreateWithFlags(&h->copy_in, cudaStreamNonBlocking));
  if (!h->copy_out) MM_CUDA(cudaStreamCreateWithFlags(&h->copy_out, cudaStreamNonBlocking));
  while (h->events.size() < nev) {
    cudaEvent_t e;
    MM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    h->events.push_back(e);
  }
  return MUMODE_OK;
}

// One pipelined host-buffer application, enqueued only: the slot's staging
// buffers (input, factors, output) alternate between consecutive calls, so
// call k+1's upload (copy_in) runs while call k's download (copy_out) drains
// -- PCIe is full duplex. The intermediate is one buffer: the compute stream
// serialises the calls. Per-slot events guard slot reuse on the device; the
// host never waits here.
constexpr int kHostChunks = 8;
constexpr int kSlotEvents = 2 * kHostChunks + 2;  // slabs, blocks, compute end, download end

static int host_tucker_enqueue(mumode_handle_t h, int d, const int64_t* m, const int64_t* n, const double* T,
                               const double* const* L, double* S) {
  constexpr int kChunks = kHostChunks;  // 8: 2.94 ms per queued C2 call; 1, 2, 3, 4: 2.99 ms
  const int slot = static_cast<int>(h->host_calls & 1);
  const bool reuse = h->host_calls >= 2;  // the slot's previous call must be done with it
  ++h->host_calls;
  MM_TRY(ensure_pipeline(h, 2 * kSlotEvents));
  cudaEvent_t* ev = h->events.data() + slot * kSlotEvents;
  cudaEvent_t ev_compute_end = ev[2 * kChunks], ev_d2h_end = ev[2 * kChunks + 1];
  const int64_t md = m[d - 1], nd = n[d - 1];
  const int64_t in_slab = prod(m, 0, d - 1);   // elements per unit of the last input mode
  const int64_t A = prod(n, 0, d - 1);         // rows of the (A x m_d) intermediate
  size_t mat_bytes = 0;
  for (int k = 0; k < d; ++k) mat_bytes += ((size_t(m[k] * n[k]) * sizeof(double) + 255) / 256) * 256;
  // growing a staging buffer frees memory that queued calls may still use
  const size_t in_bytes = size_t(in_slab * md) * sizeof(double), mid_bytes = size_t(A * md) * sizeof(double),
               out_bytes = size_t(A * nd) * sizeof(double);
  if (h->slot_mats[slot].bytes < mat_bytes + 256 || h->slot_in[slot].bytes < in_bytes ||
      h->host_mid.bytes < mid_bytes || h->slot_out[slot].bytes < out_bytes) {
    if (h->copy_in) MM_CUDA(cudaStreamSynchronize(h->copy_in));
    MM_CUDA(cudaStreamSynchronize(h->stream));
    if (h->copy_out) MM_CUDA(cudaStreamSynchronize(h->copy_out));
  }
  MM_TRY(h->slot_mats[slot].ensure(mat_bytes + 256));
  MM_TRY(h->slot_in[slot].ensure(in_bytes));
  MM_TRY(h->host_mid.ensure(mid_bytes));
  MM_TRY(h->slot_out[slot].ensure(out_bytes));
  // the slot's input and factors are free once its previous call's compute ended
  if (reuse) MM_CUDA(cudaStreamWaitEvent(h->copy_in, ev_compute_end, 0));
  std::vector<const double*> dL(d);
  size_t off = 0;
  for (int k = 0; k < d; ++k) {
    const size_t b = size_t(m[k] * n[k]) * sizeof(double);
    MM_CUDA(cudaMemcpyAsync(static_cast<char*>(h->slot_mats[slot].p) + off, L[k], b, cudaMemcpyHostToDevice,
                            h->copy_in));
    dL[k] = reinterpret_cast<const double*>(static_cast<char*>(h->slot_mats[slot].p) + off);
    off += ((b + 255) / 256) * 256;
  }
  double* dT = static_cast<double*>(h->slot_in[slot].p);
  double* dY = static_cast<double*>(h->host_mid.p);
  double* dS = static_cast<double*>(h->slot_out[slot].p);
  // input slabs of the last mode (8-aligned boundaries keep TMA bases 16-B aligned)
  auto bounds = [](int64_t total, int parts, int64_t q, int64_t align) {
    int64_t step = (total + parts - 1) / parts;
    step = (step + align - 1) / align * align;
    return std::min(total, q * step);
  };
  const cudaStream_t cs = h->stream;
  for (int q = 0; q < kChunks; ++q) {
    const int64_t c0 = bounds(md, kChunks, q, 2), c1 = bounds(md, kChunks, q + 1, 2);
    if (c1 <= c0) continue;
    MM_CUDA(cudaMemcpyAsync(dT + c0 * in_slab, T + c0 * in_slab, size_t((c1 - c0) * in_slab) * sizeof(double),
                            cudaMemcpyHostToDevice, h->copy_in));
    MM_CUDA(cudaEventRecord(ev[q], h->copy_in));
  }
  for (int q = 0; q < kChunks; ++q) {
    const int64_t c0 = bounds(md, kChunks, q, 2), c1 = bounds(md, kChunks, q + 1, 2);
    if (c1 <= c0) continue;
    MM_CUDA(cudaStreamWaitEvent(cs, ev[q], 0));
    std::vector<int64_t> ms(m, m + d), ns(n, n + d);
    ms[d - 1] = ns[d - 1] = c1 - c0;
    MM_TRY(tucker_dev(h, d, ms.data(), ns.data(), dT + c0 * in_slab, dL.data(), dY + c0 * A, false, false, 1,
                      d - 1));
  }
  // the slot's output is free once its previous call's download ended
  if (reuse) MM_CUDA(cudaStreamWaitEvent(cs, ev_d2h_end, 0));
  // last mode in row blocks of L_d -> contiguous slabs of S, streamed back
  const int64_t ym[2] = {A, md};
  for (int q = 0; q < kChunks; ++q) {
    const int64_t i0 = bounds(nd, kChunks, q, 8), i1 = bounds(nd, kChunks, q + 1, 8);
    if (i1 <= i0) continue;
    MM_TRY(mode_product_dev(h, 2, ym, 2, i1 - i0, dY, dL[d - 1] + i0, 1, nd, false, false, dS + i0 * A));
    MM_CUDA(cudaEventRecord(ev[kChunks + q], cs));
    MM_CUDA(cudaStreamWaitEvent(h->copy_out, ev[kChunks + q], 0));
    MM_CUDA(cudaMemcpyAsync(S + i0 * A, dS + i0 * A, size_t((i1 - i0) * A) * sizeof(double), cudaMemcpyDeviceToHost,
                            h->copy_out));
  }
  MM_CUDA(cudaEventRecord(ev_compute_end, cs));
  MM_CUDA(cudaEventRecord(ev_d2h_end, h->copy_out));
  return MUMODE_OK;
}

static int host_wait(mumode_handle_t h) {
  if (h->copy_in) MM_CUDA(cudaStreamSynchronize(h->copy_in));
  MM_CUDA(cudaStreamSynchronize(h->stream));
  if (h->copy_out) MM_CUDA(cudaStreamSynchronize(h->copy_out));
  return MUMODE_OK;
}

static bool host_pipelinable(int d, const int64_t* m, const int64_t* n, int adjoint, int t_el, int l_el) {
  return d >= 2 && !adjoint && t_el == 1 && l_el == 1 && m[d - 1] >= 16 && n[d - 1] >= 16 &&
         prod(m, 0, d) >= (int64_t(1) << 20);
}

static int host_tucker_impl(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                            const double* T, const double* const* L, double* S, int adjoint,
                            int t_el, int l_el) {
  if (!h) return fail(MUMODE_ERR_ARGUMENT, "null handle");
  MM_TRY(check_stack(d, m, n, T, L, S, adjoint ? "cttucker" : "tucker"));
  MM_DEVICE(h->device);
  if (host_pipelinable(d, m, n, adjoint, t_el, l_el)) {
    MM_TRY(host_tucker_enqueue(h, d, m, n, T, L, S));
    return host_wait(h);
  }
  std::vector<int64_t> lsz(d);
  for (int k = 0; k < d; ++k) lsz[k] = m[k] * n[k] * l_el;
  const double* dT;
  std::vector<const double*> dL;
  MM_TRY(upload(h, T, size_t(prod(m, 0, d)) * t_el, d, L, lsz.data(), &dT, dL));
  const size_t out_el = size_t(prod(n, 0, d)) * l_el;
  MM_TRY(h->host_out.ensure(out_el * sizeof(double)));
  double* dS = static_cast<double*>(h->host_out.p);
  if (t_el == 1 && l_el == 2)
    MM_TRY(mumode_tucker_promote(h, d, m, n, dT, dL.data(), dS, adjoint));
  else
    MM_TRY(tucker_dev(h, d, m, n, dT, dL.data(), dS, adjoint != 0, l_el == 2));
  return download(h, S, out_el);
}

int mumode_host_tucker_f64(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                           const double* T, const double* const* L, double* S, int adjoint) {
  return host_tucker_impl(h, d, m, n, T, L, S, adjoint, 1, 1);
}
int mumode_host_tucker_f64_async(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                                 const double* T, const double* const* L, double* S) {
  if (!h) return fail(MUMODE_ERR_ARGUMENT, "null handle");
  MM_TRY(check_stack(d, m, n, T, L, S, "tucker"));
  MM_DEVICE(h->device);
  if (!host_pipelinable(d, m, n, 0, 1, 1)) return host_tucker_impl(h, d, m, n, T, L, S, 0, 1, 1);
  return host_tucker_enqueue(h, d, m, n, T, L, S);
}

int mumode_host_wait(mumode_handle_t h) {
  if (!h) return fail(MUMODE_ERR_ARGUMENT, "null handle");
  MM_DEVICE(h->device);
  return host_wait(h);
}

int mumode_host_tucker_c128(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                            const double* T, const double* const* L, double* S, int adjoint) {
  return host_tucker_impl(h, d, m, n, T, L, S, adjoint, 2, 2);
}
int mumode_host_tucker_promote(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                               const double* T, const double* const* L, double* S, int adjoint) {
  return host_tucker_impl(h, d, m, n, T, L, S, adjoint, 1, 2);
}

static int host_mode_product_impl(mumode_handle_t h, int d, const int64_t* m, int mu,
                                  int64_t n_mu, const double* T, const double* L, double* S,
                                  int el) {
  if (!h) return fail(MUMODE_ERR_ARGUMENT, "null handle");
  MM_TRY(check_shape(d, m, "mode_product"));
  if (mu < 1 || mu > d)
    return fail(MUMODE_ERR_ARGUMENT, "mode index " + std::to_string(mu) + " out of range 1.." +
                                         std::to_string(d));
  if (!T || !L || !S) return fail(MUMODE_ERR_ARGUMENT, "mode_product: null pointer");
  MM_DEVICE(h->device);
  int64_t lsz = n_mu * m[mu - 1] * el;
  const double* dT;
  std::vector<const double*> dL;
  MM_TRY(upload(h, T, size_t(prod(m, 0, d)) * el, 1, &L, &lsz, &dT, dL));
  std::vector<int64_t> out(m, m + d);
  out[mu - 1] = n_mu;
  const size_t out_el = size_t(prod(out.data(), 0, d)) * el;
  MM_TRY(h->host_out.ensure(out_el * sizeof(double)));
  MM_TRY(mode_product_dev(h, d, m, mu, n_mu, dT, dL[0], 1, n_mu, el == 2, false,
                          static_cast<double*>(h->host_out.p)));
  return download(h, S, out_el);
}

int mumode_host_mode_product_f64(mumode_handle_t h, int d, const int64_t* m, int mu,
                                 int64_t n_mu, const double* T, const double* L, double* S) {
  return host_mode_product_impl(h, d, m, mu, n_mu, T, L, S, 1);
}
int mumode_host_mode_product_c128(mumode_handle_t h, int d, const int64_t* m, int mu,
                                  int64_t n_mu, const double* T, const double* L, double* S) {
  return host_mode_product_impl(h, d, m, mu, n_mu, T, L, S, 2);
}

static int host_kronsumv_impl(mumode_handle_t h, int d, const int64_t* m, const double* V, const double* const* A,
                              double* W, bool cplx) {
  if (!h) return fail(MUMODE_ERR_ARGUMENT, "null handle");
  MM_TRY(check_stack(d, m, m, V, A, W, "kronsumv"));
  MM_DEVICE(h->device);
  const int el = cplx ? 2 : 1;
  std::vector<int64_t> lsz(d);
  for (int k = 0; k < d; ++k) lsz[k] = m[k] * m[k] * el;
  const double* dV;
  std::vector<const double*> dA;
  const size_t numel = size_t(prod(m, 0, d)) * el;
  MM_TRY(upload(h, V, numel, d, A, lsz.data(), &dV, dA));
  MM_TRY(h->host_out.ensure(numel * sizeof(double)));
  MM_TRY(kronsumv_entry(h, d, m, dV, dA.data(), static_cast<double*>(h->host_out.p), cplx));
  return download(h, W, numel);
}

int mumode_host_kronsumv_f64(mumode_handle_t h, int d, const int64_t* m, const double* V, const double* const* A,
                             double* W) {
  return host_kronsumv_impl(h, d, m, V, A, W, false);
}
int mumode_host_kronsumv_c128(mumode_handle_t h, int d, const int64_t* m, const double* V, const double* const* A,
                              double* W) {
  return host_kronsumv_impl(h, d, m, V, A, W, true);
}

static int host_itucker_impl(mumode_handle_t h, int d, const int64_t* m, const double* T, const double* const* LU,
                             const int64_t* const* piv, double* S, bool cplx) {
  if (!h) return fail(MUMODE_ERR_ARGUMENT, "null handle");
  MM_TRY(check_shape(d, m, "itucker"));
  if (!T || !S || !LU || !piv) return fail(MUMODE_ERR_ARGUMENT, "itucker: null pointer");
  for (int k = 0; k < d; ++k)
    if (!LU[k] || !piv[k]) return fail(MUMODE_ERR_ARGUMENT, "itucker: null factor for mode " + std::to_string(k + 1));
  MM_DEVICE(h->device);
  const int el = cplx ? 2 : 1;
  // factors then pivots (int64 = one double slot each) through the staging upload
  std::vector<const double*> src(2 * d);
  std::vector<int64_t> lsz(2 * d);
  for (int k = 0; k < d; ++k) {
    src[k] = LU[k];
    lsz[k] = m[k] * m[k] * el;
    src[d + k] = reinterpret_cast<const double*>(piv[k]);
    lsz[d + k] = m[k];
  }
  const double* dT;
  std::vector<const double*> dL;
  const size_t numel = size_t(prod(m, 0, d)) * el;
  MM_TRY(upload(h, T, numel, 2 * d, src.data(), lsz.data(), &dT, dL));
  std::vector<const int64_t*> dpiv(d);
  for (int k = 0; k < d; ++k) dpiv[k] = reinterpret_cast<const int64_t*>(dL[d + k]);
  MM_TRY(h->host_out.ensure(numel * sizeof(double)));
  MM_TRY(itucker_dev(h, d, m, dT, dL.data(), dpiv.data(), static_cast<double*>(h->host_out.p), cplx));
  return download(h, S, numel);
}

int mumode_host_itucker_f64(mumode_handle_t h, int d, const int64_t* m, const double* T, const double* const* LU,
                            const int64_t* const* piv, double* S) {
  return host_itucker_impl(h, d, m, T, LU, piv, S, false);
}
int mumode_host_itucker_c128(mumode_handle_t h, int d, const int64_t* m, const double* T, const double* const* LU,
                             const int64_t* const* piv, double* S) {
  return host_itucker_impl(h, d, m, T, LU, piv, S, true);
}

int mumode_host_expint_f64(mumode_handle_t h, int d, const int64_t* m, const double* const* E,
                           const double* u0, double* u_out, int steps) {
  if (!h) return fail(MUMODE_ERR_ARGUMENT, "null handle");
  MM_TRY(check_stack(d, m, m, u0, E, u_out, "expint"));
  MM_DEVICE(h->device);
  std::vector<int64_t> lsz(d);
  for (int k = 0; k < d; ++k) lsz[k] = m[k] * m[k];
  const double* du;
  std::vector<const double*> dE;
  const size_t el = size_t(prod(m, 0, d));
  MM_TRY(upload(h, u0, el, d, E, lsz.data(), &du, dE));
  MM_TRY(h->host_out.ensure(el * sizeof(double)));
  MM_TRY(mumode_expint_f64(h, d, m, dE.data(), du, static_cast<double*>(h->host_out.p), steps));
  return download(h, u_out, el);
}

}  // extern "C"

#include "slab_dist.cuh"
