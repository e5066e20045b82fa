// Read-only TMA bandwidth probe for the fused C5 passes (24^6 fp64 tensor,
// 1.53 GB): a persistent kernel whose producer thread streams boxes into an
// NBUF-deep shared-memory ring and whose consumer warp only waits and
// releases. No math, so the measured rate is the access pattern's ceiling.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_pattern_probe \
//        tools/tma_pattern_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) { asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(b)), "r"(n)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t tx) { asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx)); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(b))); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(su32(b)), "r"(ph));
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
               ::"r"(su32(dst)), "l"(m), "r"(su32(bar)), "r"(x), "r"(y), "r"(z) : "memory");
}
__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y, int z, int w) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
               ::"r"(su32(dst)), "l"(m), "r"(su32(bar)), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}

struct Job {
  int kind;       // 0: 3D view, box {RA, by, bz}, per tile zsteps boxes along z. 1: 4D pass-2 view
  int RA, by, bz, zsteps;
  int ntiles;     // a tiles (3D) or a-tiles * C (4D)
  int atiles;
  int blocked;    // 1: CTA i walks a contiguous run of tiles
  uint32_t box_bytes;
  int nbuf;
};

__global__ void __launch_bounds__(64) probe_kernel(const __grid_constant__ CUtensorMap map, const Job j, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[8], empty[8];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < j.nbuf; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 32); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int per = (j.ntiles + gridDim.x - 1) / gridDim.x;
  auto tile_of = [&](int i) { return j.blocked ? blockIdx.x * per + i : blockIdx.x + i * gridDim.x; };
  const int my = j.blocked ? max(0, min(per, j.ntiles - int(blockIdx.x) * per))
                           : (j.ntiles - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x);
  const int loads = my * j.zsteps;
  if (tid == 0) {
    for (int l = 0; l < loads; ++l) {
      const int s = l % j.nbuf;
      if (l >= j.nbuf) mbar_wait(&empty[s], ((l / j.nbuf) - 1) & 1);
      const int t = tile_of(l / j.zsteps), z = l % j.zsteps;
      mbar_expect(&full[s], j.box_bytes);
      if (j.kind == 4) {
        tma4(smem + s * j.box_bytes, &map, &full[s], 0, t * (32 / j.by), 0, z * j.bz);
      } else if (j.kind == 3) {
        for (int q = 0; q < j.RA / 8; ++q)
          tma3(smem + s * j.box_bytes + q * (j.box_bytes / (j.RA / 8)), &map, &full[s], t * j.RA + 8 * q, 0, z * j.bz);
      } else if (j.kind == 0) tma3(smem + s * j.box_bytes, &map, &full[s], t * j.RA, 0, z * j.bz);
      else if (j.kind == 2) tma3(smem + s * j.box_bytes, &map, &full[s], 0, 12 * (t % 12), 2 * (t / 12));
      else tma4(smem + s * j.box_bytes, &map, &full[s], (t % j.atiles) * j.RA, 0, 0, t / j.atiles);
    }
  } else if (tid >= 32) {
    unsigned long long acc = 0;
    for (int l = 0; l < loads; ++l) {
      const int s = l % j.nbuf;
      mbar_wait(&full[s], (l / j.nbuf) & 1);
      acc += reinterpret_cast<const unsigned long long*>(smem + s * j.box_bytes)[tid - 32];
      __syncwarp();
      mbar_arrive(&empty[s]);
    }
    if (acc == 0x123456789ull) *sink = acc;
  }
}

// Store pattern of the last fused pass: output S(a, i, j) over (331776, 24, 24);
// one warp store = 8 j-rows (lanes g) x 64 B (4 lanes x 16 B). RA a's per tile,
// the RA/8 a-blocks of one (i, j-block) stored back to back.
template <int RA>
__global__ void __launch_bounds__(256) store_kernel(double* S) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int64_t A = 331776, tiles = A / RA;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x)
    for (int u = warp; u < 24 * 3; u += 8) {   // (i, jblk)
      const int i = u / 3, jb = u % 3;
      for (int ab = 0; ab < RA / 8; ++ab) {
        double* p = S + tile * RA + 8 * ab + 2 * t + A * (i + 24 * (8 * jb + g));
        asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(1.0), "d"(2.0) : "memory");
      }
    }
}

// RW-byte contiguous runs per row, 512/RW rows per warp instruction (16 B per lane)
template <int RW>
__global__ void __launch_bounds__(256) store_rows_kernel(double* S) {
  constexpr int LPR = RW / 16, RPI = 32 / LPR;  // lanes per row, rows per instruction
  constexpr int RA = RW / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t A = 331776, tiles = A / RA;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x)
    for (int rr = warp * RPI; rr < 576; rr += 8 * RPI) {
      const int row = rr + lane / LPR;
      double* p = S + tile * RA + 2 * (lane % LPR) + A * row;
      asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(1.0), "d"(2.0) : "memory");
    }
}

// TMA store of box {16, 2, 1, 24} (one i, all j; 256-B rows) per issue, from a
// fixed smem buffer; 4 bulk groups in flight.
__global__ void __launch_bounds__(32) tma_store_kernel(const __grid_constant__ CUtensorMap map) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (threadIdx.x != 0) return;
  const int tiles = 331776 / 32;
  int n = 0;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x)
    for (int i = 0; i < 24; ++i) {
      asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
                   ::"l"(&map), "r"(0), "r"(tile * 2), "r"(i), "r"(0), "r"(su32(smem + (n & 3) * 6144)) : "memory");
      asm volatile("cp.async.bulk.commit_group;");
      asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
      ++n;
    }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q));
  const uint64_t N = 191102976ull;  // 24^6
  double* buf;
  CK(cudaMalloc(&buf, N * 8));
  CK(cudaMemset(buf, 0, N * 8));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  void* flush;
  CK(cudaMalloc(&flush, 512 << 20));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);

  struct Case { const char* name; int kind, RA, by, bz, zsteps, blocked, nbuf, ctas_per_sm; };
  std::vector<Case> cases = {
      {"pass3 box{8,24,24}   interleaved", 0, 8, 24, 24, 1, 0, 4, 1},
      {"pass3 box{16,24,24}  interleaved", 0, 16, 24, 24, 1, 0, 2, 1},
      {"pass3 box{32,24,12}x2 interleaved", 0, 32, 24, 12, 2, 0, 2, 1},
      {"pass3 box{8,24,4}x6  interleaved", 0, 8, 24, 4, 6, 0, 8, 1},
      {"pass3 box{16,24,4}x6 interleaved", 0, 16, 24, 4, 6, 0, 8, 1},
      {"pass3 box{32,24,4}x6 interleaved", 0, 32, 24, 4, 6, 0, 8, 1},
      {"pass3 box{64,24,4}x6 interleaved", 0, 64, 24, 4, 6, 0, 6, 1},
      {"pass3 box{8,24,24}   blocked", 0, 8, 24, 24, 1, 1, 4, 1},
      {"pass3 box{32,24,4}x6 blocked", 0, 32, 24, 4, 6, 1, 8, 1},
      {"pass3 box{8,24,24}   2 CTA/SM", 0, 8, 24, 24, 1, 0, 2, 2},
      {"pass3 4x box{8,24,4} per stage (RA 32)", 3, 32, 24, 4, 6, 0, 8, 1},
      {"pass3 4x box{8,24,2} per stage (RA 32)", 3, 32, 24, 2, 12, 0, 8, 1},
      {"pass3 2x box{8,24,4} per stage (RA 16)", 3, 16, 24, 4, 6, 0, 8, 1},
      {"pass3 4D box{16,2,24,4} sw128", 4, 32, 16, 4, 6, 0, 8, 1},
      {"pass3 4D box{8,4,24,4} sw64", 4, 32, 8, 4, 6, 0, 8, 1},
      {"pass3 4D box{16,2,24,2} sw128", 4, 32, 16, 2, 12, 0, 8, 1},
      {"pass2 box{8,24,24,1}", 1, 8, 24, 24, 1, 0, 4, 1},
      {"pass2 box{16,24,24,1}", 1, 16, 24, 24, 1, 0, 2, 1},
      {"contiguous box{256,12,2}", 2, 256, 12, 2, 1, 0, 4, 1},
  };
  for (const Case& c : cases) {
    CUtensorMap map;
    Job j{};
    j.RA = c.RA; j.by = c.by; j.bz = c.bz; j.zsteps = c.zsteps; j.blocked = c.blocked; j.nbuf = c.nbuf;
    j.box_bytes = uint32_t(c.RA) * c.by * c.bz * 8;
    CUresult r;
    if (c.kind == 0 || c.kind == 3) {
      cuuint64_t gd[3] = {331776, 24, 24}, gs[2] = {331776 * 8ull, 331776 * 24 * 8ull};
      cuuint32_t bd[3] = {uint32_t(c.kind == 3 ? 8 : c.RA), uint32_t(c.by), uint32_t(c.bz)}, es[3] = {1, 1, 1};
      r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, buf, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      j.kind = c.kind; j.ntiles = 331776 / c.RA;
    } else if (c.kind == 4) {
      const uint32_t X = uint32_t(c.by);  // inner a run (8 or 16)
      cuuint64_t gd[4] = {X, 331776 / X, 24, 24}, gs[3] = {X * 8ull, 331776 * 8ull, 331776 * 24 * 8ull};
      cuuint32_t bd[4] = {X, 32 / X, 24, uint32_t(c.bz)}, es[4] = {1, 1, 1, 1};
      r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, buf, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              X == 16 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      j.kind = 4; j.by = int(X); j.ntiles = 331776 / 32; j.box_bytes = 32 * 24 * c.bz * 8;
    } else if (c.kind == 1) {
      cuuint64_t gd[4] = {576, 24, 24, 576}, gs[3] = {576 * 8ull, 576 * 24 * 8ull, 576 * 576 * 8ull};
      cuuint32_t bd[4] = {uint32_t(c.RA), 24, 24, 1}, es[4] = {1, 1, 1, 1};
      r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, buf, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      j.kind = 1; j.atiles = 576 / c.RA; j.ntiles = j.atiles * 576;
    } else {
      // contiguous reference: view as (256, 144, 5184), box {256, 12, 2} = 48 KB contiguous
      cuuint64_t gd[3] = {256, 144, 5184}, gs[2] = {256 * 8ull, 36864 * 8ull};
      cuuint32_t bd[3] = {256, 12, 2}, es[3] = {1, 1, 1};
      r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, buf, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      j.kind = 2; j.ntiles = 12 * 2592; j.zsteps = 1; j.box_bytes = 256 * 12 * 2 * 8;
    }
    if (r != CUDA_SUCCESS) { printf("%-40s encode failed %d\n", c.name, int(r)); continue; }
    const int grid = sms * c.ctas_per_sm;
    const size_t smem = size_t(j.box_bytes) * j.nbuf;
    if (smem > 200 * 1024) { printf("%-40s smem too big\n", c.name); continue; }
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemsetAsync(flush, rep, 512 << 20);
      cudaEventRecord(e0);
      probe_kernel<<<grid, 64, smem>>>(map, j, sink);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double bytes = double(j.box_bytes) * j.ntiles * j.zsteps;
    printf("%-40s %8.1f us  %7.0f GB/s  (%.2f GB)\n", c.name, best * 1e3, bytes / (best * 1e-3) / 1e9, bytes / 1e9);
  }
  auto time_store = [&](const char* name, void (*k)(double*)) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemsetAsync(flush, rep, 512 << 20);
      cudaEventRecord(e0);
      k<<<sms * 4, 256>>>(buf);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("%-40s %8.1f us  %7.0f GB/s\n", name, best * 1e3, N * 8.0 / (best * 1e-3) / 1e9);
  };
  time_store("store pass3 RA 8", store_kernel<8>);
  time_store("store pass3 RA 16", store_kernel<16>);
  time_store("store pass3 RA 32", store_kernel<32>);
  time_store("store rows 64B x8 per instr", store_rows_kernel<64>);
  time_store("store rows 128B x4 per instr", store_rows_kernel<128>);
  time_store("store rows 256B x2 per instr", store_rows_kernel<256>);
  time_store("store rows 512B x1 per instr", store_rows_kernel<512>);
  {
    CUtensorMap map;
    cuuint64_t gd[4] = {16, 331776 / 16, 24, 24}, gs[3] = {128ull, 331776 * 8ull, 331776 * 24 * 8ull};
    cuuint32_t bd[4] = {16, 2, 1, 24}, es[4] = {1, 1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, buf, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("store map failed %d\n", int(r));
    CK(cudaFuncSetAttribute(tma_store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 6144));
    for (int per_sm : {1, 2, 4}) {
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemsetAsync(flush, rep, 512 << 20);
        cudaEventRecord(e0);
        tma_store_kernel<<<sms * per_sm, 32, 4 * 6144>>>(map);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("TMA store box{16,2,1,24} %d CTA/SM       %8.1f us  %7.0f GB/s\n", per_sm, best * 1e3, N * 8.0 / (best * 1e-3) / 1e9);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
