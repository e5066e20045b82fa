// FP64 peak microbenchmark for B200 (sm_100a): DFMA pipe vs DMMA (mma.sync f64).
// The roofline denominator for the mu-mode product kernels is the FP64 peak,
// which MEASURED_PEAKS.json does not carry; this measures it on the box.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
//   ./fp64_peak            -> one JSON line per variant
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::printf("cuda error %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int kChains = 8;

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 1.2345) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void dmma_kernel(double* out, int iters, double a0, double b0) {
  double acc[NACC][2];
#pragma unroll
  for (int c = 0; c < NACC; ++c) { acc[c][0] = c; acc[c][1] = threadIdx.x; }
  double a = a0 + threadIdx.x * 1e-9, b = b0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < NACC; ++c)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < NACC; ++c) s += acc[c][0] + acc[c][1];
  if (s == 1.2345) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// DMMA fed from shared memory at the mode-product kernel's ratio: per k-step
// 12 conflict-free LDS.64 (8 B-frags + 4 A-frags) and 32 DMMAs (64x32 warp
// tile), 8 warps per CTA, 1 CTA per SM. Tells whether ~92 % of the DMMA pipe
// is a ceiling of the mma.sync + LDS instruction mix itself.
__global__ void __launch_bounds__(256) dmma_lds_kernel(double* out, int iters) {
  __shared__ double sm[8][512];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 8 * 512; i += blockDim.x) (&sm[0][0])[i] = 1e-3 * (i & 63);
  __syncthreads();
  double acc[8][4][2];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const double* base = &sm[warp][0];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      double pf[8], qf[4];
      const int off = (s * 96 + lane + (it & 1) * 64) & 511;
#pragma unroll
      for (int a = 0; a < 8; ++a) pf[a] = base[(off + 32 * a) & 511];
#pragma unroll
      for (int b = 0; b < 4; ++b) qf[b] = base[(off + 32 * (8 + b)) & 511];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
              : "+d"(acc[a][b][0]), "+d"(acc[a][b][1]) : "d"(qf[b]), "d"(pf[a]));
    }
  }
  double s = 0;
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) s += acc[a][b][0] + acc[a][b][1];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <class F>
float time_it(F f, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; CK(cudaMalloc(&out, 1 << 24));
  const int threads = 256;
  for (int bps : {2, 4, 8}) {
    const int blocks = sms * bps, iters = 4096;
    float ms = time_it([&] { dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-3); }, 5);
    double flops = 2.0 * blocks * threads * double(iters) * 16 * kChains;
    std::printf("{\"variant\": \"dfma\", \"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n",
                bps, ms, flops / ms / 1e9);
  }
  for (int bps : {1, 2, 4, 8}) {
    const int blocks = sms * bps, iters = 2048;
    float ms = time_it([&] { dmma_kernel<4><<<blocks, threads>>>(out, iters, 0.999, 1e-3); }, 5);
    double flops = 2.0 * 256 * (threads / 32) * double(blocks) * iters * 4 * 4;
    std::printf("{\"variant\": \"dmma_m8n8k4_acc4\", \"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n",
                bps, ms, flops / ms / 1e9);
    ms = time_it([&] { dmma_kernel<8><<<blocks, threads>>>(out, iters, 0.999, 1e-3); }, 5);
    flops = 2.0 * 256 * (threads / 32) * double(blocks) * iters * 4 * 8;
    std::printf("{\"variant\": \"dmma_m8n8k4_acc8\", \"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n",
                bps, ms, flops / ms / 1e9);
  }
  // one warp per SMSP (128-thread CTA, 1 CTA/SM): can a single warp keep the
  // DMMA pipe busy with enough independent accumulators?
  for (int acc : {4, 8, 16}) {
    const int blocks = sms, iters = 4096, thr = 128;
    float ms;
    if (acc == 4) ms = time_it([&] { dmma_kernel<4><<<blocks, thr>>>(out, iters, 0.999, 1e-3); }, 5);
    else if (acc == 8) ms = time_it([&] { dmma_kernel<8><<<blocks, thr>>>(out, iters, 0.999, 1e-3); }, 5);
    else ms = time_it([&] { dmma_kernel<16><<<blocks, thr>>>(out, iters, 0.999, 1e-3); }, 5);
    double flops = 2.0 * 256 * (thr / 32) * double(blocks) * iters * 4 * acc;
    std::printf("{\"variant\": \"dmma_1warp_per_smsp_acc%d\", \"ms\": %.3f, \"tflops\": %.3f}\n", acc, ms,
                flops / ms / 1e9);
  }
  {
    const int blocks = sms, iters = 2048;
    float ms = time_it([&] { dmma_lds_kernel<<<blocks, 256>>>(out, iters); }, 5);
    double flops = 2.0 * 256 * 8 * double(blocks) * iters * 4 * 32;
    std::printf("{\"variant\": \"dmma_with_lds_gemm_mix\", \"ms\": %.3f, \"tflops\": %.3f}\n", ms,
                flops / ms / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
