// FP64 vector (DFMA) peak vs the DMMA tensor-pipe peak on this GPU, and both
// together: can SIMT FMAs take the padded remainder of small-extent products?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dfma_probe tools/dfma_probe.cu
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MODE>  // 0: DFMA only, 1: DMMA only, 2: both interleaved (1 DMMA : 8 DFMA)
__global__ void __launch_bounds__(256) probe(double* sink, int iters, double a0) {
  double f[16], d[8][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = i * 1e-3;
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = i;
  const double a = a0 + threadIdx.x * 1e-9, b = 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (MODE != 1)
#pragma unroll
        for (int i = 0; i < 16; ++i) f[i] = fma(f[i], a, b);
      if (MODE != 0)
#pragma unroll
        for (int i = 0; i < (MODE == 2 ? 2 : 8); ++i) dmma(d[i][0], d[i][1], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += f[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  if (s == 1.2345) sink[threadIdx.x] = s;
}

template <int MODE>
static void run(int sms, double* sink) {
  const int blocks = 2 * sms, threads = 256, iters = 2048;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    probe<MODE><<<blocks, threads>>>(sink, iters, 0.999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0 && ms < best) best = ms;
  }
  const double warps = double(blocks) * threads / 32;
  const double dfma = MODE != 1 ? warps * 32 * iters * 4 * 16 * 2.0 : 0;  // flops
  const double dmmaf = MODE != 0 ? warps * iters * 4 * (MODE == 2 ? 2 : 8) * 512.0 : 0;
  printf("mode %d: %.3f ms  DFMA %.2f TF/s  DMMA %.2f TF/s  total %.2f TF/s\n", MODE, best, dfma / best / 1e9,
         dmmaf / best / 1e9, (dfma + dmmaf) / best / 1e9);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink;
  cudaMalloc(&sink, 4096 * 8);
  run<0>(sms, sink);
  run<1>(sms, sink);
  run<2>(sms, sink);
  return 0;
}
