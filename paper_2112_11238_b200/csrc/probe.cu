// FP64 tensor-pipe peak probe: the roofline denominator for the mu-mode
// kernels. MEASURED_PEAKS.json carries no fp64 figure, so bench.py measures it
// live on the same GPU and clocks as the kernels it reports. Independent
// DMMA.8x8x4 chains, 8 warps per CTA, grid = 2 CTAs per SM.
#include <cuda_runtime.h>

#include <string>

#include "../../include/mumode_gpu.h"
#include "common.cuh"

namespace mumode_gpu {
void set_error(const std::string& msg);

template <int NACC>
__global__ void __launch_bounds__(256) dmma_peak_kernel(double* sink, int iters, double a0) {
  double acc[NACC][2];
#pragma unroll
  for (int c = 0; c < NACC; ++c) acc[c][0] = acc[c][1] = c;
  const double a = a0 + threadIdx.x * 1e-9, b = 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < NACC; ++c) dmma_8x8x4(acc[c][0], acc[c][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < NACC; ++c) s += acc[c][0] + acc[c][1];
  if (s == 1.2345) sink[threadIdx.x] = s;  // never true; keeps the chains live
}
}  // namespace mumode_gpu

struct mumode_handle_s;
extern "C" void* mumode_get_stream(mumode_handle_t h);

extern "C" int mumode_probe_fp64_peak(mumode_handle_t h, double* tflops) {
  using namespace mumode_gpu;
  if (!h || !tflops) return MUMODE_ERR_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(mumode_get_stream(h));
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* sink = nullptr;
  if (cudaMalloc(&sink, 4096) != cudaSuccess) return MUMODE_ERR_OOM;
  const int blocks = 2 * sms, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(e0, s);
    dmma_peak_kernel<8><<<blocks, threads, 0, s>>>(sink, iters, 0.999);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0 && ms < best) best = ms;  // first launch is the warm-up
  }
  cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (err != cudaSuccess) {
    set_error(std::string("probe: ") + cudaGetErrorString(err));
    return MUMODE_ERR_CUDA;
  }
  const double flops = 2.0 * 256.0 * (threads / 32) * double(blocks) * iters * 4 * 8;
  *tflops = flops / (best * 1e-3) / 1e12;
  return MUMODE_OK;
}
