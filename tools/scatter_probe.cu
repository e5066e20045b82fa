// Bandwidth probe for the access patterns of a two-pass (three modes per pass)
// small-extent Tucker: a CTA owns one n^3 cube c of a d = 6 tensor (NC cubes
// of E = n^3 elements) and writes it, or reads it, as E/R pieces of R
// consecutive doubles spread NC*R elements apart ("transposed blocked"
// layout Z[p][c][r]); concurrently running CTAs own consecutive cubes, so
// together they cover whole L2 lines. Compared with contiguous streams.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/scatter_probe tools/scatter_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

template <int R, bool WRITE>
__global__ void __launch_bounds__(512) scatter_kernel(double* __restrict__ z, long NC, int E, double* sink) {
  const int pieces = E / R;
  double acc = 0;
  for (long c = blockIdx.x; c < NC; c += gridDim.x) {
    for (int p = threadIdx.x; p < pieces; p += blockDim.x) {
      double* q = z + ((long)p * NC + c) * R;
      if (WRITE) {
#pragma unroll
        for (int r = 0; r < R; r += 2) *reinterpret_cast<double2*>(q + r) = make_double2(c + p, r);
      } else {
#pragma unroll
        for (int r = 0; r < R; r += 2) { double2 v = *reinterpret_cast<const double2*>(q + r); acc += v.x + v.y; }
      }
    }
  }
  if (!WRITE && acc == 12345.678) sink[0] = acc;
}

template <bool WRITE>
__global__ void __launch_bounds__(512) contig_kernel(double* __restrict__ z, long n, double* sink) {
  double acc = 0;
  for (long i = (blockIdx.x * (long)blockDim.x + threadIdx.x) * 2; i < n; i += (long)gridDim.x * blockDim.x * 2) {
    if (WRITE) *reinterpret_cast<double2*>(z + i) = make_double2(i, 1);
    else { double2 v = *reinterpret_cast<const double2*>(z + i); acc += v.x + v.y; }
  }
  if (!WRITE && acc == 12345.678) sink[0] = acc;
}

static double* g_flush;
static void flush() { cudaMemset(g_flush, 0, 256u << 20); }

template <class F>
static float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e30f;
  for (int it = 0; it < 6; ++it) {
    flush();
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (it > 0 && ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  CK(cudaMalloc(&g_flush, 256u << 20));
  double* sink; CK(cudaMalloc(&sink, 64));
  const int ns[] = {12, 14, 16, 18, 20, 24};
  for (int n : ns) {
    const long E = (long)n * n * n, NC = E, N = E * NC;
    double* z; CK(cudaMalloc(&z, N * 8));
    const double gb = N * 8.0 / 1e9;
    auto rep = [&](const char* what, float ms) { printf("n=%2d %-22s %8.1f us  %7.0f GB/s\n", n, what, ms * 1e3, gb / (ms * 1e-3)); };
    rep("contig write", timeit([&] { contig_kernel<true><<<sms * 4, 512>>>(z, N, sink); }));
    rep("contig read", timeit([&] { contig_kernel<false><<<sms * 4, 512>>>(z, N, sink); }));
    for (int g : {1, 2, 4}) {
      char buf[64];
      if (E % 2 == 0) {
        snprintf(buf, 64, "scatter W R=2 %dCTA/SM", g); rep(buf, timeit([&] { scatter_kernel<2, true><<<sms * g, 512>>>(z, NC, (int)E, sink); }));
        snprintf(buf, 64, "scatter R R=2 %dCTA/SM", g); rep(buf, timeit([&] { scatter_kernel<2, false><<<sms * g, 512>>>(z, NC, (int)E, sink); }));
      }
      if (E % 4 == 0) {
        snprintf(buf, 64, "scatter W R=4 %dCTA/SM", g); rep(buf, timeit([&] { scatter_kernel<4, true><<<sms * g, 512>>>(z, NC, (int)E, sink); }));
        snprintf(buf, 64, "scatter R R=4 %dCTA/SM", g); rep(buf, timeit([&] { scatter_kernel<4, false><<<sms * g, 512>>>(z, NC, (int)E, sink); }));
      }
      if (E % 8 == 0) {
        snprintf(buf, 64, "scatter W R=8 %dCTA/SM", g); rep(buf, timeit([&] { scatter_kernel<8, true><<<sms * g, 512>>>(z, NC, (int)E, sink); }));
        snprintf(buf, 64, "scatter R R=8 %dCTA/SM", g); rep(buf, timeit([&] { scatter_kernel<8, false><<<sms * g, 512>>>(z, NC, (int)E, sink); }));
      }
    }
    CK(cudaGetLastError());
    cudaFree(z);
  }
  return 0;
}
