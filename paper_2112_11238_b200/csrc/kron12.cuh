// kronsumv's first two terms in ONE pass (ops::kronsumv, tucker.hpp:209-232):
//   W(:, :, c) = A1 V_c + V_c A2^T   for every slice c of the modes beyond 2,
// for small square modes 1 and 2 (even n from 10 to 24). One pass per term reads V
// twice and reads W once more than needed (24^6: 7.7 GB for the two terms
// against 3.1 GB here); the per-mode passes are at the HBM rate, so the bytes
// are the time.
//
// Both terms are computed TRANSPOSED so that their DMMA result fragments line
// up and the contiguous index i pairs up in one lane:
//   t1'(j, i) = sum_k V(k, j) A1(i, k)    A operand: V_c columns,  B operand: A1
//   t2'(j, i) = sum_k A2(j, k) V(i, k)    A operand: A2,           B operand: V_c rows
// lane (g, t) holds (j = 8 fj + g, i = 8 fi + 2t, 2t + 1) of both, adds them
// once (the reference's acc = term1; acc += term2) and stores 16 bytes. Every
// chain runs k = 0..n-1 in steps of 4 from a zero accumulator, as in the
// per-mode kernels, so the pass is bitwise equal to them (policy 26 runs the
// per-mode passes; test_kronsumv_fused_first_pair_equals_per_mode_passes).
//
// One slice per warp per iteration: the slice (n x n doubles, contiguous) is
// copied by 16-byte cp.async into a padded buffer (column pitch n + 4: both
// fragment patterns conflict-free), three buffers per warp (two slices in
// flight); A2's fragments stay in registers, A1 sits in shared memory.
#pragma once

namespace mumode_gpu {

constexpr int kKron12Warps = 12;
constexpr int kKron12Bufs = 3;

__device__ __forceinline__ void kron_cp_async16(double* dst, const double* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

template <int NB, bool FULL>  // FULL: n = 8 NB exactly (compile-time bounds)
__global__ void __launch_bounds__(32 * kKron12Warps, 1) kron12_kernel(const double* __restrict__ V,
                                                                       const double* __restrict__ A1,
                                                                       const double* __restrict__ A2,
                                                                       double* __restrict__ W, int64_t nslices,
                                                                       int n_arg) {
  // n <= N = 8 NB, n even: the buffers' rows and columns n..N-1 and the factor fragments beyond n are
  // zero, so every chain is the k-ordered chain over the true k's plus exact zero steps
  constexpr int N = 8 * NB, KS = N / 4, PS = N + 4, SL = N * PS;
  const int n = FULL ? N : n_arg, HALF = n / 2;
  extern __shared__ __align__(16) double kron_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double* buf = kron_smem + SL + warp * kKron12Bufs * SL;
  // A2's fragments (A operand of t2') in registers, A1 (B operand of t1') in shared memory with the
  // slices' column pitch: twelve warps fit the register file that way
  double* sA1 = kron_smem;
  if constexpr (!FULL) {  // the padding rows / columns are read as zeros (FULL: every element read is loaded)
    for (int e = threadIdx.x; e < (1 + kKron12Warps * kKron12Bufs) * SL; e += blockDim.x) kron_smem[e] = 0.0;
    __syncthreads();
  }
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) sA1[(e / n) * PS + (e % n)] = A1[e];
  double a2f[NB][KS];
#pragma unroll
  for (int f = 0; f < NB; ++f)
#pragma unroll
    for (int s = 0; s < KS; ++s)
      a2f[f][s] = (8 * f + g < n && 4 * s + t < n) ? A2[(8 * f + g) + n * (4 * s + t)] : 0.0;
  __syncthreads();
  const int64_t stride = int64_t(gridDim.x) * kKron12Warps;
  auto issue = [&](int64_t c, double* dst) {
    const double* src = V + c * (int64_t(n) * n);
    for (int q = lane; q < n * HALF; q += 32) {
      const int r = q / HALF, cp = q - r * HALF;
      kron_cp_async16(dst + r * PS + 2 * cp, src + 2 * q);
    }
  };
  int64_t c = int64_t(blockIdx.x) * kKron12Warps + warp;
  // prologue: two slices in flight (an empty group keeps the wait counts uniform)
  if (c < nslices) issue(c, buf);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  if (c + stride < nslices) issue(c + stride, buf + SL);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  int b = 0;
  for (; c < nslices; c += stride) {
    // the buffer two ahead was read in the previous iteration (all lanes passed the __syncwarp below)
    int b2 = b + 2;
    if (b2 >= kKron12Bufs) b2 -= kKron12Bufs;
    if (c + 2 * stride < nslices) issue(c + 2 * stride, buf + b2 * SL);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 2;\n" ::: "memory");
    __syncwarp();
    const double* v = buf + b * SL;
    double d1[NB][NB][2], d2[NB][NB][2];
#pragma unroll
    for (int fj = 0; fj < NB; ++fj)
#pragma unroll
      for (int fi = 0; fi < NB; ++fi) d1[fj][fi][0] = d1[fj][fi][1] = d2[fj][fi][0] = d2[fj][fi][1] = 0.0;
#pragma unroll
    for (int s = 0; s < KS; ++s) {
      double va[NB], vb[NB], a1[NB];
#pragma unroll
      for (int f = 0; f < NB; ++f) {
        va[f] = v[(8 * f + g) * PS + 4 * s + t];  // V(k, j): column j at j * PS
        vb[f] = v[(4 * s + t) * PS + 8 * f + g];  // V(i, k)
        a1[f] = sA1[(4 * s + t) * PS + 8 * f + g];  // A1(i, k)
      }
#pragma unroll
      for (int fj = 0; fj < NB; ++fj)
#pragma unroll
        for (int fi = 0; fi < NB; ++fi) {
          dmma_8x8x4(d1[fj][fi][0], d1[fj][fi][1], va[fj], a1[fi]);
          dmma_8x8x4(d2[fj][fi][0], d2[fj][fi][1], a2f[fj][s], vb[fi]);
        }
    }
    __syncwarp();  // every lane has read the slice: its buffer may be refilled
    double* w = W + c * (int64_t(n) * n);
#pragma unroll
    for (int fj = 0; fj < NB; ++fj)
#pragma unroll
      for (int fi = 0; fi < NB; ++fi)
        if (8 * fj + g < n && 8 * fi + 2 * t < n)
          stg_f64x2(w + (8 * fj + g) * n + 8 * fi + 2 * t, d1[fj][fi][0] + d2[fj][fi][0],
                    d1[fj][fi][1] + d2[fj][fi][1]);
    if (++b == kKron12Bufs) b = 0;
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

inline size_t kron12_smem(int nb) {  // nb = ceil(n / 8)
  return sizeof(double) * (size_t(kKron12Warps) * kKron12Bufs + 1) * size_t(8 * nb) * (8 * nb + 4);
}

}  // namespace mumode_gpu
