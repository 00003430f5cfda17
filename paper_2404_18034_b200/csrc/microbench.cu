// microbench.cu — FP64 FMA peak microbenchmark (roofline denominator for the solver kernels).
#include "kernels.cuh"

namespace ptopt_b200 {

namespace {

constexpr int kChains = 8;     // independent accumulators per thread
constexpr int kInner = 64;     // DFMAs per chain per outer iteration

__global__ void fp64_peak_kernel(double* sink, int iters) {
  double acc[kChains];
  const double a = 1.0000001, b = 1e-9 * (threadIdx.x + 1);
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = 1.0 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < kInner; ++r) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], a, b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 123.456) sink[0] = s;  // keeps the loop alive without a store in practice
}

}  // namespace

void launch_fp64_peak(double* sink, int iters, int ctas, int threads, cudaStream_t stream) {
  fp64_peak_kernel<<<ctas, threads, 0, stream>>>(sink, iters);
}

double fp64_peak_flops(int iters, int ctas, int threads) {
  return 2.0 * kChains * kInner * (double)iters * (double)ctas * (double)threads;
}

}  // namespace ptopt_b200
