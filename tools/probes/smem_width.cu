// smem_width.cu — shared-memory bytes per clock per SM by access width and pattern (one CTA of 8
// warps per SM, 8 independent loads per thread per iteration).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_width.bin smem_width.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <class T> __device__ __forceinline__ uint32_t fold(const T& t);
template <> __device__ __forceinline__ uint32_t fold<uint32_t>(const uint32_t& t) { return t; }
template <> __device__ __forceinline__ uint32_t fold<uint2>(const uint2& t) { return t.x ^ t.y; }
template <> __device__ __forceinline__ uint32_t fold<uint4>(const uint4& t) { return t.x ^ t.y ^ t.z ^ t.w; }

// pattern 0: lane-contiguous; 1: element stride 3 (conflict-free, scattered over 3x the span);
// 2: groups of 5 lanes read the same element (broadcast, like the node vectors);
// 3: element index 175*(lane/5) + 3*(lane%5)  (the partial-sum read pattern, in units of T);
// 4: the whole warp reads one element; 5: each quarter warp reads one element
template <class T>
__global__ void __launch_bounds__(256, 1) probe(int pattern, int iters, long long* clk_out, uint32_t* sink) {
  extern __shared__ __align__(16) unsigned char raw[];
  T* buf = reinterpret_cast<T*>(raw);
  constexpr int kElems = 64 * 1024 / sizeof(T);  // power of two
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(raw)[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int idx;
  if (pattern == 0) idx = threadIdx.x;
  else if (pattern == 1) idx = 3 * threadIdx.x;
  else if (pattern == 2) idx = threadIdx.x / 5;
  else if (pattern == 3) idx = 175 * (threadIdx.x / 5) + 3 * (threadIdx.x % 5);
  else if (pattern == 4) idx = warp;          // one address per warp
  else if (pattern == 5) idx = threadIdx.x / 8;  // one address per quarter warp
  else if (pattern == 6) idx = threadIdx.x / 4;  // two addresses per quarter warp
  else idx = 2 * (threadIdx.x / 8) + ((threadIdx.x & 7) >= 5);  // five lanes + three lanes per quarter warp
  (void)lane; (void)warp;
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += fold(buf[(idx + 35 * q + it) & (kElems - 1)]);
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) clk_out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <class T>
void run(const char* name, long long* d_clk, uint32_t* d_sink) {
  cudaFuncSetAttribute(probe<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const char* pats[] = {"contiguous", "stride 3", "broadcast x5", "partial-sum pattern", "one address per warp", "one address per 8 lanes", "two addresses per 8 lanes (4+4)", "two addresses per 8 lanes (5+3)"};
  for (int p = 0; p < 8; ++p) {
    const int iters = 4096;
    probe<T><<<148, 256, 64 * 1024>>>(p, iters, d_clk, d_sink);
    probe<T><<<148, 256, 64 * 1024>>>(p, iters, d_clk, d_sink);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d_clk, sizeof(h), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < 148; ++i) mean += (double)h[i] / 148;
    const double per = mean / iters / 64.0;  // clocks per warp-level load instruction
    printf("%-8s %-20s %6.2f clk per warp load  %7.1f requested B/clk/SM\n", name, pats[p], per, 32.0 * sizeof(T) / per);
  }
}

int main() {
  long long* d_clk;
  uint32_t* d_sink;
  cudaMalloc(&d_clk, 148 * sizeof(long long));
  cudaMalloc(&d_sink, 148 * 256 * sizeof(uint32_t));
  run<uint32_t>("LDS.32", d_clk, d_sink);
  run<uint2>("LDS.64", d_clk, d_sink);
  run<uint4>("LDS.128", d_clk, d_sink);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
