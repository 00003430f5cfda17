// fp64_latency.cu — dependent-issue latency of DFMA / DADD / DMUL and of an LDS -> DADD -> STS hop
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_latency.bin fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(int mode, int n, double x, double y, double* out, long long* clk) {
  __shared__ double buf[64];
  buf[threadIdx.x & 63] = x;
  __syncthreads();
  double a = x;
  const long long t0 = clock64();
  if (mode == 0) for (int i = 0; i < n; ++i) a = fma(a, y, x);
  if (mode == 1) for (int i = 0; i < n; ++i) a = a + y;
  if (mode == 2) for (int i = 0; i < n; ++i) a = a * y;
  if (mode == 3) for (int i = 0; i < n; ++i) { a = buf[(threadIdx.x + i) & 63] + a; }                // LDS feeding a chain
  if (mode == 4) for (int i = 0; i < n; ++i) { volatile double* b = buf; b[threadIdx.x & 63] = a; a = b[threadIdx.x & 63] + y; }  // STS -> LDS -> DADD hop
  if (mode == 5) for (int i = 0; i < n; ++i) a = a + __shfl_xor_sync(0xffffffffu, a, 1 << (i % 5));  // SHFL (64-bit) -> DADD hop
  const long long t1 = clock64();
  if (threadIdx.x == 0) { out[blockIdx.x] = a; clk[blockIdx.x] = t1 - t0; }
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 8 * 148); cudaMalloc(&c, 8 * 148);
  const char* names[] = {"DFMA chain", "DADD chain", "DMUL chain", "LDS + DADD (load independent of the chain)", "STS -> LDS -> DADD hop", "SHFL.64 -> DADD hop"};
  for (int mode = 0; mode < 6; ++mode)
    for (int warps : {1, 8}) {
      const int n = 4096;
      lat<<<1, 32 * warps>>>(mode, n, 1.0000001, 0.9999999, d, c);
      lat<<<1, 32 * warps>>>(mode, n, 1.0000001, 0.9999999, d, c);
      cudaDeviceSynchronize();
      long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("%-44s warps %d: %6.1f clk per step\n", names[mode], warps, (double)h / n);
    }
  return 0;
}
