// tmem_scratch.cu — can tensor memory serve as thread-private scratch for a non-MMA kernel?
// Measures, on one CTA per SM: (1) dependent latency of tcgen05.ld 32x32b.x1, (2) read throughput
// of tcgen05.ld 32x32b.x32 at 1/4/8 warps, (3) write throughput of tcgen05.st, (4) whether TMEM
// reads overlap shared-memory reads (LDS.128 stream alone, LDTM alone, both interleaved).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tmem_scratch.bin tmem_scratch.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t tmem_alloc_all(uint32_t* slot) {
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"((uint32_t)__cvta_generic_to_shared(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  return *slot;
}
__device__ __forceinline__ void tmem_free_all(uint32_t base) {
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(base));
}

#define LD32(v, addr)                                                                                     \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 "                                                  \
               "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,"   \
               "%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"                                               \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),       \
                 "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),   \
                 "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),             \
                 "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),             \
                 "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])              \
               : "r"(addr))
#define ST32(v, addr)                                                                                     \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%32], "                                           \
               "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,"   \
               "%24,%25,%26,%27,%28,%29,%30,%31};\n" ::"r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]),          \
               "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]),   \
               "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),         \
               "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]),         \
               "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]), "r"(addr))
#define WAIT_LD() asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory")
#define WAIT_ST() asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory")

// mode 0: dependent x1 loads (latency); 1: x32 read stream; 2: x32 write stream;
// 3: LDS.128 stream; 4: x32 reads + LDS.128 interleaved; 5: x32 read stream, two loads in flight
__global__ void __launch_bounds__(256, 1) probe(int mode, int iters, long long* clk_out, uint32_t* sink) {
  __shared__ uint32_t slot;
  __shared__ __align__(16) uint4 buf[1024];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_uint4(i, 1, 2, 3);
  const uint32_t base = tmem_alloc_all(&slot);
  // lanes 32*(warp%4).., columns: warps 0-3 use 0..255, warps 4-7 use 256..511
  const uint32_t mine = base + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 256);
  uint32_t v[32], w[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = (threadIdx.x * 32 + i) & 63, w[i] = 0;  // small values: valid column offsets
  for (int c = 0; c < 256; c += 32) ST32(v, mine + c);
  WAIT_ST();
  __syncthreads();
  uint32_t acc = 0;
  const long long t0 = clock64();
  if (mode == 0) {
    uint32_t col = 0;
    for (int it = 0; it < iters; ++it) {
      uint32_t r;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(r) : "r"(mine + col));
      WAIT_LD();
      col = __shfl_sync(0xffffffffu, r, 0) & 63;  // warp-uniform next column
      acc += r;
    }
  } else if (mode == 1) {
    for (int it = 0; it < iters; ++it) {
      LD32(v, mine + (it & 7) * 32);
      WAIT_LD();
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += v[i];
    }
  } else if (mode == 5) {
    for (int it = 0; it < iters; it += 2) {
      LD32(v, mine + (it & 7) * 32);
      LD32(w, mine + ((it + 1) & 7) * 32);
      WAIT_LD();
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += v[i] ^ w[i];
    }
  } else if (mode == 2) {
    for (int it = 0; it < iters; ++it) {
      v[0] = it;
      ST32(v, mine + (it & 7) * 32);
    }
    WAIT_ST();
  } else if (mode == 3) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {  // 8 x LDS.128 = 32 words per thread, conflict-free
        const uint4 t = buf[(threadIdx.x + 131 * q + it) & 1023];
        acc += t.x ^ t.y ^ t.z ^ t.w;
      }
    }
  } else if (mode == 4) {
    for (int it = 0; it < iters; ++it) {
      LD32(v, mine + (it & 7) * 32);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint4 t = buf[(threadIdx.x + 131 * q + it) & 1023];
        acc += t.x ^ t.y ^ t.z ^ t.w;
      }
      WAIT_LD();
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += v[i];
    }
  }
  const long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) clk_out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tmem_free_all(base);
}

int main() {
  long long* d_clk;
  uint32_t* d_sink;
  CK(cudaMalloc(&d_clk, 148 * sizeof(long long)));
  CK(cudaMalloc(&d_sink, 148 * 256 * sizeof(uint32_t)));
  const char* names[] = {"LDTM x1 dependent (latency)", "LDTM x32 stream, wait each", "STTM x32 stream",
                         "LDS.128 x8 stream", "LDTM x32 + LDS.128 x8 interleaved", "LDTM x32 stream, two in flight"};
  const int iters = 4096;
  for (int mode = 0; mode < 6; ++mode) {
    for (int warps : {1, 4, 8}) {
      probe<<<148, warps * 32, 0>>>(mode, iters, d_clk, d_sink);  // warm
      probe<<<148, warps * 32, 0>>>(mode, iters, d_clk, d_sink);
      CK(cudaDeviceSynchronize());
      long long h[148];
      CK(cudaMemcpy(h, d_clk, sizeof(h), cudaMemcpyDeviceToHost));
      double mean = 0;
      for (int i = 0; i < 148; ++i) mean += (double)h[i] / 148;
      const double per_it = mean / iters;  // clocks per load round (mode 5: two rounds per loop pass)
      const double bytes = mode == 0 ? 0.0 : (mode == 4 ? 2.0 : 1.0) * warps * 32 * 32 * 4;  // per load round per SM
      printf("%-36s warps %d: %8.1f clk/round", names[mode], warps, per_it);
      if (bytes > 0) printf("  %7.1f B/clk/SM", bytes / per_it);
      printf("\n");
    }
  }
  return 0;
}
