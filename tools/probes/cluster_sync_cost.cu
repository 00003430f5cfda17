// Probe: cost per iteration of different 2-CTA cluster synchronisation schemes (cycles).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned remote(unsigned local, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}

template <int kMode>
__global__ void __launch_bounds__(256, 1) probe(long long* out, int iters, int nstores) {
  __shared__ double buf[512];
  __shared__ unsigned long long bar[2];
  const unsigned rank = cg::this_cluster().block_rank();
  const int tid = threadIdx.x;
  buf[tid] = 0.0;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(&bar[0])), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(&bar[1])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  cg::this_cluster().sync();
  double* rbuf = cg::this_cluster().map_shared_rank(buf, rank ^ 1);
  const unsigned rbar = remote(saddr(&bar[0]), rank ^ 1);
  long long t0 = clock64();
  double v = tid;
  for (int i = 0; i < iters; ++i) {
    if (kMode == 5) {
      if (tid < nstores)
        asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(
                         remote(saddr(&buf[256 + tid]), rank ^ 1)),
                     "d"(v), "r"(remote(saddr(&bar[1]), rank ^ 1))
                     : "memory");
    } else if (tid < nstores) rbuf[256 + tid] = v;  // boundary values pushed to the partner
    if (kMode == 0) {
      cg::this_cluster().sync();
    } else if (kMode == 1) {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    } else if (kMode == 2) {
      __syncthreads();
    } else if (kMode == 3) {
      // local barrier, then one thread signals the partner's mbarrier (release.cluster) and
      // every thread waits on the local one
      __syncthreads();
      if (tid == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
      unsigned ok;
      do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok) : "r"(saddr(&bar[0])), "r"((unsigned)(i & 1)) : "memory");
      } while (!ok);
    } else if (kMode == 4) {
      // as 3, but only the pushing warp waits for the partner; the rest meets it at a local barrier
      __syncthreads();
      if (tid == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
      if (tid < 32) {
        unsigned ok;
        do {
          asm volatile(
              "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
              : "=r"(ok) : "r"(saddr(&bar[0])), "r"((unsigned)(i & 1)) : "memory");
        } while (!ok);
      }
      __syncthreads();
    } else if (kMode == 5) {
      // no cluster barrier at all: the pushes themselves are asynchronous stores that complete
      // transaction bytes on the partner's mbarrier; the consumer arms it and waits (one warp)
      __syncthreads();
      if (tid == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&bar[1])), "r"(nstores * 8) : "memory");
      if (tid < 32) {
        unsigned ok;
        do {
          asm volatile(
              "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
              : "=r"(ok) : "r"(saddr(&bar[1])), "r"((unsigned)(i & 1)) : "memory");
        } while (!ok);
      }
      __syncthreads();
    }
    v += buf[256 + (tid & 31)];
  }
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  buf[tid] = v;
  cg::this_cluster().sync();
}

template <int kMode>
void run(const char* name, int nstores) {
  long long* out;
  cudaMallocManaged(&out, 2 * sizeof(long long));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2); cfg.blockDim = dim3(256);
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 2; attr.val.clusterDim.y = 1; attr.val.clusterDim.z = 1;
  cfg.attrs = &attr; cfg.numAttrs = 1;
  const int iters = 20000;
  cudaLaunchKernelEx(&cfg, probe<kMode>, out, iters, nstores);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%-44s stores=%2d  %8.1f clk/iter  (%s)\n", name, nstores, (double)out[0] / iters, cudaGetErrorString(e));
  cudaFree(out);
}

int main() {
  for (int ns : {0, 32}) {
    run<2>("__syncthreads only (no cross-CTA order)", ns);
    run<0>("cg cluster.sync (arrive.release+wait.acquire)", ns);
    run<1>("barrier.cluster arrive.relaxed + wait", ns);
    run<3>("syncthreads + remote mbarrier arrive, all wait", ns);
    run<4>("syncthreads + remote mbarrier, 1 warp waits", ns);
    if (ns > 0) run<5>("st.async complete_tx pushes, 1 warp waits", ns);
  }
  return 0;
}
