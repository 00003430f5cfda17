// Probe: where do the two CTAs of a cluster land when two CTAs fit one SM?
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cluster_placement cluster_placement.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(128, 2) probe(int* smid, long long* t0, long long* t1, int spin) {
  extern __shared__ double sm[];
  unsigned id;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
  long long a;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a));
  double v = threadIdx.x;
  for (int i = 0; i < spin; ++i) {
    v = v * 1.0000001 + 1e-9;
    if ((i & 255) == 0) cg::this_cluster().sync();
  }
  sm[threadIdx.x] = v;
  long long b;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(b));
  if (threadIdx.x == 0) {
    smid[blockIdx.x] = (int)id;
    t0[blockIdx.x] = a;
    t1[blockIdx.x] = b + (sm[5] == 1234.5 ? 1 : 0);
  }
}

int main() {
  const int ctas = 148 * 4;
  int* smid; long long *t0, *t1;
  cudaMallocManaged(&smid, ctas * sizeof(int));
  cudaMallocManaged(&t0, ctas * sizeof(long long));
  cudaMallocManaged(&t1, ctas * sizeof(long long));
  const int smem = 90752;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 2; attr.val.clusterDim.y = 1; attr.val.clusterDim.z = 1;
  cfg.attrs = &attr; cfg.numAttrs = 1;
  int ncl = -1;
  cudaOccupancyMaxActiveClusters(&ncl, probe, &cfg);
  printf("max active clusters: %d\n", ncl);
  cudaError_t e = cudaLaunchKernelEx(&cfg, probe, smid, t0, t1, 200000);
  e = e == cudaSuccess ? cudaDeviceSynchronize() : e;
  printf("launch: %s\n", cudaGetErrorString(e));
  int same = 0;
  for (int c = 0; c < ctas; c += 2) same += smid[c] == smid[c + 1];
  printf("cluster pairs on the same SM: %d of %d\n", same, ctas / 2);
  long long base = t0[0];
  for (int c = 0; c < ctas; ++c) base = t0[c] < base ? t0[c] : base;
  // concurrency: how many CTAs started within the first 10 us
  int early = 0; for (int c = 0; c < ctas; ++c) early += (t0[c] - base) < 10000;
  printf("CTAs started in the first 10 us: %d (148 SMs)\n", early);
  std::vector<int> per(148, 0);
  for (int c = 0; c < ctas; ++c) if ((t0[c] - base) < 10000) per[smid[c] % 148]++;
  int h[5] = {0}; for (int s = 0; s < 148; ++s) h[per[s] > 4 ? 4 : per[s]]++;
  printf("SMs with 0/1/2/3/4+ early CTAs: %d %d %d %d %d\n", h[0], h[1], h[2], h[3], h[4]);
  for (int c = 0; c < 8; ++c) printf("cta %d sm %d start %lld end %lld\n", c, smid[c], t0[c] - base, t1[c] - base);
  return 0;
}
