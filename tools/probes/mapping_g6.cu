// mapping_g6.cu — one power-iteration trip (same operator, seed and arithmetic as the control of
// trip_ablation.cu / mapping_t3.cu) in a 2-D ownership mapping: SIX threads per node = 3 row groups
// (5 operator rows each) x 2 column halves (ch 0: the 15 columns of A-, ch 1: the 7 + 7 columns of
// B- | B+ and one zero column).  75 operator doubles per thread, 10 warps for 50 nodes (5 nodes per
// warp, lanes 15 and 31 idle), <= 200 registers.
//   * forward product: each thread multiplies its 5 x 15 block with its half of the node vector
//     (15 LDS.64, pitch-15 layout: conflict-free) and the two halves are added with ONE xor-16
//     shuffle per row;
//   * transposed product: 15 partial column sums over the thread's 5 rows, reduce-scattered over the
//     3 row-group lanes with two register-static shuffle rounds (the column groups of a thread are
//     rotated by its row group, so round s always sends register set s): no partial sums in
//     shared memory at all;
//   * only what crosses a node boundary goes through shared memory (phi_{k-1}, B+^T phi_{k-1},
//     x_{k+1}, u_{k+1}).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xptxas -v -o mapping_g6.bin mapping_g6.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#ifndef KN
#define KN 50
#endif
constexpr int kN = KN, kM = kN - 1;
constexpr int kNX = 15, kNU = 7;
constexpr int kWarps = 10, kThreads = 32 * kWarps;
constexpr int kP = 15;  // pitch of every per-node array (3 groups of 5)

__host__ __device__ inline double op_entry(int inst, int k, int i, int j) {
  uint64_t h = (uint64_t)inst * 0x9E3779B97F4A7C15ull + (uint64_t)(k * 435 + i * 29 + j) * 0xBF58476D1CE4E5B9ull;
  h ^= h >> 31; h *= 0x94D049BB133111EBull; h ^= h >> 29;
  return ((double)(h >> 11) * (1.0 / 9007199254740992.0) - 0.5) * (i == j ? 2.0 : 0.3);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// node arrays: index -1 (zero guard) .. kN + 1 (scratch for the idle lanes)
constexpr int kNodes = kN + 3;
struct Lay {
  static constexpr int xin = kP;                      // x_k            [node][15]
  static constexpr int uin = xin + kNodes * kP;       // [u_k | u_{k+1} | 0]   [node][15]
  static constexpr int php = uin + kNodes * kP;       // phi_k          [node][15]
  static constexpr int csp = php + kNodes * kP;       // column sums of the ch-1 lanes [node][15]
  static constexpr int red = csp + kNodes * kP;
  static constexpr int opx = red + 32;                 // thread-private operator overflow: entry e at opx[e * kThreads + tid]
  static constexpr int total = opx;
};

template <int ABL, int CS = 0>
__global__ void __launch_bounds__(kThreads, 1) trips_g6(int iters, double* sigma_out, long long* clk_out) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ch = lane >> 4, l16 = lane & 15;
  const int p = l16 / 3, rg = l16 - 3 * p;
  const bool idle = p == 5;
  const int k = idle ? kN + 1 : 5 * warp + p;  // idle lanes: scratch node
  const bool node = !idle && k < kN, ival = !idle && k < kM;
  const int gid = blockIdx.x;
  for (int e = tid; e < Lay::total + 5 * CS * kThreads; e += kThreads) sm[e] = 0.0;
  __syncthreads();
  // CS > 0: the last CS column slots of group 2 live in thread-private shared memory, not in registers
  double* opx = sm + Lay::opx + tid;
  auto in_smem = [](int g, int i) { return g == 2 && i >= 5 - CS; };
  auto opx_at = [&](int r, int i) -> double& { return opx[(5 * (i - (5 - CS)) + r) * kThreads]; };
  // operator block: rows 5rg..5rg+4, column slot (g, i) <-> column 5 * ((rg + g) % 3) + i of this half
  double a[5][3][5];
#pragma unroll
  for (int r = 0; r < 5; ++r)
#pragma unroll
    for (int g = 0; g < 3; ++g)
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        const int c = 5 * ((rg + g) % 3) + i;  // 0..14 inside the half
        double v = 0.0;
        if (ival && (ch == 0 || c < 14)) v = op_entry(gid, k, 5 * rg + r, ch == 0 ? c : 15 + c);
        if (in_smem(g, i)) { opx_at(r, i) = v; v = 0.0; }
        a[r][g][i] = v;
      }
  // per-thread addresses
  const double* in_k = sm + (ch ? Lay::uin : Lay::xin) + k * kP;
  int goff[3];
#pragma unroll
  for (int g = 0; g < 3; ++g) goff[g] = 5 * ((rg + g) % 3);
  const double* xnext = sm + Lay::xin + (k + 1) * kP + 5 * rg;
  double* pub = sm + (ch ? Lay::csp : Lay::php) + k * kP + 5 * rg;
  const double* nbp = sm + (ch ? Lay::csp : Lay::php) + (k - 1) * kP;
  int nboff[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) nboff[i] = ch ? min(5 * rg + 7 + i, 14) : 5 * rg + i;
  const double sgn = ch ? 1.0 : -1.0;
  // primal entries owned: ch 0: x_k[5rg + i]; ch 1: u_k[c], c = 5rg + i < 7
  int nvalid = !node ? 0 : (ch == 0 ? 5 : (rg == 0 ? 5 : (rg == 1 ? 2 : 0)));
  double* stA = ch ? sm + Lay::uin + k * kP + 5 * rg : sm + Lay::xin + k * kP + 5 * rg;
  double* stB = sm + Lay::uin + (k - 1) * kP + 5 * rg + 7;  // the same u entries as "u_{k+1}" of interval k-1
  const bool dup = ch == 1 && nvalid > 0;
  const int prev_lane = rg > 0 ? lane - 1 : lane + 2, next_lane = rg < 2 ? lane + 1 : lane - 2;
  double* red = sm + Lay::red;
  // seed: x, u = 1
  if (node) {
#pragma unroll
    for (int i = 0; i < 5; ++i)
      if (i < nvalid) {
        stA[i] = 1.0;
        if (dup) stB[i] = 1.0;
      }
  }
  __syncthreads();
  double sigma = 1.0;
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const double inv = 1.0 / sigma;
    // ---- forward product
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int g = 0; g < 3; ++g) {
      double v[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) v[i] = (ABL & 16) ? 1.0 : in_k[goff[g] + i];
#pragma unroll
      for (int r = 0; r < 5; ++r)
#pragma unroll
        for (int i = 0; i < 5; ++i) acc[r] = fma(in_smem(g, i) ? opx_at(r, i) : a[r][g][i], v[i], acc[r]);
    }
    double ph[5];
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      double t = acc[r];
      if (!(ABL & 32)) t -= (ch == 0 ? xnext[r] : 0.0);
      const double o = (ABL & 1) ? t : __shfl_xor_sync(0xffffffffu, t, 16);
      ph[r] = ival ? (t + o) * inv : 0.0;
    }
    // ---- transposed product, reduce-scatter over the row groups
    double cs[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      double q0 = a[0][0][i] * ph[0], q1 = a[0][1][i] * ph[0], q2 = (in_smem(2, i) ? opx_at(0, i) : a[0][2][i]) * ph[0];
#pragma unroll
      for (int r = 1; r < 5; ++r) {
        q0 = fma(a[r][0][i], ph[r], q0);
        q1 = fma(a[r][1][i], ph[r], q1);
        q2 = fma(in_smem(2, i) ? opx_at(r, i) : a[r][2][i], ph[r], q2);
      }
      const double r1 = (ABL & 2) ? q1 : __shfl_sync(0xffffffffu, q1, prev_lane);
      const double r2 = (ABL & 2) ? q2 : __shfl_sync(0xffffffffu, q2, next_lane);
      cs[i] = (q0 + r1) + r2;
    }
    // ---- publish what the neighbour node needs: phi_k (ch 0) / the column sums of B+ (ch 1)
    if (!(ABL & 4)) {
#pragma unroll
      for (int i = 0; i < 5; ++i) pub[i] = ch ? cs[i] : ph[i];
    }
    if (!(ABL & 512)) __syncthreads();
    // ---- owner sums
    double nrm = 0.0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const double nb = (ABL & 8) ? 0.25 : nbp[nboff[i]];
      const double nv = fma(sgn, nb, cs[i]);
      if (i < nvalid) {
        stA[i] = nv;
        if (dup) stB[i] = nv;
        nrm = fma(nv, nv, nrm);
      }
    }
    if (ch == 0 && node) {
#pragma unroll
      for (int r = 0; r < 5; ++r) nrm = fma(2.0 * ph[r], ph[r], nrm);
    }
    nrm = warp_sum(nrm);
    if (lane == 0) red[warp] = nrm;
    if (!(ABL & 1024)) __syncthreads();
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) tot += red[w];
    sigma = sqrt(tot);
  }
  const long long t1 = clock64();
  if (tid == 0) {
    sigma_out[gid] = sigma;
    clk_out[gid] = t1 - t0;
  }
}

template <int ABL, int CS = 0>
void run(const char* name, int iters, double* d_sigma, long long* d_clk, double* ref) {
  const size_t smem = (size_t)(Lay::total + 5 * CS * kThreads) * sizeof(double);
  auto kern = trips_g6<ABL, CS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = 148;
  kern<<<grid, kThreads, smem>>>(iters, d_sigma, d_clk);
  kern<<<grid, kThreads, smem>>>(iters, d_sigma, d_clk);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  static double hs[148];
  static long long hc[148];
  cudaMemcpy(hs, d_sigma, sizeof(double) * grid, cudaMemcpyDeviceToHost);
  cudaMemcpy(hc, d_clk, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
  double mean = 0, worst = 0;
  for (int i = 0; i < grid; ++i) mean += (double)hc[i] / grid;
  if (ref[0] == 0.0) for (int i = 0; i < 148; ++i) ref[i] = hs[i];
  for (int i = 0; i < 148; ++i) { const double d = fabs(hs[i] - ref[i]) / ref[i]; if (d > worst) worst = d; }
  printf("%-58s %8.1f clk per trip, smem %6.1f KB, sigma[0] %.15g, max rel diff to first %.2e\n", name,
         mean / iters, smem / 1024.0, hs[0], worst);
}

int main() {
  double* d_sigma; long long* d_clk;
  cudaMalloc(&d_sigma, sizeof(double) * 148);
  cudaMalloc(&d_clk, sizeof(long long) * 148);
  static double ref[148] = {0};
  const int iters = 3000;
  run<0>("g6: 6 threads per node, shuffle reductions", iters, d_sigma, d_clk, ref);
  run<0, 2>("g6, 10 of 75 operator entries in shared memory", iters, d_sigma, d_clk, ref);
  run<0, 3>("g6, 15 of 75 operator entries in shared memory", iters, d_sigma, d_clk, ref);
  run<0, 5>("g6, 25 of 75 operator entries in shared memory", iters, d_sigma, d_clk, ref);
  run<16>("g6, forward loads removed", iters, d_sigma, d_clk, ref);
  run<32>("g6, x_{k+1} loads removed", iters, d_sigma, d_clk, ref);
  run<1>("g6, xor-16 exchange removed", iters, d_sigma, d_clk, ref);
  run<2>("g6, reduce-scatter shuffles removed", iters, d_sigma, d_clk, ref);
  run<4 + 8>("g6, neighbour publish + loads removed", iters, d_sigma, d_clk, ref);
  run<1 + 2 + 4 + 8 + 16 + 32>("g6, FMAs + owner stores + norm only", iters, d_sigma, d_clk, ref);
  run<512 + 1024>("g6, both barriers removed (racy)", iters, d_sigma, d_clk, ref);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
