// mapping_c5.cu — one power-iteration trip (same operator, seed and arithmetic as mapping_g6.cu)
// in a COLUMN-split mapping: FIVE threads per node, all inside one warp (six nodes per warp, lanes
// 30 and 31 idle), thread c of node k holds six columns of the packed interval block
// [A-_k | B-_k | B+_k] with all fifteen rows (90 operator doubles, 8 warps, 255 registers):
//   columns of thread c: x columns 3c..3c+2 and the "u slots" c, 5+c, 10+c of
//   [u-_0..6 | u+_0..6 | pad]; the thread OWNS the primal entries its x / u- columns multiply, so the
//   forward product needs no loads for them (only the two u+ values of the next node);
//   * forward product: 15 partial row sums over the thread's columns, reduce-scattered over the five
//     lanes of the node in four shuffle rounds of three values (thread c ends up with dual rows
//     3c..3c+2 complete); the rows are stored rotated (slot t <-> rows of lane (c + t) % 5) so that
//     every round sends a compile-time register;
//   * transposed product: the new duals are all-gathered (four rounds of three values) and the six
//     column sums are thread-local: no partial sums in shared memory at all;
//   * only neighbour-node coupling goes through shared memory (x_{k+1}, u_{k+1}, phi_{k-1},
//     B+^T phi_{k-1}).
// Shuffle volume per thread and trip: 24 doubles (the row-split mapping of the library moves 29
// partial sums out and 35 in through shared memory, and 29 node-vector entries in).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xptxas -v -DKN=48 -o mapping_c5.bin mapping_c5.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#ifndef KN
#define KN 48
#endif
constexpr int kN = KN, kM = kN - 1;
constexpr int kNX = 15, kNU = 7;
constexpr int kWarps = 8, kThreads = 32 * kWarps;
constexpr int kGroups = 6 * kWarps;  // 48 in-warp groups of five lanes
static_assert(kN <= kGroups, "this probe has no odd groups: every node needs an in-warp group");

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

// node arrays: slot 0 is node -1 (zero guard), slots 1..kN the nodes, kN+1 the node behind the
// last one (zero), kN+2 scratch for the idle lanes
constexpr int kSlots = kN + 3;
struct Lay {
  static constexpr int xs = 0;                       // x_k            [slot][16]
  static constexpr int us = xs + kSlots * 16;        // u_k            [slot][8]
  static constexpr int php = us + kSlots * 8;        // phi_k          [slot][16]
  static constexpr int bps = php + kSlots * 16;      // B+_k^T phi_k   [slot][8]
  static constexpr int red = bps + kSlots * 8;       // [2][8]
  static constexpr int scratch = red + 16;           // one double per thread + one zero
  static constexpr int total = scratch + kThreads + 2;
};

template <int ABL>
__global__ void __launch_bounds__(kThreads, 1) trips_c5(int iters, double* sigma_out, long long* clk_out) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = lane / 5, c = lane - 5 * grp;
  const bool idle = grp == 6;
  const int k = idle ? kN + 1 : 6 * warp + grp;  // idle lanes: scratch node
  const bool node = !idle && k < kN, ival = !idle && k < kM;
  const int gid = blockIdx.x;
  for (int e = tid; e < Lay::total; e += kThreads) sm[e] = 0.0;
  __syncthreads();
  // columns of this thread: slot s <-> packed column col[s] (29: the pad)
  auto uslot_col = [](int q) { return q < 14 ? 15 + q : 29; };
  int col[6];
#pragma unroll
  for (int s = 0; s < 3; ++s) col[s] = 3 * c + s;
  col[3] = uslot_col(c);
  col[4] = uslot_col(5 + c);
  col[5] = uslot_col(10 + c);
  // operator: a[t][r][s] = H_k[3 * ((c + t) % 5) + r][col[s]]
  double a[5][3][6];
#pragma unroll
  for (int t = 0; t < 5; ++t)
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        const int row = 3 * ((c + t) % 5) + r;
        a[t][r][s] = (ival && col[s] < 29) ? op_entry(gid, k, row, col[s]) : 0.0;
      }
  // shuffle partners: lane of (c + t) % 5 inside the group (idle lanes talk to themselves)
  int peer[5];
#pragma unroll
  for (int t = 1; t < 5; ++t) peer[t] = idle ? lane : lane - c + (c + t) % 5;
  // addresses (slot index = node + 1)
  double* xs_k = sm + Lay::xs + (k + 1) * 16 + 3 * c;       // own x entries; node k+1 at +16
  double* us_k = sm + Lay::us + (k + 1) * 8;
  double* php_k = sm + Lay::php + (k + 1) * 16 + 3 * c;     // own dual rows; interval k-1 at -16
  double* bps_k = sm + Lay::bps + (k + 1) * 8;
  double* scratch = sm + Lay::scratch + tid;
  const double* zero = sm + Lay::scratch + kThreads;
  // slot 4: u-_{5+c} (c < 2, owned) or u+_{c-2}; slot 5: u+_{3+c} (c < 4) or the pad
  const bool own4 = c < 2;
  const double* z4 = own4 ? us_k + 5 + c : us_k + 8 + (c - 2);
  const double* z5 = c < 4 ? us_k + 8 + 3 + c : zero;
  double* pub4 = own4 ? scratch : bps_k + (c - 2);
  double* pub5 = c < 4 ? bps_k + 3 + c : scratch;
  const double* nb4 = own4 ? bps_k - 8 + 5 + c : zero;
  double* st4 = own4 ? us_k + 5 + c : scratch;
  const double keep4 = (own4 && node) ? 1.0 : 0.0, keep = node ? 1.0 : 0.0;
  double* red = sm + Lay::red;
  // seed: x, u = 1
  double z[4] = {0.0, 0.0, 0.0, 0.0};
  if (node) {
#pragma unroll
    for (int s = 0; s < 3; ++s) { z[s] = 1.0; xs_k[s] = 1.0; }
    z[3] = 1.0;
    us_k[c] = 1.0;
    if (own4) us_k[5 + c] = 1.0;
  }
  __syncthreads();
  double sigma = 1.0;
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const double inv = 1.0 / sigma;
    // ---- forward product, reduce-scattered over the node's five lanes
    const double z4v = *z4, z5v = *z5;
    double acc[3];
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      double p[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        double s0 = a[t][r][0] * z[0], s1 = a[t][r][3] * z[3];
        s0 = fma(a[t][r][1], z[1], s0);
        s1 = fma(a[t][r][4], z4v, s1);
        s0 = fma(a[t][r][2], z[2], s0);
        s1 = fma(a[t][r][5], z5v, s1);
        p[r] = s0 + s1;
      }
      if (t == 0) {
#pragma unroll
        for (int r = 0; r < 3; ++r) acc[r] = p[r];
      } else {
        // my slot t holds rows of lane (c + t) % 5; the rows I own arrive from lane (c - t) % 5
#pragma unroll
        for (int r = 0; r < 3; ++r)
          acc[r] += (ABL & 1) ? p[r] : __shfl_sync(0xffffffffu, p[r], peer[5 - t]);
      }
    }
    double ph[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) ph[r] = ival ? (acc[r] - xs_k[16 + r]) * inv : 0.0;
    // ---- all-gather of the duals, transposed product (thread-local)
    double cs[6];
#pragma unroll
    for (int s = 0; s < 6; ++s) cs[s] = 0.0;
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      double d[3];
#pragma unroll
      for (int r = 0; r < 3; ++r)
        d[r] = t == 0 ? ph[r] : ((ABL & 2) ? ph[r] : __shfl_sync(0xffffffffu, ph[r], peer[t]));
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int s = 0; s < 6; ++s) cs[s] = fma(a[t][r][s], d[r], cs[s]);
    }
    // ---- publish what the neighbour nodes need
    if (!(ABL & 4)) {
#pragma unroll
      for (int r = 0; r < 3; ++r) php_k[r] = ph[r];
      *pub4 = cs[4];
      *pub5 = cs[5];
    }
    if (!(ABL & 512)) __syncthreads();
    // ---- owner sums
    double nrm = 0.0;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const double nb = (ABL & 4) ? 0.25 : php_k[s - 16];
      const double v = keep * (cs[s] - nb);
      z[s] = v;
      xs_k[s] = v;
      nrm = fma(v, v, nrm);
    }
    {
      const double nb = (ABL & 4) ? 0.25 : bps_k[c - 8];
      const double v = keep * (cs[3] + nb);
      z[3] = v;
      us_k[c] = v;
      nrm = fma(v, v, nrm);
    }
    {
      const double nb = (ABL & 4) ? 0.25 : *nb4;
      const double v = keep4 * (cs[4] + nb);
      *st4 = v;
      nrm = fma(v, v, nrm);
    }
    if (node) {
#pragma unroll
      for (int r = 0; r < 3; ++r) nrm = fma(2.0 * ph[r], ph[r], nrm);
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


// ---------------------------------------------------------------------------------------------
// Dataflow variant: no block barriers in the loop.  Every cross-warp dependence is a one-way
// signal on an mbarrier (count 1): fdone[w] "warp w has published the duals of trip j" (awaited by
// warp w+1 before its owner sums), adone[w] "warp w has published the primal entries of trip j"
// (awaited by warp w-1 before its next forward product).  Inside a warp __syncwarp is enough.  The
// 1/sigma scale is applied by the owner sums (everything published by the forward half is
// unscaled), so the squared norm of trip j-1 is only needed half a trip after its shares were
// written: a count-8 mbarrier per parity, never a stall unless a warp is half a trip behind.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_spin(unsigned long long* bar, int phase) {
  unsigned ok, polls = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"((unsigned)(phase & 1)) : "memory");
  } while (!ok && ++polls < (1u << 24));
  if (!ok) __trap();
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, int phase) {
  unsigned ok, polls = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"((unsigned)(phase & 1)) : "memory");
  } while (!ok && ++polls < (1u << 24));
  if (!ok) __trap();
}

template <int ABL>
__global__ void __launch_bounds__(kThreads, 1) trips_c5_df(int iters, double* sigma_out, long long* clk_out) {
  extern __shared__ __align__(16) double sm[];
  __shared__ unsigned long long fdone[kWarps], adone[kWarps], nbar[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = lane / 5, c = lane - 5 * grp;
  const bool idle = grp == 6;
  const int k = idle ? kN + 1 : 6 * warp + grp;
  const bool node = !idle && k < kN, ival = !idle && k < kM;
  const int gid = blockIdx.x;
  for (int e = tid; e < Lay::total; e += kThreads) sm[e] = 0.0;
  if (tid < kWarps) { mbar_init(fdone + tid, 1); mbar_init(adone + tid, 1); }
  if (tid < 2) mbar_init(nbar + tid, kWarps);
  __syncthreads();
  auto uslot_col = [](int q) { return q < 14 ? 15 + q : 29; };
  int col[6];
#pragma unroll
  for (int s = 0; s < 3; ++s) col[s] = 3 * c + s;
  col[3] = uslot_col(c);
  col[4] = uslot_col(5 + c);
  col[5] = uslot_col(10 + c);
  double a[5][3][6];
#pragma unroll
  for (int t = 0; t < 5; ++t)
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        const int row = 3 * ((c + t) % 5) + r;
        a[t][r][s] = (ival && col[s] < 29) ? op_entry(gid, k, row, col[s]) : 0.0;
      }
  int peer[5];
#pragma unroll
  for (int t = 1; t < 5; ++t) peer[t] = idle ? lane : lane - c + (c + t) % 5;
  double* xs_k = sm + Lay::xs + (k + 1) * 16 + 3 * c;
  double* us_k = sm + Lay::us + (k + 1) * 8;
  double* php_k = sm + Lay::php + (k + 1) * 16 + 3 * c;
  double* bps_k = sm + Lay::bps + (k + 1) * 8;
  double* scratch = sm + Lay::scratch + tid;
  const double* zero = sm + Lay::scratch + kThreads;
  const bool own4 = c < 2;
  const double* z4 = own4 ? us_k + 5 + c : us_k + 8 + (c - 2);
  const double* z5 = c < 4 ? us_k + 8 + 3 + c : zero;
  double* pub4 = own4 ? scratch : bps_k + (c - 2);
  double* pub5 = c < 4 ? bps_k + 3 + c : scratch;
  const double* nb4 = own4 ? bps_k - 8 + 5 + c : zero;
  double* st4 = own4 ? us_k + 5 + c : scratch;
  const double keep4 = (own4 && node) ? 1.0 : 0.0, keep = node ? 1.0 : 0.0;
  double* red = sm + Lay::red;  // [2][8]
  double z[4] = {0.0, 0.0, 0.0, 0.0};
  if (node) {
#pragma unroll
    for (int s = 0; s < 3; ++s) { z[s] = 1.0; xs_k[s] = 1.0; }
    z[3] = 1.0;
    us_k[c] = 1.0;
    if (own4) us_k[5 + c] = 1.0;
  }
  __syncthreads();
  const bool has_next = warp + 1 < kWarps, has_prev = warp > 0;
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    // ---- forward half: needs the primal entries the next warp published in trip it-1
    if (it > 0 && has_next && !(ABL & 8)) mbar_wait(adone + warp + 1, it - 1);
    const double z4v = *z4, z5v = *z5;
    double acc[3];
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      double p[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        double s0 = a[t][r][0] * z[0], s1 = a[t][r][3] * z[3];
        s0 = fma(a[t][r][1], z[1], s0);
        s1 = fma(a[t][r][4], z4v, s1);
        s0 = fma(a[t][r][2], z[2], s0);
        s1 = fma(a[t][r][5], z5v, s1);
        p[r] = s0 + s1;
      }
      if (t == 0) {
#pragma unroll
        for (int r = 0; r < 3; ++r) acc[r] = p[r];
      } else {
#pragma unroll
        for (int r = 0; r < 3; ++r) acc[r] += __shfl_sync(0xffffffffu, p[r], peer[5 - t]);
      }
    }
    double ph[3];  // unscaled
#pragma unroll
    for (int r = 0; r < 3; ++r) ph[r] = ival ? acc[r] - xs_k[16 + r] : 0.0;
    double cs[6];
#pragma unroll
    for (int s = 0; s < 6; ++s) cs[s] = 0.0;
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      double d[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) d[r] = t == 0 ? ph[r] : __shfl_sync(0xffffffffu, ph[r], peer[t]);
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int s = 0; s < 6; ++s) cs[s] = fma(a[t][r][s], d[r], cs[s]);
    }
#pragma unroll
    for (int r = 0; r < 3; ++r) php_k[r] = ph[r];
    *pub4 = cs[4];
    *pub5 = cs[5];
    __syncwarp();
    if (lane == 0 && has_next) mbar_arrive(fdone + warp);
    // ---- owner sums: need the duals of the previous warp's last node and the norm of trip it-1
    if (has_prev && !(ABL & 8)) mbar_wait(fdone + warp - 1, it);
    double inv = 1.0;
    if (it > 0) {
      if (!(ABL & 16)) mbar_wait(nbar + (it & 1), (it - 1) >> 1);
      const double2* sh = reinterpret_cast<const double2*>(red + (it & 1) * 8);
      const double2 s0 = sh[0], s1 = sh[1], s2 = sh[2], s3 = sh[3];
      const double tot = ((s0.x + s0.y) + (s1.x + s1.y)) + ((s2.x + s2.y) + (s3.x + s3.y));
      inv = 1.0 / sqrt(tot);
    }
    double nrm = 0.0;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const double v = (keep * inv) * (cs[s] - php_k[s - 16]);
      z[s] = v;
      xs_k[s] = v;
      nrm = fma(v, v, nrm);
    }
    {
      const double v = (keep * inv) * (cs[3] + bps_k[c - 8]);
      z[3] = v;
      us_k[c] = v;
      nrm = fma(v, v, nrm);
    }
    {
      const double v = (keep4 * inv) * (cs[4] + *nb4);
      *st4 = v;
      nrm = fma(v, v, nrm);
    }
    if (node) {
#pragma unroll
      for (int r = 0; r < 3; ++r) { const double q = ph[r] * inv; nrm = fma(2.0 * q, q, nrm); }
    }
    __syncwarp();
    if (lane == 0 && has_prev) mbar_arrive(adone + warp);
    nrm = warp_sum(nrm);
    if (lane == 0) {
      red[((it + 1) & 1) * 8 + warp] = nrm;
      mbar_arrive(nbar + ((it + 1) & 1));
    }
  }
  mbar_wait(nbar + (iters & 1), (iters - 1) >> 1);
  double tot = 0.0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) tot += red[(iters & 1) * 8 + w];
  const double sigma = sqrt(tot);
  const long long t1 = clock64();
  if (tid == 0) {
    sigma_out[gid] = sigma;
    clk_out[gid] = t1 - t0;
  }
}


// ---------------------------------------------------------------------------------------------
// v2: the two block barriers stay, but (a) the shuffles of a phase are issued back to back (all
// twelve partial sums first, then twelve shuffles; all twelve gathers before the products that use
// them), and (b) the norm chain leaves the barrier-to-barrier path: the warp reduction of trip
// it-1 runs beside the forward products of trip it, the shares meet on a count-8 mbarrier, and the
// scale 1/sigma is applied by the owner sums (everything the forward half publishes is unscaled),
// so that sqrt and the reciprocal run beside the transposed products.
// ---------------------------------------------------------------------------------------------
template <int ABL>
__global__ void __launch_bounds__(kThreads, 1) trips_c5_v2(int iters, double* sigma_out, long long* clk_out) {
  extern __shared__ __align__(16) double sm[];
  __shared__ unsigned long long nbar;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = lane / 5, c = lane - 5 * grp;
  const bool idle = grp == 6;
  const int k = idle ? kN + 1 : 6 * warp + grp;
  const bool node = !idle && k < kN, ival = !idle && k < kM;
  const int gid = blockIdx.x;
  for (int e = tid; e < Lay::total; e += kThreads) sm[e] = 0.0;
  if (tid == 0) mbar_init(&nbar, kWarps);
  __syncthreads();
  auto uslot_col = [](int q) { return q < 14 ? 15 + q : 29; };
  int col[6];
#pragma unroll
  for (int s = 0; s < 3; ++s) col[s] = 3 * c + s;
  col[3] = uslot_col(c);
  col[4] = uslot_col(5 + c);
  col[5] = uslot_col(10 + c);
  double a[5][3][6];
#pragma unroll
  for (int t = 0; t < 5; ++t)
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        const int row = 3 * ((c + t) % 5) + r;
        a[t][r][s] = (ival && col[s] < 29) ? op_entry(gid, k, row, col[s]) : 0.0;
      }
  int peer[5];
#pragma unroll
  for (int t = 1; t < 5; ++t) peer[t] = idle ? lane : lane - c + (c + t) % 5;
  double* xs_k = sm + Lay::xs + (k + 1) * 16 + 3 * c;
  double* us_k = sm + Lay::us + (k + 1) * 8;
  double* php_k = sm + Lay::php + (k + 1) * 16 + 3 * c;
  double* bps_k = sm + Lay::bps + (k + 1) * 8;
  double* scratch = sm + Lay::scratch + tid;
  const double* zero = sm + Lay::scratch + kThreads;
  const bool own4 = c < 2;
  const double* z4 = own4 ? us_k + 5 + c : us_k + 8 + (c - 2);
  const double* z5 = c < 4 ? us_k + 8 + 3 + c : zero;
  double* pub4 = own4 ? scratch : bps_k + (c - 2);
  double* pub5 = c < 4 ? bps_k + 3 + c : scratch;
  const double* nb4 = own4 ? bps_k - 8 + 5 + c : zero;
  double* st4 = own4 ? us_k + 5 + c : scratch;
  const double keep4 = (own4 && node) ? 1.0 : 0.0, keep = node ? 1.0 : 0.0;
  double* red = sm + Lay::red;
  double z[4] = {0.0, 0.0, 0.0, 0.0};
  if (node) {
#pragma unroll
    for (int s = 0; s < 3; ++s) { z[s] = 1.0; xs_k[s] = 1.0; }
    z[3] = 1.0;
    us_k[c] = 1.0;
    if (own4) us_k[5 + c] = 1.0;
  }
  __syncthreads();
  double nrm = 0.0;
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    // ---- forward product: all partial sums, then the exchange
    const double z4v = *z4, z5v = *z5;
    double p[5][3];
#pragma unroll
    for (int t = 0; t < 5; ++t)
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        if (ABL & 256) { p[t][r] = a[t][r][0] * z[(t + r) & 3] + z4v + z5v; continue; }
        double s0 = a[t][r][0] * z[0], s1 = a[t][r][3] * z[3];
        s0 = fma(a[t][r][1], z[1], s0);
        s1 = fma(a[t][r][4], z4v, s1);
        s0 = fma(a[t][r][2], z[2], s0);
        s1 = fma(a[t][r][5], z5v, s1);
        p[t][r] = s0 + s1;
      }
    if (it > 0 && !(ABL & 32)) {  // the norm of the iterate this trip starts from
      const double w = warp_sum(nrm);
      if (lane == 0) {
        red[warp] = w;
        if (!(ABL & 64)) mbar_arrive(&nbar);
      }
    }
    double q[5][3];
#pragma unroll
    for (int t = 1; t < 5; ++t)
#pragma unroll
      for (int r = 0; r < 3; ++r) q[t][r] = (ABL & 1) ? p[t][r] : __shfl_sync(0xffffffffu, p[t][r], peer[5 - t]);
    double ph[3];  // unscaled
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const double acc = ((p[0][r] + q[1][r]) + (q[2][r] + q[3][r])) + q[4][r];
      ph[r] = ival ? acc - xs_k[16 + r] : 0.0;
    }
    // ---- all-gather of the duals, transposed product (thread-local)
    double d[5][3];
#pragma unroll
    for (int t = 1; t < 5; ++t)
#pragma unroll
      for (int r = 0; r < 3; ++r) d[t][r] = (ABL & 2) ? ph[r] * (double)t : __shfl_sync(0xffffffffu, ph[r], peer[t]);
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      d[0][r] = ph[r];
      php_k[r] = ph[r];
    }
    double inv = 1.0;
    if (it > 0 && !(ABL & (32 | 64))) {
      if (ABL & 128) mbar_spin(&nbar, it - 1); else mbar_wait(&nbar, it - 1);
      const double2* sh = reinterpret_cast<const double2*>(red);
      const double2 s0 = sh[0], s1 = sh[1], s2 = sh[2], s3 = sh[3];
      const double tot = ((s0.x + s0.y) + (s1.x + s1.y)) + ((s2.x + s2.y) + (s3.x + s3.y));
      inv = rsqrt(tot);
    }
    double cs[6];
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      double c0 = a[0][0][s] * d[0][0], c1 = a[0][1][s] * d[0][1], c2 = a[0][2][s] * d[0][2];
#pragma unroll
      for (int t = 1; t < ((ABL & 2048) ? 1 : 5); ++t) {
        c0 = fma(a[t][0][s], d[t][0], c0);
        c1 = fma(a[t][1][s], d[t][1], c1);
        c2 = fma(a[t][2][s], d[t][2], c2);
      }
      cs[s] = (c0 + c1) + c2;
    }
    *pub4 = cs[4];
    *pub5 = cs[5];
    if (!(ABL & 512)) __syncthreads();
    if (it > 0 && (ABL & 64)) {  // shares written before the barrier above
      const double2* sh = reinterpret_cast<const double2*>(red);
      const double2 s0 = sh[0], s1 = sh[1], s2 = sh[2], s3 = sh[3];
      const double tot = ((s0.x + s0.y) + (s1.x + s1.y)) + ((s2.x + s2.y) + (s3.x + s3.y));
      inv = rsqrt(tot);
    }
    // ---- owner sums, scaled
    nrm = 0.0;
    const double ki = keep * inv;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const double v = ki * (cs[s] - ((ABL & 4) ? 0.25 : php_k[s - 16]));
      z[s] = v;
      xs_k[s] = v;
      nrm = fma(v, v, nrm);
    }
    {
      const double v = ki * (cs[3] + ((ABL & 4) ? 0.25 : bps_k[c - 8]));
      z[3] = v;
      us_k[c] = v;
      nrm = fma(v, v, nrm);
    }
    {
      const double v = (keep4 * inv) * (cs[4] + ((ABL & 4) ? 0.25 : *nb4));
      *st4 = v;
      nrm = fma(v, v, nrm);
    }
    if (node) {
#pragma unroll
      for (int r = 0; r < 3; ++r) { const double g = ph[r] * inv; nrm = fma(2.0 * g, g, nrm); }
    }
    if (!(ABL & 1024)) __syncthreads();
  }
  nrm = warp_sum(nrm);
  if (lane == 0) red[8 + warp] = nrm;
  __syncthreads();
  double tot = 0.0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) tot += red[8 + w];
  const double sigma = sqrt(tot);
  const long long t1 = clock64();
  if (tid == 0) {
    sigma_out[gid] = sigma;
    clk_out[gid] = t1 - t0;
  }
}

template <int ABL>
void run_v2(const char* name, int iters, double* d_sigma, long long* d_clk, double* ref) {
  const size_t smem = (size_t)Lay::total * sizeof(double);
  auto kern = trips_c5_v2<ABL>;
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
  for (int i = 0; i < 148; ++i) { const double d = fabs(hs[i] - ref[i]) / ref[i]; if (d > worst) worst = d; }
  printf("%-58s %8.1f clk per trip, smem %6.1f KB, sigma[0] %.15g, max rel diff to first %.2e\n", name,
         mean / iters, smem / 1024.0, hs[0], worst);
}

template <int ABL>
void run_df(const char* name, int iters, double* d_sigma, long long* d_clk, double* ref) {
  const size_t smem = (size_t)Lay::total * sizeof(double);
  auto kern = trips_c5_df<ABL>;
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
  for (int i = 0; i < 148; ++i) { const double d = fabs(hs[i] - ref[i]) / ref[i]; if (d > worst) worst = d; }
  printf("%-58s %8.1f clk per trip, smem %6.1f KB, sigma[0] %.15g, max rel diff to first %.2e\n", name,
         mean / iters, smem / 1024.0, hs[0], worst);
}

template <int ABL>
void run(const char* name, int iters, double* d_sigma, long long* d_clk, double* ref) {
  const size_t smem = (size_t)Lay::total * sizeof(double);
  auto kern = trips_c5<ABL>;
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
  printf("N = %d nodes\n", kN);
  run<0>("c5: 5 threads per node, column split, shuffle exchange", iters, d_sigma, d_clk, ref);
  run<1>("c5, reduce-scatter shuffles removed", iters, d_sigma, d_clk, ref);
  run<2>("c5, all-gather shuffles removed", iters, d_sigma, d_clk, ref);
  run<1 + 2>("c5, all shuffles removed", iters, d_sigma, d_clk, ref);
  run<4>("c5, neighbour publish + loads removed", iters, d_sigma, d_clk, ref);
  run<512 + 1024>("c5, both barriers removed (racy)", iters, d_sigma, d_clk, ref);
  run_v2<0>("c5 v2: batched shuffles, norm chain beside the products", iters, d_sigma, d_clk, ref);
  run_v2<128>("c5 v2, test_wait spin instead of try_wait", iters, d_sigma, d_clk, ref);
  run_v2<64>("c5 v2, shares through the block barrier", iters, d_sigma, d_clk, ref);
  run_v2<32 + 256>("c5 v2, no norm, forward FMAs removed", iters, d_sigma, d_clk, ref);
  run_v2<32 + 2048>("c5 v2, no norm, transposed FMAs removed", iters, d_sigma, d_clk, ref);
  run_v2<32 + 256 + 2048>("c5 v2, no norm, all FMAs removed", iters, d_sigma, d_clk, ref);
  run_v2<32 + 1 + 2>("c5 v2, no norm, shuffles removed", iters, d_sigma, d_clk, ref);
  run_v2<32 + 4>("c5 v2, no norm, neighbour loads removed", iters, d_sigma, d_clk, ref);
  run_v2<32 + 1 + 2 + 4>("c5 v2, no norm, shuffles + neighbour loads removed", iters, d_sigma, d_clk, ref);
  run_v2<32 + 1 + 2 + 4 + 512 + 1024>("c5 v2, FMAs only (no norm/shuffles/nb/barriers)", iters, d_sigma, d_clk, ref);
  run_v2<32>("c5 v2, norm chain removed", iters, d_sigma, d_clk, ref);
  run_v2<512 + 1024>("c5 v2, both barriers removed (racy)", iters, d_sigma, d_clk, ref);
  run_df<0>("c5 dataflow: mbarrier signals between neighbour warps", iters, d_sigma, d_clk, ref);
  run_df<16>("c5 dataflow, norm wait removed (racy)", iters, d_sigma, d_clk, ref);
  run_df<8>("c5 dataflow, neighbour waits removed (racy)", iters, d_sigma, d_clk, ref);
  run_df<8 + 16>("c5 dataflow, all waits removed (racy)", iters, d_sigma, d_clk, ref);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
