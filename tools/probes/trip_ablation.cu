// trip_ablation.cu — where does a power-iteration trip spend its 2 780 clk?  The control of
// mapping_t3.cu (the library's five-threads-per-node mapping) with pieces removed one at a time
// (template parameter ABL, bit mask): 1 forward FMAs, 2 transposed FMAs, 4 transposed FMAs and
// partial-sum stores, 8 four of the five partial-sum loads, 16 forward loads, 32 warp reduction of
// the norm, 64 sqrt and division, 128 cross-warp sum, 512 / 1024 the two block barriers.  Results
// are wrong by construction; only the clocks matter.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o trip_ablation.bin trip_ablation.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#ifndef KN
#define KN 50
#endif
constexpr int kN = KN, kM = kN - 1;  // nodes, intervals
constexpr int kNX = 15, kNU = 7, kW = 29;
constexpr int kXS = 18, kUS = 10, kPH = 16;

template <int T>
struct Map {
  static constexpr int R = kNX / T;              // operator rows (and state entries) per thread
  static constexpr int UPT = (kNU + T - 1) / T;  // control entries per owner
  static constexpr int PS = T == 5 ? 51 : 53;    // partial-sum slot stride: T*PS == -1 mod 16, conflict-free
  static constexpr int TPI = T == 5 ? 256 : 160; // threads per instance
};

__host__ __device__ inline double op_entry(int inst, int k, int i, int j) {
  uint64_t h = (uint64_t)inst * 0x9E3779B97F4A7C15ull + (uint64_t)(k * 435 + i * 29 + j) * 0xBF58476D1CE4E5B9ull;
  h ^= h >> 31; h *= 0x94D049BB133111EBull; h ^= h >> 29;
  return ((double)(h >> 11) * (1.0 / 9007199254740992.0) - 0.5) * (i == j ? 2.0 : 0.3);
}

__device__ __forceinline__ void tm_ld32(uint32_t (&v)[32], uint32_t addr) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 "
               "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,"
               "%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                 "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                 "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
                 "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
                 "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
               : "r"(addr));
}
__device__ __forceinline__ void tm_ld8(uint32_t (&v)[32], uint32_t addr) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(addr));
}
__device__ __forceinline__ void tm_ld2(uint32_t (&v)[32], uint32_t addr) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n" : "=r"(v[0]), "=r"(v[1]) : "r"(addr));
}
__device__ __forceinline__ void tm_st2(uint32_t addr, double d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};\n" ::"r"(addr), "r"(__double2loint(d)), "r"(__double2hiint(d)));
}
// the staged registers pass through the wait so that no use of them can be scheduled above it
__device__ __forceinline__ void tm_wait_ld(uint32_t (&v)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]), "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31]));
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ double stage_f64(const uint32_t (&v)[32], int e) { return __hiloint2double((int)v[2 * e + 1], (int)v[2 * e]); }

template <int TPI>
__device__ __forceinline__ void inst_barrier(int inst) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(1 + inst), "n"(TPI) : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// T threads per node, INST instances per CTA; of the 29 operator columns the first CREG stay in registers,
// the next CS in thread-private shared memory, the last CT in tensor memory
// DEFER: the scale 1/sigma is applied by the owner sums instead of the forward map, so that the
// warp-level part of the norm reduction moves from the end of a trip to the top of the next one
template <int T, int INST, int CT, int CS, bool DEFER = false, int ABL = 0>
__global__ void __launch_bounds__(INST * Map<T>::TPI, 1) trips(int iters, double* sigma_out, long long* clk_out) {
  using M = Map<T>;
  constexpr int R = M::R, UPT = M::UPT, PS = M::PS, TPI = M::TPI, CREG = kW - CT - CS, CTM = kW - CT, ND = R * CT;
  constexpr int kXsz = (kN + 6) * kXS, kUsz = (kN + 6) * kUS, kPsz = (kN + 6) * kPH, kPart = (TPI + 2 * T) * PS;
  constexpr int kInst = kXsz + kUsz + kPsz + kPart + 16 + R * CS * TPI;
  extern __shared__ __align__(16) double sm[];
  __shared__ uint32_t tm_slot;
  const int inst = threadIdx.x / TPI, tt = threadIdx.x - inst * TPI, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wi = tt >> 5;  // warp inside the instance
  const int gid = blockIdx.x * INST + inst;
  const int k = tt / T, c = tt - k * T;
  const bool node = k < kN, ival = k < kM;
  double* base = sm + (size_t)inst * kInst;
  double* xs = base + kXS;                       // node -1 in front
  double* us = base + kXsz + kUS;
  double* phi = base + kXsz + kUsz + kPH;        // interval -1 in front (zero)
  double* part = base + kXsz + kUsz + kPsz + T * PS;  // T zero slots in front (interval -1)
  double* red = base + kXsz + kUsz + kPsz + kPart;
  double* opx = red + 16 + tt;  // thread-private operator columns: entry e at opx[e * TPI]
  for (int e = threadIdx.x; e < INST * kInst; e += blockDim.x) sm[e] = 0.0;
  uint32_t tm_base = 0;
  if constexpr (CT > 0) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"((uint32_t)__cvta_generic_to_shared(&tm_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
  }
  __syncthreads();
  if constexpr (CT > 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    // lanes of this warp's quarter, a column range of its own among the warps sharing the quarter
    tm_base = tm_slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * (2 * ND));
  }
  // operator rows R*c .. R*c+R-1 of [A- | B- | B+] of interval k
  double a[R][CREG];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < CREG; ++j) a[r][j] = ival ? op_entry(gid, k, R * c + r, j) : 0.0;
  if constexpr (CT > 0) {
#pragma unroll 1
    for (int e = 0; e < ND; ++e) tm_st2(tm_base + 2 * e, ival ? op_entry(gid, k, R * c + e % R, CTM + e / R) : 0.0);
    tm_wait_st();
  }
  if constexpr (CS > 0) {
#pragma unroll 1
    for (int e = 0; e < R * CS; ++e) opx[e * TPI] = ival ? op_entry(gid, k, R * c + e % R, CREG + e / R) : 0.0;
  }
  // seed: x, u = 1
  if (node) {
#pragma unroll
    for (int r = 0; r < R; ++r) xs[k * kXS + R * c + r] = 1.0;
#pragma unroll
    for (int q = 0; q < UPT; ++q)
      if (UPT * c + q < kNU) us[k * kUS + UPT * c + q] = 1.0;
  }
  __syncthreads();
  double sigma = 1.0;
  double* slot = part + (size_t)tt * PS;
  const double* part_k = part + (size_t)k * T * PS;
  auto pos_x = [](int cc, int r) { return R * cc + r; };
  const long long t0 = clock64();
#ifdef PHASES
  long long ph_clk[4] = {0, 0, 0, 0}, tc = t0;  // forward+transposed, barrier 1, owner sums, barrier 2 + norm
#define PHASE(i) { const long long tn = clock64(); ph_clk[i] += tn - tc; tc = tn; }
#else
#define PHASE(i)
#endif
#pragma unroll 1
  double carry = 0.0;  // DEFER: this thread's share of the squared norm of the last trip
  if (DEFER && tt == 0) red[0] = 1.0;  // sigma of the seed
  for (int it = 0; it < iters; ++it) {
    const double inv = DEFER ? 1.0 : ((ABL & 64) ? sigma : 1.0 / sigma);
    if (DEFER && it > 0) {
      const double w = warp_sum(carry);
      if (lane == 0) red[wi] = w;
    }
    double ph[R];
    {  // forward product, dual scaling, transposed partial sums
      uint32_t st[32];
      if constexpr (CT > 0) tm_ld32(st, tm_base);
      double v[kW];
      const double2* x2 = reinterpret_cast<const double2*>(xs + k * kXS);
#pragma unroll
      for (int q = 0; q < 7; ++q) { const double2 t = (ABL & 16) ? make_double2(1.0, 1.0) : x2[q]; v[2 * q] = t.x; v[2 * q + 1] = t.y; }
      v[14] = (ABL & 16) ? 1.0 : xs[k * kXS + 14];
      const double2* u2 = reinterpret_cast<const double2*>(us + k * kUS);
#pragma unroll
      for (int q = 0; q < 4; ++q) { const double2 t = (ABL & 16) ? make_double2(1.0, 1.0) : u2[q]; v[15 + 2 * q] = t.x; if (q < 3) v[16 + 2 * q] = t.y; }
      const double2* w2 = reinterpret_cast<const double2*>(us + (k + 1) * kUS);
#pragma unroll
      for (int q = 0; q < 4; ++q) { const double2 t = (ABL & 16) ? make_double2(1.0, 1.0) : w2[q]; v[22 + 2 * q] = t.x; if (q < 3) v[23 + 2 * q] = t.y; }
      double acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double s = 0.0;
        if constexpr ((ABL & 17) == 0) {
#pragma unroll
          for (int j = 0; j < CREG; ++j) s = fma(a[r][j], v[j], s);
        } else if constexpr ((ABL & 16) == 0) {
          long long f[kW];
#pragma unroll
          for (int j = 0; j < kW; ++j) f[j] = __double_as_longlong(v[j]);
#pragma unroll
          for (int st2 = 1; st2 < kW; st2 *= 2)
#pragma unroll
            for (int j = 0; j + st2 < kW; j += 2 * st2) f[j] ^= f[j + st2];
          s = a[r][0] * __longlong_as_double((f[0] & 0xFFFFll) | 0x3FF0000000000000ll);
        } else {
          s = a[r][0];
        }
        acc[r] = s;
      }
      if constexpr (CS > 0) {
#pragma unroll
        for (int e = 0; e < R * CS; ++e) acc[e % R] = fma(opx[e * TPI], v[CREG + e / R], acc[e % R]);
      }
      if constexpr (CT > 0) {
        constexpr int kFull = ND / 16, kRest = ND - 16 * kFull;  // x32 chunks, then x8 / x2 pieces
#pragma unroll
        for (int ch = 0; ch < kFull; ++ch) {
          tm_wait_ld(st);
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int ee = 16 * ch + e;
            acc[ee % R] = fma(stage_f64(st, e), v[CTM + ee / R], acc[ee % R]);
          }
          if (ch + 1 < kFull) tm_ld32(st, tm_base + 32 * (ch + 1));
        }
        static_assert(kRest == 0 || kRest == 5 || kRest == 4 || kRest == 1, "tail pieces");
        if constexpr (kRest >= 4) {
          tm_ld8(st, tm_base + 32 * kFull);
          tm_wait_ld(st);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int ee = 16 * kFull + e;
            acc[ee % R] = fma(stage_f64(st, e), v[CTM + ee / R], acc[ee % R]);
          }
        }
        if constexpr (kRest == 5 || kRest == 1) {
          const int ee = ND - 1;
          tm_ld2(st, tm_base + 2 * ee);
          tm_wait_ld(st);
          acc[ee % R] = fma(stage_f64(st, 0), v[CTM + ee / R], acc[ee % R]);
        }
        tm_ld32(st, tm_base);  // first chunk of the transposed pass
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        ph[r] = ival ? (acc[r] - xs[(k + 1) * kXS + R * c + r]) * inv : 0.0;
        phi[k * kPH + R * c + r] = ph[r];
      }
#pragma unroll
      for (int j = 0; j < CREG; ++j) {
        double p = (ABL & 6) ? ph[j % R] : a[0][j] * ph[0];
        if constexpr ((ABL & 6) == 0) {
#pragma unroll
          for (int r = 1; r < R; ++r) p = fma(a[r][j], ph[r], p);
        }
        const int pos = j < kNX ? j : (j < kNX + kNU ? 15 + (j - kNX) / UPT * R + (j - kNX) % UPT : 30 + (j - 22) / UPT * R + (j - 22) % UPT);
        if (!(ABL & 4) || j < R) slot[pos] = p;
      }
      if constexpr (CS > 0) {
#pragma unroll
        for (int jj = 0; jj < CS; ++jj) {
          const int j = CREG + jj;
          double p = opx[(R * jj) * TPI] * ph[0];
#pragma unroll
          for (int r = 1; r < R; ++r) p = fma(opx[(R * jj + r) * TPI], ph[r], p);
          const int pos = j < kNX ? j : (j < kNX + kNU ? 15 + (j - kNX) / UPT * R + (j - kNX) % UPT : 30 + (j - 22) / UPT * R + (j - 22) % UPT);
          slot[pos] = p;
        }
      }
      if constexpr (CT > 0) {
        constexpr int kFull = ND / 16, kRest = ND - 16 * kFull;
        double pc = 0.0;
        auto feed = [&](double op, int ee) {
          const int j = CTM + ee / R, r = ee % R;
          pc = r == 0 ? op * ph[0] : fma(op, ph[r], pc);
          if (r == R - 1) {
            const int pos = j < kNX ? j : (j < kNX + kNU ? 15 + (j - kNX) / UPT * R + (j - kNX) % UPT : 30 + (j - 22) / UPT * R + (j - 22) % UPT);
            slot[pos] = pc;
          }
        };
#pragma unroll
        for (int ch = 0; ch < kFull; ++ch) {
          tm_wait_ld(st);
#pragma unroll
          for (int e = 0; e < 16; ++e) feed(stage_f64(st, e), 16 * ch + e);
          if (ch + 1 < kFull) tm_ld32(st, tm_base + 32 * (ch + 1));
        }
        if constexpr (kRest >= 4) {
          tm_ld8(st, tm_base + 32 * kFull);
          tm_wait_ld(st);
#pragma unroll
          for (int e = 0; e < 4; ++e) feed(stage_f64(st, e), 16 * kFull + e);
        }
        if constexpr (kRest == 5 || kRest == 1) {
          tm_ld2(st, tm_base + 2 * (ND - 1));
          tm_wait_ld(st);
          feed(stage_f64(st, 0), ND - 1);
        }
      }
    }
    PHASE(0)
    if constexpr (!(ABL & 1024)) { if constexpr (INST == 1) __syncthreads(); else inst_barrier<TPI>(inst); }
    PHASE(1)
    double nrm = 0.0, sc = 1.0;
    if constexpr (DEFER) {
      double tot = 0.0;
#pragma unroll
      for (int w = 0; w < TPI / 32; ++w) tot += red[w];
      sc = rsqrt(tot);
      sigma = sqrt(tot);
    }
    if (node) {  // owner sums: x = A-^T phi_k - phi_{k-1}, u = B-^T phi_k + B+^T phi_{k-1}
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < ((ABL & 8) ? 1 : T); ++q) s += part_k[q * PS + pos_x(c, r)];
        const double x = DEFER ? (s - phi[(k - 1) * kPH + R * c + r]) * sc : s - phi[(k - 1) * kPH + R * c + r];
        xs[k * kXS + R * c + r] = x;
        nrm = fma(x, x, nrm);
      }
#pragma unroll
      for (int q = 0; q < UPT; ++q) {
        double s = 0.0;
#pragma unroll
        for (int p = 0; p < ((ABL & 8) ? 1 : T); ++p) s += part_k[p * PS + 15 + R * c + q] + part_k[(p - T) * PS + 30 + R * c + q];
        if constexpr (DEFER) s *= sc;
        if (UPT * c + q < kNU) {
          us[k * kUS + UPT * c + q] = s;
          nrm = fma(s, s, nrm);
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) nrm = DEFER ? fma(2.0 * (ph[r] * sc), ph[r] * sc, nrm) : fma(2.0 * ph[r], ph[r], nrm);
    }
    if constexpr (DEFER) {
      carry = nrm;
    } else {
      if (!(ABL & 32)) nrm = warp_sum(nrm);
      if (lane == 0) red[wi] = nrm;
    }
    PHASE(2)
    if constexpr (!(ABL & 512)) { if constexpr (INST == 1) __syncthreads(); else inst_barrier<TPI>(inst); }
    if constexpr (!DEFER) {
      double tot = 0.0;
#pragma unroll
      for (int w = 0; w < ((ABL & 128) ? 1 : TPI / 32); ++w) tot += red[w];
      sigma = (ABL & 64) ? tot * 1e-3 : sqrt(tot);
    }
    PHASE(3)
  }
  if constexpr (DEFER) {
    const double w = warp_sum(carry);
    if (lane == 0) red[wi] = w;
    if constexpr (INST == 1) __syncthreads(); else inst_barrier<TPI>(inst);
    double tot = 0.0;
#pragma unroll
    for (int w2 = 0; w2 < TPI / 32; ++w2) tot += red[w2];
    sigma = sqrt(tot);
  }
  const long long t1 = clock64();
  if (tt == 0) {
    sigma_out[gid] = sigma;
    clk_out[gid] = t1 - t0;
  }
#ifdef PHASES
  if (blockIdx.x == 0 && inst == 0 && lane == 0)
    printf("  warp %d: forward+transposed %.0f, barrier %.0f, owner sums %.0f, barrier+norm %.0f clk per trip\n", wi,
           (double)ph_clk[0] / iters, (double)ph_clk[1] / iters, (double)ph_clk[2] / iters, (double)ph_clk[3] / iters);
#endif
  if constexpr (CT > 0) {
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tm_slot));
  }
}

template <int T, int INST, int CT, int CS, bool DEFER = false, int ABL = 0>
void run(const char* name, int iters, double* d_sigma, long long* d_clk, double* ref) {
  using M = Map<T>;
  constexpr int kInst = (kN + 6) * (kXS + kUS + kPH) + (M::TPI + 2 * T) * M::PS + 16 + M::R * CS * M::TPI;
  const size_t smem = (size_t)INST * kInst * sizeof(double);
  auto kern = trips<T, INST, CT, CS, DEFER, ABL>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = 148;
  kern<<<grid, INST * M::TPI, smem>>>(iters, d_sigma, d_clk);
  kern<<<grid, INST * M::TPI, smem>>>(iters, d_sigma, d_clk);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  static double hs[148 * 2];
  static long long hc[148 * 2];
  cudaMemcpy(hs, d_sigma, sizeof(double) * grid * INST, cudaMemcpyDeviceToHost);
  cudaMemcpy(hc, d_clk, sizeof(long long) * grid * INST, cudaMemcpyDeviceToHost);
  double mean = 0, worst = 0;
  for (int i = 0; i < grid * INST; ++i) mean += (double)hc[i] / (grid * INST);
  if (ref[0] == 0.0) for (int i = 0; i < 148; ++i) ref[i] = hs[i];
  for (int i = 0; i < 148; ++i) { const double d = fabs(hs[i] - ref[i]) / ref[i]; if (d > worst) worst = d; }
  printf("%-58s %8.1f clk per trip and CTA, %8.1f clk per instance-trip, smem %6.1f KB, sigma[0] %.15g, max rel diff to first %.2e\n",
         name, mean / iters, mean / iters / INST, smem / 1024.0, hs[0], worst);
}

int main() {
  double* d_sigma; long long* d_clk;
  cudaMalloc(&d_sigma, sizeof(double) * 296);
  cudaMalloc(&d_clk, sizeof(long long) * 296);
  static double ref[148] = {0};
  const int iters = 3000;
  run<5, 1, 0, 0>("control", iters, d_sigma, d_clk, ref);
  run<5, 1, 0, 0, false, 1>("forward FMAs removed (loads kept)", iters, d_sigma, d_clk, ref);
  run<5, 1, 0, 0, false, 2>("transposed FMAs removed (stores kept)", iters, d_sigma, d_clk, ref);
  run<5, 1, 0, 0, false, 3>("all FMAs removed", iters, d_sigma, d_clk, ref);
  run<5, 1, 0, 0, false, 4>("transposed FMAs and partial stores removed", iters, d_sigma, d_clk, ref);
  run<5, 1, 0, 0, false, 8>("1 of 5 partial loads", iters, d_sigma, d_clk, ref);
  run<5, 1, 0, 0, false, 17>("forward loads and FMAs removed", iters, d_sigma, d_clk, ref);
  run<5, 1, 0, 0, false, 29>("skeleton: barriers, norm, owner stores only", iters, d_sigma, d_clk, ref);
  run<5, 1, 0, 0, false, 29 + 32>("skeleton, no warp reduction", iters, d_sigma, d_clk, ref);
  run<5, 1, 0, 0, false, 29 + 64>("skeleton, no sqrt / division", iters, d_sigma, d_clk, ref);
  run<5, 1, 0, 0, false, 29 + 32 + 64 + 128>("bare skeleton (no norm chain)", iters, d_sigma, d_clk, ref);
  run<5, 1, 0, 0, false, 29 + 32 + 64 + 128 + 512 + 1024>("bare skeleton, both barriers removed", iters, d_sigma, d_clk, ref);
  run<5, 1, 0, 0, false, 32 + 64 + 128>("full work, no norm chain", iters, d_sigma, d_clk, ref);
  run<5, 1, 0, 0, false, 512 + 1024>("full work, both barriers removed", iters, d_sigma, d_clk, ref);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
