// scp_kernels.cu — the parts of the prox-linear SCP loop that sit between the discretization
// and the convex solve, all per instance and on the device so the loop never returns to the
// host: defect norms and stopping test, scaled-subproblem assembly, power-iteration seed,
// iterate update with quaternion renormalisation, history.
//
// Follows /root/reference/proj/include/ptopt/scp.hpp:139-217 (assemble_subproblem),
// :239-249 (splitmix64 / unit_interval), :256-364 (scp_solve) and
// /root/reference/proj/include/ptopt/rocket_problem.hpp:86-92 (quaternion hook).
#include "kernels.cuh"

namespace ptopt_b200 {

namespace {

constexpr int kScpThreads = 128;

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

__device__ __forceinline__ double block_max(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s = fmax(s, red[w]);
  return s;
}

/// assemble_subproblem for one instance, scp.hpp:166-213.  Power-of-two scales make every
/// product below exact, so the evaluation order is immaterial.
__device__ void assemble_instance(const ScpConst& c, const double* init_state, const double* x,
                                  const double* u, const double* A, const double* Bm,
                                  const double* Bp, const double* x_end, double* Am, double* Bmh,
                                  double* Bph, double* wh, double* eps, double* umin,
                                  double* umax, double* init_val, double* final_val) {
  const int n = c.nodes, m = n - 1;
  const int tid = threadIdx.x, T = blockDim.x;
  for (int e = tid; e < m * kNX * kNX; e += T) {
    const int i = (e / kNX) % kNX, j = e % kNX;
    Am[e] = c.px_inv[i] * A[e] * c.px[j];
  }
  for (int e = tid; e < m * kNX * kNU; e += T) {
    const int i = (e / kNU) % kNX, j = e % kNU;
    Bmh[e] = c.px_inv[i] * Bm[e] * c.pu[j];
    Bph[e] = c.px_inv[i] * Bp[e] * c.pu[j];
  }
  for (int e = tid; e < m * kNX; e += T) {
    const int k = e / kNX, i = e % kNX;
    wh[e] = c.px_inv[i] * (x_end[e] - x[(k + 1) * kNX + i]);
  }
  for (int k = tid; k < m; k += T) {
    const double dy = x[(k + 1) * kNX + kNX - 1] - x[k * kNX + kNX - 1];
    eps[k] = c.epsilon_relax * c.px_inv[kNX - 1] - c.px_inv[kNX - 1] * dy;
  }
  for (int e = tid; e < n * kNU; e += T) {
    const int k = e / kNU, i = e % kNU;
    if (i == kNU - 1) {  // box on the dilation factor only, scp.hpp:196-200
      const double s_bar = u[k * kNU + kNU - 1];
      umin[e] = c.pu_inv[kNU - 1] * (c.s_min - s_bar);
      umax[e] = c.pu_inv[kNU - 1] * (c.s_max - s_bar);
    } else {
      umin[e] = -INFINITY;
      umax[e] = INFINITY;
    }
  }
  for (int i = tid; i < kNX; i += T) {
    const double target = i < kNXI ? init_state[i] : 0.0;
    init_val[i] = c.px_inv[i] * (target - x[i]);
  }
  for (int i = tid; i < c.n_final_fix; i += T) {
    const int idx = c.final_fix_idx[i];
    final_val[i] = c.px_inv[idx] * (c.final_fix_val[i] - x[(n - 1) * kNX + idx]);
  }
}

__global__ void __launch_bounds__(kScpThreads) assemble_kernel(
    ScpConst c, const double* init_state, const double* x, const double* u, const double* A,
    const double* Bm, const double* Bp, const double* x_end, double* Am, double* Bmh, double* Bph,
    double* wh, double* eps, double* umin, double* umax, double* init_val, double* final_val) {
  const int b = blockIdx.x;
  const size_t n = c.nodes, m = n - 1;
  const int nf = c.n_final_fix > 0 ? c.n_final_fix : 1;
  assemble_instance(c, init_state + b * kNXI, x + b * n * kNX, u + b * n * kNU,
                    A + b * m * kNX * kNX, Bm + b * m * kNX * kNU, Bp + b * m * kNX * kNU,
                    x_end + b * m * kNX, Am + b * m * kNX * kNX, Bmh + b * m * kNX * kNU,
                    Bph + b * m * kNX * kNU, wh + b * m * kNX, eps + b * m, umin + b * n * kNU,
                    umax + b * n * kNU, init_val + b * kNX, final_val + (size_t)b * nf);
}

__global__ void scp_init_kernel(ScpArgs a) {
  const int b = blockIdx.x;
  const int n = a.c.nodes, m = n - 1;
  const int tid = threadIdx.x, T = blockDim.x;
  const ScpState& s = a.s;
  // Workspace::init zeroes the warm start, pipg.hpp:122-141
  for (int e = tid; e < n * kNX; e += T) s.ws.x[(size_t)b * n * kNX + e] = 0.0;
  for (int e = tid; e < n * kNU; e += T) s.ws.u[(size_t)b * n * kNU + e] = 0.0;
  for (int e = tid; e < m * kNX; e += T) {
    s.ws.vc_pos[(size_t)b * m * kNX + e] = 0.0;
    s.ws.vc_neg[(size_t)b * m * kNX + e] = 0.0;
    s.ws.dyn_dual[(size_t)b * m * kNX + e] = 0.0;
  }
  for (int e = tid; e < m; e += T) s.ws.relax_dual[(size_t)b * m + e] = 0.0;
  for (int e = tid; e < a.c.max_iters * 5; e += T) s.history[(size_t)b * a.c.max_iters * 5 + e] = 0.0;
  for (int e = tid; e < a.c.max_iters; e += T) s.power_trips[(size_t)b * a.c.max_iters + e] = 0;
  if (tid == 0) {
    s.active[b] = 1;
    s.converged[b] = 0;
    s.solves[b] = 0;
    s.last_step[b] = INFINITY;
    s.final_defect[b] = INFINITY;
    s.status[b] = kStOk;
    s.fail_index[b] = -1;
    s.fail_key[b] = kFailKeyNone;
    s.sigma[b] = 0.0;
    s.pipg_iters[b] = 0;
  }
}

__device__ __forceinline__ unsigned long long splitmix_mix(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(kScpThreads) scp_prepare_kernel(ScpArgs a) {
  __shared__ double red[kScpThreads / 32];
  __shared__ int flag;
  const int b = blockIdx.x;
  const ScpState& s = a.s;
  const ScpConst& c = a.c;
  if (!s.active[b]) return;
  const int n = c.nodes, m = n - 1;
  const int tid = threadIdx.x, T = blockDim.x;

  // a failure inside linearize_all ends the solve (exception in the reference)
  const int key = s.fail_key[b];
  if (key != kFailKeyNone) {
    if (tid == 0) {
      s.status[b] = key & 15;
      s.fail_index[b] = key >> 4;
      s.active[b] = 0;
    }
    return;
  }

  const double* zx = s.zx + (size_t)b * n * kNX;
  const double* zu = s.zu + (size_t)b * n * kNU;
  const double* xe = s.x_end + (size_t)b * m * kNX;

  // defect norms and cost of the iterate, scp.hpp:280-292
  double dinf = 0.0, dl1 = 0.0;
  for (int e = tid; e < m * kNX; e += T) {
    const int k = e / kNX, i = e % kNX;
    const double diff = fabs(xe[e] - zx[(k + 1) * kNX + i]);
    dinf = fmax(dinf, c.px_inv[i] * diff);
    dl1 += diff;
  }
  dinf = block_max(dinf, red);
  dl1 = block_sum(dl1, red);
  double cost_lin = 0.0;
  for (int i = 0; i < kNX; ++i) cost_lin += zx[(n - 1) * kNX + i] * c.e_cost[i];
  const double iterate_cost = c.w_cost * cost_lin + c.w_ep * dl1;
  const int solves = s.solves[b];
  const bool conv = dinf <= c.tol_feas && s.last_step[b] <= c.tol_step;
  const bool stop = conv || solves == c.max_iters;
  __syncthreads();
  if (tid == 0) {
    s.final_defect[b] = dinf;
    if (conv) s.converged[b] = 1;
    if (stop) {
      s.active[b] = 0;
    } else {
      double* h = s.history + ((size_t)b * c.max_iters + solves) * 5;
      h[0] = dinf;
      h[2] = iterate_cost;
    }
  }
  if (stop) return;

  const int nf = c.n_final_fix > 0 ? c.n_final_fix : 1;
  assemble_instance(c, s.init_state + (size_t)b * kNXI, zx, zu, s.A + (size_t)b * m * kNX * kNX,
                    s.Bm + (size_t)b * m * kNX * kNU, s.Bp + (size_t)b * m * kNX * kNU, xe,
                    s.Am + (size_t)b * m * kNX * kNX, s.Bmh + (size_t)b * m * kNX * kNU,
                    s.Bph + (size_t)b * m * kNX * kNU, s.wh + (size_t)b * m * kNX,
                    s.eps + (size_t)b * m, s.umin + (size_t)b * n * kNU,
                    s.umax + (size_t)b * n * kNU, s.init_val + (size_t)b * kNX,
                    s.final_val + (size_t)b * nf);

  // seed of the power iteration, scp.hpp:303-328
  const double* wx = s.ws.x + (size_t)b * n * kNX;
  const double* wu = s.ws.u + (size_t)b * n * kNU;
  const double* wp = s.ws.vc_pos + (size_t)b * m * kNX;
  const double* wn = s.ws.vc_neg + (size_t)b * m * kNX;
  if (tid == 0) flag = 0;
  __syncthreads();
  int nonzero = 0;
  for (int e = tid; e < n * kNX; e += T) nonzero |= (wx[e] != 0.0);
  for (int e = tid; e < n * kNU; e += T) nonzero |= (wu[e] != 0.0);
  for (int e = tid; e < m * kNX; e += T) nonzero |= (wp[e] != 0.0) | (wn[e] != 0.0);
  if (nonzero) atomicOr(&flag, 1);
  __syncthreads();
  double* sx = s.seed_x + (size_t)b * n * kNX;
  double* su = s.seed_u + (size_t)b * n * kNU;
  if (flag) {  // warm start: previous primal solution
    for (int e = tid; e < n * kNX; e += T) sx[e] = wx[e];
    for (int e = tid; e < n * kNU; e += T) su[e] = wu[e];
  } else {
    // draw d (x node-major, then u) is splitmix64 at state0 + (d+1)*golden: the stateful
    // generator of scp.hpp:239-245 unrolled into a counter
    const unsigned long long state0 = s.rng_seed[b] ^ 0x5bf03635d78b41adull;
    double nsq = 0.0;
    for (int e = tid; e < n * (kNX + kNU); e += T) {
      const unsigned long long z =
          splitmix_mix(state0 + (unsigned long long)(e + 1) * 0x9e3779b97f4a7c15ull);
      const double v = 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
      nsq += v * v;
      if (e < n * kNX) sx[e] = v; else su[e - n * kNX] = v;
    }
    nsq = block_sum(nsq, red);
    const double inv = 1.0 / sqrt(nsq);
    for (int e = tid; e < n * (kNX + kNU); e += T) {
      if (e < n * kNX) sx[e] *= inv; else su[e - n * kNX] *= inv;
    }
  }
}

__global__ void __launch_bounds__(kScpThreads) scp_update_kernel(ScpArgs a) {
  __shared__ double red[kScpThreads / 32];
  const int b = blockIdx.x;
  const ScpState& s = a.s;
  const ScpConst& c = a.c;
  if (!s.active[b]) return;  // finished, or the solve of this iteration diverged
  const int n = c.nodes;
  const int tid = threadIdx.x, T = blockDim.x;
  double* zx = s.zx + (size_t)b * n * kNX;
  double* zu = s.zu + (size_t)b * n * kNU;
  const double* wx = s.ws.x + (size_t)b * n * kNX;
  const double* wu = s.ws.u + (size_t)b * n * kNU;

  // step = max_k |x_k|_inf, |u_k|_inf of the scaled solution, scp.hpp:334-338
  double step = 0.0;
  for (int e = tid; e < n * kNX; e += T) step = fmax(step, fabs(wx[e]));
  for (int e = tid; e < n * kNU; e += T) step = fmax(step, fabs(wu[e]));
  step = block_max(step, red);

  // z += P * z_hat, then the quaternion hook, scp.hpp:340-348
  for (int k = tid; k < n; k += T) {
    double* xk = zx + k * kNX;
    double* uk = zu + k * kNU;
#pragma unroll
    for (int i = 0; i < kNX; ++i) xk[i] += c.px[i] * wx[k * kNX + i];
#pragma unroll
    for (int i = 0; i < kNU; ++i) uk[i] += c.pu[i] * wu[k * kNU + i];
    if (c.renorm_quat) {
      double nq = 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i) nq += xk[7 + i] * xk[7 + i];
      nq = sqrt(nq);
      if (nq > 0.0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) xk[7 + i] /= nq;
      }
    }
  }
  if (tid == 0) {
    const int solves = s.solves[b];
    double* h = s.history + ((size_t)b * c.max_iters + solves) * 5;
    h[1] = step;
    h[3] = (double)s.pipg_iters[b];
    h[4] = s.sigma[b];
    s.solves[b] = solves + 1;
    s.last_step[b] = step;
  }
}

}  // namespace

void launch_scp_init(const ScpArgs& a, cudaStream_t stream) {
  scp_init_kernel<<<a.batch, 128, 0, stream>>>(a);
}

void launch_scp_prepare(const ScpArgs& a, cudaStream_t stream) {
  scp_prepare_kernel<<<a.batch, kScpThreads, 0, stream>>>(a);
}

void launch_scp_update(const ScpArgs& a, cudaStream_t stream) {
  scp_update_kernel<<<a.batch, kScpThreads, 0, stream>>>(a);
}

void launch_assemble(const ScpConst& c, int batch, const double* init_state, const double* x,
                     const double* u, const double* A, const double* Bm, const double* Bp,
                     const double* x_end, double* Am, double* Bmh, double* Bph, double* wh,
                     double* eps, double* umin, double* umax, double* init_val, double* final_val,
                     cudaStream_t stream) {
  assemble_kernel<<<batch, kScpThreads, 0, stream>>>(c, init_state, x, u, A, Bm, Bp, x_end, Am,
                                                     Bmh, Bph, wh, eps, umin, umax, init_val,
                                                     final_val);
}

}  // namespace ptopt_b200
