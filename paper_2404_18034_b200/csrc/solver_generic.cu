// solver_generic.cu — shape-generic power iteration and customized PIPG.
//
// One CTA per subproblem instance; iterate vectors live in shared memory, operator blocks are
// read from global memory through the read-only path.  Any run-time shape inside the
// reference's capacities (n_x <= 15, n_u <= 7, any node count whose vectors fit in shared
// memory) and an explicit A_plus are supported, so the reference's small synthetic
// subproblems run unchanged.  The rocket-shaped fast path lives in solver_fast.cu.
//
// Follows /root/reference/proj/include/ptopt/pipg.hpp:206-292 (power_iteration_custom),
// :307-326 (stopping_custom), :335-340 (step_sizes), :350-497 (pipg_custom).
#include "kernels.cuh"

namespace ptopt_b200 {

namespace {

constexpr int kMaxWarps = 32;
constexpr int kMaxGenericThreads = 768;  // 72 registers per thread must fit one SM's register file

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}


/// Row i of (block * vec): sum_j M[i][j] v[j], ascending j (mat_vec, smallmat.hpp:93-97).
__device__ __forceinline__ double row_dot(const double* __restrict__ M, int cols, int i,
                                          const double* v) {
  double acc = 0.0;
  const double* row = M + i * cols;
  for (int j = 0; j < cols; ++j) acc += __ldg(row + j) * v[j];
  return acc;
}

/// Column i of (block^T * vec): sum_r M[r][i] v[r], ascending r (smallmat.hpp:99-103).
__device__ __forceinline__ double col_dot(const double* __restrict__ M, int rows, int cols, int i,
                                          const double* v) {
  double acc = 0.0;
  for (int r = 0; r < rows; ++r) acc += __ldg(M + r * cols + i) * v[r];
  return acc;
}

__global__ void __launch_bounds__(kMaxGenericThreads, 1) power_generic_kernel(PowerArgs a) {
  extern __shared__ double sm[];
  const int b = blockIdx.x;
  if (a.active && !a.active[b]) return;
  const int nx = a.shape.nx, nu = a.shape.nu, n = a.shape.n, m = n - 1;
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = T >> 5;
  double* x = sm;
  double* u = x + n * nx;
  double* vcp = u + n * nu;
  double* vcn = vcp + m * nx;
  double* phi = vcn + m * nx;
  double* theta = phi + m * nx;
  double* red = theta + m;  // [kMaxWarps]
  double* ey = red + kMaxWarps;
  for (int i = tid; i < nx; i += T) ey[i] = a.shape.e_y[i];

  const double* Am = a.sp.A_minus + (size_t)b * m * nx * nx;
  const double* Ap = a.sp.A_plus ? a.sp.A_plus + (size_t)b * m * nx * nx : nullptr;
  const double* Bm = a.sp.B_minus + (size_t)b * m * nx * nu;
  const double* Bp = a.sp.B_plus + (size_t)b * m * nx * nu;

  double acc = 0.0;
  {
    const double* sx = a.seed_x + (size_t)b * n * nx;
    const double* su = a.seed_u + (size_t)b * n * nu;
    const double* sp = a.seed_vcp + (size_t)b * m * nx;
    const double* sn = a.seed_vcn + (size_t)b * m * nx;
    for (int e = tid; e < n * nx; e += T) { const double v = sx[e]; x[e] = v; acc += v * v; }
    for (int e = tid; e < n * nu; e += T) { const double v = su[e]; u[e] = v; acc += v * v; }
    for (int e = tid; e < m * nx; e += T) {
      const double v = sp[e], q = sn[e];
      vcp[e] = v;
      vcn[e] = q;
      acc += v * v;
      acc += q * q;
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  double sigma = 0.0;
  for (int w = 0; w < nwarps; ++w) sigma += red[w];
  if (sigma == 0.0) {  // pipg.hpp:224-225
    if (tid == 0) {
      if (a.status) a.status[b] = kStSeedZero;
      a.sigma[b] = 0.0;
      if (a.trips) a.trips[(size_t)b * a.trips_stride + (a.trips_slot ? a.trips_slot[b] : 0)] = 0;
    }
    return;
  }
  sigma = sqrt(sigma);
  __syncthreads();  // red is reused below

  int trips = 0;
  for (int j = 1; j <= a.j_max; ++j) {
    trips = j;
    const double inv = 1.0 / sigma;
    // forward map scaled by 1/sigma, pipg.hpp:234-245
    for (int e = tid; e < m * nx; e += T) {
      const int k = e / nx, i = e - k * nx;
      double r = row_dot(Am + (size_t)k * nx * nx, nx, i, x + k * nx);
      r += Ap ? row_dot(Ap + (size_t)k * nx * nx, nx, i, x + (k + 1) * nx) : -x[(k + 1) * nx + i];
      r += row_dot(Bm + (size_t)k * nx * nu, nu, i, u + k * nu);
      r += row_dot(Bp + (size_t)k * nx * nu, nu, i, u + (k + 1) * nu);
      r += vcp[e];
      r += -1.0 * vcn[e];
      phi[e] = r * inv;
    }
    for (int k = tid; k < m; k += T) {
      double d1 = 0.0, d0 = 0.0;
      for (int i = 0; i < nx; ++i) {
        d1 += ey[i] * x[(k + 1) * nx + i];
        d0 += ey[i] * x[k * nx + i];
      }
      theta[k] = (d1 - d0) / sigma;
    }
    __syncthreads();
    // adjoint map, pipg.hpp:247-275
    acc = 0.0;
    for (int e = tid; e < n * nx; e += T) {
      const int k = e / nx, i = e - k * nx;
      double r = 0.0;
      if (k < m) r = col_dot(Am + (size_t)k * nx * nx, nx, nx, i, phi + k * nx);
      if (k > 0) {
        const double t = Ap ? col_dot(Ap + (size_t)(k - 1) * nx * nx, nx, nx, i, phi + (k - 1) * nx)
                            : -phi[(k - 1) * nx + i];
        r = (k < m) ? r + t : t;
      }
      if (k < m) r += -theta[k] * ey[i];
      if (k > 0) r += theta[k - 1] * ey[i];
      x[e] = r;
      acc += r * r;
    }
    for (int e = tid; e < n * nu; e += T) {
      const int k = e / nu, i = e - k * nu;
      double r = 0.0;
      if (k < m) r = col_dot(Bm + (size_t)k * nx * nu, nx, nu, i, phi + k * nx);
      if (k > 0) {
        const double t = col_dot(Bp + (size_t)(k - 1) * nx * nu, nx, nu, i, phi + (k - 1) * nx);
        r = (k < m) ? r + t : t;
      }
      u[e] = r;
      acc += r * r;
    }
    for (int e = tid; e < m * nx; e += T) {
      const double p = phi[e];
      vcp[e] = p;
      vcn[e] = -p;
      acc += p * p;
      acc += p * p;
    }
    acc = warp_sum(acc);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    double sigma_star = 0.0;
    for (int w = 0; w < nwarps; ++w) sigma_star += red[w];
    sigma_star = sqrt(sigma_star);
    if (sigma_star == 0.0) {  // seed in the null space, pipg.hpp:280-284
      sigma = 0.0;
      break;
    }
    if (fabs(sigma_star - sigma) <= a.eps_abs + a.eps_rel * max_nn(sigma_star, sigma)) {
      sigma = sigma_star;
      break;
    }
    sigma = sigma_star;
  }
  if (tid == 0) {
    a.sigma[b] = (1.0 + a.eps_buff) * sigma;
    if (a.trips) a.trips[(size_t)b * a.trips_stride + (a.trips_slot ? a.trips_slot[b] : 0)] = trips;
  }
}

__global__ void __launch_bounds__(kMaxGenericThreads, 1) pipg_generic_kernel(PipgArgs a) {
  extern __shared__ double sm[];
  const int b = blockIdx.x;
  if (a.active && !a.active[b]) return;
  const int nx = a.shape.nx, nu = a.shape.nu, n = a.shape.n, m = n - 1;
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = T >> 5;
  const int NXn = n * nx, NUn = n * nu, NM = m * nx;
  double* x_ex = sm;
  double* u_ex = x_ex + NXn;
  double* vp_ex = u_ex + NUn;
  double* vn_ex = vp_ex + NM;
  double* ph_ex = vn_ex + NM;
  double* th_ex = ph_ex + NM;
  double* x_cur = th_ex + m;
  double* u_cur = x_cur + NXn;
  double* vp_cur = u_cur + NUn;
  double* vn_cur = vp_cur + NM;
  double* ph_cur = vn_cur + NM;
  double* th_cur = ph_cur + NM;
  double* x_rf = th_cur + m;  // reflections 2*cur - ex, pipg.hpp:436-443
  double* u_rf = x_rf + NXn;
  double* red = u_rf + NUn;  // [7][kMaxWarps]
  double* ey = red + 7 * kMaxWarps;
  double* ecost = ey + kNX;
  double* init_val = ecost + kNX;   // value per state slot at node 0
  double* final_val = init_val + kNX;
  int* init_on = reinterpret_cast<int*>(final_val + kNX);
  int* final_on = init_on + kNX;

  const double* Am = a.sp.A_minus + (size_t)b * m * nx * nx;
  const double* Ap = a.sp.A_plus ? a.sp.A_plus + (size_t)b * m * nx * nx : nullptr;
  const double* Bm = a.sp.B_minus + (size_t)b * m * nx * nu;
  const double* Bp = a.sp.B_plus + (size_t)b * m * nx * nu;
  const double* wv = a.sp.w + (size_t)b * NM;
  const double* epsr = a.sp.eps_relax + (size_t)b * m;
  const double* umin = a.sp.u_min + (size_t)b * NUn;
  const double* umax = a.sp.u_max + (size_t)b * NUn;

  if (tid == 0) {
    for (int i = 0; i < kNX; ++i) {
      init_on[i] = 0;
      final_on[i] = 0;
      ey[i] = i < nx ? a.shape.e_y[i] : 0.0;
      ecost[i] = i < nx ? a.shape.e_cost[i] : 0.0;
    }
    // later entries override earlier ones, as the assignment loops do (pipg.hpp:408-413)
    for (int i = 0; i < a.shape.n_init_fix; ++i) {
      init_on[a.shape.init_fix_idx[i]] = 1;
      init_val[a.shape.init_fix_idx[i]] = a.sp.init_fix_val[(size_t)b * a.shape.n_init_fix + i];
    }
    for (int i = 0; i < a.shape.n_final_fix; ++i) {
      final_on[a.shape.final_fix_idx[i]] = 1;
      final_val[a.shape.final_fix_idx[i]] = a.sp.final_fix_val[(size_t)b * a.shape.n_final_fix + i];
    }
  }
  // warm start: ex = cur = workspace, pipg.hpp:362-374
  for (int e = tid; e < NXn; e += T) x_ex[e] = x_cur[e] = a.ws.x[(size_t)b * NXn + e];
  for (int e = tid; e < NUn; e += T) u_ex[e] = u_cur[e] = a.ws.u[(size_t)b * NUn + e];
  for (int e = tid; e < NM; e += T) {
    vp_ex[e] = vp_cur[e] = a.ws.vc_pos[(size_t)b * NM + e];
    vn_ex[e] = vn_cur[e] = a.ws.vc_neg[(size_t)b * NM + e];
    ph_ex[e] = ph_cur[e] = a.ws.dyn_dual[(size_t)b * NM + e];
  }
  for (int e = tid; e < m; e += T) th_ex[e] = th_cur[e] = a.ws.relax_dual[(size_t)b * m + e];

  const double w_prox = a.shape.w_prox, w_ep = a.shape.w_ep, w_cost = a.shape.w_cost;
  const double sigma = a.sigma[b];
  const double alpha = 2.0 / (w_prox + sqrt(w_prox * w_prox + 4.0 * a.omega * sigma));
  const double beta = a.omega * alpha;
  const double rho = a.rho;
  __syncthreads();

  int iters = 0;
  bool converged = false, diverged = false;
  for (int j = 1; j <= a.j_max; ++j) {
    const bool check = (j % a.j_check) == 0;
    double z_cur = 0.0, z_prev = 0.0, z_del = 0.0, r_cur = 0.0, r_prev = 0.0, r_del = 0.0;
    double bad = 0.0;  // > 0 when a checked entry is not finite

    // ---- primal projected-gradient step, pipg.hpp:388-420 (extrapolation of the previous
    //      iteration, :461-467, is applied here by the element's owner)
    for (int e = tid; e < NXn; e += T) {
      const int k = e / nx, i = e - k * nx;
      double xe = x_ex[e];
      const double old = x_cur[e];
      if (j > 1) {
        xe = (1.0 - rho) * xe + rho * old;
        x_ex[e] = xe;
      }
      double grad = xe * w_prox;
      if (k < m) {
        grad += col_dot(Am + (size_t)k * nx * nx, nx, nx, i, ph_ex + k * nx);
        grad += -th_ex[k] * ey[i];
      }
      if (k > 0) {
        grad += Ap ? col_dot(Ap + (size_t)(k - 1) * nx * nx, nx, nx, i, ph_ex + (k - 1) * nx)
                   : -ph_ex[(k - 1) * nx + i];
        grad += th_ex[k - 1] * ey[i];
      }
      if (k == n - 1) grad += w_cost * ecost[i];
      double xn = xe + -alpha * grad;
      if (k == 0 && init_on[i]) xn = init_val[i];
      if (k == n - 1 && final_on[i]) xn = final_val[i];
      x_cur[e] = xn;
      x_rf[e] = 2.0 * xn - xe;
      if (check) {
        z_cur = max_nn(z_cur, fabs(xn));
        z_prev = max_nn(z_prev, fabs(old));
        z_del = max_nn(z_del, fabs(xn - old));
        if (!pt_finite(xn)) bad = 1.0;
      }
    }
    for (int e = tid; e < NUn; e += T) {
      const int k = e / nu, i = e - k * nu;
      double ue = u_ex[e];
      const double old = u_cur[e];
      if (j > 1) {
        ue = (1.0 - rho) * ue + rho * old;
        u_ex[e] = ue;
      }
      double grad = ue * w_prox;
      if (k < m) grad += col_dot(Bm + (size_t)k * nx * nu, nx, nu, i, ph_ex + k * nx);
      if (k > 0) grad += col_dot(Bp + (size_t)(k - 1) * nx * nu, nx, nu, i, ph_ex + (k - 1) * nx);
      double un = ue + -alpha * grad;
      // std::max(lo, std::min(hi, v)), pipg.hpp:418-419
      const double lo = __ldg(umin + e), hi = __ldg(umax + e);
      const double cl = (hi < un) ? hi : un;
      un = (lo < cl) ? cl : lo;
      u_cur[e] = un;
      u_rf[e] = 2.0 * un - ue;
      if (check) {
        z_cur = max_nn(z_cur, fabs(un));
        z_prev = max_nn(z_prev, fabs(old));
        z_del = max_nn(z_del, fabs(un - old));
        if (!pt_finite(un)) bad = 1.0;
      }
    }
    // ---- virtual-control slacks, pipg.hpp:423-430
    for (int e = tid; e < NM; e += T) {
      const double ph = ph_ex[e];
      const double vp = clip0(vp_ex[e] - alpha * (w_ep + ph));
      const double vn = clip0(vn_ex[e] - alpha * (w_ep - ph));
      if (check) {
        const double op = vp_cur[e], on = vn_cur[e];
        z_cur = max_nn(max_nn(z_cur, fabs(vp)), fabs(vn));
        z_prev = max_nn(max_nn(z_prev, fabs(op)), fabs(on));
        z_del = max_nn(max_nn(z_del, fabs(vp - op)), fabs(vn - on));
      }
      vp_cur[e] = vp;
      vn_cur[e] = vn;
    }
    __syncthreads();

    // ---- PI feedback of the constraint violation, pipg.hpp:433-458, with the dual and slack
    //      extrapolation (:468-472) done in place by the owner
    for (int e = tid; e < NM; e += T) {
      const int k = e / nx, i = e - k * nx;
      double resid = row_dot(Am + (size_t)k * nx * nx, nx, i, x_rf + k * nx);
      resid += Ap ? row_dot(Ap + (size_t)k * nx * nx, nx, i, x_rf + (k + 1) * nx)
                  : -x_rf[(k + 1) * nx + i];
      resid += row_dot(Bm + (size_t)k * nx * nu, nu, i, u_rf + k * nu);
      resid += row_dot(Bp + (size_t)k * nx * nu, nu, i, u_rf + (k + 1) * nu);
      const double vpc = vp_cur[e], vnc = vn_cur[e], vpe = vp_ex[e], vne = vn_ex[e];
      resid += (2.0 * vpc - vpe) - (2.0 * vnc - vne) + __ldg(wv + e);
      const double phe = ph_ex[e];
      const double phn = phe + beta * resid;
      if (check) {
        const double old = ph_cur[e];
        r_cur = max_nn(r_cur, fabs(phn));
        r_prev = max_nn(r_prev, fabs(old));
        r_del = max_nn(r_del, fabs(phn - old));
        if (!pt_finite(phn)) bad = 1.0;
      }
      ph_cur[e] = phn;
      ph_ex[e] = (1.0 - rho) * phe + rho * phn;
      vp_ex[e] = (1.0 - rho) * vpe + rho * vpc;
      vn_ex[e] = (1.0 - rho) * vne + rho * vnc;
    }
    for (int k = tid; k < m; k += T) {
      double d1 = 0.0, d0 = 0.0;
      for (int i = 0; i < nx; ++i) {
        d1 += ey[i] * x_rf[(k + 1) * nx + i];
        d0 += ey[i] * x_rf[k * nx + i];
      }
      const double drift = d1 - d0 - __ldg(epsr + k);
      const double the = th_ex[k];
      const double thn = clip0(the + beta * drift);
      if (check) {
        const double old = th_cur[k];
        r_cur = max_nn(r_cur, fabs(thn));
        r_prev = max_nn(r_prev, fabs(old));
        r_del = max_nn(r_del, fabs(thn - old));
      }
      th_cur[k] = thn;
      th_ex[k] = (1.0 - rho) * the + rho * thn;
    }
    iters = j;
    if (check) {
      z_cur = warp_max_nn(z_cur); z_prev = warp_max_nn(z_prev); z_del = warp_max_nn(z_del);
      r_cur = warp_max_nn(r_cur); r_prev = warp_max_nn(r_prev); r_del = warp_max_nn(r_del);
      bad = warp_max_nn(bad);
      if (lane == 0) {
        red[0 * kMaxWarps + warp] = z_cur; red[1 * kMaxWarps + warp] = z_prev;
        red[2 * kMaxWarps + warp] = z_del; red[3 * kMaxWarps + warp] = r_cur;
        red[4 * kMaxWarps + warp] = r_prev; red[5 * kMaxWarps + warp] = r_del;
        red[6 * kMaxWarps + warp] = bad;
      }
    }
    __syncthreads();
    if (check) {  // pipg.hpp:475-487
      double v[7];
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        double mx = 0.0;
        for (int w = 0; w < nwarps; ++w) mx = max_nn(mx, red[q * kMaxWarps + w]);
        v[q] = mx;
      }
      if (v[6] > 0.0) {
        diverged = true;
        break;
      }
      if (v[2] <= a.eps_abs + a.eps_rel * max_nn(v[0], v[1]) &&
          v[5] <= a.eps_abs + a.eps_rel * max_nn(v[3], v[4])) {
        converged = true;
        break;
      }
    }
  }

  if (diverged) {  // SolverDiverged(j): the workspace is left untouched, pipg.hpp:478
    if (tid == 0) {
      if (a.status) a.status[b] = kStSolverDiverged;
      if (a.fail_index) a.fail_index[b] = iters;
      if (a.iterations) a.iterations[b] = iters;
      if (a.converged) a.converged[b] = 0;
      if (a.active) a.active[b] = 0;
    }
    return;
  }
  // solution = the *_cur groups, pipg.hpp:490-495
  for (int e = tid; e < NXn; e += T) a.ws.x[(size_t)b * NXn + e] = x_cur[e];
  for (int e = tid; e < NUn; e += T) a.ws.u[(size_t)b * NUn + e] = u_cur[e];
  for (int e = tid; e < NM; e += T) {
    a.ws.vc_pos[(size_t)b * NM + e] = vp_cur[e];
    a.ws.vc_neg[(size_t)b * NM + e] = vn_cur[e];
    a.ws.dyn_dual[(size_t)b * NM + e] = ph_cur[e];
  }
  for (int e = tid; e < m; e += T) a.ws.relax_dual[(size_t)b * m + e] = th_cur[e];
  if (tid == 0) {
    if (a.iterations) a.iterations[b] = iters;
    if (a.converged) a.converged[b] = converged ? 1 : 0;
  }
}

}  // namespace

int solver_generic_threads(const SubShape& s) {
  int t = ((s.n * s.nx + 31) / 32) * 32;
  if (t < 64) t = 64;
  if (t > kMaxGenericThreads) t = kMaxGenericThreads;
  return t;
}

size_t power_generic_smem(const SubShape& s, int) {
  const int m = s.n - 1;
  return sizeof(double) * (size_t)(s.n * (s.nx + s.nu) + 3 * m * s.nx + m + kMaxWarps + kNX);
}

size_t pipg_generic_smem(const SubShape& s, int) {
  const int m = s.n - 1;
  const size_t vec = (size_t)(s.n * (s.nx + s.nu) + 3 * m * s.nx + m);
  return sizeof(double) * (2 * vec + (size_t)s.n * (s.nx + s.nu) + 7 * kMaxWarps + 4 * kNX) +
         sizeof(int) * 2 * kNX;
}

cudaError_t configure_solver_generic(const SubShape& s) {
  const int threads = solver_generic_threads(s);
  cudaError_t e = cudaFuncSetAttribute(power_generic_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)power_generic_smem(s, threads));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(pipg_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)pipg_generic_smem(s, threads));
}

cudaError_t launch_power_generic(const PowerArgs& a, cudaStream_t stream) {
  const int threads = solver_generic_threads(a.shape);
  power_generic_kernel<<<a.batch, threads, power_generic_smem(a.shape, threads), stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pipg_generic(const PipgArgs& a, cudaStream_t stream) {
  const int threads = solver_generic_threads(a.shape);
  pipg_generic_kernel<<<a.batch, threads, pipg_generic_smem(a.shape, threads), stream>>>(a);
  return cudaGetLastError();
}

}  // namespace ptopt_b200
