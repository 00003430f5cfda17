// mc_kernels.cu — the steps either side of scp_solve inside mc::solve_instance, on the device:
// instance generation (disperse + run_seed + initial_guess), the dense violation audit of the
// solved trajectory, and the per-instance RunRecord.
//
// Follows /root/reference/proj/include/ptopt/montecarlo.hpp:35-65 (counter-based draws,
// run_seed, disperse), :100-135 (solve_instance), /root/reference/proj/include/ptopt/
// rocket_problem.hpp:127-163 (initial_guess) and /root/reference/proj/include/ptopt/
// discretizer.hpp:153-187 (propagate_state), :249-285 (dense_violation_audit).
#include "kernels.cuh"

namespace ptopt_b200 {

namespace {

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {  // montecarlo.hpp:35-40
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/// (1-t)*a + t*b with every operation rounded separately, as the reference's non-contracted
/// build evaluates it: instance generation is bit-exact.
__device__ __forceinline__ double lerp_rn(double t, double a, double b) {
  return __dadd_rn(__dmul_rn(1.0 - t, a), __dmul_rn(t, b));
}

__global__ void generate_kernel(GenerateArgs a) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)a.batch * a.nodes) return;
  const int b = (int)(idx / a.nodes), k = (int)(idx - (long long)b * a.nodes);
  const unsigned long long run = (unsigned long long)(a.first_run_id + b);

  // disperse, montecarlo.hpp:43-65: only the initial position is drawn
  double init[kNXI];
#pragma unroll
  for (int i = 0; i < kNXI; ++i) init[i] = a.nominal[i];
  const unsigned long long key = mix64(a.seed ^ mix64(run + 1ull));
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double u = (double)(mix64(key + (unsigned long long)i) >> 11) * 0x1.0p-53;
    init[1 + i] = __dadd_rn(a.r_low[i], __dmul_rn(a.r_high[i] - a.r_low[i], u));
  }
  if (k == 0) {
    double* o = a.init_state + (size_t)b * kNXI;
#pragma unroll
    for (int i = 0; i < kNXI; ++i) o[i] = init[i];
    a.rng_seed[b] = mix64(a.seed ^ mix64(run));  // run_seed, montecarlo.hpp:51-53
  }

  // initial_guess, rocket_problem.hpp:127-163.  m_end and the slerp table depend only on the
  // nominal boundary and were evaluated on the host with the C library (exp, acos, sin).
  const double t = a.tau[k];
  double* x = a.x_guess + ((size_t)b * a.nodes + k) * kNX;
  double* u = a.u_guess + ((size_t)b * a.nodes + k) * kNU;
  const double sm = lerp_rn(t, init[0], a.m_end);
  x[0] = sm;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    x[1 + i] = lerp_rn(t, init[1 + i], a.fin[1 + i]);
    x[4 + i] = lerp_rn(t, init[4 + i], a.fin[4 + i]);
    x[11 + i] = lerp_rn(t, init[11 + i], a.fin[11 + i]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) x[7 + i] = a.qtab[k * 4 + i];
  x[kNX - 1] = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    u[i] = __dmul_rn(-sm, a.g[i]);
    u[3 + i] = 0.0;
  }
  u[kNU - 1] = a.t_f_guess;
}

/// The nine path inequalities g(xi, zeta) (rocket6dof.hpp:278-301).  Never fails.
__device__ __forceinline__ void eval_constraints(const ModelConst& P, const double* x,
                                                 const double* u, double* g) {
  const double T0 = u[0], T1 = u[1], T2 = u[2];
  const double Tn = sqrt(T0 * T0 + T1 * T1 + T2 * T2);
  const double q0 = x[7], q1 = x[8], q2 = x[9], qw = x[10];
  const double hq0 = P.H[0] * q0 + P.H[1] * q1 + P.H[2] * q2 + P.H[3] * qw;
  const double hq1 = P.H[4] * q0 + P.H[5] * q1 + P.H[6] * q2 + P.H[7] * qw;
  g[0] = P.m_dry - x[0];
  g[1] = -x[1];
  g[2] = x[4] * x[4] + x[5] * x[5] + x[6] * x[6] - P.v_max_sq;
  g[3] = 4.0 * (hq0 * hq0 + hq1 * hq1) - P.c_theta_sq;
  g[4] = x[11] * x[11] + x[12] * x[12] + x[13] * x[13] - P.w_max_sq;
  g[5] = Tn - T0 * P.sec_delta;
  g[6] = Tn - P.T_max;
  g[7] = -Tn + P.T_min;
  g[8] = u[3] * u[3] + u[4] * u[4] + u[5] * u[5] - P.gamma_max_sq;
}

/// Augmented rate f = s * (F, sum g+^2) at (x, u) (ctcs.hpp:47-74; rocket6dof.hpp:245-274).
/// Status codes as the reference throws: dilation (ctcs.hpp:66), mass (rocket6dof.hpp:246).
__device__ __forceinline__ int eval_rate(const ModelConst& P, const double* x, const double* u,
                                         double* f) {
  const double s = u[6], m = x[0];
  if (!(s > 0.0)) return kStDilation;
  if (!(m > 0.0)) return kStMass;
  const double T0 = u[0], T1 = u[1], T2 = u[2];
  const double Tn = sqrt(T0 * T0 + T1 * T1 + T2 * T2);
  const double q0 = x[7], q1 = x[8], q2 = x[9], qw = x[10];
  const double w0 = x[11], w1 = x[12], w2 = x[13];
  const double ss = q0 * q0 + q1 * q1 + q2 * q2;
  const double d = qw * qw - ss;
  double C[9];
  C[0] = d + 2.0 * q0 * q0;
  C[1] = 2.0 * q0 * q1 + 2.0 * qw * (-q2);
  C[2] = 2.0 * q0 * q2 + 2.0 * qw * q1;
  C[3] = 2.0 * q1 * q0 + 2.0 * qw * q2;
  C[4] = d + 2.0 * q1 * q1;
  C[5] = 2.0 * q1 * q2 + 2.0 * qw * (-q0);
  C[6] = 2.0 * q2 * q0 + 2.0 * qw * (-q1);
  C[7] = 2.0 * q2 * q1 + 2.0 * qw * q0;
  C[8] = d + 2.0 * q2 * q2;
  double F[kNXI];
  F[0] = -P.alpha * Tn;
  F[1] = x[4];
  F[2] = x[5];
  F[3] = x[6];
#pragma unroll
  for (int i = 0; i < 3; ++i)
    F[4 + i] = (C[i * 3] * T0 + C[i * 3 + 1] * T1 + C[i * 3 + 2] * T2) / m + P.g[i];
  F[7] = 0.5 * (qw * w0 + (q1 * w2 - q2 * w1));
  F[8] = 0.5 * (qw * w1 + (q2 * w0 - q0 * w2));
  F[9] = 0.5 * (qw * w2 + (q0 * w1 - q1 * w0));
  F[10] = -0.5 * (q0 * w0 + q1 * w1 + q2 * w2);
  double Jw[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) Jw[i] = P.J[i * 3] * w0 + P.J[i * 3 + 1] * w1 + P.J[i * 3 + 2] * w2;
  const double t0 = (P.rT[1] * T2 - P.rT[2] * T1) - (w1 * Jw[2] - w2 * Jw[1]) + u[3];
  const double t1 = (P.rT[2] * T0 - P.rT[0] * T2) - (w2 * Jw[0] - w0 * Jw[2]) + u[4];
  const double t2 = (P.rT[0] * T1 - P.rT[1] * T0) - (w0 * Jw[1] - w1 * Jw[0]) + u[5];
#pragma unroll
  for (int i = 0; i < 3; ++i)
    F[11 + i] = P.Jinv[i * 3] * t0 + P.Jinv[i * 3 + 1] * t1 + P.Jinv[i * 3 + 2] * t2;
  double g[9];
  eval_constraints(P, x, u, g);
  double integrand = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const double v = g[i] > 0.0 ? g[i] : 0.0;
    integrand += v * v;
  }
#pragma unroll
  for (int i = 0; i < kNXI; ++i) f[i] = s * F[i];
  f[kNX - 1] = s * integrand;
  return kStOk;
}

/// One thread per (instance, interval): propagate_state with the sample callback of
/// dense_violation_audit (discretizer.hpp:153-187, 262-283).
__global__ void __launch_bounds__(128) audit_kernel(AuditArgs a) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int M = a.nodes - 1;
  if (idx >= (long long)a.batch * M) return;
  const int b = (int)(idx / M), k = (int)(idx - (long long)b * M);
  if (a.skip && a.skip[b] != 0) return;  // the solve of this instance failed: nothing to audit
  const double* xk = a.x + ((size_t)b * a.nodes + k) * kNX;
  const double* uk = a.u + ((size_t)b * a.nodes + k) * kNU;
  const double tau_k = a.tau[k], tau_k1 = a.tau[k + 1];
  const double span = tau_k1 - tau_k;
  const double h = span / a.substeps;
  double x[kNX], u0[kNU], u1[kNU];
#pragma unroll
  for (int i = 0; i < kNX; ++i) x[i] = xk[i];
#pragma unroll
  for (int i = 0; i < kNU; ++i) {
    u0[i] = uk[i];
    u1[i] = uk[kNU + i];
  }
  const double y0 = x[kNX - 1];
  double gmax = -INFINITY;
  int rc = kStOk;
  double f[kNX], g[9], acc[kNX], tmp[kNX], uu[kNU];
  auto interp = [&](double tau) {  // foh_interp, discretizer.hpp:26-39
    const double lr = (tau - tau_k) / span, ll = (tau_k1 - tau) / span;
#pragma unroll
    for (int i = 0; i < kNU; ++i) uu[i] = ll * u0[i] + lr * u1[i];
  };
  // AuditSample records of this interval (discretizer.hpp:236-240), when the caller wants them
  double* sample = a.samples ? a.samples + (size_t)idx * (a.substeps + 1) * kAuditSampleDoubles : nullptr;
  auto record = [&](double tau, const double* xs) {  // sample callback, discretizer.hpp:262-276
    interp(tau);
    eval_constraints(a.model, xs, uu, g);
    double gs = -INFINITY;
#pragma unroll
    for (int i = 0; i < 9; ++i) gs = fmax(gs, g[i]);
    gmax = fmax(gmax, gs);
    if (sample) {
      sample[0] = (double)k;
      sample[1] = tau;
#pragma unroll
      for (int i = 0; i < 9; ++i) sample[2 + i] = g[i];
      sample[11] = gs;
      sample += kAuditSampleDoubles;
    }
  };
  record(tau_k, x);
  for (int step = 0; step < a.substeps && rc == kStOk; ++step) {
    const double t0 = tau_k + h * step;
    const double t_end = (step + 1 == a.substeps) ? tau_k1 : t0 + h;
    interp(t0);
    rc = eval_rate(a.model, x, uu, f);
    if (rc != kStOk) break;
#pragma unroll
    for (int i = 0; i < kNX; ++i) {
      acc[i] = x[i] + (h / 6.0) * f[i];
      tmp[i] = x[i] + (0.5 * h) * f[i];
    }
    interp(t0 + 0.5 * h);
    rc = eval_rate(a.model, tmp, uu, f);
    if (rc != kStOk) break;
#pragma unroll
    for (int i = 0; i < kNX; ++i) {
      acc[i] += (h / 3.0) * f[i];
      tmp[i] = x[i] + (0.5 * h) * f[i];
    }
    rc = eval_rate(a.model, tmp, uu, f);
    if (rc != kStOk) break;
#pragma unroll
    for (int i = 0; i < kNX; ++i) {
      acc[i] += (h / 3.0) * f[i];
      tmp[i] = x[i] + h * f[i];
    }
    interp(t_end);
    rc = eval_rate(a.model, tmp, uu, f);
    if (rc != kStOk) break;
#pragma unroll
    for (int i = 0; i < kNX; ++i) x[i] = acc[i] + (h / 6.0) * f[i];
    record(t_end, x);
  }
  if (rc != kStOk) {
    atomicMin(&a.fail_key[b], (k << 4) | rc);
    return;
  }
  a.interval_g_max[(size_t)b * M + k] = gmax;
  a.interval_y_increase[(size_t)b * M + k] = x[kNX - 1] - y0;
}

/// max over the intervals of an instance, in interval order (AuditResult::max_pointwise_g).
__global__ void audit_reduce_kernel(AuditArgs a, double* max_pointwise_g, int* status,
                                    int* fail_index) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.batch) return;
  const int M = a.nodes - 1;
  const int key = a.fail_key[b];
  if (a.skip && a.skip[b] != 0) {
    if (max_pointwise_g) max_pointwise_g[b] = 0.0;
    return;  // status stays the solve's
  }
  if (key != kFailKeyNone) {
    if (status) status[b] = key & 15;
    if (fail_index) fail_index[b] = key >> 4;
    if (max_pointwise_g) max_pointwise_g[b] = 0.0;
    return;
  }
  double gmax = -INFINITY;
  for (int k = 0; k < M; ++k) gmax = fmax(gmax, a.interval_g_max[(size_t)b * M + k]);
  if (max_pointwise_g) max_pointwise_g[b] = gmax;
}

/// RunRecord of every instance (montecarlo.hpp:100-135).
__global__ void records_kernel(RecordArgs a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.batch) return;
  RunRecordDev r;
  r.run_id = (int)(a.first_run_id + b);
  r.status = a.status[b];
  r.fail_index = a.fail_index[b];
  r.reserved_ = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i) r.initial_position[i] = a.init_state[(size_t)b * kNXI + 1 + i];
  // montecarlo.hpp:115-132: a throw inside scp_solve leaves the record at its defaults; a throw
  // inside the dense audit comes after scp_iterations, final_defect_inf and propellant_used were
  // assigned, so those stay and only `converged` is cleared.
  const bool audit_failed = r.status != kStOk && a.audit_fail_key && a.audit_fail_key[b] != kFailKeyNone;
  r.converged = 0;
  r.scp_iterations = 0;
  r.propellant_used = r.final_defect_inf = r.max_pointwise_g = r.max_node_y_increase = 0.0;
  if (r.status == kStOk || audit_failed) {
    const double* x = a.x + (size_t)b * a.nodes * kNX;
    r.scp_iterations = a.scp_iterations[b];
    r.final_defect_inf = a.final_defect[b];
    r.propellant_used = a.init_state[(size_t)b * kNXI] - x[(size_t)(a.nodes - 1) * kNX];
    if (!audit_failed) {
      r.converged = a.converged[b] ? 1 : 0;
      r.max_pointwise_g = a.max_pointwise_g[b];
      double dy_max = 0.0;
      for (int k = 0; k + 1 < a.nodes; ++k)
        dy_max = fmax(dy_max, x[(size_t)(k + 1) * kNX + kNX - 1] - x[(size_t)k * kNX + kNX - 1]);
      r.max_node_y_increase = dy_max;
    }
  }
  a.records[b] = r;
}

}  // namespace

void launch_generate(const GenerateArgs& a, cudaStream_t stream) {
  const long long total = (long long)a.batch * a.nodes;
  generate_kernel<<<(unsigned)((total + 127) / 128), 128, 0, stream>>>(a);
}

void launch_audit(const AuditArgs& a, double* max_pointwise_g, int* status, int* fail_index,
                  cudaStream_t stream) {
  const long long total = (long long)a.batch * (a.nodes - 1);
  audit_kernel<<<(unsigned)((total + 127) / 128), 128, 0, stream>>>(a);
  audit_reduce_kernel<<<(a.batch + 127) / 128, 128, 0, stream>>>(a, max_pointwise_g, status,
                                                                   fail_index);
}

void launch_records(const RecordArgs& a, cudaStream_t stream) {
  records_kernel<<<(a.batch + 127) / 128, 128, 0, stream>>>(a);
}

}  // namespace ptopt_b200
