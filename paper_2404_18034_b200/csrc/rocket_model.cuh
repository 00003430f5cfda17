// rocket_model.cuh — 6-DoF vehicle + CTCS augmentation evaluated in registers, and the two passes
// of the exact discretization (propagate_interval,
// /root/reference/proj/include/ptopt/discretizer.hpp:82-149).
//
// The state part of the RK4 bundle does not depend on the sensitivity columns.  The state pass
// (one thread per interval) therefore evaluates the model, its constraints and the Jacobian
// scalars (rocket6dof.hpp:245-402 through ctcs.hpp:47-129) once per stage and packs what the
// columns need into an 84-double stage record.  The column pass (one warp per interval, lane
// j < 29 owns column j of [Phi_x (15) | Phi_u- (7) | Phi_u+ (7)]) applies A(tau) and the B
// forcing from the record.  The Jacobian is applied in its structural sparsity: skipped entries
// are exact zeros in the reference's dense product, so results agree with the dense loops up to
// FMA contraction.
//
// Everything here is `__host__ __device__` so tests/sim can run the same code on the CPU.
#pragma once

#include <math.h>

#if defined(__CUDACC__)
#define PT_HD __host__ __device__ __forceinline__
#else
#define PT_HD inline
#endif

namespace ptopt_b200 {

constexpr int kNX = 15;
constexpr int kNU = 7;
constexpr int kNXI = 14;
constexpr int kCols = kNX + 2 * kNU;  // 29 sensitivity columns

// per-instance status codes (mirror ptopt_instance_status in include/ptopt_cuda.h)
constexpr int kStOk = 0;
constexpr int kStPropDiverged = 1;
constexpr int kStSolverDiverged = 2;
constexpr int kStDilation = 3;
constexpr int kStMass = 4;
constexpr int kStThrust = 5;
constexpr int kStSeedZero = 6;

/// Vehicle constants with everything that does not depend on the state folded on the host
/// (VehicleParams, rocket6dof.hpp:85-99; inverse3 :210-224; the cos() terms of :282, :292).
struct ModelConst {
  double alpha;
  double g[3];
  double J[9];
  double Jinv[9];
  double JinvR[9];  // Jinv * skew(r_thrust)  (rocket6dof.hpp:370-375)
  double rT[3];
  double H[8];
  double m_dry;
  double v_max_sq;
  double c_theta_sq;  // (1 - cos(theta_max))^2
  double w_max_sq;
  double sec_delta;
  double T_max;
  double T_min;
  double gamma_max_sq;
};

PT_HD bool pt_finite(double v) { return fabs(v) <= 1.79769313486231570e308; }

// ---------------------------------------------------------------------------------------------
// Stage records.  The state part of the RK4 bundle does not depend on the sensitivity columns, so
// the model is evaluated once per (interval, stage) by the state pass, which leaves everything
// the 29 column lanes need in a compact record; the column pass applies A(tau) and the B forcing
// from it.  (Evaluating the model in every column lane, as a one-pass kernel does, spends 70 % of
// the FP64 instructions on 32 identical copies of the evaluation.)
// ---------------------------------------------------------------------------------------------
constexpr int kRecS = 0;        // dilation factor
constexpr int kRecSvm = 1;      // [3]  A[v_i][m]
constexpr int kRecSvq = 4;      // [12] A[v_i][q_j]
constexpr int kRecHw = 16;      // [3]  s * 0.5 * w_k
constexpr int kRecGq = 19;      // [4]  s * 0.5 * q_k
constexpr int kRecSww = 23;     // [9]  A[w_i][w_j]
constexpr int kRecAy = 32;      // [15] row y of A (zeros unless active)
constexpr int kRecActive = 47;  // 1.0 when a path inequality is violated
constexpr int kRecBT = 48;      // [3][5] thrust columns of B: rows 0, 4, 5, 6, 14
constexpr int kRecBG = 63;      // [3] torque columns of B: row 14
constexpr int kRecBS = 66;      // [15] dilation column of B
constexpr int kRecSize = 84;    // padded to a whole number of 32-byte sectors per tile of four intervals
constexpr int kRecLamLeft = 81;   // spare record slots: the first-order-hold factors of the stage
constexpr int kRecLamRight = 82;  //   (written after the padding zeros)
static_assert(kRecBS + kNX <= kRecLamLeft && kRecLamRight < kRecSize, "record padding");

/// Evaluates one RK4 stage at augmented state x and control u: the augmented rate f[15] =
/// s * (F, sum g+^2) for the state update, and — through EMIT(field, value), every field of the
/// stage record exactly once, each as soon as it is known so that nothing stays live for the
/// record's sake — the scalars that define the nonzeros of A = df/dx and the nonzero rows of the
/// seven columns of B = df/du (ctcs.hpp:96-128; rocket6dof.hpp:333-334, 370-380, 393-400).
/// Returns a status code in the reference's throw order: dilation (ctcs.hpp:66), mass
/// (rocket6dof.hpp:246), thrust (:306); nothing has been emitted when it is not kStOk.
template <class EmitFn>
PT_HD int eval_stage_emit(const ModelConst& P, const double* x, const double* u, double* f, EmitFn EMIT) {
  const double s = u[6];
  const double m = x[0];
  const double T0 = u[0], T1 = u[1], T2 = u[2];
  if (!(s > 0.0)) return kStDilation;
  if (!(m > 0.0)) return kStMass;
  const double Tn = sqrt(T0 * T0 + T1 * T1 + T2 * T2);
  if (Tn < 1e-9) return kStThrust;
  EMIT(kRecS, s);
  const double rm = 1.0 / m;
  const double rTn = 1.0 / Tn;
  const double q0 = x[7], q1 = x[8], q2 = x[9], qw = x[10];
  const double w0 = x[11], w1 = x[12], w2 = x[13];

  // dcm, rocket6dof.hpp:176-188
  double C[9];
  {
    const double ss = q0 * q0 + q1 * q1 + q2 * q2;
    const double d = qw * qw - ss;
    C[0] = d + 2.0 * q0 * q0;
    C[1] = 2.0 * q0 * q1 + 2.0 * qw * (-q2);
    C[2] = 2.0 * q0 * q2 + 2.0 * qw * q1;
    C[3] = 2.0 * q1 * q0 + 2.0 * qw * q2;
    C[4] = d + 2.0 * q1 * q1;
    C[5] = 2.0 * q1 * q2 + 2.0 * qw * (-q0);
    C[6] = 2.0 * q2 * q0 + 2.0 * qw * (-q1);
    C[7] = 2.0 * q2 * q1 + 2.0 * qw * q0;
    C[8] = d + 2.0 * q2 * q2;
  }
  double CT[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) CT[i] = C[i * 3] * T0 + C[i * 3 + 1] * T1 + C[i * 3 + 2] * T2;

  // eval_dynamics, rocket6dof.hpp:245-274
  double F[kNXI];
  F[0] = -P.alpha * Tn;
  F[1] = x[4];
  F[2] = x[5];
  F[3] = x[6];
#pragma unroll
  for (int i = 0; i < 3; ++i) F[4 + i] = CT[i] * rm + P.g[i];
  F[7] = 0.5 * (qw * w0 + (q1 * w2 - q2 * w1));
  F[8] = 0.5 * (qw * w1 + (q2 * w0 - q0 * w2));
  F[9] = 0.5 * (qw * w2 + (q0 * w1 - q1 * w0));
  F[10] = -0.5 * (q0 * w0 + q1 * w1 + q2 * w2);
  double Jw[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) Jw[i] = P.J[i * 3] * w0 + P.J[i * 3 + 1] * w1 + P.J[i * 3 + 2] * w2;
  {
    const double lev0 = P.rT[1] * T2 - P.rT[2] * T1;
    const double lev1 = P.rT[2] * T0 - P.rT[0] * T2;
    const double lev2 = P.rT[0] * T1 - P.rT[1] * T0;
    const double gy0 = w1 * Jw[2] - w2 * Jw[1];
    const double gy1 = w2 * Jw[0] - w0 * Jw[2];
    const double gy2 = w0 * Jw[1] - w1 * Jw[0];
    const double t0 = lev0 - gy0 + u[3], t1 = lev1 - gy1 + u[4], t2 = lev2 - gy2 + u[5];
#pragma unroll
    for (int i = 0; i < 3; ++i)
      F[11 + i] = P.Jinv[i * 3] * t0 + P.Jinv[i * 3 + 1] * t1 + P.Jinv[i * 3 + 2] * t2;
  }

  // eval_constraints, rocket6dof.hpp:278-301, clipped as in ctcs.hpp:47-56
  const double hq0 = P.H[0] * q0 + P.H[1] * q1 + P.H[2] * q2 + P.H[3] * qw;
  const double hq1 = P.H[4] * q0 + P.H[5] * q1 + P.H[6] * q2 + P.H[7] * qw;
  double g[9], gp[9];
  g[0] = P.m_dry - m;
  g[1] = -x[1];
  g[2] = x[4] * x[4] + x[5] * x[5] + x[6] * x[6] - P.v_max_sq;
  g[3] = 4.0 * (hq0 * hq0 + hq1 * hq1) - P.c_theta_sq;
  g[4] = w0 * w0 + w1 * w1 + w2 * w2 - P.w_max_sq;
  g[5] = Tn - T0 * P.sec_delta;
  g[6] = Tn - P.T_max;
  g[7] = -Tn + P.T_min;
  g[8] = u[3] * u[3] + u[4] * u[4] + u[5] * u[5] - P.gamma_max_sq;
  double integrand = 0.0;
  bool active = false;
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const double v = g[i] > 0.0 ? g[i] : 0.0;
    gp[i] = v;
    integrand += v * v;
    active = active || (v > 0.0);
  }
#pragma unroll
  for (int i = 0; i < kNXI; ++i) f[i] = s * F[i];
  f[14] = s * integrand;
  // dilation column of B: the undilated rate (ctcs.hpp:99)
#pragma unroll
  for (int i = 0; i < kNXI; ++i) EMIT(kRecBS + i, F[i]);
  EMIT(kRecBS + kNXI, integrand);

  // nonzeros of A = s * dF/dxi (rocket6dof.hpp:325-369 through ctcs.hpp:96-97)
  const double rm2 = rm * rm;
#pragma unroll
  for (int i = 0; i < 3; ++i) EMIT(kRecSvm + i, s * (-CT[i] * rm2));
  {
    // dcm_times_vec_jac, rocket6dof.hpp:191-207, divided by m
    const double qT = q0 * T0 + q1 * T1 + q2 * T2;
    const double qv[3] = {q0, q1, q2};
    const double T[3] = {T0, T1, T2};
    const double Tk[9] = {0.0, -T2, T1, T2, 0.0, -T0, -T1, T0, 0.0};
    const double qxT[3] = {q1 * T2 - q2 * T1, q2 * T0 - q0 * T2, q0 * T1 - q1 * T0};
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double v = -2.0 * T[i] * qv[j] + 2.0 * qv[i] * T[j] - 2.0 * qw * Tk[i * 3 + j];
        if (i == j) v += 2.0 * qT;
        EMIT(kRecSvq + i * 4 + j, s * (v * rm));
      }
      EMIT(kRecSvq + i * 4 + 3, s * ((2.0 * qw * T[i] + 2.0 * qxT[i]) * rm));
    }
  }
  EMIT(kRecHw + 0, s * (0.5 * w0));
  EMIT(kRecHw + 1, s * (0.5 * w1));
  EMIT(kRecHw + 2, s * (0.5 * w2));
  EMIT(kRecGq + 0, s * (0.5 * q0));
  EMIT(kRecGq + 1, s * (0.5 * q1));
  EMIT(kRecGq + 2, s * (0.5 * q2));
  EMIT(kRecGq + 3, s * (0.5 * qw));
  {
    // dw/dw = Jinv * ([Jw]x - [w]x J), rocket6dof.hpp:352-369
    const double JWk[9] = {0.0, -Jw[2], Jw[1], Jw[2], 0.0, -Jw[0], -Jw[1], Jw[0], 0.0};
    const double Wk[9] = {0.0, -w2, w1, w2, 0.0, -w0, -w1, w0, 0.0};
    double M[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double acc = JWk[i * 3 + j];
#pragma unroll
        for (int k = 0; k < 3; ++k) acc -= Wk[i * 3 + k] * P.J[k * 3 + j];
        M[i * 3 + j] = acc;
      }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) acc += P.Jinv[i * 3 + k] * M[k * 3 + j];
        EMIT(kRecSww + i * 3 + j, s * acc);
      }
  }
  // row y of A: 2 s g+ dg/dxi (ctcs.hpp:108-115 with rocket6dof.hpp:383-391); zeros unless a
  // path inequality is violated
  {
    double ay[kNX];
#pragma unroll
    for (int i = 0; i < kNX; ++i) ay[i] = 0.0;
    if (active) {
      const double s2 = 2.0 * s;
      ay[0] = s2 * gp[0] * -1.0;
      ay[1] = s2 * gp[1] * -1.0;
      ay[4] = s2 * gp[2] * (2.0 * x[4]);
      ay[5] = s2 * gp[2] * (2.0 * x[5]);
      ay[6] = s2 * gp[2] * (2.0 * x[6]);
#pragma unroll
      for (int j = 0; j < 4; ++j) ay[7 + j] = s2 * gp[3] * (8.0 * (hq0 * P.H[j] + hq1 * P.H[4 + j]));
      ay[11] = s2 * gp[4] * (2.0 * w0);
      ay[12] = s2 * gp[4] * (2.0 * w1);
      ay[13] = s2 * gp[4] * (2.0 * w2);
    }
#pragma unroll
    for (int i = 0; i < kNX; ++i) EMIT(kRecAy + i, ay[i]);
    EMIT(kRecActive, active ? 1.0 : 0.0);
  }
  // thrust columns of B: rows 0, 4..6, 14 (rows 11..13 are s * Jinv R: a constant times s)
#pragma unroll
  for (int jc = 0; jc < 3; ++jc) {
    const double Tj = jc == 0 ? T0 : (jc == 1 ? T1 : T2);
    const double that = Tj * rTn;
    EMIT(kRecBT + 5 * jc, s * (-P.alpha * that));
#pragma unroll
    for (int i = 0; i < 3; ++i) EMIT(kRecBT + 5 * jc + 1 + i, s * (C[i * 3 + jc] * rm));
    double by = 0.0;
    if (active) {
      const double s2 = 2.0 * s;
      double acc = 0.0;
      acc += s2 * gp[5] * (that - (jc == 0 ? P.sec_delta : 0.0));
      acc += s2 * gp[6] * that;
      acc += s2 * gp[7] * (-that);
      by = acc;
    }
    EMIT(kRecBT + 5 * jc + 4, by);
  }
  // torque columns of B: row 14 (rows 11..13 are s * Jinv)
#pragma unroll
  for (int j = 0; j < 3; ++j) EMIT(kRecBG + j, active ? 2.0 * s * gp[8] * (2.0 * u[3 + j]) : 0.0);
#pragma unroll
  for (int i = kRecBS + kNX; i < kRecSize; ++i) EMIT(i, 0.0);
  return kStOk;
}

/// d = A * c in the structural sparsity of A (ascending column order inside every row, as
/// mat_mat does: smallmat.hpp:115-120), A taken from a stage record.
PT_HD void apply_A(const double* rec, const double* c, double* d) {
  const double s = rec[kRecS];
  const double* svm = rec + kRecSvm;
  const double* svq = rec + kRecSvq;
  const double* sww = rec + kRecSww;
  d[0] = 0.0;
  d[1] = s * c[4];
  d[2] = s * c[5];
  d[3] = s * c[6];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double acc = svm[i] * c[0];
#pragma unroll
    for (int j = 0; j < 4; ++j) acc += svq[i * 4 + j] * c[7 + j];
    d[4 + i] = acc;
  }
  const double* h = rec + kRecHw;
  const double* g = rec + kRecGq;
  d[7] = h[2] * c[8] - h[1] * c[9] + h[0] * c[10] + g[3] * c[11] - g[2] * c[12] + g[1] * c[13];
  d[8] = -h[2] * c[7] + h[0] * c[9] + h[1] * c[10] + g[2] * c[11] + g[3] * c[12] - g[0] * c[13];
  d[9] = h[1] * c[7] - h[0] * c[8] + h[2] * c[10] - g[1] * c[11] + g[0] * c[12] + g[3] * c[13];
  d[10] = -h[0] * c[7] - h[1] * c[8] - h[2] * c[9] - g[0] * c[11] - g[1] * c[12] - g[2] * c[13];
#pragma unroll
  for (int i = 0; i < 3; ++i)
    d[11 + i] = sww[i * 3] * c[11] + sww[i * 3 + 1] * c[12] + sww[i * 3 + 2] * c[13];
  double dy = 0.0;
  if (rec[kRecActive] != 0.0) {
    const double* ay = rec + kRecAy;
#pragma unroll
    for (int k = 0; k < kNXI; ++k) dy += ay[k] * c[k];
  }
  d[14] = dy;
}

/// Stage time, RK4 weights and first-order-hold factors of stage `stage` of step `step`
/// (discretizer.hpp:26-39, 118-135): shared by the state and the column pass.
struct StageTime {
  double wk, wn, lam_left, lam_right;
};
PT_HD StageTime stage_time(double tau_k, double tau_k1, int steps, int step, int stage) {
  const double span = tau_k1 - tau_k;
  const double h = span / steps;
  const double t0 = tau_k + h * step;
  const double t_end = (step + 1 == steps) ? tau_k1 : t0 + h;
  const double tau = stage == 0 ? t0 : (stage == 3 ? t_end : t0 + 0.5 * h);
  StageTime t;
  t.wk = (stage == 0 || stage == 3) ? h / 6.0 : h / 3.0;  // RK4 weight
  t.wn = stage == 2 ? h : 0.5 * h;                         // next-stage offset
  t.lam_right = (tau - tau_k) / span;
  t.lam_left = (tau_k1 - tau) / span;
  return t;
}

/// State pass of one interval (the x part of propagate_interval, discretizer.hpp:82-141):
/// 4 * steps model evaluations; EMIT(stage_number, field, value) receives every field of every
/// stage record.  On success x_end[15] holds the propagated state.
template <class EmitFn>
PT_HD int propagate_state_pass(const ModelConst& P, const double* xk, const double* uk, const double* uk1,
                               double tau_k, double tau_k1, int steps, double* x_end, EmitFn EMIT) {
  // all_finite(x_k), discretizer.hpp:89
  bool fin = true;
#pragma unroll
  for (int i = 0; i < kNX; ++i) fin = fin && pt_finite(xk[i]);
  if (!fin) return kStPropDiverged;
  double sx[kNX], ax[kNX], xin[kNX];
#pragma unroll
  for (int i = 0; i < kNX; ++i) sx[i] = xin[i] = ax[i] = xk[i];
  for (int step = 0; step < steps; ++step) {
#pragma unroll 1
    for (int stage = 0; stage < 4; ++stage) {
      const StageTime t = stage_time(tau_k, tau_k1, steps, step, stage);
      double u[kNU];
#pragma unroll
      for (int i = 0; i < kNU; ++i) u[i] = t.lam_left * uk[i] + t.lam_right * uk1[i];
      double f[kNX];
      const int stage_no = step * 4 + stage;
      const int rc = eval_stage_emit(P, xin, u, f, [&](int field, double v) { EMIT(stage_no, field, v); });
      if (rc != kStOk) return rc;
      EMIT(stage_no, kRecLamLeft, t.lam_left);  // spare record slots: the first-order-hold factors
      EMIT(stage_no, kRecLamRight, t.lam_right);
#pragma unroll
      for (int i = 0; i < kNX; ++i) {
        const double axi = (stage == 0 ? sx[i] : ax[i]) + t.wk * f[i];
        xin[i] = stage == 3 ? axi : sx[i] + t.wn * f[i];
        ax[i] = axi;
        if (stage == 3) sx[i] = axi;
      }
    }
    // all_finite(s.x) after every RK4 step, discretizer.hpp:136
    fin = true;
#pragma unroll
    for (int i = 0; i < kNX; ++i) fin = fin && pt_finite(xin[i]);
    if (!fin) return kStPropDiverged;
  }
#pragma unroll
  for (int i = 0; i < kNX; ++i) x_end[i] = xin[i];
  return kStOk;
}

/// Per-lane state of the column pass: sensitivity column `lane` of [Phi_x | Phi_u- | Phi_u+].
struct ColumnLane {
  double s_c[kNX], a_c[kNX], c[kNX];  // step start, RK4 combination, stage input
};
PT_HD void column_init(ColumnLane& L, int lane) {
#pragma unroll
  for (int i = 0; i < kNX; ++i) {
    L.s_c[i] = (i == lane) ? 1.0 : 0.0;  // Phi_x(0) = I, Phi_u(0) = 0 (discretizer.hpp:94-96)
    L.a_c[i] = L.c[i] = L.s_c[i];
  }
}

// ---------------------------------------------------------------------------------------------
// Stage slabs.  The column pass does not read a stage record as the state pass wrote it: while it
// moves the record into shared memory it scatters the B entries into a DENSE 15 x 8 array (column 7
// and every entry the record does not carry stay zero), so that every lane applies "its" column of
// B with the same fifteen multiply-adds — no branch on the kind of column (thrust / torque /
// dilation / none), which a warp whose lanes own different kinds would execute one after the other.
// The entries s * Jinv R and s * Jinv of the thrust and torque columns (rows 11..13) are the
// dilation factor times a constant: each lane keeps its three constants in registers instead.
// ---------------------------------------------------------------------------------------------
constexpr int kSlabB = 48;                  // dense B: entry (row i, control j) at kSlabB + 8 i + j
constexpr int kSlabLamLeft = kSlabB + 120;  // first-order-hold factors of the stage
constexpr int kSlabLamRight = kSlabLamLeft + 1;
constexpr int kSlabSize = kSlabLamRight + 3;  // 172: a multiple of two doubles (16-byte aligned slabs)
constexpr int kSlabZero = kSlabB + 7;         // an entry that is always zero (pad column, row 0)

/// Where field `f` of a stage record goes inside a slab.
PT_HD constexpr int slab_dest(int f) {
  if (f < kRecBT) return f;  // A scalars, row y, the active flag: same place
  if (f < kRecBG) {          // thrust columns: rows 0, 4, 5, 6, 14
    const int jc = (f - kRecBT) / 5, r = (f - kRecBT) % 5;
    const int row = r == 0 ? 0 : (r == 4 ? 14 : 3 + r);
    return kSlabB + 8 * row + jc;
  }
  if (f < kRecBS) return kSlabB + 8 * 14 + 3 + (f - kRecBG);  // torque columns: row 14
  if (f < kRecBS + kNX) return kSlabB + 8 * (f - kRecBS) + 6;  // dilation column
  if (f == kRecLamLeft) return kSlabLamLeft;
  if (f == kRecLamRight) return kSlabLamRight;
  return kSlabSize - 1;  // record padding
}

/// What a lane keeps next to its column: where its B column and its first-order-hold factor are
/// inside a slab, and s-proportional entries of rows 11..13 (thrust: Jinv R, torque: Jinv).
struct ColumnForcing {
  bool forced;   // the lane owns a column of Phi_u- / Phi_u+
  int bcol;      // slab index of row 0 of the lane's B column
  int lam;       // slab index of its first-order-hold factor
  double jr[3];
};
PT_HD void forcing_init(const ModelConst& P, int lane, ColumnForcing& Fc) {
  const bool forced = lane >= kNX && lane < kCols;
  const int jc = forced ? (lane - kNX) % kNU : 7;
  Fc.forced = forced;
  Fc.bcol = kSlabB + jc;
  Fc.lam = !forced ? kSlabZero : (lane < kNX + kNU ? kSlabLamLeft : kSlabLamRight);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double v = 0.0;
    if (jc < 3) v = jc == 0 ? P.JinvR[i * 3] : (jc == 1 ? P.JinvR[i * 3 + 1] : P.JinvR[i * 3 + 2]);
    else if (jc < 6) v = jc == 3 ? P.Jinv[i * 3] : (jc == 4 ? P.Jinv[i * 3 + 1] : P.Jinv[i * 3 + 2]);
    Fc.jr[i] = v;
  }
}

/// RK4 stage kStage of the column from a slab: d = A c + lam * b, then the RK4 combination.  Same
/// arithmetic per entry as column_stage() — rows where the column of B is structurally zero get
/// lam * 0 added, as in the reference's dense product.
template <int kStage, bool kMayForce = true>
PT_HD void column_stage_slab(ColumnLane& L, const ColumnForcing& Fc, const double* slab, double wk, double wn) {
  double d[kNX];
  apply_A(slab, kStage == 0 ? L.s_c : L.c, d);
  // One predicated region, the same code for every kind of B column; the lanes of Phi_x skip it
  // (shared memory serves requested bytes: their loads would cost as much as the others'), and a
  // warp that owns Phi_x columns only does not carry it at all (kMayForce = false).
  if (kMayForce && Fc.forced) {
    const double lam = slab[Fc.lam];
    const double* b = slab + Fc.bcol;
#pragma unroll
    for (int i = 0; i < kNX; ++i) d[i] += lam * b[8 * i];
    const double s = slab[kRecS];
#pragma unroll
    for (int i = 0; i < 3; ++i) d[11 + i] += lam * (s * Fc.jr[i]);
  }
#pragma unroll
  for (int i = 0; i < kNX; ++i) {
    if (kStage == 0) {
      L.a_c[i] = L.s_c[i] + wk * d[i];
      L.c[i] = L.s_c[i] + wn * d[i];
    } else if (kStage < 3) {
      L.a_c[i] = L.a_c[i] + wk * d[i];
      L.c[i] = L.s_c[i] + wn * d[i];
    } else {
      L.s_c[i] = L.a_c[i] + wk * d[i];
    }
  }
}

/// Record -> slab on the CPU (the kernel does it with the addresses of its asynchronous copies).
inline void expand_record(const double* rec, double lam_left, double lam_right, double* slab) {
  for (int i = 0; i < kSlabSize; ++i) slab[i] = 0.0;
  for (int f = 0; f < kRecSize; ++f) slab[slab_dest(f)] = rec[f];
  slab[kSlabLamLeft] = lam_left;
  slab[kSlabLamRight] = lam_right;
  slab[kSlabSize - 1] = 0.0;
}

/// Run-time stage index (CPU simulation).
PT_HD void column_stage_slab(ColumnLane& L, const ColumnForcing& Fc, const double* slab, const StageTime& t, int stage) {
  switch (stage) {
    case 0: column_stage_slab<0>(L, Fc, slab, t.wk, t.wn); break;
    case 1: column_stage_slab<1>(L, Fc, slab, t.wk, t.wn); break;
    case 2: column_stage_slab<2>(L, Fc, slab, t.wk, t.wn); break;
    default: column_stage_slab<3>(L, Fc, slab, t.wk, t.wn); break;
  }
}

}  // namespace ptopt_b200
