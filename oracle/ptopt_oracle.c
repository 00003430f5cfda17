/*
 * ptopt_oracle.c — TEST INFRASTRUCTURE (see ptopt_oracle.h).
 *
 * Plain-C restatement of the reference CPU algorithm for the hot path.  Flat
 * row-major arrays replace the reference's Vec/Mat templates; arithmetic is
 * kept in the reference's evaluation order so that, with FP contraction off,
 * results are bit-identical to the reference (pinned by
 * tests/test_oracle_vs_ref.py).  Citations are file:line under
 * /root/reference/proj/include/ptopt/.
 */
#define _POSIX_C_SOURCE 200809L
#include "ptopt_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define NXI PTOPT_NXI
#define NZ PTOPT_NZETA
#define NG PTOPT_NG
#define NX PTOPT_NX
#define NU PTOPT_NU

enum { K_MASS = 0, K_POS = 1, K_VEL = 4, K_ATT = 7, K_RATE = 11, K_THRUST = 0, K_TORQUE = 3 };

static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */
static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */

/* ------------------------------------------------------------------------- */
/* rocket6dof.hpp                                                             */
/* ------------------------------------------------------------------------- */

static void cross3(const double* a, const double* b, double* c) { /* :155-157 */
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}

static void skew3(const double* a, double* S) { /* :159-169 */
  for (int i = 0; i < 9; ++i) S[i] = 0.0;
  S[0 * 3 + 1] = -a[2];
  S[0 * 3 + 2] = a[1];
  S[1 * 3 + 0] = a[2];
  S[1 * 3 + 2] = -a[0];
  S[2 * 3 + 0] = -a[1];
  S[2 * 3 + 1] = a[0];
}

static double norm3(const double* a) { return sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]); }

static void dcm(const double* q, double* C) { /* :176-188 */
  const double qw = q[3];
  const double s = q[0] * q[0] + q[1] * q[1] + q[2] * q[2];
  double K[9];
  for (int i = 0; i < 9; ++i) C[i] = 0.0;
  for (int i = 0; i < 3; ++i) C[i * 3 + i] = qw * qw - s;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) C[i * 3 + j] += 2.0 * q[i] * q[j];
  skew3(q, K);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) C[i * 3 + j] += 2.0 * qw * K[i * 3 + j];
}

static void dcm_times_vec_jac(const double* q, const double* t, double* D /*3x4*/) { /* :191-207 */
  const double qw = q[3];
  const double qv[3] = {q[0], q[1], q[2]};
  const double qv_dot_t = qv[0] * t[0] + qv[1] * t[1] + qv[2] * t[2];
  double Tk[9], qv_x_t[3];
  skew3(t, Tk);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double v = -2.0 * t[i] * qv[j] + 2.0 * qv[i] * t[j] - 2.0 * qw * Tk[i * 3 + j];
      if (i == j) v += 2.0 * qv_dot_t;
      D[i * 4 + j] = v;
    }
  cross3(qv, t, qv_x_t);
  for (int i = 0; i < 3; ++i) D[i * 4 + 3] = 2.0 * qw * t[i] + 2.0 * qv_x_t[i];
}

static double det3(const double* J) { /* :139-143 */
  return J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
         J[2] * (J[3] * J[7] - J[4] * J[6]);
}

int ptor_rocket_init(ptor_rocket* r, const ptopt_vehicle_params* p) { /* :210-224, :240-241 */
  const double* J = p->inertia;
  const double det = det3(J);
  r->p = *p;
  if (det == 0.0) return -8;
  r->inertia_inv[0] = (J[4] * J[8] - J[5] * J[7]) / det;
  r->inertia_inv[1] = (J[2] * J[7] - J[1] * J[8]) / det;
  r->inertia_inv[2] = (J[1] * J[5] - J[2] * J[4]) / det;
  r->inertia_inv[3] = (J[5] * J[6] - J[3] * J[8]) / det;
  r->inertia_inv[4] = (J[0] * J[8] - J[2] * J[6]) / det;
  r->inertia_inv[5] = (J[2] * J[3] - J[0] * J[5]) / det;
  r->inertia_inv[6] = (J[3] * J[7] - J[4] * J[6]) / det;
  r->inertia_inv[7] = (J[1] * J[6] - J[0] * J[7]) / det;
  r->inertia_inv[8] = (J[0] * J[4] - J[1] * J[3]) / det;
  return 0;
}

/* eval_dynamics, :245-274 */
static int rocket_dynamics(const void* ctx, const double* xi, const double* zeta, double* F) {
  const ptor_rocket* r = (const ptor_rocket*)ctx;
  const ptopt_vehicle_params* p = &r->p;
  const double m = xi[K_MASS];
  const double* v = xi + K_VEL;
  const double* q = xi + K_ATT;
  const double* w = xi + K_RATE;
  const double* T = zeta + K_THRUST;
  const double* tq = zeta + K_TORQUE;
  double C[9], qv_x_w[3], Jw[3] = {0.0, 0.0, 0.0}, lever[3], gyro[3];
  if (!(m > 0.0)) return PTOPT_ST_MASS_NONPOSITIVE;
  F[K_MASS] = -p->alpha_mdot * norm3(T);
  for (int i = 0; i < 3; ++i) F[K_POS + i] = v[i];
  dcm(q, C);
  for (int i = 0; i < 3; ++i) {
    double acc = 0.0;
    for (int j = 0; j < 3; ++j) acc += C[i * 3 + j] * T[j];
    F[K_VEL + i] = acc / m + p->g_inertial[i];
  }
  {
    const double qv[3] = {q[0], q[1], q[2]};
    const double qw = q[3];
    cross3(qv, w, qv_x_w);
    for (int i = 0; i < 3; ++i) F[K_ATT + i] = 0.5 * (qw * w[i] + qv_x_w[i]);
    F[K_ATT + 3] = -0.5 * (qv[0] * w[0] + qv[1] * w[1] + qv[2] * w[2]);
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Jw[i] += p->inertia[i * 3 + j] * w[j];
  cross3(p->r_thrust, T, lever);
  cross3(w, Jw, gyro);
  for (int i = 0; i < 3; ++i) {
    double acc = 0.0;
    for (int j = 0; j < 3; ++j) acc += r->inertia_inv[i * 3 + j] * (lever[j] - gyro[j] + tq[j]);
    F[K_RATE + i] = acc;
  }
  return 0;
}

/* eval_constraints, :278-301 */
static void rocket_constraints(const void* ctx, const double* xi, const double* zeta, double* g) {
  const ptopt_vehicle_params* p = &((const ptor_rocket*)ctx)->p;
  const double* r = xi + K_POS;
  const double* v = xi + K_VEL;
  const double* q = xi + K_ATT;
  const double* w = xi + K_RATE;
  const double* T = zeta + K_THRUST;
  const double* tq = zeta + K_TORQUE;
  const double Tn = norm3(T);
  const double sec_delta = 1.0 / cos(p->delta_max);
  double hq_sq = 0.0;
  g[0] = p->m_dry - xi[K_MASS];
  g[1] = -r[0];
  g[2] = v[0] * v[0] + v[1] * v[1] + v[2] * v[2] - p->v_max * p->v_max;
  for (int i = 0; i < 2; ++i) {
    double acc = 0.0;
    for (int j = 0; j < 4; ++j) acc += p->H_theta[i * 4 + j] * q[j];
    hq_sq += acc * acc;
  }
  {
    const double c = 1.0 - cos(p->theta_max);
    g[3] = 4.0 * hq_sq - c * c;
  }
  g[4] = w[0] * w[0] + w[1] * w[1] + w[2] * w[2] - p->omega_max * p->omega_max;
  g[5] = Tn - T[0] * sec_delta;
  g[6] = Tn - p->T_max;
  g[7] = -Tn + p->T_min;
  g[8] = tq[0] * tq[0] + tq[1] * tq[1] + tq[2] * tq[2] - p->gamma_max * p->gamma_max;
}

/* eval_jacobians, :303-402.  Any output pointer may be NULL. */
static int rocket_jacobians(const ptor_rocket* r, const double* xi, const double* zeta,
                            double* dF_dxi, double* dF_dzeta, double* dg_dxi, double* dg_dzeta) {
  const ptopt_vehicle_params* p = &r->p;
  const double m = xi[K_MASS];
  const double* v = xi + K_VEL;
  const double* q = xi + K_ATT;
  const double* w = xi + K_RATE;
  const double* T = zeta + K_THRUST;
  const double* tq = zeta + K_TORQUE;
  const double Tn = norm3(T);
  double Fx[NXI * NXI], Fz[NXI * NZ], gx[NG * NXI], gz[NG * NZ];
  double C[9], CT[3] = {0.0, 0.0, 0.0}, dCTdq[12], Wk[9], Qk[9], Jw[3] = {0.0, 0.0, 0.0}, JWk[9],
         M[9], Rk[9];
  if (Tn < 1e-9) return PTOPT_ST_THRUST_SINGULAR;
  if (!(m > 0.0)) return PTOPT_ST_MASS_NONPOSITIVE;
  memset(Fx, 0, sizeof Fx);
  memset(Fz, 0, sizeof Fz);
  memset(gx, 0, sizeof gx);
  memset(gz, 0, sizeof gz);

  dcm(q, C);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) CT[i] += C[i * 3 + j] * T[j];

  for (int i = 0; i < 3; ++i) Fx[(K_POS + i) * NXI + K_VEL + i] = 1.0;

  for (int i = 0; i < 3; ++i) Fx[(K_VEL + i) * NXI + K_MASS] = -CT[i] / (m * m);
  dcm_times_vec_jac(q, T, dCTdq);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 4; ++j) Fx[(K_VEL + i) * NXI + K_ATT + j] = dCTdq[i * 4 + j] / m;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Fz[(K_VEL + i) * NZ + K_THRUST + j] = C[i * 3 + j] / m;

  {
    const double qv[3] = {q[0], q[1], q[2]};
    const double qw = q[3];
    skew3(w, Wk);
    for (int i = 0; i < 3; ++i) {
      for (int j = 0; j < 3; ++j) Fx[(K_ATT + i) * NXI + K_ATT + j] = -0.5 * Wk[i * 3 + j];
      Fx[(K_ATT + i) * NXI + K_ATT + 3] = 0.5 * w[i];
      Fx[(K_ATT + 3) * NXI + K_ATT + i] = -0.5 * w[i];
    }
    skew3(qv, Qk);
    for (int i = 0; i < 3; ++i) {
      for (int j = 0; j < 3; ++j)
        Fx[(K_ATT + i) * NXI + K_RATE + j] = 0.5 * ((i == j ? qw : 0.0) + Qk[i * 3 + j]);
      Fx[(K_ATT + 3) * NXI + K_RATE + i] = -0.5 * qv[i];
    }
  }

  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Jw[i] += p->inertia[i * 3 + j] * w[j];
  skew3(Jw, JWk);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double acc = JWk[i * 3 + j];
      for (int k = 0; k < 3; ++k) acc -= Wk[i * 3 + k] * p->inertia[k * 3 + j];
      M[i * 3 + j] = acc;
    }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc += r->inertia_inv[i * 3 + k] * M[k * 3 + j];
      Fx[(K_RATE + i) * NXI + K_RATE + j] = acc;
    }
  skew3(p->r_thrust, Rk);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc += r->inertia_inv[i * 3 + k] * Rk[k * 3 + j];
      Fz[(K_RATE + i) * NZ + K_THRUST + j] = acc;
      Fz[(K_RATE + i) * NZ + K_TORQUE + j] = r->inertia_inv[i * 3 + j];
    }

  for (int j = 0; j < 3; ++j) Fz[K_MASS * NZ + K_THRUST + j] = -p->alpha_mdot * T[j] / Tn;

  gx[0 * NXI + K_MASS] = -1.0;
  gx[1 * NXI + K_POS] = -1.0;
  for (int j = 0; j < 3; ++j) gx[2 * NXI + K_VEL + j] = 2.0 * v[j];
  {
    double Hq[2] = {0.0, 0.0};
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 4; ++j) Hq[i] += p->H_theta[i * 4 + j] * q[j];
    for (int j = 0; j < 4; ++j)
      gx[3 * NXI + K_ATT + j] =
          8.0 * (Hq[0] * p->H_theta[0 * 4 + j] + Hq[1] * p->H_theta[1 * 4 + j]);
  }
  for (int j = 0; j < 3; ++j) gx[4 * NXI + K_RATE + j] = 2.0 * w[j];
  {
    const double sec_delta = 1.0 / cos(p->delta_max);
    for (int j = 0; j < 3; ++j) {
      const double that = T[j] / Tn;
      gz[5 * NZ + K_THRUST + j] = that - (j == 0 ? sec_delta : 0.0);
      gz[6 * NZ + K_THRUST + j] = that;
      gz[7 * NZ + K_THRUST + j] = -that;
      gz[8 * NZ + K_TORQUE + j] = 2.0 * tq[j];
    }
  }
  if (dF_dxi) memcpy(dF_dxi, Fx, sizeof Fx);
  if (dF_dzeta) memcpy(dF_dzeta, Fz, sizeof Fz);
  if (dg_dxi) memcpy(dg_dxi, gx, sizeof gx);
  if (dg_dzeta) memcpy(dg_dzeta, gz, sizeof gz);
  return 0;
}

static int rocket_dyn_jac(const void* ctx, const double* xi, const double* zeta, double* a,
                          double* b) { /* :413-420 */
  return rocket_jacobians((const ptor_rocket*)ctx, xi, zeta, a, b, NULL, NULL);
}
static int rocket_ineq_jac(const void* ctx, const double* xi, const double* zeta, double* a,
                           double* b) { /* :422-429 */
  return rocket_jacobians((const ptor_rocket*)ctx, xi, zeta, NULL, NULL, a, b);
}

ptor_model ptor_rocket_model(const ptor_rocket* r) {
  ptor_model m;
  memset(&m, 0, sizeof m);
  m.state_dim = NXI;
  m.control_dim = NZ;
  m.ineq_dim = NG;
  m.eq_dim = 0;
  m.ctx = r;
  m.dynamics = rocket_dynamics;
  m.path_ineq = rocket_constraints;
  m.dynamics_jacobians = rocket_dyn_jac;
  m.path_ineq_jacobians = rocket_ineq_jac;
  return m;
}

int ptor_model_eval(const ptopt_vehicle_params* vp, const double* xi, const double* zeta,
                    double* F, double* g, double* dF_dxi, double* dF_dzeta, double* dg_dxi,
                    double* dg_dzeta) {
  ptor_rocket r;
  int rc = ptor_rocket_init(&r, vp);
  if (rc) return rc;
  if (F && (rc = rocket_dynamics(&r, xi, zeta, F))) return rc;
  if (g) rocket_constraints(&r, xi, zeta, g);
  if (dF_dxi) return rocket_jacobians(&r, xi, zeta, dF_dxi, dF_dzeta, dg_dxi, dg_dzeta);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* the reference's analytic test models (proj/tests/support/test_models.hpp,  */
/* proj/tests/test_discretizer.cpp:13-28)                                      */
/* ------------------------------------------------------------------------- */

static int zero_dyn(const void* c, const double* x, const double* u, double* F) {
  (void)c; (void)x; (void)u;
  F[0] = 0.0;
  F[1] = 0.0;
  return 0;
}
static void zero_ineq(const void* c, const double* x, const double* u, double* g) {
  (void)c; (void)x; (void)u;
  g[0] = -1.0;
}
static int zero_dyn_jac(const void* c, const double* x, const double* u, double* A, double* B) {
  (void)c; (void)x; (void)u;
  for (int i = 0; i < 4; ++i) A[i] = 0.0;
  B[0] = B[1] = 0.0;
  return 0;
}
static int zero_ineq_jac(const void* c, const double* x, const double* u, double* a, double* b) {
  (void)c; (void)x; (void)u;
  a[0] = a[1] = 0.0;
  b[0] = 0.0;
  return 0;
}

static int lti_dyn(const void* c, const double* x, const double* u, double* F) {
  const double* ab = (const double*)c;
  F[0] = ab[0] * x[0] + ab[1] * u[0];
  return 0;
}
static int lti_dyn_jac(const void* c, const double* x, const double* u, double* A, double* B) {
  const double* ab = (const double*)c;
  (void)x; (void)u;
  A[0] = ab[0];
  B[0] = ab[1];
  return 0;
}

static int dint_dyn(const void* c, const double* x, const double* u, double* F) {
  (void)c;
  F[0] = x[1];
  F[1] = u[0];
  return 0;
}
static int dint_dyn_jac(const void* c, const double* x, const double* u, double* A, double* B) {
  (void)c; (void)x; (void)u;
  A[0] = 0.0; A[1] = 1.0; A[2] = 0.0; A[3] = 0.0;
  B[0] = 0.0; B[1] = 1.0;
  return 0;
}

static int toy_dyn(const void* c, const double* x, const double* u, double* F) {
  (void)c;
  F[0] = -x[0] + 0.5 * x[1] * u[0];
  F[1] = x[0] * x[1] - u[1];
  return 0;
}
static void toy_ineq(const void* c, const double* x, const double* u, double* g) {
  (void)c;
  g[0] = x[0] * x[0] + 0.3 * u[0] - 1.0;
  g[1] = x[1] - 0.25 * u[1] * u[1];
}
static void toy_eq(const void* c, const double* x, const double* u, double* h) {
  (void)c;
  h[0] = 0.5 * x[0] + u[0] * u[1];
}
static int toy_dyn_jac(const void* c, const double* x, const double* u, double* A, double* B) {
  (void)c;
  A[0] = -1.0; A[1] = 0.5 * u[0]; A[2] = x[1]; A[3] = x[0];
  B[0] = 0.5 * x[1]; B[1] = 0.0; B[2] = 0.0; B[3] = -1.0;
  return 0;
}
static int toy_ineq_jac(const void* c, const double* x, const double* u, double* a, double* b) {
  (void)c;
  a[0] = 2.0 * x[0]; a[1] = 0.0; a[2] = 0.0; a[3] = 1.0;
  b[0] = 0.3; b[1] = 0.0; b[2] = 0.0; b[3] = -0.5 * u[1];
  return 0;
}
static void toy_eq_jac(const void* c, const double* x, const double* u, double* a, double* b) {
  (void)c; (void)x;
  a[0] = 0.5; a[1] = 0.0;
  b[0] = u[1]; b[1] = u[0];
}

static int blow_dyn(const void* c, const double* x, const double* u, double* F) {
  (void)c; (void)u;
  F[0] = x[0] * x[0];
  return 0;
}
static int blow_dyn_jac(const void* c, const double* x, const double* u, double* A, double* B) {
  (void)c; (void)u;
  A[0] = 2.0 * x[0];
  B[0] = 0.0;
  return 0;
}

static int test_model(int id, const double* params, ptor_model* m) {
  memset(m, 0, sizeof *m);
  m->ctx = params;
  switch (id) {
    case 0:
      m->state_dim = 2; m->control_dim = 1; m->ineq_dim = 1;
      m->dynamics = zero_dyn; m->path_ineq = zero_ineq;
      m->dynamics_jacobians = zero_dyn_jac; m->path_ineq_jacobians = zero_ineq_jac;
      return 0;
    case 1:
      m->state_dim = 1; m->control_dim = 1;
      m->dynamics = lti_dyn; m->dynamics_jacobians = lti_dyn_jac;
      return 0;
    case 2:
      m->state_dim = 2; m->control_dim = 1;
      m->dynamics = dint_dyn; m->dynamics_jacobians = dint_dyn_jac;
      return 0;
    case 3:
      m->state_dim = 2; m->control_dim = 2; m->ineq_dim = 2; m->eq_dim = 1;
      m->dynamics = toy_dyn; m->path_ineq = toy_ineq; m->path_eq = toy_eq;
      m->dynamics_jacobians = toy_dyn_jac; m->path_ineq_jacobians = toy_ineq_jac;
      m->path_eq_jacobians = toy_eq_jac;
      return 0;
    case 4:
      m->state_dim = 1; m->control_dim = 1;
      m->dynamics = blow_dyn; m->dynamics_jacobians = blow_dyn_jac;
      return 0;
    default:
      return -1;
  }
}

/* ------------------------------------------------------------------------- */
/* ctcs.hpp: Augmented<Model>                                                 */
/* ------------------------------------------------------------------------- */

static double violation_integrand(const ptor_model* m, const double* xi, const double* zeta) {
  /* :47-62 */
  double acc = 0.0;
  if (m->ineq_dim > 0) {
    double g[PTOR_MAX_G];
    m->path_ineq(m->ctx, xi, zeta, g);
    for (int i = 0; i < m->ineq_dim; ++i) {
      const double v = g[i] > 0.0 ? g[i] : 0.0;
      acc += v * v;
    }
  }
  if (m->eq_dim > 0) {
    double h[PTOR_MAX_G];
    m->path_eq(m->ctx, xi, zeta, h);
    for (int i = 0; i < m->eq_dim; ++i) acc += h[i] * h[i];
  }
  return acc;
}

static int aug_dynamics(const ptor_model* m, const double* x, const double* u, double* dx) {
  /* :64-74 */
  const int sd = m->state_dim;
  const double s = u[m->control_dim];
  double F[PTOR_MAX_X];
  int rc;
  if (!(s > 0.0)) return PTOPT_ST_DILATION_NONPOSITIVE;
  if ((rc = m->dynamics(m->ctx, x, u, F))) return rc;
  for (int i = 0; i < sd; ++i) dx[i] = s * F[i];
  dx[sd] = s * violation_integrand(m, x, u);
  return 0;
}

static int aug_jacobians(const ptor_model* m, const double* x, const double* u, double* A,
                         double* B) { /* :79-129 */
  const int sd = m->state_dim, cd = m->control_dim;
  const int nx = sd + 1, nu = cd + 1;
  const double s = u[cd];
  double dF_dx[PTOR_MAX_X * PTOR_MAX_X], dF_du[PTOR_MAX_X * PTOR_MAX_U], F[PTOR_MAX_X];
  double integrand = 0.0;
  int rc;
  if (!(s > 0.0)) return PTOPT_ST_DILATION_NONPOSITIVE;
  for (int i = 0; i < nx * nx; ++i) A[i] = 0.0;
  for (int i = 0; i < nx * nu; ++i) B[i] = 0.0;
  if ((rc = m->dynamics_jacobians(m->ctx, x, u, dF_dx, dF_du))) return rc;
  if ((rc = m->dynamics(m->ctx, x, u, F))) return rc;
  for (int i = 0; i < sd; ++i) {
    for (int j = 0; j < sd; ++j) A[i * nx + j] = s * dF_dx[i * sd + j];
    for (int j = 0; j < cd; ++j) B[i * nu + j] = s * dF_du[i * cd + j];
    B[i * nu + cd] = F[i];
  }
  if (m->ineq_dim > 0) {
    double g[PTOR_MAX_G], dg_dx[PTOR_MAX_G * PTOR_MAX_X], dg_du[PTOR_MAX_G * PTOR_MAX_U];
    m->path_ineq(m->ctx, x, u, g);
    if ((rc = m->path_ineq_jacobians(m->ctx, x, u, dg_dx, dg_du))) return rc;
    for (int i = 0; i < m->ineq_dim; ++i) {
      const double gp = g[i] > 0.0 ? g[i] : 0.0;
      integrand += gp * gp;
      if (gp > 0.0) {
        for (int j = 0; j < sd; ++j) A[sd * nx + j] += 2.0 * s * gp * dg_dx[i * sd + j];
        for (int j = 0; j < cd; ++j) B[sd * nu + j] += 2.0 * s * gp * dg_du[i * cd + j];
      }
    }
  }
  if (m->eq_dim > 0) {
    double h[PTOR_MAX_G], dh_dx[PTOR_MAX_G * PTOR_MAX_X], dh_du[PTOR_MAX_G * PTOR_MAX_U];
    m->path_eq(m->ctx, x, u, h);
    m->path_eq_jacobians(m->ctx, x, u, dh_dx, dh_du);
    for (int i = 0; i < m->eq_dim; ++i) {
      integrand += h[i] * h[i];
      for (int j = 0; j < sd; ++j) A[sd * nx + j] += 2.0 * s * h[i] * dh_dx[i * sd + j];
      for (int j = 0; j < cd; ++j) B[sd * nu + j] += 2.0 * s * h[i] * dh_du[i * cd + j];
    }
  }
  B[sd * nu + cd] = integrand;
  return 0;
}

static int aug_eval(const ptor_model* m, const double* x, const double* u, double* f, double* A,
                    double* B) {
  int rc = aug_dynamics(m, x, u, f);
  if (rc) return rc;
  return aug_jacobians(m, x, u, A, B);
}

int ptor_aug_eval(const ptopt_vehicle_params* vp, const double* x, const double* u, double* f,
                  double* A, double* B) {
  ptor_rocket r;
  ptor_model m;
  int rc = ptor_rocket_init(&r, vp);
  if (rc) return rc;
  m = ptor_rocket_model(&r);
  return aug_eval(&m, x, u, f, A, B);
}

int ptor_aug_eval_test_model(int model_id, const double* params, const double* x, const double* u,
                             double* f, double* A, double* B) {
  ptor_model m;
  if (test_model(model_id, params, &m)) return -1;
  return aug_eval(&m, x, u, f, A, B);
}

/* ------------------------------------------------------------------------- */
/* discretizer.hpp                                                            */
/* ------------------------------------------------------------------------- */

int ptor_foh_interp(int n, const double* u_k, const double* u_k1, double tau, double tau_k,
                    double tau_k1, double* u) { /* :26-39 */
  double span, lam_right, lam_left;
  if (!(tau_k < tau_k1)) return -1;
  span = tau_k1 - tau_k;
  if (tau < tau_k - 1e-12 * span || tau > tau_k1 + 1e-12 * span) return -1;
  lam_right = (tau - tau_k) / span;
  lam_left = (tau_k1 - tau) / span;
  for (int i = 0; i < n; ++i) u[i] = lam_left * u_k[i] + lam_right * u_k1[i];
  return 0;
}

typedef struct bundle { /* SensitivityBundle, :58-75 */
  double x[PTOR_MAX_X];
  double phi_x[PTOR_MAX_X * PTOR_MAX_X];
  double phi_um[PTOR_MAX_X * PTOR_MAX_U];
  double phi_up[PTOR_MAX_X * PTOR_MAX_U];
} bundle;

static void bundle_add_scaled(bundle* s, double c, const bundle* d, int nx, int nu) {
  for (int i = 0; i < nx; ++i) s->x[i] += c * d->x[i];
  for (int i = 0; i < nx * nx; ++i) s->phi_x[i] += c * d->phi_x[i];
  for (int i = 0; i < nx * nu; ++i) {
    s->phi_um[i] += c * d->phi_um[i];
    s->phi_up[i] += c * d->phi_up[i];
  }
}

static void mat_mat(const double* A, int ra, int ca, const double* B, int cb, double* C) {
  /* smallmat.hpp:109-122 */
  for (int i = 0; i < ra; ++i)
    for (int j = 0; j < cb; ++j) {
      double acc = 0.0;
      for (int k = 0; k < ca; ++k) acc += A[i * ca + k] * B[k * cb + j];
      C[i * cb + j] = acc;
    }
}

static void mat_vec(const double* A, int rows, int cols, const double* x, int transpose,
                    double* y) { /* smallmat.hpp:82-106 */
  if (!transpose) {
    for (int i = 0; i < rows; ++i) {
      double acc = 0.0;
      for (int j = 0; j < cols; ++j) acc += A[i * cols + j] * x[j];
      y[i] = acc;
    }
  } else {
    for (int j = 0; j < cols; ++j) {
      double acc = 0.0;
      for (int i = 0; i < rows; ++i) acc += A[i * cols + j] * x[i];
      y[j] = acc;
    }
  }
}

static void vec_add_scaled(double* y, double alpha, const double* x, int n) {
  for (int i = 0; i < n; ++i) y[i] += alpha * x[i]; /* smallmat.hpp:171-177 */
}

static int all_finite(const double* x, int n) {
  for (int i = 0; i < n; ++i)
    if (!isfinite(x[i])) return 0;
  return 1;
}

typedef struct interval_ctx {
  const ptor_model* m;
  const double *u_k, *u_k1;
  double tau_k, tau_k1, span;
  int nx, nu;
} interval_ctx;

static int bundle_deriv(const interval_ctx* c, double tau, const bundle* in, bundle* d) {
  /* the `deriv` lambda, :98-116 */
  const int nx = c->nx, nu = c->nu;
  double u[PTOR_MAX_U], A[PTOR_MAX_X * PTOR_MAX_X], B[PTOR_MAX_X * PTOR_MAX_U];
  double lam_right, lam_left;
  int rc;
  if ((rc = ptor_foh_interp(nu, c->u_k, c->u_k1, tau, c->tau_k, c->tau_k1, u))) return rc;
  if ((rc = aug_dynamics(c->m, in->x, u, d->x))) return rc;
  if ((rc = aug_jacobians(c->m, in->x, u, A, B))) return rc;
  mat_mat(A, nx, nx, in->phi_x, nx, d->phi_x);
  mat_mat(A, nx, nx, in->phi_um, nu, d->phi_um);
  mat_mat(A, nx, nx, in->phi_up, nu, d->phi_up);
  lam_right = (tau - c->tau_k) / c->span;
  lam_left = (c->tau_k1 - tau) / c->span;
  for (int i = 0; i < nx; ++i)
    for (int j = 0; j < nu; ++j) {
      d->phi_um[i * nu + j] += lam_left * B[i * nu + j];
      d->phi_up[i * nu + j] += lam_right * B[i * nu + j];
    }
  return 0;
}

static int propagate_generic(const ptor_model* m, const double* x_k, const double* u_k,
                             const double* u_k1, double tau_k, double tau_k1, int steps,
                             int interval_index, double* A, double* Bm, double* Bp, double* w,
                             double* x_end, int* fail_index) { /* :82-149 */
  const int nx = m->state_dim + 1, nu = m->control_dim + 1;
  interval_ctx c;
  bundle s, k1, k2, k3, k4, mid, full;
  double h, tmp[PTOR_MAX_X];
  int rc;
  if (steps < 1) return -1;
  if (!all_finite(x_k, nx)) {
    if (fail_index) *fail_index = interval_index;
    return PTOPT_ST_PROPAGATION_DIVERGED;
  }
  c.m = m;
  c.u_k = u_k;
  c.u_k1 = u_k1;
  c.tau_k = tau_k;
  c.tau_k1 = tau_k1;
  c.span = tau_k1 - tau_k;
  c.nx = nx;
  c.nu = nu;
  memset(&s, 0, sizeof s);
  for (int i = 0; i < nx; ++i) s.x[i] = x_k[i];
  for (int i = 0; i < nx; ++i) s.phi_x[i * nx + i] = 1.0;

  h = c.span / steps;
  for (int step = 0; step < steps; ++step) {
    const double t0 = tau_k + h * step;
    const double t_end = (step + 1 == steps) ? tau_k1 : t0 + h;
    if ((rc = bundle_deriv(&c, t0, &s, &k1))) return rc;
    mid = s;
    bundle_add_scaled(&mid, 0.5 * h, &k1, nx, nu);
    if ((rc = bundle_deriv(&c, t0 + 0.5 * h, &mid, &k2))) return rc;
    mid = s;
    bundle_add_scaled(&mid, 0.5 * h, &k2, nx, nu);
    if ((rc = bundle_deriv(&c, t0 + 0.5 * h, &mid, &k3))) return rc;
    full = s;
    bundle_add_scaled(&full, h, &k3, nx, nu);
    if ((rc = bundle_deriv(&c, t_end, &full, &k4))) return rc;
    bundle_add_scaled(&s, h / 6.0, &k1, nx, nu);
    bundle_add_scaled(&s, h / 3.0, &k2, nx, nu);
    bundle_add_scaled(&s, h / 3.0, &k3, nx, nu);
    bundle_add_scaled(&s, h / 6.0, &k4, nx, nu);
    if (!all_finite(s.x, nx)) {
      if (fail_index) *fail_index = interval_index;
      return PTOPT_ST_PROPAGATION_DIVERGED;
    }
  }
  memcpy(A, s.phi_x, sizeof(double) * nx * nx);
  memcpy(Bm, s.phi_um, sizeof(double) * nx * nu);
  memcpy(Bp, s.phi_up, sizeof(double) * nx * nu);
  for (int i = 0; i < nx; ++i) x_end[i] = s.x[i];
  for (int i = 0; i < nx; ++i) w[i] = s.x[i];
  mat_vec(A, nx, nx, x_k, 0, tmp);
  vec_add_scaled(w, -1.0, tmp, nx);
  mat_vec(Bm, nx, nu, u_k, 0, tmp);
  vec_add_scaled(w, -1.0, tmp, nx);
  mat_vec(Bp, nx, nu, u_k1, 0, tmp);
  vec_add_scaled(w, -1.0, tmp, nx);
  return 0;
}

int ptor_propagate_interval(const ptopt_vehicle_params* vp, const double* xk, const double* uk,
                            const double* uk1, double tau_k, double tau_k1, int steps,
                            int interval_index, double* A, double* Bm, double* Bp, double* w,
                            double* x_end, int* fail_index) {
  ptor_rocket r;
  ptor_model m;
  int rc = ptor_rocket_init(&r, vp);
  if (rc) return rc;
  m = ptor_rocket_model(&r);
  return propagate_generic(&m, xk, uk, uk1, tau_k, tau_k1, steps, interval_index, A, Bm, Bp, w,
                           x_end, fail_index);
}

int ptor_propagate_test_model(int model_id, const double* params, const double* xk,
                              const double* uk, const double* uk1, double tau_k, double tau_k1,
                              int steps, int interval_index, double* A, double* Bm, double* Bp,
                              double* w, double* x_end, int* fail_index) {
  ptor_model m;
  if (test_model(model_id, params, &m)) return -1;
  return propagate_generic(&m, xk, uk, uk1, tau_k, tau_k1, steps, interval_index, A, Bm, Bp, w,
                           x_end, fail_index);
}

static void uniform_grid(int n, double* tau) { /* trajectory.hpp:23-30 */
  for (int k = 0; k < n; ++k) tau[k] = (double)k / (n - 1);
  tau[0] = 0.0;
  tau[n - 1] = 1.0;
}

static double* grid_nodes(const ptopt_problem_desc* d, const double* tau) {
  double* g = (double*)malloc(sizeof(double) * (size_t)d->nodes);
  if (tau)
    memcpy(g, tau, sizeof(double) * (size_t)d->nodes);
  else
    uniform_grid(d->nodes, g);
  return g;
}

static int linearize_with(const ptor_model* m, const double* grid, int n, int steps,
                          const double* x, const double* u, double* A, double* Bm, double* Bp,
                          double* w, double* x_end, int* fail_index) { /* :191-232, serial */
  for (int k = 0; k < n - 1; ++k) {
    int rc = propagate_generic(m, x + k * NX, u + k * NU, u + (k + 1) * NU, grid[k], grid[k + 1],
                               steps, k, A + k * NX * NX, Bm + k * NX * NU, Bp + k * NX * NU,
                               w + k * NX, x_end + k * NX, fail_index);
    if (rc) {
      if (fail_index && rc != PTOPT_ST_PROPAGATION_DIVERGED) *fail_index = k;
      return rc;
    }
  }
  return 0;
}

int ptor_linearize_all(const ptopt_problem_desc* d, const double* tau, const double* x,
                       const double* u, int workers, double* A, double* Bm, double* Bp, double* w,
                       double* x_end, int* fail_index) {
  ptor_rocket r;
  ptor_model m;
  double* grid;
  int rc;
  (void)workers; /* results are independent of the worker count (discretizer.hpp:190) */
  if ((rc = ptor_rocket_init(&r, &d->vehicle))) return rc;
  m = ptor_rocket_model(&r);
  grid = grid_nodes(d, tau);
  rc = linearize_with(&m, grid, d->nodes, d->integrator_steps, x, u, A, Bm, Bp, w, x_end,
                      fail_index);
  free(grid);
  return rc;
}

/* propagate_state with the audit's sample sink folded in, :153-187 + :262-277 */
static int propagate_state_audit(const ptor_model* m, const double* x_k, const double* u_k,
                                 const double* u_k1, double tau_k, double tau_k1, int steps,
                                 double* x_out, double* max_g, int interval, double* samples) {
  const int nx = m->state_dim + 1, nu = m->control_dim + 1;
  double x[PTOR_MAX_X], k1[PTOR_MAX_X], k2[PTOR_MAX_X], k3[PTOR_MAX_X], k4[PTOR_MAX_X],
      tmp[PTOR_MAX_X], uu[PTOR_MAX_U], g[PTOR_MAX_G];
  const double h = (tau_k1 - tau_k) / steps;
  int rc;
  if (steps < 1) return -1;
  for (int i = 0; i < nx; ++i) x[i] = x_k[i];
#define RECORD(tau_, xs_)                                                         \
  do {                                                                            \
    double gmax = -INFINITY;                                                      \
    if ((rc = ptor_foh_interp(nu, u_k, u_k1, (tau_), tau_k, tau_k1, uu))) return rc; \
    m->path_ineq(m->ctx, (xs_), uu, g);                                           \
    for (int i_ = 0; i_ < m->ineq_dim; ++i_) gmax = dmax(gmax, g[i_]);            \
    *max_g = dmax(*max_g, gmax);                                                  \
    if (samples) { /* AuditSample{interval, tau, g, g_max}, :262-276 */           \
      samples[0] = (double)interval;                                              \
      samples[1] = (tau_);                                                        \
      for (int i_ = 0; i_ < m->ineq_dim; ++i_) samples[2 + i_] = g[i_];           \
      samples[2 + m->ineq_dim] = gmax;                                            \
      samples += PTOR_SAMPLE_DOUBLES;                                             \
    }                                                                             \
  } while (0)
#define RATE(tau_, xs_, out_)                                                     \
  do {                                                                            \
    if ((rc = ptor_foh_interp(nu, u_k, u_k1, (tau_), tau_k, tau_k1, uu))) return rc; \
    if ((rc = aug_dynamics(m, (xs_), uu, (out_)))) return rc;                     \
  } while (0)
  RECORD(tau_k, x);
  for (int step = 0; step < steps; ++step) {
    const double t0 = tau_k + h * step;
    const double t_end = (step + 1 == steps) ? tau_k1 : t0 + h;
    RATE(t0, x, k1);
    memcpy(tmp, x, sizeof x);
    vec_add_scaled(tmp, 0.5 * h, k1, nx);
    RATE(t0 + 0.5 * h, tmp, k2);
    memcpy(tmp, x, sizeof x);
    vec_add_scaled(tmp, 0.5 * h, k2, nx);
    RATE(t0 + 0.5 * h, tmp, k3);
    memcpy(tmp, x, sizeof x);
    vec_add_scaled(tmp, h, k3, nx);
    RATE(t_end, tmp, k4);
    vec_add_scaled(x, h / 6.0, k1, nx);
    vec_add_scaled(x, h / 3.0, k2, nx);
    vec_add_scaled(x, h / 3.0, k3, nx);
    vec_add_scaled(x, h / 6.0, k4, nx);
    RECORD(t_end, x);
  }
#undef RECORD
#undef RATE
  for (int i = 0; i < nx; ++i) x_out[i] = x[i];
  return 0;
}

static int dense_audit_with(const ptor_model* m, const double* grid, int n, const double* x,
                            const double* u, int substeps, double* max_pointwise_g,
                            double* total_y_increase, double* interval_y_increase, double* samples) {
  /* :249-285 */
  double total = 0.0, gmax = -INFINITY;
  if (substeps < 1) return -1;
  for (int k = 0; k < n - 1; ++k) {
    double xe[PTOR_MAX_X], dy;
    int rc = propagate_state_audit(m, x + k * NX, u + k * NU, u + (k + 1) * NU, grid[k],
                                   grid[k + 1], substeps, xe, &gmax, k,
                                   samples ? samples + (size_t)k * (substeps + 1) * PTOR_SAMPLE_DOUBLES : NULL);
    if (rc) return rc;
    dy = xe[NX - 1] - x[k * NX + NX - 1];
    if (interval_y_increase) interval_y_increase[k] = dy;
    total += dy;
  }
  *max_pointwise_g = gmax;
  *total_y_increase = total;
  return 0;
}

int ptor_dense_audit(const ptopt_problem_desc* d, const double* tau, const double* x,
                     const double* u, int substeps, double* max_pointwise_g,
                     double* total_y_increase, double* interval_y_increase) {
  ptor_rocket r;
  ptor_model m;
  double* grid;
  int rc;
  if ((rc = ptor_rocket_init(&r, &d->vehicle))) return rc;
  m = ptor_rocket_model(&r);
  grid = grid_nodes(d, tau);
  rc = dense_audit_with(&m, grid, d->nodes, x, u, substeps, max_pointwise_g, total_y_increase,
                        interval_y_increase, NULL);
  free(grid);
  return rc;
}

int ptor_dense_audit_samples(const ptopt_problem_desc* d, const double* tau, const double* x,
                             const double* u, int substeps, double* max_pointwise_g,
                             double* total_y_increase, double* interval_y_increase, double* samples) {
  ptor_rocket r;
  ptor_model m;
  double* grid;
  int rc;
  if ((rc = ptor_rocket_init(&r, &d->vehicle))) return rc;
  m = ptor_rocket_model(&r);
  grid = grid_nodes(d, tau);
  rc = dense_audit_with(&m, grid, d->nodes, x, u, substeps, max_pointwise_g, total_y_increase,
                        interval_y_increase, samples);
  free(grid);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* pipg.hpp                                                                   */
/* ------------------------------------------------------------------------- */

double ptor_step_sizes(double lambda, double omega, double sigma, double* beta) { /* :335-340 */
  const double alpha = 2.0 / (lambda + sqrt(lambda * lambda + 4.0 * omega * sigma));
  if (beta) *beta = omega * alpha;
  return alpha;
}

static double sq_norm(const double* v, int n) { /* group_sq_norm, :156-162 */
  double acc = 0.0;
  for (int i = 0; i < n; ++i) acc += v[i] * v[i];
  return acc;
}

static double inf_norm_n(const double* v, int n) { /* group_inf, :164-170 */
  double m = 0.0;
  for (int i = 0; i < n; ++i) m = dmax(m, fabs(v[i]));
  return m;
}

static double inf_diff_n(const double* a, const double* b, int n) { /* group_inf_diff, :172-178 */
  double m = 0.0;
  for (int i = 0; i < n; ++i) m = dmax(m, fabs(a[i] - b[i]));
  return m;
}

static double dot_n(const double* x, const double* y, int n) { /* smallmat.hpp:145-153 */
  double acc = 0.0;
  for (int i = 0; i < n; ++i) acc += x[i] * y[i];
  return acc;
}

/* Materialises A_plus = -I when the caller passes NULL. */
static const double* a_plus_or_negI(const ptopt_subproblem_shape* s, const double* A_plus,
                                    double** owned) {
  const int nx = s->n_x, m = s->nodes - 1;
  double* ap;
  *owned = NULL;
  if (A_plus) return A_plus;
  ap = (double*)calloc((size_t)m * nx * nx, sizeof(double));
  for (int k = 0; k < m; ++k)
    for (int i = 0; i < nx; ++i) ap[(k * nx + i) * nx + i] = -1.0;
  *owned = ap;
  return ap;
}

int ptor_power_iteration_ex(const ptopt_subproblem_shape* shape, const ptopt_subproblem_arrays* a,
                            const double* seed_x, const double* seed_u, const double* seed_vcp,
                            const double* seed_vcn, double eps_abs, double eps_rel,
                            double eps_buff, int j_max, double* sigma_out, int* trips) {
  /* power_iteration_custom, :206-292 */
  const int nx = shape->n_x, nu = shape->n_u, n = shape->nodes, m = n - 1;
  const double* e_y = shape->e_y;
  double *owned, *x, *u, *vcp, *vcn, *phi, *theta;
  const double* Ap = a_plus_or_negI(shape, a->A_plus, &owned);
  double sigma, sigma_star, r[PTOR_MAX_X], t[PTOR_MAX_X], ru[PTOR_MAX_U], tu[PTOR_MAX_U];
  int j, rc = 0, done_trips = 0;

  x = (double*)malloc(sizeof(double) * (size_t)(n * nx));
  u = (double*)malloc(sizeof(double) * (size_t)(n * nu));
  vcp = (double*)malloc(sizeof(double) * (size_t)(m * nx));
  vcn = (double*)malloc(sizeof(double) * (size_t)(m * nx));
  phi = (double*)calloc((size_t)(m * nx), sizeof(double));
  theta = (double*)calloc((size_t)m, sizeof(double));
  memcpy(x, seed_x, sizeof(double) * (size_t)(n * nx));
  memcpy(u, seed_u, sizeof(double) * (size_t)(n * nu));
  memcpy(vcp, seed_vcp, sizeof(double) * (size_t)(m * nx));
  memcpy(vcn, seed_vcn, sizeof(double) * (size_t)(m * nx));

  sigma = sq_norm(x, n * nx) + sq_norm(u, n * nu) + sq_norm(vcp, m * nx) + sq_norm(vcn, m * nx);
  if (sigma == 0.0) {
    rc = PTOPT_ST_POWER_SEED_ZERO;
    goto out;
  }
  sigma = sqrt(sigma);
  sigma_star = sigma;

  for (j = 1; j <= j_max; ++j) {
    done_trips = j;
    for (int k = 0; k < m; ++k) { /* forward map scaled by 1/sigma, :234-245 */
      mat_vec(a->A_minus + k * nx * nx, nx, nx, x + k * nx, 0, r);
      mat_vec(Ap + k * nx * nx, nx, nx, x + (k + 1) * nx, 0, t);
      vec_add_scaled(r, 1.0, t, nx);
      mat_vec(a->B_minus + k * nx * nu, nx, nu, u + k * nu, 0, t);
      vec_add_scaled(r, 1.0, t, nx);
      mat_vec(a->B_plus + k * nx * nu, nx, nu, u + (k + 1) * nu, 0, t);
      vec_add_scaled(r, 1.0, t, nx);
      vec_add_scaled(r, 1.0, vcp + k * nx, nx);
      vec_add_scaled(r, -1.0, vcn + k * nx, nx);
      for (int i = 0; i < nx; ++i) r[i] *= 1.0 / sigma;
      for (int i = 0; i < nx; ++i) phi[k * nx + i] = r[i];
      theta[k] = (dot_n(e_y, x + (k + 1) * nx, nx) - dot_n(e_y, x + k * nx, nx)) / sigma;
    }
    /* adjoint map, :247-275 */
    mat_vec(a->A_minus, nx, nx, phi, 1, r);
    vec_add_scaled(r, -theta[0], e_y, nx);
    for (int i = 0; i < nx; ++i) x[i] = r[i];
    mat_vec(a->B_minus, nx, nu, phi, 1, ru);
    for (int i = 0; i < nu; ++i) u[i] = ru[i];
    for (int i = 0; i < nx; ++i) {
      vcp[i] = phi[i];
      vcn[i] = phi[i];
      vcn[i] *= -1.0;
    }
    for (int k = 1; k < m; ++k) {
      mat_vec(a->A_minus + k * nx * nx, nx, nx, phi + k * nx, 1, r);
      mat_vec(Ap + (k - 1) * nx * nx, nx, nx, phi + (k - 1) * nx, 1, t);
      vec_add_scaled(r, 1.0, t, nx);
      vec_add_scaled(r, -theta[k], e_y, nx);
      vec_add_scaled(r, theta[k - 1], e_y, nx);
      for (int i = 0; i < nx; ++i) x[k * nx + i] = r[i];
      mat_vec(a->B_minus + k * nx * nu, nx, nu, phi + k * nx, 1, ru);
      mat_vec(a->B_plus + (k - 1) * nx * nu, nx, nu, phi + (k - 1) * nx, 1, tu);
      vec_add_scaled(ru, 1.0, tu, nu);
      for (int i = 0; i < nu; ++i) u[k * nu + i] = ru[i];
      for (int i = 0; i < nx; ++i) {
        vcp[k * nx + i] = phi[k * nx + i];
        vcn[k * nx + i] = phi[k * nx + i];
        vcn[k * nx + i] *= -1.0;
      }
    }
    mat_vec(Ap + (m - 1) * nx * nx, nx, nx, phi + (m - 1) * nx, 1, r);
    vec_add_scaled(r, theta[m - 1], e_y, nx);
    for (int i = 0; i < nx; ++i) x[(n - 1) * nx + i] = r[i];
    mat_vec(a->B_plus + (m - 1) * nx * nu, nx, nu, phi + (m - 1) * nx, 1, ru);
    for (int i = 0; i < nu; ++i) u[(n - 1) * nu + i] = ru[i];

    sigma_star =
        sq_norm(x, n * nx) + sq_norm(u, n * nu) + sq_norm(vcp, m * nx) + sq_norm(vcn, m * nx);
    sigma_star = sqrt(sigma_star);
    if (sigma_star == 0.0) {
      sigma = 0.0;
      break;
    }
    if (fabs(sigma_star - sigma) <= eps_abs + eps_rel * dmax(sigma_star, sigma)) {
      sigma = sigma_star;
      break;
    }
    sigma = sigma_star;
  }
  *sigma_out = (1.0 + eps_buff) * sigma;
out:
  if (trips) *trips = done_trips;
  free(x); free(u); free(vcp); free(vcn); free(phi); free(theta); free(owned);
  return rc;
}

int ptor_power_iteration(const ptopt_subproblem_shape* shape, const ptopt_subproblem_arrays* a,
                         const double* seed_x, const double* seed_u, const double* seed_vcp,
                         const double* seed_vcn, double eps_abs, double eps_rel, double eps_buff,
                         int j_max, double* sigma) {
  return ptor_power_iteration_ex(shape, a, seed_x, seed_u, seed_vcp, seed_vcn, eps_abs, eps_rel,
                                 eps_buff, j_max, sigma, NULL);
}

static int pipg_config_valid(const ptopt_pipg_config* c) { /* :31-37 */
  if (!(c->omega > 0.0)) return 0;
  if (!(c->rho > 0.0 && c->rho < 2.0)) return 0;
  if (c->j_check < 1) return 0;
  if (c->j_max < 1) return 0;
  if (!(c->eps_buff >= 0.0)) return 0;
  return 1;
}

int ptor_pipg(const ptopt_subproblem_shape* shape, const ptopt_subproblem_arrays* a,
              const ptopt_pipg_config* cfg, double sigma, const ptopt_workspace_arrays* w,
              int* iterations, int* converged, int* fail_index) { /* pipg_custom, :350-497 */
  const int nx = shape->n_x, nu = shape->n_u, n = shape->nodes, m = n - 1;
  const int NXn = n * nx, NUn = n * nu, NM = m * nx;
  const double* e_y = shape->e_y;
  const double w_prox = shape->w_prox, w_ep = shape->w_ep, w_cost = shape->w_cost;
  double alpha, beta, rho;
  double *owned, *buf;
  double *x_cur, *x_prev, *x_ex, *u_cur, *u_prev, *u_ex, *vp_cur, *vp_prev, *vp_ex, *vn_cur,
      *vn_prev, *vn_ex, *ph_cur, *ph_prev, *ph_ex, *th_cur, *th_prev, *th_ex;
  const double* Ap;
  int rc = 0, iters = 0, conv = 0;
  size_t total;
  if (!pipg_config_valid(cfg)) return -1;
  Ap = a_plus_or_negI(shape, a->A_plus, &owned);
  alpha = ptor_step_sizes(w_prox, cfg->omega, sigma, &beta);
  rho = cfg->rho;

  total = 3u * (size_t)(NXn + NUn + 3 * NM + m);
  buf = (double*)calloc(total, sizeof(double));
  {
    double* p = buf;
#define TAKE(ptr, len) ptr = p; p += (len)
    TAKE(x_cur, NXn); TAKE(x_prev, NXn); TAKE(x_ex, NXn);
    TAKE(u_cur, NUn); TAKE(u_prev, NUn); TAKE(u_ex, NUn);
    TAKE(vp_cur, NM); TAKE(vp_prev, NM); TAKE(vp_ex, NM);
    TAKE(vn_cur, NM); TAKE(vn_prev, NM); TAKE(vn_ex, NM);
    TAKE(ph_cur, NM); TAKE(ph_prev, NM); TAKE(ph_ex, NM);
    TAKE(th_cur, m); TAKE(th_prev, m); TAKE(th_ex, m);
#undef TAKE
  }
  memcpy(x_ex, w->x, sizeof(double) * (size_t)NXn);
  memcpy(u_ex, w->u, sizeof(double) * (size_t)NUn);
  memcpy(vp_ex, w->vc_pos, sizeof(double) * (size_t)NM);
  memcpy(vn_ex, w->vc_neg, sizeof(double) * (size_t)NM);
  memcpy(ph_ex, w->dyn_dual, sizeof(double) * (size_t)NM);
  memcpy(th_ex, w->relax_dual, sizeof(double) * (size_t)m);
  memcpy(x_cur, x_ex, sizeof(double) * (size_t)NXn);
  memcpy(u_cur, u_ex, sizeof(double) * (size_t)NUn);
  memcpy(vp_cur, vp_ex, sizeof(double) * (size_t)NM);
  memcpy(vn_cur, vn_ex, sizeof(double) * (size_t)NM);
  memcpy(ph_cur, ph_ex, sizeof(double) * (size_t)NM);
  memcpy(th_cur, th_ex, sizeof(double) * (size_t)m);

  for (int j = 1; j <= cfg->j_max; ++j) {
    double* sw;
#define SWAP(a_, b_) sw = a_; a_ = b_; b_ = sw
    SWAP(x_cur, x_prev); SWAP(u_cur, u_prev); SWAP(vp_cur, vp_prev);
    SWAP(vn_cur, vn_prev); SWAP(ph_cur, ph_prev); SWAP(th_cur, th_prev);
#undef SWAP
    /* projected gradient step on the primal variables, :388-420 */
    for (int k = 0; k < n; ++k) {
      double grad[PTOR_MAX_X], grad_u[PTOR_MAX_U], t[PTOR_MAX_X];
      double* xk = x_cur + k * nx;
      double* uk = u_cur + k * nu;
      for (int i = 0; i < nx; ++i) grad[i] = x_ex[k * nx + i] * w_prox;
      for (int i = 0; i < nu; ++i) grad_u[i] = u_ex[k * nu + i] * w_prox;
      if (k < m) {
        mat_vec(a->A_minus + k * nx * nx, nx, nx, ph_ex + k * nx, 1, t);
        vec_add_scaled(grad, 1.0, t, nx);
        vec_add_scaled(grad, -th_ex[k], e_y, nx);
        mat_vec(a->B_minus + k * nx * nu, nx, nu, ph_ex + k * nx, 1, t);
        vec_add_scaled(grad_u, 1.0, t, nu);
      }
      if (k > 0) {
        mat_vec(Ap + (k - 1) * nx * nx, nx, nx, ph_ex + (k - 1) * nx, 1, t);
        vec_add_scaled(grad, 1.0, t, nx);
        vec_add_scaled(grad, th_ex[k - 1], e_y, nx);
        mat_vec(a->B_plus + (k - 1) * nx * nu, nx, nu, ph_ex + (k - 1) * nx, 1, t);
        vec_add_scaled(grad_u, 1.0, t, nu);
      }
      if (k == n - 1) vec_add_scaled(grad, w_cost, shape->e_cost, nx);

      for (int i = 0; i < nx; ++i) xk[i] = x_ex[k * nx + i];
      vec_add_scaled(xk, -alpha, grad, nx);
      if (k == 0)
        for (int i = 0; i < shape->n_init_fix; ++i) xk[shape->init_fix_idx[i]] = a->init_fix_val[i];
      if (k == n - 1)
        for (int i = 0; i < shape->n_final_fix; ++i)
          xk[shape->final_fix_idx[i]] = a->final_fix_val[i];

      for (int i = 0; i < nu; ++i) uk[i] = u_ex[k * nu + i];
      vec_add_scaled(uk, -alpha, grad_u, nu);
      for (int i = 0; i < nu; ++i)
        uk[i] = dmax(a->u_min[k * nu + i], dmin(a->u_max[k * nu + i], uk[i]));
    }
    /* virtual-control slacks, :423-430 */
    for (int k = 0; k < m; ++k)
      for (int i = 0; i < nx; ++i) {
        vp_cur[k * nx + i] = dmax(0.0, vp_ex[k * nx + i] - alpha * (w_ep + ph_ex[k * nx + i]));
        vn_cur[k * nx + i] = dmax(0.0, vn_ex[k * nx + i] - alpha * (w_ep - ph_ex[k * nx + i]));
      }
    /* dual updates, :433-458 */
    for (int k = 0; k < m; ++k) {
      double rx[PTOR_MAX_X], rx1[PTOR_MAX_X], ru[PTOR_MAX_U], ru1[PTOR_MAX_U], resid[PTOR_MAX_X],
          t[PTOR_MAX_X], drift;
      for (int i = 0; i < nx; ++i) {
        rx[i] = 2.0 * x_cur[k * nx + i] - x_ex[k * nx + i];
        rx1[i] = 2.0 * x_cur[(k + 1) * nx + i] - x_ex[(k + 1) * nx + i];
      }
      for (int i = 0; i < nu; ++i) {
        ru[i] = 2.0 * u_cur[k * nu + i] - u_ex[k * nu + i];
        ru1[i] = 2.0 * u_cur[(k + 1) * nu + i] - u_ex[(k + 1) * nu + i];
      }
      mat_vec(a->A_minus + k * nx * nx, nx, nx, rx, 0, resid);
      mat_vec(Ap + k * nx * nx, nx, nx, rx1, 0, t);
      vec_add_scaled(resid, 1.0, t, nx);
      mat_vec(a->B_minus + k * nx * nu, nx, nu, ru, 0, t);
      vec_add_scaled(resid, 1.0, t, nx);
      mat_vec(a->B_plus + k * nx * nu, nx, nu, ru1, 0, t);
      vec_add_scaled(resid, 1.0, t, nx);
      for (int i = 0; i < nx; ++i)
        resid[i] += (2.0 * vp_cur[k * nx + i] - vp_ex[k * nx + i]) -
                    (2.0 * vn_cur[k * nx + i] - vn_ex[k * nx + i]) + a->w[k * nx + i];
      for (int i = 0; i < nx; ++i) ph_cur[k * nx + i] = ph_ex[k * nx + i];
      vec_add_scaled(ph_cur + k * nx, beta, resid, nx);
      drift = dot_n(e_y, rx1, nx) - dot_n(e_y, rx, nx) - a->eps_relax[k];
      th_cur[k] = dmax(0.0, th_ex[k] + beta * drift);
    }
    /* extrapolation, :461-472 */
    for (int i = 0; i < NXn; ++i) x_ex[i] = (1.0 - rho) * x_ex[i] + rho * x_cur[i];
    for (int i = 0; i < NUn; ++i) u_ex[i] = (1.0 - rho) * u_ex[i] + rho * u_cur[i];
    for (int i = 0; i < NM; ++i) vp_ex[i] = (1.0 - rho) * vp_ex[i] + rho * vp_cur[i];
    for (int i = 0; i < NM; ++i) vn_ex[i] = (1.0 - rho) * vn_ex[i] + rho * vn_cur[i];
    for (int i = 0; i < NM; ++i) ph_ex[i] = (1.0 - rho) * ph_ex[i] + rho * ph_cur[i];
    for (int i = 0; i < m; ++i) th_ex[i] = (1.0 - rho) * th_ex[i] + rho * th_cur[i];

    iters = j;
    if (j % cfg->j_check == 0) { /* :475-487 with stopping_custom :307-326 */
      double z_cur, z_prev, z_delta, r_cur, r_prev, r_delta;
      if (!all_finite(x_cur, NXn) || !all_finite(u_cur, NUn) || !all_finite(ph_cur, NM)) {
        rc = PTOPT_ST_SOLVER_DIVERGED;
        if (fail_index) *fail_index = j;
        goto out;
      }
      z_cur = dmax(dmax(inf_norm_n(x_cur, NXn), inf_norm_n(u_cur, NUn)),
                   dmax(inf_norm_n(vp_cur, NM), inf_norm_n(vn_cur, NM)));
      z_prev = dmax(dmax(inf_norm_n(x_prev, NXn), inf_norm_n(u_prev, NUn)),
                    dmax(inf_norm_n(vp_prev, NM), inf_norm_n(vn_prev, NM)));
      z_delta = dmax(dmax(inf_diff_n(x_cur, x_prev, NXn), inf_diff_n(u_cur, u_prev, NUn)),
                     dmax(inf_diff_n(vp_cur, vp_prev, NM), inf_diff_n(vn_cur, vn_prev, NM)));
      r_cur = dmax(inf_norm_n(ph_cur, NM), inf_norm_n(th_cur, m));
      r_prev = dmax(inf_norm_n(ph_prev, NM), inf_norm_n(th_prev, m));
      r_delta = dmax(inf_diff_n(ph_cur, ph_prev, NM), inf_diff_n(th_cur, th_prev, m));
      if (z_delta <= cfg->eps_abs + cfg->eps_rel * dmax(z_cur, z_prev) &&
          r_delta <= cfg->eps_abs + cfg->eps_rel * dmax(r_cur, r_prev)) {
        conv = 1;
        break;
      }
    }
  }
  memcpy(w->x, x_cur, sizeof(double) * (size_t)NXn);
  memcpy(w->u, u_cur, sizeof(double) * (size_t)NUn);
  memcpy(w->vc_pos, vp_cur, sizeof(double) * (size_t)NM);
  memcpy(w->vc_neg, vn_cur, sizeof(double) * (size_t)NM);
  memcpy(w->dyn_dual, ph_cur, sizeof(double) * (size_t)NM);
  memcpy(w->relax_dual, th_cur, sizeof(double) * (size_t)m);
out:
  if (iterations) *iterations = iters;
  if (converged) *converged = conv;
  free(buf);
  free(owned);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* scp.hpp                                                                    */
/* ------------------------------------------------------------------------- */

double ptor_pow2_near(double v) { return exp2(round(log2(v))); } /* :39-42 */

static uint64_t splitmix64_next(uint64_t* state) { /* :239-245 */
  uint64_t z;
  *state += 0x9e3779b97f4a7c15ull;
  z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static double unit_interval(uint64_t bits) { return (double)(bits >> 11) * 0x1.0p-53; } /* :247-249 */

void ptor_scp_seed(uint64_t rng_seed, int nodes, double* seed_x, double* seed_u) { /* :303-321 */
  uint64_t state = rng_seed ^ 0x5bf03635d78b41adull;
  double norm_sq = 0.0, inv;
  for (int i = 0; i < nodes * NX; ++i) {
    seed_x[i] = 2.0 * unit_interval(splitmix64_next(&state)) - 1.0;
    norm_sq += seed_x[i] * seed_x[i];
  }
  for (int i = 0; i < nodes * NU; ++i) {
    seed_u[i] = 2.0 * unit_interval(splitmix64_next(&state)) - 1.0;
    norm_sq += seed_u[i] * seed_u[i];
  }
  inv = 1.0 / sqrt(norm_sq);
  for (int i = 0; i < nodes * NX; ++i) seed_x[i] *= inv;
  for (int i = 0; i < nodes * NU; ++i) seed_u[i] *= inv;
}

static void shape_of_problem(const ptopt_problem_desc* d, ptopt_subproblem_shape* s) {
  memset(s, 0, sizeof *s);
  s->n_x = NX;
  s->n_u = NU;
  s->nodes = d->nodes;
  s->n_init_fix = NX;
  s->n_final_fix = d->n_final_fix;
  for (int i = 0; i < NX; ++i) s->init_fix_idx[i] = i;
  for (int i = 0; i < d->n_final_fix; ++i) s->final_fix_idx[i] = d->final_fix_idx[i];
  s->e_y[NX - 1] = 1.0;
  for (int i = 0; i < NX; ++i) s->e_cost[i] = d->px[i] * d->e_cost[i];
  s->w_cost = d->w_cost;
  s->w_prox = d->w_prox;
  s->w_ep = d->w_ep;
}

int ptor_assemble(const ptopt_problem_desc* d, const double* tau, const double* init_state,
                  const double* x, const double* u, const double* A, const double* Bm,
                  const double* Bp, const double* x_end, double* A_minus, double* A_plus,
                  double* B_minus, double* B_plus, double* w_hat, double* eps_relax, double* u_min,
                  double* u_max, double* init_fix_val, double* final_fix_val, double* e_cost_hat) {
  /* assemble_subproblem, :139-217 */
  const int n = d->nodes, m = n - 1;
  double px_inv[NX], pu_inv[NU];
  (void)tau;
  for (int i = 0; i < NX; ++i) {
    if (!(d->px[i] > 0.0)) return -1;
    px_inv[i] = 1.0 / d->px[i];
  }
  for (int i = 0; i < NU; ++i) {
    if (!(d->pu[i] > 0.0)) return -1;
    pu_inv[i] = 1.0 / d->pu[i];
  }
  for (int k = 0; k < m; ++k) {
    for (int i = 0; i < NX; ++i) {
      for (int j = 0; j < NX; ++j) {
        A_minus[(k * NX + i) * NX + j] = px_inv[i] * A[(k * NX + i) * NX + j] * d->px[j];
        if (A_plus) A_plus[(k * NX + i) * NX + j] = (i == j) ? -1.0 : 0.0;
      }
      for (int j = 0; j < NU; ++j) {
        B_minus[(k * NX + i) * NU + j] = px_inv[i] * Bm[(k * NX + i) * NU + j] * d->pu[j];
        B_plus[(k * NX + i) * NU + j] = px_inv[i] * Bp[(k * NX + i) * NU + j] * d->pu[j];
      }
    }
    for (int i = 0; i < NX; ++i)
      w_hat[k * NX + i] = px_inv[i] * (x_end[k * NX + i] - x[(k + 1) * NX + i]);
    {
      const double dy = x[(k + 1) * NX + NX - 1] - x[k * NX + NX - 1];
      eps_relax[k] = d->epsilon_relax * px_inv[NX - 1] - px_inv[NX - 1] * dy;
    }
  }
  for (int k = 0; k < n; ++k) {
    const double s_bar = u[k * NU + NU - 1];
    for (int i = 0; i < NU - 1; ++i) {
      u_min[k * NU + i] = -INFINITY;
      u_max[k * NU + i] = INFINITY;
    }
    u_min[k * NU + NU - 1] = pu_inv[NU - 1] * (d->s_min - s_bar);
    u_max[k * NU + NU - 1] = pu_inv[NU - 1] * (d->s_max - s_bar);
  }
  for (int i = 0; i < NX; ++i) {
    const double target = i < NXI ? init_state[i] : 0.0;
    init_fix_val[i] = px_inv[i] * (target - x[i]);
  }
  for (int i = 0; i < d->n_final_fix; ++i) {
    const int idx = d->final_fix_idx[i];
    final_fix_val[i] = px_inv[idx] * (d->final_fix_val[i] - x[(n - 1) * NX + idx]);
  }
  if (e_cost_hat)
    for (int i = 0; i < NX; ++i) e_cost_hat[i] = d->px[i] * d->e_cost[i];
  return 0;
}

static int scp_valid(const ptopt_problem_desc* d) { /* ScpProblem::validate, :111-120 */
  if (!(d->w_cost >= 0.0) || !(d->w_prox > 0.0) || !(d->w_ep > 0.0) || !(d->epsilon_relax > 0.0))
    return 0;
  if (!pipg_config_valid(&d->pipg)) return 0;
  if (!(d->s_min > 0.0) || !(d->s_min <= d->s_max)) return 0;
  if (d->max_iters < 1 || d->integrator_steps < 1) return 0;
  return 1;
}

int ptor_scp_solve_ex(const ptopt_problem_desc* d, const double* tau, const double* init_state,
                      const double* x_guess, const double* u_guess, uint64_t rng_seed,
                      double* x_out, double* u_out, int* scp_iterations, int* converged,
                      double* final_defect_inf, double* history, int* power_trips,
                      int* fail_index) { /* scp_solve, :256-364 */
  const int n = d->nodes, m = n - 1;
  ptor_rocket rk;
  ptor_model model;
  ptopt_subproblem_shape shape;
  ptopt_subproblem_arrays arr;
  ptopt_workspace_arrays ws;
  double *grid, *zx, *zu, *A, *Bm, *Bp, *w, *xe, *Am, *Bmh, *Bph, *wh, *eps, *umin, *umax, *wsb,
      *seed_x, *seed_u;
  double init_val[NX], final_val[NX], px_inv[NX];
  double last_step = INFINITY, defect_final = INFINITY;
  int solves = 0, conv = 0, rc = 0;
  if (!scp_valid(d)) return -1;
  if ((rc = ptor_rocket_init(&rk, &d->vehicle))) return rc;
  model = ptor_rocket_model(&rk);
  shape_of_problem(d, &shape);
  for (int i = 0; i < NX; ++i) px_inv[i] = 1.0 / d->px[i];

  grid = grid_nodes(d, tau);
  zx = (double*)malloc(sizeof(double) * (size_t)(n * NX));
  zu = (double*)malloc(sizeof(double) * (size_t)(n * NU));
  memcpy(zx, x_guess, sizeof(double) * (size_t)(n * NX));
  memcpy(zu, u_guess, sizeof(double) * (size_t)(n * NU));
  A = (double*)malloc(sizeof(double) * (size_t)(m * NX * NX));
  Bm = (double*)malloc(sizeof(double) * (size_t)(m * NX * NU));
  Bp = (double*)malloc(sizeof(double) * (size_t)(m * NX * NU));
  w = (double*)malloc(sizeof(double) * (size_t)(m * NX));
  xe = (double*)malloc(sizeof(double) * (size_t)(m * NX));
  Am = (double*)malloc(sizeof(double) * (size_t)(m * NX * NX));
  Bmh = (double*)malloc(sizeof(double) * (size_t)(m * NX * NU));
  Bph = (double*)malloc(sizeof(double) * (size_t)(m * NX * NU));
  wh = (double*)malloc(sizeof(double) * (size_t)(m * NX));
  eps = (double*)malloc(sizeof(double) * (size_t)m);
  umin = (double*)malloc(sizeof(double) * (size_t)(n * NU));
  umax = (double*)malloc(sizeof(double) * (size_t)(n * NU));
  wsb = (double*)calloc((size_t)(n * (NX + NU) + m * (3 * NX + 1)), sizeof(double));
  seed_x = (double*)malloc(sizeof(double) * (size_t)(n * NX));
  seed_u = (double*)malloc(sizeof(double) * (size_t)(n * NU));
  ws.x = wsb;
  ws.u = ws.x + n * NX;
  ws.vc_pos = ws.u + n * NU;
  ws.vc_neg = ws.vc_pos + m * NX;
  ws.dyn_dual = ws.vc_neg + m * NX;
  ws.relax_dual = ws.dyn_dual + m * NX;
  arr.A_minus = Am;
  arr.A_plus = NULL;
  arr.B_minus = Bmh;
  arr.B_plus = Bph;
  arr.w = wh;
  arr.eps_relax = eps;
  arr.u_min = umin;
  arr.u_max = umax;
  arr.init_fix_val = init_val;
  arr.final_fix_val = final_val;

  for (;;) {
    double defect_inf = 0.0, defect_l1 = 0.0, iterate_cost, sigma, step = 0.0;
    int pipg_iters = 0, pipg_conv = 0, trips = 0, all_zero = 1;
    if ((rc = linearize_with(&model, grid, n, d->integrator_steps, zx, zu, A, Bm, Bp, w, xe,
                             fail_index)))
      break;
    for (int k = 0; k < m; ++k)
      for (int i = 0; i < NX; ++i) {
        const double diff = fabs(xe[k * NX + i] - zx[(k + 1) * NX + i]);
        defect_inf = dmax(defect_inf, px_inv[i] * diff);
        defect_l1 += diff;
      }
    defect_final = defect_inf;
    iterate_cost = d->w_cost * dot_n(zx + (n - 1) * NX, d->e_cost, NX) + d->w_ep * defect_l1;
    if (defect_inf <= d->tol_feas && last_step <= d->tol_step) {
      conv = 1;
      break;
    }
    if (solves == d->max_iters) break;

    if ((rc = ptor_assemble(d, tau, init_state, zx, zu, A, Bm, Bp, xe, Am, NULL, Bmh, Bph, wh, eps,
                            umin, umax, init_val, final_val, NULL)))
      break;

    for (int i = 0; i < n * (NX + NU) + 2 * m * NX; ++i) /* primal_all_zero, pipg.hpp:143-151 */
      if (wsb[i] != 0.0) {
        all_zero = 0;
        break;
      }
    if (all_zero) {
      ptor_scp_seed(rng_seed, n, seed_x, seed_u);
      rc = ptor_power_iteration_ex(&shape, &arr, seed_x, seed_u, ws.vc_pos, ws.vc_neg,
                                   d->power_eps_abs, d->power_eps_rel, d->pipg.eps_buff,
                                   d->power_j_max, &sigma, &trips);
    } else {
      rc = ptor_power_iteration_ex(&shape, &arr, ws.x, ws.u, ws.vc_pos, ws.vc_neg,
                                   d->power_eps_abs, d->power_eps_rel, d->pipg.eps_buff,
                                   d->power_j_max, &sigma, &trips);
    }
    if (rc) break;
    if ((rc = ptor_pipg(&shape, &arr, &d->pipg, sigma, &ws, &pipg_iters, &pipg_conv, fail_index)))
      break;
    (void)pipg_conv;

    for (int k = 0; k < n; ++k) {
      step = dmax(step, inf_norm_n(ws.x + k * NX, NX));
      step = dmax(step, inf_norm_n(ws.u + k * NU, NU));
    }
    for (int k = 0; k < n; ++k) {
      double* xk = zx + k * NX;
      double* uk = zu + k * NU;
      for (int i = 0; i < NX; ++i) xk[i] += d->px[i] * ws.x[k * NX + i];
      for (int i = 0; i < NU; ++i) uk[i] += d->pu[i] * ws.u[k * NU + i];
      if (d->renormalize_quaternion) { /* rocket_problem.hpp:86-92 */
        double nq = 0.0;
        for (int i = 0; i < 4; ++i) nq += xk[K_ATT + i] * xk[K_ATT + i];
        nq = sqrt(nq);
        if (nq > 0.0)
          for (int i = 0; i < 4; ++i) xk[K_ATT + i] /= nq;
      }
    }
    if (history) {
      double* e = history + solves * PTOPT_HISTORY_FIELDS;
      e[0] = defect_inf;
      e[1] = step;
      e[2] = iterate_cost;
      e[3] = (double)pipg_iters;
      e[4] = sigma;
    }
    if (power_trips) power_trips[solves] = trips;
    ++solves;
    last_step = step;
  }

  if (!rc) {
    memcpy(x_out, zx, sizeof(double) * (size_t)(n * NX));
    memcpy(u_out, zu, sizeof(double) * (size_t)(n * NU));
    *scp_iterations = solves;
    *converged = conv;
    *final_defect_inf = defect_final;
  }
  free(grid); free(zx); free(zu); free(A); free(Bm); free(Bp); free(w); free(xe); free(Am);
  free(Bmh); free(Bph); free(wh); free(eps); free(umin); free(umax); free(wsb); free(seed_x);
  free(seed_u);
  return rc;
}

int ptor_scp_solve(const ptopt_problem_desc* d, const double* tau, const double* init_state,
                   const double* x_guess, const double* u_guess, uint64_t rng_seed, double* x_out,
                   double* u_out, int* scp_iterations, int* converged, double* final_defect_inf,
                   double* history, int* fail_index) {
  return ptor_scp_solve_ex(d, tau, init_state, x_guess, u_guess, rng_seed, x_out, u_out,
                           scp_iterations, converged, final_defect_inf, history, NULL, fail_index);
}

/* ------------------------------------------------------------------------- */
/* montecarlo.hpp + rocket_problem.hpp: instance generation and batch harness */
/* ------------------------------------------------------------------------- */

static uint64_t splitmix64_mix(uint64_t x) { /* montecarlo.hpp:35-40 */
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

static double counter_uniform(uint64_t seed, uint64_t run, uint64_t slot) { /* :43-46 */
  const uint64_t key = splitmix64_mix(seed ^ splitmix64_mix(run + 1));
  return (double)(splitmix64_mix(key + slot) >> 11) * 0x1.0p-53;
}

uint64_t ptor_run_seed(uint64_t batch_seed, int run_id) { /* :51-53 */
  return splitmix64_mix(batch_seed ^ splitmix64_mix((uint64_t)run_id));
}

void ptor_disperse(const double* r_low, const double* r_high, uint64_t seed, int run_id,
                   double* r_out) { /* :55-65 */
  for (int i = 0; i < 3; ++i) {
    const double u = counter_uniform(seed, (uint64_t)run_id, (uint64_t)i);
    r_out[i] = r_low[i] + (r_high[i] - r_low[i]) * u;
  }
}

static void slerp(const double* qa, const double* qb_in, double t, double* q) {
  /* rocket_problem.hpp:98-120 */
  double qb[4] = {qb_in[0], qb_in[1], qb_in[2], qb_in[3]};
  double d = qa[0] * qb[0] + qa[1] * qb[1] + qa[2] * qb[2] + qa[3] * qb[3];
  double nq = 0.0;
  if (d < 0.0) {
    for (int i = 0; i < 4; ++i) qb[i] = -qb[i];
    d = -d;
  }
  if (d > 1.0 - 1e-10) {
    for (int i = 0; i < 4; ++i) q[i] = (1.0 - t) * qa[i] + t * qb[i];
  } else {
    const double ang = acos(dmin(1.0, d));
    const double sa = sin(ang);
    const double ca = sin((1.0 - t) * ang) / sa;
    const double cb = sin(t * ang) / sa;
    for (int i = 0; i < 4; ++i) q[i] = ca * qa[i] + cb * qb[i];
  }
  for (int i = 0; i < 4; ++i) nq += q[i] * q[i];
  nq = sqrt(nq);
  for (int i = 0; i < 4; ++i) q[i] /= nq;
}

/* Terminal targets by model-state slot; unpinned slots default as RocketBoundary does
 * (rocket_problem.hpp:51-57). */
static void final_targets(const ptopt_problem_desc* d, double* fin /*[14]*/) {
  for (int i = 0; i < NXI; ++i) fin[i] = 0.0;
  fin[K_ATT + 3] = 1.0;
  for (int i = 0; i < d->n_final_fix; ++i)
    if (d->final_fix_idx[i] >= 0 && d->final_fix_idx[i] < NXI)
      fin[d->final_fix_idx[i]] = d->final_fix_val[i];
}

int ptor_initial_guess(const ptopt_problem_desc* d, const double* tau, const double* init_state,
                       double* x, double* u) { /* rocket_problem.hpp:127-163 */
  const int n = d->nodes;
  const ptopt_vehicle_params* p = &d->vehicle;
  const double g_norm = sqrt(p->g_inertial[0] * p->g_inertial[0] +
                             p->g_inertial[1] * p->g_inertial[1] +
                             p->g_inertial[2] * p->g_inertial[2]);
  const double m0 = init_state[K_MASS];
  const double m_end = dmax(p->m_dry, m0 * exp(-p->alpha_mdot * g_norm * d->t_f_guess));
  double fin[NXI];
  double* grid = grid_nodes(d, tau);
  final_targets(d, fin);
  for (int k = 0; k < n; ++k) {
    const double t = grid[k];
    double* xk = x + k * NX;
    double* uk = u + k * NU;
    const double sm = (1.0 - t) * m0 + t * m_end;
    xk[K_MASS] = sm;
    for (int i = 0; i < 3; ++i) {
      xk[K_POS + i] = (1.0 - t) * init_state[K_POS + i] + t * fin[K_POS + i];
      xk[K_VEL + i] = (1.0 - t) * init_state[K_VEL + i] + t * fin[K_VEL + i];
      xk[K_RATE + i] = (1.0 - t) * init_state[K_RATE + i] + t * fin[K_RATE + i];
    }
    slerp(init_state + K_ATT, fin + K_ATT, t, xk + K_ATT);
    xk[NX - 1] = 0.0;
    for (int i = 0; i < 3; ++i) {
      uk[K_THRUST + i] = -sm * p->g_inertial[i];
      uk[K_TORQUE + i] = 0.0;
    }
    uk[NU - 1] = d->t_f_guess;
  }
  free(grid);
  return 0;
}

typedef struct batch_job {
  const ptopt_problem_desc* d;
  const double* tau;
  const double* nominal;
  const double *r_low, *r_high;
  uint64_t seed;
  int batch_size, audit_substeps;
  double *records, *x_out, *u_out;
  int next; /* guarded by lock: the `next.fetch_add` work counter, montecarlo.hpp:153-162 */
  pthread_mutex_t lock;
} batch_job;

static void solve_instance(batch_job* job, int run_id) { /* montecarlo.hpp:100-135 */
  const ptopt_problem_desc* d = job->d;
  const int n = d->nodes;
  double init[NXI], *xg, *ug, *xo, *uo, *hist, *dyk;
  double* rec = job->records + run_id * 8;
  int iters = 0, conv = 0, rc, fail = 0;
  double fdef = 0.0;
  memcpy(init, job->nominal, sizeof init);
  ptor_disperse(job->r_low, job->r_high, job->seed, run_id, init + K_POS);
  xg = (double*)malloc(sizeof(double) * (size_t)(n * NX));
  ug = (double*)malloc(sizeof(double) * (size_t)(n * NU));
  xo = (double*)malloc(sizeof(double) * (size_t)(n * NX));
  uo = (double*)malloc(sizeof(double) * (size_t)(n * NU));
  hist = (double*)calloc((size_t)(d->max_iters * PTOPT_HISTORY_FIELDS), sizeof(double));
  dyk = (double*)malloc(sizeof(double) * (size_t)n);
  ptor_initial_guess(d, job->tau, init, xg, ug);
  memset(rec, 0, sizeof(double) * 8);
  rec[0] = run_id;
  rc = ptor_scp_solve(d, job->tau, init, xg, ug, ptor_run_seed(job->seed, run_id), xo, uo, &iters,
                      &conv, &fdef, hist, &fail);
  if (!rc) {
    double gmax = 0.0, ytot = 0.0, dy_max = 0.0;
    /* assigned before the audit runs (montecarlo.hpp:115-118): they survive an audit failure */
    rec[2] = iters;
    rec[3] = init[K_MASS] - xo[(n - 1) * NX + K_MASS];
    rec[4] = fdef;
    rc = ptor_dense_audit(d, job->tau, xo, uo, job->audit_substeps, &gmax, &ytot, dyk);
    if (!rc) {
      rec[1] = conv;
      rec[5] = gmax;
      for (int k = 0; k + 1 < n; ++k)
        dy_max = dmax(dy_max, xo[(k + 1) * NX + NX - 1] - xo[k * NX + NX - 1]);
      rec[6] = dy_max;
      if (job->x_out && job->u_out) {
        memcpy(job->x_out + (size_t)run_id * n * NX, xo, sizeof(double) * (size_t)(n * NX));
        memcpy(job->u_out + (size_t)run_id * n * NU, uo, sizeof(double) * (size_t)(n * NU));
      }
    }
  }
  if (rc) rec[7] = 1.0;
  free(xg); free(ug); free(xo); free(uo); free(hist); free(dyk);
}

static void* batch_worker(void* arg) {
  batch_job* job = (batch_job*)arg;
  for (;;) {
    int id;
    pthread_mutex_lock(&job->lock);
    id = job->next++;
    pthread_mutex_unlock(&job->lock);
    if (id >= job->batch_size) return NULL;
    solve_instance(job, id);
  }
}

double ptor_run_batch(const ptopt_problem_desc* d, const double* tau,
                      const double* nominal_init_state, const double* r_low, const double* r_high,
                      uint64_t seed, int batch_size, int workers, int audit_substeps,
                      double* records, double* x_out, double* u_out) { /* :140-175 */
  batch_job job;
  struct timespec t0, t1;
  pthread_t* pool;
  if (batch_size < 1 || workers < 1) return -1.0;
  job.d = d;
  job.tau = tau;
  job.nominal = nominal_init_state;
  job.r_low = r_low;
  job.r_high = r_high;
  job.seed = seed;
  job.batch_size = batch_size;
  job.audit_substeps = audit_substeps;
  job.records = records;
  job.x_out = x_out;
  job.u_out = u_out;
  job.next = 0;
  pthread_mutex_init(&job.lock, NULL);
  clock_gettime(CLOCK_MONOTONIC, &t0);
  if (workers == 1) {
    batch_worker(&job);
  } else {
    pool = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)workers);
    for (int i = 0; i < workers; ++i) pthread_create(&pool[i], NULL, batch_worker, &job);
    for (int i = 0; i < workers; ++i) pthread_join(pool[i], NULL);
    free(pool);
  }
  clock_gettime(CLOCK_MONOTONIC, &t1);
  pthread_mutex_destroy(&job.lock);
  return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}

int ptor_abi_version(void) { return PTOPT_ABI_VERSION; }
