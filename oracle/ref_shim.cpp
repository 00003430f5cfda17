// ref_shim.cpp — TEST INFRASTRUCTURE, not product code.
//
// A flat C interface around the UNMODIFIED reference headers
// (/root/reference/proj/include/ptopt/*.hpp, plus tests/support/test_models.hpp
// for the reference's analytic test models).  Built in place by
// oracle/Makefile into oracle/_ref/libptopt_ref.so (git-ignored); nothing from
// the reference is copied into this repository.  Only tests/, smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it.
//
// Error convention: return 0 = ok, >0 = ptopt_instance_status-style code with
// *fail_index set where the reference exception carries an index,
// -1 = std::invalid_argument, -9 = any other exception.

#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "ptopt/ctcs.hpp"
#include "ptopt/discretizer.hpp"
#include "ptopt/montecarlo.hpp"
#include "ptopt/pipg.hpp"
#include "ptopt/rocket6dof.hpp"
#include "ptopt/rocket_problem.hpp"
#include "ptopt/scp.hpp"
#include "ptopt/trajectory.hpp"
#include "support/test_models.hpp"

#include "ptopt_cuda.h"

using namespace ptopt;

namespace {

constexpr int NX = 15, NU = 7;
using Sub = pipg::Subproblem<NX, NU>;
using Wsp = pipg::Workspace<NX, NU>;

template <class F>
int guarded(int* fail_index, F&& body) {
  try {
    body();
    return 0;
  } catch (const PropagationDiverged& e) {
    if (fail_index) *fail_index = e.interval;
    return PTOPT_ST_PROPAGATION_DIVERGED;
  } catch (const pipg::SolverDiverged& e) {
    if (fail_index) *fail_index = e.iteration;
    return PTOPT_ST_SOLVER_DIVERGED;
  } catch (const std::domain_error& e) {
    const std::string msg = e.what();
    if (msg.find("dilation") != std::string::npos) return PTOPT_ST_DILATION_NONPOSITIVE;
    if (msg.find("mass") != std::string::npos) return PTOPT_ST_MASS_NONPOSITIVE;
    if (msg.find("thrust") != std::string::npos) return PTOPT_ST_THRUST_SINGULAR;
    return -8;
  } catch (const std::invalid_argument& e) {
    const std::string msg = e.what();
    if (msg.find("seed point must not be all zero") != std::string::npos)
      return PTOPT_ST_POWER_SEED_ZERO;
    return -1;
  } catch (...) {
    return -9;
  }
}

rocket::VehicleParams vehicle_of(const ptopt_vehicle_params& v) {
  rocket::VehicleParams p;
  p.alpha_mdot = v.alpha_mdot;
  for (int i = 0; i < 3; ++i) p.g_inertial[i] = v.g_inertial[i];
  p.inertia = Mat<3, 3>(3, 3);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) p.inertia(i, j) = v.inertia[i * 3 + j];
  for (int i = 0; i < 3; ++i) p.r_thrust[i] = v.r_thrust[i];
  p.H_theta = Mat<2, 4>(2, 4);
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 4; ++j) p.H_theta(i, j) = v.H_theta[i * 4 + j];
  p.m_dry = v.m_dry;
  p.v_max = v.v_max;
  p.theta_max = v.theta_max;
  p.omega_max = v.omega_max;
  p.delta_max = v.delta_max;
  p.T_min = v.T_min;
  p.T_max = v.T_max;
  p.gamma_max = v.gamma_max;
  return p;
}

Grid grid_of(const ptopt_problem_desc& d, const double* tau) {
  if (!tau) return Grid::uniform(d.nodes);
  return Grid(std::vector<double>(tau, tau + d.nodes));
}

RocketBoundary boundary_of(const ptopt_problem_desc& d, const double* init_state) {
  RocketBoundary bc;
  Vec<14> xi;
  for (int i = 0; i < 14; ++i) xi[i] = init_state ? init_state[i] : 0.0;
  bc.initial = rocket::VehicleState::from_vec(xi);
  // Terminal selectors of the rocket glue: r, v, q, w pinned in this order.
  for (int i = 0; i < d.n_final_fix; ++i) {
    const int idx = d.final_fix_idx[i];
    const double val = d.final_fix_val[i];
    if (idx >= rocket::kPos && idx < rocket::kPos + 3) bc.r_final[idx - rocket::kPos] = val;
    if (idx >= rocket::kVel && idx < rocket::kVel + 3) bc.v_final[idx - rocket::kVel] = val;
    if (idx >= rocket::kAtt && idx < rocket::kAtt + 4) bc.q_final[idx - rocket::kAtt] = val;
    if (idx >= rocket::kRate && idx < rocket::kRate + 3) bc.w_final[idx - rocket::kRate] = val;
  }
  return bc;
}

/// Rebuilds the reference ScpProblem from the flat description.
RocketProblem problem_of(const ptopt_problem_desc& d, const double* tau, const double* init_state,
                         std::uint64_t rng_seed) {
  const RocketBoundary bc = boundary_of(d, init_state);
  RocketProblem pb = make_rocket_problem(vehicle_of(d.vehicle), bc, grid_of(d, tau));
  // make_rocket_problem pins r,v,q,w; honour an explicit selector list instead.
  pb.final_fix_idx.assign(d.final_fix_idx, d.final_fix_idx + d.n_final_fix);
  pb.final_fix_val.assign(d.final_fix_val, d.final_fix_val + d.n_final_fix);
  for (int i = 0; i < NX; ++i) pb.e_cost[i] = d.e_cost[i];
  pb.integrator_steps = d.integrator_steps;
  pb.s_min = d.s_min;
  pb.s_max = d.s_max;
  pb.t_f_guess = d.t_f_guess;
  pb.weights.w_cost = d.w_cost;
  pb.weights.w_prox = d.w_prox;
  pb.weights.w_ep = d.w_ep;
  pb.weights.epsilon_relax = d.epsilon_relax;
  for (int i = 0; i < NX; ++i) {
    pb.scaling.px[i] = d.px[i];
    pb.scaling.px_inv[i] = 1.0 / d.px[i];
  }
  for (int i = 0; i < NU; ++i) {
    pb.scaling.pu[i] = d.pu[i];
    pb.scaling.pu_inv[i] = 1.0 / d.pu[i];
  }
  pb.pipg_cfg.omega = d.pipg.omega;
  pb.pipg_cfg.rho = d.pipg.rho;
  pb.pipg_cfg.j_max = d.pipg.j_max;
  pb.pipg_cfg.j_check = d.pipg.j_check;
  pb.pipg_cfg.eps_abs = d.pipg.eps_abs;
  pb.pipg_cfg.eps_rel = d.pipg.eps_rel;
  pb.pipg_cfg.eps_buff = d.pipg.eps_buff;
  pb.power_j_max = d.power_j_max;
  pb.power_eps_abs = d.power_eps_abs;
  pb.power_eps_rel = d.power_eps_rel;
  pb.tol_feas = d.tol_feas;
  pb.tol_step = d.tol_step;
  pb.max_iters = d.max_iters;
  pb.rng_seed = rng_seed;
  if (!d.renormalize_quaternion) pb.state_post_update = nullptr;
  return pb;
}

RocketTrajectory traj_of(int n, const double* x, const double* u) {
  RocketTrajectory z(n);
  for (int k = 0; k < n; ++k) {
    for (int i = 0; i < NX; ++i) z.x[k][i] = x[k * NX + i];
    for (int i = 0; i < NU; ++i) z.u[k][i] = u[k * NU + i];
  }
  return z;
}

void traj_out(const RocketTrajectory& z, double* x, double* u) {
  for (int k = 0; k < z.nodes(); ++k) {
    for (int i = 0; i < NX; ++i) x[k * NX + i] = z.x[k][i];
    for (int i = 0; i < NU; ++i) u[k * NU + i] = z.u[k][i];
  }
}

template <class Blocks>
void blocks_out(const Blocks& bl, int nx, int nu, double* A, double* Bm, double* Bp, double* w,
                double* x_end) {
  for (int i = 0; i < nx; ++i) {
    for (int j = 0; j < nx; ++j) A[i * nx + j] = bl.A(i, j);
    for (int j = 0; j < nu; ++j) {
      Bm[i * nu + j] = bl.B_minus(i, j);
      Bp[i * nu + j] = bl.B_plus(i, j);
    }
    w[i] = bl.w[i];
    x_end[i] = bl.x_end[i];
  }
}

std::vector<BlocksOf<rocket::Rocket6DoF>> blocks_in(int m, const double* A, const double* Bm,
                                                    const double* Bp, const double* x_end) {
  std::vector<BlocksOf<rocket::Rocket6DoF>> blocks(static_cast<std::size_t>(m));
  for (int k = 0; k < m; ++k) {
    auto& bl = blocks[k];
    for (int i = 0; i < NX; ++i) {
      for (int j = 0; j < NX; ++j) bl.A(i, j) = A[(k * NX + i) * NX + j];
      for (int j = 0; j < NU; ++j) {
        bl.B_minus(i, j) = Bm[(k * NX + i) * NU + j];
        bl.B_plus(i, j) = Bp[(k * NX + i) * NU + j];
      }
      bl.x_end[i] = x_end[k * NX + i];
    }
  }
  return blocks;
}

/// Builds a reference Subproblem<15,7> with run-time dims from flat arrays (one instance).
Sub sub_of(const ptopt_subproblem_shape& s, const ptopt_subproblem_arrays& a) {
  Sub sp;
  sp.resize(s.n_x, s.n_u, s.nodes);
  const int nx = s.n_x, nu = s.n_u, n = s.nodes, m = n - 1;
  for (int k = 0; k < m; ++k) {
    for (int i = 0; i < nx; ++i) {
      for (int j = 0; j < nx; ++j) {
        sp.A_minus[k](i, j) = a.A_minus[(k * nx + i) * nx + j];
        sp.A_plus[k](i, j) = a.A_plus ? a.A_plus[(k * nx + i) * nx + j] : (i == j ? -1.0 : 0.0);
      }
      for (int j = 0; j < nu; ++j) {
        sp.B_minus[k](i, j) = a.B_minus[(k * nx + i) * nu + j];
        sp.B_plus[k](i, j) = a.B_plus[(k * nx + i) * nu + j];
      }
      sp.w[k][i] = a.w[k * nx + i];
    }
    sp.eps_relax[k] = a.eps_relax[k];
  }
  for (int i = 0; i < nx; ++i) {
    sp.e_y[i] = s.e_y[i];
    sp.e_cost[i] = s.e_cost[i];
  }
  for (int k = 0; k < n; ++k)
    for (int i = 0; i < nu; ++i) {
      sp.u_min[k][i] = a.u_min[k * nu + i];
      sp.u_max[k][i] = a.u_max[k * nu + i];
    }
  for (int i = 0; i < s.n_init_fix; ++i) {
    sp.init_fix_idx.push_back(s.init_fix_idx[i]);
    sp.init_fix_val.push_back(a.init_fix_val[i]);
  }
  for (int i = 0; i < s.n_final_fix; ++i) {
    sp.final_fix_idx.push_back(s.final_fix_idx[i]);
    sp.final_fix_val.push_back(a.final_fix_val[i]);
  }
  sp.w_cost = s.w_cost;
  sp.w_prox = s.w_prox;
  sp.w_ep = s.w_ep;
  return sp;
}

template <int C>
std::vector<Vec<C>> group_in(int count, int len, const double* src) {
  std::vector<Vec<C>> g(static_cast<std::size_t>(count), Vec<C>(len));
  for (int k = 0; k < count; ++k)
    for (int i = 0; i < len; ++i) g[k][i] = src[k * len + i];
  return g;
}

template <int C>
void group_out(const std::vector<Vec<C>>& g, int len, double* dst) {
  for (std::size_t k = 0; k < g.size(); ++k)
    for (int i = 0; i < len; ++i) dst[k * len + i] = g[k][i];
}

// ---- the reference's analytic test models -----------------------------------

struct BlowUpModel {  // the divergence model of proj/tests/test_discretizer.cpp:13-28: xdot = x^2
  static constexpr int state_dim = 1;
  static constexpr int control_dim = 1;
  static constexpr int ineq_dim = 0;
  static constexpr int eq_dim = 0;
  Vec<1> dynamics(const Vec<1>& x, const Vec<1>&) const {
    Vec<1> f;
    f[0] = x[0] * x[0];
    return f;
  }
  void dynamics_jacobians(const Vec<1>& x, const Vec<1>&, Mat<1, 1>& A, Mat<1, 1>& B) const {
    A(0, 0) = 2.0 * x[0];
    B(0, 0) = 0.0;
  }
};

template <class Model>
int propagate_generic(const Model& m, const double* xk, const double* uk, const double* uk1,
                      double tau_k, double tau_k1, int steps, int interval_index, double* A,
                      double* Bm, double* Bp, double* w, double* x_end, int* fail_index) {
  using Aug = Augmented<Model>;
  return guarded(fail_index, [&] {
    typename Aug::State x;
    typename Aug::Control u0, u1;
    for (int i = 0; i < Aug::state_dim; ++i) x[i] = xk[i];
    for (int i = 0; i < Aug::control_dim; ++i) {
      u0[i] = uk[i];
      u1[i] = uk1[i];
    }
    const auto bl = propagate_interval(m, x, u0, u1, tau_k, tau_k1, steps, interval_index);
    blocks_out(bl, Aug::state_dim, Aug::control_dim, A, Bm, Bp, w, x_end);
  });
}

template <class Model>
int aug_eval_generic(const Model& m, const double* xin, const double* uin, double* f, double* A,
                     double* B) {
  using Aug = Augmented<Model>;
  return guarded(nullptr, [&] {
    typename Aug::State x;
    typename Aug::Control u;
    for (int i = 0; i < Aug::state_dim; ++i) x[i] = xin[i];
    for (int i = 0; i < Aug::control_dim; ++i) u[i] = uin[i];
    const auto fx = Aug::dynamics(m, x, u);
    for (int i = 0; i < Aug::state_dim; ++i) f[i] = fx[i];
    Mat<Aug::state_dim, Aug::state_dim> Am;
    Mat<Aug::state_dim, Aug::control_dim> Bmat;
    Aug::jacobians(m, x, u, Am, Bmat);
    for (int i = 0; i < Aug::state_dim; ++i) {
      for (int j = 0; j < Aug::state_dim; ++j) A[i * Aug::state_dim + j] = Am(i, j);
      for (int j = 0; j < Aug::control_dim; ++j) B[i * Aug::control_dim + j] = Bmat(i, j);
    }
  });
}

}  // namespace

extern "C" {

// ---- model layer (rocket6dof.hpp:245-402, ctcs.hpp:64-129) -------------------

int ptref_model_eval(const ptopt_vehicle_params* vp, const double* xi, const double* zeta,
                     double* F, double* g, double* dF_dxi, double* dF_dzeta, double* dg_dxi,
                     double* dg_dzeta) {
  return guarded(nullptr, [&] {
    const rocket::Rocket6DoF model(vehicle_of(*vp));
    Vec<14> x;
    Vec<6> z;
    for (int i = 0; i < 14; ++i) x[i] = xi[i];
    for (int i = 0; i < 6; ++i) z[i] = zeta[i];
    const auto s = rocket::VehicleState::from_vec(x);
    const auto c = rocket::VehicleControl::from_vec(z);
    if (F) {
      const auto d = model.eval_dynamics(s, c).to_vec();
      for (int i = 0; i < 14; ++i) F[i] = d[i];
    }
    if (g) {
      const auto gv = model.eval_constraints(s, c);
      for (int i = 0; i < 9; ++i) g[i] = gv[i];
    }
    if (dF_dxi) {
      const auto J = model.eval_jacobians(s, c);
      for (int i = 0; i < 14; ++i) {
        for (int j = 0; j < 14; ++j) dF_dxi[i * 14 + j] = J.dF_dxi(i, j);
        for (int j = 0; j < 6; ++j) dF_dzeta[i * 6 + j] = J.dF_dzeta(i, j);
      }
      for (int i = 0; i < 9; ++i) {
        for (int j = 0; j < 14; ++j) dg_dxi[i * 14 + j] = J.dg_dxi(i, j);
        for (int j = 0; j < 6; ++j) dg_dzeta[i * 6 + j] = J.dg_dzeta(i, j);
      }
    }
  });
}

int ptref_aug_eval(const ptopt_vehicle_params* vp, const double* x, const double* u, double* f,
                   double* A, double* B) {
  const rocket::Rocket6DoF model(vehicle_of(*vp));
  return aug_eval_generic(model, x, u, f, A, B);
}

// ---- discretizer (discretizer.hpp:82-149, 191-232) ---------------------------

int ptref_propagate_interval(const ptopt_vehicle_params* vp, const double* xk, const double* uk,
                             const double* uk1, double tau_k, double tau_k1, int steps,
                             int interval_index, double* A, double* Bm, double* Bp, double* w,
                             double* x_end, int* fail_index) {
  const rocket::Rocket6DoF model(vehicle_of(*vp));
  return propagate_generic(model, xk, uk, uk1, tau_k, tau_k1, steps, interval_index, A, Bm, Bp, w,
                           x_end, fail_index);
}

/// model_id: 0 ZeroModel, 1 ScalarLti(a=params[0], b=params[1]), 2 DoubleIntegrator,
/// 3 ToyConstrained, 4 BlowUp.  Dimensions are the augmented ones of that model.
int ptref_propagate_test_model(int model_id, const double* params, const double* xk,
                               const double* uk, const double* uk1, double tau_k, double tau_k1,
                               int steps, int interval_index, double* A, double* Bm, double* Bp,
                               double* w, double* x_end, int* fail_index) {
  switch (model_id) {
    case 0:
      return propagate_generic(tmodels::ZeroModel{}, xk, uk, uk1, tau_k, tau_k1, steps,
                               interval_index, A, Bm, Bp, w, x_end, fail_index);
    case 1: {
      tmodels::ScalarLti m;
      m.a = params[0];
      m.b = params[1];
      return propagate_generic(m, xk, uk, uk1, tau_k, tau_k1, steps, interval_index, A, Bm, Bp, w,
                               x_end, fail_index);
    }
    case 2:
      return propagate_generic(tmodels::DoubleIntegrator{}, xk, uk, uk1, tau_k, tau_k1, steps,
                               interval_index, A, Bm, Bp, w, x_end, fail_index);
    case 3:
      return propagate_generic(tmodels::ToyConstrained{}, xk, uk, uk1, tau_k, tau_k1, steps,
                               interval_index, A, Bm, Bp, w, x_end, fail_index);
    case 4:
      return propagate_generic(BlowUpModel{}, xk, uk, uk1, tau_k, tau_k1, steps, interval_index, A,
                               Bm, Bp, w, x_end, fail_index);
    default:
      return -1;
  }
}

int ptref_aug_eval_test_model(int model_id, const double* params, const double* x, const double* u,
                              double* f, double* A, double* B) {
  switch (model_id) {
    case 0:
      return aug_eval_generic(tmodels::ZeroModel{}, x, u, f, A, B);
    case 1: {
      tmodels::ScalarLti m;
      m.a = params[0];
      m.b = params[1];
      return aug_eval_generic(m, x, u, f, A, B);
    }
    case 2:
      return aug_eval_generic(tmodels::DoubleIntegrator{}, x, u, f, A, B);
    case 3:
      return aug_eval_generic(tmodels::ToyConstrained{}, x, u, f, A, B);
    default:
      return -1;
  }
}

int ptref_linearize_all(const ptopt_problem_desc* d, const double* tau, const double* x,
                        const double* u, int workers, double* A, double* Bm, double* Bp,
                        double* w, double* x_end, int* fail_index) {
  return guarded(fail_index, [&] {
    const rocket::Rocket6DoF model(vehicle_of(d->vehicle));
    const Grid grid = grid_of(*d, tau);
    const auto z = traj_of(d->nodes, x, u);
    const auto blocks = linearize_all(model, z, grid, d->integrator_steps, workers);
    for (int k = 0; k < grid.intervals(); ++k)
      blocks_out(blocks[k], NX, NU, A + k * NX * NX, Bm + k * NX * NU, Bp + k * NX * NU,
                 w + k * NX, x_end + k * NX);
  });
}

/// propagate_state (discretizer.hpp:153-187) + dense_violation_audit (:249-285).
int ptref_dense_audit(const ptopt_problem_desc* d, const double* tau, const double* x,
                      const double* u, int substeps, double* max_pointwise_g,
                      double* total_y_increase, double* interval_y_increase) {
  return guarded(nullptr, [&] {
    const rocket::Rocket6DoF model(vehicle_of(d->vehicle));
    const Grid grid = grid_of(*d, tau);
    const auto z = traj_of(d->nodes, x, u);
    const auto res = dense_violation_audit(model, z, grid, substeps);
    *max_pointwise_g = res.max_pointwise_g;
    *total_y_increase = res.total_y_increase;
    for (std::size_t k = 0; k < res.interval_y_increase.size(); ++k)
      interval_y_increase[k] = res.interval_y_increase[k];
  });
}

/// dense_violation_audit with its sample sink (discretizer.hpp:236-240, 262-276):
/// samples [nodes-1][substeps+1][12] = {interval, tau, g[9], g_max}.
int ptref_dense_audit_samples(const ptopt_problem_desc* d, const double* tau, const double* x,
                              const double* u, int substeps, double* max_pointwise_g,
                              double* total_y_increase, double* interval_y_increase, double* samples) {
  return guarded(nullptr, [&] {
    const rocket::Rocket6DoF model(vehicle_of(d->vehicle));
    const Grid grid = grid_of(*d, tau);
    const auto z = traj_of(d->nodes, x, u);
    std::vector<AuditSample> got;
    const auto res = dense_violation_audit(model, z, grid, substeps, &got);
    *max_pointwise_g = res.max_pointwise_g;
    *total_y_increase = res.total_y_increase;
    for (std::size_t k = 0; k < res.interval_y_increase.size(); ++k)
      interval_y_increase[k] = res.interval_y_increase[k];
    for (std::size_t i = 0; i < got.size(); ++i) {
      double* s = samples + i * 12;
      s[0] = got[i].interval;
      s[1] = got[i].tau;
      for (std::size_t q = 0; q < got[i].g.size(); ++q) s[2 + q] = got[i].g[q];
      s[11] = got[i].g_max;
    }
  });
}

// ---- SCP glue (scp.hpp:139-217, 239-249, 256-364) ----------------------------

int ptref_assemble(const ptopt_problem_desc* d, const double* tau, const double* init_state,
                   const double* x, const double* u, const double* A, const double* Bm,
                   const double* Bp, const double* x_end, double* A_minus, double* A_plus,
                   double* B_minus, double* B_plus, double* w_hat, double* eps_relax,
                   double* u_min, double* u_max, double* init_fix_val, double* final_fix_val,
                   double* e_cost_hat) {
  return guarded(nullptr, [&] {
    const auto pb = problem_of(*d, tau, init_state, 0);
    const int n = d->nodes, m = n - 1;
    const auto z = traj_of(n, x, u);
    const auto sp = assemble_subproblem(pb, z, blocks_in(m, A, Bm, Bp, x_end));
    for (int k = 0; k < m; ++k) {
      for (int i = 0; i < NX; ++i) {
        for (int j = 0; j < NX; ++j) {
          A_minus[(k * NX + i) * NX + j] = sp.A_minus[k](i, j);
          if (A_plus) A_plus[(k * NX + i) * NX + j] = sp.A_plus[k](i, j);
        }
        for (int j = 0; j < NU; ++j) {
          B_minus[(k * NX + i) * NU + j] = sp.B_minus[k](i, j);
          B_plus[(k * NX + i) * NU + j] = sp.B_plus[k](i, j);
        }
        w_hat[k * NX + i] = sp.w[k][i];
      }
      eps_relax[k] = sp.eps_relax[k];
    }
    for (int k = 0; k < n; ++k)
      for (int i = 0; i < NU; ++i) {
        u_min[k * NU + i] = sp.u_min[k][i];
        u_max[k * NU + i] = sp.u_max[k][i];
      }
    for (std::size_t i = 0; i < sp.init_fix_val.size(); ++i) init_fix_val[i] = sp.init_fix_val[i];
    for (std::size_t i = 0; i < sp.final_fix_val.size(); ++i)
      final_fix_val[i] = sp.final_fix_val[i];
    if (e_cost_hat)
      for (int i = 0; i < NX; ++i) e_cost_hat[i] = sp.e_cost[i];
  });
}

/// The cold-start seed of scp_solve (scp.hpp:303-321): n*(15+7) draws, unit 2-norm.
void ptref_scp_seed(std::uint64_t rng_seed, int nodes, double* seed_x, double* seed_u) {
  std::uint64_t state = rng_seed ^ 0x5bf03635d78b41adull;
  double norm_sq = 0.0;
  for (int i = 0; i < nodes * NX; ++i) {
    seed_x[i] = 2.0 * detail::unit_interval(detail::splitmix64(state)) - 1.0;
    norm_sq += seed_x[i] * seed_x[i];
  }
  for (int i = 0; i < nodes * NU; ++i) {
    seed_u[i] = 2.0 * detail::unit_interval(detail::splitmix64(state)) - 1.0;
    norm_sq += seed_u[i] * seed_u[i];
  }
  const double inv = 1.0 / std::sqrt(norm_sq);
  for (int i = 0; i < nodes * NX; ++i) seed_x[i] *= inv;
  for (int i = 0; i < nodes * NU; ++i) seed_u[i] *= inv;
}

int ptref_scp_solve(const ptopt_problem_desc* d, const double* tau, const double* init_state,
                    const double* x_guess, const double* u_guess, std::uint64_t rng_seed,
                    double* x_out, double* u_out, int* scp_iterations, int* converged,
                    double* final_defect_inf, double* history, int* fail_index) {
  return guarded(fail_index, [&] {
    const auto pb = problem_of(*d, tau, init_state, rng_seed);
    const auto res = scp_solve(pb, traj_of(d->nodes, x_guess, u_guess));
    traj_out(res.iterate, x_out, u_out);
    *scp_iterations = res.iterations;
    *converged = res.converged ? 1 : 0;
    *final_defect_inf = res.final_defect_inf;
    for (std::size_t i = 0; i < res.history.size(); ++i) {
      history[i * 5 + 0] = res.history[i].defect_inf;
      history[i * 5 + 1] = res.history[i].step_inf;
      history[i * 5 + 2] = res.history[i].penalized_cost;
      history[i * 5 + 3] = static_cast<double>(res.history[i].pipg_iterations);
      history[i * 5 + 4] = res.history[i].sigma;
    }
  });
}

// ---- PIPG (pipg.hpp:206-292, 350-497) ----------------------------------------

int ptref_power_iteration(const ptopt_subproblem_shape* shape, const ptopt_subproblem_arrays* a,
                          const double* seed_x, const double* seed_u, const double* seed_vcp,
                          const double* seed_vcn, double eps_abs, double eps_rel, double eps_buff,
                          int j_max, double* sigma) {
  return guarded(nullptr, [&] {
    const Sub sp = sub_of(*shape, *a);
    const int n = shape->nodes, m = n - 1;
    *sigma = pipg::power_iteration_custom(
        sp, group_in<NX>(n, shape->n_x, seed_x), group_in<NU>(n, shape->n_u, seed_u),
        group_in<NX>(m, shape->n_x, seed_vcp), group_in<NX>(m, shape->n_x, seed_vcn), eps_abs,
        eps_rel, eps_buff, j_max);
  });
}

int ptref_pipg(const ptopt_subproblem_shape* shape, const ptopt_subproblem_arrays* a,
               const ptopt_pipg_config* cfg, double sigma, const ptopt_workspace_arrays* w,
               int* iterations, int* converged, int* fail_index) {
  return guarded(fail_index, [&] {
    const Sub sp = sub_of(*shape, *a);
    const int n = shape->nodes, m = n - 1, nx = shape->n_x, nu = shape->n_u;
    Wsp ws;
    ws.init(nx, nu, n);
    ws.sigma = sigma;
    ws.x = group_in<NX>(n, nx, w->x);
    ws.u = group_in<NU>(n, nu, w->u);
    ws.vc_pos = group_in<NX>(m, nx, w->vc_pos);
    ws.vc_neg = group_in<NX>(m, nx, w->vc_neg);
    ws.dyn_dual = group_in<NX>(m, nx, w->dyn_dual);
    for (int k = 0; k < m; ++k) ws.relax_dual[k] = w->relax_dual[k];
    pipg::PipgConfig c;
    c.omega = cfg->omega;
    c.rho = cfg->rho;
    c.j_max = cfg->j_max;
    c.j_check = cfg->j_check;
    c.eps_abs = cfg->eps_abs;
    c.eps_rel = cfg->eps_rel;
    c.eps_buff = cfg->eps_buff;
    const auto res = pipg::pipg_custom(sp, c, ws);
    *iterations = res.iterations;
    *converged = res.converged ? 1 : 0;
    group_out(ws.x, nx, w->x);
    group_out(ws.u, nu, w->u);
    group_out(ws.vc_pos, nx, w->vc_pos);
    group_out(ws.vc_neg, nx, w->vc_neg);
    group_out(ws.dyn_dual, nx, w->dyn_dual);
    for (int k = 0; k < m; ++k) w->relax_dual[k] = ws.relax_dual[k];
  });
}

/// pipg_generic on build_generic_qp(sp) (pipg.hpp:563-728): the reference's own
/// dense counterpart of the customized loop.  z in generic layout, duals eta/chi.
int ptref_pipg_generic(const ptopt_subproblem_shape* shape, const ptopt_subproblem_arrays* a,
                       const ptopt_pipg_config* cfg, double sigma, double* z, double* eq_dual,
                       double* ineq_dual, int* iterations, int* converged) {
  return guarded(nullptr, [&] {
    const Sub sp = sub_of(*shape, *a);
    const auto qp = pipg::build_generic_qp(sp);
    pipg::PipgConfig c;
    c.omega = cfg->omega;
    c.rho = cfg->rho;
    c.j_max = cfg->j_max;
    c.j_check = cfg->j_check;
    c.eps_abs = cfg->eps_abs;
    c.eps_rel = cfg->eps_rel;
    c.eps_buff = cfg->eps_buff;
    const auto res = pipg::pipg_generic(qp, c, sigma);
    for (std::size_t i = 0; i < res.z.size(); ++i) z[i] = res.z[i];
    for (std::size_t i = 0; i < res.eq_dual.size(); ++i) eq_dual[i] = res.eq_dual[i];
    for (std::size_t i = 0; i < res.ineq_dual.size(); ++i) ineq_dual[i] = res.ineq_dual[i];
    *iterations = res.iterations;
    *converged = res.converged ? 1 : 0;
  });
}

double ptref_step_sizes(double lambda, double omega, double sigma, double* beta) {
  const auto s = pipg::step_sizes(lambda, omega, sigma);
  *beta = s.beta;
  return s.alpha;
}

// ---- instance generation (montecarlo.hpp:35-65, rocket_problem.hpp:127-163) --

std::uint64_t ptref_run_seed(std::uint64_t batch_seed, int run_id) {
  return mc::run_seed(batch_seed, run_id);
}

void ptref_disperse(const double* r_low, const double* r_high, std::uint64_t seed, int run_id,
                    double* r_out) {
  RocketBoundary nominal;
  mc::DispersionSpec spec;
  for (int i = 0; i < 3; ++i) {
    spec.r_low[i] = r_low[i];
    spec.r_high[i] = r_high[i];
  }
  spec.seed = seed;
  const auto bc = mc::disperse(nominal, spec, run_id);
  for (int i = 0; i < 3; ++i) r_out[i] = bc.initial.r[i];
}

int ptref_initial_guess(const ptopt_problem_desc* d, const double* tau, const double* init_state,
                        double* x, double* u) {
  return guarded(nullptr, [&] {
    const auto pb = problem_of(*d, tau, init_state, 0);
    const auto bc = boundary_of(*d, init_state);
    traj_out(initial_guess(pb, bc), x, u);
  });
}

double ptref_pow2_near(double v) { return ScalingPair<NX, NU>::pow2_near(v); }

// ---- batch harness (montecarlo.hpp:100-175): the CPU baseline ----------------

/// Runs mc::run_batch on `workers` threads and returns its own total_wall_time.
/// records: [B][8] = run_id, converged, scp_iterations, propellant_used,
/// final_defect_inf, max_pointwise_g, max_node_y_increase, failed(0/1).
/// trajectories (optional): x [B][nodes][15], u [B][nodes][7].
double ptref_run_batch(const ptopt_problem_desc* d, const double* tau,
                       const double* nominal_init_state, const double* r_low,
                       const double* r_high, std::uint64_t seed, int batch_size, int workers,
                       int audit_substeps, double* records, double* x_out, double* u_out) {
  const auto pb = problem_of(*d, tau, nominal_init_state, seed);
  const auto bc = boundary_of(*d, nominal_init_state);
  mc::DispersionSpec spec;
  for (int i = 0; i < 3; ++i) {
    spec.r_low[i] = r_low[i];
    spec.r_high[i] = r_high[i];
  }
  spec.seed = seed;
  const bool keep = x_out != nullptr && u_out != nullptr;
  const auto out = mc::run_batch(pb, bc, spec, batch_size, workers, audit_substeps, keep);
  for (int b = 0; b < batch_size; ++b) {
    const auto& r = out.records[b];
    double* rec = records + b * 8;
    rec[0] = r.run_id;
    rec[1] = r.converged ? 1.0 : 0.0;
    rec[2] = r.scp_iterations;
    rec[3] = r.propellant_used;
    rec[4] = r.final_defect_inf;
    rec[5] = r.max_pointwise_g;
    rec[6] = r.max_node_y_increase;
    rec[7] = r.failure.empty() ? 0.0 : 1.0;
    if (keep && r.failure.empty())
      traj_out(out.trajectories[b], x_out + b * d->nodes * NX, u_out + b * d->nodes * NU);
  }
  return out.total_wall_time;
}

int ptref_abi_version(void) { return PTOPT_ABI_VERSION; }

}  // extern "C"
