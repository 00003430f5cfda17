// TEST: the C++ host mirror (paper_2404_18034_b200/host/ptopt_b200.hpp) against the CPU
// oracle (oracle/ptopt_oracle.h, test infrastructure) on identical inputs.  Reads like the
// reference's own suites: build a problem, call the solver API, compare.
// Exit code 0 = all checks passed; every failed check prints a line.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ptopt_b200.hpp"
#include "ptopt_oracle.h"

namespace pb = ptopt_b200;

static int g_failed = 0;
#define CHECK(cond)                                                         \
  do {                                                                      \
    if (!(cond)) {                                                          \
      std::printf("FAILED %s:%d  %s\n", __FILE__, __LINE__, #cond);         \
      ++g_failed;                                                           \
    }                                                                       \
  } while (0)

static double rel_err(const double* a, const double* b, int n) {  // oracles.hpp:73-82
  double num = 0.0, den = 1.0;
  for (int i = 0; i < n; ++i) {
    num = std::fmax(num, std::fabs(a[i] - b[i]));
    den = std::fmax(den, std::fabs(b[i]));
  }
  return num / den;
}

// default_config() restated (config.hpp:155-197)
static pb::rocket::VehicleParams default_vehicle() {
  pb::rocket::VehicleParams p;
  p.alpha_mdot = 0.05;
  p.g_inertial = {-1.0, 0.0, 0.0};
  p.inertia(0, 0) = 0.1;
  p.inertia(1, 1) = 0.25;
  p.inertia(2, 2) = 0.25;
  p.r_thrust = {-0.5, 0.0, 0.0};
  p.m_dry = 1.0;
  p.v_max = 3.0;
  p.theta_max = 1.0471975511965976;
  p.omega_max = 1.0;
  p.delta_max = 0.3490658503988659;
  p.T_min = 1.0;
  p.T_max = 6.0;
  p.gamma_max = 0.3;
  return p;
}

static pb::RocketBoundary default_boundary() {
  pb::RocketBoundary bc;
  bc.initial.m = 2.0;
  bc.initial.r = {7.5, 4.5, 1.5};
  bc.initial.v = {-1.0, -0.5, -0.2};
  return bc;
}

static pb::RocketProblem make_problem(int nodes, int max_iters, int pipg_iters, int power_iters) {
  pb::RocketProblem p = pb::make_rocket_problem(default_vehicle(), default_boundary(), pb::Grid::uniform(nodes));
  p.t_f_guess = 5.0;
  p.s_min = 1.0;
  p.s_max = 15.0;
  pb::Vec<15> xr;
  pb::Vec<7> ur;
  const double xs[15] = {1, 8, 8, 8, 3, 3, 3, 1, 1, 1, 1, 1, 1, 1, 1};
  const double us[7] = {6, 6, 6, 0.3, 0.3, 0.3, 5};
  for (int i = 0; i < 15; ++i) xr[i] = xs[i];
  for (int i = 0; i < 7; ++i) ur[i] = us[i];
  p.scaling = pb::ScalingPair<15, 7>::from_ranges(xr, ur);
  p.max_iters = max_iters;
  p.pipg_cfg.j_max = pipg_iters;
  p.power_j_max = power_iters;
  p.rng_seed = ptor_run_seed(20260810ull, 0);
  return p;
}

int main() {
  const int n = 12, m = n - 1;
  pb::RocketProblem prob = make_problem(n, 3, 250, 300);
  const ptopt_problem_desc d = pb::detail::to_desc(prob);

  // initial guess from the oracle (rocket_problem.hpp:127-163)
  std::vector<double> init(14), xg(n * 15), ug(n * 7);
  for (int i = 0; i < 14; ++i) init[i] = prob.init_state[i];
  CHECK(ptor_initial_guess(&d, nullptr, init.data(), xg.data(), ug.data()) == 0);
  pb::RocketTrajectory z(n);
  for (int k = 0; k < n; ++k) {
    for (int i = 0; i < 15; ++i) z.x[k][i] = xg[k * 15 + i];
    for (int i = 0; i < 7; ++i) z.u[k][i] = ug[k * 7 + i];
  }

  // ---- linearize_all / propagate_interval
  std::vector<double> A(m * 225), Bm(m * 105), Bp(m * 105), w(m * 15), xe(m * 15);
  int fail = -1;
  CHECK(ptor_linearize_all(&d, nullptr, xg.data(), ug.data(), 1, A.data(), Bm.data(), Bp.data(), w.data(),
                           xe.data(), &fail) == 0);
  const auto blocks = pb::linearize_all(prob.model, z, prob.grid, prob.integrator_steps);
  CHECK((int)blocks.size() == m);
  for (int k = 0; k < m; ++k) {
    CHECK(rel_err(blocks[k].A.a.data(), &A[k * 225], 225) <= 1e-9);
    CHECK(rel_err(blocks[k].B_minus.a.data(), &Bm[k * 105], 105) <= 1e-9);
    CHECK(rel_err(blocks[k].B_plus.a.data(), &Bp[k * 105], 105) <= 1e-9);
    CHECK(rel_err(blocks[k].w.a.data(), &w[k * 15], 15) <= 1e-9);
    CHECK(rel_err(blocks[k].x_end.a.data(), &xe[k * 15], 15) <= 1e-9);
  }
  {
    const int k = 3;
    const auto b = pb::propagate_interval(prob.model, z.x[k], z.u[k], z.u[k + 1], prob.grid.nodes[k],
                                          prob.grid.nodes[k + 1], prob.integrator_steps, k);
    CHECK(rel_err(b.A.a.data(), &A[k * 225], 225) <= 1e-9);
    CHECK(rel_err(b.x_end.a.data(), &xe[k * 15], 15) <= 1e-9);
    CHECK(rel_err(b.w.a.data(), &w[k * 15], 15) <= 1e-9);
  }
  std::printf("linearize_all / propagate_interval ok\n");

  // ---- error mapping (discretizer.hpp:18-23, 89; ctcs.hpp:66)
  {
    pb::RocketTrajectory bad = z;
    bad.u[5][6] = -1.0;
    bool caught = false;
    try {
      pb::linearize_all(prob.model, bad, prob.grid, prob.integrator_steps);
    } catch (const std::domain_error& e) {
      caught = std::string(e.what()).find("dilation") != std::string::npos;
    }
    CHECK(caught);
    bad = z;
    bad.x[7][2] = std::nan("");
    int interval = -1;
    try {
      pb::linearize_all(prob.model, bad, prob.grid, prob.integrator_steps);
    } catch (const pb::PropagationDiverged& e) {
      interval = e.interval;
    }
    CHECK(interval == 7);
    caught = false;
    try {
      pb::linearize_all(prob.model, z, prob.grid, 0);
    } catch (const std::invalid_argument&) {
      caught = true;
    }
    CHECK(caught);
  }
  std::printf("error mapping ok\n");

  // ---- assemble_subproblem (exact: power-of-two scaling)
  std::vector<double> Am(m * 225), Ap(m * 225), Bmh(m * 105), Bph(m * 105), wh(m * 15), eps(m), umin(n * 7),
      umax(n * 7), iv(15), fv(15), ech(15);
  CHECK(ptor_assemble(&d, nullptr, init.data(), xg.data(), ug.data(), A.data(), Bm.data(), Bp.data(), xe.data(),
                      Am.data(), Ap.data(), Bmh.data(), Bph.data(), wh.data(), eps.data(), umin.data(), umax.data(),
                      iv.data(), fv.data(), ech.data()) == 0);
  // feed the oracle's blocks so that assembly is compared on identical inputs
  std::vector<pb::RocketBlocks> oblocks(m);
  for (int k = 0; k < m; ++k)
    for (int i = 0; i < 15; ++i) {
      for (int j = 0; j < 15; ++j) oblocks[k].A(i, j) = A[k * 225 + i * 15 + j];
      for (int j = 0; j < 7; ++j) {
        oblocks[k].B_minus(i, j) = Bm[k * 105 + i * 7 + j];
        oblocks[k].B_plus(i, j) = Bp[k * 105 + i * 7 + j];
      }
      oblocks[k].x_end[i] = xe[k * 15 + i];
    }
  const auto sp = pb::assemble_subproblem(prob, z, oblocks);
  for (int k = 0; k < m; ++k) {
    for (int e = 0; e < 225; ++e) CHECK(sp.A_minus[k].a[e] == Am[k * 225 + e]);
    for (int e = 0; e < 105; ++e) CHECK(sp.B_minus[k].a[e] == Bmh[k * 105 + e] && sp.B_plus[k].a[e] == Bph[k * 105 + e]);
    for (int i = 0; i < 15; ++i) CHECK(sp.w[k][i] == wh[k * 15 + i]);
    CHECK(sp.eps_relax[k] == eps[k]);
  }
  for (int k = 0; k < n; ++k)
    for (int i = 0; i < 7; ++i) CHECK(sp.u_min[k][i] == umin[k * 7 + i] && sp.u_max[k][i] == umax[k * 7 + i]);
  CHECK(sp.init_fix_idx.size() == 15 && sp.final_fix_idx.size() == 13);
  for (int i = 0; i < 15; ++i) CHECK(sp.init_fix_val[i] == iv[i] && sp.e_cost[i] == ech[i]);
  for (int i = 0; i < 13; ++i) CHECK(sp.final_fix_val[i] == fv[i]);
  std::printf("assemble_subproblem ok\n");

  // ---- power_iteration_custom / pipg_custom
  ptopt_subproblem_shape shape{};
  shape.n_x = 15;
  shape.n_u = 7;
  shape.nodes = n;
  shape.n_init_fix = 15;
  shape.n_final_fix = 13;
  for (int i = 0; i < 15; ++i) {
    shape.init_fix_idx[i] = i;
    shape.e_cost[i] = ech[i];
  }
  for (int i = 0; i < 13; ++i) shape.final_fix_idx[i] = d.final_fix_idx[i];
  shape.e_y[14] = 1.0;
  shape.w_cost = d.w_cost;
  shape.w_prox = d.w_prox;
  shape.w_ep = d.w_ep;
  ptopt_subproblem_arrays arr{Am.data(), nullptr, Bmh.data(), Bph.data(), wh.data(), eps.data(), umin.data(),
                              umax.data(), iv.data(), fv.data()};
  std::vector<double> sx(n * 15), su(n * 7), zero(m * 15, 0.0);
  ptor_scp_seed(prob.rng_seed, n, sx.data(), su.data());
  double sigma_ref = 0.0;
  CHECK(ptor_power_iteration(&shape, &arr, sx.data(), su.data(), zero.data(), zero.data(), 1e-12, 1e-12, 0.05,
                             10000, &sigma_ref) == 0);
  pb::pipg::Workspace<> ws;
  ws.init(15, 7, n);
  std::vector<pb::Vec<15>> seed_x(n), seed_v(m);
  std::vector<pb::Vec<7>> seed_u(n);
  for (int k = 0; k < n; ++k) {
    for (int i = 0; i < 15; ++i) seed_x[k][i] = sx[k * 15 + i];
    for (int i = 0; i < 7; ++i) seed_u[k][i] = su[k * 7 + i];
  }
  const double sigma = pb::pipg::power_iteration_custom(sp, seed_x, seed_u, seed_v, seed_v, 1e-12, 1e-12, 0.05, 10000);
  CHECK(std::fabs(sigma - sigma_ref) <= 1e-9 * sigma_ref);
  {
    bool caught = false;
    std::vector<pb::Vec<15>> zx(n);
    std::vector<pb::Vec<7>> zu(n);
    try {
      pb::pipg::power_iteration_custom(sp, zx, zu, seed_v, seed_v);
    } catch (const std::invalid_argument&) {
      caught = true;
    }
    CHECK(caught);  // all-zero seed, pipg.hpp:224-225
  }
  pb::pipg::PipgConfig cfg;
  cfg.j_max = 400;
  cfg.j_check = 25;
  ws.sigma = sigma_ref;
  const pb::pipg::PipgResult res = pb::pipg::pipg_custom(sp, cfg, ws);
  std::vector<double> rx(n * 15, 0.0), ru(n * 7, 0.0), rvp(m * 15, 0.0), rvn(m * 15, 0.0), rdd(m * 15, 0.0), rrd(m, 0.0);
  ptopt_workspace_arrays rw{rx.data(), ru.data(), rvp.data(), rvn.data(), rdd.data(), rrd.data()};
  const ptopt_pipg_config ccfg{cfg.omega, cfg.rho, cfg.j_max, cfg.j_check, cfg.eps_abs, cfg.eps_rel, cfg.eps_buff};
  int it_ref = 0, conv_ref = 0;
  CHECK(ptor_pipg(&shape, &arr, &ccfg, sigma_ref, &rw, &it_ref, &conv_ref, &fail) == 0);
  CHECK(res.iterations == it_ref && res.converged == (conv_ref != 0));
  double worst = 0.0;
  for (int k = 0; k < n; ++k) {
    for (int i = 0; i < 15; ++i) worst = std::fmax(worst, std::fabs(ws.x[k][i] - rx[k * 15 + i]));
    for (int i = 0; i < 7; ++i) worst = std::fmax(worst, std::fabs(ws.u[k][i] - ru[k * 7 + i]));
  }
  for (int k = 0; k < m; ++k) {
    for (int i = 0; i < 15; ++i) {
      worst = std::fmax(worst, std::fabs(ws.vc_pos[k][i] - rvp[k * 15 + i]));
      worst = std::fmax(worst, std::fabs(ws.vc_neg[k][i] - rvn[k * 15 + i]));
      worst = std::fmax(worst, std::fabs(ws.dyn_dual[k][i] - rdd[k * 15 + i]));
    }
    worst = std::fmax(worst, std::fabs(ws.relax_dual[k] - rrd[k]));
  }
  CHECK(worst <= 1e-6);
  std::printf("power_iteration_custom / pipg_custom ok (sigma %.12f, max |diff| %.2e)\n", sigma, worst);
  {
    // sigma = 0 is a valid workspace (Workspace::init leaves it at 0, and the power iteration returns
    // 0 for an iterate in the operator's null space, pipg.hpp:280-284): alpha = 1 / w_prox, no throw
    pb::pipg::Workspace ws0;
    ws0.init(15, 7, n);
    ws0.sigma = 0.0;
    pb::pipg::PipgConfig c0;
    c0.j_max = 10;
    c0.j_check = 5;
    std::vector<double> zx(n * 15, 0.0), zu(n * 7, 0.0), zvp(m * 15, 0.0), zvn(m * 15, 0.0), zdd(m * 15, 0.0), zrd(m, 0.0);
    ptopt_workspace_arrays zw{zx.data(), zu.data(), zvp.data(), zvn.data(), zdd.data(), zrd.data()};
    const ptopt_pipg_config cc0{c0.omega, c0.rho, c0.j_max, c0.j_check, c0.eps_abs, c0.eps_rel, c0.eps_buff};
    int it0 = 0, cv0 = 0, fl0 = -1;
    const int rc0 = ptor_pipg(&shape, &arr, &cc0, 0.0, &zw, &it0, &cv0, &fl0);
    double w0 = 0.0, scale = 1.0;
    if (rc0 == 0) {
      const pb::pipg::PipgResult r0 = pb::pipg::pipg_custom(sp, c0, ws0);
      CHECK(r0.iterations == it0 && r0.converged == (cv0 != 0));
      for (int k = 0; k < n; ++k)
        for (int i = 0; i < 15; ++i) {
          w0 = std::fmax(w0, std::fabs(ws0.x[k][i] - zx[k * 15 + i]));
          scale = std::fmax(scale, std::fabs(zx[k * 15 + i]));
        }
      CHECK(w0 <= 1e-9 * scale);
    } else {  // steps this large may blow up: then both sides report SolverDiverged at the same check
      CHECK(rc0 == PTOPT_ST_SOLVER_DIVERGED);
      int at = -1;
      try {
        pb::pipg::pipg_custom(sp, c0, ws0);
      } catch (const pb::pipg::SolverDiverged& e) {
        at = e.iteration;
      }
      CHECK(at == fl0);
    }
    std::printf("pipg_custom with sigma = 0 ok (%d iterations, max |diff| %.2e, |x| %.2e)\n", it0, w0, scale);
  }
  {
    // the texts RunRecord::failure carries are the reference's exception messages
    CHECK(ptopt_b200::detail::failure_text(PTOPT_ST_DILATION_NONPOSITIVE, 0) ==
          "augmented dynamics: dilation factor must be positive");                       // ctcs.hpp:66
    CHECK(ptopt_b200::detail::failure_text(PTOPT_ST_MASS_NONPOSITIVE, 0) == "rocket dynamics: nonpositive mass");
    CHECK(ptopt_b200::detail::failure_text(PTOPT_ST_THRUST_SINGULAR, 0) ==
          "rocket jacobians: thrust magnitude below singular-point tolerance");           // rocket6dof.hpp:307
    CHECK(ptopt_b200::detail::failure_text(PTOPT_ST_POWER_SEED_ZERO, 0) ==
          "power iteration: seed point must not be all zero");                            // pipg.hpp:225
  }

  // ---- scp_solve
  const pb::ScpResult sr = pb::scp_solve(prob, z);
  std::vector<double> xo(n * 15), uo(n * 7), hist(3 * 5, 0.0);
  int iters = 0, conv = 0;
  double fdef = 0.0;
  CHECK(ptor_scp_solve(&d, nullptr, init.data(), xg.data(), ug.data(), prob.rng_seed, xo.data(), uo.data(), &iters,
                       &conv, &fdef, hist.data(), &fail) == 0);
  CHECK(sr.iterations == iters && sr.converged == (conv != 0) && (int)sr.history.size() == iters);
  CHECK(std::fabs(sr.final_defect_inf - fdef) <= 1e-6);
  worst = 0.0;
  for (int k = 0; k < n; ++k) {
    for (int i = 0; i < 15; ++i) worst = std::fmax(worst, std::fabs(sr.iterate.x[k][i] - xo[k * 15 + i]));
    for (int i = 0; i < 7; ++i) worst = std::fmax(worst, std::fabs(sr.iterate.u[k][i] - uo[k * 7 + i]));
  }
  CHECK(worst <= 1e-6);
  for (int it = 0; it < iters; ++it) {
    CHECK(sr.history[it].pipg_iterations == (int)hist[it * 5 + 3]);
    CHECK(std::fabs(sr.history[it].sigma / hist[it * 5 + 4] - 1.0) <= 1e-8);
  }
  std::printf("scp_solve ok (%d iterations, max |diff| %.2e)\n", iters, worst);

  // ---- dense_violation_audit
  {
    double g_ref = 0.0, ytot_ref = 0.0;
    std::vector<double> dy_ref(m);
    CHECK(ptor_dense_audit(&d, nullptr, xo.data(), uo.data(), 16, &g_ref, &ytot_ref, dy_ref.data()) == 0);
    const pb::AuditResult ar = pb::dense_violation_audit(prob.model, sr.iterate, prob.grid, 16);
    CHECK(std::fabs(ar.max_pointwise_g - g_ref) <= 1e-6);
    CHECK(std::fabs(ar.total_y_increase - ytot_ref) <= 1e-6);
  }

  // ---- mc::run_batch
  {
    pb::mc::DispersionSpec spec;
    spec.r_low = {6.0, 3.0, 1.0};
    spec.r_high = {9.0, 6.0, 2.0};
    spec.seed = 20260810ull;
    const int B = 5;
    const pb::mc::BatchResult br = pb::mc::run_batch(prob, default_boundary(), spec, B, 2, 16, true);
    std::vector<double> rec(B * 8), bx(B * n * 15), bu(B * n * 7);
    ptor_run_batch(&d, nullptr, init.data(), spec.r_low.data(), spec.r_high.data(), spec.seed, B, 2, 16, rec.data(),
                   bx.data(), bu.data());
    CHECK((int)br.records.size() == B && (int)br.trajectories.size() == B);
    for (int b = 0; b < B; ++b) {
      const auto& r = br.records[b];
      CHECK(r.run_id == b && r.failure.empty() && rec[b * 8 + 7] == 0.0);
      CHECK(r.converged == (rec[b * 8 + 1] != 0.0) && r.scp_iterations == (int)rec[b * 8 + 2]);
      CHECK(std::fabs(r.propellant_used - rec[b * 8 + 3]) <= 1e-6);
      CHECK(std::fabs(r.final_defect_inf - rec[b * 8 + 4]) <= 1e-6);
      CHECK(std::fabs(r.max_pointwise_g - rec[b * 8 + 5]) <= 1e-6);
      CHECK(std::fabs(r.max_node_y_increase - rec[b * 8 + 6]) <= 1e-6);
      double wdiff = 0.0;
      for (int k = 0; k < n; ++k)
        for (int i = 0; i < 15; ++i)
          wdiff = std::fmax(wdiff, std::fabs(br.trajectories[b].x[k][i] - bx[(b * n + k) * 15 + i]));
      CHECK(wdiff <= 1e-6);
    }
    // the same batch over a device list (two handles + two host threads on device 0; three entries
    // for a batch of two leaves one worker without work): bit-identical records and trajectories
    for (const std::vector<int>& devs : {std::vector<int>{0, 0}, std::vector<int>{0, 0, 0}}) {
      const int Bm = devs.size() == 2 ? B : 2;
      std::vector<double> ms;
      const pb::mc::BatchResult bm = pb::mc::run_batch(prob, default_boundary(), spec, Bm, devs, 16, true, 0, &ms);
      CHECK((int)bm.records.size() == Bm && bm.workers == (int)devs.size() && ms.size() == devs.size());
      for (int b = 0; b < Bm; ++b) {
        const auto &r = bm.records[b], &q = br.records[b];
        CHECK(r.run_id == q.run_id && r.converged == q.converged && r.scp_iterations == q.scp_iterations);
        CHECK(r.propellant_used == q.propellant_used && r.final_defect_inf == q.final_defect_inf);
        CHECK(r.max_pointwise_g == q.max_pointwise_g && r.max_node_y_increase == q.max_node_y_increase);
        bool same = true;
        for (int k = 0; k < n; ++k) {
          for (int i = 0; i < 15; ++i) same = same && bm.trajectories[b].x[k][i] == br.trajectories[b].x[k][i];
          for (int i = 0; i < 7; ++i) same = same && bm.trajectories[b].u[k][i] == br.trajectories[b].u[k][i];
        }
        CHECK(same);
      }
    }
    {  // a boundary whose terminal targets are not the ones the problem pins is refused
      auto other = default_boundary();
      other.r_final[0] = 0.25;
      bool refused = false;
      try {
        pb::initial_guess(prob, other);
      } catch (const std::invalid_argument&) {
        refused = true;
      }
      CHECK(refused);
    }
    bool caught = false;
    try {
      pb::mc::run_batch(prob, default_boundary(), spec, 0, 1);
    } catch (const std::invalid_argument&) {
      caught = true;
    }
    CHECK(caught);
  }
  std::printf("dense_violation_audit / mc::run_batch ok\n");

  if (g_failed) {
    std::printf("%d check(s) failed\n", g_failed);
    return 1;
  }
  std::printf("all host-API checks passed\n");
  return 0;
}
