// config_formats.cpp — TEST INFRASTRUCTURE.  Loads every JSON file named on the command line and
// prints either a canonical dump of the resulting run configuration (every field, "%.17g") and of
// the problem built from it, or the error class (+ message for ConfigError, whose text is part of
// the contract).
//   default build            -> paper_2404_18034_b200/host/ptopt_b200_config.hpp
//   -DWITH_REFERENCE build   -> the reference's config.hpp + nlohmann/json (this is how
//                               tests/golden/config/expected.txt was generated)
#include <cstdio>
#include <string>

#ifdef WITH_REFERENCE
#include "ptopt/config.hpp"
namespace lib = ptopt;
#else
#include "ptopt_b200_config.hpp"
namespace lib = ptopt_b200;
#endif

namespace {

void num(const char* name, double v) { std::printf("  %s %.17g\n", name, v); }
void integer(const char* name, long long v) { std::printf("  %s %lld\n", name, v); }
template <class A>
void vec(const char* name, const A& a, int n) {
  std::printf("  %s", name);
  for (int i = 0; i < n; ++i) std::printf(" %.17g", (double)a[static_cast<std::size_t>(i)]);
  std::printf("\n");
}

void dump(const lib::RunConfig& c) {
  const auto& v = c.vehicle;
  num("vehicle.alpha_mdot", v.alpha_mdot);
  vec("vehicle.g_inertial", v.g_inertial, 3);
  std::printf("  vehicle.inertia");
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) std::printf(" %.17g", v.inertia(i, j));
  std::printf("\n");
  vec("vehicle.r_thrust", v.r_thrust, 3);
  num("vehicle.m_dry", v.m_dry); num("vehicle.v_max", v.v_max); num("vehicle.theta_max", v.theta_max);
  num("vehicle.omega_max", v.omega_max); num("vehicle.delta_max", v.delta_max); num("vehicle.T_min", v.T_min);
  num("vehicle.T_max", v.T_max); num("vehicle.gamma_max", v.gamma_max);
  const auto& b = c.boundary;
  num("boundary.m_init", b.initial.m); vec("boundary.r_init", b.initial.r, 3); vec("boundary.v_init", b.initial.v, 3);
  vec("boundary.q_init", b.initial.q, 4); vec("boundary.w_init", b.initial.w, 3); vec("boundary.r_final", b.r_final, 3);
  vec("boundary.v_final", b.v_final, 3); vec("boundary.q_final", b.q_final, 4); vec("boundary.w_final", b.w_final, 3);
  integer("grid.N", c.grid_nodes); integer("grid.integrator_substeps", c.integrator_substeps);
  integer("grid.audit_substeps", c.audit_substeps);
  num("time.t_f_guess", c.t_f_guess); num("time.s_min", c.s_min); num("time.s_max", c.s_max);
  num("scp.w_cost", c.weights.w_cost); num("scp.w_prox", c.weights.w_prox); num("scp.w_ep", c.weights.w_ep);
  num("scp.epsilon_relax", c.weights.epsilon_relax); num("scp.tol_feas", c.tol_feas); num("scp.tol_step", c.tol_step);
  integer("scp.max_iters", c.max_iters);
  num("scaling.mass", c.scaling.mass); num("scaling.position", c.scaling.position); num("scaling.velocity", c.scaling.velocity);
  num("scaling.quaternion", c.scaling.quaternion); num("scaling.omega", c.scaling.omega); num("scaling.y", c.scaling.y);
  num("scaling.thrust", c.scaling.thrust); num("scaling.torque", c.scaling.torque); num("scaling.dilation", c.scaling.dilation);
  num("pipg.omega", c.pipg_cfg.omega); num("pipg.rho", c.pipg_cfg.rho); integer("pipg.j_max", c.pipg_cfg.j_max);
  integer("pipg.j_check", c.pipg_cfg.j_check); num("pipg.eps_abs", c.pipg_cfg.eps_abs); num("pipg.eps_rel", c.pipg_cfg.eps_rel);
  num("pipg.eps_buff", c.pipg_cfg.eps_buff); integer("pipg.power_j_max", c.power_j_max);
  num("pipg.power_eps_abs", c.power_eps_abs); num("pipg.power_eps_rel", c.power_eps_rel);
  integer("montecarlo.batch_size", c.batch_size); integer("montecarlo.workers", c.workers);
  std::printf("  montecarlo.seed %llu\n", (unsigned long long)c.dispersion.seed);
  vec("montecarlo.dispersion_low", c.dispersion.r_low, 3); vec("montecarlo.dispersion_high", c.dispersion.r_high, 3);
  num("montecarlo.converged_floor", c.converged_floor);
  std::printf("  output_dir [%s]\n", c.output_dir.c_str());
  // the problem the solver entry points receive
  const auto pb = c.problem();
  integer("problem.nodes", (long long)pb.grid.nodes.size());
  num("problem.grid[1]", pb.grid.nodes[1]);
  std::printf("  problem.px");
  for (int i = 0; i < 15; ++i) std::printf(" %.17g", pb.scaling.px[i]);
  std::printf("\n  problem.pu");
  for (int i = 0; i < 7; ++i) std::printf(" %.17g", pb.scaling.pu[i]);
  std::printf("\n  problem.init_state");
  for (int i = 0; i < 14; ++i) std::printf(" %.17g", pb.init_state[i]);
  std::printf("\n  problem.final_fix");
  for (std::size_t i = 0; i < pb.final_fix_idx.size(); ++i) std::printf(" %d:%.17g", pb.final_fix_idx[i], pb.final_fix_val[i]);
  std::printf("\n  problem.rng_seed %llu max_iters %d power_j_max %d integrator_steps %d\n",
              (unsigned long long)pb.rng_seed, pb.max_iters, pb.power_j_max, pb.integrator_steps);
}

}  // namespace

int main(int argc, char** argv) {
  for (int k = 1; k < argc; ++k) {
    const std::string path = argv[k];
    const std::string name = path.substr(path.find_last_of('/') + 1);
    std::printf("== %s\n", name.c_str());
    try {
      dump(lib::load_config(path));
    } catch (const lib::ConfigError& e) {
      std::printf("  ConfigError: %s\n", e.what());
    } catch (const lib::ConfigParseError&) {
      std::printf("  ConfigParseError\n");
    }
  }
  return 0;
}
