// solve_nominal.cpp — one guidance problem from a reference configuration file, end to end on the
// GPU: JSON config -> problem -> initial guess -> scp_solve (whole SCP loop under one CUDA graph)
// -> dense violation audit -> trajectory.csv / dense_audit.csv (/ diagnostics.txt).  It is the
// work of the reference's `ptopt solve` subcommand (proj/tools/ptopt_main.cpp:46-94) written
// against this repo's host headers.
//
//   g++ -std=c++17 -O2 -Iinclude -Ipaper_2404_18034_b200/host examples/solve_nominal.cpp
//       -Lpaper_2404_18034_b200 -lptopt_cuda -Wl,-rpath,$PWD/paper_2404_18034_b200 -o solve_nominal
//   ./solve_nominal run.json
//
// Exit codes as the reference: 0 ok, 1 not converged / solve failed, 2 usage / config, 3 I/O.
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "ptopt_b200.hpp"
#include "ptopt_b200_config.hpp"
#include "ptopt_b200_io.hpp"

int main(int argc, char** argv) {
  namespace b2 = ptopt_b200;
  if (argc != 2) {
    std::fprintf(stderr, "usage: %s config.json\n", argv[0]);
    return 2;
  }
  b2::RunConfig cfg;
  try {
    cfg = b2::load_config(argv[1]);
  } catch (const b2::ConfigParseError& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  } catch (const b2::ConfigError& e) {
    std::fprintf(stderr, "invalid config: %s\n", e.what());
    return 2;
  }

  const b2::RocketProblem pb = cfg.problem();
  b2::ScpResult res;
  try {
    const b2::RocketTrajectory guess = b2::initial_guess(pb, cfg.boundary);
    res = b2::scp_solve(pb, guess);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "solve failed: %s\n", e.what());
    return 1;
  }

  try {
    std::vector<b2::AuditSample> samples;
    const b2::AuditResult audit = b2::dense_violation_audit(pb.model, res.iterate, pb.grid, cfg.audit_substeps, &samples);
    b2::csvio::write_trajectory(cfg.output_dir + "/trajectory.csv", res.iterate, pb.grid);
    b2::csvio::write_dense_audit(cfg.output_dir + "/dense_audit.csv", samples);
    const std::vector<double> t = b2::node_times(res.iterate, pb.grid);
    std::printf("converged=%d iterations=%d final_defect=%.3e t_f=%.6f mass_final=%.6f max_pointwise_g=%.3e\n",
                res.converged ? 1 : 0, res.iterations, res.final_defect_inf, t.back(),
                res.iterate.x.back()[b2::rocket::kMass], audit.max_pointwise_g);
    if (!res.converged) {
      std::ofstream diag(cfg.output_dir + "/diagnostics.txt");
      diag << "non-convergence diagnostics\n";
      diag << "iterations " << res.iterations << "\n";
      diag << "final_defect_inf " << res.final_defect_inf << "\n";
      diag << "iter defect_inf step_inf penalized_cost pipg_iterations sigma\n";
      for (std::size_t i = 0; i < res.history.size(); ++i) {
        const b2::ScpHistoryEntry& h = res.history[i];
        diag << (i + 1) << " " << h.defect_inf << " " << h.step_inf << " " << h.penalized_cost << " "
             << h.pipg_iterations << " " << h.sigma << "\n";
      }
      return 1;
    }
  } catch (const b2::csvio::IoError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "audit failed: %s\n", e.what());
    return 1;
  }
  return 0;
}
