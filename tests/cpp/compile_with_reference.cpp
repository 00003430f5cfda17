// TEST (compile-only, needs /root/reference): the host mirror accepts the reference's OWN types
// unchanged — ptopt::Trajectory, Grid, IntervalBlocks, pipg::Subproblem / Workspace / PipgConfig,
// ScpProblem<Rocket6DoF>, RocketBoundary, mc::DispersionSpec — which is what makes it a drop-in
// for the call sites named in INTEGRATION.md.  Nothing here is executed.
#include "ptopt/montecarlo.hpp"
#include "ptopt/rocket_problem.hpp"
#include "ptopt/scp.hpp"

#include "ptopt_b200.hpp"
#include "ptopt_b200_io.hpp"

namespace b2 = ptopt_b200;

double instantiate_everything(const ptopt::RocketProblem& pb, const ptopt::RocketBoundary& bc,
                              const ptopt::mc::DispersionSpec& spec) {
  const ptopt::RocketTrajectory guess = ptopt::initial_guess(pb, bc);
  // discretizer.hpp:191-194 / :82-86
  const auto blocks = b2::linearize_all(pb.model, guess, pb.grid, pb.integrator_steps, pb.linearize_workers);
  const auto one = b2::propagate_interval(pb.model, guess.x[0], guess.u[0], guess.u[1], pb.grid.nodes[0],
                                          pb.grid.nodes[1], pb.integrator_steps, 0);
  // scp.hpp:139-143, fed with the reference's own block type
  const std::vector<ptopt::BlocksOf<ptopt::rocket::Rocket6DoF>> ref_blocks =
      ptopt::linearize_all(pb.model, guess, pb.grid, pb.integrator_steps);
  const auto sp = b2::assemble_subproblem(pb, guess, ref_blocks);
  // pipg.hpp:206-211 / :350-352 on the reference's Subproblem / Workspace
  const ptopt::pipg::Subproblem<15, 7> ref_sp = ptopt::assemble_subproblem(pb, guess, ref_blocks);
  ptopt::pipg::Workspace<15, 7> ws;
  ws.init(15, 7, pb.grid.size());
  ws.sigma = b2::pipg::power_iteration_custom(ref_sp, guess.x, guess.u, ws.vc_pos, ws.vc_neg, 1e-12, 1e-12, 0.05,
                                              pb.power_j_max);
  const auto pr = b2::pipg::pipg_custom(ref_sp, pb.pipg_cfg, ws);
  // scp.hpp:256-258, discretizer.hpp:249-253, montecarlo.hpp:140-142
  const auto res = b2::scp_solve(pb, guess);
  const auto audit = b2::dense_violation_audit(pb.model, res.iterate, pb.grid, 64);
  std::vector<ptopt::AuditSample> ref_samples;  // the reference's own sample type
  b2::dense_violation_audit(pb.model, res.iterate, pb.grid, 64, &ref_samples);
  b2::csvio::write_dense_audit("/dev/null", ref_samples);
  const auto batch = b2::mc::run_batch(pb, bc, spec, 8, 4, 64, true);
  // output side (csv.hpp:34-96, montecarlo.hpp:177-209) on the reference's records / trajectory
  const std::vector<ptopt::mc::RunRecord> ref_records(2);
  const auto summary = b2::mc::aggregate(ref_records, 25, 1.0, 1);
  b2::csvio::write_runs("/dev/null", ref_records);
  b2::csvio::write_summary("/dev/null", summary);
  b2::csvio::write_trajectory("/dev/null", guess, pb.grid);
  b2::csvio::write_runs("/dev/null", batch.records);
  return blocks[0].A(0, 0) + one.w[0] + sp.w[0][0] + pr.iterations + res.final_defect_inf + audit.max_pointwise_g +
         batch.records[0].propellant_used;
}

int main() { return 0; }
