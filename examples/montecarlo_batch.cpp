// montecarlo_batch.cpp — a Monte Carlo batch from a reference configuration file, end to end on
// the GPU: JSON config -> problem -> mc::run_batch (generation, SCP solves, dense audit, records on
// the device) -> runs.csv / summary.csv (/ trajectory_NNNN.csv).  It is the work of the reference's
// `ptopt montecarlo` subcommand (proj/tools/ptopt_main.cpp:102-140) written against this repo's
// host headers; the only reference-facing types are the ones those headers mirror.
//
//   g++ -std=c++17 -O2 -Iinclude -Ipaper_2404_18034_b200/host examples/montecarlo_batch.cpp
//       -Lpaper_2404_18034_b200 -lptopt_cuda -Wl,-rpath,$PWD/paper_2404_18034_b200 -o montecarlo_batch
//   ./montecarlo_batch run.json [--runs N] [--seed S] [--dump-trajectories]
//
// Exit codes as the reference: 0 ok, 1 converged fraction below the floor, 2 usage / config,
// 3 I/O.  `output_dir` must exist.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "ptopt_b200.hpp"
#include "ptopt_b200_config.hpp"
#include "ptopt_b200_io.hpp"

int main(int argc, char** argv) {
  namespace b2 = ptopt_b200;
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s config.json [--runs N] [--seed S] [--dump-trajectories]\n", argv[0]);
    return 2;
  }
  long long runs = -1, seed = -1;
  bool dump = false;
  for (int k = 2; k < argc; ++k) {
    if (!std::strcmp(argv[k], "--runs") && k + 1 < argc) runs = std::atoll(argv[++k]);
    else if (!std::strcmp(argv[k], "--seed") && k + 1 < argc) seed = std::atoll(argv[++k]);
    else if (!std::strcmp(argv[k], "--dump-trajectories")) dump = true;
    else {
      std::fprintf(stderr, "unknown argument %s\n", argv[k]);
      return 2;
    }
  }
  b2::RunConfig cfg;
  try {
    cfg = b2::load_config(argv[1]);
    if (runs > 0) cfg.batch_size = static_cast<int>(runs);
    if (seed >= 0) cfg.dispersion.seed = static_cast<std::uint64_t>(seed);
    cfg.validate();
  } catch (const b2::ConfigParseError& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  } catch (const b2::ConfigError& e) {
    std::fprintf(stderr, "invalid config: %s\n", e.what());
    return 2;
  }

  try {
    const b2::RocketProblem pb = cfg.problem();
    const b2::mc::BatchResult batch =
        b2::mc::run_batch(pb, cfg.boundary, cfg.dispersion, cfg.batch_size, cfg.workers, cfg.audit_substeps, dump);
    const b2::mc::Summary summary = b2::mc::aggregate(batch.records, cfg.max_iters, batch.total_wall_time, batch.workers);
    b2::csvio::write_runs(cfg.output_dir + "/runs.csv", batch.records);
    b2::csvio::write_summary(cfg.output_dir + "/summary.csv", summary);
    if (dump) {
      char name[64];
      for (std::size_t i = 0; i < batch.trajectories.size(); ++i) {
        if (!batch.records[i].failure.empty()) continue;  // a failed instance has no trajectory
        std::snprintf(name, sizeof name, "/trajectory_%04zu.csv", i);
        b2::csvio::write_trajectory(cfg.output_dir + name, batch.trajectories[i], pb.grid);
      }
    }
    std::printf("runs=%d converged_fraction=%.4f wall=%.2fs workers=%d\n", summary.batch_size,
                summary.converged_fraction, summary.total_wall_time, summary.workers);
    return summary.converged_fraction >= cfg.converged_floor ? 0 : 1;
  } catch (const b2::csvio::IoError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  } catch (const b2::CudaError& e) {
    std::fprintf(stderr, "CUDA error: %s\n", e.what());
    return 3;
  }
}
