// io_formats.cpp — TEST INFRASTRUCTURE.  Writes runs.csv / summary.csv / trajectory.csv for a
// fixed synthetic batch into the directory given as argv[1]:
//   default build            -> through paper_2404_18034_b200/host/ptopt_b200_io.hpp
//   -DWITH_REFERENCE build   -> through the reference's own csv.hpp / montecarlo.hpp (this is how
//                               tests/golden/io/*.csv were generated; see tests/test_io_formats.py)
#include <cmath>
#include <cstdint>
#include <limits>
#include <string>
#include <vector>

#ifdef WITH_REFERENCE
#include "ptopt/csv.hpp"
namespace lib = ptopt;
using Record = ptopt::mc::RunRecord;
using Traj = ptopt::RocketTrajectory;
using GridT = ptopt::Grid;
#else
#include "ptopt_b200.hpp"
#include "ptopt_b200_io.hpp"
namespace lib = ptopt_b200;
using Record = ptopt_b200::mc::RunRecord;
using Traj = ptopt_b200::RocketTrajectory;
using GridT = ptopt_b200::Grid;
#endif

namespace {

// splitmix-style counter hash -> awkward but reproducible doubles
double value(std::uint64_t i) {
  std::uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  const double u = (double)(z >> 11) * (1.0 / 9007199254740992.0);
  return std::ldexp(u - 0.5, (int)(i % 40) - 20);
}

std::vector<Record> make_records() {
  std::vector<Record> recs(12);
  for (int b = 0; b < 12; ++b) {
    Record& r = recs[(std::size_t)b];
    r.run_id = 1000 + b;
    for (int i = 0; i < 3; ++i) r.initial_position[(std::size_t)i] = 6.0 + value(10 * b + i);
    r.converged = b % 3 != 1;
    r.scp_iterations = b == 4 ? 0 : 1 + (7 * b) % 25;
    r.propellant_used = 0.5 + value(100 + b);
    r.final_defect_inf = std::fabs(value(200 + b)) * 1e-6;
    r.max_pointwise_g = value(300 + b);
    r.max_node_y_increase = b == 2 ? -0.0 : std::fabs(value(400 + b));
    r.wall_time = 0.25 * b;
  }
  recs[4].failure = "propagation diverged, interval 3\nsecond line, with commas";
  recs[7].propellant_used = std::numeric_limits<double>::denorm_min();
  recs[9].max_pointwise_g = 1.0 / 3.0;
  return recs;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::string dir = argv[1];
  const std::vector<Record> recs = make_records();
  lib::csvio::write_runs(dir + "/runs.csv", recs);
  lib::csvio::write_summary(dir + "/summary.csv", lib::mc::aggregate(recs, 25, 12.5, 8));
  // a summary whose histogram grows past max_iters and with no converged record
  std::vector<Record> none(recs.begin() + 1, recs.begin() + 2);
  none[0].scp_iterations = 30;
  lib::csvio::write_summary(dir + "/summary_none.csv", lib::mc::aggregate(none, 25));

  const int n = 9;
  GridT grid = GridT::uniform(n);
  Traj z(n);
  for (int k = 0; k < n; ++k) {
    for (int i = 0; i < 15; ++i) z.x[(std::size_t)k][i] = value(1000 + 15 * k + i);
    for (int i = 0; i < 7; ++i) z.u[(std::size_t)k][i] = value(2000 + 7 * k + i);
    z.u[(std::size_t)k][6] = 4.0 + value(3000 + k);  // dilation
  }
  lib::csvio::write_trajectory(dir + "/trajectory.csv", z, grid);

  std::vector<lib::AuditSample> samples(7);
  for (int i = 0; i < 7; ++i) {
    lib::AuditSample& s = samples[(std::size_t)i];
    s.interval = i / 3;
    s.tau = 0.125 * i + value(4000 + i);
    for (int q = 0; q < 9; ++q) s.g.push_back(value(5000 + 9 * i + q));
    s.g_max = value(6000 + i);
  }
  lib::csvio::write_dense_audit(dir + "/dense_audit.csv", samples);
  lib::csvio::write_dense_audit(dir + "/dense_audit_empty.csv", std::vector<lib::AuditSample>{});
  return 0;
}
