// ptopt_b200_io.hpp — the data formats on the output side of the hot path: the Monte Carlo
// summary and the CSV files the reference CLI writes from a batch.  Host-only plumbing (no CUDA),
// kept byte-compatible with the reference so that downstream tooling which diffs or parses
// `runs.csv`, `summary.csv` and `trajectory.csv` keeps working when `mc::run_batch` comes from
// ptopt_b200.hpp:
//
//   mc::aggregate(records, max_iters, wall, workers)   montecarlo.hpp:177-209
//   node_times(z, grid)                                rocket_problem.hpp:166-176
//   csvio::fmt / write_trajectory / write_dense_audit / write_runs / write_summary   csv.hpp:20-96
//
// All functions are templates over the record / trajectory types and only use the member names
// the reference's types have, so they take the reference's objects as well as this repo's.
// Numbers are printed with "%.17g" (round-trippable), `wall_time` stays the last column of
// runs.csv so byte comparisons can strip it (csv.hpp:66).
//
// The JSON configuration on the input side is in ptopt_b200_config.hpp.
#pragma once

#include <algorithm>
#include <cstdio>
#include <fstream>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

namespace ptopt_b200 {

/// Physical time of every node: trapezoid rule over the dilation factor (last control entry).
template <class Traj, class GridT>
std::vector<double> node_times(const Traj& z, const GridT& grid) {
  const std::size_t n = grid.nodes.size();
  std::vector<double> t(n, 0.0);
  const int s_index = 6;  // RocketAug::s_index
  for (std::size_t k = 1; k < n; ++k) {
    const double dt = grid.nodes[k] - grid.nodes[k - 1];
    const double s0 = z.u[k - 1][s_index];
    const double s1 = z.u[k][s_index];
    t[k] = t[k - 1] + 0.5 * (s0 + s1) * dt;
  }
  return t;
}

namespace mc {

struct Summary {  // montecarlo.hpp:87-96
  int batch_size = 0;
  double converged_fraction = 0.0;
  std::vector<int> iteration_histogram;  // bins 1..max_iters
  double propellant_min = 0.0, propellant_mean = 0.0, propellant_max = 0.0;
  double total_wall_time = 0.0;
  int workers = 0;
};

/// Batch statistics: iteration histogram over every record, propellant statistics over the
/// converged ones (in record order, so the mean is summed as the reference sums it).
template <class Record>
Summary aggregate(const std::vector<Record>& records, int max_iters = 0, double total_wall_time = 0.0,
                  int workers = 0) {
  if (records.empty()) throw std::invalid_argument("aggregate: no records");
  Summary s;
  s.batch_size = static_cast<int>(records.size());
  s.total_wall_time = total_wall_time;
  s.workers = workers;
  int bins = max_iters;
  for (const Record& r : records) bins = std::max(bins, r.scp_iterations);
  s.iteration_histogram.assign(static_cast<std::size_t>(bins), 0);
  int n_conv = 0;
  double prop_sum = 0.0;
  for (const Record& r : records) {
    if (r.scp_iterations >= 1) ++s.iteration_histogram[static_cast<std::size_t>(r.scp_iterations - 1)];
    if (!r.converged) continue;
    prop_sum += r.propellant_used;
    if (n_conv == 0) {
      s.propellant_min = s.propellant_max = r.propellant_used;
    } else {
      s.propellant_min = std::min(s.propellant_min, r.propellant_used);
      s.propellant_max = std::max(s.propellant_max, r.propellant_used);
    }
    ++n_conv;
  }
  s.converged_fraction = static_cast<double>(n_conv) / s.batch_size;
  s.propellant_mean = n_conv > 0 ? prop_sum / n_conv : 0.0;
  return s;
}

}  // namespace mc

namespace csvio {

struct IoError : std::runtime_error {  // csv.hpp:15-17
  using std::runtime_error::runtime_error;
};

/// Round-trippable decimal float.
inline std::string fmt(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

namespace detail {

/// A failure text must not break the row structure.
inline std::string one_cell(std::string s) {
  std::replace(s.begin(), s.end(), ',', ';');
  std::replace(s.begin(), s.end(), '\n', ';');
  return s;
}

/// Opens `path`, runs `body(out)`, and reports any stream failure as IoError.
template <class Body>
void write_file(const std::string& path, Body body) {
  std::ofstream out(path);
  if (!out) throw IoError("cannot write " + path);
  body(out);
  if (!out) throw IoError("failed while writing " + path);
}

}  // namespace detail

// ---- stream forms (what the file forms write) ------------------------------------------------
template <class Traj, class GridT>
void trajectory_csv(std::ostream& out, const Traj& z, const GridT& grid) {
  out << "tau,t,m,rx,ry,rz,vx,vy,vz,qx,qy,qz,qw,wx,wy,wz,y,Tx,Ty,Tz,gx,gy,gz,s\n";
  const std::vector<double> t = node_times(z, grid);
  for (std::size_t k = 0; k < grid.nodes.size(); ++k) {
    out << fmt(grid.nodes[k]) << ',' << fmt(t[k]);
    for (int i = 0; i < 15; ++i) out << ',' << fmt(z.x[k][i]);
    for (int i = 0; i < 7; ++i) out << ',' << fmt(z.u[k][i]);
    out << '\n';
  }
}

template <class Sample>
void dense_audit_csv(std::ostream& out, const std::vector<Sample>& samples) {
  out << "interval,tau";
  const std::size_t ng = samples.empty() ? 0 : samples.front().g.size();
  for (std::size_t i = 0; i < ng; ++i) out << ",g" << (i + 1);
  out << ",g_max\n";
  for (const Sample& s : samples) {
    out << s.interval << ',' << fmt(s.tau);
    for (double g : s.g) out << ',' << fmt(g);
    out << ',' << fmt(s.g_max) << '\n';
  }
}

template <class Record>
void runs_csv(std::ostream& out, const std::vector<Record>& records) {
  out << "run_id,r0_1,r0_2,r0_3,converged,scp_iterations,propellant_used,"
         "final_defect_inf,max_pointwise_g,max_node_y_increase,failure,wall_time\n";
  for (const Record& r : records) {
    out << r.run_id;
    for (int i = 0; i < 3; ++i) out << ',' << fmt(r.initial_position[static_cast<std::size_t>(i)]);
    out << ',' << (r.converged ? 1 : 0) << ',' << r.scp_iterations;
    for (double v : {r.propellant_used, r.final_defect_inf, r.max_pointwise_g, r.max_node_y_increase})
      out << ',' << fmt(v);
    out << ',' << detail::one_cell(r.failure) << ',' << fmt(r.wall_time) << '\n';
  }
}

template <class SummaryT>
void summary_csv(std::ostream& out, const SummaryT& s) {
  out << "key,value\n";
  out << "batch_size," << s.batch_size << '\n';
  const std::pair<const char*, double> reals[] = {{"converged_fraction", s.converged_fraction},
                                                  {"propellant_min", s.propellant_min},
                                                  {"propellant_mean", s.propellant_mean},
                                                  {"propellant_max", s.propellant_max},
                                                  {"total_wall_time", s.total_wall_time}};
  for (const auto& kv : reals) out << kv.first << ',' << fmt(kv.second) << '\n';
  out << "workers," << s.workers << '\n';
  for (std::size_t i = 0; i < s.iteration_histogram.size(); ++i)
    out << "iterations_" << (i + 1) << ',' << s.iteration_histogram[i] << '\n';
}

// ---- file forms: csv.hpp:34-96 -----------------------------------------------------------------
template <class Traj, class GridT>
void write_trajectory(const std::string& path, const Traj& z, const GridT& grid) {
  detail::write_file(path, [&](std::ostream& out) { trajectory_csv(out, z, grid); });
}

template <class Sample>
void write_dense_audit(const std::string& path, const std::vector<Sample>& samples) {
  detail::write_file(path, [&](std::ostream& out) { dense_audit_csv(out, samples); });
}

template <class Record>
void write_runs(const std::string& path, const std::vector<Record>& records) {
  detail::write_file(path, [&](std::ostream& out) { runs_csv(out, records); });
}

template <class SummaryT>
void write_summary(const std::string& path, const SummaryT& s) {
  detail::write_file(path, [&](std::ostream& out) { summary_csv(out, s); });
}

}  // namespace csvio

}  // namespace ptopt_b200
