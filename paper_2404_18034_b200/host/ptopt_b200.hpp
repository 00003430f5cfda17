// ptopt_b200.hpp — C++ host mirror of the reference solver API for the SCP hot path, routed to
// the CUDA library through the C-ABI of include/ptopt_cuda.h.
//
// The reference (/root/reference/proj/include/ptopt) is a header-only template library; its
// "operator API" for this path is a handful of free functions.  This header keeps those names,
// argument meanings and error behaviour:
//
//   linearize_all(model, z, grid, steps, workers)        discretizer.hpp:191-194
//   propagate_interval(model, x_k, u_k, u_k1, ...)        discretizer.hpp:82-86
//   assemble_subproblem(pb, zbar, blocks)                 scp.hpp:139-143
//   pipg::power_iteration_custom(sp, seeds..., eps, j)    pipg.hpp:206-211
//   pipg::pipg_custom(sp, cfg, ws)                        pipg.hpp:350-352
//   scp_solve(pb, guess)                                  scp.hpp:256-258
//   dense_violation_audit(model, z, grid, substeps, &samples)  discretizer.hpp:249-253
//   initial_guess(pb, bc)                                 rocket_problem.hpp:127-163
//   mc::run_batch(nominal, bc, spec, batch, workers, ..)  montecarlo.hpp:140-142
//
// Every function is a template over its container arguments and touches them only through
// the members the reference's own types have (`v[i]`, `v.n`, `m(i, j)`, `z.x[k]`, `grid.nodes`,
// `pb.weights.w_prox`, ...).  So the reference's `ptopt::Vec`, `ptopt::Mat`, `Trajectory`,
// `Grid`, `pipg::Subproblem`, `pipg::Workspace`, `ScpProblem<Rocket6DoF>` can be passed as they
// are, and so can the equivalent plain types defined below for callers that do not have the
// reference headers.  Results come back in the types of this header (same member names).
//
// Errors follow the reference: std::invalid_argument for argument errors, std::domain_error
// for model-domain errors, PropagationDiverged{interval}, pipg::SolverDiverged{iteration}.
// A CUDA failure (or no sm_100 device) throws ptopt_b200::CudaError — there is no CPU path.
//
// Device context: the reference functions take no context argument, so the handle
// (`ptopt_cuda_handle`) is looked up in a per-thread cache keyed by the problem description.
// Handles are created on first use on device `ptopt_b200::device()` (default 0;
// `set_device(i)` switches the calling thread to another GPU).
#pragma once

#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ptopt_cuda.h"

namespace ptopt_b200 {

// =============================================================================================
// plain containers with the reference's shape (smallmat.hpp:13-72, trajectory.hpp:11-48)
// =============================================================================================
template <int Cap>
struct Vec {
  int n = Cap;
  std::array<double, static_cast<std::size_t>(Cap)> a{};
  Vec() = default;
  explicit Vec(int len) : n(len) {
    if (len < 0 || len > Cap) throw std::invalid_argument("Vec: length outside capacity");
  }
  double& operator[](int i) { return a[static_cast<std::size_t>(i)]; }
  double operator[](int i) const { return a[static_cast<std::size_t>(i)]; }
};

template <int RCap, int CCap>
struct Mat {
  int rows = RCap, cols = CCap;
  std::array<double, static_cast<std::size_t>(RCap) * static_cast<std::size_t>(CCap)> a{};
  Mat() = default;
  Mat(int r, int c) : rows(r), cols(c) {
    if (r < 0 || r > RCap || c < 0 || c > CCap) throw std::invalid_argument("Mat: shape outside capacity");
  }
  double& operator()(int i, int j) { return a[static_cast<std::size_t>(i * cols + j)]; }
  double operator()(int i, int j) const { return a[static_cast<std::size_t>(i * cols + j)]; }
};

struct Grid {
  std::vector<double> nodes;
  explicit Grid(std::vector<double> taus) : nodes(std::move(taus)) {
    if (nodes.size() < 2) throw std::invalid_argument("grid needs at least two nodes");
    if (nodes.front() != 0.0 || nodes.back() != 1.0)
      throw std::invalid_argument("grid must start at 0 and end at 1");
    for (std::size_t k = 1; k < nodes.size(); ++k)
      if (!(nodes[k] > nodes[k - 1])) throw std::invalid_argument("grid nodes must be strictly increasing");
  }
  static Grid uniform(int n) {
    if (n < 2) throw std::invalid_argument("grid needs at least two nodes");
    std::vector<double> t(static_cast<std::size_t>(n));
    for (int k = 0; k < n; ++k) t[static_cast<std::size_t>(k)] = static_cast<double>(k) / (n - 1);
    t.front() = 0.0;
    t.back() = 1.0;
    return Grid(std::move(t));
  }
  int size() const { return static_cast<int>(nodes.size()); }
  int intervals() const { return size() - 1; }
};

constexpr int kNX = PTOPT_NX, kNU = PTOPT_NU, kNXI = PTOPT_NXI;

template <int NX = kNX, int NU = kNU>
struct Trajectory {
  std::vector<Vec<NX>> x;
  std::vector<Vec<NU>> u;
  int iteration = 0;
  Trajectory() = default;
  explicit Trajectory(int n) : x(static_cast<std::size_t>(n)), u(static_cast<std::size_t>(n)) {}
  int nodes() const { return static_cast<int>(x.size()); }
};
using RocketTrajectory = Trajectory<kNX, kNU>;

template <int NX = kNX, int NU = kNU>
struct IntervalBlocks {  // discretizer.hpp:44-51
  Mat<NX, NX> A;
  Mat<NX, NU> B_minus, B_plus;
  Vec<NX> w, x_end;
};
using RocketBlocks = IntervalBlocks<kNX, kNU>;

// =============================================================================================
// errors
// =============================================================================================
struct CudaError : std::runtime_error {
  int code;
  CudaError(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

struct PropagationDiverged : std::runtime_error {  // discretizer.hpp:18-23
  int interval;
  explicit PropagationDiverged(int k)
      : std::runtime_error("state propagation diverged in interval " + std::to_string(k)), interval(k) {}
};

namespace pipg {
struct SolverDiverged : std::runtime_error {  // pipg.hpp:16-20
  int iteration;
  explicit SolverDiverged(int j)
      : std::runtime_error("pipg diverged at iteration " + std::to_string(j)), iteration(j) {}
};
}  // namespace pipg

namespace detail {

inline void check_call(int rc) {
  if (rc == PTOPT_OK) return;
  const std::string msg = ptopt_cuda_last_error();
  if (rc == PTOPT_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw CudaError(rc, msg);
}

/// Per-instance status -> the exception the reference throws for it.
[[noreturn]] inline void throw_instance(int status, int fail_index) {
  switch (status) {
    case PTOPT_ST_PROPAGATION_DIVERGED: throw PropagationDiverged(fail_index);
    case PTOPT_ST_SOLVER_DIVERGED: throw pipg::SolverDiverged(fail_index);
    case PTOPT_ST_DILATION_NONPOSITIVE: throw std::domain_error("augmented dynamics: dilation factor must be positive");  // ctcs.hpp:66
    case PTOPT_ST_MASS_NONPOSITIVE: throw std::domain_error("rocket dynamics: nonpositive mass");
    case PTOPT_ST_THRUST_SINGULAR:
      throw std::domain_error("rocket jacobians: thrust magnitude below singular-point tolerance");
    case PTOPT_ST_POWER_SEED_ZERO:
      throw std::invalid_argument("power iteration: seed point must not be all zero");
    default: throw std::runtime_error("ptopt_b200: unknown instance status " + std::to_string(status));
  }
}

inline std::string failure_text(int status, int fail_index) {
  try {
    throw_instance(status, fail_index);
  } catch (const std::exception& e) {
    return e.what();
  }
}

inline int& device_slot() {
  thread_local int dev = 0;
  return dev;
}

struct HandleDeleter {
  void operator()(ptopt_cuda_handle* h) const { ptopt_cuda_destroy(h); }
};
using HandlePtr = std::unique_ptr<ptopt_cuda_handle, HandleDeleter>;

/// Per-thread cache of handles keyed by (device, description bytes, grid).
inline ptopt_cuda_handle* context(const ptopt_problem_desc& d, const std::vector<double>& tau) {
  thread_local std::map<std::string, HandlePtr> cache;
  std::string key(reinterpret_cast<const char*>(&d), sizeof d);
  key.append(reinterpret_cast<const char*>(tau.data()), tau.size() * sizeof(double));
  const int dev = device_slot();
  key.append(reinterpret_cast<const char*>(&dev), sizeof dev);
  auto it = cache.find(key);
  if (it == cache.end()) {
    if (cache.size() >= 8) cache.clear();  // handles own device scratch: keep the cache small
    ptopt_cuda_handle* h = nullptr;
    check_call(ptopt_cuda_create(&d, tau.data(), dev, nullptr, &h));
    it = cache.emplace(std::move(key), HandlePtr(h)).first;
  }
  return it->second.get();
}

}  // namespace detail

inline int device() { return detail::device_slot(); }
inline void set_device(int dev) { detail::device_slot() = dev; }

// =============================================================================================
// vehicle model (rocket6dof.hpp:85-144, 226-241)
// =============================================================================================
namespace rocket {

constexpr int kMass = 0, kPos = 1, kVel = 4, kAtt = 7, kRate = 11;
constexpr int kThrust = 0, kTorque = 3;

struct VehicleParams {
  double alpha_mdot = 0.0;
  std::array<double, 3> g_inertial{};
  Mat<3, 3> inertia;
  std::array<double, 3> r_thrust{};
  Mat<2, 4> H_theta = tilt_selector();
  double m_dry = 0.0, v_max = 0.0, theta_max = 0.0, omega_max = 0.0, delta_max = 0.0;
  double T_min = 0.0, T_max = 0.0, gamma_max = 0.0;
  static Mat<2, 4> tilt_selector() {
    Mat<2, 4> H(2, 4);
    H(0, 1) = 1.0;
    H(1, 2) = 1.0;
    return H;
  }
};

class Rocket6DoF {
 public:
  static constexpr int state_dim = kNXI, control_dim = PTOPT_NZETA, ineq_dim = PTOPT_NG, eq_dim = 0;
  explicit Rocket6DoF(const VehicleParams& p) : p_(p) {}
  const VehicleParams& params() const { return p_; }

 private:
  VehicleParams p_;
};

struct VehicleState {  // rocket6dof.hpp:27-60
  double m = 0.0;
  std::array<double, 3> r{}, v{};
  std::array<double, 4> q{0.0, 0.0, 0.0, 1.0};
  std::array<double, 3> w{};
  Vec<kNXI> to_vec() const {
    Vec<kNXI> x;
    x[kMass] = m;
    for (int i = 0; i < 3; ++i) {
      x[kPos + i] = r[i];
      x[kVel + i] = v[i];
      x[kRate + i] = w[i];
    }
    for (int i = 0; i < 4; ++i) x[kAtt + i] = q[i];
    return x;
  }
};

}  // namespace rocket

namespace detail {

template <class VP>
ptopt_vehicle_params to_c_vehicle(const VP& p) {
  ptopt_vehicle_params c{};
  c.alpha_mdot = p.alpha_mdot;
  for (int i = 0; i < 3; ++i) {
    c.g_inertial[i] = p.g_inertial[static_cast<std::size_t>(i)];
    c.r_thrust[i] = p.r_thrust[static_cast<std::size_t>(i)];
    for (int j = 0; j < 3; ++j) c.inertia[i * 3 + j] = p.inertia(i, j);
  }
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 4; ++j) c.H_theta[i * 4 + j] = p.H_theta(i, j);
  c.m_dry = p.m_dry;
  c.v_max = p.v_max;
  c.theta_max = p.theta_max;
  c.omega_max = p.omega_max;
  c.delta_max = p.delta_max;
  c.T_min = p.T_min;
  c.T_max = p.T_max;
  c.gamma_max = p.gamma_max;
  return c;
}

/// A description that carries only what the discretizer needs; the SCP fields get the
/// reference's defaults (scp.hpp:18-22, 82-103; pipg.hpp:22-29) so that it validates.
template <class VP>
ptopt_problem_desc discretizer_desc(const VP& p, int nodes, int steps) {
  ptopt_problem_desc d{};
  d.vehicle = to_c_vehicle(p);
  d.nodes = nodes;
  d.integrator_steps = steps;
  d.s_min = 0.1;
  d.s_max = 10.0;
  d.t_f_guess = 1.0;
  d.w_cost = 1.0;
  d.w_prox = 1.0;
  d.w_ep = 100.0;
  d.epsilon_relax = 1e-4;
  for (int i = 0; i < kNX; ++i) d.px[i] = 1.0;
  for (int i = 0; i < kNU; ++i) d.pu[i] = 1.0;
  d.pipg = ptopt_pipg_config{100.0, 1.6, 2500, 25, 1e-11, 1e-11, 0.05};
  d.power_j_max = 10000;
  d.max_iters = 25;
  d.power_eps_abs = d.power_eps_rel = 1e-12;
  d.tol_feas = 1e-6;
  d.tol_step = 1e-5;
  return d;
}

template <class Traj>
void flatten_trajectory(const Traj& z, int n, std::vector<double>& x, std::vector<double>& u) {
  x.resize(static_cast<std::size_t>(n) * kNX);
  u.resize(static_cast<std::size_t>(n) * kNU);
  for (int k = 0; k < n; ++k) {
    for (int i = 0; i < kNX; ++i) x[static_cast<std::size_t>(k * kNX + i)] = z.x[static_cast<std::size_t>(k)][i];
    for (int i = 0; i < kNU; ++i) u[static_cast<std::size_t>(k * kNU + i)] = z.u[static_cast<std::size_t>(k)][i];
  }
}

}  // namespace detail

// =============================================================================================
// exact discretization (discretizer.hpp:82-149, 191-232)
// =============================================================================================

/// linearize_all: every interval of the iterate, on the device.  `workers` is accepted for
/// signature compatibility; the device runs one warp per interval regardless.
template <class Model, class Traj, class GridT>
std::vector<RocketBlocks> linearize_all(const Model& model, const Traj& z, const GridT& grid, int steps,
                                        int workers = 1) {
  if (steps < 1) throw std::invalid_argument("propagate_interval: steps must be >= 1");
  if (workers < 1) throw std::invalid_argument("linearize_all: workers must be >= 1");
  const int n = static_cast<int>(grid.nodes.size()), m = n - 1;
  if (static_cast<int>(z.x.size()) != n || static_cast<int>(z.u.size()) != n)
    throw std::invalid_argument("linearize_all: trajectory and grid sizes differ");
  const ptopt_problem_desc d = detail::discretizer_desc(model.params(), n, steps);
  ptopt_cuda_handle* h = detail::context(d, grid.nodes);
  std::vector<double> x, u;
  detail::flatten_trajectory(z, n, x, u);
  const std::size_t M = static_cast<std::size_t>(m);
  std::vector<double> A(M * kNX * kNX), Bm(M * kNX * kNU), Bp(M * kNX * kNU), w(M * kNX), xe(M * kNX);
  int32_t status = 0, fail_index = -1;
  detail::check_call(ptopt_cuda_linearize_batch(h, 1, x.data(), u.data(), A.data(), Bm.data(), Bp.data(),
                                                w.data(), xe.data(), &status, &fail_index));
  if (status != PTOPT_ST_OK) detail::throw_instance(status, fail_index);
  std::vector<RocketBlocks> out(M);
  for (std::size_t k = 0; k < M; ++k) {
    RocketBlocks& b = out[k];
    for (int i = 0; i < kNX; ++i) {
      for (int j = 0; j < kNX; ++j) b.A(i, j) = A[(k * kNX + i) * kNX + j];
      for (int j = 0; j < kNU; ++j) {
        b.B_minus(i, j) = Bm[(k * kNX + i) * kNU + j];
        b.B_plus(i, j) = Bp[(k * kNX + i) * kNU + j];
      }
      b.w[i] = w[k * kNX + i];
      b.x_end[i] = xe[k * kNX + i];
    }
  }
  return out;
}

/// propagate_interval (discretizer.hpp:82-149) of a single interval.
template <class Model, class VX, class VU>
RocketBlocks propagate_interval(const Model& model, const VX& x_k, const VU& u_k, const VU& u_k1,
                                double tau_k, double tau_k1, int steps, int interval_index = 0) {
  if (steps < 1) throw std::invalid_argument("propagate_interval: steps must be >= 1");
  const ptopt_problem_desc d = detail::discretizer_desc(model.params(), 2, steps);
  ptopt_cuda_handle* h = detail::context(d, std::vector<double>{0.0, 1.0});
  double x[kNX], u0[kNU], u1[kNU];
  for (int i = 0; i < kNX; ++i) x[i] = x_k[i];
  for (int i = 0; i < kNU; ++i) {
    u0[i] = u_k[i];
    u1[i] = u_k1[i];
  }
  double A[kNX * kNX], Bm[kNX * kNU], Bp[kNX * kNU], w[kNX], xe[kNX];
  int32_t status = 0;
  detail::check_call(ptopt_cuda_propagate_interval_batch(h, 1, x, u0, u1, &tau_k, &tau_k1, steps, A, Bm, Bp, w,
                                                         xe, &status));
  if (status != PTOPT_ST_OK) detail::throw_instance(status, interval_index);
  RocketBlocks b;
  for (int i = 0; i < kNX; ++i) {
    for (int j = 0; j < kNX; ++j) b.A(i, j) = A[i * kNX + j];
    for (int j = 0; j < kNU; ++j) {
      b.B_minus(i, j) = Bm[i * kNU + j];
      b.B_plus(i, j) = Bp[i * kNU + j];
    }
    b.w[i] = w[i];
    b.x_end[i] = xe[i];
  }
  return b;
}

struct AuditSample {  // discretizer.hpp:236-240
  int interval = 0;
  double tau = 0.0;
  std::vector<double> g;
  double g_max = 0.0;
};

struct AuditResult {  // discretizer.hpp:241-245
  double max_pointwise_g = 0.0;
  double total_y_increase = 0.0;
  std::vector<double> interval_y_increase;
};

/// dense_violation_audit (discretizer.hpp:249-285).  `samples`, when given, receives one
/// AuditSample per node / substep in the reference's order (appended, as the reference does).
template <class Model, class Traj, class GridT, class SampleT = AuditSample>
AuditResult dense_violation_audit(const Model& model, const Traj& z, const GridT& grid, int substeps,
                                  std::vector<SampleT>* samples = nullptr) {
  if (substeps < 1) throw std::invalid_argument("dense_violation_audit: substeps must be >= 1");
  const int n = static_cast<int>(grid.nodes.size());
  const ptopt_problem_desc d = detail::discretizer_desc(model.params(), n, 1);
  ptopt_cuda_handle* h = detail::context(d, grid.nodes);
  std::vector<double> x, u;
  detail::flatten_trajectory(z, n, x, u);
  AuditResult r;
  r.interval_y_increase.resize(static_cast<std::size_t>(n - 1));
  int32_t status = 0, fail_index = -1;
  if (samples) {
    const std::size_t count = static_cast<std::size_t>(n - 1) * static_cast<std::size_t>(substeps + 1);
    std::vector<double> flat(count * PTOPT_AUDIT_SAMPLE_DOUBLES);
    detail::check_call(ptopt_cuda_dense_audit_samples_batch(h, 1, substeps, x.data(), u.data(), flat.data(),
                                                            &r.max_pointwise_g, r.interval_y_increase.data(),
                                                            &status, &fail_index));
    if (status != PTOPT_ST_OK) detail::throw_instance(status, fail_index);
    samples->reserve(samples->size() + count);
    for (std::size_t i = 0; i < count; ++i) {
      const double* f = &flat[i * PTOPT_AUDIT_SAMPLE_DOUBLES];
      SampleT smp;
      smp.interval = static_cast<int>(f[0]);
      smp.tau = f[1];
      smp.g.assign(f + 2, f + 2 + PTOPT_NG);
      smp.g_max = f[2 + PTOPT_NG];
      samples->push_back(std::move(smp));
    }
  } else {
    detail::check_call(ptopt_cuda_dense_audit_batch(h, 1, substeps, x.data(), u.data(), &r.max_pointwise_g,
                                                    r.interval_y_increase.data(), &status, &fail_index));
    if (status != PTOPT_ST_OK) detail::throw_instance(status, fail_index);
  }
  for (double dy : r.interval_y_increase) r.total_y_increase += dy;
  return r;
}

// =============================================================================================
// customized PIPG (pipg.hpp)
// =============================================================================================
namespace pipg {

struct PipgConfig {  // pipg.hpp:22-38
  double omega = 100.0, rho = 1.6;
  int j_max = 2500, j_check = 25;
  double eps_abs = 1e-11, eps_rel = 1e-11, eps_buff = 0.05;
  void validate() const {
    if (!(omega > 0.0)) throw std::invalid_argument("pipg.omega must be > 0");
    if (!(rho > 0.0 && rho < 2.0)) throw std::invalid_argument("pipg.rho must lie in (0, 2)");
    if (j_check < 1) throw std::invalid_argument("pipg.j_check must be >= 1");
    if (j_max < 1) throw std::invalid_argument("pipg.j_max must be >= 1");
    if (!(eps_buff >= 0.0)) throw std::invalid_argument("pipg.eps_buff must be >= 0");
  }
};

template <int NX = kNX, int NU = kNU>
struct Subproblem {  // pipg.hpp:43-96
  int n_x = 0, n_u = 0, nodes = 0;
  std::vector<Mat<NX, NX>> A_minus, A_plus;
  std::vector<Mat<NX, NU>> B_minus, B_plus;
  std::vector<Vec<NX>> w;
  std::vector<double> eps_relax;
  Vec<NX> e_y;
  std::vector<Vec<NU>> u_min, u_max;
  std::vector<int> init_fix_idx, final_fix_idx;
  std::vector<double> init_fix_val, final_fix_val;
  Vec<NX> e_cost;
  double w_cost = 0.0, w_prox = 0.0, w_ep = 0.0;
  int intervals() const { return nodes - 1; }
  void resize(int nx, int nu, int n) {
    if (nx < 1 || nx > NX || nu < 1 || nu > NU || n < 2) throw std::invalid_argument("subproblem: bad dimensions");
    n_x = nx;
    n_u = nu;
    nodes = n;
    const auto m = static_cast<std::size_t>(n - 1);
    A_minus.assign(m, Mat<NX, NX>(nx, nx));
    A_plus.assign(m, Mat<NX, NX>(nx, nx));
    B_minus.assign(m, Mat<NX, NU>(nx, nu));
    B_plus.assign(m, Mat<NX, NU>(nx, nu));
    w.assign(m, Vec<NX>(nx));
    eps_relax.assign(m, 0.0);
    e_y = Vec<NX>(nx);
    const double inf = std::numeric_limits<double>::infinity();
    Vec<NU> lo(nu), hi(nu);
    for (int i = 0; i < nu; ++i) {
      lo[i] = -inf;
      hi[i] = inf;
    }
    u_min.assign(static_cast<std::size_t>(n), lo);
    u_max.assign(static_cast<std::size_t>(n), hi);
    init_fix_idx.clear();
    init_fix_val.clear();
    final_fix_idx.clear();
    final_fix_val.clear();
    e_cost = Vec<NX>(nx);
  }
};

template <int NX = kNX, int NU = kNU>
struct Workspace {  // warm start / solution groups of pipg.hpp:100-141 (iteration buffers live on the device)
  int n_x = 0, n_u = 0, nodes = 0;
  double sigma = 0.0;
  std::vector<Vec<NX>> x;
  std::vector<Vec<NU>> u;
  std::vector<Vec<NX>> vc_pos, vc_neg, dyn_dual;
  std::vector<double> relax_dual;
  void init(int nx, int nu, int n) {
    n_x = nx;
    n_u = nu;
    nodes = n;
    sigma = 0.0;
    x.assign(static_cast<std::size_t>(n), Vec<NX>(nx));
    u.assign(static_cast<std::size_t>(n), Vec<NU>(nu));
    vc_pos.assign(static_cast<std::size_t>(n - 1), Vec<NX>(nx));
    vc_neg = dyn_dual = vc_pos;
    relax_dual.assign(static_cast<std::size_t>(n - 1), 0.0);
  }
  bool primal_all_zero() const {
    auto any = [](const auto& group) {
      for (const auto& v : group)
        for (int i = 0; i < v.n; ++i)
          if (v[i] != 0.0) return true;
      return false;
    };
    return !(any(x) || any(u) || any(vc_pos) || any(vc_neg));
  }
};

struct PipgResult {  // pipg.hpp:342-345
  int iterations = 0;
  bool converged = false;
};

inline void step_sizes(double lambda, double omega, double sigma, double& alpha, double& beta) {  // :335-340
  alpha = 2.0 / (lambda + std::sqrt(lambda * lambda + 4.0 * omega * sigma));
  beta = omega * alpha;
}

namespace detail {

/// Dense instance-major copies of a Subproblem in the layout of ptopt_subproblem_arrays.
struct FlatSub {
  ptopt_subproblem_shape shape{};
  std::vector<double> A_minus, A_plus, B_minus, B_plus, w, eps, u_min, u_max, init_val, final_val;
  ptopt_subproblem_arrays arrays{};
};

template <class Sub>
FlatSub flatten(const Sub& sp, bool need_boundary) {
  if (sp.n_x < 1 || sp.n_x > kNX || sp.n_u < 1 || sp.n_u > kNU || sp.nodes < 2)
    throw std::invalid_argument("subproblem: bad dimensions");
  FlatSub f;
  const int nx = sp.n_x, nu = sp.n_u, n = sp.nodes, m = n - 1;
  f.shape.n_x = nx;
  f.shape.n_u = nu;
  f.shape.nodes = n;
  f.shape.n_init_fix = static_cast<int>(sp.init_fix_idx.size());
  f.shape.n_final_fix = static_cast<int>(sp.final_fix_idx.size());
  if (sp.init_fix_idx.size() != sp.init_fix_val.size() || sp.final_fix_idx.size() != sp.final_fix_val.size() ||
      f.shape.n_init_fix > kNX || f.shape.n_final_fix > kNX)
    throw std::invalid_argument("subproblem: boundary index/value size mismatch");
  for (int i = 0; i < f.shape.n_init_fix; ++i) f.shape.init_fix_idx[i] = sp.init_fix_idx[static_cast<std::size_t>(i)];
  for (int i = 0; i < f.shape.n_final_fix; ++i) f.shape.final_fix_idx[i] = sp.final_fix_idx[static_cast<std::size_t>(i)];
  for (int i = 0; i < nx; ++i) {
    f.shape.e_y[i] = sp.e_y[i];
    f.shape.e_cost[i] = sp.e_cost[i];
  }
  f.shape.w_cost = sp.w_cost;
  f.shape.w_prox = sp.w_prox;
  f.shape.w_ep = sp.w_ep;
  const std::size_t M = static_cast<std::size_t>(m);
  f.A_minus.resize(M * nx * nx);
  f.B_minus.resize(M * nx * nu);
  f.B_plus.resize(M * nx * nu);
  f.w.resize(M * nx);
  f.eps.resize(M);
  bool minus_identity = sp.A_plus.size() == M;
  for (std::size_t k = 0; k < M; ++k) {
    for (int i = 0; i < nx; ++i) {
      for (int j = 0; j < nx; ++j) {
        f.A_minus[(k * nx + i) * nx + j] = sp.A_minus[k](i, j);
        if (minus_identity && sp.A_plus[k](i, j) != (i == j ? -1.0 : 0.0)) minus_identity = false;
      }
      for (int j = 0; j < nu; ++j) {
        f.B_minus[(k * nx + i) * nu + j] = sp.B_minus[k](i, j);
        f.B_plus[(k * nx + i) * nu + j] = sp.B_plus[k](i, j);
      }
      f.w[k * nx + i] = sp.w[k][i];
    }
    f.eps[k] = sp.eps_relax[k];
  }
  if (!minus_identity) {  // A_plus = -I is implicit on the device; anything else is uploaded
    f.A_plus.resize(M * nx * nx);
    for (std::size_t k = 0; k < M; ++k)
      for (int i = 0; i < nx; ++i)
        for (int j = 0; j < nx; ++j) f.A_plus[(k * nx + i) * nx + j] = sp.A_plus[k](i, j);
  }
  f.u_min.resize(static_cast<std::size_t>(n) * nu);
  f.u_max.resize(static_cast<std::size_t>(n) * nu);
  for (int k = 0; k < n; ++k)
    for (int i = 0; i < nu; ++i) {
      f.u_min[static_cast<std::size_t>(k * nu + i)] = sp.u_min[static_cast<std::size_t>(k)][i];
      f.u_max[static_cast<std::size_t>(k * nu + i)] = sp.u_max[static_cast<std::size_t>(k)][i];
    }
  f.init_val = sp.init_fix_val;
  f.final_val = sp.final_fix_val;
  (void)need_boundary;
  f.arrays.A_minus = f.A_minus.data();
  f.arrays.A_plus = f.A_plus.empty() ? nullptr : f.A_plus.data();
  f.arrays.B_minus = f.B_minus.data();
  f.arrays.B_plus = f.B_plus.data();
  f.arrays.w = f.w.data();
  f.arrays.eps_relax = f.eps.data();
  f.arrays.u_min = f.u_min.data();
  f.arrays.u_max = f.u_max.data();
  f.arrays.init_fix_val = f.init_val.empty() ? nullptr : f.init_val.data();
  f.arrays.final_fix_val = f.final_val.empty() ? nullptr : f.final_val.data();
  return f;
}

template <class Group>
std::vector<double> flatten_group(const Group& g, int count, int len) {
  if (static_cast<int>(g.size()) != count) throw std::invalid_argument("workspace/seed group has the wrong size");
  std::vector<double> out(static_cast<std::size_t>(count) * len);
  for (int k = 0; k < count; ++k)
    for (int i = 0; i < len; ++i) out[static_cast<std::size_t>(k * len + i)] = g[static_cast<std::size_t>(k)][i];
  return out;
}

template <class Group>
void unflatten_group(const std::vector<double>& flat, int count, int len, Group& g) {
  for (int k = 0; k < count; ++k)
    for (int i = 0; i < len; ++i) g[static_cast<std::size_t>(k)][i] = flat[static_cast<std::size_t>(k * len + i)];
}

/// Handle for shape-generic subproblem calls: any valid description will do.
inline ptopt_cuda_handle* generic_context() {
  rocket::VehicleParams p;
  p.alpha_mdot = 1.0;
  p.inertia(0, 0) = p.inertia(1, 1) = p.inertia(2, 2) = 1.0;
  p.m_dry = p.v_max = p.theta_max = p.omega_max = p.gamma_max = 1.0;
  p.delta_max = 0.5;
  p.T_min = 1.0;
  p.T_max = 2.0;
  const ptopt_problem_desc d = ptopt_b200::detail::discretizer_desc(p, 2, 1);
  return ptopt_b200::detail::context(d, std::vector<double>{0.0, 1.0});
}

}  // namespace detail

/// power_iteration_custom (pipg.hpp:206-292): (1 + eps_buff) * estimate of max spec H^T H.
template <class Sub, class GX, class GU, class GV>
double power_iteration_custom(const Sub& sp, const GX& seed_x, const GU& seed_u, const GV& seed_vcp,
                              const GV& seed_vcn, double eps_abs = 1e-10, double eps_rel = 1e-10,
                              double eps_buff = 0.05, int j_max = 5000) {
  if (j_max < 1) throw std::invalid_argument("power iteration: j_max must be >= 1");
  const detail::FlatSub f = detail::flatten(sp, false);
  const int n = sp.nodes, m = n - 1;
  const std::vector<double> sx = detail::flatten_group(seed_x, n, sp.n_x), su = detail::flatten_group(seed_u, n, sp.n_u);
  const std::vector<double> sp_ = detail::flatten_group(seed_vcp, m, sp.n_x), sn = detail::flatten_group(seed_vcn, m, sp.n_x);
  double sigma = 0.0;
  int32_t trips = 0, status = 0;
  ptopt_b200::detail::check_call(ptopt_cuda_power_iteration_batch(
      detail::generic_context(), 1, &f.shape, &f.arrays, sx.data(), su.data(), sp_.data(), sn.data(), eps_abs,
      eps_rel, eps_buff, j_max, &sigma, &trips, &status));
  if (status != PTOPT_ST_OK) ptopt_b200::detail::throw_instance(status, -1);
  return sigma;
}

/// pipg_custom (pipg.hpp:350-497): warm start in, solution out, through `ws`.
template <class Sub, class Cfg, class Ws>
PipgResult pipg_custom(const Sub& sp, const Cfg& cfg, Ws& ws) {
  cfg.validate();
  if (ws.n_x != sp.n_x || ws.n_u != sp.n_u || ws.nodes != sp.nodes)
    throw std::invalid_argument("pipg: workspace shape does not match the subproblem");
  // the reference accepts any sigma (Workspace::init leaves 0, and the power iteration returns 0
  // for an iterate in the operator's null space, pipg.hpp:280-284): alpha = 1 / w_prox then
  const detail::FlatSub f = detail::flatten(sp, true);
  const int n = sp.nodes, m = n - 1, nx = sp.n_x, nu = sp.n_u;
  std::vector<double> x = detail::flatten_group(ws.x, n, nx), u = detail::flatten_group(ws.u, n, nu);
  std::vector<double> vp = detail::flatten_group(ws.vc_pos, m, nx), vn = detail::flatten_group(ws.vc_neg, m, nx);
  std::vector<double> dd = detail::flatten_group(ws.dyn_dual, m, nx);
  std::vector<double> rd(ws.relax_dual.begin(), ws.relax_dual.end());
  ptopt_workspace_arrays w{x.data(), u.data(), vp.data(), vn.data(), dd.data(), rd.data()};
  const ptopt_pipg_config c{cfg.omega, cfg.rho, cfg.j_max, cfg.j_check, cfg.eps_abs, cfg.eps_rel, cfg.eps_buff};
  const double sigma = ws.sigma;
  int32_t iters = 0, status = 0, fail_index = -1;
  uint8_t conv = 0;
  ptopt_b200::detail::check_call(ptopt_cuda_pipg_batch(detail::generic_context(), 1, &f.shape, &f.arrays, &c, &sigma,
                                                       &w, &iters, &conv, &status, &fail_index));
  if (status != PTOPT_ST_OK) ptopt_b200::detail::throw_instance(status, fail_index);
  detail::unflatten_group(x, n, nx, ws.x);
  detail::unflatten_group(u, n, nu, ws.u);
  detail::unflatten_group(vp, m, nx, ws.vc_pos);
  detail::unflatten_group(vn, m, nx, ws.vc_neg);
  detail::unflatten_group(dd, m, nx, ws.dyn_dual);
  for (int k = 0; k < m; ++k) ws.relax_dual[static_cast<std::size_t>(k)] = rd[static_cast<std::size_t>(k)];
  return PipgResult{iters, conv != 0};
}

}  // namespace pipg

// =============================================================================================
// SCP driver (scp.hpp)
// =============================================================================================
struct ScpWeights {  // scp.hpp:18-30
  double w_cost = 1.0, w_prox = 1.0, w_ep = 100.0, epsilon_relax = 1e-4;
};

template <int NX = kNX, int NU = kNU>
struct ScalingPair {  // scp.hpp:34-68
  Vec<NX> px, px_inv;
  Vec<NU> pu, pu_inv;
  static double pow2_near(double v) {
    if (!(v > 0.0)) throw std::invalid_argument("scaling ranges must be positive");
    return std::exp2(std::round(std::log2(v)));
  }
  static ScalingPair from_ranges(const Vec<NX>& xr, const Vec<NU>& ur) {
    ScalingPair s;
    s.px = s.px_inv = Vec<NX>(xr.n);
    s.pu = s.pu_inv = Vec<NU>(ur.n);
    for (int i = 0; i < xr.n; ++i) {
      s.px[i] = pow2_near(xr[i]);
      s.px_inv[i] = 1.0 / s.px[i];
    }
    for (int i = 0; i < ur.n; ++i) {
      s.pu[i] = pow2_near(ur[i]);
      s.pu_inv[i] = 1.0 / s.pu[i];
    }
    return s;
  }
  static ScalingPair identity(int nx, int nu) {
    Vec<NX> xr(nx);
    Vec<NU> ur(nu);
    for (int i = 0; i < nx; ++i) xr[i] = 1.0;
    for (int i = 0; i < nu; ++i) ur[i] = 1.0;
    return from_ranges(xr, ur);
  }
};

/// ScpProblem<Rocket6DoF> (scp.hpp:73-121) with the same member names.
struct RocketProblem {
  static constexpr int NX = kNX, NU = kNU;
  rocket::Rocket6DoF model;
  Grid grid = Grid::uniform(2);
  int integrator_steps = 16;
  int linearize_workers = 1;
  Vec<kNXI> init_state;
  std::vector<int> final_fix_idx;
  std::vector<double> final_fix_val;
  Vec<kNX> e_cost;
  double s_min = 0.1, s_max = 10.0, t_f_guess = 1.0;
  ScpWeights weights;
  ScalingPair<kNX, kNU> scaling = ScalingPair<kNX, kNU>::identity(kNX, kNU);
  pipg::PipgConfig pipg_cfg;
  int power_j_max = 10000;
  double power_eps_abs = 1e-12, power_eps_rel = 1e-12;
  double tol_feas = 1e-6, tol_step = 1e-5;
  int max_iters = 25;
  std::uint64_t rng_seed = 0;
  /// Present = quaternion renormalisation after every update (rocket_problem.hpp:86-92); the
  /// device implements exactly that hook, the callable itself is never invoked.
  std::function<void(Vec<kNX>&)> state_post_update;
  explicit RocketProblem(rocket::Rocket6DoF m) : model(std::move(m)) {}
};

namespace detail {

template <class Problem>
ptopt_problem_desc to_desc(const Problem& pb) {
  ptopt_problem_desc d{};
  d.vehicle = to_c_vehicle(pb.model.params());
  d.nodes = static_cast<int>(pb.grid.nodes.size());
  d.integrator_steps = pb.integrator_steps;
  d.s_min = pb.s_min;
  d.s_max = pb.s_max;
  d.t_f_guess = pb.t_f_guess;
  d.w_cost = pb.weights.w_cost;
  d.w_prox = pb.weights.w_prox;
  d.w_ep = pb.weights.w_ep;
  d.epsilon_relax = pb.weights.epsilon_relax;
  for (int i = 0; i < kNX; ++i) {
    d.px[i] = pb.scaling.px[i];
    d.e_cost[i] = pb.e_cost[i];
  }
  for (int i = 0; i < kNU; ++i) d.pu[i] = pb.scaling.pu[i];
  d.pipg = ptopt_pipg_config{pb.pipg_cfg.omega, pb.pipg_cfg.rho, pb.pipg_cfg.j_max, pb.pipg_cfg.j_check,
                             pb.pipg_cfg.eps_abs, pb.pipg_cfg.eps_rel, pb.pipg_cfg.eps_buff};
  d.power_j_max = pb.power_j_max;
  d.max_iters = pb.max_iters;
  d.power_eps_abs = pb.power_eps_abs;
  d.power_eps_rel = pb.power_eps_rel;
  d.tol_feas = pb.tol_feas;
  d.tol_step = pb.tol_step;
  if (pb.final_fix_idx.size() != pb.final_fix_val.size())
    throw std::invalid_argument("scp: final boundary index/value size mismatch");
  if (pb.final_fix_idx.size() > static_cast<std::size_t>(kNX))
    throw std::invalid_argument("scp: too many final boundary rows");
  d.n_final_fix = static_cast<int>(pb.final_fix_idx.size());
  for (int i = 0; i < d.n_final_fix; ++i) {
    d.final_fix_idx[i] = pb.final_fix_idx[static_cast<std::size_t>(i)];
    d.final_fix_val[i] = pb.final_fix_val[static_cast<std::size_t>(i)];
  }
  d.renormalize_quaternion = pb.state_post_update ? 1 : 0;
  return d;
}

}  // namespace detail

/// assemble_subproblem (scp.hpp:139-217): blocks + iterate -> scaled subproblem.
template <class Problem, class Traj, class BlocksVec>
pipg::Subproblem<kNX, kNU> assemble_subproblem(const Problem& pb, const Traj& zbar, const BlocksVec& blocks) {
  const int n = static_cast<int>(pb.grid.nodes.size()), m = n - 1;
  if (static_cast<int>(zbar.x.size()) != n || static_cast<int>(blocks.size()) != m)
    throw std::invalid_argument("assemble_subproblem: size mismatch");
  const ptopt_problem_desc d = detail::to_desc(pb);
  ptopt_cuda_handle* h = detail::context(d, pb.grid.nodes);
  std::vector<double> x, u;
  detail::flatten_trajectory(zbar, n, x, u);
  const std::size_t M = static_cast<std::size_t>(m);
  std::vector<double> A(M * kNX * kNX), Bm(M * kNX * kNU), Bp(M * kNX * kNU), xe(M * kNX);
  for (std::size_t k = 0; k < M; ++k)
    for (int i = 0; i < kNX; ++i) {
      for (int j = 0; j < kNX; ++j) A[(k * kNX + i) * kNX + j] = blocks[k].A(i, j);
      for (int j = 0; j < kNU; ++j) {
        Bm[(k * kNX + i) * kNU + j] = blocks[k].B_minus(i, j);
        Bp[(k * kNX + i) * kNU + j] = blocks[k].B_plus(i, j);
      }
      xe[k * kNX + i] = blocks[k].x_end[i];
    }
  std::vector<double> init(kNXI);
  for (int i = 0; i < kNXI; ++i) init[static_cast<std::size_t>(i)] = pb.init_state[i];
  const int nf = d.n_final_fix;
  std::vector<double> Am(M * kNX * kNX), Bmh(M * kNX * kNU), Bph(M * kNX * kNU), wh(M * kNX), eps(M);
  std::vector<double> umin(static_cast<std::size_t>(n) * kNU), umax(static_cast<std::size_t>(n) * kNU), iv(kNX),
      fv(static_cast<std::size_t>(nf > 0 ? nf : 1));
  detail::check_call(ptopt_cuda_assemble_batch(h, 1, init.data(), x.data(), u.data(), A.data(), Bm.data(), Bp.data(),
                                               xe.data(), Am.data(), Bmh.data(), Bph.data(), wh.data(), eps.data(),
                                               umin.data(), umax.data(), iv.data(), fv.data()));
  ptopt_subproblem_shape shape{};
  detail::check_call(ptopt_cuda_subproblem_shape(h, &shape));
  pipg::Subproblem<kNX, kNU> sp;
  sp.resize(kNX, kNU, n);
  for (std::size_t k = 0; k < M; ++k) {
    for (int i = 0; i < kNX; ++i) {
      for (int j = 0; j < kNX; ++j) {
        sp.A_minus[k](i, j) = Am[(k * kNX + i) * kNX + j];
        sp.A_plus[k](i, j) = i == j ? -1.0 : 0.0;
      }
      for (int j = 0; j < kNU; ++j) {
        sp.B_minus[k](i, j) = Bmh[(k * kNX + i) * kNU + j];
        sp.B_plus[k](i, j) = Bph[(k * kNX + i) * kNU + j];
      }
      sp.w[k][i] = wh[k * kNX + i];
    }
    sp.eps_relax[k] = eps[k];
  }
  for (int k = 0; k < n; ++k)
    for (int i = 0; i < kNU; ++i) {
      sp.u_min[static_cast<std::size_t>(k)][i] = umin[static_cast<std::size_t>(k * kNU + i)];
      sp.u_max[static_cast<std::size_t>(k)][i] = umax[static_cast<std::size_t>(k * kNU + i)];
    }
  for (int i = 0; i < kNX; ++i) {
    sp.e_y[i] = shape.e_y[i];
    sp.e_cost[i] = shape.e_cost[i];
  }
  for (int i = 0; i < shape.n_init_fix; ++i) {
    sp.init_fix_idx.push_back(shape.init_fix_idx[i]);
    sp.init_fix_val.push_back(iv[static_cast<std::size_t>(i)]);
  }
  for (int i = 0; i < shape.n_final_fix; ++i) {
    sp.final_fix_idx.push_back(shape.final_fix_idx[i]);
    sp.final_fix_val.push_back(fv[static_cast<std::size_t>(i)]);
  }
  sp.w_cost = shape.w_cost;
  sp.w_prox = shape.w_prox;
  sp.w_ep = shape.w_ep;
  return sp;
}

struct ScpHistoryEntry {  // scp.hpp:219-226
  double defect_inf = 0.0, step_inf = 0.0, penalized_cost = 0.0;
  int pipg_iterations = 0;
  double sigma = 0.0;
};

struct ScpResult {  // scp.hpp:228-235
  RocketTrajectory iterate;
  int iterations = 0;
  bool converged = false;
  double final_defect_inf = std::numeric_limits<double>::infinity();
  std::vector<ScpHistoryEntry> history;
};

/// scp_solve (scp.hpp:256-364): the whole loop on the device under one CUDA graph.
/// Non-convergence is reported, not thrown; a failing instance throws what the reference throws.
template <class Problem, class Traj>
ScpResult scp_solve(const Problem& pb, const Traj& guess) {
  const int n = static_cast<int>(pb.grid.nodes.size());
  if (static_cast<int>(guess.x.size()) != n || static_cast<int>(guess.u.size()) != n)
    throw std::invalid_argument("scp_solve: guess and grid sizes differ");
  const ptopt_problem_desc d = detail::to_desc(pb);
  ptopt_cuda_handle* h = detail::context(d, pb.grid.nodes);
  std::vector<double> xg, ug;
  detail::flatten_trajectory(guess, n, xg, ug);
  std::vector<double> init(kNXI);
  for (int i = 0; i < kNXI; ++i) init[static_cast<std::size_t>(i)] = pb.init_state[i];
  const uint64_t seed = pb.rng_seed;
  std::vector<double> xo(xg.size()), uo(ug.size());
  std::vector<double> hist(static_cast<std::size_t>(d.max_iters) * PTOPT_HISTORY_FIELDS);
  int32_t iters = 0, status = 0, fail_index = -1;
  uint8_t conv = 0;
  double fdef = 0.0;
  detail::check_call(ptopt_cuda_scp_solve_batch(h, 1, init.data(), xg.data(), ug.data(), &seed, xo.data(), uo.data(),
                                                &iters, &conv, &fdef, hist.data(), nullptr, &status, &fail_index));
  if (status != PTOPT_ST_OK) detail::throw_instance(status, fail_index);
  ScpResult r;
  r.iterate = RocketTrajectory(n);
  for (int k = 0; k < n; ++k) {
    for (int i = 0; i < kNX; ++i) r.iterate.x[static_cast<std::size_t>(k)][i] = xo[static_cast<std::size_t>(k * kNX + i)];
    for (int i = 0; i < kNU; ++i) r.iterate.u[static_cast<std::size_t>(k)][i] = uo[static_cast<std::size_t>(k * kNU + i)];
  }
  r.iterate.iteration = iters;
  r.iterations = iters;
  r.converged = conv != 0;
  r.final_defect_inf = fdef;
  for (int it = 0; it < iters; ++it) {
    const double* e = &hist[static_cast<std::size_t>(it) * PTOPT_HISTORY_FIELDS];
    r.history.push_back(ScpHistoryEntry{e[0], e[1], e[2], static_cast<int>(e[3]), e[4]});
  }
  return r;
}

// =============================================================================================
// rocket glue (rocket_problem.hpp) and the Monte Carlo harness (montecarlo.hpp)
// =============================================================================================
struct RocketBoundary {  // rocket_problem.hpp:51-57
  rocket::VehicleState initial;
  std::array<double, 3> r_final{}, v_final{};
  std::array<double, 4> q_final{0.0, 0.0, 0.0, 1.0};
  std::array<double, 3> w_final{};
};

inline RocketProblem make_rocket_problem(const rocket::VehicleParams& params, const RocketBoundary& bc,
                                         const Grid& grid) {  // rocket_problem.hpp:59-94
  RocketProblem pb{rocket::Rocket6DoF(params)};
  pb.grid = grid;
  pb.init_state = bc.initial.to_vec();
  auto pin = [&](int base, const double* v, int count) {
    for (int i = 0; i < count; ++i) {
      pb.final_fix_idx.push_back(base + i);
      pb.final_fix_val.push_back(v[i]);
    }
  };
  pin(rocket::kPos, bc.r_final.data(), 3);
  pin(rocket::kVel, bc.v_final.data(), 3);
  pin(rocket::kAtt, bc.q_final.data(), 4);
  pin(rocket::kRate, bc.w_final.data(), 3);
  pb.e_cost[rocket::kMass] = -1.0;  // maximise terminal mass
  pb.state_post_update = [](Vec<kNX>&) {};  // marks the quaternion hook as present
  return pb;
}

namespace detail {
/// The device generator interpolates toward the terminal targets pinned in `pb`
/// (final_fix_idx / final_fix_val; an unpinned position, velocity or rate slot reads 0, an unpinned
/// attitude the identity), while the reference interpolates toward bc.*_final
/// (rocket_problem.hpp:144-148).  The two agree whenever `pb` was built from `bc`
/// (make_rocket_problem); anything else is refused instead of silently producing another guess.
template <class Problem, class Boundary>
inline void check_terminal_targets(const Problem& pb, const Boundary& bc) {
  double want[kNXI] = {0.0};
  for (int i = 0; i < 3; ++i) {
    want[1 + i] = bc.r_final[static_cast<std::size_t>(i)];
    want[4 + i] = bc.v_final[static_cast<std::size_t>(i)];
    want[11 + i] = bc.w_final[static_cast<std::size_t>(i)];
  }
  for (int i = 0; i < 4; ++i) want[7 + i] = bc.q_final[static_cast<std::size_t>(i)];
  double have[kNXI] = {0.0};
  have[10] = 1.0;  // identity attitude, scalar last
  for (std::size_t j = 0; j < pb.final_fix_idx.size(); ++j) {
    const int idx = pb.final_fix_idx[j];
    if (idx >= 0 && idx < kNXI) have[idx] = pb.final_fix_val[j];
  }
  for (int i = 1; i < kNXI; ++i)
    if (have[i] != want[i])
      throw std::invalid_argument("initial_guess: the boundary's terminal targets differ from the ones the problem pins "
                                  "(build the problem with make_rocket_problem from the same boundary)");
}
}  // namespace detail

/// initial_guess (rocket_problem.hpp:127-163): straight-line state interpolation, slerp of the
/// attitude and a gravity-cancelling thrust profile.  Evaluated by the device generator that
/// run_batch uses (ptopt_cuda_generate_batch with a dispersion box of zero width around the
/// initial position, which leaves it bit-for-bit unchanged), so there is one implementation.
/// The terminal targets are the ones `pb` was built with (make_rocket_problem).
template <class Problem, class Boundary>
RocketTrajectory initial_guess(const Problem& pb, const Boundary& bc) {
  detail::check_terminal_targets(pb, bc);
  const int n = static_cast<int>(pb.grid.nodes.size());
  const ptopt_problem_desc d = detail::to_desc(pb);
  ptopt_cuda_handle* h = detail::context(d, pb.grid.nodes);
  const auto init = bc.initial.to_vec();
  double nominal[kNXI];
  for (int i = 0; i < kNXI; ++i) nominal[i] = init[i];
  ptopt_dispersion_spec box{};
  for (int i = 0; i < 3; ++i) box.r_low[i] = box.r_high[i] = bc.initial.r[static_cast<std::size_t>(i)];
  std::vector<double> x(static_cast<std::size_t>(n) * kNX), u(static_cast<std::size_t>(n) * kNU);
  double init_out[kNXI];
  std::uint64_t seed_out = 0;
  detail::check_call(ptopt_cuda_generate_batch(h, 1, 0, nominal, &box, init_out, x.data(), u.data(), &seed_out));
  RocketTrajectory z(n);
  for (int k = 0; k < n; ++k) {
    for (int i = 0; i < kNX; ++i) z.x[static_cast<std::size_t>(k)][i] = x[static_cast<std::size_t>(k) * kNX + i];
    for (int i = 0; i < kNU; ++i) z.u[static_cast<std::size_t>(k)][i] = u[static_cast<std::size_t>(k) * kNU + i];
  }
  return z;
}

namespace mc {

struct DispersionSpec {  // montecarlo.hpp:20-31
  std::array<double, 3> r_low{}, r_high{};
  std::uint64_t seed = 0;
};

struct RunRecord {  // montecarlo.hpp:67-78
  int run_id = 0;
  std::array<double, 3> initial_position{};
  bool converged = false;
  int scp_iterations = 0;
  double propellant_used = 0.0, final_defect_inf = 0.0, max_pointwise_g = 0.0, max_node_y_increase = 0.0;
  std::string failure;
  double wall_time = 0.0;  // batch device+transfer time divided by the batch size
};

struct BatchResult {  // montecarlo.hpp:80-85
  std::vector<RunRecord> records;
  std::vector<RocketTrajectory> trajectories;
  double total_wall_time = 0.0;
  int workers = 0;
};

namespace detail {

template <class Spec>
inline ptopt_dispersion_spec to_c_spec(const Spec& spec) {
  ptopt_dispersion_spec cs{};
  for (int i = 0; i < 3; ++i) {
    cs.r_low[i] = spec.r_low[static_cast<std::size_t>(i)];
    cs.r_high[i] = spec.r_high[static_cast<std::size_t>(i)];
  }
  cs.seed = spec.seed;
  return cs;
}

/// ptopt_run_record[] (+ flat trajectories) -> BatchResult, montecarlo.hpp:67-85.
inline BatchResult to_batch_result(const std::vector<ptopt_run_record>& rec, const std::vector<double>& xo,
                                   const std::vector<double>& uo, int n, bool keep_trajectories, int workers,
                                   double wall_s) {
  BatchResult out;
  out.workers = workers;
  out.total_wall_time = wall_s;
  out.records.resize(rec.size());
  if (keep_trajectories) out.trajectories.resize(rec.size());
  for (std::size_t b = 0; b < rec.size(); ++b) {
    RunRecord& r = out.records[b];
    r.run_id = rec[b].run_id;
    for (int i = 0; i < 3; ++i) r.initial_position[static_cast<std::size_t>(i)] = rec[b].initial_position[i];
    r.converged = rec[b].converged != 0;
    r.scp_iterations = rec[b].scp_iterations;
    r.propellant_used = rec[b].propellant_used;
    r.final_defect_inf = rec[b].final_defect_inf;
    r.max_pointwise_g = rec[b].max_pointwise_g;
    r.max_node_y_increase = rec[b].max_node_y_increase;
    if (rec[b].status != PTOPT_ST_OK) r.failure = ptopt_b200::detail::failure_text(rec[b].status, rec[b].fail_index);
    r.wall_time = wall_s / static_cast<double>(rec.size());
    if (keep_trajectories && rec[b].status == PTOPT_ST_OK) {
      RocketTrajectory z(n);
      for (int k = 0; k < n; ++k) {
        for (int i = 0; i < kNX; ++i) z.x[static_cast<std::size_t>(k)][i] = xo[(b * n + k) * kNX + i];
        for (int i = 0; i < kNU; ++i) z.u[static_cast<std::size_t>(k)][i] = uo[(b * n + k) * kNU + i];
      }
      out.trajectories[b] = std::move(z);
    }
  }
  return out;
}

}  // namespace detail

/// run_batch (montecarlo.hpp:140-175): instance generation, solve, audit and records all on
/// the device, one CTA per instance.  `workers` is validated and echoed only; `first_run_id`
/// (an extension) lets several GPUs / processes take disjoint run-id ranges of one batch.
template <class Problem, class Boundary, class Spec>
BatchResult run_batch(const Problem& nominal, const Boundary& nominal_bc, const Spec& spec, int batch_size,
                      int workers, int audit_substeps = 64, bool keep_trajectories = false,
                      std::int64_t first_run_id = 0) {
  if (batch_size < 1) throw std::invalid_argument("montecarlo.batch_size must be >= 1");
  if (workers < 1) throw std::invalid_argument("montecarlo.workers must be >= 1");
  ptopt_b200::detail::check_terminal_targets(nominal, nominal_bc);
  const int n = static_cast<int>(nominal.grid.nodes.size());
  const ptopt_problem_desc d = ptopt_b200::detail::to_desc(nominal);
  ptopt_cuda_handle* h = ptopt_b200::detail::context(d, nominal.grid.nodes);
  const auto init = nominal_bc.initial.to_vec();
  double nominal_init[kNXI];
  for (int i = 0; i < kNXI; ++i) nominal_init[i] = init[i];
  const ptopt_dispersion_spec cs = detail::to_c_spec(spec);
  std::vector<ptopt_run_record> rec(static_cast<std::size_t>(batch_size));
  std::vector<double> xo, uo;
  if (keep_trajectories) {
    xo.resize(static_cast<std::size_t>(batch_size) * n * kNX);
    uo.resize(static_cast<std::size_t>(batch_size) * n * kNU);
  }
  const auto t0 = std::chrono::steady_clock::now();
  ptopt_b200::detail::check_call(ptopt_cuda_run_batch(h, batch_size, first_run_id, nominal_init, &cs, audit_substeps,
                                                      rec.data(), keep_trajectories ? xo.data() : nullptr,
                                                      keep_trajectories ? uo.data() : nullptr));
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return detail::to_batch_result(rec, xo, uo, n, keep_trajectories, workers, wall);
}

/// run_batch over the listed devices of this node: the reference's worker pool
/// (montecarlo.hpp:153-171) with one worker per device.  Entry g of `devices` solves the
/// contiguous run ids [g*batch/G, (g+1)*batch/G) on its own handle and host thread and writes
/// into the record slots of those ids, so the result equals the single-device batch bit for
/// bit whatever the device list (an ordinal may repeat).  `workers` of the result is the
/// number of device entries.
template <class Problem, class Boundary, class Spec>
BatchResult run_batch(const Problem& nominal, const Boundary& nominal_bc, const Spec& spec, int batch_size,
                      const std::vector<int>& devices, int audit_substeps = 64, bool keep_trajectories = false,
                      std::int64_t first_run_id = 0, std::vector<double>* device_ms = nullptr) {
  if (batch_size < 1) throw std::invalid_argument("montecarlo.batch_size must be >= 1");
  if (devices.empty()) throw std::invalid_argument("montecarlo.workers must be >= 1");
  ptopt_b200::detail::check_terminal_targets(nominal, nominal_bc);
  const int n = static_cast<int>(nominal.grid.nodes.size());
  const ptopt_problem_desc d = ptopt_b200::detail::to_desc(nominal);
  const auto init = nominal_bc.initial.to_vec();
  double nominal_init[kNXI];
  for (int i = 0; i < kNXI; ++i) nominal_init[i] = init[i];
  const ptopt_dispersion_spec cs = detail::to_c_spec(spec);
  std::vector<ptopt_run_record> rec(static_cast<std::size_t>(batch_size));
  std::vector<double> xo, uo;
  if (keep_trajectories) {
    xo.resize(static_cast<std::size_t>(batch_size) * n * kNX);
    uo.resize(static_cast<std::size_t>(batch_size) * n * kNU);
  }
  std::vector<double> tau(nominal.grid.nodes.begin(), nominal.grid.nodes.end());
  if (device_ms) device_ms->assign(devices.size(), 0.0);
  const auto t0 = std::chrono::steady_clock::now();
  ptopt_b200::detail::check_call(ptopt_cuda_run_batch_multi(
      &d, tau.data(), devices.data(), static_cast<int>(devices.size()), batch_size, first_run_id, nominal_init, &cs,
      audit_substeps, rec.data(), keep_trajectories ? xo.data() : nullptr, keep_trajectories ? uo.data() : nullptr,
      device_ms ? device_ms->data() : nullptr));
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return detail::to_batch_result(rec, xo, uo, n, keep_trajectories, static_cast<int>(devices.size()), wall);
}

}  // namespace mc

}  // namespace ptopt_b200
