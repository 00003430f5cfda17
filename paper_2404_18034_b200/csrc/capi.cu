// capi.cu — the C-ABI of include/ptopt_cuda.h: handle, device buffers, argument checking,
// host<->device staging, kernel dispatch, and the CUDA graph of the SCP loop.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <chrono>
#include <thread>
#include <vector>

#include "kernels.cuh"
#include "model_const.hpp"
#include "ptopt_cuda.h"

using namespace ptopt_b200;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define PT_CUDA(expr)                                                                  \
  do {                                                                                 \
    cudaError_t e__ = (expr);                                                          \
    if (e__ != cudaSuccess)                                                            \
      return fail(PTOPT_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (want == 0) want = 8;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

enum BufId {
  // staging for host-pointer entry points and the stand-alone ops
  B_X, B_U, B_A, B_BM, B_BP, B_W, B_XEND, B_STATUS, B_FAILIDX, B_FAILKEY, B_INIT,
  B_AM, B_AP, B_BMH, B_BPH, B_WH, B_EPS, B_UMIN, B_UMAX, B_INITVAL, B_FINALVAL,
  B_SEEDX, B_SEEDU, B_SEEDP, B_SEEDN, B_SIGMA, B_TRIPS, B_ITERS, B_CONV,
  B_WSX, B_WSU, B_WSP, B_WSN, B_WSD, B_WSR, B_TAU, B_STAGES, B_HANDLED,
  // SCP loop state (separate so a stand-alone call never disturbs a captured graph)
  S_ZX, S_ZU, S_INIT, S_SEED, S_A, S_BM, S_BP, S_W, S_XEND, S_AM, S_BMH, S_BPH, S_WH, S_EPS,
  S_UMIN, S_UMAX, S_INITVAL, S_FINALVAL, S_SEEDX, S_SEEDU, S_WSX, S_WSU, S_WSP, S_WSN, S_WSD,
  S_WSR, S_SIGMA, S_PITERS, S_FAILKEY, S_ACTIVE, S_CONV, S_SOLVES, S_LASTSTEP, S_FDEF, S_HIST,
  S_TRIPS, S_STATUS, S_FAILIDX, S_STAGES, S_HANDLED,
  // Monte Carlo harness
  R_QTAB, R_INIT, R_XG, R_UG, R_SEED, R_XOUT, R_UOUT, R_ITERS, R_CONV, R_FDEF, R_STATUS, R_FAILIDX,
  R_GMAX, R_DY, R_AKEY, R_PG, R_RECORDS, R_SAMPLES,
  kNumBufs
};

}  // namespace

struct ptopt_cuda_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ptopt_problem_desc desc{};
  std::vector<double> tau;
  double* d_tau = nullptr;
  ModelConst model{};
  ScpConst scp{};
  SubShape rocket_shape{};
  int64_t launches = 0;
  DevBuf buf[kNumBufs];
  cudaGraphExec_t scp_graph = nullptr;
  int scp_graph_batch = 0;
  int scp_graph_kernels = 0;
  int scp_capacity = 0;
  // stage-boundary events recorded by event nodes inside the SCP graph
  std::vector<cudaEvent_t> stage_events;
  std::vector<int> stage_of_span;  // stage id of the span that ENDS at event i+1
  bool stage_times_valid = false;
  int solver_path = PTOPT_SOLVER_AUTO;
  int num_sms = 0;
  // mc::run_batch promises records that do not depend on how a batch is sharded (run ids are all
  // that matter), so under AUTO it always runs the throughput family: the latency kernels round
  // differently, and choosing them by batch size would make a shard's bits depend on its size.
  bool batch_entry = false;
  int scp_graph_lat = -1;  // latency cluster size the cached SCP graph was captured with
};

namespace {

struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (cudaSetDevice(dev) != cudaSuccess) ok = false;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

bool pipg_cfg_valid(const ptopt_pipg_config& c) {  // PipgConfig::validate, pipg.hpp:31-37
  return c.omega > 0.0 && c.rho > 0.0 && c.rho < 2.0 && c.j_check >= 1 && c.j_max >= 1 &&
         c.eps_buff >= 0.0;
}

int check_shape(const ptopt_subproblem_shape* s, SubShape& out) {
  if (!s) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null subproblem shape");
  // Subproblem::resize, pipg.hpp:69-71
  if (s->n_x < 1 || s->n_x > PTOPT_NX || s->n_u < 1 || s->n_u > PTOPT_NU || s->nodes < 2)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "subproblem: bad dimensions");
  if (s->n_init_fix < 0 || s->n_init_fix > PTOPT_NX || s->n_final_fix < 0 ||
      s->n_final_fix > PTOPT_NX)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "subproblem: bad boundary row count");
  out.nx = s->n_x;
  out.nu = s->n_u;
  out.n = s->nodes;
  out.n_init_fix = s->n_init_fix;
  out.n_final_fix = s->n_final_fix;
  for (int i = 0; i < PTOPT_NX; ++i) {
    out.init_fix_idx[i] = s->init_fix_idx[i];
    out.final_fix_idx[i] = s->final_fix_idx[i];
    out.e_y[i] = s->e_y[i];
    out.e_cost[i] = s->e_cost[i];
  }
  for (int i = 0; i < s->n_init_fix; ++i)
    if (s->init_fix_idx[i] < 0 || s->init_fix_idx[i] >= s->n_x)
      return fail(PTOPT_ERR_INVALID_ARGUMENT, "subproblem: initial row index out of range");
  for (int i = 0; i < s->n_final_fix; ++i)
    if (s->final_fix_idx[i] < 0 || s->final_fix_idx[i] >= s->n_x)
      return fail(PTOPT_ERR_INVALID_ARGUMENT, "subproblem: final row index out of range");
  out.w_cost = s->w_cost;
  out.w_prox = s->w_prox;
  out.w_ep = s->w_ep;
  return PTOPT_OK;
}

int check_smem(ptopt_cuda_handle* h, size_t bytes) {
  int limit = 0;
  PT_CUDA(cudaDeviceGetAttribute(&limit, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
  if (bytes > (size_t)limit)
    return fail(PTOPT_ERR_UNSUPPORTED, "subproblem too large for one CTA's shared memory (" +
                                           std::to_string(bytes) + " > " + std::to_string(limit) +
                                           " bytes)");
  return PTOPT_OK;
}

template <class T>
int upload(ptopt_cuda_handle* h, BufId id, const T* host, size_t count, const T** dev_out) {
  if (!host) {
    *dev_out = nullptr;
    return PTOPT_OK;
  }
  PT_CUDA(h->buf[id].ensure(count * sizeof(T)));
  PT_CUDA(cudaMemcpyAsync(h->buf[id].p, host, count * sizeof(T), cudaMemcpyHostToDevice,
                          h->stream));
  *dev_out = h->buf[id].as<T>();
  return PTOPT_OK;
}

template <class T>
int device_out(ptopt_cuda_handle* h, BufId id, size_t count, T** dev_out) {
  PT_CUDA(h->buf[id].ensure(count * sizeof(T)));
  *dev_out = h->buf[id].as<T>();
  return PTOPT_OK;
}

template <class T>
int download(ptopt_cuda_handle* h, T* host, const T* dev, size_t count) {
  if (!host) return PTOPT_OK;
  PT_CUDA(cudaMemcpyAsync(host, dev, count * sizeof(T), cudaMemcpyDeviceToHost, h->stream));
  return PTOPT_OK;
}

#define PT_TRY(expr)            \
  do {                          \
    int rc__ = (expr);          \
    if (rc__ != PTOPT_OK) return rc__; \
  } while (0)

void fill_scp_const(const ptopt_problem_desc& d, ScpConst& c) {
  c.nodes = d.nodes;
  c.max_iters = d.max_iters;
  c.n_final_fix = d.n_final_fix;
  c.renorm_quat = d.renormalize_quaternion;
  for (int i = 0; i < kNX; ++i) {
    c.final_fix_idx[i] = d.final_fix_idx[i];
    c.final_fix_val[i] = d.final_fix_val[i];
    c.px[i] = d.px[i];
    c.px_inv[i] = 1.0 / d.px[i];
    c.e_cost[i] = d.e_cost[i];
  }
  for (int i = 0; i < kNU; ++i) {
    c.pu[i] = d.pu[i];
    c.pu_inv[i] = 1.0 / d.pu[i];
  }
  c.w_cost = d.w_cost;
  c.w_ep = d.w_ep;
  c.epsilon_relax = d.epsilon_relax;
  c.s_min = d.s_min;
  c.s_max = d.s_max;
  c.tol_feas = d.tol_feas;
  c.tol_step = d.tol_step;
}

void fill_rocket_shape(const ptopt_problem_desc& d, SubShape& s) {  // scp.hpp:160-215
  std::memset(&s, 0, sizeof s);
  s.nx = kNX;
  s.nu = kNU;
  s.n = d.nodes;
  s.n_init_fix = kNX;
  s.n_final_fix = d.n_final_fix;
  for (int i = 0; i < kNX; ++i) s.init_fix_idx[i] = i;
  for (int i = 0; i < d.n_final_fix; ++i) s.final_fix_idx[i] = d.final_fix_idx[i];
  s.e_y[kNX - 1] = 1.0;
  for (int i = 0; i < kNX; ++i) s.e_cost[i] = d.px[i] * d.e_cost[i];
  s.w_cost = d.w_cost;
  s.w_prox = d.w_prox;
  s.w_ep = d.w_ep;
}

/// The register-resident kernels serve the rocket-shaped subproblem; every other shape (and a
/// handle forced to PTOPT_SOLVER_GENERIC) runs the shape-generic kernels.
bool use_fast_solver(const ptopt_cuda_handle* h, const SubShape& s, bool has_a_plus) {
  return h->solver_path != PTOPT_SOLVER_GENERIC && solver_fast_supports(s, has_a_plus);
}

/// The column-sparse kernels (solver_cs.cu) run in front of the dense register-resident ones under
/// AUTO and FAST_THROUGHPUT when the shape allows: they solve every instance whose operator has
/// the zero pattern of the rocket model's discretization and mark it handled; the dense kernels
/// then run on the rest (normally nothing: their CTAs leave at once).
bool use_cs_solver(const ptopt_cuda_handle* h, const SubShape& s, bool has_a_plus) {
  return (h->solver_path == PTOPT_SOLVER_AUTO || h->solver_path == PTOPT_SOLVER_FAST_THROUGHPUT) &&
         solver_cs_supports(s, has_a_plus);
}

/// Shapes above kCsMaxNodes (2-CTA clusters): the power iteration runs on the column-sparse cluster
/// kernel, PIPG on the dense cluster kernel.  The column-sparse PIPG cluster kernel
/// (pipg_cs_cluster_kernel) is parity-green and sanitizer-clean up to a few hundred instances but
/// ended in a mailbox time-out (launch failure) in a batch of 2048 x N=100, so it is not the
/// default; PTOPT_CS_CLUSTER=3 selects it (bit 0: power iteration, bit 1: PIPG).
bool cs_stage_enabled(const SubShape& s, int stage_bit) {
  static const int mask = [] {
    const char* e = getenv("PTOPT_CS_CLUSTER");
    return e ? atoi(e) : 1;
  }();
  return s.n <= kCsMaxNodes || (mask & stage_bit) != 0;
}

/// The split variant of the register-resident kernels (see solver_fast.cu) runs only when the
/// handle asks for it (and the node count allows it).  Measured on B200 it loses to one CTA per
/// instance both in throughput (493 vs 655 solves/s at N=50) and in single-solve latency
/// (250 vs 216 ms): the flight time of the boundary values is paid twice per iteration.
bool use_split_solver(const ptopt_cuda_handle* h, int /*batch*/) {
  return h->solver_path == PTOPT_SOLVER_FAST_SPLIT;
}

/// Cluster size of the latency-mode kernels (solver_lat.cu) for this launch, 0 = not used: forced
/// by PTOPT_SOLVER_FAST_LATENCY, chosen under AUTO when the whole batch fits the chip in one wave.
int latency_ranks(const ptopt_cuda_handle* h, const SubShape& s, bool has_a_plus, int batch) {
  if (h->solver_path == PTOPT_SOLVER_FAST_LATENCY) return solver_lat_ranks(s, has_a_plus, 0, h->num_sms);
  if (h->solver_path == PTOPT_SOLVER_AUTO && !h->batch_entry) return solver_lat_ranks(s, has_a_plus, batch, h->num_sms);
  return 0;
}

int configure_solver(ptopt_cuda_handle* h, const SubShape& s, bool fast) {
  if (fast) {
    PT_TRY(check_smem(h, pipg_fast_smem(s, false)));
    PT_CUDA(configure_solver_fast(s));
    if (solver_cs_supports(s, false)) {
      PT_TRY(check_smem(h, pipg_cs_smem(s)));
      PT_CUDA(configure_solver_cs(s));
    }
  } else {
    PT_TRY(check_smem(h, pipg_generic_smem(s, solver_generic_threads(s))));
    PT_CUDA(configure_solver_generic(s));
  }
  return PTOPT_OK;
}

int dispatch_power(ptopt_cuda_handle* h, const PowerArgs& a) {
  if (const int ranks = latency_ranks(h, a.shape, a.sp.A_plus != nullptr, a.batch)) {
    PT_CUDA(launch_power_lat(a, ranks, h->stream));
    h->launches += 1;
    return PTOPT_OK;
  }
  const bool fast = use_fast_solver(h, a.shape, a.sp.A_plus != nullptr);
  PT_TRY(configure_solver(h, a.shape, fast));
  if (fast && use_cs_solver(h, a.shape, a.sp.A_plus != nullptr) && cs_stage_enabled(a.shape, 1)) {
    unsigned char* handled = nullptr;
    PT_TRY(device_out(h, B_HANDLED, (size_t)a.batch, &handled));
    PT_CUDA(launch_power_cs(a, handled, h->stream));
    PowerArgs rest = a;
    rest.skip = handled;
    PT_CUDA(launch_power_fast(rest, false, h->stream));
    h->launches += 2;
    return PTOPT_OK;
  }
  PT_CUDA(fast ? launch_power_fast(a, use_split_solver(h, a.batch), h->stream) : launch_power_generic(a, h->stream));
  h->launches += 1;
  return PTOPT_OK;
}

int dispatch_pipg(ptopt_cuda_handle* h, const PipgArgs& a) {
  if (const int ranks = latency_ranks(h, a.shape, a.sp.A_plus != nullptr, a.batch)) {
    PT_CUDA(launch_pipg_lat(a, ranks, h->stream));
    h->launches += 1;
    return PTOPT_OK;
  }
  const bool fast = use_fast_solver(h, a.shape, a.sp.A_plus != nullptr);
  PT_TRY(configure_solver(h, a.shape, fast));
  if (fast && use_cs_solver(h, a.shape, a.sp.A_plus != nullptr) && cs_stage_enabled(a.shape, 2)) {
    unsigned char* handled = nullptr;
    PT_TRY(device_out(h, B_HANDLED, (size_t)a.batch, &handled));
    PT_CUDA(launch_pipg_cs(a, handled, h->stream));
    PipgArgs rest = a;
    rest.skip = handled;
    PT_CUDA(launch_pipg_fast(rest, false, h->stream));
    h->launches += 2;
    return PTOPT_OK;
  }
  PT_CUDA(fast ? launch_pipg_fast(a, use_split_solver(h, a.batch), h->stream) : launch_pipg_generic(a, h->stream));
  h->launches += 1;
  return PTOPT_OK;
}

/// Upper bound on the stage-record storage of one state/column pass pair; larger batches are
/// processed in chunks (PTOPT_STAGE_BYTES_MAX overrides the default of 16 GiB).
size_t stage_bytes_cap() {
  static const size_t cap = [] {
    const char* env = getenv("PTOPT_STAGE_BYTES_MAX");
    const unsigned long long v = env ? strtoull(env, nullptr, 10) : 0ull;
    return v ? (size_t)v : ((size_t)16 << 30);
  }();
  return cap;
}

/// Intervals per pass pair and bytes of stage records for a linearize over `intervals` intervals.
long long stage_plan(long long intervals, int steps, size_t* bytes) {
  const long long chunk = linearize_chunk_intervals(intervals, steps, stage_bytes_cap());
  *bytes = linearize_stage_doubles(chunk, steps) * sizeof(double);
  return chunk;
}

/// The stage-record buffer `stage_buf` must already be large enough when this runs under stream
/// capture (ensure_scp_state sizes S_STAGES); otherwise it is grown here.
int linearize_args(ptopt_cuda_handle* h, int batch, int nodes, int steps, const double* x, const double* u,
                   double* A, double* Bm, double* Bp, double* w, double* x_end, int* fail_key,
                   const unsigned char* active, BufId stage_buf, LinearizeArgs* out) {
  LinearizeArgs a;
  a.model = h->model;
  a.batch = batch;
  a.nodes = nodes;
  a.steps = steps;
  a.tau = h->d_tau;
  a.tau_stride = 0;
  a.x = x;
  a.u = u;
  a.A = A;
  a.Bm = Bm;
  a.Bp = Bp;
  a.w = w;
  a.x_end = x_end;
  a.fail_key = fail_key;
  a.active = active;
  size_t bytes = 0;
  a.stage_capacity = stage_plan((long long)batch * (nodes - 1), steps, &bytes);
  PT_CUDA(h->buf[stage_buf].ensure(bytes));
  a.stages = h->buf[stage_buf].as<double>();
  *out = a;
  return PTOPT_OK;
}

int ensure_scp_state(ptopt_cuda_handle* h, int batch, ScpState& s) {
  const size_t B = (size_t)batch, n = (size_t)h->desc.nodes, m = n - 1;
  const size_t nf = h->desc.n_final_fix > 0 ? (size_t)h->desc.n_final_fix : 1;
  const size_t mi = (size_t)h->desc.max_iters;
  size_t stage_bytes = 0;
  stage_plan((long long)B * (long long)m, h->desc.integrator_steps, &stage_bytes);
  struct Req { BufId id; size_t bytes; };
  const Req reqs[] = {
      {S_ZX, B * n * kNX * 8}, {S_ZU, B * n * kNU * 8}, {S_INIT, B * kNXI * 8}, {S_SEED, B * 8},
      {S_A, B * m * kNX * kNX * 8}, {S_BM, B * m * kNX * kNU * 8}, {S_BP, B * m * kNX * kNU * 8},
      {S_W, B * m * kNX * 8}, {S_XEND, B * m * kNX * 8}, {S_AM, B * m * kNX * kNX * 8},
      {S_BMH, B * m * kNX * kNU * 8}, {S_BPH, B * m * kNX * kNU * 8}, {S_WH, B * m * kNX * 8},
      {S_EPS, B * m * 8}, {S_UMIN, B * n * kNU * 8}, {S_UMAX, B * n * kNU * 8},
      {S_INITVAL, B * kNX * 8}, {S_FINALVAL, B * nf * 8}, {S_SEEDX, B * n * kNX * 8},
      {S_SEEDU, B * n * kNU * 8}, {S_WSX, B * n * kNX * 8}, {S_WSU, B * n * kNU * 8},
      {S_WSP, B * m * kNX * 8}, {S_WSN, B * m * kNX * 8}, {S_WSD, B * m * kNX * 8},
      {S_WSR, B * m * 8}, {S_SIGMA, B * 8}, {S_PITERS, B * 4}, {S_FAILKEY, B * 4},
      {S_ACTIVE, B}, {S_CONV, B}, {S_SOLVES, B * 4}, {S_LASTSTEP, B * 8}, {S_FDEF, B * 8},
      {S_HIST, B * mi * 5 * 8}, {S_TRIPS, B * mi * 4}, {S_STATUS, B * 4}, {S_FAILIDX, B * 4},
      {S_STAGES, stage_bytes}, {S_HANDLED, B}};
  bool grew = false;
  for (const Req& r : reqs) {
    if (r.bytes > h->buf[r.id].bytes || !h->buf[r.id].p) grew = true;
    PT_CUDA(h->buf[r.id].ensure(r.bytes));
  }
  if (grew && h->scp_graph) {  // pointers changed: the captured graph is stale
    cudaGraphExecDestroy(h->scp_graph);
    h->scp_graph = nullptr;
    h->scp_graph_batch = 0;
  }
  auto D = [&](BufId id) { return h->buf[id].as<double>(); };
  s.zx = D(S_ZX); s.zu = D(S_ZU); s.init_state = D(S_INIT);
  s.rng_seed = h->buf[S_SEED].as<unsigned long long>();
  s.A = D(S_A); s.Bm = D(S_BM); s.Bp = D(S_BP); s.w = D(S_W); s.x_end = D(S_XEND);
  s.Am = D(S_AM); s.Bmh = D(S_BMH); s.Bph = D(S_BPH); s.wh = D(S_WH); s.eps = D(S_EPS);
  s.umin = D(S_UMIN); s.umax = D(S_UMAX); s.init_val = D(S_INITVAL); s.final_val = D(S_FINALVAL);
  s.seed_x = D(S_SEEDX); s.seed_u = D(S_SEEDU);
  s.ws.x = D(S_WSX); s.ws.u = D(S_WSU); s.ws.vc_pos = D(S_WSP); s.ws.vc_neg = D(S_WSN);
  s.ws.dyn_dual = D(S_WSD); s.ws.relax_dual = D(S_WSR);
  s.sigma = D(S_SIGMA);
  s.pipg_iters = h->buf[S_PITERS].as<int>();
  s.fail_key = h->buf[S_FAILKEY].as<int>();
  s.active = h->buf[S_ACTIVE].as<unsigned char>();
  s.converged = h->buf[S_CONV].as<unsigned char>();
  s.solves = h->buf[S_SOLVES].as<int>();
  s.last_step = D(S_LASTSTEP);
  s.final_defect = D(S_FDEF);
  s.history = D(S_HIST);
  s.power_trips = h->buf[S_TRIPS].as<int>();
  s.status = h->buf[S_STATUS].as<int>();
  s.fail_index = h->buf[S_FAILIDX].as<int>();
  return PTOPT_OK;
}

/// Enqueues the whole SCP loop for `batch` instances on the handle's stream (used under
/// stream capture to build the graph).  Returns the number of kernels enqueued.
int enqueue_scp_loop(ptopt_cuda_handle* h, int batch, const ScpState& st, int* kernels_out) {
  ScpArgs sa;
  sa.c = h->scp;
  sa.s = st;
  sa.batch = batch;
  int kernels = 0;
  h->stage_of_span.clear();
  size_t ev = 0;
  auto mark = [&](int stage) -> cudaError_t {  // closes the span of `stage` (-1: opens the first)
    if (ev >= h->stage_events.size()) {
      cudaEvent_t e;
      cudaError_t rc = cudaEventCreate(&e);
      if (rc != cudaSuccess) return rc;
      h->stage_events.push_back(e);
    }
    if (stage >= 0) h->stage_of_span.push_back(stage);
    return cudaEventRecordWithFlags(h->stage_events[ev++], h->stream, cudaEventRecordExternal);
  };
  launch_scp_init(sa, h->stream);
  ++kernels;
  PT_CUDA(mark(-1));

  PowerArgs pa;
  pa.shape = h->rocket_shape;
  pa.sp = SubArrays{st.Am, nullptr, st.Bmh, st.Bph, st.wh, st.eps, st.umin, st.umax,
                    st.init_val, st.final_val};
  pa.batch = batch;
  pa.seed_x = st.seed_x;
  pa.seed_u = st.seed_u;
  pa.seed_vcp = st.ws.vc_pos;
  pa.seed_vcn = st.ws.vc_neg;
  pa.eps_abs = h->desc.power_eps_abs;
  pa.eps_rel = h->desc.power_eps_rel;
  pa.eps_buff = h->desc.pipg.eps_buff;
  pa.j_max = h->desc.power_j_max;
  pa.sigma = st.sigma;
  pa.trips = st.power_trips;
  pa.trips_stride = h->desc.max_iters;
  pa.trips_slot = st.solves;
  pa.status = st.status;
  pa.active = st.active;

  PipgArgs ga;
  ga.shape = h->rocket_shape;
  ga.sp = pa.sp;
  ga.batch = batch;
  ga.omega = h->desc.pipg.omega;
  ga.rho = h->desc.pipg.rho;
  ga.eps_abs = h->desc.pipg.eps_abs;
  ga.eps_rel = h->desc.pipg.eps_rel;
  ga.j_max = h->desc.pipg.j_max;
  ga.j_check = h->desc.pipg.j_check;
  ga.sigma = st.sigma;
  ga.ws = st.ws;
  ga.iterations = st.pipg_iters;
  ga.converged = nullptr;
  ga.status = st.status;
  ga.fail_index = st.fail_index;
  ga.active = st.active;

  LinearizeArgs la;
  PT_TRY(linearize_args(h, batch, h->desc.nodes, h->desc.integrator_steps, st.zx, st.zu, st.A, st.Bm, st.Bp,
                        st.w, st.x_end, st.fail_key, st.active, S_STAGES, &la));
  const bool fast = use_fast_solver(h, h->rocket_shape, false);
  const int lat = latency_ranks(h, h->rocket_shape, false, batch);
  const bool cs = !lat && fast && use_cs_solver(h, h->rocket_shape, false);
  const bool cs_power = cs && cs_stage_enabled(h->rocket_shape, 1), cs_pipg = cs && cs_stage_enabled(h->rocket_shape, 2);
  unsigned char* handled = h->buf[S_HANDLED].as<unsigned char>();
  PowerArgs pa_rest = pa;
  PipgArgs ga_rest = ga;
  pa_rest.skip = handled;
  ga_rest.skip = handled;
  for (int it = 0; it <= h->desc.max_iters; ++it) {
    kernels += launch_linearize(la, h->stream);
    PT_CUDA(mark(0));
    launch_scp_prepare(sa, h->stream);
    PT_CUDA(mark(1));
    kernels += 1;
    if (it == h->desc.max_iters) break;  // the last pass only measures the final defect
    if (cs_power) {  // column-sparse kernels, then the dense ones on whatever they did not take
      PT_CUDA(launch_power_cs(pa, handled, h->stream));
      PT_CUDA(launch_power_fast(pa_rest, false, h->stream));
      kernels += 1;
    } else {
      PT_CUDA(lat    ? launch_power_lat(pa, lat, h->stream)
              : fast ? launch_power_fast(pa, use_split_solver(h, batch), h->stream)
                     : launch_power_generic(pa, h->stream));
    }
    PT_CUDA(mark(2));
    if (cs_pipg) {
      PT_CUDA(launch_pipg_cs(ga, handled, h->stream));
      PT_CUDA(launch_pipg_fast(ga_rest, false, h->stream));
      kernels += 1;
    } else {
      PT_CUDA(lat    ? launch_pipg_lat(ga, lat, h->stream)
              : fast ? launch_pipg_fast(ga, use_split_solver(h, batch), h->stream)
                     : launch_pipg_generic(ga, h->stream));
    }
    PT_CUDA(mark(3));
    launch_scp_update(sa, h->stream);
    PT_CUDA(mark(4));
    kernels += 3;
  }
  PT_CUDA(cudaGetLastError());
  *kernels_out = kernels;
  return PTOPT_OK;
}

int ensure_scp_graph(ptopt_cuda_handle* h, int batch, const ScpState& st) {
  const int lat = latency_ranks(h, h->rocket_shape, false, batch);
  if (h->scp_graph && h->scp_graph_batch == batch && h->scp_graph_lat == lat) return PTOPT_OK;
  if (h->scp_graph) {
    cudaGraphExecDestroy(h->scp_graph);
    h->scp_graph = nullptr;
  }
  PT_TRY(configure_solver(h, h->rocket_shape, use_fast_solver(h, h->rocket_shape, false)));
  cudaGraph_t graph = nullptr;
  PT_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  int kernels = 0;
  const int rc = enqueue_scp_loop(h, batch, st, &kernels);
  cudaError_t e = cudaStreamEndCapture(h->stream, &graph);
  if (rc != PTOPT_OK) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (e != cudaSuccess)
    return fail(PTOPT_ERR_CUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e));
  e = cudaGraphInstantiate(&h->scp_graph, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess)
    return fail(PTOPT_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
  h->scp_graph_batch = batch;
  h->scp_graph_lat = lat;
  h->scp_graph_kernels = kernels;
  return PTOPT_OK;
}

int scp_solve_common(ptopt_cuda_handle* h, int batch, const double* init_state,
                     const double* x_guess, const double* u_guess, const uint64_t* rng_seed,
                     double* x_out, double* u_out, int32_t* scp_iterations, uint8_t* converged,
                     double* final_defect_inf, double* history, int32_t* power_trips,
                     int32_t* status, int32_t* fail_index, cudaMemcpyKind in_kind,
                     cudaMemcpyKind out_kind) {
  if (!h) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null handle");
  if (batch < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  if (!init_state || !x_guess || !u_guess || !rng_seed)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "scp_solve: null input");
  DeviceGuard guard(h->device);
  if (!guard.ok) return fail(PTOPT_ERR_CUDA, "cudaSetDevice failed");
  const size_t B = (size_t)batch, n = (size_t)h->desc.nodes, mi = (size_t)h->desc.max_iters;
  ScpState st;
  PT_TRY(ensure_scp_state(h, batch, st));
  PT_TRY(ensure_scp_graph(h, batch, st));
  PT_CUDA(cudaMemcpyAsync(st.zx, x_guess, B * n * kNX * 8, in_kind, h->stream));
  PT_CUDA(cudaMemcpyAsync(st.zu, u_guess, B * n * kNU * 8, in_kind, h->stream));
  PT_CUDA(cudaMemcpyAsync(const_cast<double*>(st.init_state), init_state, B * kNXI * 8, in_kind,
                          h->stream));
  PT_CUDA(cudaMemcpyAsync(const_cast<unsigned long long*>(st.rng_seed), rng_seed, B * 8, in_kind,
                          h->stream));
  PT_CUDA(cudaGraphLaunch(h->scp_graph, h->stream));
  h->launches += h->scp_graph_kernels;
  h->stage_times_valid = true;
  auto out = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
    if (!dst) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, bytes, out_kind, h->stream);
  };
  PT_CUDA(out(x_out, st.zx, B * n * kNX * 8));
  PT_CUDA(out(u_out, st.zu, B * n * kNU * 8));
  PT_CUDA(out(scp_iterations, st.solves, B * 4));
  PT_CUDA(out(converged, st.converged, B));
  PT_CUDA(out(final_defect_inf, st.final_defect, B * 8));
  PT_CUDA(out(history, st.history, B * mi * 5 * 8));
  PT_CUDA(out(power_trips, st.power_trips, B * mi * 4));
  PT_CUDA(out(status, st.status, B * 4));
  PT_CUDA(out(fail_index, st.fail_index, B * 4));
  if (out_kind == cudaMemcpyDeviceToHost) PT_CUDA(cudaStreamSynchronize(h->stream));
  return PTOPT_OK;
}

}  // namespace

extern "C" {

int ptopt_cuda_abi_version(void) { return PTOPT_ABI_VERSION; }

const char* ptopt_cuda_last_error(void) { return g_last_error.c_str(); }

int64_t ptopt_cuda_launch_count(const ptopt_cuda_handle* h) { return h ? h->launches : 0; }

int ptopt_cuda_create(const ptopt_problem_desc* desc, const double* tau, int device, void* stream,
                      ptopt_cuda_handle** out) {
  if (!desc || !out) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  const ptopt_problem_desc& d = *desc;
  // Grid (trajectory.hpp:14-21) and ScpProblem::validate (scp.hpp:111-120)
  if (d.nodes < 2) return fail(PTOPT_ERR_INVALID_ARGUMENT, "grid needs at least two nodes");
  std::vector<double> grid((size_t)d.nodes);
  if (tau) {
    for (int k = 0; k < d.nodes; ++k) grid[k] = tau[k];
    if (grid.front() != 0.0 || grid.back() != 1.0)
      return fail(PTOPT_ERR_INVALID_ARGUMENT, "grid must start at 0 and end at 1");
    for (int k = 1; k < d.nodes; ++k)
      if (!(grid[k] > grid[k - 1]))
        return fail(PTOPT_ERR_INVALID_ARGUMENT, "grid nodes must be strictly increasing");
  } else {
    for (int k = 0; k < d.nodes; ++k) grid[k] = (double)k / (d.nodes - 1);
    grid.front() = 0.0;
    grid.back() = 1.0;
  }
  if (!(d.w_cost >= 0.0)) return fail(PTOPT_ERR_INVALID_ARGUMENT, "scp.w_cost must be >= 0");
  if (!(d.w_prox > 0.0)) return fail(PTOPT_ERR_INVALID_ARGUMENT, "scp.w_prox must be > 0");
  if (!(d.w_ep > 0.0)) return fail(PTOPT_ERR_INVALID_ARGUMENT, "scp.w_ep must be > 0");
  if (!(d.epsilon_relax > 0.0))
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "scp.epsilon_relax must be > 0");
  if (!pipg_cfg_valid(d.pipg)) return fail(PTOPT_ERR_INVALID_ARGUMENT, "invalid pipg config");
  if (!(d.s_min > 0.0) || !(d.s_min <= d.s_max))
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "scp: need 0 < s_min <= s_max");
  if (d.max_iters < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "scp.max_iters must be >= 1");
  if (d.integrator_steps < 1)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "grid.integrator_substeps must be >= 1");
  if (d.power_j_max < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "pipg.power_j_max must be >= 1");
  if (d.n_final_fix < 0 || d.n_final_fix > PTOPT_NX)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "scp: bad final boundary row count");
  for (int i = 0; i < d.n_final_fix; ++i)
    if (d.final_fix_idx[i] < 0 || d.final_fix_idx[i] >= PTOPT_NX)
      return fail(PTOPT_ERR_INVALID_ARGUMENT, "scp: final boundary index out of range");
  for (int i = 0; i < PTOPT_NX; ++i)  // assemble_subproblem, scp.hpp:155-158
    if (!(d.px[i] > 0.0))
      return fail(PTOPT_ERR_INVALID_ARGUMENT, "assemble_subproblem: nonpositive state scale");
  for (int i = 0; i < PTOPT_NU; ++i)
    if (!(d.pu[i] > 0.0))
      return fail(PTOPT_ERR_INVALID_ARGUMENT, "assemble_subproblem: nonpositive control scale");

  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count < 1)
    return fail(PTOPT_ERR_CUDA, std::string("no CUDA device: ") +
                                    (e != cudaSuccess ? cudaGetErrorString(e) : "device count 0"));
  if (device < 0 || device >= count) return fail(PTOPT_ERR_INVALID_ARGUMENT, "bad device index");
  int major = 0;
  PT_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  if (major != 10)
    return fail(PTOPT_ERR_CUDA, "device is not sm_100 (this library ships sm_100a code only)");

  ptopt_cuda_handle* h = new (std::nothrow) ptopt_cuda_handle();
  if (!h) return fail(PTOPT_ERR_ALLOC, "out of host memory");
  h->device = device;
  h->desc = d;
  h->tau = grid;
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (!make_model_const(d.vehicle, h->model)) {
    delete h;
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "inverse3: singular matrix");
  }
  fill_scp_const(d, h->scp);
  fill_rocket_shape(d, h->rocket_shape);
  DeviceGuard guard(device);
  if (!guard.ok) {
    delete h;
    return fail(PTOPT_ERR_CUDA, "cudaSetDevice failed");
  }
  if (stream) {
    h->stream = static_cast<cudaStream_t>(stream);
  } else {
    e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete h;
      return fail(PTOPT_ERR_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    }
    h->own_stream = true;
  }
  e = cudaMalloc(&h->d_tau, sizeof(double) * grid.size());
  if (e == cudaSuccess)
    e = cudaMemcpy(h->d_tau, grid.data(), sizeof(double) * grid.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    ptopt_cuda_destroy(h);
    return fail(PTOPT_ERR_CUDA, std::string("grid upload: ") + cudaGetErrorString(e));
  }
  *out = h;
  return PTOPT_OK;
}

int ptopt_cuda_destroy(ptopt_cuda_handle* h) {
  if (!h) return PTOPT_OK;
  DeviceGuard guard(h->device);
  cudaStreamSynchronize(h->stream);
  if (h->scp_graph) cudaGraphExecDestroy(h->scp_graph);
  for (cudaEvent_t e : h->stage_events) cudaEventDestroy(e);
  for (DevBuf& b : h->buf) b.release();
  if (h->d_tau) cudaFree(h->d_tau);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return PTOPT_OK;
}

int ptopt_cuda_set_solver_path(ptopt_cuda_handle* h, int path) {
  if (!h) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null handle");
  if (path < PTOPT_SOLVER_AUTO || path > PTOPT_SOLVER_FAST_DENSE)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "unknown solver path");
  if (path != h->solver_path && h->scp_graph) {  // the captured graph names the other kernels
    DeviceGuard guard(h->device);
    cudaStreamSynchronize(h->stream);
    cudaGraphExecDestroy(h->scp_graph);
    h->scp_graph = nullptr;
    h->scp_graph_batch = 0;
  }
  h->solver_path = path;
  return PTOPT_OK;
}

int ptopt_cuda_synchronize(ptopt_cuda_handle* h) {
  if (!h) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null handle");
  DeviceGuard guard(h->device);
  PT_CUDA(cudaStreamSynchronize(h->stream));
  return PTOPT_OK;
}

// ---- exact discretization -------------------------------------------------------------

int ptopt_cuda_linearize_batch_dev(ptopt_cuda_handle* h, int batch, const double* x,
                                   const double* u, double* A, double* Bm, double* Bp, double* w,
                                   double* x_end, int32_t* status, int32_t* fail_index) {
  if (!h) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null handle");
  if (batch < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  if (!x || !u || !A || !Bm || !Bp || !w || !x_end)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "linearize: null array");
  DeviceGuard guard(h->device);
  if (!guard.ok) return fail(PTOPT_ERR_CUDA, "cudaSetDevice failed");
  int* fail_key = nullptr;
  PT_TRY(device_out(h, B_FAILKEY, (size_t)batch, &fail_key));
  LinearizeArgs la;
  PT_TRY(linearize_args(h, batch, h->desc.nodes, h->desc.integrator_steps, x, u, A, Bm, Bp, w, x_end,
                        fail_key, nullptr, B_STAGES, &la));
  launch_init_fail_key(fail_key, batch, h->stream);
  h->launches += 1 + launch_linearize(la, h->stream);
  if (status || fail_index) {
    launch_decode_fail_key(fail_key, batch, status, fail_index, h->stream);
    h->launches += 1;
  }
  PT_CUDA(cudaGetLastError());
  return PTOPT_OK;
}

int ptopt_cuda_linearize_batch(ptopt_cuda_handle* h, int batch, const double* x, const double* u,
                               double* A, double* Bm, double* Bp, double* w, double* x_end,
                               int32_t* status, int32_t* fail_index) {
  if (!h) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null handle");
  if (batch < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  if (!x || !u || !A || !Bm || !Bp || !w || !x_end)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "linearize: null array");
  DeviceGuard guard(h->device);
  if (!guard.ok) return fail(PTOPT_ERR_CUDA, "cudaSetDevice failed");
  const size_t B = (size_t)batch, n = (size_t)h->desc.nodes, m = n - 1;
  const double *dx, *du;
  double *dA, *dBm, *dBp, *dw, *dxe;
  int *dst, *dfi;
  PT_TRY(upload(h, B_X, x, B * n * kNX, &dx));
  PT_TRY(upload(h, B_U, u, B * n * kNU, &du));
  PT_TRY(device_out(h, B_A, B * m * kNX * kNX, &dA));
  PT_TRY(device_out(h, B_BM, B * m * kNX * kNU, &dBm));
  PT_TRY(device_out(h, B_BP, B * m * kNX * kNU, &dBp));
  PT_TRY(device_out(h, B_W, B * m * kNX, &dw));
  PT_TRY(device_out(h, B_XEND, B * m * kNX, &dxe));
  PT_TRY(device_out(h, B_STATUS, B, &dst));
  PT_TRY(device_out(h, B_FAILIDX, B, &dfi));
  PT_TRY(ptopt_cuda_linearize_batch_dev(h, batch, dx, du, dA, dBm, dBp, dw, dxe, dst, dfi));
  PT_TRY(download(h, A, dA, B * m * kNX * kNX));
  PT_TRY(download(h, Bm, dBm, B * m * kNX * kNU));
  PT_TRY(download(h, Bp, dBp, B * m * kNX * kNU));
  PT_TRY(download(h, w, dw, B * m * kNX));
  PT_TRY(download(h, x_end, dxe, B * m * kNX));
  PT_TRY(download(h, status, dst, B));
  PT_TRY(download(h, fail_index, dfi, B));
  PT_CUDA(cudaStreamSynchronize(h->stream));
  return PTOPT_OK;
}

int ptopt_cuda_propagate_interval_batch(ptopt_cuda_handle* h, int batch, const double* x_k,
                                        const double* u_k, const double* u_k1, const double* tau_k,
                                        const double* tau_k1, int steps, double* A, double* Bm,
                                        double* Bp, double* w, double* x_end, int32_t* status) {
  if (!h) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null handle");
  if (batch < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  if (steps < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "propagate_interval: steps must be >= 1");
  if (!x_k || !u_k || !u_k1 || !tau_k || !tau_k1 || !A || !Bm || !Bp || !w || !x_end)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "propagate_interval: null array");
  for (int b = 0; b < batch; ++b)  // discretizer.hpp:29 (also rejects NaN bounds, as the reference's !(a < b) does)
    if (!(tau_k[b] < tau_k1[b])) return fail(PTOPT_ERR_INVALID_ARGUMENT, "foh_interp: empty interval");
  DeviceGuard guard(h->device);
  if (!guard.ok) return fail(PTOPT_ERR_CUDA, "cudaSetDevice failed");
  const size_t B = (size_t)batch;
  // every interval becomes a two-node instance with its own grid {tau_k, tau_k1}
  std::vector<double> hx(B * 2 * kNX, 0.0), hu(B * 2 * kNU), ht(B * 2);
  for (size_t b = 0; b < B; ++b) {
    for (int i = 0; i < kNX; ++i) hx[b * 2 * kNX + i] = x_k[b * kNX + i];
    for (int i = 0; i < kNU; ++i) {
      hu[b * 2 * kNU + i] = u_k[b * kNU + i];
      hu[b * 2 * kNU + kNU + i] = u_k1[b * kNU + i];
    }
    ht[b * 2] = tau_k[b];
    ht[b * 2 + 1] = tau_k1[b];
  }
  const double *dx, *du, *dt;
  double *dA, *dBm, *dBp, *dw, *dxe;
  int *dst, *dfi, *dkey;
  PT_TRY(upload(h, B_X, hx.data(), hx.size(), &dx));
  PT_TRY(upload(h, B_U, hu.data(), hu.size(), &du));
  PT_TRY(upload(h, B_TAU, ht.data(), ht.size(), &dt));
  PT_CUDA(cudaStreamSynchronize(h->stream));  // the staging vectors die with this call
  PT_TRY(device_out(h, B_A, B * kNX * kNX, &dA));
  PT_TRY(device_out(h, B_BM, B * kNX * kNU, &dBm));
  PT_TRY(device_out(h, B_BP, B * kNX * kNU, &dBp));
  PT_TRY(device_out(h, B_W, B * kNX, &dw));
  PT_TRY(device_out(h, B_XEND, B * kNX, &dxe));
  PT_TRY(device_out(h, B_STATUS, B, &dst));
  PT_TRY(device_out(h, B_FAILIDX, B, &dfi));
  PT_TRY(device_out(h, B_FAILKEY, B, &dkey));
  LinearizeArgs a;
  PT_TRY(linearize_args(h, batch, 2, steps, dx, du, dA, dBm, dBp, dw, dxe, dkey, nullptr, B_STAGES, &a));
  a.tau = dt;
  a.tau_stride = 2;
  launch_init_fail_key(dkey, batch, h->stream);
  h->launches += 2 + launch_linearize(a, h->stream);
  launch_decode_fail_key(dkey, batch, dst, dfi, h->stream);
  PT_CUDA(cudaGetLastError());
  PT_TRY(download(h, A, dA, B * kNX * kNX));
  PT_TRY(download(h, Bm, dBm, B * kNX * kNU));
  PT_TRY(download(h, Bp, dBp, B * kNX * kNU));
  PT_TRY(download(h, w, dw, B * kNX));
  PT_TRY(download(h, x_end, dxe, B * kNX));
  PT_TRY(download(h, status, dst, B));
  PT_CUDA(cudaStreamSynchronize(h->stream));
  return PTOPT_OK;
}

// ---- scaled subproblem assembly -------------------------------------------------------

int ptopt_cuda_subproblem_shape(const ptopt_cuda_handle* h, ptopt_subproblem_shape* shape) {
  if (!h || !shape) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null argument");
  const SubShape& s = h->rocket_shape;
  std::memset(shape, 0, sizeof *shape);
  shape->n_x = s.nx;
  shape->n_u = s.nu;
  shape->nodes = s.n;
  shape->n_init_fix = s.n_init_fix;
  shape->n_final_fix = s.n_final_fix;
  for (int i = 0; i < kNX; ++i) {
    shape->init_fix_idx[i] = s.init_fix_idx[i];
    shape->final_fix_idx[i] = s.final_fix_idx[i];
    shape->e_y[i] = s.e_y[i];
    shape->e_cost[i] = s.e_cost[i];
  }
  shape->w_cost = s.w_cost;
  shape->w_prox = s.w_prox;
  shape->w_ep = s.w_ep;
  return PTOPT_OK;
}

int ptopt_cuda_assemble_batch(ptopt_cuda_handle* h, int batch, const double* init_state,
                              const double* x, const double* u, const double* A, const double* Bm,
                              const double* Bp, const double* x_end, double* A_minus,
                              double* B_minus, double* B_plus, double* w_hat, double* eps_relax,
                              double* u_min, double* u_max, double* init_fix_val,
                              double* final_fix_val) {
  if (!h) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null handle");
  if (batch < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  if (!init_state || !x || !u || !A || !Bm || !Bp || !x_end)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "assemble: null input");
  DeviceGuard guard(h->device);
  if (!guard.ok) return fail(PTOPT_ERR_CUDA, "cudaSetDevice failed");
  const size_t B = (size_t)batch, n = (size_t)h->desc.nodes, m = n - 1;
  const size_t nf = h->desc.n_final_fix > 0 ? (size_t)h->desc.n_final_fix : 1;
  const double *dinit, *dx, *du, *dA, *dBm, *dBp, *dxe;
  double *oAm, *oBm, *oBp, *ow, *oeps, *oumin, *oumax, *oiv, *ofv;
  PT_TRY(upload(h, B_INIT, init_state, B * kNXI, &dinit));
  PT_TRY(upload(h, B_X, x, B * n * kNX, &dx));
  PT_TRY(upload(h, B_U, u, B * n * kNU, &du));
  PT_TRY(upload(h, B_A, A, B * m * kNX * kNX, &dA));
  PT_TRY(upload(h, B_BM, Bm, B * m * kNX * kNU, &dBm));
  PT_TRY(upload(h, B_BP, Bp, B * m * kNX * kNU, &dBp));
  PT_TRY(upload(h, B_XEND, x_end, B * m * kNX, &dxe));
  PT_TRY(device_out(h, B_AM, B * m * kNX * kNX, &oAm));
  PT_TRY(device_out(h, B_BMH, B * m * kNX * kNU, &oBm));
  PT_TRY(device_out(h, B_BPH, B * m * kNX * kNU, &oBp));
  PT_TRY(device_out(h, B_WH, B * m * kNX, &ow));
  PT_TRY(device_out(h, B_EPS, B * m, &oeps));
  PT_TRY(device_out(h, B_UMIN, B * n * kNU, &oumin));
  PT_TRY(device_out(h, B_UMAX, B * n * kNU, &oumax));
  PT_TRY(device_out(h, B_INITVAL, B * kNX, &oiv));
  PT_TRY(device_out(h, B_FINALVAL, B * nf, &ofv));
  launch_assemble(h->scp, batch, dinit, dx, du, dA, dBm, dBp, dxe, oAm, oBm, oBp, ow, oeps, oumin,
                  oumax, oiv, ofv, h->stream);
  h->launches += 1;
  PT_CUDA(cudaGetLastError());
  PT_TRY(download(h, A_minus, oAm, B * m * kNX * kNX));
  PT_TRY(download(h, B_minus, oBm, B * m * kNX * kNU));
  PT_TRY(download(h, B_plus, oBp, B * m * kNX * kNU));
  PT_TRY(download(h, w_hat, ow, B * m * kNX));
  PT_TRY(download(h, eps_relax, oeps, B * m));
  PT_TRY(download(h, u_min, oumin, B * n * kNU));
  PT_TRY(download(h, u_max, oumax, B * n * kNU));
  PT_TRY(download(h, init_fix_val, oiv, B * kNX));
  PT_TRY(download(h, final_fix_val, ofv, B * (size_t)h->desc.n_final_fix));
  PT_CUDA(cudaStreamSynchronize(h->stream));
  return PTOPT_OK;
}

// ---- power iteration ------------------------------------------------------------------

int ptopt_cuda_power_iteration_batch_dev(ptopt_cuda_handle* h, int batch,
                                         const ptopt_subproblem_shape* shape,
                                         const ptopt_subproblem_arrays* sp, const double* seed_x,
                                         const double* seed_u, const double* seed_vcp,
                                         const double* seed_vcn, double eps_abs, double eps_rel,
                                         double eps_buff, int j_max, double* sigma, int32_t* trips,
                                         int32_t* status) {
  if (!h) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null handle");
  if (batch < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  if (!sp || !seed_x || !seed_u || !seed_vcp || !seed_vcn || !sigma)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "power iteration: null argument");
  if (!sp->A_minus || !sp->B_minus || !sp->B_plus)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "power iteration: null operator block");
  DeviceGuard guard(h->device);
  if (!guard.ok) return fail(PTOPT_ERR_CUDA, "cudaSetDevice failed");
  PowerArgs a;
  PT_TRY(check_shape(shape, a.shape));
  a.sp = SubArrays{sp->A_minus, sp->A_plus, sp->B_minus, sp->B_plus, sp->w, sp->eps_relax,
                   sp->u_min, sp->u_max, sp->init_fix_val, sp->final_fix_val};
  a.batch = batch;
  a.seed_x = seed_x;
  a.seed_u = seed_u;
  a.seed_vcp = seed_vcp;
  a.seed_vcn = seed_vcn;
  a.eps_abs = eps_abs;
  a.eps_rel = eps_rel;
  a.eps_buff = eps_buff;
  a.j_max = j_max;
  a.sigma = sigma;
  a.trips = trips;
  a.trips_stride = 1;
  a.trips_slot = nullptr;
  a.status = status;
  a.active = nullptr;
  if (status) PT_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * (size_t)batch, h->stream));
  return dispatch_power(h, a);
}

namespace {

/// Uploads the per-instance arrays of a subproblem batch; returns device views.
int upload_sub(ptopt_cuda_handle* h, int batch, const SubShape& s,
               const ptopt_subproblem_arrays* sp, ptopt_subproblem_arrays* dev) {
  const size_t B = (size_t)batch, n = (size_t)s.n, m = n - 1, nx = (size_t)s.nx, nu = (size_t)s.nu;
  PT_TRY(upload(h, B_AM, sp->A_minus, B * m * nx * nx, &dev->A_minus));
  PT_TRY(upload(h, B_AP, sp->A_plus, B * m * nx * nx, &dev->A_plus));
  PT_TRY(upload(h, B_BMH, sp->B_minus, B * m * nx * nu, &dev->B_minus));
  PT_TRY(upload(h, B_BPH, sp->B_plus, B * m * nx * nu, &dev->B_plus));
  PT_TRY(upload(h, B_WH, sp->w, B * m * nx, &dev->w));
  PT_TRY(upload(h, B_EPS, sp->eps_relax, B * m, &dev->eps_relax));
  PT_TRY(upload(h, B_UMIN, sp->u_min, B * n * nu, &dev->u_min));
  PT_TRY(upload(h, B_UMAX, sp->u_max, B * n * nu, &dev->u_max));
  PT_TRY(upload(h, B_INITVAL, sp->init_fix_val, B * (size_t)s.n_init_fix, &dev->init_fix_val));
  PT_TRY(upload(h, B_FINALVAL, sp->final_fix_val, B * (size_t)s.n_final_fix, &dev->final_fix_val));
  return PTOPT_OK;
}

}  // namespace

int ptopt_cuda_power_iteration_batch(ptopt_cuda_handle* h, int batch,
                                     const ptopt_subproblem_shape* shape,
                                     const ptopt_subproblem_arrays* sp, const double* seed_x,
                                     const double* seed_u, const double* seed_vcp,
                                     const double* seed_vcn, double eps_abs, double eps_rel,
                                     double eps_buff, int j_max, double* sigma, int32_t* trips,
                                     int32_t* status) {
  if (!h) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null handle");
  if (batch < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  if (!sp || !seed_x || !seed_u || !seed_vcp || !seed_vcn || !sigma)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "power iteration: null argument");
  DeviceGuard guard(h->device);
  if (!guard.ok) return fail(PTOPT_ERR_CUDA, "cudaSetDevice failed");
  SubShape s;
  PT_TRY(check_shape(shape, s));
  const size_t B = (size_t)batch, n = (size_t)s.n, m = n - 1, nx = (size_t)s.nx, nu = (size_t)s.nu;
  ptopt_subproblem_arrays dev{};
  PT_TRY(upload_sub(h, batch, s, sp, &dev));
  const double *dsx, *dsu, *dsp, *dsn;
  double* dsig;
  int *dtr, *dst;
  PT_TRY(upload(h, B_SEEDX, seed_x, B * n * nx, &dsx));
  PT_TRY(upload(h, B_SEEDU, seed_u, B * n * nu, &dsu));
  PT_TRY(upload(h, B_SEEDP, seed_vcp, B * m * nx, &dsp));
  PT_TRY(upload(h, B_SEEDN, seed_vcn, B * m * nx, &dsn));
  PT_TRY(device_out(h, B_SIGMA, B, &dsig));
  PT_TRY(device_out(h, B_TRIPS, B, &dtr));
  PT_TRY(device_out(h, B_STATUS, B, &dst));
  PT_TRY(ptopt_cuda_power_iteration_batch_dev(h, batch, shape, &dev, dsx, dsu, dsp, dsn, eps_abs,
                                              eps_rel, eps_buff, j_max, dsig, dtr, dst));
  PT_TRY(download(h, sigma, dsig, B));
  PT_TRY(download(h, trips, dtr, B));
  PT_TRY(download(h, status, dst, B));
  PT_CUDA(cudaStreamSynchronize(h->stream));
  return PTOPT_OK;
}

// ---- customized PIPG ------------------------------------------------------------------

int ptopt_cuda_pipg_batch_dev(ptopt_cuda_handle* h, int batch, const ptopt_subproblem_shape* shape,
                              const ptopt_subproblem_arrays* sp, const ptopt_pipg_config* cfg,
                              const double* sigma, const ptopt_workspace_arrays* ws,
                              int32_t* iterations, uint8_t* converged, int32_t* status,
                              int32_t* fail_index) {
  if (!h) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null handle");
  if (batch < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  if (!sp || !cfg || !sigma || !ws)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "pipg: null argument");
  if (!pipg_cfg_valid(*cfg)) return fail(PTOPT_ERR_INVALID_ARGUMENT, "invalid pipg config");
  if (!sp->A_minus || !sp->B_minus || !sp->B_plus || !sp->w || !sp->eps_relax || !sp->u_min ||
      !sp->u_max)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "pipg: null subproblem array");
  if (!ws->x || !ws->u || !ws->vc_pos || !ws->vc_neg || !ws->dyn_dual || !ws->relax_dual)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "pipg: null workspace array");
  DeviceGuard guard(h->device);
  if (!guard.ok) return fail(PTOPT_ERR_CUDA, "cudaSetDevice failed");
  PipgArgs a;
  PT_TRY(check_shape(shape, a.shape));
  if ((a.shape.n_init_fix > 0 && !sp->init_fix_val) || (a.shape.n_final_fix > 0 && !sp->final_fix_val))
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "pipg: null boundary values");
  a.sp = SubArrays{sp->A_minus, sp->A_plus, sp->B_minus, sp->B_plus, sp->w, sp->eps_relax,
                   sp->u_min, sp->u_max, sp->init_fix_val, sp->final_fix_val};
  a.batch = batch;
  a.omega = cfg->omega;
  a.rho = cfg->rho;
  a.eps_abs = cfg->eps_abs;
  a.eps_rel = cfg->eps_rel;
  a.j_max = cfg->j_max;
  a.j_check = cfg->j_check;
  a.sigma = sigma;
  a.ws = WsArrays{ws->x, ws->u, ws->vc_pos, ws->vc_neg, ws->dyn_dual, ws->relax_dual};
  a.iterations = iterations;
  a.converged = converged;
  a.status = status;
  a.fail_index = fail_index;
  a.active = nullptr;
  if (status) PT_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * (size_t)batch, h->stream));
  if (fail_index)
    PT_CUDA(cudaMemsetAsync(fail_index, 0xff, sizeof(int32_t) * (size_t)batch, h->stream));
  return dispatch_pipg(h, a);
}

int ptopt_cuda_pipg_batch(ptopt_cuda_handle* h, int batch, const ptopt_subproblem_shape* shape,
                          const ptopt_subproblem_arrays* sp, const ptopt_pipg_config* cfg,
                          const double* sigma, const ptopt_workspace_arrays* ws,
                          int32_t* iterations, uint8_t* converged, int32_t* status,
                          int32_t* fail_index) {
  if (!h) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null handle");
  if (batch < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  if (!sp || !cfg || !sigma || !ws)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "pipg: null argument");
  if (!ws->x || !ws->u || !ws->vc_pos || !ws->vc_neg || !ws->dyn_dual || !ws->relax_dual)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "pipg: null workspace array");
  DeviceGuard guard(h->device);
  if (!guard.ok) return fail(PTOPT_ERR_CUDA, "cudaSetDevice failed");
  SubShape s;
  PT_TRY(check_shape(shape, s));
  const size_t B = (size_t)batch, n = (size_t)s.n, m = n - 1, nx = (size_t)s.nx, nu = (size_t)s.nu;
  ptopt_subproblem_arrays dev{};
  PT_TRY(upload_sub(h, batch, s, sp, &dev));
  const double* dsig;
  PT_TRY(upload(h, B_SIGMA, sigma, B, &dsig));
  ptopt_workspace_arrays dws{};
  const double* tmp;
  PT_TRY(upload(h, B_WSX, (const double*)ws->x, B * n * nx, &tmp)); dws.x = const_cast<double*>(tmp);
  PT_TRY(upload(h, B_WSU, (const double*)ws->u, B * n * nu, &tmp)); dws.u = const_cast<double*>(tmp);
  PT_TRY(upload(h, B_WSP, (const double*)ws->vc_pos, B * m * nx, &tmp)); dws.vc_pos = const_cast<double*>(tmp);
  PT_TRY(upload(h, B_WSN, (const double*)ws->vc_neg, B * m * nx, &tmp)); dws.vc_neg = const_cast<double*>(tmp);
  PT_TRY(upload(h, B_WSD, (const double*)ws->dyn_dual, B * m * nx, &tmp)); dws.dyn_dual = const_cast<double*>(tmp);
  PT_TRY(upload(h, B_WSR, (const double*)ws->relax_dual, B * m, &tmp)); dws.relax_dual = const_cast<double*>(tmp);
  int *dit, *dst, *dfi;
  unsigned char* dcv;
  PT_TRY(device_out(h, B_ITERS, B, &dit));
  PT_TRY(device_out(h, B_CONV, B, &dcv));
  PT_TRY(device_out(h, B_STATUS, B, &dst));
  PT_TRY(device_out(h, B_FAILIDX, B, &dfi));
  PT_TRY(ptopt_cuda_pipg_batch_dev(h, batch, shape, &dev, cfg, dsig, &dws, dit, dcv, dst, dfi));
  PT_TRY(download(h, ws->x, dws.x, B * n * nx));
  PT_TRY(download(h, ws->u, dws.u, B * n * nu));
  PT_TRY(download(h, ws->vc_pos, dws.vc_pos, B * m * nx));
  PT_TRY(download(h, ws->vc_neg, dws.vc_neg, B * m * nx));
  PT_TRY(download(h, ws->dyn_dual, dws.dyn_dual, B * m * nx));
  PT_TRY(download(h, ws->relax_dual, dws.relax_dual, B * m));
  PT_TRY(download(h, iterations, dit, B));
  PT_TRY(download(h, converged, dcv, B));
  PT_TRY(download(h, status, dst, B));
  PT_TRY(download(h, fail_index, dfi, B));
  PT_CUDA(cudaStreamSynchronize(h->stream));
  return PTOPT_OK;
}

// ---- SCP loop -------------------------------------------------------------------------

int ptopt_cuda_scp_solve_batch(ptopt_cuda_handle* h, int batch, const double* init_state,
                               const double* x_guess, const double* u_guess,
                               const uint64_t* rng_seed, double* x_out, double* u_out,
                               int32_t* scp_iterations, uint8_t* converged,
                               double* final_defect_inf, double* history, int32_t* power_trips,
                               int32_t* status, int32_t* fail_index) {
  return scp_solve_common(h, batch, init_state, x_guess, u_guess, rng_seed, x_out, u_out,
                          scp_iterations, converged, final_defect_inf, history, power_trips,
                          status, fail_index, cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost);
}

int ptopt_cuda_scp_solve_batch_dev(ptopt_cuda_handle* h, int batch, const double* init_state,
                                   const double* x_guess, const double* u_guess,
                                   const uint64_t* rng_seed, double* x_out, double* u_out,
                                   int32_t* scp_iterations, uint8_t* converged,
                                   double* final_defect_inf, double* history, int32_t* power_trips,
                                   int32_t* status, int32_t* fail_index) {
  return scp_solve_common(h, batch, init_state, x_guess, u_guess, rng_seed, x_out, u_out,
                          scp_iterations, converged, final_defect_inf, history, power_trips,
                          status, fail_index, cudaMemcpyDeviceToDevice, cudaMemcpyDeviceToDevice);
}

// ---- Monte Carlo harness ---------------------------------------------------------------

namespace {

/// slerp of rocket_problem.hpp:98-120, evaluated on the host with the C library.
void slerp_host(const double* qa, const double* qb_in, double t, double* q) {
  double qb[4] = {qb_in[0], qb_in[1], qb_in[2], qb_in[3]};
  double d = qa[0] * qb[0] + qa[1] * qb[1] + qa[2] * qb[2] + qa[3] * qb[3];
  if (d < 0.0) {
    for (double& c : qb) c = -c;
    d = -d;
  }
  if (d > 1.0 - 1e-10) {
    for (int i = 0; i < 4; ++i) q[i] = (1.0 - t) * qa[i] + t * qb[i];
  } else {
    const double ang = std::acos(d < 1.0 ? d : 1.0);
    const double sa = std::sin(ang);
    const double ca = std::sin((1.0 - t) * ang) / sa;
    const double cb = std::sin(t * ang) / sa;
    for (int i = 0; i < 4; ++i) q[i] = ca * qa[i] + cb * qb[i];
  }
  double nq = 0.0;
  for (int i = 0; i < 4; ++i) nq += q[i] * q[i];
  nq = std::sqrt(nq);
  for (int i = 0; i < 4; ++i) q[i] /= nq;
}

int generate_dev(ptopt_cuda_handle* h, int batch, int64_t first_run_id, const double* nominal,
                 const ptopt_dispersion_spec* spec, double* init_state, double* x_guess,
                 double* u_guess, uint64_t* rng_seed) {
  if (!nominal || !spec || !init_state || !x_guess || !u_guess || !rng_seed)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "generate: null argument");
  for (int i = 0; i < 3; ++i)  // DispersionSpec::validate, montecarlo.hpp:25-30
    if (!(spec->r_low[i] <= spec->r_high[i]))
      return fail(PTOPT_ERR_INVALID_ARGUMENT,
                  "montecarlo.dispersion: low > high on axis " + std::to_string(i + 1));
  const ptopt_problem_desc& d = h->desc;
  GenerateArgs a;
  a.batch = batch;
  a.nodes = d.nodes;
  a.first_run_id = first_run_id;
  for (int i = 0; i < kNXI; ++i) {
    a.nominal[i] = nominal[i];
    a.fin[i] = 0.0;
  }
  a.fin[10] = 1.0;  // RocketBoundary defaults: identity attitude, everything else zero
  for (int i = 0; i < d.n_final_fix; ++i)
    if (d.final_fix_idx[i] >= 0 && d.final_fix_idx[i] < kNXI) a.fin[d.final_fix_idx[i]] = d.final_fix_val[i];
  for (int i = 0; i < 3; ++i) {
    a.r_low[i] = spec->r_low[i];
    a.r_high[i] = spec->r_high[i];
    a.g[i] = d.vehicle.g_inertial[i];
  }
  a.seed = spec->seed;
  a.t_f_guess = d.t_f_guess;
  const double* g = d.vehicle.g_inertial;
  const double g_norm = std::sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
  const double burn = nominal[0] * std::exp(-d.vehicle.alpha_mdot * g_norm * d.t_f_guess);
  a.m_end = d.vehicle.m_dry < burn ? burn : d.vehicle.m_dry;  // std::max(m_dry, burn)
  std::vector<double> qtab((size_t)d.nodes * 4);
  for (int k = 0; k < d.nodes; ++k) slerp_host(nominal + 7, a.fin + 7, h->tau[k], &qtab[(size_t)k * 4]);
  PT_CUDA(h->buf[R_QTAB].ensure(qtab.size() * 8));
  // the table is consumed by the kernel enqueued right after this copy; wait for earlier
  // consumers of the staging buffer first
  PT_CUDA(cudaStreamSynchronize(h->stream));
  PT_CUDA(cudaMemcpyAsync(h->buf[R_QTAB].p, qtab.data(), qtab.size() * 8, cudaMemcpyHostToDevice,
                          h->stream));
  PT_CUDA(cudaStreamSynchronize(h->stream));  // qtab is a stack-lifetime host buffer
  a.tau = h->d_tau;
  a.qtab = h->buf[R_QTAB].as<double>();
  a.init_state = init_state;
  a.x_guess = x_guess;
  a.u_guess = u_guess;
  a.rng_seed = reinterpret_cast<unsigned long long*>(rng_seed);
  launch_generate(a, h->stream);
  h->launches += 1;
  PT_CUDA(cudaGetLastError());
  return PTOPT_OK;
}

int audit_dev(ptopt_cuda_handle* h, int batch, int substeps, const double* x, const double* u,
              const int* skip, double* max_pointwise_g, double* interval_y_increase,
              int32_t* status, int32_t* fail_index, double* samples = nullptr,
              const int** fail_key_out = nullptr) {
  if (substeps < 1)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "dense_violation_audit: substeps must be >= 1");
  const size_t B = (size_t)batch, m = (size_t)h->desc.nodes - 1;
  AuditArgs a;
  a.model = h->model;
  a.batch = batch;
  a.nodes = h->desc.nodes;
  a.substeps = substeps;
  a.tau = h->d_tau;
  a.x = x;
  a.u = u;
  a.skip = skip;
  a.samples = samples;
  PT_TRY(device_out(h, R_GMAX, B * m, &a.interval_g_max));
  if (interval_y_increase) {
    a.interval_y_increase = interval_y_increase;
  } else {
    PT_TRY(device_out(h, R_DY, B * m, &a.interval_y_increase));
  }
  PT_TRY(device_out(h, R_AKEY, B, &a.fail_key));
  launch_init_fail_key(a.fail_key, batch, h->stream);
  if (fail_key_out) *fail_key_out = a.fail_key;
  launch_audit(a, max_pointwise_g, status, fail_index, h->stream);
  h->launches += 3;
  PT_CUDA(cudaGetLastError());
  return PTOPT_OK;
}

}  // namespace

int ptopt_cuda_generate_batch_dev(ptopt_cuda_handle* h, int batch, int64_t first_run_id,
                                  const double* nominal_init_state,
                                  const ptopt_dispersion_spec* spec, double* init_state,
                                  double* x_guess, double* u_guess, uint64_t* rng_seed) {
  if (!h) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null handle");
  if (batch < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "montecarlo.batch_size must be >= 1");
  DeviceGuard guard(h->device);
  if (!guard.ok) return fail(PTOPT_ERR_CUDA, "cudaSetDevice failed");
  return generate_dev(h, batch, first_run_id, nominal_init_state, spec, init_state, x_guess,
                      u_guess, rng_seed);
}

int ptopt_cuda_generate_batch(ptopt_cuda_handle* h, int batch, int64_t first_run_id,
                              const double* nominal_init_state, const ptopt_dispersion_spec* spec,
                              double* init_state, double* x_guess, double* u_guess,
                              uint64_t* rng_seed) {
  if (!h) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null handle");
  if (batch < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "montecarlo.batch_size must be >= 1");
  if (!init_state || !x_guess || !u_guess || !rng_seed)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "generate: null output");
  DeviceGuard guard(h->device);
  if (!guard.ok) return fail(PTOPT_ERR_CUDA, "cudaSetDevice failed");
  const size_t B = (size_t)batch, n = (size_t)h->desc.nodes;
  double *di, *dx, *du;
  uint64_t* ds;
  PT_TRY(device_out(h, R_INIT, B * kNXI, &di));
  PT_TRY(device_out(h, R_XG, B * n * kNX, &dx));
  PT_TRY(device_out(h, R_UG, B * n * kNU, &du));
  PT_TRY(device_out(h, R_SEED, B, &ds));
  PT_TRY(generate_dev(h, batch, first_run_id, nominal_init_state, spec, di, dx, du, ds));
  PT_TRY(download(h, init_state, di, B * kNXI));
  PT_TRY(download(h, x_guess, dx, B * n * kNX));
  PT_TRY(download(h, u_guess, du, B * n * kNU));
  PT_TRY(download(h, rng_seed, ds, B));
  PT_CUDA(cudaStreamSynchronize(h->stream));
  return PTOPT_OK;
}

int ptopt_cuda_dense_audit_batch_dev(ptopt_cuda_handle* h, int batch, int substeps,
                                     const double* x, const double* u, double* max_pointwise_g,
                                     double* interval_y_increase, int32_t* status,
                                     int32_t* fail_index) {
  if (!h) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null handle");
  if (batch < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  if (!x || !u) return fail(PTOPT_ERR_INVALID_ARGUMENT, "audit: null trajectory");
  DeviceGuard guard(h->device);
  if (!guard.ok) return fail(PTOPT_ERR_CUDA, "cudaSetDevice failed");
  if (status) PT_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * (size_t)batch, h->stream));
  if (fail_index)
    PT_CUDA(cudaMemsetAsync(fail_index, 0xff, sizeof(int32_t) * (size_t)batch, h->stream));
  return audit_dev(h, batch, substeps, x, u, nullptr, max_pointwise_g, interval_y_increase, status,
                   fail_index);
}

int ptopt_cuda_dense_audit_batch(ptopt_cuda_handle* h, int batch, int substeps, const double* x,
                                 const double* u, double* max_pointwise_g,
                                 double* interval_y_increase, int32_t* status,
                                 int32_t* fail_index) {
  if (!h) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null handle");
  if (batch < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  if (!x || !u) return fail(PTOPT_ERR_INVALID_ARGUMENT, "audit: null trajectory");
  DeviceGuard guard(h->device);
  if (!guard.ok) return fail(PTOPT_ERR_CUDA, "cudaSetDevice failed");
  const size_t B = (size_t)batch, n = (size_t)h->desc.nodes, m = n - 1;
  const double *dx, *du;
  double *dg, *dy;
  int *dst, *dfi;
  PT_TRY(upload(h, B_X, x, B * n * kNX, &dx));
  PT_TRY(upload(h, B_U, u, B * n * kNU, &du));
  PT_TRY(device_out(h, R_PG, B, &dg));
  PT_TRY(device_out(h, R_DY, B * m, &dy));
  PT_TRY(device_out(h, B_STATUS, B, &dst));
  PT_TRY(device_out(h, B_FAILIDX, B, &dfi));
  PT_TRY(ptopt_cuda_dense_audit_batch_dev(h, batch, substeps, dx, du, dg, dy, dst, dfi));
  PT_TRY(download(h, max_pointwise_g, dg, B));
  PT_TRY(download(h, interval_y_increase, dy, B * m));
  PT_TRY(download(h, status, dst, B));
  PT_TRY(download(h, fail_index, dfi, B));
  PT_CUDA(cudaStreamSynchronize(h->stream));
  return PTOPT_OK;
}

int ptopt_cuda_dense_audit_samples_batch(ptopt_cuda_handle* h, int batch, int substeps, const double* x,
                                         const double* u, double* samples, double* max_pointwise_g,
                                         double* interval_y_increase, int32_t* status,
                                         int32_t* fail_index) {
  if (!h) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null handle");
  if (batch < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  if (!x || !u || !samples) return fail(PTOPT_ERR_INVALID_ARGUMENT, "audit: null array");
  if (substeps < 1)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "dense_violation_audit: substeps must be >= 1");
  DeviceGuard guard(h->device);
  if (!guard.ok) return fail(PTOPT_ERR_CUDA, "cudaSetDevice failed");
  const size_t B = (size_t)batch, n = (size_t)h->desc.nodes, m = n - 1;
  const size_t per_instance = m * (size_t)(substeps + 1) * kAuditSampleDoubles;
  const double *dx, *du;
  double *dg, *dy, *ds;
  int *dst, *dfi;
  PT_TRY(upload(h, B_X, x, B * n * kNX, &dx));
  PT_TRY(upload(h, B_U, u, B * n * kNU, &du));
  PT_TRY(device_out(h, R_PG, B, &dg));
  PT_TRY(device_out(h, R_DY, B * m, &dy));
  PT_TRY(device_out(h, R_SAMPLES, B * per_instance, &ds));
  PT_TRY(device_out(h, B_STATUS, B, &dst));
  PT_TRY(device_out(h, B_FAILIDX, B, &dfi));
  PT_CUDA(cudaMemsetAsync(ds, 0, sizeof(double) * B * per_instance, h->stream));
  PT_CUDA(cudaMemsetAsync(dst, 0, sizeof(int32_t) * B, h->stream));
  PT_CUDA(cudaMemsetAsync(dfi, 0xff, sizeof(int32_t) * B, h->stream));
  PT_TRY(audit_dev(h, batch, substeps, dx, du, nullptr, dg, dy, dst, dfi, ds));
  PT_TRY(download(h, samples, ds, B * per_instance));
  PT_TRY(download(h, max_pointwise_g, dg, B));
  PT_TRY(download(h, interval_y_increase, dy, B * m));
  PT_TRY(download(h, status, dst, B));
  PT_TRY(download(h, fail_index, dfi, B));
  PT_CUDA(cudaStreamSynchronize(h->stream));
  return PTOPT_OK;
}

int ptopt_cuda_run_batch(ptopt_cuda_handle* h, int batch, int64_t first_run_id,
                         const double* nominal_init_state, const ptopt_dispersion_spec* spec,
                         int audit_substeps, ptopt_run_record* records, double* x_out,
                         double* u_out) {
  static_assert(sizeof(ptopt_run_record) == sizeof(RunRecordDev), "record layouts must agree");
  if (!h) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null handle");
  if (batch < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "montecarlo.batch_size must be >= 1");
  if (!records) return fail(PTOPT_ERR_INVALID_ARGUMENT, "run_batch: null records");
  if (audit_substeps < 1)
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "dense_violation_audit: substeps must be >= 1");
  DeviceGuard guard(h->device);
  if (!guard.ok) return fail(PTOPT_ERR_CUDA, "cudaSetDevice failed");
  const size_t B = (size_t)batch, n = (size_t)h->desc.nodes;
  double *di, *dxg, *dug, *dxo, *duo, *dfd, *dpg;
  uint64_t* ds;
  int *dit, *dst, *dfi;
  unsigned char* dcv;
  RunRecordDev* drec;
  PT_TRY(device_out(h, R_INIT, B * kNXI, &di));
  PT_TRY(device_out(h, R_XG, B * n * kNX, &dxg));
  PT_TRY(device_out(h, R_UG, B * n * kNU, &dug));
  PT_TRY(device_out(h, R_SEED, B, &ds));
  PT_TRY(device_out(h, R_XOUT, B * n * kNX, &dxo));
  PT_TRY(device_out(h, R_UOUT, B * n * kNU, &duo));
  PT_TRY(device_out(h, R_ITERS, B, &dit));
  PT_TRY(device_out(h, R_CONV, B, &dcv));
  PT_TRY(device_out(h, R_FDEF, B, &dfd));
  PT_TRY(device_out(h, R_STATUS, B, &dst));
  PT_TRY(device_out(h, R_FAILIDX, B, &dfi));
  PT_TRY(device_out(h, R_PG, B, &dpg));
  PT_TRY(device_out(h, R_RECORDS, B, &drec));
  PT_TRY(generate_dev(h, batch, first_run_id, nominal_init_state, spec, di, dxg, dug, ds));
  h->batch_entry = true;
  const int solve_rc = scp_solve_common(h, batch, di, dxg, dug, ds, dxo, duo, dit, dcv, dfd, nullptr, nullptr,
                                        dst, dfi, cudaMemcpyDeviceToDevice, cudaMemcpyDeviceToDevice);
  h->batch_entry = false;
  PT_TRY(solve_rc);
  const int* audit_key = nullptr;
  PT_TRY(audit_dev(h, batch, audit_substeps, dxo, duo, dst, dpg, nullptr, dst, dfi, nullptr, &audit_key));
  RecordArgs ra;
  ra.audit_fail_key = audit_key;
  ra.batch = batch;
  ra.nodes = h->desc.nodes;
  ra.first_run_id = first_run_id;
  ra.init_state = di;
  ra.x = dxo;
  ra.scp_iterations = dit;
  ra.converged = dcv;
  ra.final_defect = dfd;
  ra.max_pointwise_g = dpg;
  ra.status = dst;
  ra.fail_index = dfi;
  ra.records = drec;
  launch_records(ra, h->stream);
  h->launches += 1;
  PT_CUDA(cudaGetLastError());
  PT_CUDA(cudaMemcpyAsync(records, drec, B * sizeof(ptopt_run_record), cudaMemcpyDeviceToHost,
                          h->stream));
  PT_TRY(download(h, x_out, dxo, B * n * kNX));
  PT_TRY(download(h, u_out, duo, B * n * kNU));
  PT_CUDA(cudaStreamSynchronize(h->stream));
  return PTOPT_OK;
}

int ptopt_cuda_run_batch_multi(const ptopt_problem_desc* desc, const double* tau, const int* devices,
                               int n_devices, int batch, int64_t first_run_id,
                               const double* nominal_init_state, const ptopt_dispersion_spec* spec,
                               int audit_substeps, ptopt_run_record* records, double* x_out,
                               double* u_out, double* device_ms) {
  if (!desc || !devices) return fail(PTOPT_ERR_INVALID_ARGUMENT, "run_batch_multi: null argument");
  if (n_devices < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "run_batch_multi: n_devices must be >= 1");
  if (batch < 1) return fail(PTOPT_ERR_INVALID_ARGUMENT, "montecarlo.batch_size must be >= 1");
  if (!records) return fail(PTOPT_ERR_INVALID_ARGUMENT, "run_batch: null records");
  const size_t n = (size_t)desc->nodes;
  const int G = n_devices;
  std::vector<int> rc(G, PTOPT_OK);
  std::vector<std::string> err(G);
  std::vector<double> ms(G, 0.0);
  // handles first, on this thread: a bad description or device fails the call before any work
  std::vector<ptopt_cuda_handle*> hs(G, nullptr);
  int created = PTOPT_OK;
  for (int g = 0; g < G && created == PTOPT_OK; ++g) {
    const int64_t lo = (int64_t)g * batch / G, hi = (int64_t)(g + 1) * batch / G;
    if (hi > lo) created = ptopt_cuda_create(desc, tau, devices[g], nullptr, &hs[g]);
  }
  if (created == PTOPT_OK) {
    std::vector<std::thread> pool;
    for (int g = 0; g < G; ++g) {
      if (!hs[g]) continue;
      pool.emplace_back([&, g] {
        const int64_t lo = (int64_t)g * batch / G, hi = (int64_t)(g + 1) * batch / G;
        const auto t0 = std::chrono::steady_clock::now();
        rc[g] = ptopt_cuda_run_batch(hs[g], (int)(hi - lo), first_run_id + lo, nominal_init_state, spec,
                                     audit_substeps, records + lo, x_out ? x_out + (size_t)lo * n * kNX : nullptr,
                                     u_out ? u_out + (size_t)lo * n * kNU : nullptr);
        ms[g] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (rc[g] != PTOPT_OK) err[g] = g_last_error;  // thread-local: carry it to the caller
      });
    }
    for (auto& t : pool) t.join();
  }
  const std::string create_err = created == PTOPT_OK ? std::string() : g_last_error;
  for (auto* h : hs)
    if (h) ptopt_cuda_destroy(h);
  if (created != PTOPT_OK) return fail(created, create_err);
  if (device_ms)
    for (int g = 0; g < G; ++g) device_ms[g] = ms[g];
  for (int g = 0; g < G; ++g)
    if (rc[g] != PTOPT_OK) return fail(rc[g], "device entry " + std::to_string(g) + ": " + err[g]);
  return PTOPT_OK;
}

// ---- measurement ----------------------------------------------------------------------

int ptopt_cuda_scp_stage_times(ptopt_cuda_handle* h, double* ms) {
  if (!h || !ms) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null argument");
  if (!h->stage_times_valid || h->stage_of_span.empty())
    return fail(PTOPT_ERR_INVALID_ARGUMENT, "no scp_solve_batch launch to report on");
  DeviceGuard guard(h->device);
  PT_CUDA(cudaStreamSynchronize(h->stream));
  for (int i = 0; i < PTOPT_STAGE_COUNT; ++i) ms[i] = 0.0;
  for (size_t i = 0; i < h->stage_of_span.size(); ++i) {
    float t = 0.f;
    PT_CUDA(cudaEventElapsedTime(&t, h->stage_events[i], h->stage_events[i + 1]));
    ms[h->stage_of_span[i]] += t;
  }
  float total = 0.f;
  PT_CUDA(cudaEventElapsedTime(&total, h->stage_events.front(),
                               h->stage_events[h->stage_of_span.size()]));
  ms[5] = total;
  return PTOPT_OK;
}

int ptopt_cuda_measure_fp64_peak(ptopt_cuda_handle* h, double* tflops) {
  if (!h || !tflops) return fail(PTOPT_ERR_INVALID_ARGUMENT, "null argument");
  DeviceGuard guard(h->device);
  int sms = 0;
  PT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
  double* sink = nullptr;
  PT_TRY(device_out(h, B_SIGMA, 8, &sink));
  cudaEvent_t e0, e1;
  PT_CUDA(cudaEventCreate(&e0));
  PT_CUDA(cudaEventCreate(&e1));
  const int ctas = sms * 4, threads = 256, iters = 4000;
  launch_fp64_peak(sink, iters / 10, ctas, threads, h->stream);  // warm-up
  double best = 0.0;
  for (int rep = 0; rep < 5; ++rep) {
    PT_CUDA(cudaEventRecord(e0, h->stream));
    launch_fp64_peak(sink, iters, ctas, threads, h->stream);
    PT_CUDA(cudaEventRecord(e1, h->stream));
    PT_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    PT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    const double tf = fp64_peak_flops(iters, ctas, threads) / (ms * 1e-3) * 1e-12;
    if (tf > best) best = tf;
  }
  h->launches += 6;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *tflops = best;
  return PTOPT_OK;
}

}  // extern "C"
