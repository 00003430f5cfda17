/*
 * ptopt_cuda.h — C-ABI of the B200 (sm_100a) implementation of the batched
 * 6-DoF powered-descent SCP hot path:
 *     exact discretization -> power iteration -> customized PIPG -> SCP loop.
 *
 * This header is the drop-in boundary.  The reference (/root/reference/proj)
 * is a header-only C++ template library with no FFI of its own; the entry
 * points below are what a binding for this path would bind.  Each one names
 * the reference interface it replaces (file:line relative to
 * /root/reference/).  Plain C, `extern "C"`, plain pointers and sizes, no C++
 * or torch types.
 *
 * Conventions
 *   - All arrays are dense, row-major, IEEE fp64, instance-major
 *     ([B][...] with B the batch size).  Matrices follow the reference's
 *     Mat<R,C> row-major order a[i*cols+j] (proj/include/ptopt/smallmat.hpp:60).
 *   - Every call returns a ptopt_call_status: 0 = the call ran; negative = a
 *     call-level error (bad argument, CUDA failure) described by
 *     ptopt_cuda_last_error().  A failing *instance* never fails the call:
 *     per-instance outcomes come back in status[B] / fail_index[B], mirroring
 *     mc::solve_instance which converts exceptions into RunRecord::failure
 *     (proj/include/ptopt/montecarlo.hpp:114-132).
 *   - Functions without the `_dev` suffix take HOST pointers and perform the
 *     host<->device copies themselves (pageable or pinned memory both work).
 *     `_dev` variants take DEVICE pointers valid on the handle's device and
 *     enqueue work on the handle's stream without synchronising.
 *   - The caller owns every buffer; the library allocates only its private
 *     per-handle scratch.  A handle is not thread-safe; use one handle per
 *     (device, host thread).
 *   - There is no CPU fallback: every entry point fails with PTOPT_ERR_CUDA
 *     when no sm_100 device is usable.
 */
#ifndef PTOPT_CUDA_H_
#define PTOPT_CUDA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PTOPT_ABI_VERSION 1

/* Dimensions of the rocket path (proj/include/ptopt/rocket6dof.hpp:13-15,
 * proj/include/ptopt/ctcs.hpp:25-28). */
#define PTOPT_NXI 14   /* model state  xi = (m, r, v, q, w)              */
#define PTOPT_NZETA 6  /* model control zeta = (T_body, torque_body)     */
#define PTOPT_NG 9     /* path inequalities                              */
#define PTOPT_NX 15    /* augmented state  x = (xi, y)                   */
#define PTOPT_NU 7     /* augmented control u = (zeta, s)                */
#define PTOPT_HISTORY_FIELDS 5 /* defect_inf, step_inf, penalized_cost, pipg_iterations, sigma
                                  (proj/include/ptopt/scp.hpp:219-226) */

/* Call-level status. */
typedef enum ptopt_call_status {
  PTOPT_OK = 0,
  PTOPT_ERR_INVALID_ARGUMENT = -1, /* std::invalid_argument in the reference   */
  PTOPT_ERR_CUDA = -2,             /* CUDA runtime / no usable device          */
  PTOPT_ERR_UNSUPPORTED = -3,      /* shape outside what the kernels implement */
  PTOPT_ERR_ALLOC = -4
} ptopt_call_status;

/* Per-instance status (what the reference reports by throwing). */
typedef enum ptopt_instance_status {
  PTOPT_ST_OK = 0,
  /* PropagationDiverged{interval} (proj/include/ptopt/discretizer.hpp:18-23, 89, 136);
   * fail_index = interval. */
  PTOPT_ST_PROPAGATION_DIVERGED = 1,
  /* pipg::SolverDiverged{iteration} (proj/include/ptopt/pipg.hpp:16-20, 476-478);
   * fail_index = PIPG iteration. */
  PTOPT_ST_SOLVER_DIVERGED = 2,
  /* std::domain_error "dilation factor must be positive" (proj/include/ptopt/ctcs.hpp:66, 82);
   * fail_index = interval. */
  PTOPT_ST_DILATION_NONPOSITIVE = 3,
  /* std::domain_error "nonpositive mass" (proj/include/ptopt/rocket6dof.hpp:246, 308). */
  PTOPT_ST_MASS_NONPOSITIVE = 4,
  /* std::domain_error "thrust magnitude below singular-point tolerance"
   * (proj/include/ptopt/rocket6dof.hpp:306-307). */
  PTOPT_ST_THRUST_SINGULAR = 5,
  /* std::invalid_argument "seed point must not be all zero"
   * (proj/include/ptopt/pipg.hpp:224-225). */
  PTOPT_ST_POWER_SEED_ZERO = 6
} ptopt_instance_status;

/* rocket::VehicleParams (proj/include/ptopt/rocket6dof.hpp:85-99). */
typedef struct ptopt_vehicle_params {
  double alpha_mdot;
  double g_inertial[3];
  double inertia[9];  /* row-major 3x3 */
  double r_thrust[3];
  double H_theta[8];  /* row-major 2x4 tilt selector */
  double m_dry;
  double v_max;
  double theta_max;
  double omega_max;
  double delta_max;
  double T_min;
  double T_max;
  double gamma_max;
} ptopt_vehicle_params;

/* pipg::PipgConfig (proj/include/ptopt/pipg.hpp:22-38). */
typedef struct ptopt_pipg_config {
  double omega;
  double rho;
  int32_t j_max;
  int32_t j_check;
  double eps_abs;
  double eps_rel;
  double eps_buff;
} ptopt_pipg_config;

/* Flattened ScpProblem<Rocket6DoF> minus the per-instance fields (init_state,
 * rng_seed) (proj/include/ptopt/scp.hpp:73-121; proj/include/ptopt/rocket_problem.hpp:59-94).
 * px/pu are the already power-of-two-rounded scales of ScalingPair
 * (proj/include/ptopt/scp.hpp:39-59); their reciprocals are exact. */
typedef struct ptopt_problem_desc {
  ptopt_vehicle_params vehicle;
  int32_t nodes;            /* grid.size()                       */
  int32_t integrator_steps; /* RK4 substeps per interval         */
  double s_min;
  double s_max;
  double t_f_guess;
  double w_cost;            /* ScpWeights (scp.hpp:18-22)        */
  double w_prox;
  double w_ep;
  double epsilon_relax;
  double px[PTOPT_NX];
  double pu[PTOPT_NU];
  ptopt_pipg_config pipg;
  int32_t power_j_max;
  int32_t max_iters;
  double power_eps_abs;
  double power_eps_rel;
  double tol_feas;
  double tol_step;
  int32_t n_final_fix;
  int32_t renormalize_quaternion; /* state_post_update hook present (rocket_problem.hpp:86-92) */
  int32_t final_fix_idx[PTOPT_NX];
  int32_t reserved_;
  double final_fix_val[PTOPT_NX];
  double e_cost[PTOPT_NX];
} ptopt_problem_desc;

/* Shape + shared data of a batch of pipg::Subproblem<NX,NU>
 * (proj/include/ptopt/pipg.hpp:43-96).  Dimensions are run-time values inside
 * the fixed capacities, exactly as in the reference. */
typedef struct ptopt_subproblem_shape {
  int32_t n_x;   /* 1..15 */
  int32_t n_u;   /* 1..7  */
  int32_t nodes; /* >= 2  */
  int32_t n_init_fix;
  int32_t n_final_fix;
  int32_t reserved_;
  int32_t init_fix_idx[PTOPT_NX];
  int32_t final_fix_idx[PTOPT_NX];
  double e_y[PTOPT_NX];
  double e_cost[PTOPT_NX];
  double w_cost;
  double w_prox;
  double w_ep;
} ptopt_subproblem_shape;

/* Per-instance arrays of a batch of subproblems; M = nodes-1.  All [B][...]. */
typedef struct ptopt_subproblem_arrays {
  const double* A_minus;       /* [B][M][n_x][n_x]                          */
  const double* A_plus;        /* [B][M][n_x][n_x] or NULL meaning -I       */
  const double* B_minus;       /* [B][M][n_x][n_u]                          */
  const double* B_plus;        /* [B][M][n_x][n_u]                          */
  const double* w;             /* [B][M][n_x]                               */
  const double* eps_relax;     /* [B][M]                                    */
  const double* u_min;         /* [B][nodes][n_u]  (+-inf allowed)          */
  const double* u_max;         /* [B][nodes][n_u]                           */
  const double* init_fix_val;  /* [B][n_init_fix]                           */
  const double* final_fix_val; /* [B][n_final_fix]                          */
} ptopt_subproblem_arrays;

/* pipg::Workspace warm start / solution groups (proj/include/ptopt/pipg.hpp:100-141). */
typedef struct ptopt_workspace_arrays {
  double* x;          /* [B][nodes][n_x] */
  double* u;          /* [B][nodes][n_u] */
  double* vc_pos;     /* [B][M][n_x]     */
  double* vc_neg;     /* [B][M][n_x]     */
  double* dyn_dual;   /* [B][M][n_x]     */
  double* relax_dual; /* [B][M]          */
} ptopt_workspace_arrays;

typedef struct ptopt_cuda_handle ptopt_cuda_handle;

/* ---- library ---------------------------------------------------------- */

int ptopt_cuda_abi_version(void);
/* Thread-local description of the last call-level error on this thread. */
const char* ptopt_cuda_last_error(void);
/* Number of kernel launches issued through `h` since creation (graph nodes
 * count once per graph launch). */
int64_t ptopt_cuda_launch_count(const ptopt_cuda_handle* h);

/* Creates a solver handle for one problem description on one device.
 * Replaces constructing ScpProblem<Rocket6DoF> + Grid
 * (proj/include/ptopt/scp.hpp:73-121, proj/include/ptopt/trajectory.hpp:11-34).
 * `tau` = grid nodes [nodes] (strictly increasing, tau[0]=0, tau[nodes-1]=1),
 * or NULL for Grid::uniform(nodes).  `stream` = a cudaStream_t to run on, or
 * NULL for a private non-blocking stream owned by the handle. */
int ptopt_cuda_create(const ptopt_problem_desc* desc, const double* tau, int device, void* stream,
                      ptopt_cuda_handle** out);
int ptopt_cuda_destroy(ptopt_cuda_handle* h);
/* Kernel family used for power iteration and PIPG.  No reference counterpart.
 *   AUTO       for the rocket-shaped subproblem (n_x = 15, n_u = 7, A_plus = -I, e_y = last
 *              state): the latency-mode kernels whenever the whole batch fits the chip in one
 *              wave (batch x cluster size <= SM count: one CTA per instance up to 16 nodes,
 *              else up to 18 / 37 / 74 instances with 8 / 4 / 2 CTAs per instance), else the
 *              throughput kernels; the shape-generic kernels for every other shape.
 *   GENERIC    forces the shape-generic kernels (the parity tests run every family on the same
 *              inputs).
 *   FAST_SPLIT throughput kernels with every instance of 4..50 nodes shared by a 2-CTA
 *              cluster of 128-thread CTAs, two CTAs (halves of different instances) resident per
 *              SM; other node counts run as under FAST_THROUGHPUT.  Experimental: slower than
 *              FAST_THROUGHPUT on B200.
 *   FAST_LATENCY    latency mode whatever the batch size: one instance spread over a cluster of
 *              up to eight CTAs, sixteen threads per node (a short dependent instruction
 *              stream per thread); up to 128 nodes.  Lowest single-solve latency, lower
 *              throughput per SM.
 *   FAST_THROUGHPUT register-resident throughput kernels whatever the batch size.  Up to 102 nodes
 *              the column-sparse kernels run first (four role-uniform warps per 32 nodes, the
 *              structural zeros of the rocket model's state-transition blocks skipped at compile
 *              time; one CTA per instance up to 61 nodes; above, the power iteration over a 2-CTA
 *              cluster and PIPG on the dense cluster kernel); they verify the
 *              zero pattern of every instance while loading it and leave instances without it to
 *              the dense kernels (FAST_DENSE), which run right behind.
 *   FAST_DENSE the dense register-resident kernels alone: five threads per node, one CTA per
 *              instance up to 51 nodes, a 2-CTA cluster up to 102; any operator values. */
#define PTOPT_SOLVER_AUTO 0
#define PTOPT_SOLVER_GENERIC 1
#define PTOPT_SOLVER_FAST_SPLIT 2
#define PTOPT_SOLVER_FAST_LATENCY 3
#define PTOPT_SOLVER_FAST_THROUGHPUT 4
#define PTOPT_SOLVER_FAST_DENSE 5
int ptopt_cuda_set_solver_path(ptopt_cuda_handle* h, int path);
/* Blocks until all work enqueued on the handle's stream has finished. */
int ptopt_cuda_synchronize(ptopt_cuda_handle* h);

/* ---- exact discretization --------------------------------------------- */

/* Batched linearize_all (proj/include/ptopt/discretizer.hpp:191-232), i.e.
 * propagate_interval (discretizer.hpp:82-149) over every interval of every
 * instance.  x [B][nodes][15], u [B][nodes][7] ->
 * A [B][M][15][15], Bm/Bp [B][M][15][7], w/x_end [B][M][15].
 * status[b] != 0 marks the FIRST failing interval of instance b (the
 * reference throws from the lowest interval index) and fail_index[b] holds it;
 * blocks of a failed instance are unspecified. */
int ptopt_cuda_linearize_batch(ptopt_cuda_handle* h, int batch, const double* x, const double* u,
                               double* A, double* Bm, double* Bp, double* w, double* x_end,
                               int32_t* status, int32_t* fail_index);
int ptopt_cuda_linearize_batch_dev(ptopt_cuda_handle* h, int batch, const double* x,
                                   const double* u, double* A, double* Bm, double* Bp, double* w,
                                   double* x_end, int32_t* status, int32_t* fail_index);

/* Batched propagate_interval (proj/include/ptopt/discretizer.hpp:82-149): independent
 * intervals, each with its own end points.  x_k [B][15], u_k/u_k1 [B][7],
 * tau_k/tau_k1 [B] -> A [B][15][15], Bm/Bp [B][15][7], w/x_end [B][15].
 * status[b] != 0 is what the reference throws for interval b (the caller knows
 * the interval index it passed as `interval_index`). */
int ptopt_cuda_propagate_interval_batch(ptopt_cuda_handle* h, int batch, const double* x_k,
                                        const double* u_k, const double* u_k1, const double* tau_k,
                                        const double* tau_k1, int steps, double* A, double* Bm,
                                        double* Bp, double* w, double* x_end, int32_t* status);

/* ---- scaled subproblem assembly ---------------------------------------- */

/* Batched assemble_subproblem (proj/include/ptopt/scp.hpp:139-217) for the
 * handle's problem: blocks + iterate -> scaled Subproblem arrays.
 * init_state [B][14]; outputs: A_minus [B][M][15][15] (A_plus is -I and not
 * materialised), B_minus/B_plus [B][M][15][7], w_hat [B][M][15],
 * eps_relax [B][M], u_min/u_max [B][nodes][7], init_fix_val [B][15],
 * final_fix_val [B][n_final_fix]. */
int ptopt_cuda_assemble_batch(ptopt_cuda_handle* h, int batch, const double* init_state,
                              const double* x, const double* u, const double* A, const double* Bm,
                              const double* Bp, const double* x_end, double* A_minus,
                              double* B_minus, double* B_plus, double* w_hat, double* eps_relax,
                              double* u_min, double* u_max, double* init_fix_val,
                              double* final_fix_val);
/* Fills `shape` with the subproblem shape assemble_subproblem produces for the
 * handle's problem (n_x=15, n_u=7, fix index lists, e_y, scaled e_cost, weights). */
int ptopt_cuda_subproblem_shape(const ptopt_cuda_handle* h, ptopt_subproblem_shape* shape);

/* ---- power iteration ---------------------------------------------------- */

/* Batched pipg::power_iteration_custom (proj/include/ptopt/pipg.hpp:206-292).
 * Seeds: seed_x [B][nodes][n_x], seed_u [B][nodes][n_u], seed_vcp/seed_vcn
 * [B][M][n_x].  sigma[b] = (1+eps_buff) * estimate; trips[b] = iterations run
 * (may be NULL).  status[b] = PTOPT_ST_POWER_SEED_ZERO for an all-zero seed.
 * Known deviation: the kernels normalise with a reciprocal square root and add
 * the norm as a tree, so the stopping test |sigma* - sigma| <= eps (1e-12 by
 * default) can be met a few trips earlier or later than on the CPU: sigma agrees
 * to 1e-9 relative, trips to max(3, 2 %) (tests/test_gpu_parity.py:
 * test_power_iteration_random_subproblems); inside the SCP loop to max(5, 5 %). */
int ptopt_cuda_power_iteration_batch(ptopt_cuda_handle* h, int batch,
                                     const ptopt_subproblem_shape* shape,
                                     const ptopt_subproblem_arrays* sp, const double* seed_x,
                                     const double* seed_u, const double* seed_vcp,
                                     const double* seed_vcn, double eps_abs, double eps_rel,
                                     double eps_buff, int j_max, double* sigma, int32_t* trips,
                                     int32_t* status);
int ptopt_cuda_power_iteration_batch_dev(ptopt_cuda_handle* h, int batch,
                                         const ptopt_subproblem_shape* shape,
                                         const ptopt_subproblem_arrays* sp, const double* seed_x,
                                         const double* seed_u, const double* seed_vcp,
                                         const double* seed_vcn, double eps_abs, double eps_rel,
                                         double eps_buff, int j_max, double* sigma, int32_t* trips,
                                         int32_t* status);

/* ---- customized PIPG ---------------------------------------------------- */

/* Batched pipg::pipg_custom (proj/include/ptopt/pipg.hpp:350-497).  `ws` holds
 * the warm start on entry and the solution (the *_cur groups, pipg.hpp:490-495)
 * on return; sigma [B] is Workspace::sigma.  iterations [B], converged [B]
 * mirror PipgResult (pipg.hpp:342-345).  status/fail_index report
 * SolverDiverged{j}. */
int ptopt_cuda_pipg_batch(ptopt_cuda_handle* h, int batch, const ptopt_subproblem_shape* shape,
                          const ptopt_subproblem_arrays* sp, const ptopt_pipg_config* cfg,
                          const double* sigma, const ptopt_workspace_arrays* ws,
                          int32_t* iterations, uint8_t* converged, int32_t* status,
                          int32_t* fail_index);
int ptopt_cuda_pipg_batch_dev(ptopt_cuda_handle* h, int batch, const ptopt_subproblem_shape* shape,
                              const ptopt_subproblem_arrays* sp, const ptopt_pipg_config* cfg,
                              const double* sigma, const ptopt_workspace_arrays* ws,
                              int32_t* iterations, uint8_t* converged, int32_t* status,
                              int32_t* fail_index);

/* ---- SCP loop ------------------------------------------------------------ */

/* Batched scp_solve (proj/include/ptopt/scp.hpp:256-364) for the handle's
 * problem, the whole loop on the device under one CUDA graph.
 * Inputs: init_state [B][14] (ScpProblem::init_state), x_guess [B][nodes][15],
 * u_guess [B][nodes][7], rng_seed [B] (ScpProblem::rng_seed).
 * Outputs: x_out/u_out (ScpResult::iterate), scp_iterations [B], converged [B],
 * final_defect_inf [B], history [B][max_iters][5] (rows past scp_iterations are
 * zero; pipg_iterations stored as a double), power_trips [B][max_iters] (may be
 * NULL; extra diagnostic the reference does not expose; see the deviation note
 * at ptopt_cuda_power_iteration_batch), status/fail_index [B]. */
int ptopt_cuda_scp_solve_batch(ptopt_cuda_handle* h, int batch, const double* init_state,
                               const double* x_guess, const double* u_guess,
                               const uint64_t* rng_seed, double* x_out, double* u_out,
                               int32_t* scp_iterations, uint8_t* converged,
                               double* final_defect_inf, double* history, int32_t* power_trips,
                               int32_t* status, int32_t* fail_index);
int ptopt_cuda_scp_solve_batch_dev(ptopt_cuda_handle* h, int batch, const double* init_state,
                                   const double* x_guess, const double* u_guess,
                                   const uint64_t* rng_seed, double* x_out, double* u_out,
                                   int32_t* scp_iterations, uint8_t* converged,
                                   double* final_defect_inf, double* history, int32_t* power_trips,
                                   int32_t* status, int32_t* fail_index);

/* ---- Monte Carlo harness around the solve --------------------------------- */

/* mc::DispersionSpec (proj/include/ptopt/montecarlo.hpp:20-31). */
typedef struct ptopt_dispersion_spec {
  double r_low[3];
  double r_high[3];
  uint64_t seed;
} ptopt_dispersion_spec;

/* mc::RunRecord (proj/include/ptopt/montecarlo.hpp:67-78).  `failure` becomes
 * status/fail_index (ptopt_instance_status); a failed record keeps the
 * reference's defaults (converged 0, zeros).  wall_time has no per-instance
 * meaning on the device and is not reported. */
typedef struct ptopt_run_record {
  int32_t run_id;
  int32_t converged;
  int32_t scp_iterations;
  int32_t status;
  int32_t fail_index;
  int32_t reserved_;
  double initial_position[3];
  double propellant_used;
  double final_defect_inf;
  double max_pointwise_g;
  double max_node_y_increase;
} ptopt_run_record;

/* Instance generation exactly as mc::solve_instance does it for run ids
 * first_run_id .. first_run_id+batch-1: mc::disperse (montecarlo.hpp:55-65),
 * mc::run_seed (:51-53) and initial_guess (proj/include/ptopt/rocket_problem.hpp:127-163)
 * about the handle's problem.  nominal_init_state [14] is RocketBoundary::initial; the
 * terminal targets are the handle's final_fix values (unpinned slots default as
 * RocketBoundary does).  Outputs: init_state [B][14], x_guess [B][nodes][15],
 * u_guess [B][nodes][7], rng_seed [B].  Integer draws and every floating-point
 * operation are bit-exact with the reference. */
int ptopt_cuda_generate_batch(ptopt_cuda_handle* h, int batch, int64_t first_run_id,
                              const double* nominal_init_state, const ptopt_dispersion_spec* spec,
                              double* init_state, double* x_guess, double* u_guess,
                              uint64_t* rng_seed);
int ptopt_cuda_generate_batch_dev(ptopt_cuda_handle* h, int batch, int64_t first_run_id,
                                  const double* nominal_init_state,
                                  const ptopt_dispersion_spec* spec, double* init_state,
                                  double* x_guess, double* u_guess, uint64_t* rng_seed);

/* Batched dense_violation_audit (proj/include/ptopt/discretizer.hpp:249-285) with
 * propagate_state (:153-187): x [B][nodes][15], u [B][nodes][7] ->
 * max_pointwise_g [B], interval_y_increase [B][M] (total_y_increase is their
 * in-order sum).  status/fail_index report a domain error inside the propagation
 * (first failing interval). */
int ptopt_cuda_dense_audit_batch(ptopt_cuda_handle* h, int batch, int substeps, const double* x,
                                 const double* u, double* max_pointwise_g,
                                 double* interval_y_increase, int32_t* status,
                                 int32_t* fail_index);
int ptopt_cuda_dense_audit_batch_dev(ptopt_cuda_handle* h, int batch, int substeps,
                                     const double* x, const double* u, double* max_pointwise_g,
                                     double* interval_y_increase, int32_t* status,
                                     int32_t* fail_index);

/* The same audit with its sample sink (the `samples` argument of dense_violation_audit,
 * discretizer.hpp:253, 262-276; AuditSample :236-240): samples
 * [B][M][substeps+1][PTOPT_AUDIT_SAMPLE_DOUBLES] = {interval, tau, g[9], g_max}, in the
 * reference's order (interval by interval, the node sample first, then one per substep).
 * Samples of an instance whose propagation fails are unspecified from the failing interval on. */
#define PTOPT_AUDIT_SAMPLE_DOUBLES 12
int ptopt_cuda_dense_audit_samples_batch(ptopt_cuda_handle* h, int batch, int substeps, const double* x,
                                         const double* u, double* samples, double* max_pointwise_g,
                                         double* interval_y_increase, int32_t* status,
                                         int32_t* fail_index);

/* mc::run_batch (proj/include/ptopt/montecarlo.hpp:140-175) for run ids
 * first_run_id .. first_run_id+batch-1, everything on the device: generation ->
 * scp_solve -> audit -> records.  Only the records (and, when x_out/u_out are
 * non-NULL, the final trajectories [B][nodes][15] / [B][nodes][7]) cross to the
 * host.  The reference's `workers` argument has no counterpart: every instance
 * is its own CTA.  Sharding a batch over GPUs = one handle per device with
 * disjoint run-id ranges (records are pure functions of the run id). */
int ptopt_cuda_run_batch(ptopt_cuda_handle* h, int batch, int64_t first_run_id,
                         const double* nominal_init_state, const ptopt_dispersion_spec* spec,
                         int audit_substeps, ptopt_run_record* records, double* x_out,
                         double* u_out);

/* mc::run_batch over several devices of one node.  The reference's batch entry
 * owns its parallelism -- a pool of `workers` threads pulling run ids, results
 * written into slots indexed by run id so the output does not depend on the
 * worker count (proj/include/ptopt/montecarlo.hpp:153-171).  Here a worker is
 * one device: the call creates one handle and one host thread per entry of
 * `devices` (an ordinal may be listed more than once: several handles then share
 * that GPU), gives entry g the contiguous run ids
 *   first_run_id + [g*batch/G .. (g+1)*batch/G)      (sizes differ by at most one)
 * and every thread writes its records (and trajectories, when x_out/u_out are
 * non-NULL) straight into the caller's arrays at the slots of its run ids, so the
 * result is bit-identical to one ptopt_cuda_run_batch over the whole range.  No
 * data-path collective: instances are independent (BASELINE north_star).
 * `device_ms` (NULL or [n_devices]) receives each worker's wall time of its
 * ptopt_cuda_run_batch call in milliseconds; the slowest one is the batch time.
 * An entry whose range is empty (batch < n_devices) does nothing.  The first
 * failing worker's error becomes the call's error. */
int ptopt_cuda_run_batch_multi(const ptopt_problem_desc* desc, const double* tau, const int* devices,
                               int n_devices, int batch, int64_t first_run_id,
                               const double* nominal_init_state, const ptopt_dispersion_spec* spec,
                               int audit_substeps, ptopt_run_record* records, double* x_out,
                               double* u_out, double* device_ms);

/* ---- measurement --------------------------------------------------------- */

#define PTOPT_STAGE_COUNT 6
/* Device time in milliseconds of the most recent scp_solve_batch[_dev] graph launch on this
 * handle, split by stage and measured by event nodes inside the graph:
 * [0] discretization (linearize_all), [1] defect test + assemble_subproblem + seed,
 * [2] power iteration, [3] PIPG, [4] iterate update, [5] whole graph.
 * Blocks until the launch has finished.  (No reference counterpart: the reference only keeps
 * wall-clock times per instance, proj/include/ptopt/montecarlo.hpp:113, 133.) */
int ptopt_cuda_scp_stage_times(ptopt_cuda_handle* h, double* ms);

/* Measures the FP64 FMA throughput of the device (dependent-chain-free DFMA loop filling every
 * SM) in TFLOP/s: the roofline denominator for this path, which MEASURED_PEAKS.json lacks. */
int ptopt_cuda_measure_fp64_peak(ptopt_cuda_handle* h, double* tflops);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* PTOPT_CUDA_H_ */
