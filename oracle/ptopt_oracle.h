/*
 * ptopt_oracle.h — TEST INFRASTRUCTURE.  CPU restatement (plain C, flat arrays)
 * of the reference algorithm for the batched 6-DoF SCP hot path.  It is the
 * parity checker for the CUDA library and the "port" CPU baseline; the product
 * (paper_2404_18034_b200/, include/) never includes, links or calls it.
 *
 * Parity pin: every function is checked bit-for-bit (both built with
 * -ffp-contract=off) against the unmodified reference compiled in place
 * (oracle/_ref, see oracle/Makefile) by tests/test_oracle_vs_ref.py, and against
 * the committed vectors in tests/golden/ that the reference generated.
 *
 * Return convention (same as oracle/ref_shim.cpp): 0 = ok, >0 = a
 * ptopt_instance_status code (fail_index set where the reference exception
 * carries one), -1 = std::invalid_argument in the reference.
 */
#ifndef PTOPT_ORACLE_H_
#define PTOPT_ORACLE_H_

#include <stdint.h>

#include "ptopt_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

#define PTOR_MAX_X 16
#define PTOR_MAX_U 8
#define PTOR_MAX_G 16

/* The model concept of proj/include/ptopt/ctcs.hpp:10-17 as a table of
 * callbacks.  Jacobians are row-major with the model's own dims. */
typedef struct ptor_model {
  int state_dim, control_dim, ineq_dim, eq_dim;
  const void* ctx;
  int (*dynamics)(const void* ctx, const double* xi, const double* zeta, double* F);
  void (*path_ineq)(const void* ctx, const double* xi, const double* zeta, double* g);
  void (*path_eq)(const void* ctx, const double* xi, const double* zeta, double* h);
  int (*dynamics_jacobians)(const void* ctx, const double* xi, const double* zeta, double* dF_dx,
                            double* dF_du);
  int (*path_ineq_jacobians)(const void* ctx, const double* xi, const double* zeta, double* dg_dx,
                             double* dg_du);
  void (*path_eq_jacobians)(const void* ctx, const double* xi, const double* zeta, double* dh_dx,
                            double* dh_du);
} ptor_model;

/* Rocket6DoF with its cached inertia inverse (rocket6dof.hpp:231-241). */
typedef struct ptor_rocket {
  ptopt_vehicle_params p;
  double inertia_inv[9];
} ptor_rocket;

int ptor_rocket_init(ptor_rocket* r, const ptopt_vehicle_params* p);
ptor_model ptor_rocket_model(const ptor_rocket* r);

/* model layer */
int ptor_model_eval(const ptopt_vehicle_params* vp, const double* xi, const double* zeta,
                    double* F, double* g, double* dF_dxi, double* dF_dzeta, double* dg_dxi,
                    double* dg_dzeta);
int ptor_aug_eval(const ptopt_vehicle_params* vp, const double* x, const double* u, double* f,
                  double* A, double* B);
int ptor_aug_eval_test_model(int model_id, const double* params, const double* x, const double* u,
                             double* f, double* A, double* B);

/* discretizer */
int ptor_foh_interp(int n, const double* u_k, const double* u_k1, double tau, double tau_k,
                    double tau_k1, double* u);
int ptor_propagate_interval(const ptopt_vehicle_params* vp, const double* xk, const double* uk,
                            const double* uk1, double tau_k, double tau_k1, int steps,
                            int interval_index, double* A, double* Bm, double* Bp, double* w,
                            double* x_end, int* fail_index);
int ptor_propagate_test_model(int model_id, const double* params, const double* xk,
                              const double* uk, const double* uk1, double tau_k, double tau_k1,
                              int steps, int interval_index, double* A, double* Bm, double* Bp,
                              double* w, double* x_end, int* fail_index);
int ptor_linearize_all(const ptopt_problem_desc* d, const double* tau, const double* x,
                       const double* u, int workers, double* A, double* Bm, double* Bp, double* w,
                       double* x_end, int* fail_index);
int ptor_dense_audit(const ptopt_problem_desc* d, const double* tau, const double* x,
                     const double* u, int substeps, double* max_pointwise_g,
                     double* total_y_increase, double* interval_y_increase);
/* The same with the per-sample records of dense_violation_audit (discretizer.hpp:236-240,
 * 262-276): samples [nodes-1][substeps+1][PTOR_SAMPLE_DOUBLES] = {interval, tau, g[9], g_max}. */
#define PTOR_SAMPLE_DOUBLES 12
int ptor_dense_audit_samples(const ptopt_problem_desc* d, const double* tau, const double* x,
                             const double* u, int substeps, double* max_pointwise_g,
                             double* total_y_increase, double* interval_y_increase, double* samples);

/* SCP glue */
int ptor_assemble(const ptopt_problem_desc* d, const double* tau, const double* init_state,
                  const double* x, const double* u, const double* A, const double* Bm,
                  const double* Bp, const double* x_end, double* A_minus, double* A_plus,
                  double* B_minus, double* B_plus, double* w_hat, double* eps_relax, double* u_min,
                  double* u_max, double* init_fix_val, double* final_fix_val, double* e_cost_hat);
void ptor_scp_seed(uint64_t rng_seed, int nodes, double* seed_x, double* seed_u);
int ptor_scp_solve(const ptopt_problem_desc* d, const double* tau, const double* init_state,
                   const double* x_guess, const double* u_guess, uint64_t rng_seed, double* x_out,
                   double* u_out, int* scp_iterations, int* converged, double* final_defect_inf,
                   double* history, int* fail_index);
/* Same, also reporting the power-iteration trip count of every SCP iteration. */
int ptor_scp_solve_ex(const ptopt_problem_desc* d, const double* tau, const double* init_state,
                      const double* x_guess, const double* u_guess, uint64_t rng_seed,
                      double* x_out, double* u_out, int* scp_iterations, int* converged,
                      double* final_defect_inf, double* history, int* power_trips,
                      int* fail_index);

/* PIPG */
int ptor_power_iteration(const ptopt_subproblem_shape* shape, const ptopt_subproblem_arrays* a,
                         const double* seed_x, const double* seed_u, const double* seed_vcp,
                         const double* seed_vcn, double eps_abs, double eps_rel, double eps_buff,
                         int j_max, double* sigma);
int ptor_power_iteration_ex(const ptopt_subproblem_shape* shape, const ptopt_subproblem_arrays* a,
                            const double* seed_x, const double* seed_u, const double* seed_vcp,
                            const double* seed_vcn, double eps_abs, double eps_rel,
                            double eps_buff, int j_max, double* sigma, int* trips);
int ptor_pipg(const ptopt_subproblem_shape* shape, const ptopt_subproblem_arrays* a,
              const ptopt_pipg_config* cfg, double sigma, const ptopt_workspace_arrays* w,
              int* iterations, int* converged, int* fail_index);
double ptor_step_sizes(double lambda, double omega, double sigma, double* beta);

/* instance generation */
uint64_t ptor_run_seed(uint64_t batch_seed, int run_id);
void ptor_disperse(const double* r_low, const double* r_high, uint64_t seed, int run_id,
                   double* r_out);
int ptor_initial_guess(const ptopt_problem_desc* d, const double* tau, const double* init_state,
                       double* x, double* u);
double ptor_pow2_near(double v);

/* batch harness on `workers` pthreads; returns wall seconds (instance generation excluded
 * exactly as mc::run_batch does not exclude it: generation is inside solve_instance). */
double ptor_run_batch(const ptopt_problem_desc* d, const double* tau,
                      const double* nominal_init_state, const double* r_low, const double* r_high,
                      uint64_t seed, int batch_size, int workers, int audit_substeps,
                      double* records, double* x_out, double* u_out);

int ptor_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PTOPT_ORACLE_H_ */
