"""Small workload for compute-sanitizer: every kernel of the path once (reduced budgets).
usage: python tools/sanitizer_workload.py <nodes> [auto|generic|split]"""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2404_18034_b200 import scenario
from paper_2404_18034_b200.binding import Solver
sc = scenario.default_scenario(int(sys.argv[1]))
path = sys.argv[2] if len(sys.argv) > 2 else "auto"
sc.max_iters, sc.pipg_j_max, sc.power_j_max = 2, 60, 40
d = sc.problem_desc()
batch = scenario.make_batch(sc, range(3))
with Solver(d) as s:
    s.set_solver_path(path)
    out = s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"], batch["rng_seed"])
    rec = s.run_batch(3, 0, sc.initial_state, sc.dispersion.r_low, sc.dispersion.r_high, sc.dispersion.seed, audit_substeps=8)
print("status", out["status"], rec["status"], float(out["x"].sum()))
