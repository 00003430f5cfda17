"""Workload for ncu captures: one wave (148 instances, N nodes) through every kernel of the path
with a reduced iteration budget.  usage: python tools/ncu_workload.py [nodes] [batch] [path]"""
import sys
sys.path.insert(0, ".")
from paper_2404_18034_b200 import scenario
from paper_2404_18034_b200.binding import Solver

nodes = int(sys.argv[1]) if len(sys.argv) > 1 else 50
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 148
path = sys.argv[3] if len(sys.argv) > 3 else "auto"
sc = scenario.default_scenario(nodes)
sc.max_iters, sc.pipg_j_max, sc.power_j_max = 2, 500, 400
with Solver(sc.problem_desc()) as s:
    s.set_solver_path(path)
    rec = s.run_batch(batch, 0, sc.initial_state, sc.dispersion.r_low, sc.dispersion.r_high,
                      sc.dispersion.seed, audit_substeps=64)
print("records", len(rec), "failed", int((rec["status"] != 0).sum()))
