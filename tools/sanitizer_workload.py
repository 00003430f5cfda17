import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from paper_2404_18034_b200 import scenario
from paper_2404_18034_b200.binding import Solver
sc = scenario.default_scenario(int(sys.argv[1]))
sc.max_iters, sc.pipg_j_max, sc.power_j_max = 2, 60, 40
d = sc.problem_desc()
batch = scenario.make_batch(sc, range(3))
with Solver(d) as s:
    out = s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"], batch["rng_seed"])
    rec = s.run_batch(3, 0, sc.initial_state, sc.dispersion.r_low, sc.dispersion.r_high, sc.dispersion.seed, audit_substeps=8)
print("status", out["status"], rec["status"], float(out["x"].sum()))
