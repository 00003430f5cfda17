"""Throughput of full SCP solves at N=100 (BASELINE config 5 shape: 296 instances, 2-CTA cluster per instance)."""
import sys, time
sys.path.insert(0, ".")
from paper_2404_18034_b200 import scenario
from paper_2404_18034_b200.binding import Solver
n, B = 100, 296
sc = scenario.default_scenario(n)
batch = scenario.make_batch(sc, range(B))
with Solver(sc.problem_desc()) as s:
    s.scp_solve(batch["init_state"][:4], batch["x_guess"][:4], batch["u_guess"][:4], batch["rng_seed"][:4])
    res = s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"], batch["rng_seed"])
    st = s.scp_stage_times()
print("n100 solves/s", B / (st["graph_total"] * 1e-3), st)
