"""Single-solve latency by stage: one N-node instance through ptopt_cuda_scp_solve_batch."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2404_18034_b200 import scenario
from paper_2404_18034_b200.binding import Solver

nodes = int(sys.argv[1]) if len(sys.argv) > 1 else 50
for path in sys.argv[2:] or ["auto"]:
    sc = scenario.default_scenario(nodes)
    b = scenario.make_batch(sc, [0])
    with Solver(sc.problem_desc()) as s:
        s.set_solver_path(path)
        s.scp_solve(b["init_state"], b["x_guess"], b["u_guess"], b["rng_seed"])
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            out = s.scp_solve(b["init_state"], b["x_guess"], b["u_guess"], b["rng_seed"])
            ts.append(1e3 * (time.perf_counter() - t0))
        print(path, "nodes", nodes, "latency ms", [round(t, 2) for t in ts], "stages", s.scp_stage_times(),
              "trips", int(out["power_trips"][0].sum()))
