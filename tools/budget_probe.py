"""One instance through scp_solve with chosen budgets: python tools/budget_probe.py nodes path max_iters pipg_j_max power_j_max"""
import sys, time
sys.path.insert(0, ".")
from paper_2404_18034_b200 import scenario
from paper_2404_18034_b200.binding import Solver
nodes, path, mi, pj, wj = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
sc = scenario.default_scenario(nodes)
sc.max_iters, sc.pipg_j_max, sc.power_j_max = mi, pj, wj
b = scenario.make_batch(sc, [0, 1])
with Solver(sc.problem_desc()) as s:
    s.set_solver_path(path)
    t0 = time.perf_counter()
    out = s.scp_solve(b["init_state"], b["x_guess"], b["u_guess"], b["rng_seed"])
    print(nodes, path, mi, pj, wj, "ms", round(1e3 * (time.perf_counter() - t0), 1), "trips", out["power_trips"][0][:mi],
          "pipg", out["history"][0][:mi, 3], flush=True)
