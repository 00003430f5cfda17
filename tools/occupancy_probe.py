import sys; sys.path.insert(0,'.')
from paper_2404_18034_b200 import scenario
from paper_2404_18034_b200.binding import Solver
sc = scenario.default_scenario(50); sc.max_iters=1; sc.pipg_j_max=50; sc.power_j_max=50
b = scenario.make_batch(sc, range(4))
with Solver(sc.problem_desc()) as s:
    s.set_solver_path("split")
    s.scp_solve(b["init_state"], b["x_guess"], b["u_guess"], b["rng_seed"])
