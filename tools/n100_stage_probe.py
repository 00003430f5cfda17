"""Per-stage clocks of ONE SCP iteration at N=100 (296 instances = four waves of 74 two-CTA clusters): clk per
power trip / PIPG iteration of the column-sparse cluster kernels.  usage: python tools/n100_stage_probe.py"""
import sys
sys.path.insert(0, ".")
from paper_2404_18034_b200 import scenario
from paper_2404_18034_b200.binding import Solver
n, B = 100, 296
sc = scenario.default_scenario(n)
sc.max_iters = 1
batch = scenario.make_batch(sc, range(B))
with Solver(sc.problem_desc()) as s:
    s.scp_solve(batch["init_state"][:4], batch["x_guess"][:4], batch["u_guess"][:4], batch["rng_seed"][:4])
    res = s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"], batch["rng_seed"])
    st = s.scp_stage_times()
trips = res["power_trips"].sum(axis=-1).mean() if res["power_trips"].ndim > 1 else res["power_trips"].mean()
its = res["history"][:, :, 3].sum(axis=1).mean()
waves = B / 74.0
print("power ms", st["power_iteration"], "trips", trips,
      "clk/trip", st["power_iteration"] * 1e-3 / waves / trips * 1.965e9,
      "pipg ms", st["pipg"], "its", its, "clk/it", st["pipg"] * 1e-3 / waves / its * 1.965e9)
