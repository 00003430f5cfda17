"""One GPU's share of BASELINE config 5 (65 536 x N=100 over 8 GPUs = 8 192 run ids per GPU) through
ptopt_cuda_run_batch: generation, full-budget SCP solves on the column-sparse cluster kernels, audit and
records on the device.  usage: python tools/config5_shard_probe.py [batch] [first_run_id] [path]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2404_18034_b200 import scenario
from paper_2404_18034_b200.binding import Solver

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
path = sys.argv[3] if len(sys.argv) > 3 else "auto"
sc = scenario.default_scenario(100)
with Solver(sc.problem_desc()) as s:
    s.set_solver_path(path)
    t0 = time.perf_counter()
    rec = s.run_batch(B, first, sc.initial_state, sc.dispersion.r_low, sc.dispersion.r_high,
                      sc.dispersion.seed, audit_substeps=64)
    dt = time.perf_counter() - t0
    st = s.scp_stage_times()
ok = rec["status"] == 0
print("config5 shard:", path, "batch", B, "first run id", first, "wall s %.2f" % dt, "solves/s %.1f" % (B / dt),
      "failed", int((~ok).sum()), "scp_iterations min/max", int(rec["scp_iterations"][ok].min()),
      int(rec["scp_iterations"][ok].max()), "propellant mean %.6f" % float(rec["propellant_used"][ok].mean()),
      "stages", {k: round(v, 1) for k, v in st.items()})
