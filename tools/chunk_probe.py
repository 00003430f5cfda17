"""Prints a digest of linearize_all and a short scp_solve over a small batch; run with and without
PTOPT_STAGE_BYTES_MAX to compare the chunked discretization with the one-pass-pair one
(tests/test_gpu_parity.py::test_linearize_chunked_stage_records)."""
import hashlib
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2404_18034_b200 import scenario
from paper_2404_18034_b200.binding import Solver

sc = scenario.default_scenario(15)
sc.max_iters, sc.pipg_j_max, sc.power_j_max = 2, 60, 40
b = scenario.make_batch(sc, range(23))
x = b["x_guess"].copy()
x[5, 3, 0] = -1.0   # a failing instance (mass <= 0) in the middle of a chunk
with Solver(sc.problem_desc()) as s:
    lin = s.linearize_all(x, b["u_guess"])
    out = s.scp_solve(b["init_state"], b["x_guess"], b["u_guess"], b["rng_seed"])
h = hashlib.sha256()
ok = lin["status"] == 0
for k in ("A", "Bm", "Bp", "w", "x_end"):
    h.update(np.ascontiguousarray(lin[k][ok]).tobytes())
h.update(lin["status"].tobytes()); h.update(lin["fail_index"].tobytes())
h.update(out["x"].tobytes()); h.update(out["u"].tobytes())
print("digest", h.hexdigest(), "status", lin["status"].tolist(), "fail", lin["fail_index"].tolist())
