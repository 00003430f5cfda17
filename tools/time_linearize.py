"""Times ptopt_cuda_linearize_batch_dev on device-resident inputs (B x N nodes; BASELINE config 2
is B=1024, N=50).  usage: python tools/time_linearize.py [B] [nodes]"""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2404_18034_b200 import scenario
from paper_2404_18034_b200.binding import Solver
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50
sc = scenario.default_scenario(n)
small = scenario.make_batch(sc, range(64))
idx = np.arange(B) % 64
dev = torch.device("cuda", 0)
x = torch.from_numpy(small["x_guess"][idx]).to(dev); u = torch.from_numpy(small["u_guess"][idx]).to(dev)
m = n - 1
A = torch.empty((B, m, 15, 15), dtype=torch.float64, device=dev); Bm = torch.empty((B, m, 15, 7), dtype=torch.float64, device=dev)
Bp = torch.empty_like(Bm); w = torch.empty((B, m, 15), dtype=torch.float64, device=dev); xe = torch.empty_like(w)
stream = torch.cuda.Stream(device=dev)
with Solver(sc.problem_desc(), stream=stream) as s, torch.cuda.stream(stream):
    for _ in range(3): s.linearize_all_dev(x, u, A, Bm, Bp, w, xe)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(5): s.linearize_all_dev(x, u, A, Bm, Bp, w, xe)
    e1.record(stream); stream.synchronize()
    ms = e0.elapsed_time(e1) / 5
flop = B * m * 836070
print(f"linearize B={B} N={n}: {ms:.3f} ms/call  {flop/ms*1e-9:.2f} TFLOP/s (algorithmic)  checksum {float(A.sum()):.12e}")
