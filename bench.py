#!/usr/bin/env python
"""bench.py — SCP solves/sec of the batched 6-DoF powered-descent hot path on B200.

    python bench.py --gpus N --steps K --warmup W            # this repo's CUDA path
    python bench.py --impl reference --gpus N --steps K ...  # the reference's CPU path

One "step" = one full batched ``scp_solve`` (26 discretizations + 25 power iterations +
25 x 2500 PIPG iterations per instance at the shipped defaults) over one batch of dispersed
landing scenarios, N=50 nodes, 4096 instances per GPU (BASELINE.json configs[3]).  Instances
are independent, so ranks shard run ids with no data-path collective (weak scaling).

JSON line keys: see the bench contract; additionally ``stages_ms`` (device time per stage
of the last timed graph launch), ``roofline`` (dominant kernel vs the FP64 DFMA peak measured
in the same run and vs the compulsory-HBM bound) and ``cpu_baseline`` (the unmodified
reference compiled in place, oracle/_ref, timed on the host cores on a bounded sample).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

NX, NU = 15, 7


# --------------------------------------------------------------------------- helpers
def algorithmic_flops(nodes: int):
    """dense block-product flops only."""
    m = nodes - 1
    disc = m * (16 * 4 * 2 * NX * NX * (NX + 2 * NU) + 2 * (NX * NX + 2 * NX * NU))
    op = m * 2 * 2 * (NX * NX + 2 * NX * NU)  # one PIPG iteration or one power trip
    return disc, op


class ClockSampler:
    """Samples nvidia-smi clocks / throttle reasons while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                     "-i", str(self.index)], capture_output=True, text=True, timeout=5).stdout
                parts = [p.strip() for p in out.strip().split(",")]
                if len(parts) >= 7:
                    self.rows.append(parts)
            except Exception:
                pass
            self._stop.wait(0.25)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = [n for i, n in enumerate(names) if any(r[3 + i] == "Active" for r in self.rows)]
        pw = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None,
                "samples": len(self.rows), "reasons": reasons}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


# --------------------------------------------------------------------------- CPU baseline
def cpu_reference_run(nodes: int, instances: int, workers: int):
    """Times the reference's own mc::run_batch (oracle/_ref when built, else the C restatement)
    on `workers` host threads.  Returns (solves_per_s, kind, wall_s)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import CpuOracle, ref_available
    from paper_2404_18034_b200 import scenario

    sc = scenario.default_scenario(nodes)
    desc = sc.problem_desc()
    if ref_available():
        oracle, kind = CpuOracle("ptref", fast=True), "reference"
    else:
        oracle, kind = CpuOracle("ptor"), "port"
    wall, rec, _, _ = oracle.run_batch(desc, sc.initial_state, sc.dispersion.r_low,
                                       sc.dispersion.r_high, sc.dispersion.seed, instances,
                                       workers, sc.audit_substeps)
    assert (rec[:, 7] == 0).all(), "reference CPU run reported a failed instance"
    return instances / wall, kind, wall


def cpu_stage_timings(nodes: int = 50):
    """the reference's CPU time of the stages BASELINE configs 2 and 3
    isolate -- linearize_all (N=50) and pipg_custom with j_max = 2000, j_check = 2001 at the initial
    guess -- on one core and on all cores (independent instances on a thread pool; ctypes releases
    the GIL).  Bounded: a few seconds."""
    import ctypes
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import NU as _NU, NX as _NX, CpuOracle, SubArrays, Workspace, ref_available, rocket_shape
    from paper_2404_18034_b200 import abi, scenario

    cores = os.cpu_count() or 1
    cpu, kind = (CpuOracle("ptref", fast=True), "reference") if ref_available() else (CpuOracle("ptor"), "port")
    sc = scenario.default_scenario(nodes)
    d = sc.problem_desc()
    shape = rocket_shape(d)
    ids = list(range(2 * cores))
    batch = scenario.make_batch(sc, ids)

    def lin(b):
        return cpu.linearize_all(d, batch["x_guess"][b], batch["u_guess"][b])

    t0 = time.perf_counter()
    blocks = [lin(b) for b in range(4)]
    lin_1 = (time.perf_counter() - t0) / 4
    with ThreadPoolExecutor(max_workers=cores) as pool:
        t0 = time.perf_counter()
        rest = list(pool.map(lin, ids * 2))
        lin_all = len(ids) * 2 / (time.perf_counter() - t0)
    # config 3: subproblem at the initial guess, sigma from the CPU power iteration, cold start
    cfg = abi.PipgConfig(omega=100.0, rho=1.6, j_max=2000, j_check=2001, eps_abs=1e-11, eps_rel=1e-11,
                         eps_buff=0.05)
    subs = []
    for b in range(min(cores, len(ids))):
        rc, blk = rest[b]
        rc2, sub, _ = cpu.assemble(d, batch["init_state"][b], batch["x_guess"][b], batch["u_guess"][b], blk)
        sx, su = cpu.scp_seed(int(batch["rng_seed"][b]), nodes)
        z = np.zeros((nodes - 1, _NX))
        rc3, sigma = cpu.power_iteration(shape, sub, sx, su, z, z, 1e-12, 1e-12, 0.05, 10000)[:2]
        subs.append((sub, sigma))

    def pipg(i):
        sub, sigma = subs[i % len(subs)]
        return cpu.pipg(shape, sub, cfg, sigma, Workspace(_NX, _NU, nodes))

    t0 = time.perf_counter()
    for i in range(2):
        pipg(i)
    pipg_1 = (time.perf_counter() - t0) / 2
    with ThreadPoolExecutor(max_workers=cores) as pool:
        t0 = time.perf_counter()
        list(pool.map(pipg, range(2 * cores)))
        pipg_all = 2 * cores / (time.perf_counter() - t0)
    return {"kind": kind, "cores": cores, "nodes": nodes,
            "linearize_all": {"ms_per_call_1_core": 1e3 * lin_1, "calls_per_s_all_cores": lin_all},
            "pipg_custom_2000_iterations": {"ms_per_solve_1_core": 1e3 * pipg_1,
                                            "solves_per_s_all_cores": pipg_all}}


def cpu_sample_size(args, cores):
    """B_cpu = 2 * nproc instances on nproc workers."""
    return args.cpu_instances or 2 * cores


def run_reference_arm(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    inst = cpu_sample_size(args, cores)
    walls = []
    kind = "reference"
    for i in range(args.warmup + args.steps):
        _, kind, wall = cpu_reference_run(args.nodes, inst, cores)
        if i >= args.warmup:
            walls.append(wall)
    total = sum(walls)
    value = inst * len(walls) / total
    sample = (f"{inst} instances of the {args.batch}-instance N={args.nodes} batch per step "
              f"(run ids 0..{inst - 1}), mc::run_batch on {cores} threads")
    line = {
        "impl": "reference", "metric": "SCP solves/sec (batched, N=50)", "value": value,
        "unit": "solves/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(walls), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def workload_config(args, world):
    return {"workload": f"full SCP loop (trust region + virtual control), batch {args.batch} per GPU, "
                        f"N={args.nodes} nodes, default 6-DoF landing scenario, dispersed initial "
                        f"positions (BASELINE.json configs[3])",
            "batch_per_gpu": args.batch, "global_batch": args.batch * world, "nodes": args.nodes,
            "scp_max_iters": 25, "pipg_j_max": 2500, "power_j_max": 10000,
            "parallelism": f"instances sharded over {world} GPU(s), no collective",
            "l2": "per-step working set (operator blocks + iterates of the whole batch) exceeds "
                  "the 126 MB L2; inputs are re-uploaded/re-initialised every step"}


def other_configs(device_index, fp64_peak):
    """Informational timings of the other BASELINE configs' shapes on this GPU (rank 0 only, after
    the headline measurement; they are parity-test cases, not the metric): config 2 = exact
    discretization only, 1024 x N=50, device-resident; config 5 shape = full SCP solves at N=100
    (two waves of 2-CTA clusters)."""
    import numpy as np
    import torch

    from paper_2404_18034_b200 import scenario
    from paper_2404_18034_b200.binding import Solver

    dev = torch.device("cuda", device_index)
    out = {}
    # ---- config 2
    B, n = 1024, 50
    sc = scenario.default_scenario(n)
    small = scenario.make_batch(sc, range(64))
    idx = np.arange(B) % 64
    x = torch.from_numpy(small["x_guess"][idx]).to(dev)
    u = torch.from_numpy(small["u_guess"][idx]).to(dev)
    m = n - 1
    A = torch.empty((B, m, NX, NX), dtype=torch.float64, device=dev)
    Bm = torch.empty((B, m, NX, NU), dtype=torch.float64, device=dev)
    Bp = torch.empty_like(Bm)
    w = torch.empty((B, m, NX), dtype=torch.float64, device=dev)
    xe = torch.empty_like(w)
    stream = torch.cuda.Stream(device=dev)
    with Solver(sc.problem_desc(), device=device_index, stream=stream) as s, torch.cuda.stream(stream):
        for _ in range(3):
            s.linearize_all_dev(x, u, A, Bm, Bp, w, xe)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            s.linearize_all_dev(x, u, A, Bm, Bp, w, xe)
        e1.record(stream)
        stream.synchronize()
        ms = e0.elapsed_time(e1) / 5
    disc_flop, _ = algorithmic_flops(n)
    tf = B * disc_flop / (ms * 1e-3) * 1e-12
    out["config2_discretization_1024xN50"] = {"ms_per_call": ms, "algorithmic_tflops": tf, "frac_fp64_peak": tf / fp64_peak}
    # single-instance discretization latency (north_star: sub-millisecond): one N=50 instance,
    # device-resident (CUDA events around 20 calls) and through the host-pointer call (wall clock,
    # H2D of the iterate and D2H of the blocks included)
    with Solver(sc.problem_desc(), device=device_index, stream=stream) as s, torch.cuda.stream(stream):
        x1, u1 = x[:1].contiguous(), u[:1].contiguous()
        for _ in range(3):
            s.linearize_all_dev(x1, u1, A[:1], Bm[:1], Bp[:1], w[:1], xe[:1])
        e0.record(stream)
        for _ in range(20):
            s.linearize_all_dev(x1, u1, A[:1], Bm[:1], Bp[:1], w[:1], xe[:1])
        e1.record(stream)
        stream.synchronize()
        dev_ms = e0.elapsed_time(e1) / 20
        hx, hu = small["x_guess"][:1], small["u_guess"][:1]
        s.linearize_all(hx, hu)
        lat = []
        for _ in range(10):
            t0 = time.perf_counter()
            s.linearize_all(hx, hu)
            lat.append(1e3 * (time.perf_counter() - t0))
    out["single_instance_discretization_N50"] = {
        "device_ms_per_call": dev_ms, "host_buffers_ms_p50": statistics.median(lat),
        "what": "linearize_all of ONE N=50 instance (49 intervals x 16 RK4 steps): device-resident inputs "
                "timed with CUDA events, and ptopt_cuda_linearize_batch with host buffers timed by wall clock "
                "(the reference takes 26 ms on one core, BASELINE.md section 2)"}
    # ---- config 3: PIPG only, fixed 2000 iterations (j_check = 2001 disables the stop test), batch
    #      1024, N=50, subproblems assembled at the initial guess, sigma from the power iteration,
    #      cold start; device-resident, CUDA events on the handle's stream
    import ctypes as C

    from paper_2404_18034_b200 import abi
    from paper_2404_18034_b200.binding import _check, _dp
    with Solver(sc.problem_desc(), device=device_index, stream=stream) as s, torch.cuda.stream(stream):
        base = 64
        blk = s.linearize_all(small["x_guess"], small["u_guess"])
        sub = s.assemble_subproblem(small["init_state"], small["x_guess"], small["u_guess"], blk)
        shape = s.subproblem_shape()
        sx = np.full((base, n, NX), 1.0 / np.sqrt(n * (NX + NU)))
        su = np.full((base, n, NU), 1.0 / np.sqrt(n * (NX + NU)))
        zz = np.zeros((base, m, NX))
        sigma, _, st = s.power_iteration_custom(shape, sub, sx, su, zz, zz, 1e-12, 1e-12, 0.05, 10000)
        assert (st == 0).all()
        dsub = {k: torch.from_numpy(np.ascontiguousarray(v[idx])).to(dev) for k, v in sub.items() if v is not None}
        arrs = abi.SubproblemArrays()
        for f, _ in abi.SubproblemArrays._fields_:
            setattr(arrs, f, dsub[f].data_ptr() if f in dsub else None)
        dsig = torch.from_numpy(sigma[idx]).to(dev)
        ws = {"x": torch.zeros((B, n, NX), dtype=torch.float64, device=dev),
              "u": torch.zeros((B, n, NU), dtype=torch.float64, device=dev),
              "vc_pos": torch.zeros((B, m, NX), dtype=torch.float64, device=dev),
              "vc_neg": torch.zeros((B, m, NX), dtype=torch.float64, device=dev),
              "dyn_dual": torch.zeros((B, m, NX), dtype=torch.float64, device=dev),
              "relax_dual": torch.zeros((B, m), dtype=torch.float64, device=dev)}
        wsa = abi.WorkspaceArrays()
        for f, _ in abi.WorkspaceArrays._fields_:
            setattr(wsa, f, ws[f].data_ptr())
        cfg = abi.PipgConfig(omega=100.0, rho=1.6, j_max=2000, j_check=2001, eps_abs=1e-11, eps_rel=1e-11,
                             eps_buff=0.05)
        its = torch.zeros(B, dtype=torch.int32, device=dev)

        def pipg_once():
            for t in ws.values():
                t.zero_()
            _check(s.lib.ptopt_cuda_pipg_batch_dev(s._h, C.c_int(B), C.byref(shape), C.byref(arrs), C.byref(cfg),
                                                   _dp(dsig), C.byref(wsa), _dp(its), None, None, None))

        pipg_once()
        stream.synchronize()
        e0.record(stream)
        for _ in range(3):
            pipg_once()
        e1.record(stream)
        stream.synchronize()
        ms3 = e0.elapsed_time(e1) / 3
        assert int(its.min()) == 2000 and int(its.max()) == 2000
    _, op_flop = algorithmic_flops(n)
    tf3 = B * 2000 * op_flop / (ms3 * 1e-3) * 1e-12
    out["config3_pipg_2000_iterations_1024xN50"] = {
        "ms_per_call": ms3, "solves_per_s": B / (ms3 * 1e-3), "algorithmic_tflops": tf3,
        "frac_fp64_peak": tf3 / fp64_peak,
        "what": "pipg_custom only, j_max = 2000 with the stop test disabled, cold start, 1024 subproblems "
                "assembled at the initial guess (64 distinct, tiled), device-resident"}
    # ---- config 5 shape
    n, B = 100, 296
    sc = scenario.default_scenario(n)
    batch = scenario.make_batch(sc, range(B))
    with Solver(sc.problem_desc(), device=device_index) as s:
        s.scp_solve(batch["init_state"][:4], batch["x_guess"][:4], batch["u_guess"][:4], batch["rng_seed"][:4])
        res = s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"], batch["rng_seed"])
        st = s.scp_stage_times()
    out["config5_shape_296xN100"] = {
        "solves_per_s": B / (st["graph_total"] * 1e-3), "graph_ms": st["graph_total"],
        "stages_ms": {k: st[k] for k in ("linearize", "power_iteration", "pipg")},
        "power_trips_mean": float(res["power_trips"].sum(axis=1).mean()),
        "what": "full SCP solves at N=100 on one GPU (one instance over a 2-CTA cluster, 74 instances at a time, "
                "four waves: column-sparse power iteration, dense cluster PIPG), device time of the graph"}
    # ---- the headline configuration on the dense register-resident kernels alone (round-1 path), for
    #      the gain of the column-sparse kernels in the same run
    n, B = 50, 4096
    sc = scenario.default_scenario(n)
    batch = scenario.make_batch(sc, range(B))
    with Solver(sc.problem_desc(), device=device_index) as s:
        s.set_solver_path("dense")
        s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"], batch["rng_seed"])
        s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"], batch["rng_seed"])
        st = s.scp_stage_times()
    out["config4_on_the_dense_kernels_4096xN50"] = {
        "solves_per_s": B / (st["graph_total"] * 1e-3), "stages_ms": st,
        "what": "the step of the headline metric with ptopt_cuda_set_solver_path(PTOPT_SOLVER_FAST_DENSE): five "
                "threads per node, dense operator (no zero pattern assumed), device time of the graph"}
    # ---- config 1 shape: the default scenario (N=15), one instance, full SCP loop
    sc = scenario.default_scenario(15)
    one = scenario.make_batch(sc, range(1))
    with Solver(sc.problem_desc(), device=device_index) as s:
        s.scp_solve(one["init_state"], one["x_guess"], one["u_guess"], one["rng_seed"])
        lat = []
        for _ in range(3):
            t0 = time.perf_counter()
            s.scp_solve(one["init_state"], one["x_guess"], one["u_guess"], one["rng_seed"])
            lat.append(1e3 * (time.perf_counter() - t0))
    out["config1_default_scenario_single_instance_N15"] = {
        "latency_ms_p50": statistics.median(lat),
        "what": "SPEC default 6-DoF landing scenario, one instance, full SCP loop, host buffers "
                "(the reference takes 3.3-3.8 s on one core, SURVEY 8d)"}
    return out


# --------------------------------------------------------------------------- own arm
def run_own_arm(args):
    import numpy as np
    import torch

    from paper_2404_18034_b200 import scenario, sharding
    from paper_2404_18034_b200.binding import RECORD_DTYPE, Solver

    rank, local_rank, world = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device — the product path has no CPU fallback")
    # PTOPT_BENCH_SHARE_GPU=1 (plumbing check only, numbers meaningless): all ranks time-slice the
    # GPUs that exist and rendezvous over gloo, so the multi-rank path can be exercised on one GPU
    share_gpu = os.environ.get("PTOPT_BENCH_SHARE_GPU") == "1"
    if share_gpu:
        local_rank %= torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    use_dist = world > 1
    if use_dist:
        import torch.distributed as dist
        if share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()

    B, n = args.batch, args.nodes
    sc = scenario.default_scenario(n)
    desc = sc.problem_desc()
    mi = int(desc.max_iters)
    first_id, count = sharding.shard_range(world * B, world, rank)  # weak scaling: B ids per rank
    assert count == B
    batch = scenario.make_batch(sc, range(first_id, first_id + B))

    stream = torch.cuda.Stream(device=dev)
    solver = Solver(desc, device=local_rank, stream=stream)
    solver.set_solver_path(args.solver_path)

    # device-resident inputs / outputs for the kernel-only number
    d_init = torch.from_numpy(batch["init_state"]).to(dev)
    d_xg = torch.from_numpy(batch["x_guess"]).to(dev)
    d_ug = torch.from_numpy(batch["u_guess"]).to(dev)
    d_seed = torch.from_numpy(batch["rng_seed"].view(np.int64)).to(dev)
    d_x = torch.empty((B, n, NX), dtype=torch.float64, device=dev)
    d_u = torch.empty((B, n, NU), dtype=torch.float64, device=dev)
    d_iters = torch.empty(B, dtype=torch.int32, device=dev)
    d_conv = torch.empty(B, dtype=torch.uint8, device=dev)
    d_fdef = torch.empty(B, dtype=torch.float64, device=dev)
    d_hist = torch.empty((B, mi, 5), dtype=torch.float64, device=dev)
    d_trips = torch.empty((B, mi), dtype=torch.int32, device=dev)
    d_status = torch.empty(B, dtype=torch.int32, device=dev)
    d_fail = torch.empty(B, dtype=torch.int32, device=dev)

    def step_dev():
        solver.scp_solve_dev(d_init, d_xg, d_ug, d_seed, d_x, d_u, d_iters, d_conv, d_fdef,
                             d_hist, d_trips, d_status, d_fail)

    fp64_peak = solver.measure_fp64_peak()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step_dev()
        stream.synchronize()
        barrier()
        launches0 = solver.launch_count
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local_rank) as clocks:
            ev0.record(stream)
            for _ in range(args.steps):
                step_dev()
            ev1.record(stream)
            stream.synchronize()
        barrier()
        launches = solver.launch_count - launches0
    ms_total = ev0.elapsed_time(ev1)
    stages = solver.scp_stage_times()
    trips = d_trips.cpu().numpy().astype(np.int64)
    hist = d_hist.cpu().numpy()
    status = d_status.cpu().numpy()
    scp_iters = d_iters.cpu().numpy()

    # ---- end to end through the host-pointer C-ABI call, pinned host buffers
    def pinned(shape, dtype):
        return torch.empty(shape, dtype=dtype).pin_memory().numpy()

    h_in = {}
    for k in ("init_state", "x_guess", "u_guess", "rng_seed"):
        src = batch[k].view(np.int64) if batch[k].dtype == np.uint64 else batch[k]
        h_in[k] = pinned(src.shape, torch.from_numpy(src).dtype)
        h_in[k][...] = src
    h_out = dict(x=pinned((B, n, NX), torch.float64), u=pinned((B, n, NU), torch.float64),
                 scp_iterations=pinned((B,), torch.int32), converged=pinned((B,), torch.uint8),
                 final_defect_inf=pinned((B,), torch.float64),
                 history=pinned((B, mi, 5), torch.float64),
                 power_trips=pinned((B, mi), torch.int32), status=pinned((B,), torch.int32),
                 fail_index=pinned((B,), torch.int32))
    h2d = sum(int(v.nbytes) for v in h_in.values())
    d2h = sum(int(v.nbytes) for v in h_out.values())

    def step_e2e():
        solver.scp_solve_into(h_in["init_state"], h_in["x_guess"], h_in["u_guess"],
                              h_in["rng_seed"], h_out)

    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    step_e2e()  # the graph is warm already; one untimed pass for the staging path
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        step_e2e()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    assert np.array_equal(h_out["x"], d_x.cpu().numpy()), "e2e and device-resident results differ"

    # ---- the reference-facing batch call, mc::run_batch: generation, solve, audit and records on
    #      the device; only the dispersion spec goes in and the RunRecords come back
    spec = sc.dispersion
    records = torch.empty(B * RECORD_DTYPE.itemsize, dtype=torch.uint8).pin_memory().numpy().view(RECORD_DTYPE)
    barrier()
    t0 = time.perf_counter()
    solver.run_batch(B, first_id, sc.initial_state, spec.r_low, spec.r_high, spec.seed,
                     audit_substeps=sc.audit_substeps, records=records)
    torch.cuda.synchronize()
    rb_s = time.perf_counter() - t0
    assert (records["run_id"] == np.arange(first_id, first_id + B)).all()
    assert np.array_equal(records["scp_iterations"], h_out["scp_iterations"])

    # ---- p50 latency of a single full solve (batch of one) through the host-pointer call
    lat_ms = []
    lat_fast_ms = None
    if rank == 0 and args.latency_runs > 0:
        one = {k: np.ascontiguousarray(h_in[k][:1]) for k in h_in}
        one_out = {k: np.ascontiguousarray(v[:1]) for k, v in h_out.items()}
        with Solver(desc, device=local_rank) as single:
            single.scp_solve_into(one["init_state"], one["x_guess"], one["u_guess"], one["rng_seed"], one_out)
            for _ in range(args.latency_runs):
                t0 = time.perf_counter()
                single.scp_solve_into(one["init_state"], one["x_guess"], one["u_guess"], one["rng_seed"],
                                      one_out)
                lat_ms.append(1e3 * (time.perf_counter() - t0))
        # the two kernel families round differently (1e-14); both are checked against the CPU in tests/
        assert np.abs(one_out["x"][0] - h_out["x"][0]).max() <= 1e-6, "batch-of-one result differs"
        with Solver(desc, device=local_rank) as single:  # the same solve on the throughput kernels
            single.set_solver_path("fast")
            single.scp_solve_into(one["init_state"], one["x_guess"], one["u_guess"], one["rng_seed"], one_out)
            t0 = time.perf_counter()
            single.scp_solve_into(one["init_state"], one["x_guess"], one["u_guess"], one["rng_seed"], one_out)
            lat_fast_ms = 1e3 * (time.perf_counter() - t0)

    # ---- max over ranks
    if use_dist:
        ms_total = sharding.max_over_ranks(ms_total)
        e2e_s = sharding.max_over_ranks(e2e_s)
        rb_s = sharding.max_over_ranks(rb_s)
        bad = torch.tensor([int((status != 0).sum())], device=torch.device("cpu") if share_gpu else dev)
        dist.all_reduce(bad)
        n_bad = int(bad[0])
    else:
        n_bad = int((status != 0).sum())

    if rank == 0:
        disc_flop, op_flop = algorithmic_flops(n)
        sum_trips = float(trips.sum())
        pipg_iters = float(hist[:, :, 3].sum())
        n_lin = float((scp_iters + 1).sum())
        flop = {"linearize": n_lin * disc_flop, "power_iteration": sum_trips * op_flop,
                "pipg": pipg_iters * op_flop}
        dom = max(("linearize", "power_iteration", "pipg"), key=lambda k: stages[k])
        achieved = flop[dom] / (stages[dom] * 1e-3) * 1e-12
        total_flop = sum(flop.values())
        # DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
        # (profiles/ncu_traffic.json: bytes for a 148-instance launch), scaled to this batch
        traffic = None
        kernel_of = {"linearize": "column_pass_kernel",
                     "power_iteration": "power_cs_kernel",   # (n > 61: its 2-CTA cluster variant)
                     "pipg": "pipg_cs_kernel" if n <= 61 else "pipg_fast_kernel"}
        tpath = ROOT / "profiles" / "ncu_traffic.json"
        if tpath.exists() and n in (50, 100):
            tj = json.loads(tpath.read_text())
            tk = (tj["kernels"] if n == 50 else tj.get("kernels_n100", {}).get("kernels", {})).get(kernel_of[dom])
            if tk:
                per_instance = (tk["dram_read_bytes"] + tk["dram_write_bytes"]) / float(tk.get("instances", 148))
                traffic = per_instance * B
        m_int = n - 1
        compulsory = {"linearize": B * (n * 22 + m_int * 465) * 8,
                      "power_iteration": B * (m_int * 435 + n * 22 + 2 * m_int * 15) * 8,
                      "pipg": B * (m_int * 435 + 2 * (n * 22 + m_int * 46) + m_int * 16 + 2 * n * 7) * 8}
        value = world * B * args.steps / (ms_total * 1e-3)
        # Shared-memory view of the two solver kernels (one CTA = one instance = one SM): clocks per
        # trip / iteration from the stage time at the sampled SM clock, against the shared-memory
        # wavefronts one trip / iteration issues (ncu source counters of the hot loops of the
        # column-sparse kernels: 376 / 446 per pass of the four role bodies x 2 warps per role,
        # profiles/r02_cs_power_loop_stalls.txt and r02_cs_pipg_loop_stalls.txt; one wavefront per
        # clock and SM, tools/probes/smem_width.cu)
        smem_view = None
        clk_info = clocks.summary()
        if n == 50 and args.solver_path == "auto" and clk_info.get("sm_mhz"):
            sms = min(torch.cuda.get_device_properties(dev).multi_processor_count, B)
            units = {"power_iteration": sum_trips, "pipg": pipg_iters}
            wavefronts = {"power_iteration": 376.0 * 2, "pipg": 446.0 * 2}
            smem_view = {}
            for k in units:
                clk = stages[k] * 1e-3 * clk_info["sm_mhz"] * 1e6 * sms / units[k]  # stage times: last launch
                smem_view[k] = {"clk_per_iteration": clk, "smem_wavefronts_per_iteration": wavefronts[k],
                                "frac_of_smem_floor": wavefronts[k] / clk}
        line = {
            "metric": "SCP solves/sec (batched, N=50)", "value": value, "unit": "solves/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_total / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, world),
            "clocks": clocks.summary(),
            "e2e": {"value": world * B * e2e_steps / e2e_s, "unit": "solves/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": e2e_steps},
            "e2e_run_batch": {"value": world * B / rb_s, "unit": "solves/s",
                              "call": "ptopt_cuda_run_batch (mc::run_batch: generation + solve + audit "
                                      "+ records on the device)",
                              "h2d_bytes_per_step": 8 * (14 + 7 + 4 * n),
                              "d2h_bytes_per_step": int(records.nbytes),
                              "converged_fraction": float(records["converged"].mean()),
                              "propellant_mean": float(records["propellant_used"].mean())},
            "single_solve_latency_ms": {"p50": statistics.median(lat_ms) if lat_ms else None,
                                        "min": min(lat_ms) if lat_ms else None, "runs": len(lat_ms),
                                        "what": "one N=50 instance, full 25-iteration budget, "
                                                "ptopt_cuda_scp_solve_batch with host buffers; under AUTO a batch "
                                                "of one runs the latency-mode kernels (one instance over a cluster "
                                                "of 8 CTAs, 16 threads per node)",
                                        "throughput_kernels_ms": lat_fast_ms},
            "gpu_launches": int(launches),
            "stages_ms": stages,
            "work": {"power_trips_mean": sum_trips / B, "pipg_iterations_mean": pipg_iters / B,
                     "scp_iterations_mean": float(scp_iters.mean()), "failed_instances": n_bad,
                     "algorithmic_gflop_per_solve": total_flop / B * 1e-9,
                     "algorithmic_tflops_whole_step": total_flop / (stages["graph_total"] * 1e-3) * 1e-12},
            "roofline": {
                "bound": "fp64", "kernel": dom, "achieved": achieved, "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": achieved / fp64_peak,
                "peak_source": "DFMA microbenchmark measured in this run (MEASURED_PEAKS.json has "
                               "no fp64 entry)",
                "traffic": traffic,
                "traffic_source": "profiles/ncu_traffic.json: dram__bytes_read.sum + dram__bytes_write.sum of a "
                                  "committed ncu --set full capture (148 instances, first launch), scaled to "
                                  "this batch; not re-measured in this run",
                "traffic_unit": "bytes per launch (ncu dram read+write, scaled from a "
                                                    "148-instance capture)",
                "compulsory_hbm_bytes_per_launch": compulsory[dom],
                "per_stage": {k: {"tflops": flop[k] / (stages[k] * 1e-3) * 1e-12,
                                  "frac": flop[k] / (stages[k] * 1e-3) * 1e-12 / fp64_peak,
                                  "share_of_step": stages[k] / stages["graph_total"]}
                              for k in ("linearize", "power_iteration", "pipg")},
                "shared_memory_view": smem_view,
            },
        }
        if world == 1 and not args.no_other_configs:
            line["other_configs"] = other_configs(local_rank, fp64_peak)
        if world == 1 and not args.no_cpu_baseline:
            cores = os.cpu_count() or 1
            inst = cpu_sample_size(args, cores)
            v, kind, wall = cpu_reference_run(n, inst, cores)
            v1, _, wall1 = cpu_reference_run(n, 1, 1)
            line["cpu_baseline"] = {
                "value": v, "unit": "solves/s", "cores": cores, "kind": kind,
                "sample": f"run ids 0..{inst - 1} of the same batch ({inst} full N={n} solves, "
                          f"mc::run_batch on {cores} threads, {wall:.1f} s)",
                "workers_1": {"value": v1, "unit": "solves/s", "cores": 1,
                              "sample": f"run id 0, mc::run_batch with workers = 1, {wall1:.1f} s"},
                "build": "g++ -O3 -march=x86-64-v3 (AVX2 + FMA): the library is built where /root/reference "
                         "exists and shipped to the GPU box, so -march=native of the build container is not "
                         "portable to the box's host CPU",
                "stages": cpu_stage_timings(n)}
        print(json.dumps(line), flush=True)
    solver.close()
    if use_dist:
        dist.destroy_process_group()


def run_own_arm_multi(args):
    """`python bench.py --gpus N` WITHOUT torchrun: one process drives N devices through the host-layer
    entry ptopt_cuda_run_batch_multi (one handle + host thread per device, contiguous run-id ranges,
    records written into their run-id slots) -- mc::run_batch with its worker pool mapped onto GPUs
    (montecarlo.hpp:153-171).  Weak scaling: args.batch instances per device; the step time is the
    slowest device's wall time of its ptopt_cuda_run_batch call (generation, solve, audit, records
    and the D2H of the records included)."""
    import numpy as np
    import torch

    from paper_2404_18034_b200 import scenario
    from paper_2404_18034_b200.binding import RECORD_DTYPE, run_batch_multi

    n_dev = torch.cuda.device_count()
    if n_dev < 1:
        raise SystemExit("bench.py: no CUDA device -- the product path has no CPU fallback")
    # fewer physical devices than asked for: entries wrap around (plumbing check, numbers meaningless)
    devices = [g % n_dev for g in range(args.gpus)]
    B, n = args.batch, args.nodes
    sc = scenario.default_scenario(n)
    desc = sc.problem_desc()
    spec = sc.dispersion
    total = B * args.gpus
    records = np.empty(total, RECORD_DTYPE)
    times = []
    for i in range(args.warmup + args.steps):
        _, ms = run_batch_multi(desc, devices, total, 0, sc.initial_state, spec.r_low, spec.r_high, spec.seed,
                                audit_substeps=sc.audit_substeps, records=records)
        if i >= args.warmup:
            times.append(float(ms.max()))
    assert (records["run_id"] == np.arange(total)).all() and (records["status"] == 0).all()
    step_ms = sum(times) / len(times)
    value = total / (step_ms * 1e-3)
    line = {"metric": "SCP solves/sec (batched, N=50)", "value": value, "unit": "solves/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(workload_config(args, args.gpus), launcher="single process, ptopt_cuda_run_batch_multi",
                           devices=devices, distinct_devices=len(set(devices))),
            "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 8 * (14 + 7 + 4 * n) * args.gpus,
                    "d2h_bytes_per_step": int(records.nbytes),
                    "call": "ptopt_cuda_run_batch_multi (mc::run_batch: generation + solve + audit + records on "
                            "each device)"},
            "gpu_launches": None,
            "note": "value is measured through the host-buffer call (wall clock of the slowest device's worker), so "
                    "value == e2e here; the device-timed number and the roofline come from the torchrun path"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--batch", type=int, default=4096, help="instances per GPU")
    ap.add_argument("--nodes", type=int, default=50)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--solver-path", choices=("auto", "generic", "split", "latency", "fast", "dense"), default="auto",
                    help="kernel family for power iteration / PIPG (ptopt_cuda_set_solver_path)")
    ap.add_argument("--cpu-instances", type=int, default=0,
                    help="instances in the CPU sample (default: one per host core)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the informational timings of the other BASELINE config shapes")
    ap.add_argument("--latency-runs", type=int, default=5,
                    help="batch-of-one solves timed for the p50 single-solve latency (0 = skip)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        run_own_arm_multi(args)
    else:
        run_own_arm(args)


if __name__ == "__main__":
    main()
