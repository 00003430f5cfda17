#!/usr/bin/env python
"""Generates tests/golden/reference_vectors.npz from the UNMODIFIED reference compiled in place
(oracle/_ref/libptopt_ref.so, built by `make -C oracle ref` from /root/reference/proj/include,
-O2 -ffp-contract=off).  Run in the container that has /root/reference:

    python tests/golden/make_golden.py

The vectors pin the CPU oracle (bit-for-bit, tests/test_golden.py) and the CUDA path (within the
north_star tolerances, tests/test_gpu_parity.py::test_cuda_path_against_golden_vectors) on
machines where the reference tree does not exist (the GPU box).
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle_lib import CpuOracle, Workspace, random_subproblem, rocket_shape  # noqa: E402
from paper_2404_18034_b200 import abi, scenario  # noqa: E402


def main():
    ref = CpuOracle("ptref")
    out = {}

    # ---- model + one interval at seeded points (rocket6dof.hpp:245-402, discretizer.hpp:82-149)
    sc = scenario.default_scenario(15)
    d = sc.problem_desc()
    rng = np.random.default_rng(20240418)
    xs, us, u1s = [], [], []
    for _ in range(6):
        x = np.zeros(15)
        x[0] = rng.uniform(1.2, 2.0)
        x[1:4] = rng.uniform(-1, 8, 3)
        x[4:7] = rng.uniform(-2.5, 2.5, 3)   # some speeds exceed v_max: active y-row
        q = rng.normal(size=4)
        x[7:11] = q / np.linalg.norm(q)
        x[11:14] = rng.uniform(-0.9, 0.9, 3)
        u = np.concatenate([rng.uniform(0.6, 3.0, 3), rng.uniform(-0.2, 0.2, 3), [rng.uniform(2, 8)]])
        u1 = u + rng.normal(0, 0.2, 7)
        u1[6] = abs(u1[6]) + 0.5
        xs.append(x); us.append(u); u1s.append(u1)
    xs, us, u1s = np.array(xs), np.array(us), np.array(u1s)
    out["pi_x"], out["pi_u"], out["pi_u1"] = xs, us, u1s
    out["pi_tau"] = np.array([0.25, 0.4375])
    A, Bm, Bp, w, xe, f, Aj, Bj = [], [], [], [], [], [], [], []
    for x, u, u1 in zip(xs, us, u1s):
        rc, o = ref.propagate_interval(d.vehicle, x, u, u1, 0.25, 0.4375, 16)
        assert rc == 0
        A.append(o["A"]); Bm.append(o["Bm"]); Bp.append(o["Bp"]); w.append(o["w"]); xe.append(o["x_end"])
        rc, ff, AA, BB = ref.aug_eval(d.vehicle, x, u)
        assert rc == 0
        f.append(ff); Aj.append(AA); Bj.append(BB)
    out.update(pi_A=np.array(A), pi_Bm=np.array(Bm), pi_Bp=np.array(Bp), pi_w=np.array(w),
               pi_x_end=np.array(xe), aug_f=np.array(f), aug_A=np.array(Aj), aug_B=np.array(Bj))

    # ---- instance generation (montecarlo.hpp:43-65, rocket_problem.hpp:127-163)
    sc10 = scenario.default_scenario(10)
    d10 = sc10.problem_desc()
    ids = np.array([0, 1, 7, 4095, 65535])
    spec = sc10.dispersion
    gen_r, gen_seed, gen_x, gen_u = [], [], [], []
    for rid in ids:
        r = ref.disperse(spec.r_low, spec.r_high, spec.seed, int(rid))
        init = np.array(sc10.initial_state)
        init[1:4] = r
        rc, x, u = ref.initial_guess(d10, init)
        assert rc == 0
        gen_r.append(r); gen_seed.append(ref.run_seed(spec.seed, int(rid))); gen_x.append(x); gen_u.append(u)
    out.update(gen_ids=ids, gen_r=np.array(gen_r), gen_seed=np.array(gen_seed, dtype=np.uint64),
               gen_x=np.array(gen_x), gen_u=np.array(gen_u))

    # ---- linearize + assemble at the first generated instance (scp.hpp:139-217)
    init0 = np.array(sc10.initial_state)
    init0[1:4] = gen_r[0]
    rc, blocks = ref.linearize_all(d10, gen_x[0], gen_u[0])
    assert rc == 0
    rc, sub, e_cost = ref.assemble(d10, init0, gen_x[0], gen_u[0], blocks)
    assert rc == 0
    out.update(lin_A=blocks["A"], lin_Bm=blocks["Bm"], lin_Bp=blocks["Bp"], lin_w=blocks["w"],
               lin_x_end=blocks["x_end"], asm_A_minus=sub.A_minus, asm_B_minus=sub.B_minus,
               asm_B_plus=sub.B_plus, asm_w=sub.w, asm_eps=sub.eps_relax, asm_u_min=sub.u_min,
               asm_u_max=sub.u_max, asm_init=sub.init_fix_val, asm_final=sub.final_fix_val,
               asm_e_cost=e_cost)

    # ---- power iteration + PIPG on the assembled rocket subproblem (pipg.hpp:206-292, 350-497)
    shape = rocket_shape(d10)
    sx, su = ref.scp_seed(int(gen_seed[0]), 10)
    z = np.zeros((9, 15))
    rc, sigma, _ = ref.power_iteration(shape, sub, sx, su, z, z, 1e-12, 1e-12, 0.05, 10000)
    assert rc == 0
    cfg = abi.PipgConfig(omega=100.0, rho=1.6, j_max=300, j_check=301, eps_abs=1e-11, eps_rel=1e-11,
                         eps_buff=0.05)
    ws = Workspace(15, 7, 10)
    rc, iters, conv, _ = ref.pipg(shape, sub, cfg, sigma, ws)
    assert rc == 0 and iters == 300
    out.update(pw_seed_x=sx, pw_seed_u=su, pw_sigma=np.array(sigma),
               **{f"pipg_{f}": getattr(ws, f) for f in ws.FIELDS})

    # ---- full SCP loop, reduced budget (scp.hpp:256-364) and run_batch records
    sc10.max_iters = 4
    sc10.pipg_j_max = 300
    sc10.power_j_max = 400
    d10r = sc10.problem_desc()
    rc, res = ref.scp_solve(d10r, init0, gen_x[0], gen_u[0], int(gen_seed[0]))
    assert rc == 0
    out.update(scp_x=res["x"], scp_u=res["u"], scp_history=res["history"],
               scp_meta=np.array([res["scp_iterations"], int(res["converged"])]),
               scp_final_defect=np.array(res["final_defect_inf"]))
    wall, rec, xb, ub = ref.run_batch(d10r, sc10.initial_state, spec.r_low, spec.r_high, spec.seed, 3,
                                      1, 16, keep=True)
    out.update(rb_records=rec, rb_x=xb, rb_u=ub)

    path = Path(__file__).resolve().parent / "reference_vectors.npz"
    np.savez_compressed(path, **out)
    print("wrote", path, path.stat().st_size, "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
