"""Pins the plain-C oracle (oracle/ptopt_oracle.c) to the UNMODIFIED reference
compiled in place (oracle/_ref): identical inputs, bit-identical outputs (both are
built with -ffp-contract=off).  Skipped where oracle/_ref is absent."""
import ctypes as C

import numpy as np
import pytest

from oracle_lib import NU, NX, Workspace, random_subproblem, rocket_shape
from paper_2404_18034_b200 import abi, scenario


def rocket_point(rng):
    """A random vehicle state/control like tmodels::random_rocket_point
    (proj/tests/support/test_models.hpp:162-197)."""
    u = lambda: rng.uniform(-1.0, 1.0)  # noqa: E731
    xi = np.zeros(14)
    xi[0] = 1.2 + 0.6 * abs(u())
    for i in range(3):
        xi[1 + i], xi[4 + i], xi[11 + i] = 4.0 * u(), 1.5 * u(), 0.6 * u()
    q = np.array([u(), u(), u(), u() + 1.5])
    xi[7:11] = q / np.linalg.norm(q)
    zeta = np.array([1.5 * u() + 2.5, 1.5 * u(), 1.5 * u(), 0.2 * u(), 0.2 * u(), 0.2 * u()])
    return xi, zeta


def same(a, b):
    np.testing.assert_array_equal(np.asarray(a), np.asarray(b))


def small_scenario(nodes=8):
    sc = scenario.default_scenario(nodes)
    sc.max_iters = 3
    sc.pipg_j_max = 150
    sc.power_j_max = 200
    return sc


def test_model_layer_bitwise(ptor, ptref):
    vp = scenario.default_scenario().problem_desc().vehicle
    rng = np.random.default_rng(2024)
    for _ in range(50):
        xi, zeta = rocket_point(rng)
        ra, a = ptor.model_eval(vp, xi, zeta)
        rb, b = ptref.model_eval(vp, xi, zeta)
        assert ra == rb == 0
        for k in a:
            same(a[k], b[k])
        x = np.concatenate([xi, [rng.uniform(0, 0.1)]])
        u = np.concatenate([zeta, [rng.uniform(0.5, 6.0)]])
        ra, fa, Aa, Ba = ptor.aug_eval(vp, x, u)
        rb, fb, Ab, Bb = ptref.aug_eval(vp, x, u)
        assert ra == rb == 0
        same(fa, fb), same(Aa, Ab), same(Ba, Bb)


def test_model_domain_errors_match(ptor, ptref):
    vp = scenario.default_scenario().problem_desc().vehicle
    xi, zeta = rocket_point(np.random.default_rng(1))
    x, u = np.concatenate([xi, [0.0]]), np.concatenate([zeta, [2.0]])
    for mutate in ("s0", "sneg", "m0", "T0", "snan"):
        xx, uu = x.copy(), u.copy()
        if mutate == "s0":
            uu[6] = 0.0
        if mutate == "sneg":
            uu[6] = -1.0
        if mutate == "snan":
            uu[6] = np.nan
        if mutate == "m0":
            xx[0] = 0.0
        if mutate == "T0":
            uu[0:3] = 0.0
        ra = ptor.aug_eval(vp, xx, uu)[0]
        rb = ptref.aug_eval(vp, xx, uu)[0]
        assert ra == rb and ra > 0, mutate


def test_propagate_interval_bitwise(ptor, ptref):
    vp = scenario.default_scenario().problem_desc().vehicle
    rng = np.random.default_rng(7)
    for trial in range(6):
        xi, zeta = rocket_point(rng)
        xi2, zeta2 = rocket_point(rng)
        x = np.concatenate([xi, [0.0]])
        u0 = np.concatenate([zeta, [rng.uniform(1.0, 6.0)]])
        u1 = np.concatenate([0.5 * (zeta + zeta2), [rng.uniform(1.0, 6.0)]])
        if trial % 2:  # force active path constraints so the y-row is exercised
            x[4:7] *= 4.0
        ra, a = ptor.propagate_interval(vp, x, u0, u1, 0.2, 0.3, 16, trial)
        rb, b = ptref.propagate_interval(vp, x, u0, u1, 0.2, 0.3, 16, trial)
        assert ra == rb == 0
        for k in ("A", "Bm", "Bp", "w", "x_end"):
            same(a[k], b[k])
        if trial % 2:
            assert np.abs(a["A"][14, :14]).max() > 0.0


@pytest.mark.parametrize("model_id,nx,nu,params", [(0, 3, 2, [0, 0]), (1, 2, 2, [-1.0, 1.0]),
                                                   (2, 3, 2, [0, 0]), (3, 3, 3, [0, 0])])
def test_propagate_test_models_bitwise(ptor, ptref, model_id, nx, nu, params):
    rng = np.random.default_rng(100 + model_id)
    x = rng.uniform(-0.5, 0.5, nx)
    u0, u1 = rng.uniform(-0.5, 0.5, nu), rng.uniform(-0.5, 0.5, nu)
    u0[-1], u1[-1] = 1.0, 1.3
    ra, a = ptor.propagate_test_model(model_id, params, x, u0, u1, 0.1, 0.35, 8)
    rb, b = ptref.propagate_test_model(model_id, params, x, u0, u1, 0.1, 0.35, 8)
    assert ra == rb == 0
    for k in ("A", "Bm", "Bp", "w", "x_end"):
        same(a[k], b[k])
    ra, fa, Aa, Ba = ptor.aug_eval_test_model(model_id, params, x, u0)
    rb, fb, Ab, Bb = ptref.aug_eval_test_model(model_id, params, x, u0)
    assert ra == rb == 0
    same(fa, fb), same(Aa, Ab), same(Ba, Bb)


def test_divergence_names_interval(ptor, ptref):
    for lib in (ptor, ptref):
        rc, out = lib.propagate_test_model(4, [0, 0], [5.0, 0.0], [0.0, 4.0], [0.0, 4.0], 0.0,
                                           1.0, 3, 7)
        assert rc == abi.ST_PROPAGATION_DIVERGED and out["fail_index"] == 7
        rc, _ = lib.propagate_test_model(4, [0, 0], [5.0, 0.0], [0.0, 4.0], [0.0, 4.0], 0.0, 1.0,
                                         0)
        assert rc == -1


def test_instance_generation_bitwise(ptor, ptref):
    sc = scenario.default_scenario(15)
    d = sc.problem_desc()
    for run_id in (0, 1, 2, 77, 4095, 65535):
        a = ptor.run_seed(sc.dispersion.seed, run_id)
        assert a == ptref.run_seed(sc.dispersion.seed, run_id) == scenario.run_seed(
            sc.dispersion.seed, run_id)
        ra = ptor.disperse(sc.dispersion.r_low, sc.dispersion.r_high, sc.dispersion.seed, run_id)
        rb = ptref.disperse(sc.dispersion.r_low, sc.dispersion.r_high, sc.dispersion.seed, run_id)
        init = scenario.disperse(sc, run_id)
        same(ra, rb), same(ra, init[1:4])
        _, xa, ua = ptor.initial_guess(d, init)
        _, xb, ub = ptref.initial_guess(d, init)
        xc, uc = scenario.initial_guess(sc, init)
        same(xa, xb), same(ua, ub), same(xa, xc), same(ua, uc)
    for v in (1.0, 8.0, 3.0, 6.0, 0.3, 5.0, 0.7, 1.5, 2.9, 1e-3):
        assert ptor.pow2_near(v) == ptref.pow2_near(v) == scenario.pow2_near(v)
    for seed in (0, 1, 2**63 + 5):
        for a, b in zip(ptor.scp_seed(seed, 9), ptref.scp_seed(seed, 9)):
            same(a, b)


def test_slerp_branch_bitwise(ptor, ptref):
    sc = scenario.default_scenario(6)
    d = sc.problem_desc()
    init = np.array(sc.initial_state)
    q = np.array([0.3, -0.2, 0.1, 0.9])
    init[7:11] = q / np.linalg.norm(q)
    _, xa, ua = ptor.initial_guess(d, init)
    _, xb, ub = ptref.initial_guess(d, init)
    xc, uc = scenario.initial_guess(sc, init)
    same(xa, xb), same(ua, ub), same(xa, xc), same(ua, uc)


def test_linearize_assemble_bitwise(ptor, ptref):
    sc = scenario.default_scenario(15)
    d = sc.problem_desc()
    init = scenario.disperse(sc, 3)
    x, u = scenario.initial_guess(sc, init)
    ra, a = ptor.linearize_all(d, x, u)
    rb, b = ptref.linearize_all(d, x, u, workers=3)
    assert ra == rb == 0
    for k in ("A", "Bm", "Bp", "w", "x_end"):
        same(a[k], b[k])
    ra, sa, ea = ptor.assemble(d, init, x, u, a, with_a_plus=True)
    rb, sb, eb = ptref.assemble(d, init, x, u, b, with_a_plus=True)
    assert ra == rb == 0
    same(ea, eb)
    for f in sa.FIELDS:
        same(getattr(sa, f), getattr(sb, f))
    # non-uniform grid
    tau = np.sort(np.concatenate([[0.0, 1.0], np.random.default_rng(3).uniform(0.05, 0.95, 13)]))
    ra, a = ptor.linearize_all(d, x, u, tau=tau)
    rb, b = ptref.linearize_all(d, x, u, tau=tau)
    assert ra == rb == 0
    same(a["A"], b["A"]), same(a["w"], b["w"])


def test_power_and_pipg_random_bitwise(ptor, ptref):
    rng = np.random.default_rng(2025)
    cfg = abi.PipgConfig(omega=20.0, rho=1.6, j_max=100, j_check=10, eps_abs=1e-12,
                         eps_rel=1e-12, eps_buff=0.05)
    for _ in range(10):
        shape, sub = random_subproblem(rng)
        nx, nu, n = shape.n_x, shape.n_u, shape.nodes
        m = n - 1
        seeds = [rng.uniform(-1, 1, s) for s in ((n, nx), (n, nu), (m, nx), (m, nx))]
        ra, siga, _ = ptor.power_iteration(shape, sub, *seeds, 1e-13, 1e-13, 0.05, 200000)
        rb, sigb, _ = ptref.power_iteration(shape, sub, *seeds, 1e-13, 1e-13, 0.05, 200000)
        assert ra == rb == 0 and siga == sigb
        wa, wb = Workspace(nx, nu, n), Workspace(nx, nu, n)
        outa = ptor.pipg(shape, sub, cfg, siga, wa)
        outb = ptref.pipg(shape, sub, cfg, sigb, wb)
        assert outa == outb
        for f in wa.FIELDS:
            same(getattr(wa, f), getattr(wb, f))
        # warm-started second call
        outa = ptor.pipg(shape, sub, cfg, siga, wa)
        outb = ptref.pipg(shape, sub, cfg, sigb, wb)
        assert outa == outb
        for f in wa.FIELDS:
            same(getattr(wa, f), getattr(wb, f))


def test_power_zero_seed_and_divergence_codes(ptor, ptref):
    rng = np.random.default_rng(42)
    shape, sub = random_subproblem(rng)
    nx, nu, n = shape.n_x, shape.n_u, shape.nodes
    m = n - 1
    z = [np.zeros(s) for s in ((n, nx), (n, nu), (m, nx), (m, nx))]
    for lib in (ptor, ptref):
        assert lib.power_iteration(shape, sub, *z, 1e-12, 1e-12, 0.05, 100)[0] == \
            abi.ST_POWER_SEED_ZERO
    cfg = abi.PipgConfig(omega=1e8, rho=1.6, j_max=20000, j_check=5, eps_abs=1e-11,
                         eps_rel=1e-11, eps_buff=0.05)
    outs = []
    for lib in (ptor, ptref):
        ws = Workspace(nx, nu, n)
        ws.x[:] = 0.5
        outs.append(lib.pipg(shape, sub, cfg, 1e-16, ws))
    # on SolverDiverged the reference reports only the iteration it threw at
    assert (outs[0][0], outs[0][3]) == (outs[1][0], outs[1][3])


def test_scp_solve_bitwise(ptor, ptref):
    sc = small_scenario(8)
    d = sc.problem_desc()
    for run_id in (0, 5):
        b = scenario.make_batch(sc, [run_id])
        args = (d, b["init_state"][0], b["x_guess"][0], b["u_guess"][0], int(b["rng_seed"][0]))
        ra, a = ptor.scp_solve(*args, with_trips=True)
        rb, r = ptref.scp_solve(*args)
        assert ra == rb == 0
        assert a["scp_iterations"] == r["scp_iterations"] == sc.max_iters
        assert a["converged"] == r["converged"]
        assert a["final_defect_inf"] == r["final_defect_inf"]
        same(a["history"], r["history"]), same(a["x"], r["x"]), same(a["u"], r["u"])
        assert (a["power_trips"] > 0).all()


def test_dense_audit_and_run_batch_bitwise(ptor, ptref):
    sc = small_scenario(6)
    d = sc.problem_desc()
    x, u = scenario.initial_guess(sc, np.array(sc.initial_state))
    a = ptor.dense_audit(d, x, u, 16)
    b = ptref.dense_audit(d, x, u, 16)
    assert a[0] == b[0] == 0 and a[1] == b[1] and a[2] == b[2]
    same(a[3], b[3])
    # the sample sink: {interval, tau, g[9], g_max} per node / substep, in the reference's order
    sa = ptor.dense_audit_samples(d, x, u, 5)
    sb = ptref.dense_audit_samples(d, x, u, 5)
    assert sa[0] == sb[0] == 0 and sa[1] == sb[1]
    same(sa[4], sb[4])
    assert sa[4].shape == (5, 6, 12) and (sa[4][:, :, 0] == np.arange(5)[:, None]).all()
    assert sa[4][:, :, 11].max() == sa[1]
    spec = sc.dispersion
    wa, reca, xa, ua = ptor.run_batch(d, sc.initial_state, spec.r_low, spec.r_high, spec.seed, 4,
                                      2, 16, keep=True)
    wb, recb, xb, ub = ptref.run_batch(d, sc.initial_state, spec.r_low, spec.r_high, spec.seed, 4,
                                       1, 16, keep=True)
    assert wa > 0 and wb > 0
    same(reca, recb), same(xa, xb), same(ua, ub)
