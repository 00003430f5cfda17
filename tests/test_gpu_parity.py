"""GPU parity tests: the CUDA library (through the C-ABI) against the CPU oracle on
identical inputs.  Tolerances are the ones BASELINE.json's north_star states:
discretization blocks <= 1e-9 relative, PIPG iterates / final trajectories <= 1e-6."""
import numpy as np
import pytest

from oracle_lib import (NU, NX, SubArrays, Workspace, dense_operator, pack_primal,
                        random_subproblem, rocket_shape)
from paper_2404_18034_b200 import abi, scenario

pytestmark = pytest.mark.gpu

TOL_DISC = 1e-9   # relative, scaled by max(1, |block|_inf) as oracles.hpp:73-82 does
TOL_ITER = 1e-6   # absolute on scaled iterates / final trajectories
TOL_SIGMA = 1e-9  # relative


def rel_err(a, b):
    return np.abs(a - b).max() / max(1.0, np.abs(b).max())


@pytest.fixture(scope="module", params=["fast", "dense", "generic", "split", "latency"])
def solver15(request):
    """The default-scenario handle, once per kernel family: 'fast' runs the register-resident
    throughput kernels on rocket-shaped subproblems (the column-sparse kernels -- four role-uniform
    warps per 32 nodes -- with the dense ones behind them for operators without the rocket model's
    zero pattern), 'dense' the dense ones alone (five threads per node, one CTA per instance),
    'generic' forces the shape-generic ones, 'split' shares every rocket-shaped instance between
    the two CTAs of a cluster, 'latency' spreads every instance over a cluster of up to eight CTAs
    with sixteen threads per node.  ('auto' picks 'latency' for batches that fit the chip in one
    wave and 'fast' otherwise: test_auto_path_selection.)"""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(15)
    with Solver(sc.problem_desc()) as s:
        s.set_solver_path(request.param)
        yield sc, s


def stressed_iterate(sc, run_id, rng):
    """An iterate with large defects and active path constraints (y-row of A nonzero)."""
    init = scenario.disperse(sc, run_id)
    x, u = scenario.initial_guess(sc, init)
    x = x + rng.normal(0, 0.05, x.shape)
    x[:, 4:7] *= 3.0                      # speed above v_max
    x[:, 11:14] += rng.normal(0, 0.6, (x.shape[0], 3))
    q = x[:, 7:11] + rng.normal(0, 0.3, (x.shape[0], 4))
    x[:, 7:11] = q / np.linalg.norm(q, axis=1, keepdims=True)
    u = u + rng.normal(0, 0.3, u.shape)
    u[:, 6] = np.abs(u[:, 6]) + 1.0
    u[:, 3:6] += rng.normal(0, 0.3, (u.shape[0], 3))
    return init, x, u


def test_linearize_parity_initial_guess_and_stressed(solver15, ptor):
    sc, s = solver15
    d = sc.problem_desc()
    rng = np.random.default_rng(11)
    xs, us = [], []
    for run_id in range(24):
        if run_id % 2 == 0:
            init = scenario.disperse(sc, run_id)
            x, u = scenario.initial_guess(sc, init)
        else:
            _, x, u = stressed_iterate(sc, run_id, rng)
        xs.append(x), us.append(u)
    out = s.linearize_all(np.stack(xs), np.stack(us))
    assert (out["status"] == 0).all()
    active_rows = 0
    for b in range(len(xs)):
        rc, ref = ptor.linearize_all(d, xs[b], us[b])
        assert rc == 0
        for k in ("A", "Bm", "Bp", "w", "x_end"):
            assert rel_err(out[k][b], ref[k]) <= TOL_DISC, (b, k)
        active_rows += int(np.abs(ref["A"][:, 14, :14]).max() > 0)
    assert active_rows >= 8  # the stressed set really exercises the CTCS row


def test_linearize_batch1024_n50_subset_parity(ptor):
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(50)
    d = sc.problem_desc()
    B = 1024
    batch = scenario.make_batch(sc, range(B))
    with Solver(d) as s:
        out = s.linearize_all(batch["x_guess"], batch["u_guess"])
    assert (out["status"] == 0).all()
    for b in (0, 1, 511, 1023):
        rc, ref = ptor.linearize_all(d, batch["x_guess"][b], batch["u_guess"][b])
        assert rc == 0
        for k in ("A", "Bm", "Bp", "w", "x_end"):
            assert rel_err(out[k][b], ref[k]) <= TOL_DISC, (b, k)
    # forward-shot property (test_discretizer.cpp:152-190): x_end of interval k equals the
    # state reached by the nonlinear propagation, so A x + B u + w reproduces it
    k = 7
    lin = (np.einsum("bij,bj->bi", out["A"][:, k], batch["x_guess"][:, k])
           + np.einsum("bij,bj->bi", out["Bm"][:, k], batch["u_guess"][:, k])
           + np.einsum("bij,bj->bi", out["Bp"][:, k], batch["u_guess"][:, k + 1]) + out["w"][:, k])
    assert np.abs(lin - out["x_end"][:, k]).max() < 1e-11


def test_linearize_chunked_stage_records():
    """Batches whose stage records would exceed PTOPT_STAGE_BYTES_MAX run the state / column passes
    in chunks that reuse the record buffer (e.g. 8192 x N=100 per GPU in BASELINE config 5).  A cap
    of 3 record tiles forces 4 chunks for 23 x 14 intervals; blocks, failure codes (one failing
    instance inside a chunk) and a short SCP solve must be bit-identical to the unchunked run."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    tile_bytes = 32 * 64 * 84 * 8

    def digest(env_extra):
        env = dict(os.environ, **env_extra)
        out = subprocess.run([sys.executable, str(root / "tools" / "chunk_probe.py")], cwd=str(root), env=env,
                             capture_output=True, text=True, timeout=300)
        assert out.returncode == 0, out.stderr
        return [l for l in out.stdout.splitlines() if l.startswith("digest")][0]

    whole = digest({})
    chunked = digest({"PTOPT_STAGE_BYTES_MAX": str(3 * tile_bytes)})
    assert "status [0, 0, 0, 0, 0, 4," in whole  # instance 5 fails with the mass code
    assert whole == chunked


def test_linearize_failure_codes_match_oracle(solver15, ptor):
    sc, s = solver15
    d = sc.problem_desc()
    init = scenario.disperse(sc, 0)
    x0, u0 = scenario.initial_guess(sc, init)
    cases = []
    for kind in ("dilation", "mass", "thrust", "nan", "dilation_two", "ok"):
        x, u = x0.copy(), u0.copy()
        if kind == "dilation":
            u[6, 6] = 0.0          # used by intervals 5 and 6 -> first failure at 5
        if kind == "dilation_two":
            u[9, 6] = -1.0
            u[3, 6] = -2.0
        if kind == "mass":
            x[4, 0] = -0.5
        if kind == "thrust":
            u[8, 0:3] = 0.0        # |T| = 0 exactly at node 8: start of interval 8, end of 7
        if kind == "nan":
            x[10, 2] = np.nan
        cases.append((kind, x, u))
    out = s.linearize_all(np.stack([c[1] for c in cases]), np.stack([c[2] for c in cases]))
    for b, (kind, x, u) in enumerate(cases):
        rc, ref = ptor.linearize_all(d, x, u)
        assert out["status"][b] == rc, kind
        if rc:
            assert out["fail_index"][b] == ref["fail_index"], kind
    assert out["status"][-1] == 0


def test_assemble_is_exact(solver15, ptor):
    sc, s = solver15
    d = sc.problem_desc()
    rng = np.random.default_rng(5)
    init, x, u = stressed_iterate(sc, 3, rng)
    rc, blocks = ptor.linearize_all(d, x, u)
    assert rc == 0
    rc, sub, e_cost = ptor.assemble(d, init, x, u, blocks)
    out = s.assemble_subproblem(init[None], x[None], u[None],
                                {k: v[None] for k, v in blocks.items() if k != "fail_index"})
    for f in ("A_minus", "B_minus", "B_plus", "w", "eps_relax", "u_min", "u_max", "init_fix_val"):
        np.testing.assert_array_equal(out[f][0], getattr(sub, f))
    np.testing.assert_array_equal(out["final_fix_val"][0], sub.final_fix_val)
    shape = s.subproblem_shape()
    ref_shape = rocket_shape(d)
    assert bytes(shape) == bytes(ref_shape)
    np.testing.assert_array_equal(np.array(shape.e_cost[:]), e_cost)


def batch1(sub: SubArrays):
    return {f: (None if getattr(sub, f) is None else getattr(sub, f)[None]) for f in sub.FIELDS}


def test_power_iteration_random_subproblems(solver15, ptor):
    """test_pipg.cpp:108-119: tracks the dense Gram oracle to 1e-6; plus parity with the port."""
    _, s = solver15
    rng = np.random.default_rng(2025)
    for trial in range(20):
        shape, sub = random_subproblem(rng)
        nx, nu, n = shape.n_x, shape.n_u, shape.nodes
        m = n - 1
        seeds = [rng.uniform(-1, 1, sh) for sh in ((n, nx), (n, nu), (m, nx), (m, nx))]
        rc, sig_ref, trips_ref = ptor.power_iteration(shape, sub, *seeds, 1e-13, 1e-13, 0.05,
                                                      200000, with_trips=True)
        assert rc == 0
        sigma, trips, status = s.power_iteration_custom(shape, batch1(sub),
                                                        *[a[None] for a in seeds], 1e-13, 1e-13,
                                                        0.05, 200000)
        assert status[0] == 0
        assert abs(sigma[0] - sig_ref) <= TOL_SIGMA * sig_ref
        G, H = dense_operator(shape, sub)
        K = np.vstack([G, H])
        lam = np.linalg.eigvalsh(K.T @ K).max()
        assert abs(sigma[0] / 1.05 - lam) <= 1e-6 * lam and sigma[0] > lam
        assert abs(int(trips[0]) - trips_ref) <= max(3, trips_ref // 50)


def test_power_iteration_zero_seed_and_explicit_a_plus(solver15, ptor):
    _, s = solver15
    rng = np.random.default_rng(9)
    shape, sub = random_subproblem(rng, nx=3, nu=2, nodes=4)
    n, m = 4, 3
    z = [np.zeros(sh) for sh in ((1, n, 3), (1, n, 2), (1, m, 3), (1, m, 3))]
    sigma, trips, status = s.power_iteration_custom(shape, batch1(sub), *z, 1e-12, 1e-12, 0.05, 100)
    assert status[0] == abi.ST_POWER_SEED_ZERO
    # a general A_plus (the reference stores it explicitly so synthetic instances can vary it)
    sub.A_plus = -np.eye(3)[None].repeat(m, 0) + 0.1 * rng.uniform(-1, 1, (m, 3, 3))
    seeds = [rng.uniform(-1, 1, sh) for sh in ((n, 3), (n, 2), (m, 3), (m, 3))]
    rc, sig_ref, _ = ptor.power_iteration(shape, sub, *seeds, 1e-13, 1e-13, 0.0, 100000)
    sigma, _, status = s.power_iteration_custom(shape, batch1(sub), *[a[None] for a in seeds],
                                                1e-13, 1e-13, 0.0, 100000)
    assert status[0] == 0 and abs(sigma[0] - sig_ref) <= TOL_SIGMA * sig_ref


@pytest.mark.parametrize("nodes", [15, 50])
def test_power_iteration_zero_seed_on_the_rocket_kernels(ptor, nodes):
    """pipg.hpp:224-225 on every register-resident family: a zero seed next to a regular one in the same
    batch (the latency family finds it inside its first trip when the instance is spread over a
    cluster, in front of the loop when it is not)."""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(nodes)
    d, shape, sub = rocket_subproblem(sc, ptor, 0)
    n, m = d.nodes, d.nodes - 1
    sx, su = ptor.scp_seed(scenario.run_seed(sc.dispersion.seed, 0), n)
    z = np.zeros((m, NX))
    rc, sig_ref, _ = ptor.power_iteration(shape, sub, sx, su, z, z, 1e-12, 1e-12, 0.05, 300, with_trips=True)
    assert rc == 0
    two = {f: (None if getattr(sub, f) is None else np.stack([getattr(sub, f)] * 2)) for f in sub.FIELDS}
    seeds = [np.stack([np.zeros_like(a), a]) for a in (sx, su, z, z)]
    for path in ("fast", "dense", "latency"):
        with Solver(d) as s:
            s.set_solver_path(path)
            sigma, trips, status = s.power_iteration_custom(shape, two, *seeds, 1e-12, 1e-12, 0.05, 300)
        assert status[0] == abi.ST_POWER_SEED_ZERO and sigma[0] == 0.0 and trips[0] == 0, path
        assert status[1] == 0 and abs(sigma[1] - sig_ref) <= TOL_SIGMA * sig_ref, path


def ws_dict(ws: Workspace):
    return {f: getattr(ws, f)[None].copy() for f in ws.FIELDS}


def test_pipg_matches_oracle_at_fixed_iteration_counts(solver15, ptor):
    """test_pipg.cpp:279-314 style: identical iterates (primal and dual) at 1/10/100 iterations."""
    _, s = solver15
    rng = np.random.default_rng(5150)
    for trial in range(6):
        shape, sub = random_subproblem(rng)
        if trial == 5:
            m = shape.nodes - 1
            sub.A_plus = -np.eye(shape.n_x)[None].repeat(m, 0) + 0.05 * rng.uniform(
                -1, 1, (m, shape.n_x, shape.n_x))
        nx, nu, n = shape.n_x, shape.n_u, shape.nodes
        m = n - 1
        seeds = [rng.uniform(-1, 1, sh) for sh in ((n, nx), (n, nu), (m, nx), (m, nx))]
        _, sigma, _ = ptor.power_iteration(shape, sub, *seeds, 1e-13, 1e-13, 0.05, 200000)
        for iters in (1, 10, 100):
            cfg = abi.PipgConfig(omega=20.0, rho=1.6, j_max=iters, j_check=iters + 1,
                                 eps_abs=0.0, eps_rel=0.0, eps_buff=0.05)
            ref = Workspace(nx, nu, n)
            rc, it_ref, conv_ref, _ = ptor.pipg(shape, sub, cfg, sigma, ref)
            assert rc == 0 and it_ref == iters
            ws = ws_dict(Workspace(nx, nu, n))
            it, conv, status, _ = s.pipg_custom(shape, batch1(sub), cfg, [sigma], ws)
            assert status[0] == 0 and it[0] == iters and not conv[0]
            for f in ref.FIELDS:
                assert np.abs(ws[f][0] - getattr(ref, f)).max() < 1e-10, (trial, iters, f)
            # invariants of test_pipg.cpp:227-248
            assert (ws["vc_pos"] >= 0).all() and (ws["vc_neg"] >= 0).all()
            assert (ws["relax_dual"] >= 0).all()
            for i in range(shape.n_init_fix):
                assert ws["x"][0, 0, shape.init_fix_idx[i]] == sub.init_fix_val[i]
            for i in range(shape.n_final_fix):
                assert ws["x"][0, -1, shape.final_fix_idx[i]] == sub.final_fix_val[i]
            assert (ws["u"][0] >= sub.u_min).all() and (ws["u"][0] <= sub.u_max).all()


def test_pipg_stopping_and_warm_start(solver15, ptor):
    """Converges like the oracle (same iteration count at the same check), and a warm start at
    the solution stops at the first check (test_pipg.cpp:210-225)."""
    _, s = solver15
    rng = np.random.default_rng(77)
    shape, sub = random_subproblem(rng)
    nx, nu, n = shape.n_x, shape.n_u, shape.nodes
    m = n - 1
    seeds = [rng.uniform(-1, 1, sh) for sh in ((n, nx), (n, nu), (m, nx), (m, nx))]
    _, sigma, _ = ptor.power_iteration(shape, sub, *seeds, 1e-13, 1e-13, 0.05, 200000)
    cfg = abi.PipgConfig(omega=20.0, rho=1.6, j_max=60000, j_check=10, eps_abs=1e-12,
                         eps_rel=1e-12, eps_buff=0.05)
    ref = Workspace(nx, nu, n)
    rc, it_ref, conv_ref, _ = ptor.pipg(shape, sub, cfg, sigma, ref)
    ws = ws_dict(Workspace(nx, nu, n))
    it, conv, status, _ = s.pipg_custom(shape, batch1(sub), cfg, [sigma], ws)
    assert conv[0] == conv_ref and conv[0]
    assert abs(int(it[0]) - it_ref) <= 20
    for f in ref.FIELDS:
        assert np.abs(ws[f][0] - getattr(ref, f)).max() < 1e-9
    cfg2 = abi.PipgConfig(omega=20.0, rho=1.6, j_max=5000, j_check=25, eps_abs=1e-9,
                          eps_rel=1e-9, eps_buff=0.05)
    it, conv, status, _ = s.pipg_custom(shape, batch1(sub), cfg2, [sigma], ws)
    assert conv[0] and it[0] == 25


def test_pipg_divergence_is_reported_per_instance(solver15, ptor):
    """test_pipg.cpp:402-422: a wildly underestimated sigma diverges; one bad instance in a
    batch does not disturb its neighbour."""
    _, s = solver15
    rng = np.random.default_rng(42)
    shape, sub = random_subproblem(rng)
    nx, nu, n = shape.n_x, shape.n_u, shape.nodes
    cfg = abi.PipgConfig(omega=1e8, rho=1.6, j_max=20000, j_check=5, eps_abs=1e-11,
                         eps_rel=1e-11, eps_buff=0.05)
    ref = Workspace(nx, nu, n)
    ref.x[:] = 0.5
    rc, _, _, fail_ref = ptor.pipg(shape, sub, cfg, 1e-16, ref)
    ws = Workspace(nx, nu, n)
    ws.x[:] = 0.5
    wsd = ws_dict(ws)
    it, conv, status, fail = s.pipg_custom(shape, batch1(sub), cfg, [1e-16], wsd)
    assert status[0] == rc
    if rc == abi.ST_SOLVER_DIVERGED:
        assert fail[0] == fail_ref
        np.testing.assert_array_equal(wsd["x"][0], ws.x)  # workspace untouched on divergence


def rocket_subproblem(sc, ptor, run_id=0):
    d = sc.problem_desc()
    init = scenario.disperse(sc, run_id)
    x, u = scenario.initial_guess(sc, init)
    rc, blocks = ptor.linearize_all(d, x, u)
    assert rc == 0
    rc, sub, _ = ptor.assemble(d, init, x, u, blocks)
    assert rc == 0
    return d, rocket_shape(d), sub


def test_pipg_rocket_2000_iterations(solver15, ptor):
    """BASELINE config 3 at the default node count: fixed 2000 iterations, sigma injected from
    the CPU power iteration, cold start, stop test disabled."""
    sc, s = solver15
    d, shape, sub = rocket_subproblem(sc, ptor, 2)
    n, m = d.nodes, d.nodes - 1
    sx, su = ptor.scp_seed(scenario.run_seed(sc.dispersion.seed, 2), n)
    z = np.zeros((m, NX))
    rc, sigma, trips_ref = ptor.power_iteration(shape, sub, sx, su, z, z, 1e-12, 1e-12, 0.05,
                                                10000, with_trips=True)
    assert rc == 0
    sig_gpu, trips, status = s.power_iteration_custom(shape, batch1(sub), sx[None], su[None],
                                                      z[None], z[None], 1e-12, 1e-12, 0.05, 10000)
    assert status[0] == 0 and abs(sig_gpu[0] - sigma) <= TOL_SIGMA * sigma
    assert abs(int(trips[0]) - trips_ref) <= max(3, trips_ref // 50)
    cfg = abi.PipgConfig(omega=100.0, rho=1.6, j_max=2000, j_check=2001, eps_abs=1e-11,
                         eps_rel=1e-11, eps_buff=0.05)
    ref = Workspace(NX, NU, n)
    rc, it_ref, _, _ = ptor.pipg(shape, sub, cfg, sigma, ref)
    assert rc == 0 and it_ref == 2000
    ws = ws_dict(Workspace(NX, NU, n))
    it, conv, status, _ = s.pipg_custom(shape, batch1(sub), cfg, [sigma], ws)
    assert status[0] == 0 and it[0] == 2000
    for f in ref.FIELDS:
        assert np.abs(ws[f][0] - getattr(ref, f)).max() <= TOL_ITER, f


@pytest.mark.parametrize("nodes", [50, 100])
def test_pipg_rocket_stopping_and_divergence_on_the_column_sparse_kernels(ptor, nodes):
    """stopping_custom and the divergence test (pipg.hpp:307-326, 475-487) on the rocket-shaped
    subproblem: the column-sparse kernel with one CTA per instance at N=50; a 2-CTA cluster at
    N=100 (by default the dense cluster PIPG kernel, with PTOPT_CS_CLUSTER=3 the column-sparse one),
    where the maxima of the two halves are combined between cluster barriers and both CTAs
    have to take the same verdict.  (a) loose tolerances: the solve stops early at the oracle's
    iteration; (b) a wildly underestimated sigma diverges: status, iteration index as the oracle
    reports them, workspace untouched; the neighbour instance in the batch is not disturbed."""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(nodes)
    d, shape, sub = rocket_subproblem(sc, ptor, 1)
    n, m = d.nodes, d.nodes - 1
    sx, su = ptor.scp_seed(scenario.run_seed(sc.dispersion.seed, 1), n)
    z = np.zeros((m, NX))
    rc, sigma, _ = ptor.power_iteration(shape, sub, sx, su, z, z, 1e-12, 1e-12, 0.05, 2000, with_trips=True)
    assert rc == 0
    with Solver(d) as s:
        s.set_solver_path("fast")
        # (a) early stop
        cfg = abi.PipgConfig(omega=100.0, rho=1.6, j_max=4000, j_check=5, eps_abs=2e-3, eps_rel=2e-3,
                             eps_buff=0.05)
        ref = Workspace(NX, NU, n)
        rc, it_ref, conv_ref, _ = ptor.pipg(shape, sub, cfg, sigma, ref)
        assert rc == 0 and conv_ref and it_ref < 4000
        ws = ws_dict(Workspace(NX, NU, n))
        it, conv, status, _ = s.pipg_custom(shape, batch1(sub), cfg, [sigma], ws)
        assert status[0] == 0 and conv[0] == 1 and it[0] == it_ref
        for f in ref.FIELDS:
            assert np.abs(ws[f][0] - getattr(ref, f)).max() <= TOL_ITER, f
        # (b) divergence in the first instance of a batch of two
        bad = abi.PipgConfig(omega=1e8, rho=1.6, j_max=20000, j_check=5, eps_abs=1e-11, eps_rel=1e-11,
                             eps_buff=0.05)
        ref_bad, ref_ok = Workspace(NX, NU, n), Workspace(NX, NU, n)
        ref_bad.x[:] = 0.5
        ref_ok.x[:] = 0.5
        rc_bad, _, _, fail_ref = ptor.pipg(shape, sub, bad, 1e-16, ref_bad)
        rc_ok, it_ok, conv_ok, _ = ptor.pipg(shape, sub, bad, sigma, ref_ok)
        assert rc_bad == abi.ST_SOLVER_DIVERGED
        start = Workspace(NX, NU, n)
        start.x[:] = 0.5
        ws2 = {f: np.concatenate([v, v]) for f, v in ws_dict(start).items()}
        two = {f: (None if getattr(sub, f) is None else np.stack([getattr(sub, f)] * 2)) for f in sub.FIELDS}
        it, conv, status, fail = s.pipg_custom(shape, two, bad, [1e-16, sigma], ws2)
        assert status[0] == abi.ST_SOLVER_DIVERGED and fail[0] == fail_ref
        np.testing.assert_array_equal(ws2["x"][0], start.x)  # workspace untouched on divergence
        assert status[1] == rc_ok and it[1] == it_ok and conv[1] == conv_ok
        if rc_ok == 0:
            for f in ref_ok.FIELDS:
                assert np.abs(ws2[f][1] - getattr(ref_ok, f)).max() <= TOL_ITER * max(1.0, np.abs(getattr(ref_ok, f)).max()), f


@pytest.mark.parametrize("nodes,where", [(15, 3), (100, 3), (100, 80)])
def test_column_sparse_kernels_leave_foreign_operators_to_the_dense_ones(ptor, nodes, where):
    """The column-sparse kernels check the zero pattern of every instance while they load it.  A
    batch of three rocket subproblems whose middle one carries an entry outside the pattern (rate
    row, position column: never produced by the model) and whose last one a NaN there: under
    'fast' the first instance is solved by the column-sparse kernels, the other two by the dense
    kernels behind them -- all three as the CPU oracle solves them.  At N=100 an instance is shared
    by a cluster of two CTAs and the foreign entry sits in the half of rank 0 (interval 3) or of
    rank 1 (interval 80): the CTA that does not see it has to leave with its partner."""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(nodes)
    d, shape, sub = rocket_subproblem(sc, ptor, 1)
    n, m = d.nodes, d.nodes - 1
    subs = [sub]
    for bad in (0.37, np.nan):
        other = SubArrays(**{f: (None if getattr(sub, f) is None else getattr(sub, f).copy())
                             for f in sub.FIELDS})
        other.A_minus[where, 11, 2] = bad
        subs.append(other)

    def stack(items):
        return {f: (None if getattr(items[0], f) is None else np.stack([getattr(x, f) for x in items]))
                for f in sub.FIELDS}

    sx, su = ptor.scp_seed(scenario.run_seed(sc.dispersion.seed, 1), n)
    z = np.zeros((m, NX))
    cfg = abi.PipgConfig(omega=100.0, rho=1.6, j_max=300, j_check=10, eps_abs=1e-11,
                         eps_rel=1e-11, eps_buff=0.05)
    with Solver(d) as s:
        s.set_solver_path("fast")
        sig, trips, status = s.power_iteration_custom(shape, stack(subs), np.stack([sx] * 3),
                                                      np.stack([su] * 3), np.stack([z] * 3),
                                                      np.stack([z] * 3), 1e-12, 1e-12, 0.05, 400)
        sig_ref = []
        for b in range(2):
            rc, sigma, _ = ptor.power_iteration(shape, subs[b], sx, su, z, z, 1e-12, 1e-12, 0.05, 400,
                                                with_trips=True)
            assert rc == 0 and status[b] == 0
            assert abs(sig[b] - sigma) <= TOL_SIGMA * sigma
            sig_ref.append(sigma)
        assert sig_ref[0] != sig_ref[1]
        assert not np.isfinite(sig[2])
        ws = {f: np.concatenate([v, v]) for f, v in ws_dict(Workspace(NX, NU, n)).items()}
        it, conv, status, _ = s.pipg_custom(shape, stack(subs[:2]), cfg, sig_ref, ws)
        for b in range(2):
            ref = Workspace(NX, NU, n)
            rc, it_ref, _, _ = ptor.pipg(shape, subs[b], cfg, sig_ref[b], ref)
            assert rc == 0 and status[b] == 0 and it[b] == it_ref
            for f in ref.FIELDS:
                assert np.abs(ws[f][b] - getattr(ref, f)).max() <= TOL_ITER, (b, f)


def test_scp_solve_general_vehicle_fills_the_whole_pattern(ptor):
    """The default vehicle (diagonal inertia, thrust lever along the body x axis) leaves entries of
    the structural pattern zero (tests/test_block_structure.py); a vehicle with a full inertia matrix
    and an oblique lever arm does not.  The pattern is parameter-independent, so the column-sparse
    kernels take these instances too, and the solves agree with the oracle on both families."""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(20)
    sc.inertia = (0.1, 0.01, -0.02, 0.01, 0.25, 0.015, -0.02, 0.015, 0.22)
    sc.r_thrust = (-0.5, 0.03, -0.02)
    sc.max_iters, sc.pipg_j_max, sc.power_j_max = 3, 250, 300
    d = sc.problem_desc()
    batch = scenario.make_batch(sc, [0, 5, 9])
    refs = [ptor.scp_solve(d, batch["init_state"][b], batch["x_guess"][b], batch["u_guess"][b],
                           int(batch["rng_seed"][b]), with_trips=True) for b in range(3)]
    rc, blocks = ptor.linearize_all(d, batch["x_guess"][0], batch["u_guess"][0])
    assert rc == 0 and np.abs(blocks["Bm"][:, 11, 1]).max() > 0  # a torque row reached by a thrust column the default vehicle leaves at zero
    for path in ("fast", "dense"):
        with Solver(d) as s:
            s.set_solver_path(path)
            out = s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"], batch["rng_seed"])
        for b, (rc, ref) in enumerate(refs):
            assert rc == 0
            check_scp_against_oracle(sc, out, b, ref, ref["power_trips"])


def check_scp_against_oracle(sc, out, b, ref, trips_ref=None):
    assert out["status"][b] == 0
    assert out["scp_iterations"][b] == ref["scp_iterations"]
    assert bool(out["converged"][b]) == ref["converged"]
    k = ref["scp_iterations"]
    assert np.abs(out["x"][b] - ref["x"]).max() <= TOL_ITER
    assert np.abs(out["u"][b] - ref["u"]).max() <= TOL_ITER
    h, hr = out["history"][b][:k], ref["history"][:k]
    np.testing.assert_array_equal(h[:, 3], hr[:, 3])                       # pipg_iterations
    assert np.abs(h[:, 4] / hr[:, 4] - 1.0).max() <= 1e-8                  # sigma
    assert np.abs(h[:, 0] - hr[:, 0]).max() <= TOL_ITER                    # defect_inf
    assert np.abs(h[:, 1] - hr[:, 1]).max() <= TOL_ITER                    # step_inf
    assert np.abs(h[:, 2] - hr[:, 2]).max() <= 1e-6 * np.abs(hr[:, 2]).max()  # penalized cost
    assert abs(out["final_defect_inf"][b] - ref["final_defect_inf"]) <= TOL_ITER
    assert (out["history"][b][k:] == 0).all()
    if trips_ref is not None:
        t = out["power_trips"][b][:k]
        assert (np.abs(t - trips_ref[:k]) <= np.maximum(5, trips_ref[:k] // 20)).all(), (t, trips_ref[:k])


def test_scp_solve_default_scenario_full_budget(solver15, ptor):
    """BASELINE config 1: the shipped N=15 scenario, full 25 x 2500 budget, nominal instance +
    two dispersed ones in one batch."""
    sc, s = solver15
    d = sc.problem_desc()
    nominal = np.array(sc.initial_state)
    xg, ug = scenario.initial_guess(sc, nominal)
    batch = scenario.make_batch(sc, [0, 1])
    init = np.concatenate([nominal[None], batch["init_state"]])
    x0 = np.concatenate([xg[None], batch["x_guess"]])
    u0 = np.concatenate([ug[None], batch["u_guess"]])
    seeds = np.concatenate([[sc.dispersion.seed], batch["rng_seed"]]).astype(np.uint64)
    out = s.scp_solve(init, x0, u0, seeds)
    for b in range(3):
        rc, ref = ptor.scp_solve(d, init[b], x0[b], u0[b], int(seeds[b]), with_trips=True)
        assert rc == 0
        check_scp_against_oracle(sc, out, b, ref, ref["power_trips"])
    # spot value of SURVEY.md 6.3-4 for the nominal instance
    assert abs(out["x"][0, -1, 0] - 1.416480459) < 1e-6


@pytest.mark.parametrize("path", ["fast", "dense", "latency"])
def test_scp_solve_reduced_budget_batch(ptor, path):
    """Many dispersed instances with a reduced iteration budget (fast on the CPU oracle), one
    of them poisoned so that the per-instance failure path is exercised inside the loop."""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(12)
    sc.max_iters = 4
    sc.pipg_j_max = 300
    sc.power_j_max = 400
    d = sc.problem_desc()
    B = 10
    batch = scenario.make_batch(sc, range(B))
    batch["u_guess"][4, 5, 6] = -1.0  # nonpositive dilation at node 5 of instance 4
    with Solver(d) as s:
        s.set_solver_path(path)
        out = s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"],
                          batch["rng_seed"])
        out2 = s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"],
                           batch["rng_seed"])  # graph relaunch: identical results
    for k in ("x", "u", "history", "status", "scp_iterations"):
        np.testing.assert_array_equal(out[k], out2[k])
    for b in range(B):
        rc, ref = ptor.scp_solve(d, batch["init_state"][b], batch["x_guess"][b],
                                 batch["u_guess"][b], int(batch["rng_seed"][b]), with_trips=True)
        if b == 4:
            assert rc == abi.ST_DILATION_NONPOSITIVE and out["status"][b] == rc
            assert out["fail_index"][b] == 4  # interval 4 is the first to touch node 5
            continue
        assert rc == 0
        check_scp_against_oracle(sc, out, b, ref, ref["power_trips"])


@pytest.mark.parametrize("path", ["fast", "dense", "latency"])
def test_scp_solve_n50_two_instances(ptor, path):
    """BASELINE config 4 shape (N=50, all defaults) on two dispersed instances."""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(50)
    d = sc.problem_desc()
    batch = scenario.make_batch(sc, [0, 1])
    with Solver(d) as s:
        s.set_solver_path(path)
        out = s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"],
                          batch["rng_seed"])
        launches = s.launch_count
    # init + 25 x (state pass, column pass, prepare, power, PIPG, update) + the final defect pass;
    # 'fast' launches the column-sparse and the dense kernel of both solver stages
    assert launches == 1 + (8 if path == "fast" else 6) * 25 + 3
    spec = sc.dispersion
    wall, rec, xr, ur = ptor.run_batch(d, sc.initial_state, spec.r_low, spec.r_high, spec.seed, 2,
                                       2, 8, keep=True)
    for b in range(2):
        assert rec[b, 7] == 0
        assert out["scp_iterations"][b] == rec[b, 2] and bool(out["converged"][b]) == bool(rec[b, 1])
        assert np.abs(out["x"][b] - xr[b]).max() <= TOL_ITER
        assert np.abs(out["u"][b] - ur[b]).max() <= TOL_ITER
        assert abs(out["final_defect_inf"][b] - rec[b, 4]) <= TOL_ITER
    # sigma history spot values of SURVEY.md 6.3-4 are for the nominal instance; here we only
    # require the first power iteration to need thousands of trips as the survey observed
    assert out["power_trips"][0, 0] > 1000


# ---------------------------------------------------------------- Monte Carlo harness
def test_generate_batch_is_bit_exact(ptor):
    """disperse + run_seed + initial_guess on the device equal the oracle bit for bit (integer
    draws and separately rounded floating-point operations), incl. a slerp that takes the
    trigonometric branch."""
    from paper_2404_18034_b200.binding import Solver

    for q_init in ((0.0, 0.0, 0.0, 1.0), (0.1, -0.2, 0.05, 0.97)):
        sc = scenario.default_scenario(23)
        q = np.array(q_init) / np.linalg.norm(q_init)
        nominal = np.array(sc.initial_state)
        nominal[7:11] = q
        d = sc.problem_desc()
        spec = sc.dispersion
        first, B = 1000, 37
        with Solver(d) as s:
            out = s.generate_batch(B, first, nominal, spec.r_low, spec.r_high, spec.seed)
        for b in range(B):
            rid = first + b
            init = nominal.copy()
            init[1:4] = ptor.disperse(spec.r_low, spec.r_high, spec.seed, rid)
            rc, xg, ug = ptor.initial_guess(d, init)
            assert rc == 0
            np.testing.assert_array_equal(out["init_state"][b], init)
            np.testing.assert_array_equal(out["x_guess"][b], xg)
            np.testing.assert_array_equal(out["u_guess"][b], ug)
            assert int(out["rng_seed"][b]) == ptor.run_seed(spec.seed, rid)


def test_dense_audit_matches_oracle(solver15, ptor):
    sc, s = solver15
    d = sc.problem_desc()
    rng = np.random.default_rng(99)
    xs, us = [], []
    for rid in range(6):
        init = scenario.disperse(sc, rid)
        x, u = scenario.initial_guess(sc, init)
        if rid >= 3:  # active constraints: the violation integrator grows
            _, x, u = stressed_iterate(sc, rid, rng)
        xs.append(x)
        us.append(u)
    xs, us = np.stack(xs), np.stack(us)
    bad = xs.copy()
    bad_u = us.copy()
    bad_u[2, 7, 6] = -0.5  # nonpositive dilation at node 7: first failing interval is 6
    out = s.dense_violation_audit(bad, bad_u, 16)
    for b in range(6):
        rc, g, ytot, dy = ptor.dense_audit(d, bad[b], bad_u[b], 16)
        if b == 2:
            assert rc == abi.ST_DILATION_NONPOSITIVE and out["status"][b] == rc
            assert out["fail_index"][b] == 6
            continue
        assert rc == 0 and out["status"][b] == 0
        assert abs(out["max_pointwise_g"][b] - g) <= TOL_DISC * max(1.0, abs(g))
        assert np.abs(out["interval_y_increase"][b] - dy).max() <= TOL_DISC * max(1.0, np.abs(dy).max())
        assert abs(out["interval_y_increase"][b].sum() - ytot) <= 1e-9 * max(1.0, abs(ytot))
    # the sample sink of the audit (AuditSample: interval, tau, g[9], g_max), reference order
    smp = s.dense_violation_audit_samples(bad, bad_u, 6)
    assert smp["samples"].shape == (6, d.nodes - 1, 7, 12)
    for b in range(6):
        rc, g, ytot, dy, ref = ptor.dense_audit_samples(d, bad[b], bad_u[b], 6)
        if b == 2:
            assert smp["status"][b] == abi.ST_DILATION_NONPOSITIVE and smp["fail_index"][b] == 6
            got, ref = smp["samples"][b][:6], ref[:6]   # intervals before the failing one are complete
        else:
            assert rc == 0 and smp["status"][b] == 0
            assert abs(smp["max_pointwise_g"][b] - g) <= TOL_DISC * max(1.0, abs(g))
            got = smp["samples"][b]
        assert np.array_equal(got[..., 0], ref[..., 0])                       # interval index
        assert np.abs(got[..., 1] - ref[..., 1]).max() <= 1e-15               # tau
        assert np.abs(got[..., 2:] - ref[..., 2:]).max() <= TOL_DISC * max(1.0, np.abs(ref[..., 2:]).max())


def test_run_batch_records_match_oracle(ptor):
    """mc::run_batch on the device (generation -> scp_solve -> audit -> records) against the
    CPU oracle's run_batch, reduced budget; run ids are offset to exercise first_run_id."""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(12)
    sc.max_iters = 3
    sc.pipg_j_max = 250
    sc.power_j_max = 300
    d = sc.problem_desc()
    spec = sc.dispersion
    B = 9
    with Solver(d) as s:
        rec, xo, uo = s.run_batch(B, 0, sc.initial_state, spec.r_low, spec.r_high, spec.seed,
                                  audit_substeps=16, keep_trajectories=True)
        tail = s.run_batch(4, 5, sc.initial_state, spec.r_low, spec.r_high, spec.seed,
                           audit_substeps=16)
    wall, ref, xr, ur = ptor.run_batch(d, sc.initial_state, spec.r_low, spec.r_high, spec.seed, B,
                                       2, 16, keep=True)
    for b in range(B):
        assert rec["run_id"][b] == b and rec["status"][b] == 0 and ref[b, 7] == 0
        assert rec["converged"][b] == ref[b, 1] and rec["scp_iterations"][b] == ref[b, 2]
        assert abs(rec["propellant_used"][b] - ref[b, 3]) <= TOL_ITER
        assert abs(rec["final_defect_inf"][b] - ref[b, 4]) <= TOL_ITER
        assert abs(rec["max_pointwise_g"][b] - ref[b, 5]) <= TOL_ITER
        assert abs(rec["max_node_y_increase"][b] - ref[b, 6]) <= TOL_ITER
        np.testing.assert_array_equal(rec["initial_position"][b],
                                      ptor.disperse(spec.r_low, spec.r_high, spec.seed, b))
        assert np.abs(xo[b] - xr[b]).max() <= TOL_ITER and np.abs(uo[b] - ur[b]).max() <= TOL_ITER
    # records are pure functions of the run id: a shard starting at run 5 reproduces them
    for f in ("run_id", "converged", "scp_iterations", "propellant_used", "final_defect_inf",
              "max_pointwise_g", "max_node_y_increase"):
        np.testing.assert_array_equal(tail[f], rec[f][5:9])


def test_cuda_path_against_golden_vectors():
    """The CUDA path against the vectors the unmodified reference produced
    (tests/golden/make_golden.py) — no oracle in the loop."""
    from pathlib import Path

    from paper_2404_18034_b200.binding import Solver

    gold = dict(np.load(Path(__file__).resolve().parent / "golden" / "reference_vectors.npz"))
    sc15 = scenario.default_scenario(15)
    with Solver(sc15.problem_desc()) as s:
        B = gold["pi_x"].shape[0]
        out = s.propagate_interval(gold["pi_x"], gold["pi_u"], gold["pi_u1"],
                                   np.full(B, gold["pi_tau"][0]), np.full(B, gold["pi_tau"][1]), 16)
        assert (out["status"] == 0).all()
        for k, g in (("A", "pi_A"), ("Bm", "pi_Bm"), ("Bp", "pi_Bp"), ("w", "pi_w"), ("x_end", "pi_x_end")):
            for b in range(B):
                assert rel_err(out[k][b], gold[g][b]) <= TOL_DISC, (k, b)
    sc = scenario.default_scenario(10)
    spec = sc.dispersion
    init = np.array(sc.initial_state)
    init[1:4] = gold["gen_r"][0]
    with Solver(sc.problem_desc()) as s:
        gen = s.generate_batch(1, 4095, sc.initial_state, spec.r_low, spec.r_high, spec.seed)
        np.testing.assert_array_equal(gen["x_guess"][0], gold["gen_x"][3])
        np.testing.assert_array_equal(gen["u_guess"][0], gold["gen_u"][3])
        assert gen["rng_seed"][0] == gold["gen_seed"][3]
        lin = s.linearize_all(gold["gen_x"][:1], gold["gen_u"][:1])
        for k, g in (("A", "lin_A"), ("Bm", "lin_Bm"), ("Bp", "lin_Bp"), ("w", "lin_w"), ("x_end", "lin_x_end")):
            assert rel_err(lin[k][0], gold[g]) <= TOL_DISC, k
        gb = {k: gold[g][None] for k, g in (("A", "lin_A"), ("Bm", "lin_Bm"), ("Bp", "lin_Bp"),
                                            ("x_end", "lin_x_end"))}
        asm = s.assemble_subproblem(init[None], gold["gen_x"][:1], gold["gen_u"][:1], gb)
        for f, g in (("A_minus", "asm_A_minus"), ("B_minus", "asm_B_minus"), ("B_plus", "asm_B_plus"),
                     ("w", "asm_w"), ("eps_relax", "asm_eps"), ("u_min", "asm_u_min"),
                     ("u_max", "asm_u_max"), ("init_fix_val", "asm_init"), ("final_fix_val", "asm_final")):
            np.testing.assert_array_equal(asm[f][0], gold[g])  # power-of-two scaling: exact
        shape = s.subproblem_shape()
        sub = {f: asm[f] for f in ("A_minus", "B_minus", "B_plus", "w", "eps_relax", "u_min", "u_max",
                                    "init_fix_val", "final_fix_val")}
        z = np.zeros((1, 9, 15))
        sigma, _, st = s.power_iteration_custom(shape, sub, gold["pw_seed_x"][None], gold["pw_seed_u"][None],
                                                z, z, 1e-12, 1e-12, 0.05, 10000)
        assert st[0] == 0 and abs(sigma[0] / float(gold["pw_sigma"]) - 1.0) <= TOL_SIGMA
        cfg = abi.PipgConfig(omega=100.0, rho=1.6, j_max=300, j_check=301, eps_abs=1e-11, eps_rel=1e-11,
                             eps_buff=0.05)
        ws = ws_dict(Workspace(NX, NU, 10))
        it, _, st, _ = s.pipg_custom(shape, sub, cfg, [float(gold["pw_sigma"])], ws)
        assert st[0] == 0 and it[0] == 300
        for f in Workspace.FIELDS:
            assert np.abs(ws[f][0] - gold[f"pipg_{f}"]).max() <= TOL_ITER, f
    sc.max_iters, sc.pipg_j_max, sc.power_j_max = 4, 300, 400
    with Solver(sc.problem_desc()) as s:
        res = s.scp_solve(init[None], gold["gen_x"][:1], gold["gen_u"][:1], gold["gen_seed"][:1])
        assert res["status"][0] == 0 and res["scp_iterations"][0] == gold["scp_meta"][0]
        assert np.abs(res["x"][0] - gold["scp_x"]).max() <= TOL_ITER
        assert np.abs(res["u"][0] - gold["scp_u"]).max() <= TOL_ITER
        np.testing.assert_array_equal(res["history"][0][:, 3], gold["scp_history"][:, 3])
        rec = s.run_batch(3, 0, sc.initial_state, spec.r_low, spec.r_high, spec.seed, audit_substeps=16)
        ref = gold["rb_records"]
        assert (rec["status"] == 0).all() and (ref[:, 7] == 0).all()
        np.testing.assert_array_equal(rec["scp_iterations"], ref[:, 2].astype(np.int32))
        for f, c in (("propellant_used", 3), ("final_defect_inf", 4), ("max_pointwise_g", 5),
                     ("max_node_y_increase", 6)):
            assert np.abs(rec[f] - ref[:, c]).max() <= TOL_ITER, f


# ---------------------------------------------------------------- BASELINE configs at full size
def test_config3_pipg_2000_iterations_batch1024_n50(ptor):
    """BASELINE config 3: fixed 2000 PIPG iterations, batch 1024, N=50.  Subproblems of the first
    8 dispersed instances (CPU-assembled, sigma injected from the CPU power iteration) tiled to
    1024; a subset is compared with the oracle, the rest through invariants: identical inputs
    give identical outputs wherever they sit in the batch, slacks / relaxation dual are
    nonnegative, boundary rows equal their targets, controls stay in the box."""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(50)
    d = sc.problem_desc()
    n, m, base, B = 50, 49, 8, 1024
    subs, sigmas = [], []
    shape = rocket_shape(d)
    for rid in range(base):
        init = scenario.disperse(sc, rid)
        x, u = scenario.initial_guess(sc, init)
        rc, blocks = ptor.linearize_all(d, x, u)
        assert rc == 0
        rc, sub, _ = ptor.assemble(d, init, x, u, blocks)
        assert rc == 0
        sx, su = ptor.scp_seed(scenario.run_seed(sc.dispersion.seed, rid), n)
        z = np.zeros((m, NX))
        rc, sigma, _ = ptor.power_iteration(shape, sub, sx, su, z, z, 1e-12, 1e-12, 0.05, 10000)
        assert rc == 0
        subs.append(sub)
        sigmas.append(sigma)
    tile = np.arange(B) % base
    fields = ("A_minus", "B_minus", "B_plus", "w", "eps_relax", "u_min", "u_max", "init_fix_val",
              "final_fix_val")
    batch = {f: np.stack([getattr(subs[i], f) for i in range(base)])[tile] for f in fields}
    sig = np.array(sigmas)[tile]
    cfg = abi.PipgConfig(omega=100.0, rho=1.6, j_max=2000, j_check=2001, eps_abs=1e-11, eps_rel=1e-11,
                         eps_buff=0.05)
    ws = {f: np.zeros((B,) + getattr(Workspace(NX, NU, n), f).shape) for f in Workspace.FIELDS}
    with Solver(d) as s:
        it, conv, status, _ = s.pipg_custom(s.subproblem_shape(), batch, cfg, sig, ws)
    assert (status == 0).all() and (it == 2000).all() and not conv.any()
    for i in (0, 5):  # oracle parity on two of the base instances (the CPU needs ~0.3 s each)
        ref = Workspace(NX, NU, n)
        rc, it_ref, _, _ = ptor.pipg(shape, subs[i], cfg, sigmas[i], ref)
        assert rc == 0 and it_ref == 2000
        for f in Workspace.FIELDS:
            assert np.abs(ws[f][i] - getattr(ref, f)).max() <= TOL_ITER, f
    for f in Workspace.FIELDS:  # position independence / determinism across the batch
        np.testing.assert_array_equal(ws[f], ws[f][:base][tile])
    assert (ws["vc_pos"] >= 0).all() and (ws["vc_neg"] >= 0).all() and (ws["relax_dual"] >= 0).all()
    np.testing.assert_array_equal(ws["x"][:, 0, :], batch["init_fix_val"])
    fin_idx = [int(i) for i in d.final_fix_idx[: d.n_final_fix]]
    np.testing.assert_array_equal(ws["x"][:, -1, fin_idx], batch["final_fix_val"])
    assert (ws["u"] >= batch["u_min"]).all() and (ws["u"] <= batch["u_max"]).all()


def test_config4_scp_batch4096_n50_properties():
    """BASELINE config 4 shape (batch 4096, N=50) with a reduced iteration budget: the graph
    relaunch is deterministic, every instance's result is independent of where it sits in the
    batch (a permuted batch gives permuted results), all instances finish with status ok and
    unit quaternions, and the history rows past the last iteration are zero."""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(50)
    sc.max_iters, sc.pipg_j_max, sc.power_j_max = 2, 60, 80
    d = sc.problem_desc()
    B, base = 4096, 64
    small = scenario.make_batch(sc, range(base))
    rng = np.random.default_rng(7)
    tile = rng.integers(0, base, B)
    tile[:base] = np.arange(base)
    big = {k: small[k][tile] for k in ("init_state", "x_guess", "u_guess", "rng_seed")}
    with Solver(d) as s:
        out = s.scp_solve(big["init_state"], big["x_guess"], big["u_guess"], big["rng_seed"])
        again = s.scp_solve(big["init_state"], big["x_guess"], big["u_guess"], big["rng_seed"])
    assert (out["status"] == 0).all() and (out["scp_iterations"] == 2).all()
    for k in ("x", "u", "history", "power_trips", "final_defect_inf"):
        np.testing.assert_array_equal(out[k], again[k])
        np.testing.assert_array_equal(out[k], out[k][:base][tile])
    q = out["x"][:, :, 7:11]
    assert np.abs(np.linalg.norm(q, axis=2) - 1.0).max() <= 1e-14
    assert (out["history"][:, :, 3] == 60).all() and (out["power_trips"] > 0).all()


@pytest.mark.parametrize("path", ["fast", "generic", "latency"])
def test_config5_n100_cluster_and_generic_kernels(ptor, path):
    """BASELINE config 5 shape (N=100): above the single-CTA node limit, so each instance is split
    over a two-CTA cluster ('fast': the column-sparse kernels with a copy of the partner's boundary
    node on either side of the cut); the shape-generic kernels serve it too ('generic'), and the
    latency mode spreads it over eight CTAs of 12-13 nodes ('latency').  Reduced
    budget with stopping checks, parity with the oracle on three instances."""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(100)
    sc.max_iters, sc.pipg_j_max, sc.power_j_max = 2, 150, 200
    d = sc.problem_desc()
    batch = scenario.make_batch(sc, [3, 65535, 12])
    with Solver(d) as s:
        s.set_solver_path(path)
        out = s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"], batch["rng_seed"])
    for b in range(3):
        rc, ref = ptor.scp_solve(d, batch["init_state"][b], batch["x_guess"][b], batch["u_guess"][b],
                                 int(batch["rng_seed"][b]), with_trips=True)
        assert rc == 0
        check_scp_against_oracle(sc, out, b, ref, ref["power_trips"])


@pytest.mark.parametrize("nodes", [2, 3, 30, 31, 32, 50, 51, 52, 61, 62, 63, 64, 77, 102, 103])
def test_scp_solve_node_count_edges(ptor, nodes):
    """Node counts at the edges of the register-resident kernels: the minimum grid, the last count
    the column-sparse kernels hold in one warp per role (31) and its neighbours (30; 32: two warps
    per role with a halo lane each), their largest single-CTA count (61) and the first ones they
    split over a two-CTA cluster (62, 63: the copy of the partner's boundary node falls on the
    halo lanes between the two warps of a role; 64), the largest dense single-CTA count (51) and
    the first one the dense kernels split (52), an odd cluster split (77), the largest cluster
    count (102) and the first one that falls back to the shape-generic kernels (103)."""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(nodes)
    sc.max_iters, sc.pipg_j_max, sc.power_j_max = 2, 120, 150
    d = sc.problem_desc()
    batch = scenario.make_batch(sc, [0, 11])
    with Solver(d) as s:
        s.set_solver_path("fast")
        outs = [s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"], batch["rng_seed"])]
    for b in range(2):
        rc, ref = ptor.scp_solve(d, batch["init_state"][b], batch["x_guess"][b], batch["u_guess"][b],
                                 int(batch["rng_seed"][b]), with_trips=True)
        assert rc == 0
        for out in outs:
            check_scp_against_oracle(sc, out, b, ref, ref["power_trips"])


@pytest.mark.parametrize("nodes", [4, 5, 26, 49, 50, 51])
def test_scp_solve_split_path_node_counts(ptor, nodes):
    """The split variant (every instance shared by a 2-CTA cluster of 128-thread CTAs, two CTAs per
    SM): the smallest and largest node counts it accepts (4, 50), odd counts (uneven halves), a
    count whose halves leave idle threads (26), and one above its range (51, runs single-CTA)."""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(nodes)
    sc.max_iters, sc.pipg_j_max, sc.power_j_max = 2, 120, 150
    d = sc.problem_desc()
    batch = scenario.make_batch(sc, [0, 11, 5])
    with Solver(d) as s:
        s.set_solver_path("split")
        out = s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"], batch["rng_seed"])
    for b in range(3):
        rc, ref = ptor.scp_solve(d, batch["init_state"][b], batch["x_guess"][b], batch["u_guess"][b],
                                 int(batch["rng_seed"][b]), with_trips=True)
        assert rc == 0
        check_scp_against_oracle(sc, out, b, ref, ref["power_trips"])


def test_solver_divergence_inside_the_scp_loop(ptor):
    """A spectral estimate cut off after one power-iteration trip is far too small, the step
    sizes are too large and PIPG blows up: the reference throws SolverDiverged at the stopping
    check that first sees a non-finite iterate.  Inside the batched loop every instance stops
    with the same status and iteration index (they differ between instances)."""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(12)
    sc.max_iters, sc.pipg_j_max, sc.power_j_max = 3, 2500, 1
    sc.pipg_eps_buff = 0.0
    d = sc.problem_desc()
    batch = scenario.make_batch(sc, [0, 1])
    refs = []
    for b in range(2):
        rc, ref = ptor.scp_solve(d, batch["init_state"][b], batch["x_guess"][b], batch["u_guess"][b],
                                 int(batch["rng_seed"][b]))
        assert rc == abi.ST_SOLVER_DIVERGED, rc
        refs.append(ref["fail_index"])
    assert refs[0] != refs[1]
    for path in ("fast", "dense", "generic", "split", "latency"):
        with Solver(d) as s:
            s.set_solver_path(path)
            out = s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"], batch["rng_seed"])
        assert (out["status"] == abi.ST_SOLVER_DIVERGED).all()
        assert list(out["fail_index"]) == refs, (out["fail_index"], refs)
        assert (out["scp_iterations"] == 0).all() and not out["converged"].any()


# ------------------------------------------------- full-size configs at their real budgets
def cpu_reference_solves(d, batch, ids):
    """Full SCP solves of batch rows `ids` on the CPU, one host thread per core (ctypes releases
    the GIL).  Uses the unmodified reference compiled in place when it travelled with the repo
    (oracle/_ref, -O3 build), else the plain-C oracle; both are pinned to each other bit for bit
    in their -ffp-contract=off builds (tests/test_oracle_vs_ref.py)."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    from oracle_lib import CpuOracle, ref_available

    cpu = CpuOracle("ptref", fast=True) if ref_available() else CpuOracle("ptor")

    def solve(b):
        return cpu.scp_solve(d, batch["init_state"][b], batch["x_guess"][b], batch["u_guess"][b],
                             int(batch["rng_seed"][b]))

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as pool:
        return dict(zip(ids, pool.map(solve, ids)))


def test_config4_full_budget_batch4096_subset_vs_cpu():
    """BASELINE config 4 as the bench runs it: 4096 dispersed N=50 instances, every default
    (25 SCP iterations x 2500 PIPG iterations, power iteration capped at 10 000 trips).  Run ids
    0..63 plus 64 seeded-random ids of the batch are solved by the CPU reference as well
    (SURVEY.md 8d row 4): final x, u <= 1e-6, history (defect, step, cost, pipg_iterations, sigma
    1e-8), scp_iterations, converged and final_defect_inf equal."""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(50)
    d = sc.problem_desc()
    B = 4096
    batch = scenario.make_batch(sc, range(B))
    with Solver(d) as s:
        out = s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"], batch["rng_seed"])
    assert (out["status"] == 0).all()
    rng = np.random.default_rng(20260810)
    ids = list(range(64)) + sorted(int(i) for i in rng.choice(np.arange(64, B), 64, replace=False))
    refs = cpu_reference_solves(d, batch, ids)
    for b in ids:
        rc, ref = refs[b]
        assert rc == 0, b
        check_scp_against_oracle(sc, out, b, ref)
    q = out["x"][:, :, 7:11]
    assert np.abs(np.linalg.norm(q, axis=2) - 1.0).max() <= 1e-14


@pytest.mark.parametrize("path", ["fast", "latency"])
def test_config5_n100_full_budget_cluster_kernels_vs_cpu(path):
    """BASELINE config 5 at the depth it runs: N=100 on the two-CTA cluster kernels ('fast': column-sparse) and on
    the eight-CTA latency-mode clusters ('latency') with the full budget -- the power iteration
    mostly runs to its 10 000-trip cap, 25 x 2500 PIPG iterations, so the mailbox protocols run
    ~300 000 hand-offs per instance -- six dispersed ids against the CPU reference."""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(100)
    d = sc.problem_desc()
    ids = [0, 1, 2, 4097, 32768, 65535]
    batch = scenario.make_batch(sc, ids)
    with Solver(d) as s:
        s.set_solver_path(path)
        out = s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"], batch["rng_seed"])
    assert (out["power_trips"] == 10000).sum() >= 25  # the mailbox protocol ran at its real depth
    refs = cpu_reference_solves(d, batch, list(range(len(ids))))
    for b in range(len(ids)):
        rc, ref = refs[b]
        assert rc == 0, b
        check_scp_against_oracle(sc, out, b, ref)


def test_scp_converged_early_exit_mixed_batch(solver15, ptor):
    """scp.hpp:294-297: an instance leaves the loop as soon as its defect and last step meet the
    tolerances.  With tolerances loosened to (1e-3, 1.35e-2) and at most 12 iterations the twelve
    dispersed instances of this batch converge after 7, 8, 9, 10 and 12 solves and four never do,
    so the per-instance gating of the batched loop is exercised on every kernel family: iteration
    counts, converged flags, history rows (zero past the exit) and final iterates against the
    oracle."""
    from paper_2404_18034_b200.binding import Solver

    sc0, s0 = solver15
    sc = scenario.default_scenario(15)
    sc.tol_feas, sc.tol_step, sc.max_iters = 1e-3, 1.35e-2, 12
    d = sc.problem_desc()
    batch = scenario.make_batch(sc, range(12))
    with Solver(d) as s:
        s.set_solver_path(s0.solver_path)
        out = s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"], batch["rng_seed"])
    its, conv = [], []
    for b in range(12):
        rc, ref = ptor.scp_solve(d, batch["init_state"][b], batch["x_guess"][b], batch["u_guess"][b],
                                 int(batch["rng_seed"][b]), with_trips=True)
        assert rc == 0
        check_scp_against_oracle(sc, out, b, ref, ref["power_trips"])
        its.append(ref["scp_iterations"])
        conv.append(ref["converged"])
    assert len(set(its)) >= 4 and min(its) < 12          # different exit iterations ...
    assert sum(conv) >= 6 and sum(not c for c in conv) >= 2  # ... and some that never converge
    assert [bool(c) for c in out["converged"]] == conv


def test_run_batch_multi_device_list_is_bit_identical():
    """ptopt_cuda_run_batch_multi (the reference's worker pool, montecarlo.hpp:153-171, with one
    worker per device entry): two and three handles on device 0, each with its own host thread and
    contiguous run-id range, reproduce the single-handle batch bit for bit -- records written into
    their run-id slots, trajectories too; an entry with an empty range is skipped; a bad device
    ordinal fails the call."""
    from paper_2404_18034_b200.binding import PtoptError, Solver, run_batch_multi

    sc = scenario.default_scenario(11)
    sc.max_iters, sc.pipg_j_max, sc.power_j_max, sc.audit_substeps = 3, 150, 200, 8
    d = sc.problem_desc()
    spec = sc.dispersion
    B, first = 9, 40
    with Solver(d) as s:
        rec, x, u = s.run_batch(B, first, sc.initial_state, spec.r_low, spec.r_high, spec.seed,
                                audit_substeps=8, keep_trajectories=True)
    for devices, batch in (([0, 0], B), ([0, 0, 0], B), ([0, 0, 0], 2)):
        rm, xm, um, ms = run_batch_multi(d, devices, batch, first, sc.initial_state, spec.r_low, spec.r_high,
                                         spec.seed, audit_substeps=8, keep_trajectories=True)
        assert rm.tobytes() == rec[:batch].tobytes()
        np.testing.assert_array_equal(xm, x[:batch])
        np.testing.assert_array_equal(um, u[:batch])
        assert len(ms) == len(devices) and (ms > 0).sum() == min(batch, len(devices))
    with pytest.raises(PtoptError):
        run_batch_multi(d, [0, 99], B, first, sc.initial_state, spec.r_low, spec.r_high, spec.seed)


@pytest.mark.parametrize("nodes", [2, 3, 5, 8, 9, 15, 17, 33, 50, 128, 129])
def test_scp_solve_latency_mode_node_counts(ptor, nodes):
    """Latency mode (one instance over a cluster, sixteen threads per node) at the edges of its
    decomposition: clusters of two CTAs (2, 3 nodes), four (5), eight with one node per CTA (8),
    uneven shares (9, 15, 17, 33, 50), the largest supported count (128 = 8 x 16) and the first one
    that falls back to the shape-generic kernels (129)."""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(nodes)
    sc.max_iters, sc.pipg_j_max, sc.power_j_max = 2, 120, 150
    d = sc.problem_desc()
    batch = scenario.make_batch(sc, [0, 11, 5])
    with Solver(d) as s:
        s.set_solver_path("latency")
        out = s.scp_solve(batch["init_state"], batch["x_guess"], batch["u_guess"], batch["rng_seed"])
    for b in range(3):
        rc, ref = ptor.scp_solve(d, batch["init_state"][b], batch["x_guess"][b], batch["u_guess"][b],
                                 int(batch["rng_seed"][b]), with_trips=True)
        assert rc == 0
        check_scp_against_oracle(sc, out, b, ref, ref["power_trips"])


def test_auto_path_selection():
    """AUTO runs the latency-mode kernels when batch x cluster size fits the chip in one wave and the
    throughput kernels otherwise; mc::run_batch always uses the throughput family so that a shard's
    records do not depend on its size.  Detected through bit-identity with the forced paths."""
    from paper_2404_18034_b200.binding import Solver

    sc = scenario.default_scenario(15)
    sc.max_iters, sc.pipg_j_max, sc.power_j_max, sc.audit_substeps = 2, 100, 120, 8
    d = sc.problem_desc()
    spec = sc.dispersion
    B = 200  # more instances than SMs: throughput kernels; the first 3 alone: latency kernels
    batch = scenario.make_batch(sc, range(B))
    args = lambda k: (batch["init_state"][:k], batch["x_guess"][:k], batch["u_guess"][:k], batch["rng_seed"][:k])
    res = {}
    for path in ("auto", "fast", "latency"):
        with Solver(d) as s:
            s.set_solver_path(path)
            res[path, 3] = s.scp_solve(*args(3))["x"]
            res[path, B] = s.scp_solve(*args(B))["x"]
            res[path, "rb"] = s.run_batch(3, 0, sc.initial_state, spec.r_low, spec.r_high, spec.seed,
                                          audit_substeps=8, keep_trajectories=True)[1]
    assert not np.array_equal(res["fast", 3], res["latency", 3])  # the two families round differently
    np.testing.assert_array_equal(res["auto", 3], res["latency", 3])
    np.testing.assert_array_equal(res["auto", B], res["fast", B])
    np.testing.assert_array_equal(res["auto", "rb"], res["fast", "rb"])
    np.testing.assert_array_equal(res["fast", B][:3], res["fast", 3])
    assert np.abs(res["fast", 3] - res["latency", 3]).max() <= TOL_ITER
