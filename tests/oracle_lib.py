"""TEST INFRASTRUCTURE: ctypes access to the CPU oracles.

``CpuOracle("ptor")`` wraps oracle/_build/libptopt_oracle.so (the plain-C
restatement) and ``CpuOracle("ptref")`` wraps oracle/_ref/libptopt_ref.so (the
unmodified reference compiled in place).  Both export the same functions with a
different prefix, so every test can be parametrised over the two.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_2404_18034_b200 import abi

ROOT = Path(__file__).resolve().parent.parent
ORACLE_SO = ROOT / "oracle" / "_build" / "libptopt_oracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libptopt_ref.so"
REF_FAST_SO = ROOT / "oracle" / "_ref" / "libptopt_ref_fast.so"

NX, NU, NXI, NZ, NG = abi.NX, abi.NU, abi.NXI, abi.NZETA, abi.NG


def build_oracle():
    """Compiles the C restatement (and the reference shim when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "oracle"], check=True)
    if Path("/root/reference/proj/include/ptopt").is_dir() and not REF_SO.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "ref"], check=True)


def ref_available() -> bool:
    return REF_SO.exists()


def _p(a):
    """numpy array (or None) -> void pointer."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be contiguous"
    return a.ctypes.data_as(C.c_void_p)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class SubArrays:
    """Owns the numpy arrays behind a ptopt_subproblem_arrays (one instance)."""

    FIELDS = ("A_minus", "A_plus", "B_minus", "B_plus", "w", "eps_relax", "u_min", "u_max",
              "init_fix_val", "final_fix_val")

    def __init__(self, **kw):
        for f in self.FIELDS:
            v = kw.get(f)
            setattr(self, f, None if v is None else f64(v))

    def struct(self) -> abi.SubproblemArrays:
        s = abi.SubproblemArrays()
        for f in self.FIELDS:
            v = getattr(self, f)
            setattr(s, f, None if v is None else v.ctypes.data)
        return s


class Workspace:
    """Owns the arrays behind a ptopt_workspace_arrays (one instance)."""

    FIELDS = ("x", "u", "vc_pos", "vc_neg", "dyn_dual", "relax_dual")

    def __init__(self, nx, nu, nodes):
        m = nodes - 1
        self.x = np.zeros((nodes, nx))
        self.u = np.zeros((nodes, nu))
        self.vc_pos = np.zeros((m, nx))
        self.vc_neg = np.zeros((m, nx))
        self.dyn_dual = np.zeros((m, nx))
        self.relax_dual = np.zeros(m)

    def copy(self):
        w = Workspace.__new__(Workspace)
        for f in self.FIELDS:
            setattr(w, f, getattr(self, f).copy())
        return w

    def struct(self) -> abi.WorkspaceArrays:
        s = abi.WorkspaceArrays()
        for f in self.FIELDS:
            setattr(s, f, getattr(self, f).ctypes.data)
        return s


class CpuOracle:
    def __init__(self, prefix: str = "ptor", fast: bool = False):
        self.prefix = prefix
        if prefix == "ptor":
            path = ORACLE_SO
            if not path.exists():
                build_oracle()
        elif prefix == "ptref":
            path = REF_FAST_SO if fast else REF_SO
        else:
            raise ValueError(prefix)
        if not path.exists():
            raise FileNotFoundError(path)
        self.path = path
        self.lib = C.CDLL(str(path))
        self._f("run_seed").restype = C.c_uint64
        self._f("run_batch").restype = C.c_double
        self._f("step_sizes").restype = C.c_double
        self._f("pow2_near").restype = C.c_double

    def _f(self, name):
        return getattr(self.lib, f"{self.prefix}_{name}")

    # ---- model layer
    def model_eval(self, vp, xi, zeta, jac=True):
        xi, zeta = f64(xi), f64(zeta)
        F, g = np.zeros(NXI), np.zeros(NG)
        Fx, Fz = np.zeros((NXI, NXI)), np.zeros((NXI, NZ))
        gx, gz = np.zeros((NG, NXI)), np.zeros((NG, NZ))
        rc = self._f("model_eval")(C.byref(vp), _p(xi), _p(zeta), _p(F), _p(g),
                                    _p(Fx) if jac else None, _p(Fz), _p(gx), _p(gz))
        return rc, dict(F=F, g=g, dF_dxi=Fx, dF_dzeta=Fz, dg_dxi=gx, dg_dzeta=gz)

    def aug_eval(self, vp, x, u):
        x, u = f64(x), f64(u)
        f, A, B = np.zeros(NX), np.zeros((NX, NX)), np.zeros((NX, NU))
        rc = self._f("aug_eval")(C.byref(vp), _p(x), _p(u), _p(f), _p(A), _p(B))
        return rc, f, A, B

    def aug_eval_test_model(self, model_id, params, x, u):
        x, u, params = f64(x), f64(u), f64(params)
        nx, nu = len(x), len(u)
        f, A, B = np.zeros(nx), np.zeros((nx, nx)), np.zeros((nx, nu))
        rc = self._f("aug_eval_test_model")(C.c_int(model_id), _p(params), _p(x), _p(u), _p(f),
                                             _p(A), _p(B))
        return rc, f, A, B

    # ---- discretizer
    def propagate_interval(self, vp, xk, uk, uk1, tau_k, tau_k1, steps, interval_index=0):
        xk, uk, uk1 = f64(xk), f64(uk), f64(uk1)
        out = dict(A=np.zeros((NX, NX)), Bm=np.zeros((NX, NU)), Bp=np.zeros((NX, NU)),
                   w=np.zeros(NX), x_end=np.zeros(NX))
        fail = C.c_int(-1)
        rc = self._f("propagate_interval")(
            C.byref(vp), _p(xk), _p(uk), _p(uk1), C.c_double(tau_k), C.c_double(tau_k1),
            C.c_int(steps), C.c_int(interval_index), _p(out["A"]), _p(out["Bm"]), _p(out["Bp"]),
            _p(out["w"]), _p(out["x_end"]), C.byref(fail))
        out["fail_index"] = fail.value
        return rc, out

    def propagate_test_model(self, model_id, params, xk, uk, uk1, tau_k, tau_k1, steps,
                             interval_index=0):
        xk, uk, uk1, params = f64(xk), f64(uk), f64(uk1), f64(params)
        nx, nu = len(xk), len(uk)
        out = dict(A=np.zeros((nx, nx)), Bm=np.zeros((nx, nu)), Bp=np.zeros((nx, nu)),
                   w=np.zeros(nx), x_end=np.zeros(nx))
        fail = C.c_int(-1)
        rc = self._f("propagate_test_model")(
            C.c_int(model_id), _p(params), _p(xk), _p(uk), _p(uk1), C.c_double(tau_k),
            C.c_double(tau_k1), C.c_int(steps), C.c_int(interval_index), _p(out["A"]),
            _p(out["Bm"]), _p(out["Bp"]), _p(out["w"]), _p(out["x_end"]), C.byref(fail))
        out["fail_index"] = fail.value
        return rc, out

    def linearize_all(self, desc, x, u, tau=None, workers=1):
        n, m = desc.nodes, desc.nodes - 1
        x, u = f64(x), f64(u)
        tau = None if tau is None else f64(tau)
        out = dict(A=np.zeros((m, NX, NX)), Bm=np.zeros((m, NX, NU)), Bp=np.zeros((m, NX, NU)),
                   w=np.zeros((m, NX)), x_end=np.zeros((m, NX)))
        fail = C.c_int(-1)
        rc = self._f("linearize_all")(C.byref(desc), _p(tau), _p(x), _p(u), C.c_int(workers),
                                       _p(out["A"]), _p(out["Bm"]), _p(out["Bp"]), _p(out["w"]),
                                       _p(out["x_end"]), C.byref(fail))
        out["fail_index"] = fail.value
        return rc, out

    def dense_audit(self, desc, x, u, substeps, tau=None):
        x, u = f64(x), f64(u)
        tau = None if tau is None else f64(tau)
        gmax, ytot = C.c_double(0), C.c_double(0)
        dy = np.zeros(desc.nodes - 1)
        rc = self._f("dense_audit")(C.byref(desc), _p(tau), _p(x), _p(u), C.c_int(substeps),
                                     C.byref(gmax), C.byref(ytot), _p(dy))
        return rc, gmax.value, ytot.value, dy

    def dense_audit_samples(self, desc, x, u, substeps, tau=None):
        """dense_violation_audit with its sample sink: samples [M][substeps+1][12] =
        {interval, tau, g[9], g_max}."""
        x, u = f64(x), f64(u)
        tau = None if tau is None else f64(tau)
        gmax, ytot = C.c_double(0), C.c_double(0)
        dy = np.zeros(desc.nodes - 1)
        samples = np.zeros((desc.nodes - 1, substeps + 1, 12))
        rc = self._f("dense_audit_samples")(C.byref(desc), _p(tau), _p(x), _p(u), C.c_int(substeps),
                                             C.byref(gmax), C.byref(ytot), _p(dy), _p(samples))
        return rc, gmax.value, ytot.value, dy, samples

    # ---- SCP glue
    def assemble(self, desc, init_state, x, u, blocks, tau=None, with_a_plus=False):
        n, m = desc.nodes, desc.nodes - 1
        nf = desc.n_final_fix
        init_state, x, u = f64(init_state), f64(x), f64(u)
        sub = SubArrays(A_minus=np.zeros((m, NX, NX)),
                        A_plus=np.zeros((m, NX, NX)) if with_a_plus else None,
                        B_minus=np.zeros((m, NX, NU)), B_plus=np.zeros((m, NX, NU)),
                        w=np.zeros((m, NX)), eps_relax=np.zeros(m), u_min=np.zeros((n, NU)),
                        u_max=np.zeros((n, NU)), init_fix_val=np.zeros(NX),
                        final_fix_val=np.zeros(max(nf, 1)))
        e_cost = np.zeros(NX)
        rc = self._f("assemble")(
            C.byref(desc), _p(None if tau is None else f64(tau)), _p(init_state), _p(x), _p(u),
            _p(f64(blocks["A"])), _p(f64(blocks["Bm"])), _p(f64(blocks["Bp"])),
            _p(f64(blocks["x_end"])), _p(sub.A_minus), _p(sub.A_plus), _p(sub.B_minus),
            _p(sub.B_plus), _p(sub.w), _p(sub.eps_relax), _p(sub.u_min), _p(sub.u_max),
            _p(sub.init_fix_val), _p(sub.final_fix_val), _p(e_cost))
        return rc, sub, e_cost

    def scp_seed(self, rng_seed, nodes):
        sx, su = np.zeros((nodes, NX)), np.zeros((nodes, NU))
        self._f("scp_seed")(C.c_uint64(int(rng_seed)), C.c_int(nodes), _p(sx), _p(su))
        return sx, su

    def scp_solve(self, desc, init_state, x_guess, u_guess, rng_seed, tau=None,
                  with_trips=False):
        n = desc.nodes
        init_state, x_guess, u_guess = f64(init_state), f64(x_guess), f64(u_guess)
        xo, uo = np.zeros((n, NX)), np.zeros((n, NU))
        iters, conv, fail = C.c_int(0), C.c_int(0), C.c_int(-1)
        fdef = C.c_double(0)
        hist = np.zeros((desc.max_iters, abi.HISTORY_FIELDS))
        trips = np.zeros(desc.max_iters, dtype=np.int32)
        tau_p = _p(None if tau is None else f64(tau))
        if with_trips and self.prefix == "ptor":
            rc = self._f("scp_solve_ex")(
                C.byref(desc), tau_p, _p(init_state), _p(x_guess), _p(u_guess),
                C.c_uint64(int(rng_seed)), _p(xo), _p(uo), C.byref(iters), C.byref(conv),
                C.byref(fdef), _p(hist), _p(trips), C.byref(fail))
        else:
            rc = self._f("scp_solve")(
                C.byref(desc), tau_p, _p(init_state), _p(x_guess), _p(u_guess),
                C.c_uint64(int(rng_seed)), _p(xo), _p(uo), C.byref(iters), C.byref(conv),
                C.byref(fdef), _p(hist), C.byref(fail))
        return rc, dict(x=xo, u=uo, scp_iterations=iters.value, converged=bool(conv.value),
                        final_defect_inf=fdef.value, history=hist, power_trips=trips,
                        fail_index=fail.value)

    # ---- PIPG
    def power_iteration(self, shape, sub, seed_x, seed_u, seed_vcp, seed_vcn, eps_abs, eps_rel,
                        eps_buff, j_max, with_trips=False):
        sigma = C.c_double(0)
        trips = C.c_int(0)
        s = sub.struct()
        args = [C.byref(shape), C.byref(s), _p(f64(seed_x)), _p(f64(seed_u)), _p(f64(seed_vcp)),
                _p(f64(seed_vcn)), C.c_double(eps_abs), C.c_double(eps_rel), C.c_double(eps_buff),
                C.c_int(j_max), C.byref(sigma)]
        if with_trips and self.prefix == "ptor":
            rc = self._f("power_iteration_ex")(*args, C.byref(trips))
        else:
            rc = self._f("power_iteration")(*args)
        return rc, sigma.value, trips.value

    def pipg(self, shape, sub, cfg, sigma, ws):
        iters, conv, fail = C.c_int(0), C.c_int(0), C.c_int(-1)
        s, w = sub.struct(), ws.struct()
        rc = self._f("pipg")(C.byref(shape), C.byref(s), C.byref(cfg), C.c_double(sigma),
                              C.byref(w), C.byref(iters), C.byref(conv), C.byref(fail))
        return rc, iters.value, bool(conv.value), fail.value

    def pipg_generic(self, shape, sub, cfg, sigma):
        assert self.prefix == "ptref"
        nx, nu, n = shape.n_x, shape.n_u, shape.nodes
        m = n - 1
        dim = n * (nx + nu) + 2 * m * nx
        z, eq, ineq = np.zeros(dim), np.zeros(m * nx), np.zeros(m)
        iters, conv = C.c_int(0), C.c_int(0)
        s = sub.struct()
        rc = self.lib.ptref_pipg_generic(C.byref(shape), C.byref(s), C.byref(cfg),
                                         C.c_double(sigma), _p(z), _p(eq), _p(ineq),
                                         C.byref(iters), C.byref(conv))
        return rc, z, eq, ineq, iters.value, bool(conv.value)

    def step_sizes(self, lam, omega, sigma):
        beta = C.c_double(0)
        alpha = self._f("step_sizes")(C.c_double(lam), C.c_double(omega), C.c_double(sigma),
                                       C.byref(beta))
        return alpha, beta.value

    # ---- instance generation
    def run_seed(self, batch_seed, run_id):
        return int(self._f("run_seed")(C.c_uint64(int(batch_seed)), C.c_int(run_id)))

    def disperse(self, r_low, r_high, seed, run_id):
        out = np.zeros(3)
        self._f("disperse")(_p(f64(r_low)), _p(f64(r_high)), C.c_uint64(int(seed)),
                             C.c_int(run_id), _p(out))
        return out

    def initial_guess(self, desc, init_state, tau=None):
        n = desc.nodes
        x, u = np.zeros((n, NX)), np.zeros((n, NU))
        rc = self._f("initial_guess")(C.byref(desc), _p(None if tau is None else f64(tau)),
                                       _p(f64(init_state)), _p(x), _p(u))
        return rc, x, u

    def pow2_near(self, v):
        return self._f("pow2_near")(C.c_double(v))

    def run_batch(self, desc, nominal_init, r_low, r_high, seed, batch, workers,
                  audit_substeps=64, keep=False, tau=None):
        n = desc.nodes
        rec = np.zeros((batch, 8))
        xo = np.zeros((batch, n, NX)) if keep else None
        uo = np.zeros((batch, n, NU)) if keep else None
        wall = self._f("run_batch")(
            C.byref(desc), _p(None if tau is None else f64(tau)), _p(f64(nominal_init)),
            _p(f64(r_low)), _p(f64(r_high)), C.c_uint64(int(seed)), C.c_int(batch),
            C.c_int(workers), C.c_int(audit_substeps), _p(rec), _p(xo), _p(uo))
        return wall, rec, xo, uo


def make_shape(nx, nu, nodes, init_fix_idx=(), final_fix_idx=(), e_y=None, e_cost=None,
               w_cost=0.0, w_prox=1.0, w_ep=1.0) -> abi.SubproblemShape:
    s = abi.SubproblemShape()
    s.n_x, s.n_u, s.nodes = nx, nu, nodes
    s.n_init_fix, s.n_final_fix = len(init_fix_idx), len(final_fix_idx)
    for i, v in enumerate(init_fix_idx):
        s.init_fix_idx[i] = v
    for i, v in enumerate(final_fix_idx):
        s.final_fix_idx[i] = v
    if e_y is not None:
        for i, v in enumerate(e_y):
            s.e_y[i] = v
    if e_cost is not None:
        for i, v in enumerate(e_cost):
            s.e_cost[i] = v
    s.w_cost, s.w_prox, s.w_ep = w_cost, w_prox, w_ep
    return s


def rocket_shape(desc) -> abi.SubproblemShape:
    """Shape assemble_subproblem yields for the rocket problem (scp.hpp:160-215)."""
    return make_shape(NX, NU, desc.nodes, init_fix_idx=range(NX),
                      final_fix_idx=[desc.final_fix_idx[i] for i in range(desc.n_final_fix)],
                      e_y=[0.0] * (NX - 1) + [1.0],
                      e_cost=[desc.px[i] * desc.e_cost[i] for i in range(NX)],
                      w_cost=desc.w_cost, w_prox=desc.w_prox, w_ep=desc.w_ep)


def random_subproblem(rng: np.random.Generator, nx=None, nu=None, nodes=None):
    """Small random scaled subproblem in the spirit of the reference's
    tmodels::random_subproblem (proj/tests/support/test_models.hpp:201-241): A_plus = -I,
    box on the last control slot only, all initial rows and a random subset of final rows
    pinned.  (Drawn from numpy's generator, so instances differ from the reference's mt19937
    stream; the tests compare implementations on identical instances.)"""
    nx = int(rng.integers(2, 5)) if nx is None else nx
    nu = int(rng.integers(1, 4)) if nu is None else nu
    n = int(rng.integers(2, 6)) if nodes is None else nodes
    m = n - 1
    u = lambda *shape: rng.uniform(-1.0, 1.0, size=shape)  # noqa: E731
    A_minus = 0.8 * u(m, nx, nx) + np.eye(nx)
    B_minus, B_plus = 0.5 * u(m, nx, nu), 0.5 * u(m, nx, nu)
    w = 0.5 * u(m, nx)
    eps = 0.15 + 0.1 * u(m)
    u_min = np.full((n, nu), -np.inf)
    u_max = np.full((n, nu), np.inf)
    u_min[:, nu - 1] = -0.2 - 0.6 * np.abs(u(n))
    u_max[:, nu - 1] = 0.2 + 0.6 * np.abs(u(n))
    final_idx = [i for i in range(nx) if u() > 0.0]
    e_y = np.zeros(nx)
    e_y[nx - 1] = 1.0
    shape = make_shape(nx, nu, n, init_fix_idx=range(nx), final_fix_idx=final_idx, e_y=e_y,
                       e_cost=u(nx), w_cost=float(abs(u())), w_prox=float(0.5 + 2.5 * abs(u())),
                       w_ep=float(0.5 + 1.5 * abs(u())))
    sub = SubArrays(A_minus=A_minus, A_plus=None, B_minus=B_minus, B_plus=B_plus, w=w,
                    eps_relax=eps, u_min=u_min, u_max=u_max, init_fix_val=0.4 * u(nx),
                    final_fix_val=0.4 * u(max(len(final_idx), 1)))
    return shape, sub


def dense_operator(shape, sub):
    """Materialises the stacked constraint operator [G; H] of build_generic_qp
    (proj/include/ptopt/pipg.hpp:563-631) with numpy, in the generic layout
    (x nodes | u nodes | vc_neg | vc_pos).  Independent of every solver path."""
    nx, nu, n = shape.n_x, shape.n_u, shape.nodes
    m = n - 1
    dim = n * (nx + nu) + 2 * m * nx
    x_off = lambda k: k * nx  # noqa: E731
    u_off = lambda k: n * nx + k * nu  # noqa: E731
    vcn_off = lambda k: n * (nx + nu) + k * nx  # noqa: E731
    vcp_off = lambda k: n * (nx + nu) + m * nx + k * nx  # noqa: E731
    G = np.zeros((m * nx, dim))
    H = np.zeros((m, dim))
    e_y = np.array([shape.e_y[i] for i in range(nx)])
    for k in range(m):
        rows = slice(k * nx, (k + 1) * nx)
        G[rows, x_off(k):x_off(k) + nx] = sub.A_minus[k]
        G[rows, x_off(k + 1):x_off(k + 1) + nx] = (-np.eye(nx) if sub.A_plus is None
                                                   else sub.A_plus[k])
        G[rows, u_off(k):u_off(k) + nu] = sub.B_minus[k]
        G[rows, u_off(k + 1):u_off(k + 1) + nu] = sub.B_plus[k]
        G[rows, vcp_off(k):vcp_off(k) + nx] = np.eye(nx)
        G[rows, vcn_off(k):vcn_off(k) + nx] = -np.eye(nx)
        H[k, x_off(k):x_off(k) + nx] = -e_y
        H[k, x_off(k + 1):x_off(k + 1) + nx] = e_y
    return G, H


def pack_primal(shape, ws):
    """pack_primal (pipg.hpp:731-749)."""
    return np.concatenate([ws.x.ravel(), ws.u.ravel(), ws.vc_neg.ravel(), ws.vc_pos.ravel()])
