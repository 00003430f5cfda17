"""ctypes binding of ``libptopt_cuda.so`` (the C-ABI of ``include/ptopt_cuda.h``).

``Solver`` mirrors the reference's solver API for the hot path — ``linearize_all``,
``assemble_subproblem``, ``power_iteration_custom``, ``pipg_custom``, ``scp_solve`` — batched
over instances.  Host arrays are numpy (the library stages them); ``*_dev`` methods take
torch CUDA tensors and run on the handle's stream without synchronising.

There is no CPU fallback: if the library is missing or no sm_100 device is usable the
calls raise.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from . import abi

_LIB_PATH = Path(__file__).resolve().parent / "libptopt_cuda.so"
_lib = None

EXPORTS = [
    "ptopt_cuda_abi_version", "ptopt_cuda_last_error", "ptopt_cuda_launch_count",
    "ptopt_cuda_create", "ptopt_cuda_destroy", "ptopt_cuda_synchronize",
    "ptopt_cuda_set_solver_path",
    "ptopt_cuda_linearize_batch", "ptopt_cuda_linearize_batch_dev",
    "ptopt_cuda_propagate_interval_batch",
    "ptopt_cuda_assemble_batch", "ptopt_cuda_subproblem_shape",
    "ptopt_cuda_power_iteration_batch", "ptopt_cuda_power_iteration_batch_dev",
    "ptopt_cuda_pipg_batch", "ptopt_cuda_pipg_batch_dev",
    "ptopt_cuda_scp_solve_batch", "ptopt_cuda_scp_solve_batch_dev",
    "ptopt_cuda_generate_batch", "ptopt_cuda_generate_batch_dev",
    "ptopt_cuda_dense_audit_batch", "ptopt_cuda_dense_audit_batch_dev",
    "ptopt_cuda_dense_audit_samples_batch",
    "ptopt_cuda_run_batch", "ptopt_cuda_run_batch_multi",
    "ptopt_cuda_scp_stage_times", "ptopt_cuda_measure_fp64_peak",
]

RECORD_DTYPE = np.dtype([
    ("run_id", np.int32), ("converged", np.int32), ("scp_iterations", np.int32),
    ("status", np.int32), ("fail_index", np.int32), ("reserved_", np.int32),
    ("initial_position", np.float64, (3,)), ("propellant_used", np.float64),
    ("final_defect_inf", np.float64), ("max_pointwise_g", np.float64),
    ("max_node_y_increase", np.float64)])

STAGE_NAMES = ("linearize", "prepare", "power_iteration", "pipg", "update", "graph_total")


class PtoptError(RuntimeError):
    def __init__(self, code, message):
        super().__init__(f"ptopt_cuda error {code}: {message}")
        self.code = code


class InstanceError(RuntimeError):
    """A per-instance failure (what the reference reports by throwing)."""

    def __init__(self, status, fail_index):
        super().__init__(f"{abi.STATUS_NAMES.get(status, status)} (index {fail_index})")
        self.status = status
        self.fail_index = fail_index


def load_library():
    """Loads the CUDA library; raises if it has not been built (no silent fallback)."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise FileNotFoundError(
                f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` or `make -C paper_2404_18034_b200/csrc`")
        lib = C.CDLL(str(_LIB_PATH))
        lib.ptopt_cuda_last_error.restype = C.c_char_p
        lib.ptopt_cuda_launch_count.restype = C.c_int64
        lib.ptopt_cuda_launch_count.argtypes = [C.c_void_p]
        _lib = lib
    return _lib


def _check(rc):
    if rc != abi.OK:
        raise PtoptError(rc, load_library().ptopt_cuda_last_error().decode())


def _np(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


def _hp(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _dp(t):
    """torch CUDA tensor -> device pointer."""
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous()
    return C.c_void_p(t.data_ptr())


class Solver:
    """One ``ptopt_cuda_handle``: a problem description bound to one device and stream."""

    def __init__(self, desc: abi.ProblemDesc, tau=None, device: int = 0, stream=None):
        self.lib = load_library()
        self.desc = desc
        self.nodes = int(desc.nodes)
        self.device = device
        self.solver_path = "auto"
        self._h = C.c_void_p()
        tau_arr = None if tau is None else _np(tau)
        stream_ptr = None
        if stream is not None:
            stream_ptr = C.c_void_p(getattr(stream, "cuda_stream", stream))
        _check(self.lib.ptopt_cuda_create(C.byref(desc), _hp(tau_arr), C.c_int(device), stream_ptr,
                                          C.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self.lib.ptopt_cuda_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_solver_path(self, path: str):
        """'auto' (latency-mode kernels when the batch fits the chip in one wave, else the
        throughput kernels; generic kernels for non-rocket shapes), 'generic', 'split'
        (PTOPT_SOLVER_FAST_SPLIT), 'latency' (PTOPT_SOLVER_FAST_LATENCY) or 'fast'
        (PTOPT_SOLVER_FAST_THROUGHPUT: column-sparse kernels with the dense ones behind them) or
        'dense' (PTOPT_SOLVER_FAST_DENSE: the dense register-resident kernels alone)."""
        code = {"auto": 0, "generic": 1, "split": 2, "latency": 3, "fast": 4, "dense": 5}[path]
        _check(self.lib.ptopt_cuda_set_solver_path(self._h, C.c_int(code)))
        self.solver_path = path

    def synchronize(self):
        _check(self.lib.ptopt_cuda_synchronize(self._h))

    @property
    def launch_count(self) -> int:
        return int(self.lib.ptopt_cuda_launch_count(self._h))

    def scp_stage_times(self) -> dict:
        """Device milliseconds per stage of the last scp_solve graph launch."""
        ms = (C.c_double * 6)()
        _check(self.lib.ptopt_cuda_scp_stage_times(self._h, ms))
        return dict(zip(STAGE_NAMES, [float(v) for v in ms]))

    def measure_fp64_peak(self) -> float:
        """DFMA microbenchmark, TFLOP/s."""
        tf = C.c_double(0.0)
        _check(self.lib.ptopt_cuda_measure_fp64_peak(self._h, C.byref(tf)))
        return tf.value

    # ---------------------------------------------------------------- discretization
    def linearize_all(self, x, u):
        """Batched linearize_all (discretizer.hpp:191-232). x [B,N,15], u [B,N,7]."""
        x, u = _np(x), _np(u)
        B, n = x.shape[0], self.nodes
        m = n - 1
        assert x.shape == (B, n, abi.NX) and u.shape == (B, n, abi.NU)
        out = dict(A=np.empty((B, m, abi.NX, abi.NX)), Bm=np.empty((B, m, abi.NX, abi.NU)),
                   Bp=np.empty((B, m, abi.NX, abi.NU)), w=np.empty((B, m, abi.NX)),
                   x_end=np.empty((B, m, abi.NX)), status=np.empty(B, np.int32),
                   fail_index=np.empty(B, np.int32))
        _check(self.lib.ptopt_cuda_linearize_batch(
            self._h, C.c_int(B), _hp(x), _hp(u), _hp(out["A"]), _hp(out["Bm"]), _hp(out["Bp"]),
            _hp(out["w"]), _hp(out["x_end"]), _hp(out["status"]), _hp(out["fail_index"])))
        return out

    def propagate_interval(self, x_k, u_k, u_k1, tau_k, tau_k1, steps):
        """Batched propagate_interval (discretizer.hpp:82-149): one row per interval."""
        x_k, u_k, u_k1 = _np(x_k), _np(u_k), _np(u_k1)
        tau_k, tau_k1 = _np(tau_k), _np(tau_k1)
        B = x_k.shape[0]
        out = dict(A=np.empty((B, abi.NX, abi.NX)), Bm=np.empty((B, abi.NX, abi.NU)),
                   Bp=np.empty((B, abi.NX, abi.NU)), w=np.empty((B, abi.NX)),
                   x_end=np.empty((B, abi.NX)), status=np.empty(B, np.int32))
        _check(self.lib.ptopt_cuda_propagate_interval_batch(
            self._h, C.c_int(B), _hp(x_k), _hp(u_k), _hp(u_k1), _hp(tau_k), _hp(tau_k1),
            C.c_int(steps), _hp(out["A"]), _hp(out["Bm"]), _hp(out["Bp"]), _hp(out["w"]),
            _hp(out["x_end"]), _hp(out["status"])))
        return out

    def linearize_all_dev(self, x, u, A, Bm, Bp, w, x_end, status=None, fail_index=None):
        _check(self.lib.ptopt_cuda_linearize_batch_dev(
            self._h, C.c_int(x.shape[0]), _dp(x), _dp(u), _dp(A), _dp(Bm), _dp(Bp), _dp(w),
            _dp(x_end), _dp(status), _dp(fail_index)))

    # ---------------------------------------------------------------------- assembly
    def subproblem_shape(self) -> abi.SubproblemShape:
        s = abi.SubproblemShape()
        _check(self.lib.ptopt_cuda_subproblem_shape(self._h, C.byref(s)))
        return s

    def assemble_subproblem(self, init_state, x, u, blocks):
        """Batched assemble_subproblem (scp.hpp:139-217)."""
        init_state, x, u = _np(init_state), _np(x), _np(u)
        B, n = x.shape[0], self.nodes
        m = n - 1
        nf = max(int(self.desc.n_final_fix), 1)
        out = dict(A_minus=np.empty((B, m, abi.NX, abi.NX)), B_minus=np.empty((B, m, abi.NX, abi.NU)),
                   B_plus=np.empty((B, m, abi.NX, abi.NU)), w=np.empty((B, m, abi.NX)),
                   eps_relax=np.empty((B, m)), u_min=np.empty((B, n, abi.NU)),
                   u_max=np.empty((B, n, abi.NU)), init_fix_val=np.empty((B, abi.NX)),
                   final_fix_val=np.zeros((B, nf)))
        _check(self.lib.ptopt_cuda_assemble_batch(
            self._h, C.c_int(B), _hp(init_state), _hp(x), _hp(u), _hp(_np(blocks["A"])),
            _hp(_np(blocks["Bm"])), _hp(_np(blocks["Bp"])), _hp(_np(blocks["x_end"])),
            _hp(out["A_minus"]), _hp(out["B_minus"]), _hp(out["B_plus"]), _hp(out["w"]),
            _hp(out["eps_relax"]), _hp(out["u_min"]), _hp(out["u_max"]), _hp(out["init_fix_val"]),
            _hp(out["final_fix_val"])))
        return out

    # ------------------------------------------------------------------------ solver
    @staticmethod
    def _sub_struct(sub: dict):
        """dict of numpy arrays (batch axis first; A_plus may be None) -> C struct."""
        s = abi.SubproblemArrays()
        keep = []
        for f, _ in abi.SubproblemArrays._fields_:
            v = sub.get(f)
            if v is None:
                setattr(s, f, None)
                continue
            v = _np(v)
            keep.append(v)
            setattr(s, f, v.ctypes.data)
        return s, keep

    def power_iteration_custom(self, shape, sub, seed_x, seed_u, seed_vcp, seed_vcn, eps_abs,
                               eps_rel, eps_buff, j_max):
        """Batched pipg::power_iteration_custom (pipg.hpp:206-292); arrays carry a batch axis."""
        seed_x, seed_u, seed_vcp, seed_vcn = map(_np, (seed_x, seed_u, seed_vcp, seed_vcn))
        B = seed_x.shape[0]
        s, keep = self._sub_struct(sub)
        sigma, trips, status = np.empty(B), np.empty(B, np.int32), np.empty(B, np.int32)
        _check(self.lib.ptopt_cuda_power_iteration_batch(
            self._h, C.c_int(B), C.byref(shape), C.byref(s), _hp(seed_x), _hp(seed_u),
            _hp(seed_vcp), _hp(seed_vcn), C.c_double(eps_abs), C.c_double(eps_rel),
            C.c_double(eps_buff), C.c_int(j_max), _hp(sigma), _hp(trips), _hp(status)))
        return sigma, trips, status

    def pipg_custom(self, shape, sub, cfg, sigma, ws):
        """Batched pipg::pipg_custom (pipg.hpp:350-497).  ``ws``: dict of the six workspace
        groups with a batch axis, updated in place."""
        sigma = _np(sigma)
        B = sigma.shape[0]
        s, keep = self._sub_struct(sub)
        w = abi.WorkspaceArrays()
        for f, _ in abi.WorkspaceArrays._fields_:
            assert ws[f].dtype == np.float64 and ws[f].flags["C_CONTIGUOUS"]
            setattr(w, f, ws[f].ctypes.data)
        iters, conv = np.empty(B, np.int32), np.empty(B, np.uint8)
        status, fail = np.empty(B, np.int32), np.empty(B, np.int32)
        _check(self.lib.ptopt_cuda_pipg_batch(
            self._h, C.c_int(B), C.byref(shape), C.byref(s), C.byref(cfg), _hp(sigma), C.byref(w),
            _hp(iters), _hp(conv), _hp(status), _hp(fail)))
        return iters, conv.astype(bool), status, fail

    # ------------------------------------------------------------- Monte Carlo harness
    @staticmethod
    def _spec(r_low, r_high, seed):
        sp = abi.DispersionSpec()
        sp.r_low[:] = list(r_low)
        sp.r_high[:] = list(r_high)
        sp.seed = int(seed)
        return sp

    def generate_batch(self, batch, first_run_id, nominal_init_state, r_low, r_high, seed):
        """disperse + run_seed + initial_guess on the device (montecarlo.hpp:43-65,
        rocket_problem.hpp:127-163) for run ids first_run_id .. first_run_id+batch-1."""
        n = self.nodes
        out = dict(init_state=np.empty((batch, abi.NXI)), x_guess=np.empty((batch, n, abi.NX)),
                   u_guess=np.empty((batch, n, abi.NU)), rng_seed=np.empty(batch, np.uint64))
        sp = self._spec(r_low, r_high, seed)
        _check(self.lib.ptopt_cuda_generate_batch(
            self._h, C.c_int(batch), C.c_int64(first_run_id), _hp(_np(nominal_init_state)),
            C.byref(sp), _hp(out["init_state"]), _hp(out["x_guess"]), _hp(out["u_guess"]),
            _hp(out["rng_seed"])))
        return out

    def dense_violation_audit(self, x, u, substeps):
        """Batched dense_violation_audit (discretizer.hpp:249-285)."""
        x, u = _np(x), _np(u)
        B, m = x.shape[0], self.nodes - 1
        out = dict(max_pointwise_g=np.empty(B), interval_y_increase=np.empty((B, m)),
                   status=np.empty(B, np.int32), fail_index=np.empty(B, np.int32))
        _check(self.lib.ptopt_cuda_dense_audit_batch(
            self._h, C.c_int(B), C.c_int(substeps), _hp(x), _hp(u), _hp(out["max_pointwise_g"]),
            _hp(out["interval_y_increase"]), _hp(out["status"]), _hp(out["fail_index"])))
        return out

    def dense_violation_audit_samples(self, x, u, substeps):
        """dense_violation_audit with its sample sink: adds samples [B, M, substeps+1, 12] =
        {interval, tau, g[9], g_max} (discretizer.hpp:236-240, 262-276)."""
        x, u = _np(x), _np(u)
        B, m = x.shape[0], self.nodes - 1
        out = dict(samples=np.empty((B, m, substeps + 1, 12)), max_pointwise_g=np.empty(B),
                   interval_y_increase=np.empty((B, m)), status=np.empty(B, np.int32),
                   fail_index=np.empty(B, np.int32))
        _check(self.lib.ptopt_cuda_dense_audit_samples_batch(
            self._h, C.c_int(B), C.c_int(substeps), _hp(x), _hp(u), _hp(out["samples"]),
            _hp(out["max_pointwise_g"]), _hp(out["interval_y_increase"]), _hp(out["status"]),
            _hp(out["fail_index"])))
        return out

    def run_batch(self, batch, first_run_id, nominal_init_state, r_low, r_high, seed,
                  audit_substeps=64, keep_trajectories=False, records=None, x_out=None,
                  u_out=None):
        """mc::run_batch (montecarlo.hpp:140-175) on the device; returns a structured array of
        ptopt_run_record (and the trajectories when asked)."""
        n = self.nodes
        rec = np.empty(batch, RECORD_DTYPE) if records is None else records
        if keep_trajectories and x_out is None:
            x_out, u_out = np.empty((batch, n, abi.NX)), np.empty((batch, n, abi.NU))
        sp = self._spec(r_low, r_high, seed)
        _check(self.lib.ptopt_cuda_run_batch(
            self._h, C.c_int(batch), C.c_int64(first_run_id), _hp(_np(nominal_init_state)),
            C.byref(sp), C.c_int(audit_substeps), _hp(rec), _hp(x_out), _hp(u_out)))
        return (rec, x_out, u_out) if keep_trajectories else rec

    # ---------------------------------------------------------------------- SCP loop
    def scp_solve(self, init_state, x_guess, u_guess, rng_seed):
        """Batched scp_solve (scp.hpp:256-364) through the host-pointer entry point."""
        init_state, x_guess, u_guess = _np(init_state), _np(x_guess), _np(u_guess)
        rng_seed = _np(rng_seed, np.uint64)
        B, n, mi = x_guess.shape[0], self.nodes, int(self.desc.max_iters)
        out = dict(x=np.empty((B, n, abi.NX)), u=np.empty((B, n, abi.NU)),
                   scp_iterations=np.empty(B, np.int32), converged=np.empty(B, np.uint8),
                   final_defect_inf=np.empty(B), history=np.empty((B, mi, abi.HISTORY_FIELDS)),
                   power_trips=np.empty((B, mi), np.int32), status=np.empty(B, np.int32),
                   fail_index=np.empty(B, np.int32))
        _check(self.lib.ptopt_cuda_scp_solve_batch(
            self._h, C.c_int(B), _hp(init_state), _hp(x_guess), _hp(u_guess), _hp(rng_seed),
            _hp(out["x"]), _hp(out["u"]), _hp(out["scp_iterations"]), _hp(out["converged"]),
            _hp(out["final_defect_inf"]), _hp(out["history"]), _hp(out["power_trips"]),
            _hp(out["status"]), _hp(out["fail_index"])))
        out["converged"] = out["converged"].astype(bool)
        return out

    def scp_solve_into(self, init_state, x_guess, u_guess, rng_seed, out: dict):
        """Host-pointer entry point writing into caller-provided (e.g. pinned) numpy arrays."""
        B = x_guess.shape[0]
        _check(self.lib.ptopt_cuda_scp_solve_batch(
            self._h, C.c_int(B), _hp(init_state), _hp(x_guess), _hp(u_guess), _hp(rng_seed),
            _hp(out["x"]), _hp(out["u"]), _hp(out["scp_iterations"]), _hp(out["converged"]),
            _hp(out["final_defect_inf"]), _hp(out["history"]), _hp(out["power_trips"]),
            _hp(out["status"]), _hp(out["fail_index"])))

    def scp_solve_dev(self, init_state, x_guess, u_guess, rng_seed, x_out, u_out,
                      scp_iterations=None, converged=None, final_defect_inf=None, history=None,
                      power_trips=None, status=None, fail_index=None):
        """Device-pointer entry point (torch CUDA tensors); asynchronous on the handle's stream."""
        _check(self.lib.ptopt_cuda_scp_solve_batch_dev(
            self._h, C.c_int(x_guess.shape[0]), _dp(init_state), _dp(x_guess), _dp(u_guess),
            _dp(rng_seed), _dp(x_out), _dp(u_out), _dp(scp_iterations), _dp(converged),
            _dp(final_defect_inf), _dp(history), _dp(power_trips), _dp(status), _dp(fail_index)))


def run_batch_multi(desc: abi.ProblemDesc, devices, batch, first_run_id, nominal_init_state, r_low,
                    r_high, seed, audit_substeps=64, keep_trajectories=False, tau=None,
                    records=None):
    """ptopt_cuda_run_batch_multi: mc::run_batch with one worker (handle + host thread) per entry
    of `devices`, contiguous run-id ranges, records written into their run-id slots.  Returns
    (records, per-device wall ms) or (records, x, u, per-device wall ms)."""
    lib = load_library()
    n = int(desc.nodes)
    devs = (C.c_int * len(devices))(*[int(d) for d in devices])
    rec = np.empty(batch, RECORD_DTYPE) if records is None else records
    x_out = u_out = None
    if keep_trajectories:
        x_out, u_out = np.empty((batch, n, abi.NX)), np.empty((batch, n, abi.NU))
    ms = np.zeros(len(devices))
    sp = Solver._spec(r_low, r_high, seed)
    tau_arr = None if tau is None else _np(tau)
    _check(lib.ptopt_cuda_run_batch_multi(
        C.byref(desc), _hp(tau_arr), devs, C.c_int(len(devices)), C.c_int(batch),
        C.c_int64(first_run_id), _hp(_np(nominal_init_state)), C.byref(sp), C.c_int(audit_substeps),
        _hp(rec), _hp(x_out), _hp(u_out), _hp(ms)))
    return (rec, x_out, u_out, ms) if keep_trajectories else (rec, ms)
