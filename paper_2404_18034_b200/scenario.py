"""Host-side problem setup for the rocket landing path.

Restates the reference's shipped scenario (``default_config()``,
proj/include/ptopt/config.hpp:155-197 with the RunConfig defaults at :27-55),
the power-of-two scaling (proj/include/ptopt/scp.hpp:39-59,
proj/include/ptopt/rocket_problem.hpp:33-47), the boundary selectors
(rocket_problem.hpp:59-94) and the deterministic instance generators
(proj/include/ptopt/montecarlo.hpp:35-65, rocket_problem.hpp:98-163).

All of this is per-problem / per-instance *setup*; the hot path itself runs in
the CUDA library.  The integer generators are bit-exact (uint64 arithmetic on
Python ints); the floating-point parts use the same libm as the reference.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import abi

_M64 = (1 << 64) - 1

K_MASS, K_POS, K_VEL, K_ATT, K_RATE = 0, 1, 4, 7, 11
K_THRUST, K_TORQUE = 0, 3
Y_INDEX = abi.NX - 1
S_INDEX = abi.NU - 1


# --------------------------------------------------------------------------- RNG
def _splitmix64(x: int) -> int:
    """Stateless mix (montecarlo.hpp:35-40)."""
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def counter_uniform(seed: int, run: int, slot: int) -> float:
    """Uniform in [0,1) as a pure function of (seed, run, slot) (montecarlo.hpp:43-46)."""
    key = _splitmix64(seed ^ _splitmix64((run + 1) & _M64))
    return float(_splitmix64((key + slot) & _M64) >> 11) * 2.0 ** -53


def run_seed(batch_seed: int, run_id: int) -> int:
    """mc::run_seed (montecarlo.hpp:51-53)."""
    return _splitmix64(batch_seed ^ _splitmix64(run_id & _M64))


def pow2_near(v: float) -> float:
    """ScalingPair::pow2_near (scp.hpp:39-42)."""
    if not v > 0.0:
        raise ValueError("scaling ranges must be positive")
    lg = math.log2(v)
    r = math.copysign(math.floor(abs(lg) + 0.5), lg)  # std::round: halves away from zero
    return math.ldexp(1.0, int(r))


# ---------------------------------------------------------------------- scenario
@dataclass
class DispersionSpec:
    """mc::DispersionSpec (montecarlo.hpp:20-31)."""

    r_low: tuple = (6.0, 3.0, 1.0)
    r_high: tuple = (9.0, 6.0, 2.0)
    seed: int = 20260810


@dataclass
class Scenario:
    """RunConfig restated (config.hpp:27-55) with the default_config() values (:155-197)."""

    # vehicle
    alpha_mdot: float = 0.05
    g_inertial: tuple = (-1.0, 0.0, 0.0)
    inertia: tuple = (0.1, 0.0, 0.0, 0.0, 0.25, 0.0, 0.0, 0.0, 0.25)
    r_thrust: tuple = (-0.5, 0.0, 0.0)
    H_theta: tuple = (0.0, 1.0, 0.0, 0.0, 0.0, 0.0, 1.0, 0.0)
    m_dry: float = 1.0
    v_max: float = 3.0
    theta_max: float = 1.0471975511965976
    omega_max: float = 1.0
    delta_max: float = 0.3490658503988659
    T_min: float = 1.0
    T_max: float = 6.0
    gamma_max: float = 0.3
    # boundary
    initial_state: tuple = (2.0, 7.5, 4.5, 1.5, -1.0, -0.5, -0.2, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0)
    r_final: tuple = (0.0, 0.0, 0.0)
    v_final: tuple = (0.0, 0.0, 0.0)
    q_final: tuple = (0.0, 0.0, 0.0, 1.0)
    w_final: tuple = (0.0, 0.0, 0.0)
    # grid / time
    grid_nodes: int = 15
    integrator_substeps: int = 16
    audit_substeps: int = 64
    t_f_guess: float = 5.0
    s_min: float = 1.0
    s_max: float = 15.0
    # SCP
    w_cost: float = 1.0
    w_prox: float = 1.0
    w_ep: float = 100.0
    epsilon_relax: float = 1e-4
    tol_feas: float = 1e-6
    tol_step: float = 1e-5
    max_iters: int = 25
    # scaling ranges (mass, position, velocity, quaternion, omega, y, thrust, torque, dilation)
    scaling: tuple = (1.0, 8.0, 3.0, 1.0, 1.0, 1.0, 6.0, 0.3, 5.0)
    # PIPG
    pipg_omega: float = 100.0
    pipg_rho: float = 1.6
    pipg_j_max: int = 2500
    pipg_j_check: int = 25
    pipg_eps_abs: float = 1e-11
    pipg_eps_rel: float = 1e-11
    pipg_eps_buff: float = 0.05
    power_j_max: int = 10000
    power_eps_abs: float = 1e-12
    power_eps_rel: float = 1e-12
    dispersion: DispersionSpec = field(default_factory=DispersionSpec)

    def scaling_px_pu(self):
        """rocket_scaling + ScalingPair::from_ranges (rocket_problem.hpp:33-47, scp.hpp:44-59)."""
        mass, pos, vel, quat, omega, y, thrust, torque, dil = self.scaling
        xr = [mass] + [pos] * 3 + [vel] * 3 + [quat] * 4 + [omega] * 3 + [y]
        ur = [thrust] * 3 + [torque] * 3 + [dil]
        return [pow2_near(v) for v in xr], [pow2_near(v) for v in ur]

    def problem_desc(self) -> abi.ProblemDesc:
        """make_rocket_problem + RunConfig::problem (rocket_problem.hpp:59-94, config.hpp:79-96)."""
        d = abi.ProblemDesc()
        v = d.vehicle
        v.alpha_mdot = self.alpha_mdot
        v.g_inertial[:] = self.g_inertial
        v.inertia[:] = self.inertia
        v.r_thrust[:] = self.r_thrust
        v.H_theta[:] = self.H_theta
        for name in ("m_dry", "v_max", "theta_max", "omega_max", "delta_max", "T_min", "T_max",
                     "gamma_max"):
            setattr(v, name, getattr(self, name))
        d.nodes = self.grid_nodes
        d.integrator_steps = self.integrator_substeps
        d.s_min, d.s_max, d.t_f_guess = self.s_min, self.s_max, self.t_f_guess
        d.w_cost, d.w_prox, d.w_ep = self.w_cost, self.w_prox, self.w_ep
        d.epsilon_relax = self.epsilon_relax
        px, pu = self.scaling_px_pu()
        d.px[:] = px
        d.pu[:] = pu
        d.pipg.omega, d.pipg.rho = self.pipg_omega, self.pipg_rho
        d.pipg.j_max, d.pipg.j_check = self.pipg_j_max, self.pipg_j_check
        d.pipg.eps_abs, d.pipg.eps_rel = self.pipg_eps_abs, self.pipg_eps_rel
        d.pipg.eps_buff = self.pipg_eps_buff
        d.power_j_max = self.power_j_max
        d.power_eps_abs, d.power_eps_rel = self.power_eps_abs, self.power_eps_rel
        d.tol_feas, d.tol_step, d.max_iters = self.tol_feas, self.tol_step, self.max_iters
        idx = ([K_POS + i for i in range(3)] + [K_VEL + i for i in range(3)]
               + [K_ATT + i for i in range(4)] + [K_RATE + i for i in range(3)])
        val = list(self.r_final) + list(self.v_final) + list(self.q_final) + list(self.w_final)
        d.n_final_fix = len(idx)
        for i, (a, b) in enumerate(zip(idx, val)):
            d.final_fix_idx[i] = a
            d.final_fix_val[i] = b
        d.e_cost[K_MASS] = -1.0  # maximise terminal mass
        d.renormalize_quaternion = 1
        return d

    def grid(self) -> np.ndarray:
        return uniform_grid(self.grid_nodes)


def default_scenario(nodes: int = 15) -> Scenario:
    """``default_config()`` with only ``grid.N`` changed."""
    return Scenario(grid_nodes=nodes)


def uniform_grid(n: int) -> np.ndarray:
    """Grid::uniform (proj/include/ptopt/trajectory.hpp:23-30)."""
    if n < 2:
        raise ValueError("grid needs at least two nodes")
    tau = np.arange(n, dtype=np.float64) / float(n - 1)
    tau[0], tau[-1] = 0.0, 1.0
    return tau


# ------------------------------------------------------------ instance generation
def disperse(sc: Scenario, run_id: int) -> np.ndarray:
    """mc::disperse (montecarlo.hpp:55-65): the dispersed 14-vector initial state."""
    spec = sc.dispersion
    x0 = np.array(sc.initial_state, dtype=np.float64)
    for i in range(3):
        u = counter_uniform(spec.seed, run_id, i)
        x0[K_POS + i] = spec.r_low[i] + (spec.r_high[i] - spec.r_low[i]) * u
    return x0


def _slerp(qa, qb, t):
    """detail::slerp (rocket_problem.hpp:98-120)."""
    qb = list(qb)
    d = qa[0] * qb[0] + qa[1] * qb[1] + qa[2] * qb[2] + qa[3] * qb[3]
    if d < 0.0:
        qb = [-c for c in qb]
        d = -d
    if d > 1.0 - 1e-10:
        q = [(1.0 - t) * qa[i] + t * qb[i] for i in range(4)]
    else:
        ang = math.acos(min(1.0, d))
        sa = math.sin(ang)
        ca = math.sin((1.0 - t) * ang) / sa
        cb = math.sin(t * ang) / sa
        q = [ca * qa[i] + cb * qb[i] for i in range(4)]
    nq = 0.0
    for c in q:
        nq += c * c
    nq = math.sqrt(nq)
    return [c / nq for c in q]


def initial_guess(sc: Scenario, init_state: np.ndarray, tau: np.ndarray | None = None):
    """initial_guess (rocket_problem.hpp:127-163) -> x [N,15], u [N,7]."""
    n = sc.grid_nodes
    tau = uniform_grid(n) if tau is None else np.asarray(tau, dtype=np.float64)
    g = sc.g_inertial
    g_norm = math.sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2])
    m0 = float(init_state[K_MASS])
    m_end = max(sc.m_dry, m0 * math.exp(-sc.alpha_mdot * g_norm * sc.t_f_guess))
    x = np.zeros((n, abi.NX))
    u = np.zeros((n, abi.NU))
    q0 = [float(c) for c in init_state[K_ATT:K_ATT + 4]]
    for k in range(n):
        t = float(tau[k])
        sm = (1.0 - t) * m0 + t * m_end
        x[k, K_MASS] = sm
        for i in range(3):
            x[k, K_POS + i] = (1.0 - t) * float(init_state[K_POS + i]) + t * sc.r_final[i]
            x[k, K_VEL + i] = (1.0 - t) * float(init_state[K_VEL + i]) + t * sc.v_final[i]
            x[k, K_RATE + i] = (1.0 - t) * float(init_state[K_RATE + i]) + t * sc.w_final[i]
        x[k, K_ATT:K_ATT + 4] = _slerp(q0, sc.q_final, t)
        for i in range(3):
            u[k, K_THRUST + i] = -sm * g[i]
        u[k, S_INDEX] = sc.t_f_guess
    return x, u


def make_batch(sc: Scenario, run_ids) -> dict:
    """Inputs of one batch exactly as mc::solve_instance builds them (montecarlo.hpp:100-111)."""
    run_ids = list(run_ids)
    tau = sc.grid()
    init = np.stack([disperse(sc, r) for r in run_ids])
    xs, us = zip(*(initial_guess(sc, s, tau) for s in init))
    seeds = np.array([run_seed(sc.dispersion.seed, r) for r in run_ids], dtype=np.uint64)
    return {
        "run_id": np.array(run_ids, dtype=np.int64),
        "init_state": np.ascontiguousarray(init),
        "x_guess": np.ascontiguousarray(np.stack(xs)),
        "u_guess": np.ascontiguousarray(np.stack(us)),
        "rng_seed": seeds,
    }
