"""ctypes mirror of ``include/ptopt_cuda.h`` (structs, enums, constants).

Field order and types follow the header one-to-one; ``tests/test_abi.py`` checks
``ctypes.sizeof`` of every struct against the sizes the C compiler reports.
"""
from __future__ import annotations

import ctypes as C

ABI_VERSION = 1

NXI = 14
NZETA = 6
NG = 9
NX = 15
NU = 7
HISTORY_FIELDS = 5

# ptopt_call_status
OK = 0
ERR_INVALID_ARGUMENT = -1
ERR_CUDA = -2
ERR_UNSUPPORTED = -3
ERR_ALLOC = -4

# ptopt_instance_status
ST_OK = 0
ST_PROPAGATION_DIVERGED = 1
ST_SOLVER_DIVERGED = 2
ST_DILATION_NONPOSITIVE = 3
ST_MASS_NONPOSITIVE = 4
ST_THRUST_SINGULAR = 5
ST_POWER_SEED_ZERO = 6

c_double_p = C.POINTER(C.c_double)
c_int32_p = C.POINTER(C.c_int32)
c_uint8_p = C.POINTER(C.c_uint8)
c_uint64_p = C.POINTER(C.c_uint64)


class VehicleParams(C.Structure):
    """rocket::VehicleParams (proj/include/ptopt/rocket6dof.hpp:85-99)."""

    _fields_ = [
        ("alpha_mdot", C.c_double),
        ("g_inertial", C.c_double * 3),
        ("inertia", C.c_double * 9),
        ("r_thrust", C.c_double * 3),
        ("H_theta", C.c_double * 8),
        ("m_dry", C.c_double),
        ("v_max", C.c_double),
        ("theta_max", C.c_double),
        ("omega_max", C.c_double),
        ("delta_max", C.c_double),
        ("T_min", C.c_double),
        ("T_max", C.c_double),
        ("gamma_max", C.c_double),
    ]


class PipgConfig(C.Structure):
    """pipg::PipgConfig (proj/include/ptopt/pipg.hpp:22-38)."""

    _fields_ = [
        ("omega", C.c_double),
        ("rho", C.c_double),
        ("j_max", C.c_int32),
        ("j_check", C.c_int32),
        ("eps_abs", C.c_double),
        ("eps_rel", C.c_double),
        ("eps_buff", C.c_double),
    ]


class ProblemDesc(C.Structure):
    """Flattened ScpProblem<Rocket6DoF> (proj/include/ptopt/scp.hpp:73-121)."""

    _fields_ = [
        ("vehicle", VehicleParams),
        ("nodes", C.c_int32),
        ("integrator_steps", C.c_int32),
        ("s_min", C.c_double),
        ("s_max", C.c_double),
        ("t_f_guess", C.c_double),
        ("w_cost", C.c_double),
        ("w_prox", C.c_double),
        ("w_ep", C.c_double),
        ("epsilon_relax", C.c_double),
        ("px", C.c_double * NX),
        ("pu", C.c_double * NU),
        ("pipg", PipgConfig),
        ("power_j_max", C.c_int32),
        ("max_iters", C.c_int32),
        ("power_eps_abs", C.c_double),
        ("power_eps_rel", C.c_double),
        ("tol_feas", C.c_double),
        ("tol_step", C.c_double),
        ("n_final_fix", C.c_int32),
        ("renormalize_quaternion", C.c_int32),
        ("final_fix_idx", C.c_int32 * NX),
        ("reserved_", C.c_int32),
        ("final_fix_val", C.c_double * NX),
        ("e_cost", C.c_double * NX),
    ]


class SubproblemShape(C.Structure):
    """Shape + shared data of pipg::Subproblem (proj/include/ptopt/pipg.hpp:43-96)."""

    _fields_ = [
        ("n_x", C.c_int32),
        ("n_u", C.c_int32),
        ("nodes", C.c_int32),
        ("n_init_fix", C.c_int32),
        ("n_final_fix", C.c_int32),
        ("reserved_", C.c_int32),
        ("init_fix_idx", C.c_int32 * NX),
        ("final_fix_idx", C.c_int32 * NX),
        ("e_y", C.c_double * NX),
        ("e_cost", C.c_double * NX),
        ("w_cost", C.c_double),
        ("w_prox", C.c_double),
        ("w_ep", C.c_double),
    ]


class SubproblemArrays(C.Structure):
    _fields_ = [
        ("A_minus", C.c_void_p),
        ("A_plus", C.c_void_p),
        ("B_minus", C.c_void_p),
        ("B_plus", C.c_void_p),
        ("w", C.c_void_p),
        ("eps_relax", C.c_void_p),
        ("u_min", C.c_void_p),
        ("u_max", C.c_void_p),
        ("init_fix_val", C.c_void_p),
        ("final_fix_val", C.c_void_p),
    ]


class WorkspaceArrays(C.Structure):
    """pipg::Workspace warm-start groups (proj/include/ptopt/pipg.hpp:100-141)."""

    _fields_ = [
        ("x", C.c_void_p),
        ("u", C.c_void_p),
        ("vc_pos", C.c_void_p),
        ("vc_neg", C.c_void_p),
        ("dyn_dual", C.c_void_p),
        ("relax_dual", C.c_void_p),
    ]


class DispersionSpec(C.Structure):
    """mc::DispersionSpec (proj/include/ptopt/montecarlo.hpp:20-31)."""

    _fields_ = [("r_low", C.c_double * 3), ("r_high", C.c_double * 3), ("seed", C.c_uint64)]


class RunRecord(C.Structure):
    """mc::RunRecord (proj/include/ptopt/montecarlo.hpp:67-78) as ptopt_run_record."""

    _fields_ = [
        ("run_id", C.c_int32),
        ("converged", C.c_int32),
        ("scp_iterations", C.c_int32),
        ("status", C.c_int32),
        ("fail_index", C.c_int32),
        ("reserved_", C.c_int32),
        ("initial_position", C.c_double * 3),
        ("propellant_used", C.c_double),
        ("final_defect_inf", C.c_double),
        ("max_pointwise_g", C.c_double),
        ("max_node_y_increase", C.c_double),
    ]


STATUS_NAMES = {
    ST_OK: "ok",
    ST_PROPAGATION_DIVERGED: "propagation diverged",
    ST_SOLVER_DIVERGED: "pipg diverged",
    ST_DILATION_NONPOSITIVE: "dilation factor must be positive",
    ST_MASS_NONPOSITIVE: "nonpositive mass",
    ST_THRUST_SINGULAR: "thrust magnitude below singular-point tolerance",
    ST_POWER_SEED_ZERO: "power iteration: seed point must not be all zero",
}
