// model_const.hpp — host-side folding of rocket::VehicleParams into the constants the kernels
// use (inverse inertia by cofactors, Jinv*[r_T]x, squared limits, sec(delta_max)).
// Follows /root/reference/proj/include/ptopt/rocket6dof.hpp:139-143, 210-224, 282, 292, 370-375.
#pragma once

#include <cmath>

#include "ptopt_cuda.h"
#include "rocket_model.cuh"

namespace ptopt_b200 {

/// Returns false when the inertia matrix is singular (inverse3 throws std::domain_error).
inline bool make_model_const(const ptopt_vehicle_params& p, ModelConst& mc) {
  const double* J = p.inertia;
  const double det = J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
                     J[2] * (J[3] * J[7] - J[4] * J[6]);
  if (det == 0.0) return false;
  mc.alpha = p.alpha_mdot;
  for (int i = 0; i < 3; ++i) mc.g[i] = p.g_inertial[i];
  for (int i = 0; i < 9; ++i) mc.J[i] = J[i];
  mc.Jinv[0] = (J[4] * J[8] - J[5] * J[7]) / det;
  mc.Jinv[1] = (J[2] * J[7] - J[1] * J[8]) / det;
  mc.Jinv[2] = (J[1] * J[5] - J[2] * J[4]) / det;
  mc.Jinv[3] = (J[5] * J[6] - J[3] * J[8]) / det;
  mc.Jinv[4] = (J[0] * J[8] - J[2] * J[6]) / det;
  mc.Jinv[5] = (J[2] * J[3] - J[0] * J[5]) / det;
  mc.Jinv[6] = (J[3] * J[7] - J[4] * J[6]) / det;
  mc.Jinv[7] = (J[1] * J[6] - J[0] * J[7]) / det;
  mc.Jinv[8] = (J[0] * J[4] - J[1] * J[3]) / det;
  for (int i = 0; i < 3; ++i) mc.rT[i] = p.r_thrust[i];
  const double* a = p.r_thrust;
  const double Rk[9] = {0.0, -a[2], a[1], a[2], 0.0, -a[0], -a[1], a[0], 0.0};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc += mc.Jinv[i * 3 + k] * Rk[k * 3 + j];
      mc.JinvR[i * 3 + j] = acc;
    }
  for (int i = 0; i < 8; ++i) mc.H[i] = p.H_theta[i];
  mc.m_dry = p.m_dry;
  mc.v_max_sq = p.v_max * p.v_max;
  const double c = 1.0 - std::cos(p.theta_max);
  mc.c_theta_sq = c * c;
  mc.w_max_sq = p.omega_max * p.omega_max;
  mc.sec_delta = 1.0 / std::cos(p.delta_max);
  mc.T_max = p.T_max;
  mc.T_min = p.T_min;
  mc.gamma_max_sq = p.gamma_max * p.gamma_max;
  return true;
}

}  // namespace ptopt_b200
