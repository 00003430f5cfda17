// sim_kernels.cpp — TEST INFRASTRUCTURE.  Runs the device thread / lane code of
// paper_2404_18034_b200/csrc/*.cuh on the CPU, one "lane" after another, so the
// kernel arithmetic can be checked against the oracle without a GPU.  Not part of
// the product library and never loaded by it.
#include <cstring>
#include <vector>

#include "model_const.hpp"
#include "rocket_model.cuh"

using namespace ptopt_b200;

extern "C" {

/// One interval through the state pass (records kept in memory) and the column pass of every
/// lane, then the kernel's epilogue.
int sim_propagate_interval(const ptopt_vehicle_params* vp, const double* xk, const double* uk,
                           const double* uk1, double tau_k, double tau_k1, int steps, double* A,
                           double* Bm, double* Bp, double* w, double* x_end) {
  ModelConst mc;
  if (!make_model_const(*vp, mc)) return -8;
  double block[kNX][kCols];
  double xe[kNX];
  std::vector<double> recs((size_t)4 * steps * kRecSize);
  const int rc = propagate_state_pass(mc, xk, uk, uk1, tau_k, tau_k1, steps, xe,
                                      [&](int stage_no, int field, double v) {
                                        recs[(size_t)stage_no * kRecSize + field] = v;
                                      });
  if (rc) return rc;
  for (int lane = 0; lane < kCols; ++lane) {
    ColumnLane L;
    column_init(L, lane);
    ColumnForcing Fc;
    forcing_init(mc, lane, Fc);
    double slab[kSlabSize];
    for (int sn = 0; sn < 4 * steps; ++sn) {
      const StageTime t = stage_time(tau_k, tau_k1, steps, sn >> 2, sn & 3);
      expand_record(&recs[(size_t)sn * kRecSize], t.lam_left, t.lam_right, slab);
      column_stage_slab(L, Fc, slab, t, sn & 3);
    }
    for (int i = 0; i < kNX; ++i) block[i][lane] = L.s_c[i];
  }
  for (int i = 0; i < kNX; ++i) {
    double acc = 0.0;
    for (int j = 0; j < kNX; ++j) acc += block[i][j] * xk[j];
    double wv = xe[i] + -1.0 * acc;
    acc = 0.0;
    for (int j = 0; j < kNU; ++j) acc += block[i][kNX + j] * uk[j];
    wv += -1.0 * acc;
    acc = 0.0;
    for (int j = 0; j < kNU; ++j) acc += block[i][kNX + kNU + j] * uk1[j];
    wv += -1.0 * acc;
    w[i] = wv;
    x_end[i] = xe[i];
    for (int j = 0; j < kNX; ++j) A[i * kNX + j] = block[i][j];
    for (int j = 0; j < kNU; ++j) {
      Bm[i * kNU + j] = block[i][kNX + j];
      Bp[i * kNU + j] = block[i][kNX + kNU + j];
    }
  }
  return 0;
}

}  // extern "C"
