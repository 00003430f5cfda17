// linearize.cu — exact discretization: batched linearize_all
// (/root/reference/proj/include/ptopt/discretizer.hpp:191-232) in two passes over every
// (instance, interval):
//   * state pass   — one THREAD per interval integrates the 15 augmented states through the
//                    4 * steps RK4 stages (the only place the model and its Jacobian are
//                    evaluated) and leaves one 84-double record per stage in HBM;
//   * column pass  — one WARP per interval, lane j < 29 owns column j of
//                    [Phi_x | Phi_u- | Phi_u+]; every stage it fetches the record (coalesced,
//                    prefetched one stage ahead, staged in shared memory) and applies A(tau) and
//                    the B forcing to its column in registers; then stages the 15 x 29 block in
//                    shared memory for w = x_end - A x - B- u - B+ u+ and the coalesced write.
// See rocket_model.cuh for the per-thread / per-lane algorithms.
#include <type_traits>

#include "kernels.cuh"
#include "rocket_model.cuh"

namespace ptopt_b200 {

namespace {

constexpr int kWarpsPerCta = 4;
constexpr int kStageStride = kCols + 1;  // 30: row stride of the staged [15][29] block
constexpr int kRecLamLeft = 81;          // spare record slots: the first-order-hold factors
constexpr int kRecLamRight = 82;
static_assert(kRecLamRight < kRecSize, "record padding");

// Records of 32 consecutive intervals are interleaved (field-major inside a tile) so that the
// state pass -- one thread per interval -- writes them coalesced.  The four warps of a
// column-pass CTA read four neighbouring intervals, i.e. the same 32-byte sectors.
__host__ __device__ inline size_t record_index(long long local_interval, int nst, int stage_no) {
  const long long tile = local_interval >> 5;
  const int r = (int)(local_interval & 31);
  return (((size_t)tile * nst + stage_no) * kRecSize) * 32 + r;
}

__global__ void __launch_bounds__(128) state_pass_kernel(LinearizeArgs a, long long first, long long count) {
  const long long local = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (local >= count) return;
  const long long widx = first + local;
  const int M = a.nodes - 1;
  const int b = (int)(widx / M);
  const int k = (int)(widx - (long long)b * M);
  if (a.active && !a.active[b]) return;  // instance already finished (SCP loop)
  const double* xg = a.x + ((size_t)b * a.nodes + k) * kNX;
  const double* ug = a.u + ((size_t)b * a.nodes + k) * kNU;
  double xk[kNX], uk[kNU], uk1[kNU], x_end[kNX];
#pragma unroll
  for (int i = 0; i < kNX; ++i) xk[i] = xg[i];
#pragma unroll
  for (int i = 0; i < kNU; ++i) {
    uk[i] = ug[i];
    uk1[i] = ug[kNU + i];
  }
  const double* tau = a.tau + (size_t)b * a.tau_stride;
  const double tau_k = tau[k], tau_k1 = tau[k + 1];
  const int nst = 4 * a.steps;
  double* out = a.stages;
  const ModelConst& P = a.model;
  const int rc = propagate_state_pass(
      P, xk, uk, uk1, tau_k, tau_k1, a.steps, x_end, [&](int stage_no, const Stage& st, const double* u) {
        double rec[kRecSize];
        pack_stage_record(P, st, u, rec);
        const StageTime t = stage_time(tau_k, tau_k1, a.steps, stage_no >> 2, stage_no & 3);
        rec[kRecLamLeft] = t.lam_left;
        rec[kRecLamRight] = t.lam_right;
        double* o = out + record_index(local, nst, stage_no);
#pragma unroll
        for (int f = 0; f < kRecSize; ++f) o[(size_t)f * 32] = rec[f];
      });
  if (rc != kStOk) {
    // first failing interval wins, as the serial reference loop would report it
    atomicMin(&a.fail_key[b], (k << 4) | rc);
    return;
  }
  double* xe = a.x_end + ((size_t)b * M + k) * kNX;
#pragma unroll
  for (int i = 0; i < kNX; ++i) xe[i] = x_end[i];
}

constexpr int kRecRing = 4;  // stage records in flight per warp (cp.async ring)

struct __align__(16) WarpSmem {
  double rec[kRecRing][kRecSize];    // ring of stage records
  double block[kNX * kStageStride];  // staged [A | B- | B+], row-major
  double xk[kNX], uk[kNU], uk1[kNU], xe[kNX];
};

__global__ void __launch_bounds__(kWarpsPerCta * 32)
column_pass_kernel(LinearizeArgs a, long long first, long long count) {
  __shared__ WarpSmem smem[kWarpsPerCta];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const long long local = (long long)blockIdx.x * kWarpsPerCta + wib;
  if (local >= count) return;
  const long long widx = first + local;
  const int M = a.nodes - 1;
  const int b = (int)(widx / M);
  const int k = (int)(widx - (long long)b * M);
  if (a.active && !a.active[b]) return;  // instance already finished (SCP loop)
  // an instance with a failed interval has no blocks (its records stop at the failure)
  if (a.fail_key[b] != kFailKeyNone) return;

  WarpSmem& ws = smem[wib];
  const size_t iv = (size_t)b * M + k;
  const double* xg = a.x + ((size_t)b * a.nodes + k) * kNX;
  const double* ug = a.u + ((size_t)b * a.nodes + k) * kNU;
  if (lane < kNX) {
    ws.xk[lane] = xg[lane];
    ws.xe[lane] = a.x_end[iv * kNX + lane];
  }
  if (lane < kNU) {
    ws.uk[lane] = ug[lane];
    ws.uk1[lane] = ug[kNU + lane];
  }

  const double* tau = a.tau + (size_t)b * a.tau_stride;
  const double h = (tau[k + 1] - tau[k]) / a.steps;
  const double h6 = h / 6.0, h3 = h / 3.0, hh = 0.5 * h;  // as stage_time forms them
  const int nst = 4 * a.steps;
  const double* recs = a.stages + record_index(local, nst, 0);
  const size_t rec_stride = (size_t)kRecSize * 32;  // between consecutive stages of an interval
  const bool third = lane + 64 < kRecSize;
  // record `sn` -> ring slot sn % kRecRing, three 8-byte asynchronous copies per lane, one
  // commit group per record (an empty group past the last record keeps the counting uniform)
  auto fetch = [&](int sn) {
    if (sn < nst) {
      const double* src = recs + (size_t)sn * rec_stride + (size_t)lane * 32;
      const unsigned dst = (unsigned)__cvta_generic_to_shared(&ws.rec[sn % kRecRing][lane]);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 32 * 8), "l"(src + 32 * 32) : "memory");
      if (third)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 64 * 8), "l"(src + 64 * 32) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int sn = 0; sn < kRecRing - 1; ++sn) fetch(sn);

  ColumnLane L;
  column_init(L, lane);
  const bool is_col = lane < kCols;
  // one stage: wait for its record, start the copy of the record kRecRing - 1 stages ahead into
  // the slot everybody finished reading a stage ago, apply the record to the column
  auto run_stage = [&](auto stage_tag, int sn, double wk, double wn) {
    constexpr int kStage = decltype(stage_tag)::value;
    asm volatile("cp.async.wait_group %0;" ::"n"(kRecRing - 2) : "memory");
    __syncwarp();
    fetch(sn + kRecRing - 1);
    const double* rec = ws.rec[sn % kRecRing];
    // lanes 29..31 carry an all-zero dummy column (no branch around the stage)
    column_stage<kStage>(a.model, L, rec, wk, wn, rec[kRecLamLeft], rec[kRecLamRight]);
  };
  for (int step = 0; step < a.steps; ++step) {
    run_stage(std::integral_constant<int, 0>{}, 4 * step, h6, hh);
    run_stage(std::integral_constant<int, 1>{}, 4 * step + 1, h3, hh);
    run_stage(std::integral_constant<int, 2>{}, 4 * step + 2, h3, h);
    run_stage(std::integral_constant<int, 3>{}, 4 * step + 3, h6, hh);
  }

  // stage the 15x29 block, then w = x_end - A x_k - B- u_k - B+ u_k1 row by row in the
  // reference's order (discretizer.hpp:144-147)
  if (is_col) {
#pragma unroll
    for (int i = 0; i < kNX; ++i) ws.block[i * kStageStride + lane] = L.s_c[i];
  }
  __syncwarp();
  if (lane < kNX) {
    const double* row = ws.block + lane * kStageStride;
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < kNX; ++j) acc += row[j] * ws.xk[j];
    double wv = ws.xe[lane] + -1.0 * acc;
    acc = 0.0;
#pragma unroll
    for (int j = 0; j < kNU; ++j) acc += row[kNX + j] * ws.uk[j];
    wv += -1.0 * acc;
    acc = 0.0;
#pragma unroll
    for (int j = 0; j < kNU; ++j) acc += row[kNX + kNU + j] * ws.uk1[j];
    wv += -1.0 * acc;
    a.w[iv * kNX + lane] = wv;
  }
  double* Ag = a.A + iv * kNX * kNX;
  for (int e = lane; e < kNX * kNX; e += 32) Ag[e] = ws.block[(e / kNX) * kStageStride + e % kNX];
  double* Bmg = a.Bm + iv * kNX * kNU;
  double* Bpg = a.Bp + iv * kNX * kNU;
  for (int e = lane; e < kNX * kNU; e += 32) {
    const int i = e / kNU, j = e % kNU;
    Bmg[e] = ws.block[i * kStageStride + kNX + j];
    Bpg[e] = ws.block[i * kStageStride + kNX + kNU + j];
  }
}

__global__ void init_fail_key_kernel(int* fail_key, int batch) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < batch) fail_key[b] = kFailKeyNone;
}

__global__ void decode_fail_key_kernel(const int* fail_key, int batch, int* status,
                                       int* fail_index) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const int key = fail_key[b];
  if (key == kFailKeyNone) {
    if (status) status[b] = kStOk;
    if (fail_index) fail_index[b] = -1;
  } else {
    if (status) status[b] = key & 15;
    if (fail_index) fail_index[b] = key >> 4;
  }
}

}  // namespace

void launch_init_fail_key(int* fail_key, int batch, cudaStream_t stream) {
  init_fail_key_kernel<<<(batch + 255) / 256, 256, 0, stream>>>(fail_key, batch);
}

void launch_decode_fail_key(const int* fail_key, int batch, int* status, int* fail_index,
                            cudaStream_t stream) {
  decode_fail_key_kernel<<<(batch + 255) / 256, 256, 0, stream>>>(fail_key, batch, status,
                                                                  fail_index);
}

size_t linearize_stage_doubles(long long intervals, int steps) {
  const long long tiles = (intervals + 31) / 32;
  return (size_t)tiles * 32 * (size_t)(4 * steps) * kRecSize;
}

long long linearize_chunk_intervals(long long intervals, int steps, size_t max_bytes) {
  const size_t per_tile = 32 * (size_t)(4 * steps) * kRecSize * sizeof(double);
  long long tiles = (long long)(max_bytes / per_tile);
  if (tiles < 1) tiles = 1;
  const long long cap = tiles * 32;
  return intervals < cap ? (intervals + 31) / 32 * 32 : cap;
}

int launch_linearize(const LinearizeArgs& a, cudaStream_t stream) {
  const long long total = (long long)a.batch * (a.nodes - 1);
  int launches = 0;
  for (long long first = 0; first < total; first += a.stage_capacity) {
    const long long count = total - first < a.stage_capacity ? total - first : a.stage_capacity;
    state_pass_kernel<<<(unsigned)((count + 127) / 128), 128, 0, stream>>>(a, first, count);
    column_pass_kernel<<<(unsigned)((count + kWarpsPerCta - 1) / kWarpsPerCta), kWarpsPerCta * 32, 0, stream>>>(
        a, first, count);
    launches += 2;
  }
  return launches;
}

}  // namespace ptopt_b200
