// linearize.cu — exact discretization kernel: batched linearize_all
// (/root/reference/proj/include/ptopt/discretizer.hpp:191-232) with one warp per
// (instance, interval).  See rocket_model.cuh for the per-lane algorithm.
#include "kernels.cuh"
#include "rocket_model.cuh"

namespace ptopt_b200 {

namespace {

constexpr int kWarpsPerCta = 4;
constexpr int kStageStride = kCols + 1;  // 30: row stride of the staged [15][29] block

struct __align__(16) WarpSmem {
  StateScratch sc;
  double block[kNX * kStageStride];  // staged [A | B- | B+], row-major
  double xk[kNX], uk[kNU], uk1[kNU], xe[kNX];
};

struct WarpSync {
  __device__ __forceinline__ void operator()() const { __syncwarp(); }
};

__global__ void __launch_bounds__(kWarpsPerCta * 32)
linearize_kernel(LinearizeArgs a) {
  __shared__ WarpSmem smem[kWarpsPerCta];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const long long widx = (long long)blockIdx.x * kWarpsPerCta + wib;
  const int M = a.nodes - 1;
  if (widx >= (long long)a.batch * M) return;
  const int b = (int)(widx / M);
  const int k = (int)(widx - (long long)b * M);
  if (a.active && !a.active[b]) return;  // instance already finished (SCP loop)

  WarpSmem& ws = smem[wib];
  const double* xg = a.x + ((size_t)b * a.nodes + k) * kNX;
  const double* ug = a.u + ((size_t)b * a.nodes + k) * kNU;
  if (lane < kNX) ws.xk[lane] = xg[lane];
  if (lane < kNU) {
    ws.uk[lane] = ug[lane];
    ws.uk1[lane] = ug[kNU + lane];
  }
  __syncwarp();
  double xk[kNX], uk[kNU], uk1[kNU];
#pragma unroll
  for (int i = 0; i < kNX; ++i) xk[i] = ws.xk[i];
#pragma unroll
  for (int i = 0; i < kNU; ++i) {
    uk[i] = ws.uk[i];
    uk1[i] = ws.uk1[i];
  }

  double col[kNX], x_end[kNX];
  const double* tau = a.tau + (size_t)b * a.tau_stride;
  const int rc = propagate_lane(a.model, lane, lane == 0, ws.sc, xk, uk, uk1, tau[k], tau[k + 1],
                                a.steps, col, x_end, WarpSync());
  if (rc != kStOk) {
    // first failing interval wins, as the serial reference loop would report it
    if (lane == 0) atomicMin(&a.fail_key[b], (k << 4) | rc);
    return;
  }

  // stage the 15x29 block, then w = x_end - A x_k - B- u_k - B+ u_k1 row by row in the
  // reference's order (discretizer.hpp:144-147)
  if (lane < kCols) {
#pragma unroll
    for (int i = 0; i < kNX; ++i) ws.block[i * kStageStride + lane] = col[i];
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < kNX; ++i) ws.xe[i] = x_end[i];
  }
  __syncwarp();
  const size_t iv = (size_t)b * M + k;
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
    a.x_end[iv * kNX + lane] = ws.xe[lane];
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

void launch_linearize(const LinearizeArgs& a, cudaStream_t stream) {
  const long long warps = (long long)a.batch * (a.nodes - 1);
  const int ctas = (int)((warps + kWarpsPerCta - 1) / kWarpsPerCta);
  linearize_kernel<<<ctas, kWarpsPerCta * 32, 0, stream>>>(a);
}

}  // namespace ptopt_b200
