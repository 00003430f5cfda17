// linearize.cu — exact discretization: batched linearize_all
// (/root/reference/proj/include/ptopt/discretizer.hpp:191-232) in two passes over every
// (instance, interval):
//   * state pass   — one THREAD per interval integrates the 15 augmented states through the
//                    4 * steps RK4 stages (the only place the model and its Jacobian are
//                    evaluated) and leaves one 84-double record per stage in HBM;
//   * column pass  — one lane per column of [Phi_x | Phi_u- | Phi_u+] (29 per interval); the four
//                    warps of a CTA take four neighbouring intervals -- two warps their Phi_x
//                    columns, two their Phi_u columns, each warp two intervals side by side --
//                    whose records of a stage form one contiguous chunk: the CTA copies it
//                    with coalesced asynchronous copies three stages ahead, every 8-byte word
//                    straight to its place in the slab of its interval (rocket_model.cuh); each
//                    lane applies A(tau) and the B forcing to its column in registers; then the
//                    15 x 29 block is staged in shared memory for w = x_end - A x - B- u - B+ u+
//                    and the coalesced write.
// See rocket_model.cuh for the per-thread / per-lane algorithms.
#include <type_traits>

#include "kernels.cuh"
#include "rocket_model.cuh"

namespace ptopt_b200 {

namespace {

constexpr int kWarpsPerCta = 4;
constexpr int kStageStride = kCols + 1;  // 30: row stride of the staged [15][29] block

// Records of kWarpsPerCta (4) consecutive intervals are interleaved word by word, one contiguous
// chunk of 4 * kRecSize doubles per (tile, stage): the state pass -- one thread per interval --
// fills whole 32-byte sectors with the four lanes of a tile, and a column-pass CTA (one tile) reads
// a stage as one contiguous 2 688-byte piece.
constexpr int kTile = kWarpsPerCta;
constexpr int kChunk = kTile * kRecSize;  // doubles per (tile, stage)
__host__ __device__ inline size_t record_index(long long local_interval, int nst, int stage_no) {
  const long long tile = local_interval / kTile;
  const int r = (int)(local_interval - tile * kTile);
  return ((size_t)tile * nst + stage_no) * kChunk + r;
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
  // every field goes straight from the register it was computed in to its place in the tile's chunk
  double* out0 = out + record_index(local, nst, 0);
  const int rc = propagate_state_pass(P, xk, uk, uk1, tau_k, tau_k1, a.steps, x_end, [&](int stage_no, int field, double v) {
    out0[(size_t)stage_no * kChunk + (size_t)field * kTile] = v;
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

constexpr int kRecRing = 4;  // stage slabs in flight per warp (cp.async ring)

struct __align__(16) WarpSmem {
  double slab[kRecRing][kSlabSize];  // ring of stage slabs (records with the B entries scattered, rocket_model.cuh)
  double block[kNX * kStageStride];  // staged [A | B- | B+], row-major
  double xk[kNX], uk[kNU], uk1[kNU], xe[kNX];
};

__global__ void __launch_bounds__(kWarpsPerCta * 32, 3)
column_pass_kernel(LinearizeArgs a, long long first, long long count) {
  __shared__ WarpSmem smem[kWarpsPerCta];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int M = a.nodes - 1;
  // Interval t of the tile: is there work (inside the range, instance neither finished nor failed)?
  // An interval without work still has its records copied and its columns computed (on whatever
  // the slab holds); nothing is stored for it.
  auto locate = [&](int t, int& b, int& k) {
    const long long local = (long long)blockIdx.x * kTile + t;
    b = k = 0;
    if (local >= count) return false;
    const long long widx = first + local;
    b = (int)(widx / M);
    k = (int)(widx - (long long)b * M);
    if (a.active && !a.active[b]) return false;  // instance already finished (SCP loop)
    // an instance with a failed interval has no blocks (its records stop at the failure)
    return a.fail_key[b] == kFailKeyNone;
  };
  // Roles.  Shared memory serves requested bytes, and the 32 A scalars of a stage are the bulk of
  // what a lane reads; a warp therefore works on TWO intervals, one per half warp (the sixteen
  // lanes of a half read one address: a broadcast), and warps are uniform in what their columns
  // need: warps 0, 1 own the Phi_x columns (no forcing: they never touch the B part of a slab),
  // warps 2, 3 the Phi_u- | Phi_u+ columns.  Afterwards warp w assembles and stores interval w.
  const bool u_role = wib >= 2;
  const int half = lane >> 4, l16 = lane & 15;
  const int mine = 2 * (wib & 1) + half;                      // interval of the tile this lane works on
  const bool is_col = u_role ? l16 < 2 * kNU : l16 < kNX;
  const int col = !is_col ? 31 : (u_role ? kNX + l16 : l16);  // column of [Phi_x | Phi_u- | Phi_u+]; 31: a zero dummy
  int b, k, bm, km;
  const bool alive = locate(wib, b, k);
  const bool alive_mine = locate(mine, bm, km);
  if (!__syncthreads_or(alive)) return;

  WarpSmem& ws = smem[wib];
  const size_t iv = (size_t)b * M + k;
  const double* xg = a.x + ((size_t)b * a.nodes + k) * kNX;
  const double* ug = a.u + ((size_t)b * a.nodes + k) * kNU;
  if (alive && lane < kNX) {
    ws.xk[lane] = xg[lane];
    ws.xe[lane] = a.x_end[iv * kNX + lane];
  }
  if (alive && lane < kNU) {
    ws.uk[lane] = ug[lane];
    ws.uk1[lane] = ug[kNU + lane];
  }
  // the entries of a slab no record field lands on (the zeros of the dense B) are cleared once
  for (int e = lane; e < kRecRing * kSlabSize; e += 32) (&ws.slab[0][0])[e] = 0.0;
  __syncthreads();  // before any thread's copies land in another warp's slabs

  double h = 0.0;
  if (alive_mine) {
    const double* tau = a.tau + (size_t)bm * a.tau_stride;
    h = (tau[km + 1] - tau[km]) / a.steps;
  }
  const double h6 = h / 6.0, h3 = h / 3.0, hh = 0.5 * h;  // as stage_time forms them
  const int nst = 4 * a.steps;
  // Stage `sn` of the tile: kChunk consecutive words; thread t copies words t, t + 128, t + 256
  // (coalesced), word w = field w / 4 of interval w % 4, to slab_dest(field) of that interval's
  // ring slot sn % kRecRing.  One commit group per stage (an empty group past the last stage keeps
  // the counting uniform).
  const double* chunk0 = a.stages + (size_t)blockIdx.x * nst * kChunk + threadIdx.x;
  constexpr int kThreads = kWarpsPerCta * 32;
  constexpr int kCopies = (kChunk + kThreads - 1) / kThreads;
  unsigned dst[kCopies];
#pragma unroll
  for (int c = 0; c < kCopies; ++c) {
    const int w = threadIdx.x + c * kThreads;
    const int field = w < kChunk ? w / kTile : kRecSize - 1;
    dst[c] = (unsigned)__cvta_generic_to_shared(&smem[w % kTile].slab[0][slab_dest(field)]);
  }
  const bool last_copy = threadIdx.x + (kCopies - 1) * kThreads < kChunk;
  auto fetch = [&](int sn) {
    if (sn < nst) {
      const double* src = chunk0 + (size_t)sn * kChunk;
      const unsigned ring = (unsigned)(sn % kRecRing) * (unsigned)(kSlabSize * sizeof(double));
#pragma unroll
      for (int c = 0; c < kCopies; ++c)
        if (c + 1 < kCopies || last_copy)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst[c] + ring), "l"(src + c * kThreads) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int sn = 0; sn < kRecRing - 1; ++sn) fetch(sn);

  ColumnLane L;
  column_init(L, col);
  ColumnForcing Fc;
  forcing_init(a.model, col, Fc);
  const double* my_slabs = &smem[mine].slab[0][0];
  // one stage: wait for this thread's copies of its chunk, meet the CTA (every copy of the chunk
  // has landed, and every warp is done with the stage before), start the copies of the stage
  // kRecRing - 1 ahead into the slot that was read last, apply the slab to the column
  auto run_stage = [&](auto stage_tag, int sn, double wk, double wn) {
    constexpr int kStage = decltype(stage_tag)::value;
    asm volatile("cp.async.wait_group %0;" ::"n"(kRecRing - 2) : "memory");
    __syncthreads();
    fetch(sn + kRecRing - 1);
    const double* slab = my_slabs + (sn % kRecRing) * kSlabSize;
    if (u_role) column_stage_slab<kStage, true>(L, Fc, slab, wk, wn);
    else column_stage_slab<kStage, false>(L, Fc, slab, wk, wn);
  };
  for (int step = 0; step < a.steps; ++step) {
    run_stage(std::integral_constant<int, 0>{}, 4 * step, h6, hh);
    run_stage(std::integral_constant<int, 1>{}, 4 * step + 1, h3, hh);
    run_stage(std::integral_constant<int, 2>{}, 4 * step + 2, h3, h);
    run_stage(std::integral_constant<int, 3>{}, 4 * step + 3, h6, hh);
  }

  // stage the 15x29 blocks (every lane into the block of the interval it worked on), then warp w
  // forms w = x_end - A x_k - B- u_k - B+ u_k1 of interval w row by row in the reference's order
  // (discretizer.hpp:144-147) and writes its block
  if (is_col) {
    double* blk = smem[mine].block;
#pragma unroll
    for (int i = 0; i < kNX; ++i) blk[i * kStageStride + col] = L.s_c[i];
  }
  __syncthreads();
  if (!alive) return;
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
  const long long tiles = (intervals + 31) / 32;  // capacity in whole state-pass warps (a multiple of kTile)
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
