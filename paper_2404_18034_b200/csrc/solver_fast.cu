// solver_fast.cu — register-resident power iteration and customized PIPG for the rocket-shaped
// subproblem (n_x = 15, n_u = 7, A_plus = -I, e_y = unit vector of the last state, at most
// kFastMaxNodes nodes).
//
// One CTA per instance, five threads per node.  Thread (k, g) keeps rows 3g..3g+2 of the packed
// interval block [A-_k | B-_k | B+_k] (3 x 29 doubles) in registers for the whole kernel, so the
// operator is read from HBM exactly once per launch and never touches shared memory:
//   * the forward product  H z  (dual update / power-iteration forward map) is thread-local:
//     29 FMAs per row against the node vectors, which are broadcast from shared memory;
//   * the transposed product H^T phi uses the thread's own three dual entries: it forms the
//     29 partial column sums of its three rows and publishes them to shared memory, where the
//     owner of each primal entry adds the five partials of its column.
// Every primal/dual entry has one owner thread that keeps its extrapolated copy in registers;
// only what a neighbour needs (reflections, extrapolated duals, partial sums) lives in shared
// memory.  Two block-wide barriers per iteration.
//
// Follows /root/reference/proj/include/ptopt/pipg.hpp:206-292 (power_iteration_custom),
// :307-326 (stopping_custom), :335-340 (step_sizes), :350-497 (pipg_custom).  Sums over the
// fifteen rows of a column are grouped three rows at a time, and FMA contraction is on; both
// change rounding only (measured sensitivity of the whole loop: 1e-13).
#include <type_traits>

#include "kernels.cuh"

namespace ptopt_b200 {

namespace {

constexpr int kG = 5;        // threads per node
constexpr int kR = 3;        // operator rows per thread
constexpr int kW = kNX + 2 * kNU;  // 29 columns of [A- | B- | B+]
constexpr int kXS = 18;      // node stride of x vectors in shared memory (16-byte aligned, conflict-free)
constexpr int kUS = 10;      // node stride of u vectors
constexpr int kPS = 35;      // stride of one thread's partial-sum slot (== 3 mod 16: conflict-free)
constexpr int kFastThreads = 256;
constexpr int kFastWarps = kFastThreads / 32;
static_assert((kFastThreads - 1) / kG <= kFastMaxNodes, "every thread needs a (scratch) node inside the layout");
static_assert(kG * kFastMaxNodes <= kFastThreads, "five threads per node");

// position of a column's partial sum inside a slot: x columns first, then the B- / B+ columns
// interleaved so that the five owners of a node read with a 3-double spacing (no bank conflicts)
__host__ __device__ constexpr int pos_bm(int ju) { return ju < 5 ? 15 + 3 * ju : 16 + 3 * (ju - 5); }
__host__ __device__ constexpr int pos_bp(int ju) { return ju < 5 ? 17 + 3 * ju : 22 + 3 * (ju - 5); }
__host__ __device__ constexpr int pos_col(int j) {
  return j < kNX ? j : (j < kNX + kNU ? pos_bm(j - kNX) : pos_bp(j - kNX - kNU));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

/// Loads rows 3g..3g+2 of [A-_k | B-_k | B+_k] of instance b into registers.
__device__ __forceinline__ void load_rows(const SubArrays& sp, int b, int m, int k, int g,
                                          double (&a)[kR][kW]) {
  const size_t iv = (size_t)b * m + k;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const int i = kR * g + r;
    const double* ra = sp.A_minus + (iv * kNX + i) * kNX;
    const double* rm = sp.B_minus + (iv * kNX + i) * kNU;
    const double* rp = sp.B_plus + (iv * kNX + i) * kNU;
#pragma unroll
    for (int j = 0; j < kNX; ++j) a[r][j] = __ldg(ra + j);
#pragma unroll
    for (int j = 0; j < kNU; ++j) {
      a[r][kNX + j] = __ldg(rm + j);
      a[r][kNX + kNU + j] = __ldg(rp + j);
    }
  }
}

/// Reads the node vectors the forward product of interval k needs: x_k, u_k, u_{k+1}.
__device__ __forceinline__ void load_node_vectors(const double* xs_k, const double* us_k,
                                                  double (&v)[kW]) {
  const double2* x2 = reinterpret_cast<const double2*>(xs_k);
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    const double2 t = x2[q];
    v[2 * q] = t.x;
    v[2 * q + 1] = t.y;
  }
  v[14] = xs_k[14];
  const double2* u2 = reinterpret_cast<const double2*>(us_k);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double2 t = u2[q];  // entry 7 is padding
    v[kNX + 2 * q] = t.x;
    if (q < 3) v[kNX + 2 * q + 1] = t.y;
  }
  const double2* w2 = reinterpret_cast<const double2*>(us_k + kUS);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double2 t = w2[q];
    v[kNX + kNU + 2 * q] = t.x;
    if (q < 3) v[kNX + kNU + 2 * q + 1] = t.y;
  }
}

/// Row r of the forward product: A- x_k, B- u_k, B+ u_{k+1}, each summed in ascending column
/// order (mat_vec, smallmat.hpp:93-97).
__device__ __forceinline__ void row_products(const double (&a)[kR][kW], const double (&v)[kW], int r,
                                             double& pa, double& pm, double& pp) {
  double sa = 0.0, sm = 0.0, sp = 0.0;
#pragma unroll
  for (int j = 0; j < kNX; ++j) sa += a[r][j] * v[j];
#pragma unroll
  for (int j = 0; j < kNU; ++j) {
    sm += a[r][kNX + j] * v[kNX + j];
    sp += a[r][kNX + kNU + j] * v[kNX + kNU + j];
  }
  pa = sa;
  pm = sm;
  pp = sp;
}

/// Publishes the partial column sums of this thread's three rows against its three dual entries.
__device__ __forceinline__ void store_partials(const double (&a)[kR][kW], const double (&d)[kR],
                                               double* slot) {
#pragma unroll
  for (int j = 0; j < kW; ++j) {
    double p = a[0][j] * d[0];
    p += a[1][j] * d[1];
    p += a[2][j] * d[2];
    slot[pos_col(j)] = p;
  }
}

/// Sum over the five partial slots of an interval (part_k: its first slot) for one position.
__device__ __forceinline__ double column_sum(const double* part_k, int pos) {
  const double* p = part_k + pos;
  const double p0 = p[0], p1 = p[kPS], p2 = p[2 * kPS], p3 = p[3 * kPS], p4 = p[4 * kPS];
  return ((p0 + p1) + (p2 + p3)) + p4;  // short dependency chain; rounding-only change
}

struct FastLayout {
  int xs, us, phi, theta, part, red, total;  // offsets in doubles
  // PIPG only
  int wv, eps, umin, umax, snap, bnd;
};

// One snapshot of the *_cur groups (pipg.hpp:490-495), with room for the scratch entries the
// idle threads write: x [n+2][15], u [n+2][7 (+3)], vc+, vc-, dyn dual [n+2][15], relax dual [n+2].
struct SnapLayout {
  int x, u, vp, vn, ph, th, total;
};
__host__ __device__ constexpr SnapLayout snap_layout() {
  constexpr int n = kFastMaxNodes + 2;
  SnapLayout S{};
  int o = 0;
  S.x = o; o += n * kNX;
  S.u = o; o += n * kNU + 4;
  S.vp = o; o += n * kNX;
  S.vn = o; o += n * kNX;
  S.ph = o; o += n * kNX;
  S.th = o; o += n;
  S.total = (o + 1) & ~1;
  return S;
}

__host__ __device__ constexpr int even_up(int v) { return (v + 1) & ~1; }

// Arrays carry guard entries so that the hot loops need no boundary branches: node arrays have
// two extra nodes (n: scratch node of the idle threads, n+1: its right neighbour); interval
// arrays have one zero interval in front (index -1, read by node 0) and are sized for every
// thread; partial-sum slots exist for every thread plus five zero slots in front.
__host__ __device__ constexpr FastLayout fast_layout(bool pipg) {
  constexpr int n = kFastMaxNodes;  // fixed offsets: every address is base + immediate
  FastLayout L{};
  int o = 0;
  L.xs = o; o += (n + 2) * kXS;
  L.us = o; o += (n + 2) * kUS;
  L.phi = o + kNX + 1; o += even_up((n + 2) * kNX + 2);
  L.theta = o + 2; o += even_up(n + 4);
  L.part = o + kG * kPS + 1; o += even_up(kG * kPS + 1 + (n + 2) * kG * kPS);
  L.red = o; o += 16 * kFastWarps;
  if (pipg) {
    L.wv = o; o += even_up((n + 2) * kNX);
    L.eps = o; o += even_up(n + 2);
    L.umin = o; o += 2 * kFastThreads;  // {lo, hi} of each thread's first control entry
    L.umax = o; o += 2 * kFastThreads;  // {lo, hi} of its second one (+-inf where it has none)
    L.snap = o; o += 2 * snap_layout().total;
    L.bnd = o; o += 6 * 16;  // ecost, init_val, final_val, init_on, final_on (as doubles)
  }
  L.total = o;
  return L;
}

// ---------------------------------------------------------------------------------------------
// power iteration (pipg.hpp:206-292)
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kFastThreads, 1) power_fast_kernel(PowerArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  if (a.active && !a.active[b]) return;
  const int n = a.shape.n, m = n - 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = blockDim.x, nwarps = T >> 5;  // launched with just enough warps for 5 threads per node
  const int k = tid / kG, g = tid - k * kG;
  const bool node = k < n, ival = k < m;
  const int kc = k;  // threads past the last node work on scratch nodes of their own (layout has kFastMaxNodes + 2)
  constexpr FastLayout L = fast_layout(false);
  for (int e = tid; e < L.total; e += T) sm[e] = 0.0;
  __syncthreads();
  double* xs_k = sm + L.xs + kc * kXS;          // x_k; x_{k+1} at +kXS
  double* us_k = sm + L.us + kc * kUS;
  double* phi_k = sm + L.phi + kc * kNX + kR * g;  // own dual entries; interval k-1 at -kNX
  double* th_k = sm + L.theta + kc;
  double* part = sm + L.part;
  double* slot = part + (size_t)tid * kPS;
  const double* part_k = part + (size_t)kc * kG * kPS;  // slots of interval k; k-1 at -kG*kPS
  double* red = sm + L.red;
  const int ju1 = g + 5;                        // second control entry (g >= 2: a padding slot of its own)

  double aop[kR][kW];
  double vcp[kR], vcn[kR];
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    vcp[r] = vcn[r] = 0.0;
#pragma unroll
    for (int j = 0; j < kW; ++j) aop[r][j] = 0.0;
  }
  if (ival) load_rows(a.sp, b, m, k, g, aop);

  // seed (pipg.hpp:213-230): x, u, vc+, vc-; sigma0 = ||seed||_2
  double acc = 0.0;
  if (node) {
    const double* sx = a.seed_x + ((size_t)b * n + k) * kNX;
    const double* su = a.seed_u + ((size_t)b * n + k) * kNU;
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const double v = sx[kR * g + r];
      xs_k[kR * g + r] = v;
      acc += v * v;
    }
    {
      const double v = su[g];
      us_k[g] = v;
      acc += v * v;
    }
    if (g < 2) {
      const double v = su[g + 5];
      us_k[g + 5] = v;
      acc += v * v;
    }
  }
  if (ival) {
    const double* sp = a.seed_vcp + ((size_t)b * m + k) * kNX;
    const double* sn = a.seed_vcn + ((size_t)b * m + k) * kNX;
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      vcp[r] = sp[kR * g + r];
      vcn[r] = sn[kR * g + r];
      acc += vcp[r] * vcp[r];
      acc += vcn[r] * vcn[r];
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  double sigma = 0.0;
#pragma unroll
  for (int w = 0; w < kFastWarps; ++w) sigma += w < nwarps ? red[w] : 0.0;
  if (sigma == 0.0) {  // pipg.hpp:224-225
    if (tid == 0) {
      if (a.status) a.status[b] = kStSeedZero;
      a.sigma[b] = 0.0;
      if (a.trips) a.trips[(size_t)b * a.trips_stride + (a.trips_slot ? a.trips_slot[b] : 0)] = 0;
    }
    return;
  }
  sigma = sqrt(sigma);

  // The norm of trip j-1 is reduced while trip j's forward products are already running: the
  // products do not need sigma until they are scaled, so the block reduction, the square root
  // and the reciprocal overlap with them instead of forming a serial stage of their own.
  int trips = 0;
  bool done = false;
  for (int j = 1; j <= a.j_max; ++j) {
    // ---- forward map (pipg.hpp:234-245): products first, then the scale 1/sigma
    double v[kW];
    load_node_vectors(xs_k, us_k, v);
    double s[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      double pa, pm, pp;
      row_products(aop, v, r, pa, pm, pp);
      double t = pa + -xs_k[kXS + kR * g + r];
      t += pm;
      t += pp;
      t += vcp[r];
      t += -1.0 * vcn[r];
      s[r] = t;
    }
    const double dy = xs_k[kXS + 14] - v[14];
    if (j > 1) {  // stopping test of trip j-1 (pipg.hpp:277-289)
      const double* rd = red + (((j - 1) & 1) ? kFastWarps : 0);
      double sq = 0.0;
#pragma unroll
      for (int w = 0; w < kFastWarps; ++w) sq += w < nwarps ? rd[w] : 0.0;
      const double sigma_star = sqrt(sq);
      if (sigma_star == 0.0) {  // iterate in the null space, pipg.hpp:280-284
        sigma = 0.0;
        done = true;
        break;
      }
      const bool hit = fabs(sigma_star - sigma) <= a.eps_abs + a.eps_rel * fmax(sigma_star, sigma);
      sigma = sigma_star;
      if (hit) {
        done = true;
        break;
      }
    }
    trips = j;
    const double inv = 1.0 / sigma;
    double phi[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      phi[r] = ival ? s[r] * inv : 0.0;
      phi_k[r] = phi[r];
    }
    if (g == 4) th_k[0] = ival ? dy / sigma : 0.0;
    store_partials(aop, phi, slot);
    // vc+ = phi, vc- = -phi and their share of the norm (pipg.hpp:268-279)
    double acc_d = 0.0;
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      vcp[r] = phi[r];
      vcn[r] = -phi[r];
      acc_d += phi[r] * phi[r];
      acc_d += phi[r] * phi[r];
    }
    __syncthreads();
    // ---- adjoint map (pipg.hpp:247-275): every primal entry is assembled by its owner
    double sx[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) sx[r] = column_sum(part_k, kR * g + r);
    const double su0 = column_sum(part_k, 15 + 3 * g) + column_sum(part_k - kG * kPS, 17 + 3 * g);
    const double su1 = column_sum(part_k, 16 + 3 * g) + column_sum(part_k - kG * kPS, 22 + 3 * g);
    double acc_x = 0.0;
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      double t = sx[r] + -phi_k[r - kNX];
      if (r == kR - 1 && g == 4) {
        t += -th_k[0];
        t += th_k[-1];
      }
      xs_k[kR * g + r] = t;
      acc_x += t * t;
    }
    us_k[g] = su0;
    us_k[ju1] = su1;
    double acc_u = su0 * su0;
    acc_u += g < 2 ? su1 * su1 : 0.0;
    acc = node ? (acc_x + acc_u) + acc_d : 0.0;
    acc = warp_sum(acc);
    if (lane == 0) red[((j & 1) ? kFastWarps : 0) + warp] = acc;
    __syncthreads();
  }
  if (!done) {  // j_max trips without meeting the tolerance: sigma is the last norm
    const double* rd = red + ((a.j_max & 1) ? kFastWarps : 0);
    double sq = 0.0;
#pragma unroll
    for (int w = 0; w < kFastWarps; ++w) sq += w < nwarps ? rd[w] : 0.0;
    sigma = sqrt(sq);
  }
  if (tid == 0) {
    a.sigma[b] = (1.0 + a.eps_buff) * sigma;
    if (a.trips) a.trips[(size_t)b * a.trips_stride + (a.trips_slot ? a.trips_slot[b] : 0)] = trips;
  }
}

// ---------------------------------------------------------------------------------------------
// customized PIPG (pipg.hpp:350-497)
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kFastThreads, 1) pipg_fast_kernel(PipgArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  if (a.active && !a.active[b]) return;
  const int n = a.shape.n, m = n - 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = blockDim.x, nwarps = T >> 5;  // launched with just enough warps for 5 threads per node
  const int k = tid / kG, g = tid - k * kG;
  const bool node = k < n, ival = k < m;
  const int kc = k;  // threads past the last node work on scratch nodes of their own (layout has kFastMaxNodes + 2)
  constexpr FastLayout L = fast_layout(true);
  constexpr SnapLayout S = snap_layout();
  for (int e = tid; e < L.total; e += T) sm[e] = 0.0;
  __syncthreads();
  double* xr_k = sm + L.xs + kc * kXS;   // reflections 2*cur - ex (pipg.hpp:436-443); k+1 at +kXS
  double* ur_k = sm + L.us + kc * kUS;
  double* phx_k = sm + L.phi + kc * kNX + kR * g;  // extrapolated dynamics dual; k-1 at -kNX
  double* thx_k = sm + L.theta + kc;               // extrapolated relaxation dual
  double* part = sm + L.part;
  double* slot = part + (size_t)tid * kPS;
  const double* part_k = part + (size_t)kc * kG * kPS;
  double* red = sm + L.red;
  const double* wv_k = sm + L.wv + kc * kNX + kR * g;
  const double* eps_k = sm + L.eps + kc;
  double2* bnd0 = reinterpret_cast<double2*>(sm + L.umin) + tid;  // conflict-free 16-byte slots
  double2* bnd1 = reinterpret_cast<double2*>(sm + L.umax) + tid;
  double* snap0 = sm + L.snap;  // two snapshots of the *_cur groups, written alternately
  double* ecost = sm + L.bnd;
  double* init_val = ecost + 16;
  double* final_val = init_val + 16;
  double* init_on = final_val + 16;
  double* final_on = init_on + 16;
  const int ju1 = g + 5;  // second control entry (g >= 2: a padding slot of its own)

  const int NXn = n * kNX, NUn = n * kNU, NM = m * kNX;
  if (tid < kNX) ecost[tid] = a.shape.e_cost[tid];
  if (tid == 0) {
    // later entries override earlier ones, as the assignment loops do (pipg.hpp:408-413)
    for (int i = 0; i < a.shape.n_init_fix; ++i) {
      init_on[a.shape.init_fix_idx[i]] = 1.0;
      init_val[a.shape.init_fix_idx[i]] = a.sp.init_fix_val[(size_t)b * a.shape.n_init_fix + i];
    }
    for (int i = 0; i < a.shape.n_final_fix; ++i) {
      final_on[a.shape.final_fix_idx[i]] = 1.0;
      final_val[a.shape.final_fix_idx[i]] = a.sp.final_fix_val[(size_t)b * a.shape.n_final_fix + i];
    }
  }
  for (int e = tid; e < NM; e += T) sm[L.wv + e] = a.sp.w[(size_t)b * NM + e];
  for (int e = tid; e < m; e += T) sm[L.eps + e] = a.sp.eps_relax[(size_t)b * m + e];
  {  // box of this thread's control entries (pipg.hpp:418-419); scratch entries are unbounded
    const double* lo = a.sp.u_min + (size_t)b * NUn + k * kNU;
    const double* hi = a.sp.u_max + (size_t)b * NUn + k * kNU;
    *bnd0 = node ? make_double2(lo[g], hi[g]) : make_double2(-INFINITY, INFINITY);
    *bnd1 = (node && g < 2) ? make_double2(lo[g + 5], hi[g + 5]) : make_double2(-INFINITY, INFINITY);
  }
  // warm start: ex = cur = workspace (pipg.hpp:362-374); it is snapshot 0
  for (int e = tid; e < NXn; e += T) snap0[S.x + e] = a.ws.x[(size_t)b * NXn + e];
  for (int e = tid; e < NUn; e += T) snap0[S.u + e] = a.ws.u[(size_t)b * NUn + e];
  for (int e = tid; e < NM; e += T) {
    snap0[S.vp + e] = a.ws.vc_pos[(size_t)b * NM + e];
    snap0[S.vn + e] = a.ws.vc_neg[(size_t)b * NM + e];
    snap0[S.ph + e] = a.ws.dyn_dual[(size_t)b * NM + e];
  }
  for (int e = tid; e < m; e += T) snap0[S.th + e] = a.ws.relax_dual[(size_t)b * m + e];

  double aop[kR][kW];
#pragma unroll
  for (int r = 0; r < kR; ++r)
#pragma unroll
    for (int j = 0; j < kW; ++j) aop[r][j] = 0.0;
  if (ival) load_rows(a.sp, b, m, k, g, aop);
  __syncthreads();

  // boundary rows of this thread (pipg.hpp:408-413): bit r set when row 3g+r is assigned
  int fix_bits = 0;
  const double* fix_val = init_val;
  if (k == 0 || k == n - 1) {
    const double* on = k == n - 1 ? final_on : init_on;
    fix_val = k == n - 1 ? final_val : init_val;
#pragma unroll
    for (int r = 0; r < kR; ++r)
      if (on[kR * g + r] != 0.0) fix_bits |= 1 << r;
  }
  const bool last_node = k == n - 1;
  const bool warp_fix = __any_sync(0xffffffffu, fix_bits != 0);  // warp-uniform

  // owner-private extrapolated copies
  double xe[kR], ue[2], vpe[kR], vne[kR], phe[kR], the = 0.0;
  ue[0] = ue[1] = 0.0;
#pragma unroll
  for (int r = 0; r < kR; ++r) xe[r] = vpe[r] = vne[r] = phe[r] = 0.0;
  if (node) {
#pragma unroll
    for (int r = 0; r < kR; ++r) xe[r] = snap0[S.x + k * kNX + kR * g + r];
    ue[0] = snap0[S.u + k * kNU + g];
    if (g < 2) ue[1] = snap0[S.u + k * kNU + g + 5];
  }
  if (ival) {
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const int e = k * kNX + kR * g + r;
      vpe[r] = snap0[S.vp + e];
      vne[r] = snap0[S.vn + e];
      phe[r] = snap0[S.ph + e];
      phx_k[r] = phe[r];
    }
    if (g == 4) {
      the = snap0[S.th + k];
      thx_k[0] = the;
    }
  }
  store_partials(aop, phe, slot);

  const double sigma = a.sigma[b];
  const double alpha = 2.0 / (a.shape.w_prox + sqrt(a.shape.w_prox * a.shape.w_prox + 4.0 * a.omega * sigma));
  const double beta = a.omega * alpha;
  const double one_m_rho = 1.0 - a.rho;
  __syncthreads();

  // One iteration.  kStore additionally writes the new *_cur values of every owner into the
  // snapshot `snap` (threads without a node / interval write scratch entries).
  auto iteration = [&](auto store_tag, double* snap) {
    constexpr bool kStore = decltype(store_tag)::value;
    // ---- primal projected-gradient step (pipg.hpp:388-420) by the owner of each entry.  The
    //      terms that do not need the partial sums are gathered first so that the dependent
    //      chain behind the shared-memory loads stays short.
    double base[kR], fv[kR], sx[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const int i = kR * g + r;
      fv[r] = warp_fix ? fix_val[i] : 0.0;
      double t = xe[r] * a.shape.w_prox;
      if (last_node) t += a.shape.w_cost * ecost[i];
      t += -phx_k[r - kNX];
      if (r == kR - 1 && g == 4) t += thx_k[-1] - thx_k[0];
      base[r] = t;
    }
#pragma unroll
    for (int r = 0; r < kR; ++r) sx[r] = column_sum(part_k, kR * g + r);
    double su[2], lo[2], hi[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int ju = q == 0 ? g : ju1;
      const double2 bq = q == 0 ? *bnd0 : *bnd1;
      lo[q] = bq.x;
      hi[q] = bq.y;
      su[q] = column_sum(part_k, q == 0 ? 15 + 3 * g : 16 + 3 * g) +
              column_sum(part_k - kG * kPS, q == 0 ? 17 + 3 * g : 22 + 3 * g);
    }
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const int i = kR * g + r;
      const double x0 = xe[r];
      const double grad = base[r] + sx[r];
      double xn = x0 + -alpha * grad;
      xn = (fix_bits & (1 << r)) ? fv[r] : xn;
      xr_k[i] = fma(2.0, xn, -x0);
      if (kStore) snap[S.x + kc * kNX + i] = xn;
      xe[r] = one_m_rho * x0 + a.rho * xn;  // extrapolation, pipg.hpp:461-467
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int ju = q == 0 ? g : ju1;
      const double u0 = ue[q];
      const double grad = u0 * a.shape.w_prox + su[q];
      double un = u0 + -alpha * grad;
      // std::max(lo, std::min(hi, v)), pipg.hpp:418-419
      const double cl = (hi[q] < un) ? hi[q] : un;
      un = (lo[q] < cl) ? cl : lo[q];
      ur_k[ju] = fma(2.0, un, -u0);
      if (kStore) {
        if (q == 0 || g < 2) snap[S.u + kc * kNU + ju] = un;
      }
      ue[q] = one_m_rho * u0 + a.rho * un;
    }
    __syncthreads();

    // ---- slacks (pipg.hpp:423-430), PI feedback of the constraint violation (:433-458),
    //      extrapolation of the dual groups (:468-472) and the partial sums of H^T phi_ex for
    //      the next primal step
    {
      double v[kW];
      load_node_vectors(xr_k, ur_k, v);
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        double pa, pm, pp;
        row_products(aop, v, r, pa, pm, pp);
        double resid = pa + -xr_k[kXS + kR * g + r];
        resid += pm;
        resid += pp;
        const double p0 = phe[r], vp0 = vpe[r], vn0 = vne[r];
        const double vp = fmax(0.0, vp0 - alpha * (a.shape.w_ep + p0));
        const double vn = fmax(0.0, vn0 - alpha * (a.shape.w_ep - p0));
        resid += (2.0 * vp - vp0) - (2.0 * vn - vn0) + wv_k[r];
        const double pn = p0 + beta * resid;
        if (kStore) {
          const int e = kc * kNX + kR * g + r;
          snap[S.vp + e] = vp;
          snap[S.vn + e] = vn;
          snap[S.ph + e] = pn;
        }
        const double pe = one_m_rho * p0 + a.rho * pn;
        phe[r] = ival ? pe : 0.0;
        vpe[r] = one_m_rho * vp0 + a.rho * vp;
        vne[r] = one_m_rho * vn0 + a.rho * vn;
        phx_k[r] = phe[r];
      }
      if (g == 4) {
        const double drift = xr_k[kXS + 14] - v[14] - eps_k[0];
        const double tn = fmax(0.0, the + beta * drift);
        if (kStore) snap[S.th + kc] = tn;
        the = ival ? one_m_rho * the + a.rho * tn : 0.0;
        thx_k[0] = the;
      }
      store_partials(aop, phe, slot);
    }
  };

  int iters = 0, cur_set = 0;  // snapshot holding the latest materialised *_cur groups
  bool converged = false, diverged = false;
  int to_check = a.j_check;  // iterations left until the next stopping test (counts down to 0)
  for (int j = 1; j <= a.j_max; ++j) {
    --to_check;
    const bool check = to_check == 0;
    // cur values are materialised when the next iteration checks against them, when this one
    // checks (a converged exit returns them), and on the last iteration
    const bool keep = to_check <= 1 || j == a.j_max;
    if (check) to_check = a.j_check;
    if (keep) {
      cur_set ^= 1;
      iteration(std::true_type{}, snap0 + cur_set * S.total);
    } else {
      iteration(std::false_type{}, nullptr);
    }
    iters = j;
    __syncthreads();
    if (check) {  // stopping_custom(cur, prev) and the divergence test, pipg.hpp:475-487
      const double* cur = snap0 + cur_set * S.total;
      const double* prev = snap0 + (cur_set ^ 1) * S.total;
      double z_cur = 0.0, z_prev = 0.0, z_del = 0.0, r_cur = 0.0, r_prev = 0.0, r_del = 0.0;
      double bad = 0.0;
      auto primal = [&](int off, int count, bool finite_checked) {
        for (int e = tid; e < count; e += T) {
          const double c = cur[off + e], o = prev[off + e];
          z_cur = fmax(z_cur, fabs(c));
          z_prev = fmax(z_prev, fabs(o));
          z_del = fmax(z_del, fabs(c - o));
          if (finite_checked && !pt_finite(c)) bad = 1.0;
        }
      };
      auto dual = [&](int off, int count, bool finite_checked) {
        for (int e = tid; e < count; e += T) {
          const double c = cur[off + e], o = prev[off + e];
          r_cur = fmax(r_cur, fabs(c));
          r_prev = fmax(r_prev, fabs(o));
          r_del = fmax(r_del, fabs(c - o));
          if (finite_checked && !pt_finite(c)) bad = 1.0;
        }
      };
      primal(S.x, NXn, true);
      primal(S.u, NUn, true);
      primal(S.vp, NM, false);
      primal(S.vn, NM, false);
      dual(S.ph, NM, true);
      dual(S.th, m, false);
      z_cur = warp_max(z_cur); z_prev = warp_max(z_prev); z_del = warp_max(z_del);
      r_cur = warp_max(r_cur); r_prev = warp_max(r_prev); r_del = warp_max(r_del);
      bad = warp_max(bad);
      if (lane == 0) {
        double* rw = red + warp * 8;
        rw[0] = z_cur; rw[1] = z_prev; rw[2] = z_del; rw[3] = r_cur; rw[4] = r_prev; rw[5] = r_del;
        rw[6] = bad;
      }
      __syncthreads();
      double v[7];
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        double mx = 0.0;
#pragma unroll
        for (int w = 0; w < kFastWarps; ++w) mx = fmax(mx, w < nwarps ? red[w * 8 + q] : 0.0);
        v[q] = mx;
      }
      __syncthreads();  // red and the snapshots are rewritten later
      if (v[6] > 0.0) {
        diverged = true;
        break;
      }
      if (v[2] <= a.eps_abs + a.eps_rel * fmax(v[0], v[1]) &&
          v[5] <= a.eps_abs + a.eps_rel * fmax(v[3], v[4])) {
        converged = true;
        break;
      }
    }
  }

  if (diverged) {  // SolverDiverged(j): the workspace is left untouched, pipg.hpp:478
    if (tid == 0) {
      if (a.status) a.status[b] = kStSolverDiverged;
      if (a.fail_index) a.fail_index[b] = iters;
      if (a.iterations) a.iterations[b] = iters;
      if (a.converged) a.converged[b] = 0;
      if (a.active) a.active[b] = 0;
    }
    return;
  }
  // solution = the *_cur groups, pipg.hpp:490-495 (all threads passed a barrier after the last
  // snapshot write)
  const double* cur = snap0 + cur_set * S.total;
  for (int e = tid; e < NXn; e += T) a.ws.x[(size_t)b * NXn + e] = cur[S.x + e];
  for (int e = tid; e < NUn; e += T) a.ws.u[(size_t)b * NUn + e] = cur[S.u + e];
  for (int e = tid; e < NM; e += T) {
    a.ws.vc_pos[(size_t)b * NM + e] = cur[S.vp + e];
    a.ws.vc_neg[(size_t)b * NM + e] = cur[S.vn + e];
    a.ws.dyn_dual[(size_t)b * NM + e] = cur[S.ph + e];
  }
  for (int e = tid; e < m; e += T) a.ws.relax_dual[(size_t)b * m + e] = cur[S.th + e];
  if (tid == 0) {
    if (a.iterations) a.iterations[b] = iters;
    if (a.converged) a.converged[b] = converged ? 1 : 0;
  }
}

}  // namespace

bool solver_fast_supports(const SubShape& s, bool has_a_plus) {
  if (has_a_plus || s.nx != kNX || s.nu != kNU) return false;
  if (s.n < 2 || s.n > kFastMaxNodes) return false;
  for (int i = 0; i < kNX; ++i)
    if (s.e_y[i] != (i == kNX - 1 ? 1.0 : 0.0)) return false;
  return true;
}

size_t power_fast_smem(const SubShape&) { return sizeof(double) * (size_t)fast_layout(false).total; }
size_t pipg_fast_smem(const SubShape&) { return sizeof(double) * (size_t)fast_layout(true).total; }

cudaError_t configure_solver_fast(const SubShape& s) {
  cudaError_t e = cudaFuncSetAttribute(power_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)power_fast_smem(s));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(pipg_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)pipg_fast_smem(s));
}

/// Just enough warps for five threads per node (the kernels size their loops by blockDim).
static int fast_threads(const SubShape& s) { return ((kG * s.n + 31) / 32) * 32; }

cudaError_t launch_power_fast(const PowerArgs& a, cudaStream_t stream) {
  power_fast_kernel<<<a.batch, fast_threads(a.shape), power_fast_smem(a.shape), stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pipg_fast(const PipgArgs& a, cudaStream_t stream) {
  pipg_fast_kernel<<<a.batch, fast_threads(a.shape), pipg_fast_smem(a.shape), stream>>>(a);
  return cudaGetLastError();
}

}  // namespace ptopt_b200
