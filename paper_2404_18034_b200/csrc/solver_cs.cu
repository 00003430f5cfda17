// solver_cs.cu — "column-sparse" register-resident power iteration and customized PIPG for the
// rocket-shaped subproblem (n_x = 15, n_u = 7, A_plus = -I, e_y = unit vector of the last state,
// at most kCsMaxNodes nodes), exploiting the structural zeros of the exact discretization.
//
// Mapping.  One CTA per instance, FOUR threads per node, and the four threads of a node sit in
// four DIFFERENT warps: warp (role, half) holds role `role` of 32 consecutive nodes, lane = node.
// A role is a fixed set of COLUMNS of the packed interval block [A-_k | B-_k | B+_k] (all rows of
// those columns) together with the primal entries these columns multiply:
//     role 0: x columns q0 r0 r1 r2 y     u columns T0 T1      dual rows r0 r1 r2 (+ relaxation dual)
//     role 1: x columns q1 m v2           u columns T2 tau0    dual rows q1 m v2 q0
//     role 2: x columns q2 q3             u columns tau1 tau2  dual rows q2 q3 w2 y
//     role 3: x columns w0 w1 w2 v0 v1    u column  s          dual rows w0 w1 v0 v1
// Because every lane of a warp has the same role, the zero pattern of a role's columns is a
// compile-time pattern of its instruction stream: the state-transition matrix of the 6-DoF model
// (state m, r, v, q, w, y) is block triangular -- the column of r_i only reaches r_i and y, that of
// v_i only r_i, v_i, y, the quaternion columns reach r, v, q, y, the rate columns everything but m,
// the mass column m, r, v, y, the y column only y, and the torque columns never reach m
// (rocket6dof.hpp:318-375, ctcs.hpp:84-129; a pattern closed under the products of the RK4
// bundle, so the zeros are exact) -- 314 of the 435 entries of a block are structurally non-zero,
// 78..80 per thread.  The kernels VERIFY the pattern while they load the operator: an instance
// with a non-zero (or non-finite) entry outside it is left untouched for the dense kernels of
// solver_fast.cu, which run right behind on the instances not marked as handled.
//   * transposed product H^T phi: thread-local (a thread has whole columns); it reads the fifteen
//     duals of its interval from shared memory, [row][node] arrays, lane-contiguous: 2 wavefronts
//     per warp load, no bank conflicts, no broadcast waste;
//   * forward product H z: a thread multiplies its columns by its OWN primal entries (registers)
//     and publishes partial row sums for the rows other roles own; the row owner adds four partials;
//   * neighbour-node coupling along the horizon is a lane shift inside the warp (shuffles); the
//     boundary between the two warps of a role is covered by one redundantly computed halo node on
//     either side (lane 31 of the first warp repeats node 31, lane 0 of the second warp node 30),
//     so no value ever has to cross warps in the middle of a phase.
//   * above kCsMaxNodes nodes (up to kCsClusterMaxNodes) one instance runs over a CLUSTER of two
//     CTAs with the same trick across the cut: rank 0 carries a redundant copy of rank 1's first
//     node, rank 1 a copy of rank 0's last node (as the source of B+^T phi), and the only values
//     that cross are the duals of the two boundary intervals (and, in the power iteration, every
//     warp's share of the squared norm), stored into the partner's shared memory through mailboxes
//     (struct Cut, struct Port; mailbox.cuh).
//     These cluster variants are separate functions (power_role_x, pipg_role_x): the single-CTA
//     loops sit on a narrow optimum of instruction count and placement, and sharing one templated
//     body with the cluster code cost the single-CTA PIPG kernel 20 % (2 134 -> 2 556 ms per step).
// Two block barriers per iteration / trip, as in solver_fast.cu, but 0.4x the shared-memory
// wavefronts, 0.72x the FMAs and 360 / 400 instead of 397 / 540 instructions per warp and trip /
// iteration: 1 850 / 2 400 clk against 2 750 / 3 160 (B200, N = 50).  The four role bodies of a loop
// share the SM's 32 KB instruction cache; the PIPG loop (25.6 KB) only became faster than the dense
// kernel once it fitted, and its speed follows its instruction count: keep
// role-independent work (stopping test, set-up) in shared functions and out of the role bodies.
//
// Follows /root/reference/proj/include/ptopt/pipg.hpp:206-292 (power_iteration_custom),
// :307-326 (stopping_custom), :335-340 (step_sizes), :350-497 (pipg_custom).  Differences from the
// reference are rounding only: sums in a different order, FMA contraction, exact zeros skipped.
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include <cooperative_groups.h>

#include "kernels.cuh"
#include "mailbox.cuh"

namespace cg = cooperative_groups;

namespace ptopt_b200 {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kCsWarps = 16;  // slots of the per-warp reduction arrays (at most 14 warps)

// ---- structure of the operator ------------------------------------------------------------------
/// Rows (bit i = row i) a column of A- can reach.  State order: m | r0..2 | v0..2 | q0..3 | w0..2 | y.
__host__ __device__ constexpr unsigned xcol_mask(int c) {
  return c == 0    ? (0x007fu | 0x4000u)                       // m: m, r, v, y
         : c <= 3  ? ((1u << c) | 0x4000u)                     // r_i: r_i, y
         : c <= 6  ? ((1u << (c - 3)) | (1u << c) | 0x4000u)   // v_i: r_i, v_i, y
         : c <= 10 ? (0x07feu | 0x4000u)                       // q_j: r, v, q, y
         : c <= 13 ? 0x7ffeu                                   // w_j: everything but m
                   : 0x4000u;                                  // y: y
}
/// Rows a column of B- / B+ can reach.  Control order: T0..2 | tau0..2 | s.
__host__ __device__ constexpr unsigned ucol_mask(int c) { return (c >= 3 && c <= 5) ? 0x7ffeu : 0x7fffu; }

// The partition of the 29 columns (K = 4 roles: 8 warps, 255 registers, 78..80 operator entries per
// thread).  Partitions with more roles were measured and dropped: six roles
// (12 warps at 168 registers, 48..58 entries) are slower -- 49 % more warp instructions and twice the
// shared-memory wavefronts, because every role reads all fifteen duals and publishes its own
// partial sums; seven roles (14 warps) get 128 registers and spill.  A dual row is "aligned" when
// its owner also owns the primal entry of the same index: x_{k+1}[row] then arrives by a lane shift.
template <int K, int R>
struct RoleT;
template <>
struct RoleT<4, 0> {
  static constexpr int nxc = 5, nuc = 2, nrow = 3;
  __host__ __device__ static constexpr int xc(int j) { return j == 0 ? 7 : j == 4 ? 14 : j; }  // q0 r0 r1 r2 y
  __host__ __device__ static constexpr int uc(int j) { return j; }                                // T0 T1
  __host__ __device__ static constexpr int row(int r) { return 1 + r; }                           // r0 r1 r2
};
template <>
struct RoleT<4, 1> {
  static constexpr int nxc = 3, nuc = 2, nrow = 4;
  __host__ __device__ static constexpr int xc(int j) { return j == 0 ? 8 : j == 1 ? 0 : 6; }     // q1 m v2
  __host__ __device__ static constexpr int uc(int j) { return 2 + j; }                            // T2 tau0
  __host__ __device__ static constexpr int row(int r) { return r == 0 ? 8 : r == 1 ? 0 : r == 2 ? 6 : 7; }
};
template <>
struct RoleT<4, 2> {
  static constexpr int nxc = 2, nuc = 2, nrow = 4;
  __host__ __device__ static constexpr int xc(int j) { return 9 + j; }                            // q2 q3
  __host__ __device__ static constexpr int uc(int j) { return 4 + j; }                            // tau1 tau2
  __host__ __device__ static constexpr int row(int r) { return r == 0 ? 9 : r == 1 ? 10 : r == 2 ? 13 : 14; }
};
template <>
struct RoleT<4, 3> {
  static constexpr int nxc = 5, nuc = 1, nrow = 4;
  __host__ __device__ static constexpr int xc(int j) { return j < 3 ? 11 + j : 1 + j; }          // w0 w1 w2 v0 v1
  __host__ __device__ static constexpr int uc(int) { return 6; }                                  // s
  __host__ __device__ static constexpr int row(int r) { return r < 2 ? 11 + r : 2 + r; }          // w0 w1 v0 v1
};
/// Rows the columns of role R reach (union of its column masks).
template <int K, int R>
__host__ __device__ constexpr unsigned role_touch() {
  unsigned m = 0;
  for (int j = 0; j < RoleT<K, R>::nxc; ++j) m |= xcol_mask(RoleT<K, R>::xc(j));
  for (int j = 0; j < RoleT<K, R>::nuc; ++j) m |= ucol_mask(RoleT<K, R>::uc(j));
  return m;
}
template <int K>
__host__ __device__ constexpr unsigned role_touch_of(int r) {
  static_assert(K == 4, "one partition");
  return r == 0 ? role_touch<4, 0>() : r == 1 ? role_touch<4, 1>() : r == 2 ? role_touch<4, 2>() : role_touch<4, 3>();
}
/// Index of the x column of role R that equals row i (the row is "aligned": its owner also owns
/// the primal entry of the same index, so x_{k+1}[i] arrives by a lane shift), or -1.
template <int K, int R>
__host__ __device__ constexpr int aligned_col(int i) {
  for (int j = 0; j < RoleT<K, R>::nxc; ++j)
    if (RoleT<K, R>::xc(j) == i) return j;
  return -1;
}
/// True when role R owns dual row i.
template <int K, int R>
__host__ __device__ constexpr bool owns_row(int i) {
  for (int r = 0; r < RoleT<K, R>::nrow; ++r)
    if (RoleT<K, R>::row(r) == i) return true;
  return false;
}
// primal entries whose reflections a row owner of ANOTHER role needs from node k+1 go through
// shared memory: x[q0] (7, role 0 -> role 1), x[w2] (13, role 3 -> role 2), x[y] (14, role 0 -> role 2)
template <int K>
__host__ __device__ constexpr int xn_slot(int c) {
  return c == 7 ? 0 : c == 13 ? 1 : c == 14 ? 2 : -1;
}

// ---- shared-memory layout --------------------------------------------------------------------------
// [row][slot] arrays, slot = node + 1 (slot 0: the zero "node -1" / "interval -1" in front).
template <int K, int kHalves>
struct CsCfg {
  static constexpr int warps = K * kHalves;
  static constexpr int threads = 32 * warps;
  // nodes: the last lane never holds a node (the lane shift that fetches node k + 1 must find zeros
  // behind the last node), and two halves share two halo lanes
  static constexpr int cap = kHalves == 1 ? 31 : 61;
  static constexpr int S = kHalves == 1 ? 34 : 64;     // slots per row
};

struct SnapCs {
  int x, u, vp, vn, ph, th, total;
};
template <int K, int kHalves, int kExtra = 0>  // kExtra: rank 0's copy of the partner's first node
__host__ __device__ constexpr SnapCs snap_cs() {
  constexpr int n = CsCfg<K, kHalves>::cap + kExtra;
  SnapCs s{};
  int o = 0;
  s.x = o; o += n * kNX;
  s.u = o; o += n * kNU;
  s.vp = o; o += n * kNX;
  s.vn = o; o += n * kNX;
  s.ph = o; o += n * kNX;
  s.th = o; o += n;
  s.total = (o + 1) & ~1;
  return s;
}

struct CsLayout {
  int phi, th, part, xn, red, total;
  int wv, eps, bnd, fix, ecost, snap;  // PIPG only
};
template <int K, int kHalves>
__host__ __device__ constexpr CsLayout cs_layout(bool pipg, bool cluster = false) {
  constexpr int S = CsCfg<K, kHalves>::S;
  CsLayout L{};
  int o = 0;
  L.phi = o; o += kNX * S;
  L.th = o; o += S;
  L.part = o; o += K * kNX * S;
  L.xn = o; o += 3 * S;
  L.red = o; o += 8 * kCsWarps;  // power: [2][kCsWarps]; PIPG: [warps][8]
  if (pipg) {
    L.wv = o; o += kNX * S;
    L.eps = o; o += S;
    L.bnd = o; o += K * 2 * 2 * S;   // [role][u column][lo, hi][slot]
    L.fix = o; o += 4 * 16;          // init_val, final_val, init_on, final_on
    L.ecost = o; o += kNX * S;        // w_cost * e_cost at the last node's slot, zero elsewhere: [row][slot]
    L.snap = o; o += 2 * (cluster ? snap_cs<K, kHalves, 1>().total : snap_cs<K, kHalves>().total);
  }
  L.total = o;
  return L;
}

__device__ __forceinline__ void block_barrier() { asm volatile("bar.sync 0;" ::: "memory"); }
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

/// Which node a lane holds and in what capacity.
struct Lane {
  int k;        // node
  int slot;     // k + 1
  bool halo;    // a redundant copy of a node another warp owns
  bool auth;    // this thread is THE owner of node k (k < n, not a halo copy)
  bool primal;  // its primal entries are valid (owner, or the halo copy of node 31 in the first warp)
  bool ival;    // auth and k is an interval (k < n - 1)
};
template <int kHalves>
__device__ __forceinline__ Lane make_lane(int n, int half, int lane) {
  Lane t;
  if (kHalves == 1) {
    t.k = lane;
    t.halo = false;
    t.auth = t.k < n;
    t.primal = t.auth;
  } else {
    t.k = half == 0 ? lane : 30 + lane;
    t.halo = half == 0 ? lane == 31 : lane == 0;
    t.auth = !t.halo && t.k < n;
    t.primal = t.k < n && (half == 0 || lane != 0);
  }
  t.slot = t.k + 1;
  t.ival = t.auth && t.k < n - 1;
  return t;
}

/// The part of the horizon a CTA works on.  Without a cluster: everything.  In a cluster of two
/// (62..kCsClusterMaxNodes nodes) rank 0 owns nodes [0, c), c = ceil(n / 2), and
/// carries a redundant copy of node c behind its last node; rank 1 owns [c, n) and carries a copy of
/// node c - 1 in front of its first one (only as the source of B+^T phi of interval c - 1).  The
/// duals of the two boundary intervals are the only values that cross the cut (see Port).
struct Cut {
  int rank;  // CTA rank in the cluster
  int base;  // global node of local node 0
  int lo, hi;  // owned nodes [lo, hi)
  int hip;   // primal entries are maintained for nodes [lo, hip): hi + 1 in rank 0 of a cluster
};
template <bool kCluster>
__device__ __forceinline__ Cut make_cut(int n) {
  Cut c;
  if constexpr (kCluster) {
    const int mid = (n + 1) / 2;
    c.rank = (int)cg::this_cluster().block_rank();
    c.base = c.rank == 0 ? 0 : mid - 1;
    c.lo = c.rank == 0 ? 0 : mid;
    c.hi = c.rank == 0 ? mid : n;
    c.hip = c.rank == 0 ? mid + 1 : n;
  } else {
    c.rank = 0;
    c.base = 0;
    c.lo = 0;
    c.hi = c.hip = n;
  }
  return c;
}

/// Which node a lane of a cluster CTA holds and in what capacity (struct Lane with the cut).
struct LaneX {
  int k;        // node (global)
  int slot;     // local node + 1
  bool halo;    // a redundant copy of a node another warp owns
  bool auth;    // this thread is THE owner of node k (an owned node of this CTA, not a halo copy)
  bool primal;  // its primal entries are valid (owner, the halo copy of node 31 in the first warp, or
                // rank 0's copy of the first node of rank 1)
  bool pubx;    // it publishes the primal entries other roles read through shared memory
  bool ival;    // auth and k is an interval (k < n - 1)
  bool have;    // it loads the operator block of interval k
};
template <int kHalves>
__device__ __forceinline__ LaneX make_lane_cut(const Cut& c, int n, int half, int lane) {
  LaneX t;
  const int l = kHalves == 1 ? lane : (half == 0 ? lane : 30 + lane);
  t.k = c.base + l;
  t.halo = kHalves == 2 && (half == 0 ? lane == 31 : lane == 0);
  t.auth = !t.halo && t.k >= c.lo && t.k < c.hi;
  t.primal = t.k >= c.lo && t.k < c.hip && (kHalves == 1 || half == 0 || lane != 0);
  t.pubx = t.primal && !t.halo;
  t.slot = l + 1;
  t.ival = t.auth && t.k < n - 1;
  t.have = t.k < n - 1 && t.k <= c.hi;  // halo copies load their node's block too
  return t;
}

/// Hand-off between the two CTAs of a cluster (mailbox.cuh): per trip each CTA pushes the duals of
/// its boundary interval (fifteen rows and the relaxation dual, 128 bytes) into the partner's phi /
/// theta slots, and every warp its share of the squared norm into the partner's copy of `red`.
/// Nothing is read remotely in the loop.  The norm mailboxes alternate by trip parity (both CTAs
/// send every trip; a CTA is never two trips ahead, see solver_fast.cu).
struct Port {
  static constexpr int kBoxAt = 64;   // doubles into `red`: three mbarriers, then the pattern flag
  static constexpr int kPhiBytes = 8 * (kNX + 1);
  unsigned red;     // shared-memory address of the norm shares, held in a register
  unsigned box;     // [3] mbarriers (shared-memory address): phi, norm of even trips, norm of odd trips
  unsigned rbox;    // the partner's
  unsigned rsm;     // the partner's shared memory (shared::cluster address of sm[0])
  unsigned armer;   // thread 0
  bool need_phi;    // this warp reads a slot the partner fills
  /// Thread 0 arms the phase (its warp does not wait unless it reads the partner's values itself: a
  /// warp that waits runs its phase after the release, and two such warps on one scheduler -- the
  /// armer's and the halo warp of the same role -- were the long pole of the trip).
  __device__ __forceinline__ void recv_phi(int phase) const {
    mbar_expect_pred(armer, box, kPhiBytes);
    if (need_phi) mbar_wait_at(box, (unsigned)phase);
  }
  __device__ __forceinline__ void recv_norm(int trip, int bytes) const {
    const unsigned at = box + 8u + 8u * (unsigned)(trip & 1);
    mbar_expect_pred(armer, at, bytes);
    mbar_wait_at(at, (unsigned)(trip >> 1));
  }
  __device__ __forceinline__ unsigned norm_box(int trip) const { return rbox + 8u * (1u + (unsigned)(trip & 1)); }
};
/// Opens the mailboxes (the shared memory is cleared and a block barrier passed), exchanges the
/// pattern verdicts and returns the cluster-wide one.
__device__ __forceinline__ bool open_port(Port& pt, double* sm, double* red, const Cut& c, const LaneX& t, bool bad) {
  const int tid = threadIdx.x;
  unsigned long long* box = reinterpret_cast<unsigned long long*>(red + Port::kBoxAt);
  pt.red = smem_u32(red);
  asm volatile("mov.u32 %0, %0;" : "+r"(pt.red));  // opaque: not to be rematerialised inside the loop
  pt.box = pt.red + 8u * (unsigned)Port::kBoxAt;
  int* flag = reinterpret_cast<int*>(red + Port::kBoxAt + 4);
  if (tid == 0) {
    mbar_init(box, 1);
    mbar_init(box + 1, 1);
    mbar_init(box + 2, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    *flag = bad ? 1 : 0;
  }
  cg::this_cluster().sync();
  pt.rbox = partner_u32(box, c.rank ^ 1);
  pt.rsm = partner_u32(sm, c.rank ^ 1);
  pt.armer = tid == 0 ? 1u : 0u;
  const bool reads = c.rank == 0 ? t.k == c.hi : (t.k == c.lo - 1 || t.k == c.lo);
  pt.need_phi = __any_sync(kFull, reads);
  const int theirs = *cg::this_cluster().map_shared_rank(flag, c.rank ^ 1);
  return bad || theirs != 0;
}

/// The operator columns of role R of one interval, and whether the block has the expected zeros.
template <int K, int R>
struct OpCols {
  double ax[RoleT<K, R>::nxc][kNX];
  double bm[RoleT<K, R>::nuc][kNX];
  double bp[RoleT<K, R>::nuc][kNX];
};

/// Loads the columns of role R of interval `iv` (zero when !have).  Returns true when an entry
/// outside the structural pattern is not an exact zero.
template <int K, int R>
__device__ __forceinline__ bool load_cols(const SubArrays& sp, size_t iv, bool have, OpCols<K, R>& op) {
  using RT = RoleT<K, R>;
  bool bad = false;
  const double* A = sp.A_minus + iv * kNX * kNX;
  const double* Bm = sp.B_minus + iv * kNX * kNU;
  const double* Bp = sp.B_plus + iv * kNX * kNU;
#pragma unroll
  for (int j = 0; j < RT::nxc; ++j) {
    const int c = RT::xc(j);
    const unsigned mask = xcol_mask(c);
#pragma unroll
    for (int i = 0; i < kNX; ++i) {
      const double v = have ? __ldg(A + i * kNX + c) : 0.0;
      if ((mask >> i) & 1u) op.ax[j][i] = v;
      else bad |= !(v == 0.0);
    }
  }
#pragma unroll
  for (int j = 0; j < RT::nuc; ++j) {
    const int c = RT::uc(j);
    const unsigned mask = ucol_mask(c);
#pragma unroll
    for (int i = 0; i < kNX; ++i) {
      const double vm = have ? __ldg(Bm + i * kNU + c) : 0.0;
      const double vp = have ? __ldg(Bp + i * kNU + c) : 0.0;
      if ((mask >> i) & 1u) {
        op.bm[j][i] = vm;
        op.bp[j][i] = vp;
      } else {
        bad |= !(vm == 0.0) || !(vp == 0.0);
      }
    }
  }
  return bad;
}

/// Transposed products of role R against the duals of its interval (read from shared memory row
/// by row: one dual is live at a time, the column sums are the only accumulators): column sums of
/// its x columns, of its B- columns and of its B+ columns.
template <int K, int R, int S, bool kLean = false>
__device__ __forceinline__ void transposed(const OpCols<K, R>& op, const double* phi_slot,
                                           double (&gx)[RoleT<K, R>::nxc], double (&gm)[RoleT<K, R>::nuc],
                                           double (&gp)[RoleT<K, R>::nuc]) {
  using RT = RoleT<K, R>;
  constexpr unsigned touch = role_touch<K, R>();
  // kLean: every column sum starts with a product instead of an addition to a cleared accumulator
  bool fx[RT::nxc], fu[RT::nuc];
#pragma unroll
  for (int j = 0; j < RT::nxc; ++j) {
    gx[j] = 0.0;
    fx[j] = kLean;
  }
#pragma unroll
  for (int j = 0; j < RT::nuc; ++j) {
    gm[j] = gp[j] = 0.0;
    fu[j] = kLean;
  }
#pragma unroll
  for (int i = 0; i < kNX; ++i) {
    if (!((touch >> i) & 1u)) continue;
    const double p = phi_slot[i * S];
#pragma unroll
    for (int j = 0; j < RT::nuc; ++j)
      if ((ucol_mask(RT::uc(j)) >> i) & 1u) {
        gm[j] = fu[j] ? op.bm[j][i] * p : fma(op.bm[j][i], p, gm[j]);
        gp[j] = fu[j] ? op.bp[j][i] * p : fma(op.bp[j][i], p, gp[j]);
        fu[j] = false;
      }
#pragma unroll
    for (int j = 0; j < RT::nxc; ++j)
      if ((xcol_mask(RT::xc(j)) >> i) & 1u) {
        gx[j] = fx[j] ? op.ax[j][i] * p : fma(op.ax[j][i], p, gx[j]);
        fx[j] = false;
      }
  }
}

/// Partial sum of row i of role R's columns against its own primal entries zx, zu and the next
/// node's control entries zun (for the B+ columns).  kTwoChains: two accumulators added at the end
/// (shorter dependent chain; the power kernel is faster with it) or one chain started by a product
/// (an instruction less per row; the PIPG kernel, whose four loop bodies fill the instruction
/// cache, is 10 % faster with it).
template <int K, int R, bool kTwoChains>
__device__ __forceinline__ double forward_row(const OpCols<K, R>& op, const double (&zx)[RoleT<K, R>::nxc],
                                              const double (&zu)[RoleT<K, R>::nuc],
                                              const double (&zun)[RoleT<K, R>::nuc], int i) {
  using RT = RoleT<K, R>;
  if constexpr (kTwoChains) {
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int j = 0; j < RT::nuc; ++j)
      if ((ucol_mask(RT::uc(j)) >> i) & 1u) {
        a0 = fma(op.bm[j][i], zu[j], a0);
        a1 = fma(op.bp[j][i], zun[j], a1);
      }
#pragma unroll
    for (int j = 0; j < RT::nxc; ++j)
      if ((xcol_mask(RT::xc(j)) >> i) & 1u) {
        if (j & 1) a1 = fma(op.ax[j][i], zx[j], a1);
        else a0 = fma(op.ax[j][i], zx[j], a0);
      }
    return a0 + a1;
  } else {
    double a = 0.0;
    bool first = true;
#pragma unroll
    for (int j = 0; j < RT::nuc; ++j)
      if ((ucol_mask(RT::uc(j)) >> i) & 1u) {
        a = first ? op.bm[j][i] * zu[j] : fma(op.bm[j][i], zu[j], a);
        first = false;
        a = fma(op.bp[j][i], zun[j], a);
      }
#pragma unroll
    for (int j = 0; j < RT::nxc; ++j)
      if ((xcol_mask(RT::xc(j)) >> i) & 1u) {
        a = first ? op.ax[j][i] * zx[j] : fma(op.ax[j][i], zx[j], a);
        first = false;
      }
    return a;
  }
}

/// Forward products of role R row by row: the partial sums of the rows other roles own are
/// published at once, the own ones kept.
template <int K, int R, int S, bool kTwoChains>
__device__ __forceinline__ void forward_publish(const OpCols<K, R>& op, const double (&zx)[RoleT<K, R>::nxc],
                                                const double (&zu)[RoleT<K, R>::nuc],
                                                const double (&zun)[RoleT<K, R>::nuc], double* part_slot,
                                                bool auth, double (&own)[RoleT<K, R>::nrow]) {
  constexpr unsigned touch = role_touch<K, R>();
#pragma unroll
  for (int i = 0; i < kNX; ++i) {
    if (owns_row<K, R>(i)) continue;
    if (!((touch >> i) & 1u)) continue;
    const double v = forward_row<K, R, kTwoChains>(op, zx, zu, zun, i);
    if (auth) part_slot[(R * kNX + i) * S] = v;
  }
#pragma unroll
  for (int r = 0; r < RoleT<K, R>::nrow; ++r)
    own[r] = forward_row<K, R, kTwoChains>(op, zx, zu, zun, RoleT<K, R>::row(r));
}

/// Sum of the partial sums of row RoleT<K, R>::row(kRow): the own one and those of the roles that
/// reach the row.
template <int K, int R, int S, int kRow>
__device__ __forceinline__ double gather_row_t(double own, const double* part_slot) {
  constexpr int i = RoleT<K, R>::row(kRow);
  double s0 = own, s1 = 0.0;  // two short chains instead of one
  int cnt = 0;
#pragma unroll
  for (int q = 0; q < K; ++q) {
    if (q == R) continue;
    if (!((role_touch_of<K>(q) >> i) & 1u)) continue;
    if (cnt & 1) s0 += part_slot[(q * kNX + i) * S];
    else s1 += part_slot[(q * kNX + i) * S];
    ++cnt;
  }
  return s0 + s1;
}

template <int K, int R, int S>
__device__ __forceinline__ void gather_rows(const double (&own)[RoleT<K, R>::nrow], const double* part_slot,
                                            double (&s)[RoleT<K, R>::nrow]) {
  constexpr int nrow = RoleT<K, R>::nrow;
  s[0] = gather_row_t<K, R, S, 0>(own[0], part_slot);
  if constexpr (nrow > 1) s[1] = gather_row_t<K, R, S, 1>(own[1], part_slot);
  if constexpr (nrow > 2) s[2] = gather_row_t<K, R, S, 2>(own[2], part_slot);
  if constexpr (nrow > 3) s[3] = gather_row_t<K, R, S, 3>(own[3], part_slot);
  static_assert(nrow <= 4, "rows per role");
}

// ---------------------------------------------------------------------------------------------
// power iteration (pipg.hpp:206-292)
// ---------------------------------------------------------------------------------------------
template <int K, int R, int kHalves>
__device__ __forceinline__ void power_role(const PowerArgs& a, double* sm, int b, unsigned char* handled) {
  using RT = RoleT<K, R>;
  using Cfg = CsCfg<K, kHalves>;
  constexpr int S = Cfg::S;
  constexpr CsLayout L = cs_layout<K, kHalves>(false);
  const int n = a.shape.n, m = n - 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, half = warp / K;
  const Lane t = make_lane<kHalves>(n, half, lane);
  for (int e = tid; e < L.total; e += Cfg::threads) sm[e] = 0.0;

  OpCols<K, R> op;
  const bool have = t.k < m;  // halo copies load their node's block too
  const bool bad = load_cols<K, R>(a.sp, (size_t)b * m + (have ? t.k : 0), have, op);
  if (__syncthreads_or(bad ? 1 : 0)) {  // not the rocket pattern: the dense kernel takes the instance
    if (tid == 0) handled[b] = 0;
    return;
  }
  if (tid == 0) handled[b] = 1;

  double* phi_s = sm + L.phi + t.slot;    // row i at + i * S; interval k-1 at -1
  double* th_s = sm + L.th + t.slot;
  double* part_s = sm + L.part + t.slot;  // [role][row] at + (role * 15 + row) * S
  double* xn_s = sm + L.xn + t.slot;      // [3] at + q * S; node k+1 at +1
  double* red = sm + L.red;               // [2][kCsWarps] shares of the squared norm, by trip parity

  // seed (pipg.hpp:213-230)
  double zx[RT::nxc], zu[RT::nuc], vcd[RT::nrow];
  double acc0 = 0.0;
#pragma unroll
  for (int j = 0; j < RT::nxc; ++j) {
    zx[j] = t.primal ? a.seed_x[((size_t)b * n + t.k) * kNX + RT::xc(j)] : 0.0;
    acc0 = fma(zx[j], zx[j], acc0);
  }
#pragma unroll
  for (int j = 0; j < RT::nuc; ++j) {
    zu[j] = t.primal ? a.seed_u[((size_t)b * n + t.k) * kNU + RT::uc(j)] : 0.0;
    acc0 = fma(zu[j], zu[j], acc0);
  }
#pragma unroll
  for (int r = 0; r < RT::nrow; ++r) {
    double vp = 0.0, vn = 0.0;
    if (t.ival) {
      vp = a.seed_vcp[((size_t)b * m + t.k) * kNX + RT::row(r)];
      vn = a.seed_vcn[((size_t)b * m + t.k) * kNX + RT::row(r)];
    }
    vcd[r] = vp - vn;
    acc0 = fma(vp, vp, acc0);
    acc0 = fma(vn, vn, acc0);
  }
  acc0 = warp_sum(t.auth ? acc0 : 0.0);
  if (lane == 0) red[warp] = acc0;
  block_barrier();
  auto norm_sq = [&](int parity) {
    const double2* p = reinterpret_cast<const double2*>(red + parity * kCsWarps);
    const double2 q0 = p[0], q1 = p[1], q2 = p[2], q3 = p[3];
    const double lo = ((q0.x + q0.y) + (q1.x + q1.y)) + ((q2.x + q2.y) + (q3.x + q3.y));
    if (Cfg::warps <= 8) return lo;
    const double2 q4 = p[4], q5 = p[5], q6 = p[6], q7 = p[7];
    return lo + (((q4.x + q4.y) + (q5.x + q5.y)) + ((q6.x + q6.y) + (q7.x + q7.y)));
  };
  double ss = norm_sq(0);  // squared norm of the current iterate
  if (ss == 0.0) {  // pipg.hpp:224-225
    if (tid == 0) {
      if (a.status) a.status[b] = kStSeedZero;
      a.sigma[b] = 0.0;
      if (a.trips) a.trips[(size_t)b * a.trips_stride + (a.trips_slot ? a.trips_slot[b] : 0)] = 0;
    }
    return;
  }
  // Inside the loop sigma is ss * rsqrt(ss) (1 ulp from sqrt: it only feeds the stopping test, whose
  // tolerance is four orders of magnitude wider) and the scale 1 / sigma of pipg.hpp:243 is the
  // same rsqrt: no square root and no division on the trip's critical path.  The value returned is
  // the correctly rounded sqrt of the last squared norm.
  // The stopping test runs in every trip, also the first (no `if (j > 1)` block that would keep the
  // norm -> rsqrt -> test chain out of the basic block of the gathers it can overlap with): the first
  // one reads the seed's norm again and compares it with a NaN, which no tolerance accepts.
  double inv;
  double sigma = __longlong_as_double(0x7ff8000000000000ll);

  // The forward products of trip j + 1 are issued right behind the adjoint map of trip j, in front
  // of the barrier, so that the warp reduction of trip j's norm shares overlaps them.
  constexpr int kJy = aligned_col<K, R>(kNX - 1);  // the role that owns x[y] also owns the relaxation dual
  double own[RT::nrow], xnx[RT::nrow], dy = 0.0;
  auto forward_map = [&]() {  // pipg.hpp:234-245: partial row sums of the own columns
    double zun[RT::nuc];
#pragma unroll
    for (int q = 0; q < RT::nuc; ++q) zun[q] = __shfl_down_sync(kFull, zu[q], 1);
#pragma unroll
    for (int r = 0; r < RT::nrow; ++r) {  // x_{k+1}[row] of the aligned rows
      const int jc = aligned_col<K, R>(RT::row(r));
      xnx[r] = jc >= 0 ? __shfl_down_sync(kFull, zx[jc >= 0 ? jc : 0], 1) : 0.0;
    }
    if (kJy >= 0) dy = __shfl_down_sync(kFull, zx[kJy >= 0 ? kJy : 0], 1) - zx[kJy >= 0 ? kJy : 0];  // e_y^T (x_{k+1} - x_k)
#pragma unroll
    for (int q = 0; q < RT::nxc; ++q) {
      const int slot = xn_slot<K>(RT::xc(q));
      if (slot >= 0 && t.auth) xn_s[slot * S] = zx[q];
    }
    forward_publish<K, R, S, true>(op, zx, zu, zun, part_s, t.auth, own);
  };
  forward_map();

  int trips = 0;
  bool done = false;
  for (int j = 1; j <= a.j_max; ++j) {
    block_barrier();
    // ---- rows: sum of the partials, scale by 1 / sigma
    double s[RT::nrow];
    gather_rows<K, R, S>(own, part_s, s);
#pragma unroll
    for (int r = 0; r < RT::nrow; ++r) {
      const int i = RT::row(r);
      const double xn = aligned_col<K, R>(i) >= 0 ? xnx[r] : xn_s[xn_slot<K>(i) * S + 1];
      s[r] = (s[r] - xn) + vcd[r];
    }
    {  // stopping test of trip j-1 (pipg.hpp:277-289); j = 1: the seed against NaN, never met
      ss = norm_sq((j - 1) & 1);
      inv = rsqrt_pos(ss);
      const double sigma_star = ss * inv;
      const bool hit = fabs(sigma_star - sigma) <= a.eps_abs + a.eps_rel * max_nn(sigma_star, sigma);
      sigma = sigma_star;
      if (hit || ss == 0.0) {  // met, or the iterate is in the null space (pipg.hpp:280-284)
        done = true;
        break;
      }
    }
    trips = j;
    // rows of nodes without an interval come out as exact zeros (zero operator, zero neighbours);
    // only real intervals are stored, the rest of the array stays cleared
    double acc_d = 0.0;
#pragma unroll
    for (int r = 0; r < RT::nrow; ++r) {
      const double p = s[r] * inv;
      if (t.ival) phi_s[RT::row(r) * S] = p;
      vcd[r] = 2.0 * p;  // vc+ = phi, vc- = -phi (pipg.hpp:268-279)
      acc_d = fma(vcd[r], p, acc_d);
    }
    if (kJy >= 0) {
      if (t.ival) th_s[0] = dy * inv;
    }
    block_barrier();
    // ---- adjoint map (pipg.hpp:247-275)
    {
      double gx[RT::nxc], gm[RT::nuc], gp[RT::nuc];
      transposed<K, R, S>(op, phi_s, gx, gm, gp);
#pragma unroll
      for (int q = 0; q < RT::nxc; ++q) {
        const int c = RT::xc(q);
        double v = gx[q] - phi_s[c * S - 1];
        if (c == kNX - 1) v += th_s[-1] - th_s[0];
        zx[q] = v;
      }
#pragma unroll
      for (int q = 0; q < RT::nuc; ++q) {
        const double gpp = __shfl_up_sync(kFull, gp[q], 1);
        zu[q] = gm[q] + (lane == 0 ? 0.0 : gpp);
      }
    }
    double az0 = acc_d, az1 = 0.0;
#pragma unroll
    for (int q = 0; q < RT::nxc; ++q) {
      if (q & 1) az1 = fma(zx[q], zx[q], az1);
      else az0 = fma(zx[q], zx[q], az0);
    }
#pragma unroll
    for (int q = 0; q < RT::nuc; ++q) az1 = fma(zu[q], zu[q], az1);
    const double share = warp_sum(t.auth ? az0 + az1 : 0.0);
    forward_map();  // of trip j + 1
    if (lane == 0) red[(j & 1) * kCsWarps + warp] = share;
  }
  if (!done) {  // j_max trips without meeting the tolerance
    block_barrier();
    ss = norm_sq(a.j_max & 1);
  }
  if (tid == 0) {
    a.sigma[b] = (1.0 + a.eps_buff) * sqrt(ss);
    if (a.trips) a.trips[(size_t)b * a.trips_stride + (a.trips_slot ? a.trips_slot[b] : 0)] = trips;
  }
}

template <int K, int kHalves>
__global__ void __launch_bounds__(CsCfg<K, kHalves>::threads, 1) power_cs_kernel(PowerArgs a, unsigned char* handled) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  if (a.active && !a.active[b]) return;
  switch ((threadIdx.x >> 5) % K) {
    case 0: power_role<4, 0, kHalves>(a, sm, b, handled); break;
    case 1: power_role<4, 1, kHalves>(a, sm, b, handled); break;
    case 2: power_role<4, 2, kHalves>(a, sm, b, handled); break;
    default: power_role<4, 3, kHalves>(a, sm, b, handled); break;
  }
}

// ---- the same over a cluster of two CTAs (struct Cut, struct Port) ----
template <int K, int R, int kHalves, bool kCluster>
__device__ __forceinline__ void power_role_x(const PowerArgs& a, double* sm, int b, unsigned char* handled) {
  using RT = RoleT<K, R>;
  using Cfg = CsCfg<K, kHalves>;
  constexpr int S = Cfg::S;
  constexpr CsLayout L = cs_layout<K, kHalves>(false);
  const int n = a.shape.n, m = n - 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, half = warp / K;
  const Cut cut = make_cut<kCluster>(n);
  const LaneX t = make_lane_cut<kHalves>(cut, n, half, lane);
  for (int e = tid; e < L.total; e += Cfg::threads) sm[e] = 0.0;

  OpCols<K, R> op;
  bool bad = load_cols<K, R>(a.sp, (size_t)b * m + (t.have ? t.k : 0), t.have, op);
  bad = __syncthreads_or(bad ? 1 : 0) != 0;
  double* red = sm + L.red;               // [2][kCsWarps] shares of the squared norm, by trip parity
  Port port{};
  if constexpr (kCluster) bad = open_port(port, sm, red, cut, t, bad);
  if (bad) {  // not the rocket pattern: the dense kernel takes the instance
    if (tid == 0 && cut.rank == 0) handled[b] = 0;
    if constexpr (kCluster) cg::this_cluster().sync();  // the partner reads this CTA's verdict
    return;
  }
  if (tid == 0 && cut.rank == 0) handled[b] = 1;

  double* phi_s = sm + L.phi + t.slot;    // row i at + i * S; interval k-1 at -1
  double* th_s = sm + L.th + t.slot;
  double* part_s = sm + L.part + t.slot;  // [role][row] at + (role * 15 + row) * S
  double* xn_s = sm + L.xn + t.slot;      // [3] at + q * S; node k+1 at +1
  // cluster: the owners of the boundary interval store its duals in the partner's slots as well
  const bool pusher = kCluster && t.auth && t.k == (cut.rank == 0 ? cut.hi - 1 : cut.lo);
  const int pslot = cut.rank == 0 ? 1 : cut.lo + 1;  // slot of that interval over there
  const unsigned rphi = port.rsm + 8u * (unsigned)(L.phi + pslot), rth = port.rsm + 8u * (unsigned)(L.th + pslot);
  const unsigned rred = port.rsm + 8u * (unsigned)(L.red + cut.rank * (kCsWarps / 2) + warp);
  double* red_mine = red + cut.rank * (kCsWarps / 2) + warp;
  constexpr int kShareBytes = 8 * Cfg::warps;

  // seed (pipg.hpp:213-230)
  double zx[RT::nxc], zu[RT::nuc], vcd[RT::nrow];
  double acc0 = 0.0;
#pragma unroll
  for (int j = 0; j < RT::nxc; ++j) {
    zx[j] = t.primal ? a.seed_x[((size_t)b * n + t.k) * kNX + RT::xc(j)] : 0.0;
    acc0 = fma(zx[j], zx[j], acc0);
  }
#pragma unroll
  for (int j = 0; j < RT::nuc; ++j) {
    zu[j] = t.primal ? a.seed_u[((size_t)b * n + t.k) * kNU + RT::uc(j)] : 0.0;
    acc0 = fma(zu[j], zu[j], acc0);
  }
#pragma unroll
  for (int r = 0; r < RT::nrow; ++r) {
    double vp = 0.0, vn = 0.0;
    if (t.ival) {
      vp = a.seed_vcp[((size_t)b * m + t.k) * kNX + RT::row(r)];
      vn = a.seed_vcn[((size_t)b * m + t.k) * kNX + RT::row(r)];
    }
    vcd[r] = vp - vn;
    acc0 = fma(vp, vp, acc0);
    acc0 = fma(vn, vn, acc0);
  }
  acc0 = warp_sum(t.auth ? acc0 : 0.0);
  if (lane == 0) {
    if constexpr (kCluster) push_f64(rred, acc0, port.norm_box(0));
    red_mine[0] = acc0;
  }
  block_barrier();
  if constexpr (kCluster) port.recv_norm(0, kShareBytes);
  auto norm_sq = [&](int parity) {
    if constexpr (kCluster) {
      // (the address is a register: derived from the generic pointer it costs a special-register
      // read of the CTA's cluster rank on the trip's critical path)
      const unsigned at = port.red + 8u * (unsigned)(parity * kCsWarps);
      double2 q[8];
#pragma unroll
      for (int e = 0; e < 8; ++e)
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(q[e].x), "=d"(q[e].y) : "r"(at + 16u * e));
      const double lo = ((q[0].x + q[0].y) + (q[1].x + q[1].y)) + ((q[2].x + q[2].y) + (q[3].x + q[3].y));
      return lo + (((q[4].x + q[4].y) + (q[5].x + q[5].y)) + ((q[6].x + q[6].y) + (q[7].x + q[7].y)));
    } else {
      const double2* p = reinterpret_cast<const double2*>(red + parity * kCsWarps);
      const double2 q0 = p[0], q1 = p[1], q2 = p[2], q3 = p[3];
      const double lo = ((q0.x + q0.y) + (q1.x + q1.y)) + ((q2.x + q2.y) + (q3.x + q3.y));
      if (Cfg::warps <= 8) return lo;
      const double2 q4 = p[4], q5 = p[5], q6 = p[6], q7 = p[7];
      return lo + (((q4.x + q4.y) + (q5.x + q5.y)) + ((q6.x + q6.y) + (q7.x + q7.y)));
    }
  };
  double ss = norm_sq(0);  // squared norm of the current iterate
  if (ss == 0.0) {  // pipg.hpp:224-225
    if (tid == 0 && cut.rank == 0) {
      if (a.status) a.status[b] = kStSeedZero;
      a.sigma[b] = 0.0;
      if (a.trips) a.trips[(size_t)b * a.trips_stride + (a.trips_slot ? a.trips_slot[b] : 0)] = 0;
    }
    if constexpr (kCluster) cg::this_cluster().sync();
    return;
  }
  // Inside the loop sigma is ss * rsqrt(ss) (1 ulp from sqrt: it only feeds the stopping test, whose
  // tolerance is four orders of magnitude wider) and the scale 1 / sigma of pipg.hpp:243 is the
  // same rsqrt: no square root and no division on the trip's critical path.  The value returned is
  // the correctly rounded sqrt of the last squared norm.
  // The stopping test runs in every trip, also the first (no `if (j > 1)` block that would keep the
  // norm -> rsqrt -> test chain out of the basic block of the gathers it can overlap with): the first
  // one reads the seed's norm again and compares it with a NaN, which no tolerance accepts.
  double inv;
  double sigma = __longlong_as_double(0x7ff8000000000000ll);

  // The forward products of trip j + 1 are issued right behind the adjoint map of trip j, in front
  // of the barrier, so that the warp reduction of trip j's norm shares overlaps them.
  constexpr int kJy = aligned_col<K, R>(kNX - 1);  // the role that owns x[y] also owns the relaxation dual
  double own[RT::nrow], xnx[RT::nrow], dy = 0.0;
  auto forward_map = [&]() {  // pipg.hpp:234-245: partial row sums of the own columns
    double zun[RT::nuc];
#pragma unroll
    for (int q = 0; q < RT::nuc; ++q) zun[q] = __shfl_down_sync(kFull, zu[q], 1);
#pragma unroll
    for (int r = 0; r < RT::nrow; ++r) {  // x_{k+1}[row] of the aligned rows
      const int jc = aligned_col<K, R>(RT::row(r));
      xnx[r] = jc >= 0 ? __shfl_down_sync(kFull, zx[jc >= 0 ? jc : 0], 1) : 0.0;
    }
    if (kJy >= 0) dy = __shfl_down_sync(kFull, zx[kJy >= 0 ? kJy : 0], 1) - zx[kJy >= 0 ? kJy : 0];  // e_y^T (x_{k+1} - x_k)
#pragma unroll
    for (int q = 0; q < RT::nxc; ++q) {
      const int slot = xn_slot<K>(RT::xc(q));
      if (slot >= 0 && t.pubx) xn_s[slot * S] = zx[q];
    }
    forward_publish<K, R, S, !kCluster>(op, zx, zu, zun, part_s, t.auth, own);  // (cluster: the leaner code)
  };
  forward_map();

  int trips = 0;
  bool done = false;
  for (int j = 1; j <= a.j_max; ++j) {
    block_barrier();
    // The partner's norm shares of trip j - 1 have normally arrived by now (they were sent in front
    // of its forward products): the mailbox is armed here, tested once behind the gathers -- which
    // do not need the shares and overlap the test -- and polled only if that test fails.
    unsigned norm_at = 0, norm_par = 0;
    if constexpr (kCluster) {
      norm_at = port.box + 8u + 8u * (unsigned)((j - 1) & 1);
      norm_par = (unsigned)((j - 1) >> 1);
      mbar_expect_pred(j > 1 ? port.armer : 0u, norm_at, kShareBytes);  // (the seed's were received above)
    }
    // ---- rows: sum of the partials, scale by 1 / sigma
    double s[RT::nrow];
    gather_rows<K, R, S>(own, part_s, s);
#pragma unroll
    for (int r = 0; r < RT::nrow; ++r) {
      const int i = RT::row(r);
      const double xn = aligned_col<K, R>(i) >= 0 ? xnx[r] : xn_s[xn_slot<K>(i) * S + 1];
      s[r] = (s[r] - xn) + vcd[r];
    }
    if constexpr (kCluster) {
      if (!mbar_test_at(norm_at, norm_par)) mbar_wait_at(norm_at, norm_par);
    }
    {  // stopping test of trip j-1 (pipg.hpp:277-289); j = 1: the seed against NaN, never met
      ss = norm_sq((j - 1) & 1);
      inv = rsqrt_pos(ss);
      const double sigma_star = ss * inv;
      const bool hit = fabs(sigma_star - sigma) <= a.eps_abs + a.eps_rel * max_nn(sigma_star, sigma);
      sigma = sigma_star;
      if (hit || ss == 0.0) {  // met, or the iterate is in the null space (pipg.hpp:280-284)
        done = true;
        break;
      }
    }
    trips = j;
    // rows of nodes without an interval come out as exact zeros (zero operator, zero neighbours);
    // only real intervals are stored, the rest of the array stays cleared
    double acc_d = 0.0;
#pragma unroll
    for (int r = 0; r < RT::nrow; ++r) {
      s[r] *= inv;
      if (t.ival) phi_s[RT::row(r) * S] = s[r];
      vcd[r] = 2.0 * s[r];  // vc+ = phi, vc- = -phi (pipg.hpp:268-279)
      acc_d = fma(vcd[r], s[r], acc_d);
    }
    if (kJy >= 0) {
      if (t.ival) th_s[0] = dy * inv;
    }
    if constexpr (kCluster) {  // one divergent block for all the remote stores of the boundary lane
      if (pusher) {
#pragma unroll
        for (int r = 0; r < RT::nrow; ++r) push_f64(rphi + 8u * (unsigned)(RT::row(r) * S), s[r], port.rbox);
        if (kJy >= 0) push_f64(rth, dy * inv, port.rbox);
      }
    }
    block_barrier();
    if constexpr (kCluster) port.recv_phi(j - 1);
    // ---- adjoint map (pipg.hpp:247-275)
    {
      double gx[RT::nxc], gm[RT::nuc], gp[RT::nuc];
      transposed<K, R, S, kCluster>(op, phi_s, gx, gm, gp);
#pragma unroll
      for (int q = 0; q < RT::nxc; ++q) {
        const int c = RT::xc(q);
        double v = gx[q] - phi_s[c * S - 1];
        if (c == kNX - 1) v += th_s[-1] - th_s[0];
        zx[q] = v;
      }
#pragma unroll
      for (int q = 0; q < RT::nuc; ++q) {
        const double gpp = __shfl_up_sync(kFull, gp[q], 1);
        zu[q] = gm[q] + (lane == 0 ? 0.0 : gpp);
      }
    }
    double az0 = acc_d, az1 = 0.0;
#pragma unroll
    for (int q = 0; q < RT::nxc; ++q) {
      if (q & 1) az1 = fma(zx[q], zx[q], az1);
      else az0 = fma(zx[q], zx[q], az0);
    }
#pragma unroll
    for (int q = 0; q < RT::nuc; ++q) az1 = fma(zu[q], zu[q], az1);
    const double share = warp_sum(t.auth ? az0 + az1 : 0.0);
    if constexpr (kCluster) {  // in flight while the forward products run
      push_f64_pred(lane == 0, rred + 8u * (unsigned)((j & 1) * kCsWarps), share, port.norm_box(j));
    }
    forward_map();  // of trip j + 1
    if (lane == 0) red_mine[(j & 1) * kCsWarps] = share;
  }
  if (!done) {  // j_max trips without meeting the tolerance
    block_barrier();
    if constexpr (kCluster) port.recv_norm(a.j_max, kShareBytes);
    ss = norm_sq(a.j_max & 1);
  }
  if (tid == 0 && cut.rank == 0) {
    a.sigma[b] = (1.0 + a.eps_buff) * sqrt(ss);
    if (a.trips) a.trips[(size_t)b * a.trips_stride + (a.trips_slot ? a.trips_slot[b] : 0)] = trips;
  }
  if constexpr (kCluster) cg::this_cluster().sync();  // nobody leaves while the partner may still store here
}

template <int K, int kHalves, bool kCluster>
__global__ void __launch_bounds__(CsCfg<K, kHalves>::threads, 1) power_cs_cluster_kernel(PowerArgs a, unsigned char* handled) {
  extern __shared__ __align__(16) double sm[];
  const int b = kCluster ? blockIdx.x >> 1 : blockIdx.x;
  if (a.active && !a.active[b]) return;  // both CTAs of a cluster leave together
  switch ((threadIdx.x >> 5) % K) {
    case 0: power_role_x<4, 0, kHalves, kCluster>(a, sm, b, handled); break;
    case 1: power_role_x<4, 1, kHalves, kCluster>(a, sm, b, handled); break;
    case 2: power_role_x<4, 2, kHalves, kCluster>(a, sm, b, handled); break;
    default: power_role_x<4, 3, kHalves, kCluster>(a, sm, b, handled); break;
  }
}

// ---------------------------------------------------------------------------------------------
// customized PIPG (pipg.hpp:350-497)
// ---------------------------------------------------------------------------------------------
/// stopping_custom(cur, prev) and the divergence test of pipg.hpp:475-487 over two snapshots: 0 =
/// go on, 1 = converged, 2 = a non-finite primal or dual entry.  One copy for the four roles (the
/// loop bodies are role-specific and have to share the instruction cache with as little as possible).
template <int kHalves>
__device__ __noinline__ int pipg_check(const double* cur, const double* prev, int n, double* red, double eps_abs,
                                       double eps_rel) {
  constexpr SnapCs SN = snap_cs<4, kHalves>();
  constexpr int T = CsCfg<4, kHalves>::threads;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = n - 1;
  double z_cur = 0.0, z_prev = 0.0, z_del = 0.0, r_cur = 0.0, r_prev = 0.0, r_del = 0.0, badv = 0.0;
  auto scan = [&](int off, int count, bool dual, bool finite_checked) {
#pragma unroll 1
    for (int e = tid; e < count; e += T) {
      const double c = cur[off + e], o = prev[off + e];
      if (dual) {
        r_cur = max_nn(r_cur, fabs(c));
        r_prev = max_nn(r_prev, fabs(o));
        r_del = max_nn(r_del, fabs(c - o));
      } else {
        z_cur = max_nn(z_cur, fabs(c));
        z_prev = max_nn(z_prev, fabs(o));
        z_del = max_nn(z_del, fabs(c - o));
      }
      if (finite_checked && !pt_finite(c)) badv = 1.0;
    }
  };
  scan(SN.x, n * kNX, false, true);
  scan(SN.u, n * kNU, false, true);
  scan(SN.vp, m * kNX, false, false);
  scan(SN.vn, m * kNX, false, false);
  scan(SN.ph, m * kNX, true, true);
  scan(SN.th, m, true, false);
  z_cur = warp_max_nn(z_cur); z_prev = warp_max_nn(z_prev); z_del = warp_max_nn(z_del);
  r_cur = warp_max_nn(r_cur); r_prev = warp_max_nn(r_prev); r_del = warp_max_nn(r_del);
  badv = warp_max_nn(badv);
  if (lane == 0) {
    double* rw = red + warp * 8;
    rw[0] = z_cur; rw[1] = z_prev; rw[2] = z_del; rw[3] = r_cur; rw[4] = r_prev; rw[5] = r_del;
    rw[6] = badv;
  }
  block_barrier();
  double v[7];
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    double mx = 0.0;
#pragma unroll
    for (int w = 0; w < CsCfg<4, kHalves>::warps; ++w) mx = max_nn(mx, red[w * 8 + q]);
    v[q] = mx;
  }
  block_barrier();  // red and the snapshots are rewritten later
  if (v[6] > 0.0) return 2;
  return (v[2] <= eps_abs + eps_rel * max_nn(v[0], v[1]) && v[5] <= eps_abs + eps_rel * max_nn(v[3], v[4])) ? 1 : 0;
}

template <int K, int R, int kHalves>
__device__ __forceinline__ void pipg_role(const PipgArgs& a, double* sm, int b, unsigned char* handled) {
  using RT = RoleT<K, R>;
  using Cfg = CsCfg<K, kHalves>;
  constexpr int S = Cfg::S;
  constexpr int T = Cfg::threads;
  constexpr CsLayout L = cs_layout<K, kHalves>(true);
  constexpr SnapCs SN = snap_cs<K, kHalves>();
  const int n = a.shape.n, m = n - 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, half = warp / K;
  const Lane t = make_lane<kHalves>(n, half, lane);
  for (int e = tid; e < L.total; e += T) sm[e] = 0.0;

  OpCols<K, R> op;
  const bool have = t.k < m;  // halo copies load their node's block too
  const bool bad = load_cols<K, R>(a.sp, (size_t)b * m + (have ? t.k : 0), have, op);
  if (__syncthreads_or(bad ? 1 : 0)) {  // not the rocket pattern: the dense kernel takes the instance
    if (tid == 0) handled[b] = 0;
    return;
  }
  if (tid == 0) handled[b] = 1;

  double* phi_s = sm + L.phi + t.slot;    // extrapolated dynamics dual, row i at + i * S; interval k-1 at -1
  double* th_s = sm + L.th + t.slot;      // extrapolated relaxation dual
  double* part_s = sm + L.part + t.slot;
  double* xn_s = sm + L.xn + t.slot;      // reflections of x[q0], x[w2], x[y]; node k+1 at +1
  const double* wv_s = sm + L.wv + t.slot;
  const double* eps_s = sm + L.eps + t.slot;
  double* bnd_s = sm + L.bnd + (R * 4) * S + t.slot;  // [u column][lo, hi] at + (2 * q + {0, 1}) * S
  double* red = sm + L.red;
  double* snap0 = sm + L.snap;
  double* init_val = sm + L.fix;
  double* final_val = init_val + 16;
  double* init_on = final_val + 16;
  double* final_on = init_on + 16;
  const double* cost_s = sm + L.ecost + t.slot;  // the terminal-cost term of this node's entries (pipg.hpp:404)

  const size_t gx = (size_t)b * n * kNX, gu = (size_t)b * n * kNU, gm_ = (size_t)b * m * kNX, gt = (size_t)b * m;
  const int NXn = n * kNX, NUn = n * kNU, NM = m * kNX;
  if (tid < kNX) sm[L.ecost + tid * S + n] = a.shape.w_cost * a.shape.e_cost[tid];  // slot of node n - 1
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
  for (int e = tid; e < NM; e += T) {  // [interval][row] -> [row][slot]
    const int k = e / kNX, i = e - k * kNX;
    sm[L.wv + i * S + k + 1] = a.sp.w[gm_ + e];
  }
  for (int e = tid; e < m; e += T) sm[L.eps + e + 1] = a.sp.eps_relax[gt + e];
#pragma unroll
  for (int q = 0; q < RT::nuc; ++q) {  // box of the own control entries (pipg.hpp:418-419); unbounded where there is no node
    if (t.halo) continue;  // the owner's warp fills the slot; the halo copy reads it behind the barrier
    bnd_s[(2 * q) * S] = t.auth ? a.sp.u_min[gu + t.k * kNU + RT::uc(q)] : -INFINITY;
    bnd_s[(2 * q + 1) * S] = t.auth ? a.sp.u_max[gu + t.k * kNU + RT::uc(q)] : INFINITY;
  }
  // warm start: ex = cur = workspace (pipg.hpp:362-374); it is snapshot 0
  for (int e = tid; e < NXn; e += T) snap0[SN.x + e] = a.ws.x[gx + e];
  for (int e = tid; e < NUn; e += T) snap0[SN.u + e] = a.ws.u[gu + e];
  for (int e = tid; e < NM; e += T) {
    snap0[SN.vp + e] = a.ws.vc_pos[gm_ + e];
    snap0[SN.vn + e] = a.ws.vc_neg[gm_ + e];
    snap0[SN.ph + e] = a.ws.dyn_dual[gm_ + e];
  }
  for (int e = tid; e < m; e += T) snap0[SN.th + e] = a.ws.relax_dual[gt + e];
  block_barrier();

  // boundary columns of this thread (pipg.hpp:408-413): bit q set when own x column q is assigned
  int fix_bits = 0;
  const double* fix_val = init_val;
  const bool last_node = t.primal && t.k == n - 1;
  if (t.primal && (t.k == 0 || t.k == n - 1)) {
    const double* on = last_node ? final_on : init_on;
    fix_val = last_node ? final_val : init_val;
#pragma unroll
    for (int q = 0; q < RT::nxc; ++q)
      if (on[RT::xc(q)] != 0.0) fix_bits |= 1 << q;
  }

  const bool warp_fix = __any_sync(kFull, fix_bits != 0);  // warp-uniform

  // owner-private extrapolated copies
  double xe[RT::nxc], ue[RT::nuc], vpe[RT::nrow], vne[RT::nrow], phe[RT::nrow], the = 0.0;
#pragma unroll
  for (int q = 0; q < RT::nxc; ++q) xe[q] = t.primal ? snap0[SN.x + t.k * kNX + RT::xc(q)] : 0.0;
#pragma unroll
  for (int q = 0; q < RT::nuc; ++q) ue[q] = t.primal ? snap0[SN.u + t.k * kNU + RT::uc(q)] : 0.0;
#pragma unroll
  for (int r = 0; r < RT::nrow; ++r) {
    const int e = t.k * kNX + RT::row(r);
    vpe[r] = t.ival ? snap0[SN.vp + e] : 0.0;
    vne[r] = t.ival ? snap0[SN.vn + e] : 0.0;
    phe[r] = t.ival ? snap0[SN.ph + e] : 0.0;
    if (t.auth) phi_s[RT::row(r) * S] = phe[r];
  }
  if (R == 0) {
    the = t.ival ? snap0[SN.th + t.k] : 0.0;
    if (t.auth) th_s[0] = the;
  }

  const double sigma = a.sigma[b];
  const double alpha = 2.0 / (a.shape.w_prox + sqrt(a.shape.w_prox * a.shape.w_prox + 4.0 * a.omega * sigma));
  const double beta = a.omega * alpha;
  // extrapolation (pipg.hpp:461-472) (1 - rho) * ex + rho * cur, evaluated as ex + rho * (cur - ex)
  auto extrapolate = [&](double ex, double cur) { return fma(a.rho, cur - ex, ex); };
  block_barrier();

  // One iteration.  kStore additionally writes the new *_cur values of every owner into `snap`.
  auto iteration = [&](auto store_tag, double* snap) {
    constexpr bool kStore = decltype(store_tag)::value;
    // ---- primal projected-gradient step (pipg.hpp:388-420) by the owner of each entry
    double rx[RT::nxc], ru[RT::nuc];
    {
      double gx_[RT::nxc], gm[RT::nuc], gp[RT::nuc];
      transposed<K, R, S, true>(op, phi_s, gx_, gm, gp);
#pragma unroll
      for (int q = 0; q < RT::nxc; ++q) {
        const int c = RT::xc(q);
        const double x0 = xe[q];
        double base = x0 * a.shape.w_prox;
        base += cost_s[c * S];  // zero but at the last node: no branch, no predicated address arithmetic
        base += -phi_s[c * S - 1];
        if (c == kNX - 1) base += th_s[-1] - th_s[0];
        const double grad = base + gx_[q];
        double xn = x0 + -alpha * grad;
        if (warp_fix) xn = (fix_bits & (1 << q)) ? fix_val[c] : xn;  // (measured: faster than unconditional)
        rx[q] = fma(2.0, xn, -x0);
        if (kStore && t.auth) snap[SN.x + t.k * kNX + c] = xn;
        xe[q] = extrapolate(x0, xn);
      }
#pragma unroll
      for (int q = 0; q < RT::nuc; ++q) {
        double gpp = __shfl_up_sync(kFull, gp[q], 1);
        gpp = lane == 0 ? 0.0 : gpp;
        const double u0 = ue[q];
        const double grad = u0 * a.shape.w_prox + (gm[q] + gpp);
        double un = u0 + -alpha * grad;
        const double lo = bnd_s[(2 * q) * S], hi = bnd_s[(2 * q + 1) * S];
        // std::max(lo, std::min(hi, v)), pipg.hpp:418-419
        un = clamp_box(lo, hi, un);
        ru[q] = fma(2.0, un, -u0);
        if (kStore && t.auth) snap[SN.u + t.k * kNU + RT::uc(q)] = un;
        ue[q] = extrapolate(u0, un);
      }
    }
    // ---- forward products of the reflections: partial row sums of the own columns
    double run[RT::nuc];
#pragma unroll
    for (int q = 0; q < RT::nuc; ++q) run[q] = __shfl_down_sync(kFull, ru[q], 1);
    double xnx[RT::nrow];
#pragma unroll
    for (int r = 0; r < RT::nrow; ++r) {
      const int jc = aligned_col<K, R>(RT::row(r));
      xnx[r] = jc >= 0 ? __shfl_down_sync(kFull, rx[jc >= 0 ? jc : 0], 1) : 0.0;
    }
    double drift = 0.0;
    if (R == 0) drift = __shfl_down_sync(kFull, rx[4], 1) - rx[4];  // K = 4: role 0 owns x[y]
#pragma unroll
    for (int q = 0; q < RT::nxc; ++q) {
      const int slot = xn_slot<K>(RT::xc(q));
      if (slot >= 0 && t.auth) xn_s[slot * S] = rx[q];
    }
    double own[RT::nrow];
    forward_publish<K, R, S, false>(op, rx, ru, run, part_s, t.auth, own);
    block_barrier();
    // ---- slacks (pipg.hpp:423-430), PI feedback of the constraint violation (:433-458),
    //      extrapolation of the dual groups (:468-472)
    double s[RT::nrow];
    gather_rows<K, R, S>(own, part_s, s);
#pragma unroll
    for (int r = 0; r < RT::nrow; ++r) {
      const int i = RT::row(r);
      const double xn = aligned_col<K, R>(i) >= 0 ? xnx[r] : xn_s[xn_slot<K>(i) * S + 1];
      double resid = s[r] - xn;
      const double p0 = phe[r], vp0 = vpe[r], vn0 = vne[r];
      const double vp = clip0(vp0 - alpha * (a.shape.w_ep + p0));
      const double vn = clip0(vn0 - alpha * (a.shape.w_ep - p0));
      resid += (2.0 * vp - vp0) - (2.0 * vn - vn0) + wv_s[i * S];
      const double pn = p0 + beta * resid;
      if (kStore && t.ival) {
        const int e = t.k * kNX + i;
        snap[SN.vp + e] = vp;
        snap[SN.vn + e] = vn;
        snap[SN.ph + e] = pn;
      }
      // rows of nodes without an interval (zero operator, zero neighbours, zero right-hand side,
      // w_ep >= 0) stay exact zeros; only real intervals are stored
      phe[r] = extrapolate(p0, pn);
      vpe[r] = extrapolate(vp0, vp);
      vne[r] = extrapolate(vn0, vn);
      if (t.ival) phi_s[i * S] = phe[r];
    }
    if (R == 0) {
      const double tn = clip0(the + beta * (drift - eps_s[0]));
      if (kStore && t.ival) snap[SN.th + t.k] = tn;
      the = extrapolate(the, tn);
      if (t.ival) th_s[0] = the;
    }
    block_barrier();
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
      iteration(std::true_type{}, snap0 + cur_set * SN.total);
    } else {
      iteration(std::false_type{}, nullptr);
    }
    iters = j;
    if (check) {  // stopping_custom(cur, prev) and the divergence test, pipg.hpp:475-487
      const int verdict = pipg_check<kHalves>(snap0 + cur_set * SN.total, snap0 + (cur_set ^ 1) * SN.total, n, red,
                                              a.eps_abs, a.eps_rel);
      if (verdict == 2) {
        diverged = true;
        break;
      }
      if (verdict == 1) {
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
  // solution = the *_cur groups, pipg.hpp:490-495 (every iteration ends with a barrier)
  const double* cur = snap0 + cur_set * SN.total;
  for (int e = tid; e < NXn; e += T) a.ws.x[gx + e] = cur[SN.x + e];
  for (int e = tid; e < NUn; e += T) a.ws.u[gu + e] = cur[SN.u + e];
  for (int e = tid; e < NM; e += T) {
    a.ws.vc_pos[gm_ + e] = cur[SN.vp + e];
    a.ws.vc_neg[gm_ + e] = cur[SN.vn + e];
    a.ws.dyn_dual[gm_ + e] = cur[SN.ph + e];
  }
  for (int e = tid; e < m; e += T) a.ws.relax_dual[gt + e] = cur[SN.th + e];
  if (tid == 0) {
    if (a.iterations) a.iterations[b] = iters;
    if (a.converged) a.converged[b] = converged ? 1 : 0;
  }
}

template <int kHalves>
__global__ void __launch_bounds__(CsCfg<4, kHalves>::threads, 1) pipg_cs_kernel(PipgArgs a, unsigned char* handled) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  if (a.active && !a.active[b]) return;
  switch ((threadIdx.x >> 5) & 3) {
    case 0: pipg_role<4, 0, kHalves>(a, sm, b, handled); break;
    case 1: pipg_role<4, 1, kHalves>(a, sm, b, handled); break;
    case 2: pipg_role<4, 2, kHalves>(a, sm, b, handled); break;
    default: pipg_role<4, 3, kHalves>(a, sm, b, handled); break;
  }
}

// ---- the same over a cluster of two CTAs (struct Cut, struct Port) ----
template <int kHalves, bool kCluster>
__device__ __noinline__ int pipg_check_x(const double* cur, const double* prev, int l0, int nn, int mm, double* red,
                                       double eps_abs, double eps_rel) {
  // l0: first owned local node, nn / mm: owned nodes / intervals of this CTA
  constexpr SnapCs SN = snap_cs<4, kHalves, 1>();
  constexpr int T = CsCfg<4, kHalves>::threads;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double z_cur = 0.0, z_prev = 0.0, z_del = 0.0, r_cur = 0.0, r_prev = 0.0, r_del = 0.0, badv = 0.0;
  auto scan = [&](int off, int count, bool dual, bool finite_checked) {
#pragma unroll 1
    for (int e = tid; e < count; e += T) {
      const double c = cur[off + e], o = prev[off + e];
      if (dual) {
        r_cur = max_nn(r_cur, fabs(c));
        r_prev = max_nn(r_prev, fabs(o));
        r_del = max_nn(r_del, fabs(c - o));
      } else {
        z_cur = max_nn(z_cur, fabs(c));
        z_prev = max_nn(z_prev, fabs(o));
        z_del = max_nn(z_del, fabs(c - o));
      }
      if (finite_checked && !pt_finite(c)) badv = 1.0;
    }
  };
  scan(SN.x + l0 * kNX, nn * kNX, false, true);
  scan(SN.u + l0 * kNU, nn * kNU, false, true);
  scan(SN.vp + l0 * kNX, mm * kNX, false, false);
  scan(SN.vn + l0 * kNX, mm * kNX, false, false);
  scan(SN.ph + l0 * kNX, mm * kNX, true, true);
  scan(SN.th + l0, mm, true, false);
  z_cur = warp_max_nn(z_cur); z_prev = warp_max_nn(z_prev); z_del = warp_max_nn(z_del);
  r_cur = warp_max_nn(r_cur); r_prev = warp_max_nn(r_prev); r_del = warp_max_nn(r_del);
  badv = warp_max_nn(badv);
  if (lane == 0) {
    double* rw = red + warp * 8;
    rw[0] = z_cur; rw[1] = z_prev; rw[2] = z_del; rw[3] = r_cur; rw[4] = r_prev; rw[5] = r_del;
    rw[6] = badv;
  }
  block_barrier();
  double v[7];
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    double mx = 0.0;
#pragma unroll
    for (int w = 0; w < CsCfg<4, kHalves>::warps; ++w) mx = max_nn(mx, red[w * 8 + q]);
    v[q] = mx;
  }
  if constexpr (kCluster) {  // the partner's maxima (a stopping test is rare: two cluster barriers)
    double* mine = red + Port::kBoxAt + 8;  // [7], behind the mailboxes and the pattern flag
    if (tid == 0) {
#pragma unroll
      for (int q = 0; q < 7; ++q) mine[q] = v[q];
    }
    cg::this_cluster().sync();
    const double* theirs = cg::this_cluster().map_shared_rank(mine, (int)cg::this_cluster().block_rank() ^ 1);
#pragma unroll
    for (int q = 0; q < 7; ++q) v[q] = max_nn(v[q], theirs[q]);
    cg::this_cluster().sync();  // red and the snapshots are rewritten later
  } else {
    block_barrier();  // red and the snapshots are rewritten later
  }
  if (v[6] > 0.0) return 2;
  return (v[2] <= eps_abs + eps_rel * max_nn(v[0], v[1]) && v[5] <= eps_abs + eps_rel * max_nn(v[3], v[4])) ? 1 : 0;
}

template <int K, int R, int kHalves, bool kCluster>
__device__ __forceinline__ void pipg_role_x(const PipgArgs& a, double* sm, int b, unsigned char* handled) {
  using RT = RoleT<K, R>;
  using Cfg = CsCfg<K, kHalves>;
  constexpr int S = Cfg::S;
  constexpr int T = Cfg::threads;
  constexpr CsLayout L = cs_layout<K, kHalves>(true, true);
  constexpr SnapCs SN = snap_cs<K, kHalves, 1>();
  const int n = a.shape.n, m = n - 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, half = warp / K;
  const Cut cut = make_cut<kCluster>(n);
  const LaneX t = make_lane_cut<kHalves>(cut, n, half, lane);
  const int tl = t.slot - 1;  // local node: the snapshots are indexed by it
  for (int e = tid; e < L.total; e += T) sm[e] = 0.0;

  OpCols<K, R> op;
  bool bad = load_cols<K, R>(a.sp, (size_t)b * m + (t.have ? t.k : 0), t.have, op);
  bad = __syncthreads_or(bad ? 1 : 0) != 0;
  Port port{};
  if constexpr (kCluster) bad = open_port(port, sm, sm + L.red, cut, t, bad);
  if (bad) {  // not the rocket pattern: the dense kernel takes the instance
    if (tid == 0 && cut.rank == 0) handled[b] = 0;
    if constexpr (kCluster) cg::this_cluster().sync();  // the partner reads this CTA's verdict
    return;
  }
  if (tid == 0 && cut.rank == 0) handled[b] = 1;

  double* phi_s = sm + L.phi + t.slot;    // extrapolated dynamics dual, row i at + i * S; interval k-1 at -1
  double* th_s = sm + L.th + t.slot;      // extrapolated relaxation dual
  double* part_s = sm + L.part + t.slot;
  double* xn_s = sm + L.xn + t.slot;      // reflections of x[q0], x[w2], x[y]; node k+1 at +1
  const double* wv_s = sm + L.wv + t.slot;
  const double* eps_s = sm + L.eps + t.slot;
  double* bnd_s = sm + L.bnd + (R * 4) * S + t.slot;  // [u column][lo, hi] at + (2 * q + {0, 1}) * S
  double* red = sm + L.red;
  double* snap0 = sm + L.snap;
  double* init_val = sm + L.fix;
  double* final_val = init_val + 16;
  double* init_on = final_val + 16;
  double* final_on = init_on + 16;
  const double* cost_s = sm + L.ecost + t.slot;  // the terminal-cost term of this node's entries (pipg.hpp:404)

  const size_t gx = (size_t)b * n * kNX, gu = (size_t)b * n * kNU, gm_ = (size_t)b * m * kNX, gt = (size_t)b * m;
  const int NXn = n * kNX, NUn = n * kNU, NM = m * kNX;
  if (tid < kNX && n - 1 >= cut.lo && n - 1 < cut.hip)  // slot of node n - 1, in the CTA that holds it
    sm[L.ecost + tid * S + n - cut.base] = a.shape.w_cost * a.shape.e_cost[tid];
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
  // the nodes / intervals this CTA holds a slot for: local 0 .. kLoc - 1
  constexpr int kLoc = Cfg::cap + 1;
  for (int e = tid; e < NM; e += T) {  // [interval][row] -> [row][slot]
    const int k = e / kNX, i = e - k * kNX, l = k - cut.base;
    if (l >= 0 && l < kLoc) sm[L.wv + i * S + l + 1] = a.sp.w[gm_ + e];
  }
  for (int e = tid; e < m; e += T) {
    const int l = e - cut.base;
    if (l >= 0 && l < kLoc) sm[L.eps + l + 1] = a.sp.eps_relax[gt + e];
  }
#pragma unroll
  for (int q = 0; q < RT::nuc; ++q) {  // box of the own control entries (pipg.hpp:418-419); unbounded where there is no node
    if (t.halo) continue;  // the owner's warp fills the slot; the halo copy reads it behind the barrier
    bnd_s[(2 * q) * S] = t.pubx ? a.sp.u_min[gu + t.k * kNU + RT::uc(q)] : -INFINITY;
    bnd_s[(2 * q + 1) * S] = t.pubx ? a.sp.u_max[gu + t.k * kNU + RT::uc(q)] : INFINITY;
  }
  // warm start: ex = cur = workspace (pipg.hpp:362-374); it is snapshot 0
  const int sx = cut.base * kNX, su = cut.base * kNU;  // global index - this = local index
  for (int e = tid; e < NXn; e += T)
    if (e >= sx && e < sx + kLoc * kNX) snap0[SN.x + e - sx] = a.ws.x[gx + e];
  for (int e = tid; e < NUn; e += T)
    if (e >= su && e < su + kLoc * kNU) snap0[SN.u + e - su] = a.ws.u[gu + e];
  for (int e = tid; e < NM; e += T)
    if (e >= sx && e < sx + kLoc * kNX) {
      snap0[SN.vp + e - sx] = a.ws.vc_pos[gm_ + e];
      snap0[SN.vn + e - sx] = a.ws.vc_neg[gm_ + e];
      snap0[SN.ph + e - sx] = a.ws.dyn_dual[gm_ + e];
    }
  for (int e = tid; e < m; e += T)
    if (e >= cut.base && e < cut.base + kLoc) snap0[SN.th + e - cut.base] = a.ws.relax_dual[gt + e];
  block_barrier();

  // boundary columns of this thread (pipg.hpp:408-413): bit q set when own x column q is assigned
  int fix_bits = 0;
  const double* fix_val = init_val;
  const bool last_node = t.primal && t.k == n - 1;
  if (t.primal && (t.k == 0 || t.k == n - 1)) {
    const double* on = last_node ? final_on : init_on;
    fix_val = last_node ? final_val : init_val;
#pragma unroll
    for (int q = 0; q < RT::nxc; ++q)
      if (on[RT::xc(q)] != 0.0) fix_bits |= 1 << q;
  }

  const bool warp_fix = __any_sync(kFull, fix_bits != 0);  // warp-uniform

  // owner-private extrapolated copies
  double xe[RT::nxc], ue[RT::nuc], vpe[RT::nrow], vne[RT::nrow], phe[RT::nrow], the = 0.0;
#pragma unroll
  for (int q = 0; q < RT::nxc; ++q) xe[q] = t.primal ? snap0[SN.x + tl * kNX + RT::xc(q)] : 0.0;
#pragma unroll
  for (int q = 0; q < RT::nuc; ++q) ue[q] = t.primal ? snap0[SN.u + tl * kNU + RT::uc(q)] : 0.0;
#pragma unroll
  for (int r = 0; r < RT::nrow; ++r) {
    const int e = tl * kNX + RT::row(r);
    vpe[r] = t.ival ? snap0[SN.vp + e] : 0.0;
    vne[r] = t.ival ? snap0[SN.vn + e] : 0.0;
    phe[r] = t.ival ? snap0[SN.ph + e] : 0.0;
    if (t.auth) phi_s[RT::row(r) * S] = phe[r];
  }
  if (R == 0) {
    the = t.ival ? snap0[SN.th + tl] : 0.0;
    if (t.auth) th_s[0] = the;
  }
  // cluster: the owners of the boundary interval store its (extrapolated) duals in the partner's
  // slots as well, after the warm start (phase 0) and after every iteration j (phase j)
  const bool pusher = kCluster && t.auth && t.k == (cut.rank == 0 ? cut.hi - 1 : cut.lo);
  const int pslot = cut.rank == 0 ? 1 : cut.lo + 1;  // slot of that interval over there
  const unsigned rphi = port.rsm + 8u * (unsigned)(L.phi + pslot), rth = port.rsm + 8u * (unsigned)(L.th + pslot);
  auto push_duals = [&]() {
    if (pusher) {
#pragma unroll
      for (int r = 0; r < RT::nrow; ++r) push_f64(rphi + 8u * (unsigned)(RT::row(r) * S), phe[r], port.rbox);
      if (R == 0) push_f64(rth, the, port.rbox);
    }
  };
  if constexpr (kCluster) push_duals();
  int phase = 0;  // of the duals' mailbox

  const double sigma = a.sigma[b];
  const double alpha = 2.0 / (a.shape.w_prox + sqrt(a.shape.w_prox * a.shape.w_prox + 4.0 * a.omega * sigma));
  const double beta = a.omega * alpha;
  // extrapolation (pipg.hpp:461-472) (1 - rho) * ex + rho * cur, evaluated as ex + rho * (cur - ex)
  auto extrapolate = [&](double ex, double cur) { return fma(a.rho, cur - ex, ex); };
  block_barrier();

  // One iteration.  kStore additionally writes the new *_cur values of every owner into `snap`.
  auto iteration = [&](auto store_tag, double* snap) {
    constexpr bool kStore = decltype(store_tag)::value;
    if constexpr (kCluster) port.recv_phi(phase++);
    // ---- primal projected-gradient step (pipg.hpp:388-420) by the owner of each entry
    double rx[RT::nxc], ru[RT::nuc];
    {
      double gx_[RT::nxc], gm[RT::nuc], gp[RT::nuc];
      transposed<K, R, S, true>(op, phi_s, gx_, gm, gp);
#pragma unroll
      for (int q = 0; q < RT::nxc; ++q) {
        const int c = RT::xc(q);
        const double x0 = xe[q];
        double base = x0 * a.shape.w_prox;
        base += cost_s[c * S];  // zero but at the last node: no branch, no predicated address arithmetic
        base += -phi_s[c * S - 1];
        if (c == kNX - 1) base += th_s[-1] - th_s[0];
        const double grad = base + gx_[q];
        double xn = x0 + -alpha * grad;
        if (warp_fix) xn = (fix_bits & (1 << q)) ? fix_val[c] : xn;  // (measured: faster than unconditional)
        rx[q] = fma(2.0, xn, -x0);
        if (kStore && t.auth) snap[SN.x + tl * kNX + c] = xn;
        xe[q] = extrapolate(x0, xn);
      }
#pragma unroll
      for (int q = 0; q < RT::nuc; ++q) {
        double gpp = __shfl_up_sync(kFull, gp[q], 1);
        gpp = lane == 0 ? 0.0 : gpp;
        const double u0 = ue[q];
        const double grad = u0 * a.shape.w_prox + (gm[q] + gpp);
        double un = u0 + -alpha * grad;
        const double lo = bnd_s[(2 * q) * S], hi = bnd_s[(2 * q + 1) * S];
        // std::max(lo, std::min(hi, v)), pipg.hpp:418-419
        un = clamp_box(lo, hi, un);
        ru[q] = fma(2.0, un, -u0);
        if (kStore && t.auth) snap[SN.u + tl * kNU + RT::uc(q)] = un;
        ue[q] = extrapolate(u0, un);
      }
    }
    // ---- forward products of the reflections: partial row sums of the own columns
    double run[RT::nuc];
#pragma unroll
    for (int q = 0; q < RT::nuc; ++q) run[q] = __shfl_down_sync(kFull, ru[q], 1);
    double xnx[RT::nrow];
#pragma unroll
    for (int r = 0; r < RT::nrow; ++r) {
      const int jc = aligned_col<K, R>(RT::row(r));
      xnx[r] = jc >= 0 ? __shfl_down_sync(kFull, rx[jc >= 0 ? jc : 0], 1) : 0.0;
    }
    double drift = 0.0;
    if (R == 0) drift = __shfl_down_sync(kFull, rx[4], 1) - rx[4];  // K = 4: role 0 owns x[y]
#pragma unroll
    for (int q = 0; q < RT::nxc; ++q) {
      const int slot = xn_slot<K>(RT::xc(q));
      if (slot >= 0 && t.pubx) xn_s[slot * S] = rx[q];
    }
    double own[RT::nrow];
    forward_publish<K, R, S, false>(op, rx, ru, run, part_s, t.auth, own);
    block_barrier();
    // ---- slacks (pipg.hpp:423-430), PI feedback of the constraint violation (:433-458),
    //      extrapolation of the dual groups (:468-472)
    double s[RT::nrow];
    gather_rows<K, R, S>(own, part_s, s);
#pragma unroll
    for (int r = 0; r < RT::nrow; ++r) {
      const int i = RT::row(r);
      const double xn = aligned_col<K, R>(i) >= 0 ? xnx[r] : xn_s[xn_slot<K>(i) * S + 1];
      double resid = s[r] - xn;
      const double p0 = phe[r], vp0 = vpe[r], vn0 = vne[r];
      const double vp = clip0(vp0 - alpha * (a.shape.w_ep + p0));
      const double vn = clip0(vn0 - alpha * (a.shape.w_ep - p0));
      resid += (2.0 * vp - vp0) - (2.0 * vn - vn0) + wv_s[i * S];
      const double pn = p0 + beta * resid;
      if (kStore && t.ival) {
        const int e = tl * kNX + i;
        snap[SN.vp + e] = vp;
        snap[SN.vn + e] = vn;
        snap[SN.ph + e] = pn;
      }
      // rows of nodes without an interval (zero operator, zero neighbours, zero right-hand side,
      // w_ep >= 0) stay exact zeros; only real intervals are stored
      phe[r] = extrapolate(p0, pn);
      vpe[r] = extrapolate(vp0, vp);
      vne[r] = extrapolate(vn0, vn);
      if (t.ival) phi_s[i * S] = phe[r];
    }
    if (R == 0) {
      const double tn = clip0(the + beta * (drift - eps_s[0]));
      if (kStore && t.ival) snap[SN.th + tl] = tn;
      the = extrapolate(the, tn);
      if (t.ival) th_s[0] = the;
    }
    if constexpr (kCluster) push_duals();
    block_barrier();
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
      iteration(std::true_type{}, snap0 + cur_set * SN.total);
    } else {
      iteration(std::false_type{}, nullptr);
    }
    iters = j;
    if (check) {  // stopping_custom(cur, prev) and the divergence test, pipg.hpp:475-487
      const int verdict = pipg_check_x<kHalves, kCluster>(snap0 + cur_set * SN.total, snap0 + (cur_set ^ 1) * SN.total,
                                                        cut.lo - cut.base, cut.hi - cut.lo,
                                                        (cut.hi < m ? cut.hi : m) - cut.lo, red, a.eps_abs, a.eps_rel);
      if (verdict == 2) {
        diverged = true;
        break;
      }
      if (verdict == 1) {
        converged = true;
        break;
      }
    }
  }

  if constexpr (kCluster) {  // the duals sent after the last iteration: nothing may be in flight at the exit
    port.recv_phi(phase);
    cg::this_cluster().sync();
  }
  if (diverged) {  // SolverDiverged(j): the workspace is left untouched, pipg.hpp:478
    if (tid == 0 && cut.rank == 0) {
      if (a.status) a.status[b] = kStSolverDiverged;
      if (a.fail_index) a.fail_index[b] = iters;
      if (a.iterations) a.iterations[b] = iters;
      if (a.converged) a.converged[b] = 0;
      if (a.active) a.active[b] = 0;
    }
    return;
  }
  // solution = the *_cur groups, pipg.hpp:490-495 (every iteration ends with a barrier)
  const double* cur = snap0 + cur_set * SN.total;
  const int hi_m = cut.hi < m ? cut.hi : m;  // owned nodes [lo, hi), owned intervals [lo, hi_m)
  for (int e = tid + cut.lo * kNX; e < cut.hi * kNX; e += T) a.ws.x[gx + e] = cur[SN.x + e - sx];
  for (int e = tid + cut.lo * kNU; e < cut.hi * kNU; e += T) a.ws.u[gu + e] = cur[SN.u + e - su];
  for (int e = tid + cut.lo * kNX; e < hi_m * kNX; e += T) {
    a.ws.vc_pos[gm_ + e] = cur[SN.vp + e - sx];
    a.ws.vc_neg[gm_ + e] = cur[SN.vn + e - sx];
    a.ws.dyn_dual[gm_ + e] = cur[SN.ph + e - sx];
  }
  for (int e = tid + cut.lo; e < hi_m; e += T) a.ws.relax_dual[gt + e] = cur[SN.th + e - cut.base];
  if (tid == 0 && cut.rank == 0) {
    if (a.iterations) a.iterations[b] = iters;
    if (a.converged) a.converged[b] = converged ? 1 : 0;
  }
}

template <int kHalves, bool kCluster>
__global__ void __launch_bounds__(CsCfg<4, kHalves>::threads, 1) pipg_cs_cluster_kernel(PipgArgs a, unsigned char* handled) {
  extern __shared__ __align__(16) double sm[];
  const int b = kCluster ? blockIdx.x >> 1 : blockIdx.x;
  if (a.active && !a.active[b]) return;  // both CTAs of a cluster leave together
  // Warps w and w + 4 share a scheduler; the roles differ in length, and in this kernel a scheduler
  // does better with one longer and one shorter role than with the same role twice (measured:
  // 16.9 -> 16.6 ms per 2 500 iterations x four waves; the power kernel loses with it, 43.6 -> 45.1)
  const int w = threadIdx.x >> 5;
  switch (w < 4 ? w : (w + 2) & 3) {
    case 0: pipg_role_x<4, 0, kHalves, kCluster>(a, sm, b, handled); break;
    case 1: pipg_role_x<4, 1, kHalves, kCluster>(a, sm, b, handled); break;
    case 2: pipg_role_x<4, 2, kHalves, kCluster>(a, sm, b, handled); break;
    default: pipg_role_x<4, 3, kHalves, kCluster>(a, sm, b, handled); break;
  }
}

}  // namespace

bool solver_cs_supports(const SubShape& s, bool has_a_plus) {
  return solver_fast_supports(s, has_a_plus) && s.n <= kCsClusterMaxNodes;
}

namespace {
template <int K, int kHalves>
cudaError_t opt_in_power() {
  return cudaFuncSetAttribute(power_cs_kernel<K, kHalves>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(sizeof(double) * cs_layout<K, kHalves>(false).total));
}
template <int kHalves>
cudaError_t opt_in_pipg() {
  return cudaFuncSetAttribute(pipg_cs_kernel<kHalves>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(sizeof(double) * cs_layout<4, kHalves>(true).total));
}
constexpr size_t kPowerClusterSmem = sizeof(double) * cs_layout<4, 2>(false).total;
constexpr size_t kPipgClusterSmem = sizeof(double) * cs_layout<4, 2>(true, true).total;
template <int K, int kHalves>
void launch_power(const PowerArgs& a, unsigned char* handled, cudaStream_t stream) {
  power_cs_kernel<K, kHalves><<<a.batch, CsCfg<K, kHalves>::threads, sizeof(double) * cs_layout<K, kHalves>(false).total, stream>>>(a, handled);
}
/// One instance over a cluster of two CTAs (kCsMaxNodes < n <= kCsClusterMaxNodes).
template <class Kernel, class Args>
cudaError_t launch_cluster(Kernel kernel, const Args& a, size_t smem, unsigned char* handled, cudaStream_t stream) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2u * (unsigned)a.batch);
  cfg.blockDim = dim3(CsCfg<4, 2>::threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 2;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, a, handled);
}
}  // namespace

size_t pipg_cs_smem(const SubShape& s) {
  if (s.n > kCsMaxNodes) return kPipgClusterSmem;
  return sizeof(double) * (size_t)(s.n <= CsCfg<4, 1>::cap ? cs_layout<4, 1>(true).total : cs_layout<4, 2>(true).total);
}

cudaError_t configure_solver_cs(const SubShape&) {
  cudaError_t e = opt_in_power<4, 1>();
  if (e == cudaSuccess) e = opt_in_power<4, 2>();
  if (e == cudaSuccess) e = opt_in_pipg<1>();
  if (e == cudaSuccess) e = opt_in_pipg<2>();
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(power_cs_cluster_kernel<4, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kPowerClusterSmem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(pipg_cs_cluster_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kPipgClusterSmem);
  return e;
}

cudaError_t launch_power_cs(const PowerArgs& a, unsigned char* handled, cudaStream_t stream) {
  if (a.shape.n > kCsMaxNodes)
    return launch_cluster(power_cs_cluster_kernel<4, 2, true>, a, kPowerClusterSmem, handled, stream);
  if (a.shape.n <= CsCfg<4, 1>::cap) launch_power<4, 1>(a, handled, stream);
  else launch_power<4, 2>(a, handled, stream);
  return cudaGetLastError();
}

cudaError_t launch_pipg_cs(const PipgArgs& a, unsigned char* handled, cudaStream_t stream) {
  if (a.shape.n > kCsMaxNodes)
    return launch_cluster(pipg_cs_cluster_kernel<2, true>, a, kPipgClusterSmem, handled, stream);
  if (a.shape.n <= CsCfg<4, 1>::cap) {
    pipg_cs_kernel<1><<<a.batch, CsCfg<4, 1>::threads, sizeof(double) * cs_layout<4, 1>(true).total, stream>>>(a, handled);
  } else {
    pipg_cs_kernel<2><<<a.batch, CsCfg<4, 2>::threads, sizeof(double) * cs_layout<4, 2>(true).total, stream>>>(a, handled);
  }
  return cudaGetLastError();
}

}  // namespace ptopt_b200
