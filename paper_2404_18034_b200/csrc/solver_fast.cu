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
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"
#include "mailbox.cuh"

namespace ptopt_b200 {

namespace cg = cooperative_groups;

namespace {

constexpr int kG = 5;        // threads per node
constexpr int kR = 3;        // operator rows per thread
constexpr int kW = kNX + 2 * kNU;  // 29 columns of [A- | B- | B+]
constexpr int kXS = 18;      // node stride of x vectors in shared memory (16-byte aligned, conflict-free)
constexpr int kUS = 10;      // node stride of u vectors
constexpr int kPS = 35;      // stride of one thread's partial-sum slot (== 3 mod 16: conflict-free)
constexpr int kFastWarps = 8;  // slots of the reduction arrays (any variant has at most this many warps)
constexpr int kPipgClusterSpill = 14;  // operator entries per thread the cluster PIPG kernel keeps in shared memory

// Two compile-time shapes of a CTA.  kCap = kFastMaxNodes (51 nodes, 256 threads, one CTA per SM)
// holds a whole instance of up to 51 nodes, or half of a 2-CTA cluster for up to 102.  kCap =
// kSplitMaxNodes (25 nodes, 128 threads, 112 KB of shared memory) is half of an instance of up to
// 50 nodes: two such CTAs -- halves of two different instances -- share one SM, so that the
// shared-memory phases of one overlap the FP64 phases of the other instead of running in lockstep.
template <int kCap>
struct FastCfg {
  static constexpr int threads = (kG * kCap + 31) / 32 * 32;
  static constexpr int ctas_per_sm = kCap <= kSplitMaxNodes ? 2 : 1;
  static_assert((threads - 1) / kG <= kCap, "every thread needs a (scratch) node inside the layout");
  static_assert(threads / 32 <= kFastWarps, "reduction slots");
};

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

// The PIPG kernel of the cluster variants needs a dozen registers more than the 255 a thread can
// have next to its 174 of operator; ptxas then spills operator entries to local memory and reloads
// them every iteration.  Those variants keep the last kSpill entries of a thread's third row
// (B+ columns) in a thread-private shared-memory column instead (`opx[c * stride]`, consecutive
// threads in consecutive words: conflict-free) -- chosen, not left to the register allocator.
template <int kSpill>
struct OpTail {
  const double* opx;  // this thread's entry of column 0
  int stride;         // doubles between columns (the CTA's thread count)
  __device__ __forceinline__ static constexpr bool spilled(int r, int j) { return r == kR - 1 && j >= kW - kSpill; }
  __device__ __forceinline__ double get(const double (&a)[kR][kW], int r, int j) const {
    return spilled(r, j) ? opx[(j - (kW - kSpill)) * stride] : a[r][j];
  }
};

/// Row r of the forward product: A- x_k, B- u_k, B+ u_{k+1}, each summed in ascending column
/// order (mat_vec, smallmat.hpp:93-97).
template <int kSpill>
__device__ __forceinline__ void row_products(const double (&a)[kR][kW], const OpTail<kSpill>& tail,
                                             const double (&v)[kW], int r, double& pa, double& pm, double& pp) {
  double sa = 0.0, sm = 0.0, sp = 0.0;
#pragma unroll
  for (int j = 0; j < kNX; ++j) sa += tail.get(a, r, j) * v[j];
#pragma unroll
  for (int j = 0; j < kNU; ++j) {
    sm += tail.get(a, r, kNX + j) * v[kNX + j];
    sp += tail.get(a, r, kNX + kNU + j) * v[kNX + kNU + j];
  }
  pa = sa;
  pm = sm;
  pp = sp;
}

/// Publishes the partial column sums of this thread's three rows against its three dual entries.
template <int kSpill>
__device__ __forceinline__ void store_partials(const double (&a)[kR][kW], const OpTail<kSpill>& tail,
                                               const double (&d)[kR], double* slot) {
#pragma unroll
  for (int j = 0; j < kW; ++j) {
    double p = a[0][j] * d[0];
    p += a[1][j] * d[1];
    p += tail.get(a, 2, j) * d[2];
    slot[pos_col(j)] = p;
  }
}

/// Moves the entries OpTail serves out of the register copy (after load_rows).
template <int kSpill>
__device__ __forceinline__ void park_tail(double (&a)[kR][kW], double* opx, int stride) {
#pragma unroll
  for (int c = 0; c < kSpill; ++c) {
    opx[c * stride] = a[kR - 1][kW - kSpill + c];
    a[kR - 1][kW - kSpill + c] = 0.0;
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
  int wv, eps, umin, umax, snap, bnd, opx;
};

// One snapshot of the *_cur groups (pipg.hpp:490-495), with room for the scratch entries the
// idle threads write: x [n+2][15], u [n+2][7 (+3)], vc+, vc-, dyn dual [n+2][15], relax dual [n+2].
struct SnapLayout {
  int x, u, vp, vn, ph, th, total;
};
template <int kCap>
__host__ __device__ constexpr SnapLayout snap_layout() {
  constexpr int n = kCap + 3;
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
template <int kCap>
__host__ __device__ constexpr FastLayout fast_layout(bool pipg) {
  constexpr int n = kCap;  // fixed offsets: every address is base + immediate
  constexpr int kThreads = FastCfg<kCap>::threads;
  FastLayout L{};
  int o = 0;
  L.xs = o; o += (n + 4) * kXS;
  L.us = o; o += (n + 4) * kUS;
  L.phi = o + kNX + 1; o += even_up((n + 3) * kNX + 2);
  L.theta = o + 2; o += even_up(n + 6);
  L.part = o + kG * kPS + 1; o += even_up(kG * kPS + 1 + (n + 3) * kG * kPS);
  L.red = o; o += 16 * kFastWarps;  // power: [2][warps] own + [2][warps] partner; pipg: [warps][8]
  if (pipg) {
    L.wv = o; o += even_up((n + 3) * kNX);
    L.eps = o; o += even_up(n + 4);
    L.umin = o; o += 2 * kThreads;  // {lo, hi} of each thread's first control entry
    L.umax = o; o += 2 * kThreads;  // {lo, hi} of its second one (+-inf where it has none)
    L.snap = o; o += 2 * snap_layout<kCap>().total;
    L.bnd = o; o += 6 * 16;  // ecost, init_val, final_val, init_on, final_on (as doubles)
    L.opx = o; o += kPipgClusterSpill * kThreads;  // OpTail columns (cluster variants)
  }
  L.total = o;
  return L;
}

// ---------------------------------------------------------------------------------------------
// Horizon split.  Up to kFastMaxNodes nodes one CTA holds the whole instance.  Above that (up to
// 2 * kFastMaxNodes) a thread-block cluster of two CTAs shares it: rank 0 takes the first
// ceil(n/2) nodes, rank 1 the rest; each keeps its operator rows in its own SM's registers.  The
// only coupling across the cut is the one between neighbouring nodes, so the owners of the boundary
// values store them twice: locally, and through distributed shared memory into the guard entries
// the partner's single-CTA code already reads — rank 1's first node vectors into rank 0's "next
// node" slot, rank 0's last interval (B+ partial sums, duals) into rank 1's "previous interval"
// slots, every warp's share of a reduction into the partner's copy.  Nothing is ever read remotely.
//
// Hand-off.  A release/acquire cluster barrier costs ~500 cycles on B200 and the hot loops would
// need two per iteration (tools/probes/cluster_sync_cost.cu).  Instead every remote store is an
// asynchronous store that completes transaction bytes on an mbarrier in the RECEIVER's shared
// memory ("mailbox"): the receiver arms the barrier with the byte count of the phase and only the
// warps that read the guard entries wait for it; phase boundaries inside a CTA stay plain block
// barriers.  One way, no fence (~150 cycles).  Overwriting a guard entry before the partner has
// read it is excluded by data dependence: a CTA can only produce the next value after it has
// received everything the partner computed from the previous one.
// ---------------------------------------------------------------------------------------------
enum Mailbox { kBoxPrev = 0, kBoxNext = 1, kBoxNorm = 2 /* and 3: by trip parity */, kBoxes = 4 };
constexpr int kBoxOffset = 12 * kFastWarps;                 // mbarriers live in the unused tail of `red`
constexpr int kPrevBytes = 8 * (kNX + 1 + kG * kNU);        // duals + relaxation dual + B+ partial sums
constexpr int kNextBytes = 8 * (kNX + kNU);                 // first node vectors of rank 1

/// Per-thread view of the mailboxes of a cluster CTA.
struct Boxes {
  unsigned long long* local;  // [kBoxes] in this CTA's shared memory
  unsigned remote;            // the partner's [kBoxes] (shared::cluster address)
  bool prev_warp, next_warp;  // this warp reads the "previous interval" / "next node" guard entries
  bool prev_armer, next_armer, norm_armer;
  int norm_bytes;
  __device__ __forceinline__ unsigned box(int which) const { return remote + 8u * (unsigned)which; }
  /// Arms mailbox `which` for `phase` (one thread) and waits until its bytes have arrived.
  __device__ __forceinline__ void receive(int which, bool mine, bool armer, int bytes, int phase) const {
    if (!mine) return;
    if (armer) mbar_expect(local + which, bytes);
    mbar_wait(local + which, phase);
  }
  __device__ __forceinline__ void recv_prev(int phase) const { receive(kBoxPrev, prev_warp, prev_armer, kPrevBytes, phase); }
  __device__ __forceinline__ void recv_next(int phase) const { receive(kBoxNext, next_warp, next_armer, kNextBytes, phase); }
  /// Norm shares of trip `trip` (0: the seed).  This exchange is not a ping-pong -- both CTAs send
  /// every trip, and rank 0 may run up to one trip ahead of rank 1 (only its NEXT forward map needs
  /// rank 1's boundary node) -- so one mailbox would see the shares of trip t + 1 before trip t is
  /// armed or polled (lost bytes, or a phase parity that flips twice under a slow warp).  Two
  /// mailboxes alternate by trip parity instead: a CTA can never be two trips ahead.
  __device__ __forceinline__ unsigned norm_box(int trip) const { return box(kBoxNorm + (trip & 1)); }
  __device__ __forceinline__ void recv_norm(int trip) const {
    receive(kBoxNorm + (trip & 1), true, norm_armer, norm_bytes, trip >> 1);
  }
};

/// Initialises the mailboxes (after the shared memory has been cleared) and meets the partner, so
/// that both CTAs are running, cleared and armed before any remote store.
template <bool kCluster>
__device__ __forceinline__ Boxes open_boxes(double* red, const struct Split& cut, int tid, int warp, int nwarps);

struct Split {
  int rank;   // CTA rank inside the cluster (0 without clusters)
  int node0;  // first global node of this CTA
  int nloc;   // nodes of this CTA
  int half;   // nodes of rank 0
};

template <bool kCluster>
__device__ __forceinline__ Split make_split(int n) {
  Split sp;
  if constexpr (kCluster) {
    sp.rank = (int)cg::this_cluster().block_rank();
    sp.half = (n + 1) / 2;
    sp.node0 = sp.rank * sp.half;
    sp.nloc = sp.rank == 0 ? sp.half : n - sp.half;
  } else {
    sp.rank = 0;
    sp.half = n;
    sp.node0 = 0;
    sp.nloc = n;
  }
  return sp;
}

/// Address of `local` (a pointer into this CTA's shared memory) inside CTA `rank` of the cluster.
template <class T>
__device__ __forceinline__ T* in_cta(T* local, int rank) {
  return cg::this_cluster().map_shared_rank(local, rank);
}

template <bool kCluster>
__device__ __forceinline__ Boxes open_boxes(double* red, const Split& cut, int tid, int warp, int nwarps) {
  Boxes bx{};
  if constexpr (kCluster) {
    bx.local = reinterpret_cast<unsigned long long*>(red + kBoxOffset);
    __syncthreads();  // the clearing loop is done
    if (tid == 0) {
#pragma unroll
      for (int i = 0; i < kBoxes; ++i) mbar_init(bx.local + i, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cg::this_cluster().sync();
    bx.remote = partner_u32(bx.local, cut.rank ^ 1);
    const int bfirst = kG * (cut.half - 1);  // threads of rank 0's last node: bfirst .. bfirst + kG - 1
    bx.prev_warp = cut.rank == 1 && warp == 0;
    bx.next_warp = cut.rank == 0 && (warp == (bfirst >> 5) || warp == ((bfirst + kG - 1) >> 5));
    bx.prev_armer = cut.rank == 1 && tid == 0;
    bx.next_armer = cut.rank == 0 && tid == bfirst;
    bx.norm_armer = tid == 0;
    bx.norm_bytes = 8 * nwarps;
  } else {
    __syncthreads();
  }
  return bx;
}

/// Sends the B+ partial sums a thread has just published in `slot` to `remote_slot` (the matching
/// "previous interval" guard slot of the partner CTA).
__device__ __forceinline__ void push_bp_partials(const double* slot, unsigned remote_slot, unsigned box) {
#pragma unroll
  for (int c = 0; c < kNU; ++c) push_f64(remote_slot + 8u * pos_bp(c), slot[pos_bp(c)], box);
}

// ---------------------------------------------------------------------------------------------
// power iteration (pipg.hpp:206-292)
// ---------------------------------------------------------------------------------------------
template <bool kCluster, int kCap>
__global__ void __launch_bounds__(FastCfg<kCap>::threads, FastCfg<kCap>::ctas_per_sm)
power_fast_kernel(PowerArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int b = kCluster ? blockIdx.x >> 1 : blockIdx.x;
  if (a.active && !a.active[b]) return;  // both CTAs of a cluster leave together
  if (a.skip && a.skip[b]) return;       // solved by the column-sparse kernels (solver_cs.cu)
  const int n = a.shape.n, m = n - 1;
  const Split cut = make_split<kCluster>(n);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = blockDim.x, nwarps = T >> 5;  // launched with just enough warps for 5 threads per node
  const int k = tid / kG, g = tid - k * kG;   // local node, row group
  const int kg = cut.node0 + k;               // global node
  const bool node = k < cut.nloc, ival = node && kg < m;
  // threads past the last node work on scratch nodes of their own; in a cluster node `nloc` of
  // rank 0 is not scratch (the partner pushes its first node there), so they start one further
  const int kc = (kCluster && k >= cut.nloc) ? k + 1 : k;
  constexpr FastLayout L = fast_layout<kCap>(false);
  for (int e = tid; e < L.total; e += T) sm[e] = 0.0;
  const Boxes bx = open_boxes<kCluster>(sm + L.red, cut, tid, warp, nwarps);
  double* xs_k = sm + L.xs + kc * kXS;          // x_k; x_{k+1} at +kXS
  double* us_k = sm + L.us + kc * kUS;
  double* phi_k = sm + L.phi + kc * kNX + kR * g;  // own dual entries; interval k-1 at -kNX
  double* th_k = sm + L.theta + kc;
  double* part = sm + L.part;
  double* slot = part + (size_t)tid * kPS;
  const double* part_k = part + (size_t)kc * kG * kPS;  // slots of interval k; k-1 at -kG*kPS
  double* red = sm + L.red;       // [2][kFastWarps] own partial sums of the norm, by trip parity
  double* redp = red + 2 * kFastWarps;  // the partner's (clusters only)
  const int ju1 = g + 5;                        // second control entry (g >= 2: a padding slot of its own)
  // boundary owners of a cluster: the last node of rank 0 feeds rank 1's "previous interval"
  // guard entries, the first node of rank 1 feeds rank 0's "next node" entries
  const bool push_prev = kCluster && cut.rank == 0 && k == cut.half - 1;
  const bool push_next = kCluster && cut.rank == 1 && k == 0 && node;
  // Sum of the warps' shares of one parity (slots of warps that do not exist stay zero), as a
  // pairwise tree: three dependent additions instead of seven on every thread's critical path.
  auto share_sum = [&](const double* shares) {
    static_assert(kFastWarps == 8, "tree below");
    const double2* p = reinterpret_cast<const double2*>(shares);
    const double2 a = p[0], b = p[1], c = p[2], d = p[3];
    return ((a.x + a.y) + (b.x + b.y)) + ((c.x + c.y) + (d.x + d.y));
  };
  auto norm_sq = [&](int parity) {  // both CTAs' shares, rank 0's first
    const double own = share_sum(red + parity * kFastWarps);
    if constexpr (kCluster) {
      const double other = share_sum(redp + parity * kFastWarps);
      return cut.rank == 0 ? own + other : other + own;
    }
    return own;
  };

  double aop[kR][kW];
  double vcd[kR];  // vc+ - vc-: the only combination of the two groups the forward map uses
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    vcd[r] = 0.0;
#pragma unroll
    for (int j = 0; j < kW; ++j) aop[r][j] = 0.0;
  }
  if (ival) load_rows(a.sp, b, m, kg, g, aop);

  // seed (pipg.hpp:213-230): x, u, vc+, vc-; sigma0 = ||seed||_2
  double acc = 0.0;
  if (node) {
    const double* sx = a.seed_x + ((size_t)b * n + kg) * kNX;
    const double* su = a.seed_u + ((size_t)b * n + kg) * kNU;
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
    const double* sp = a.seed_vcp + ((size_t)b * m + kg) * kNX;
    const double* sn = a.seed_vcn + ((size_t)b * m + kg) * kNX;
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const double vp = sp[kR * g + r], vn = sn[kR * g + r];
      vcd[r] = vp - vn;
      acc += vp * vp;
      acc += vn * vn;
    }
  }
  if constexpr (kCluster) {  // rank 0's "next node" is the partner's first node
    if (cut.rank == 0 && tid < kNX + kNU) {
      const size_t gn = (size_t)b * n + cut.half;
      if (tid < kNX) sm[L.xs + cut.nloc * kXS + tid] = a.seed_x[gn * kNX + tid];
      else sm[L.us + cut.nloc * kUS + tid - kNX] = a.seed_u[gn * kNU + tid - kNX];
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) {
    red[warp] = acc;
    if constexpr (kCluster) push_f64(partner_u32(redp + warp, cut.rank ^ 1), acc, bx.norm_box(0));
  }
  __syncthreads();
  if constexpr (kCluster) bx.recv_norm(0);  // the seed's shares
  double sigma = norm_sq(0);
  if (sigma == 0.0) {  // pipg.hpp:224-225
    if (tid == 0 && cut.rank == 0) {
      if (a.status) a.status[b] = kStSeedZero;
      a.sigma[b] = 0.0;
      if (a.trips) a.trips[(size_t)b * a.trips_stride + (a.trips_slot ? a.trips_slot[b] : 0)] = 0;
    }
    if constexpr (kCluster) cg::this_cluster().sync();  // the partner may still be reading
    return;
  }
  // Inside the loop sigma is ss * rsqrt(ss) (1 ulp from sqrt: it only feeds the stopping test) and
  // the scale 1 / sigma of pipg.hpp:243 the same rsqrt: no square root and no division on the
  // trip's critical path.  The value returned is the correctly rounded sqrt of the last squared norm.
  double ss_last = sigma;
  double inv = rsqrt(ss_last);
  sigma = ss_last * inv;

  // The norm of trip j-1 is reduced while trip j's forward products are already running: the
  // products do not need sigma until they are scaled, so the block reduction, the square root
  // and the reciprocal overlap with them instead of forming a serial stage of their own.
  int trips = 0;
  bool done = false;
  for (int j = 1; j <= a.j_max; ++j) {
    // ---- forward map (pipg.hpp:234-245): products first, then the scale 1/sigma
    if constexpr (kCluster) {
      if (j > 1) bx.recv_next(j - 2);  // rank 1's first node of trip j-1 ("next" phase j-2)
    }
    double v[kW];
    load_node_vectors(xs_k, us_k, v);
    double s[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      double pa, pm, pp;
      row_products(aop, OpTail<0>{}, v, r, pa, pm, pp);
      // pipg.hpp:235-241 adds the six terms one after the other; paired here (three dependent
      // additions instead of five)
      s[r] = ((pa - xs_k[kXS + kR * g + r]) + (pm + pp)) + vcd[r];
    }
    const double dy = xs_k[kXS + 14] - v[14];
    if (j > 1) {  // stopping test of trip j-1 (pipg.hpp:277-289)
      if constexpr (kCluster) bx.recv_norm(j - 1);
      const double ss = norm_sq((j - 1) & 1);
      ss_last = ss;
      if (ss == 0.0) {  // iterate in the null space, pipg.hpp:280-284
        done = true;
        break;
      }
      inv = rsqrt_pos(ss);
      const double sigma_star = ss * inv;
      const bool hit = fabs(sigma_star - sigma) <= a.eps_abs + a.eps_rel * max_nn(sigma_star, sigma);
      sigma = sigma_star;
      if (hit) {
        done = true;
        break;
      }
    }
    trips = j;
    double phi[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      phi[r] = ival ? s[r] * inv : 0.0;
      phi_k[r] = phi[r];
    }
    // pipg.hpp:244 divides by sigma; the reciprocal is already there (1 ulp, and one division
    // chain less on every thread's critical path)
    const double th = ival ? dy * inv : 0.0;
    if (g == 4) th_k[0] = th;
    if (push_prev) {  // the same values into rank 1's guard entries for interval -1
      const unsigned rphi = partner_u32(sm + L.phi - kNX + kR * g, 1);
#pragma unroll
      for (int r = 0; r < kR; ++r) push_f64(rphi + 8u * r, phi[r], bx.box(kBoxPrev));
      if (g == 4) push_f64(partner_u32(sm + L.theta - 1, 1), th, bx.box(kBoxPrev));
    }
    store_partials(aop, OpTail<0>{}, phi, slot);
    if (push_prev) push_bp_partials(slot, partner_u32(part - kG * kPS + g * kPS, 1), bx.box(kBoxPrev));
    // vc+ = phi, vc- = -phi (so vc+ - vc- = 2 phi, exactly) and their share of the norm,
    // phi^2 + phi^2 (pipg.hpp:268-279)
    double acc_d = 0.0;
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      vcd[r] = 2.0 * phi[r];
      acc_d = fma(vcd[r], phi[r], acc_d);
    }
    __syncthreads();
    // ---- adjoint map (pipg.hpp:247-275): every primal entry is assembled by its owner.  The sums
    //      over the thread's own interval come first: in a cluster they hide part of the flight
    //      time of the partner's boundary values, which only the previous-interval terms need.
    double sx[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) sx[r] = column_sum(part_k, kR * g + r);
    const double su0_own = column_sum(part_k, 15 + 3 * g), su1_own = column_sum(part_k, 16 + 3 * g);
    if constexpr (kCluster) bx.recv_prev(j - 1);  // rank 0's last interval of this trip
    const double su0 = su0_own + column_sum(part_k - kG * kPS, 17 + 3 * g);
    const double su1 = su1_own + column_sum(part_k - kG * kPS, 22 + 3 * g);
    double acc_x = 0.0;
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      double t = sx[r] + -phi_k[r - kNX];
      if (r == kR - 1 && g == 4) {
        t += -th_k[0];
        t += th_k[-1];
      }
      xs_k[kR * g + r] = t;
      if (push_next) push_f64(partner_u32(sm + L.xs + cut.half * kXS + kR * g + r, 0), t, bx.box(kBoxNext));
      acc_x += t * t;
    }
    us_k[g] = su0;
    us_k[ju1] = su1;
    if (push_next) {
      const unsigned ru = partner_u32(sm + L.us + cut.half * kUS, 0);
      push_f64(ru + 8u * g, su0, bx.box(kBoxNext));
      if (g < 2) push_f64(ru + 8u * (g + 5), su1, bx.box(kBoxNext));
    }
    double acc_u = su0 * su0;
    acc_u += g < 2 ? su1 * su1 : 0.0;
    acc = node ? (acc_x + acc_u) + acc_d : 0.0;
    acc = warp_sum(acc);
    if (lane == 0) {
      red[(j & 1) * kFastWarps + warp] = acc;
      if constexpr (kCluster)
        push_f64(partner_u32(redp + (j & 1) * kFastWarps + warp, cut.rank ^ 1), acc, bx.norm_box(j));
    }
    __syncthreads();
  }
  if (!done) {  // j_max trips without meeting the tolerance
    if constexpr (kCluster) {
      if (a.j_max >= 1) {  // what the partner sent in the last trip is still on its way
        bx.recv_next(a.j_max - 1);
        bx.recv_norm(a.j_max);
      }
    }
    ss_last = norm_sq(a.j_max & 1);
  }
  if (tid == 0 && cut.rank == 0) {
    a.sigma[b] = (1.0 + a.eps_buff) * sqrt(ss_last);
    if (a.trips) a.trips[(size_t)b * a.trips_stride + (a.trips_slot ? a.trips_slot[b] : 0)] = trips;
  }
  if constexpr (kCluster) cg::this_cluster().sync();  // the partner may still be reading
}

// ---------------------------------------------------------------------------------------------
// customized PIPG (pipg.hpp:350-497)
// ---------------------------------------------------------------------------------------------
template <bool kCluster, int kCap>
__global__ void __launch_bounds__(FastCfg<kCap>::threads, FastCfg<kCap>::ctas_per_sm)
pipg_fast_kernel(PipgArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int b = kCluster ? blockIdx.x >> 1 : blockIdx.x;
  if (a.active && !a.active[b]) return;  // both CTAs of a cluster leave together
  if (a.skip && a.skip[b]) return;       // solved by the column-sparse kernels (solver_cs.cu)
  const int n = a.shape.n, m = n - 1;
  const Split cut = make_split<kCluster>(n);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = blockDim.x, nwarps = T >> 5;  // launched with just enough warps for 5 threads per node
  const int k = tid / kG, g = tid - k * kG;   // local node, row group
  const int kg = cut.node0 + k;               // global node
  const bool node = k < cut.nloc, ival = node && kg < m;
  // threads past the last node work on scratch nodes of their own; in a cluster node `nloc` of
  // rank 0 is not scratch (the partner pushes its first node there), so they start one further
  const int kc = (kCluster && k >= cut.nloc) ? k + 1 : k;
  const int mloc = cut.nloc - (cut.node0 + cut.nloc == n ? 1 : 0);  // intervals owned by this CTA
  constexpr FastLayout L = fast_layout<kCap>(true);
  constexpr SnapLayout S = snap_layout<kCap>();
  for (int e = tid; e < L.total; e += T) sm[e] = 0.0;
  const Boxes bx = open_boxes<kCluster>(sm + L.red, cut, tid, warp, nwarps);
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
  // boundary owners of a cluster: the last node of rank 0 feeds rank 1's "previous interval"
  // guard entries, the first node of rank 1 feeds rank 0's "next node" entries
  const bool push_prev = kCluster && cut.rank == 0 && k == cut.half - 1;
  const bool push_next = kCluster && cut.rank == 1 && k == 0 && node;

  // this CTA's share of the instance-major global arrays
  const size_t gx = ((size_t)b * n + cut.node0) * kNX, gu = ((size_t)b * n + cut.node0) * kNU;
  const size_t gm = ((size_t)b * m + cut.node0) * kNX, gt = (size_t)b * m + cut.node0;
  const int NXn = cut.nloc * kNX, NUn = cut.nloc * kNU, NM = mloc * kNX;
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
  for (int e = tid; e < NM; e += T) sm[L.wv + e] = a.sp.w[gm + e];
  for (int e = tid; e < mloc; e += T) sm[L.eps + e] = a.sp.eps_relax[gt + e];
  {  // box of this thread's control entries (pipg.hpp:418-419); scratch entries are unbounded
    const double* lo = a.sp.u_min + gu + k * kNU;
    const double* hi = a.sp.u_max + gu + k * kNU;
    *bnd0 = node ? make_double2(lo[g], hi[g]) : make_double2(-INFINITY, INFINITY);
    *bnd1 = (node && g < 2) ? make_double2(lo[g + 5], hi[g + 5]) : make_double2(-INFINITY, INFINITY);
  }
  // warm start: ex = cur = workspace (pipg.hpp:362-374); it is snapshot 0
  for (int e = tid; e < NXn; e += T) snap0[S.x + e] = a.ws.x[gx + e];
  for (int e = tid; e < NUn; e += T) snap0[S.u + e] = a.ws.u[gu + e];
  for (int e = tid; e < NM; e += T) {
    snap0[S.vp + e] = a.ws.vc_pos[gm + e];
    snap0[S.vn + e] = a.ws.vc_neg[gm + e];
    snap0[S.ph + e] = a.ws.dyn_dual[gm + e];
  }
  for (int e = tid; e < mloc; e += T) snap0[S.th + e] = a.ws.relax_dual[gt + e];

  double aop[kR][kW];
#pragma unroll
  for (int r = 0; r < kR; ++r)
#pragma unroll
    for (int j = 0; j < kW; ++j) aop[r][j] = 0.0;
  if (ival) load_rows(a.sp, b, m, kg, g, aop);
  constexpr int kSpill = kCluster ? kPipgClusterSpill : 0;
  park_tail<kSpill>(aop, sm + L.opx + tid, T);
  const OpTail<kSpill> tail{sm + L.opx + tid, T};
  __syncthreads();
  auto publish_duals = [&](const double (&phe)[kR], double the) {  // extrapolated duals + partial sums
#pragma unroll
    for (int r = 0; r < kR; ++r) phx_k[r] = phe[r];
    if (g == 4) thx_k[0] = the;
    if (push_prev) {
      const unsigned rphx = partner_u32(sm + L.phi - kNX + kR * g, 1);
#pragma unroll
      for (int r = 0; r < kR; ++r) push_f64(rphx + 8u * r, phe[r], bx.box(kBoxPrev));
      if (g == 4) push_f64(partner_u32(sm + L.theta - 1, 1), the, bx.box(kBoxPrev));
    }
    store_partials(aop, tail, phe, slot);
    if (push_prev) push_bp_partials(slot, partner_u32(part - kG * kPS + g * kPS, 1), bx.box(kBoxPrev));
  };

  // boundary rows of this thread (pipg.hpp:408-413): bit r set when row 3g+r is assigned
  int fix_bits = 0;
  const double* fix_val = init_val;
  const bool last_node = node && kg == n - 1;
  if (node && (kg == 0 || kg == n - 1)) {
    const double* on = last_node ? final_on : init_on;
    fix_val = last_node ? final_val : init_val;
#pragma unroll
    for (int r = 0; r < kR; ++r)
      if (on[kR * g + r] != 0.0) fix_bits |= 1 << r;
  }
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
    }
    if (g == 4) the = snap0[S.th + k];
  }
  publish_duals(phe, the);

  const double sigma = a.sigma[b];
  const double alpha = 2.0 / (a.shape.w_prox + sqrt(a.shape.w_prox * a.shape.w_prox + 4.0 * a.omega * sigma));
  const double beta = a.omega * alpha;
  // extrapolation (pipg.hpp:461-472) (1 - rho) * ex + rho * cur, evaluated as ex + rho * (cur - ex):
  // the same two operations without a loop-long register pair for 1 - rho
  auto extrapolate = [&](double ex, double cur) { return fma(a.rho, cur - ex, ex); };
  __syncthreads();
  // "previous interval" mailbox: phase j = what rank 0 sends after iteration j (0: the warm start);
  // it is received inside the next primal step, or after the loop
  int iter_no = 0;  // iteration the lambda below is running

  // One iteration.  kStore additionally writes the new *_cur values of every owner into the
  // snapshot `snap` (threads without a node / interval write scratch entries).
  auto iteration = [&](auto store_tag, double* snap) {
    constexpr bool kStore = decltype(store_tag)::value;
    // ---- primal projected-gradient step (pipg.hpp:388-420) by the owner of each entry.  The
    //      terms that do not need the partial sums are gathered first so that the dependent
    //      chain behind the shared-memory loads stays short.
    double base[kR], sx[kR];
    double su[2];
    // the sums over the thread's own interval first: in a cluster they hide part of the flight
    // time of the partner's boundary values, which only the previous-interval terms below need
#pragma unroll
    for (int r = 0; r < kR; ++r) sx[r] = column_sum(part_k, kR * g + r);
#pragma unroll
    for (int q = 0; q < 2; ++q) su[q] = column_sum(part_k, q == 0 ? 15 + 3 * g : 16 + 3 * g);
    if constexpr (kCluster) bx.recv_prev(iter_no - 1);  // rank 0's last interval after iteration iter_no - 1 (0: warm start)
#pragma unroll
    for (int q = 0; q < 2; ++q) su[q] += column_sum(part_k - kG * kPS, q == 0 ? 17 + 3 * g : 22 + 3 * g);
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const int i = kR * g + r;
      double t = xe[r] * a.shape.w_prox;
      if (last_node) t += a.shape.w_cost * ecost[i];
      t += -phx_k[r - kNX];
      if (r == kR - 1 && g == 4) t += thx_k[-1] - thx_k[0];
      base[r] = t;
    }
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const int i = kR * g + r;
      const double x0 = xe[r];
      const double grad = base[r] + sx[r];
      double xn = x0 + -alpha * grad;
      if (warp_fix) xn = (fix_bits & (1 << r)) ? fix_val[i] : xn;
      const double xrf = fma(2.0, xn, -x0);
      xr_k[i] = xrf;
      if (push_next) push_f64(partner_u32(sm + L.xs + cut.half * kXS + i, 0), xrf, bx.box(kBoxNext));
      if (kStore) snap[S.x + kc * kNX + i] = xn;
      xe[r] = extrapolate(x0, xn);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int ju = q == 0 ? g : ju1;
      const double u0 = ue[q];
      const double grad = u0 * a.shape.w_prox + su[q];
      double un = u0 + -alpha * grad;
      const double2 bq = q == 0 ? *bnd0 : *bnd1;
      un = clamp_box(bq.x, bq.y, un);  // std::max(lo, std::min(hi, v)), pipg.hpp:418-419
      const double urf = fma(2.0, un, -u0);
      ur_k[ju] = urf;
      if (push_next && (q == 0 || g < 2))
        push_f64(partner_u32(sm + L.us + cut.half * kUS + ju, 0), urf, bx.box(kBoxNext));
      if (kStore) {
        if (q == 0 || g < 2) snap[S.u + kc * kNU + ju] = un;
      }
      ue[q] = extrapolate(u0, un);
    }
    __syncthreads();
    if constexpr (kCluster) bx.recv_next(iter_no - 1);  // rank 1's first node of this iteration

    // ---- slacks (pipg.hpp:423-430), PI feedback of the constraint violation (:433-458),
    //      extrapolation of the dual groups (:468-472) and the partial sums of H^T phi_ex for
    //      the next primal step
    {
      double v[kW];
      load_node_vectors(xr_k, ur_k, v);
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        double pa, pm, pp;
        row_products(aop, tail, v, r, pa, pm, pp);
        double resid = pa + -xr_k[kXS + kR * g + r];
        resid += pm;
        resid += pp;
        const double p0 = phe[r], vp0 = vpe[r], vn0 = vne[r];
        const double vp = clip0(vp0 - alpha * (a.shape.w_ep + p0));
        const double vn = clip0(vn0 - alpha * (a.shape.w_ep - p0));
        resid += (2.0 * vp - vp0) - (2.0 * vn - vn0) + wv_k[r];
        const double pn = p0 + beta * resid;
        if (kStore) {
          const int e = kc * kNX + kR * g + r;
          snap[S.vp + e] = vp;
          snap[S.vn + e] = vn;
          snap[S.ph + e] = pn;
        }
        const double pe = extrapolate(p0, pn);
        phe[r] = ival ? pe : 0.0;
        vpe[r] = extrapolate(vp0, vp);
        vne[r] = extrapolate(vn0, vn);
      }
      if (g == 4) {
        const double drift = xr_k[kXS + 14] - v[14] - eps_k[0];
        const double tn = clip0(the + beta * drift);
        if (kStore) snap[S.th + kc] = tn;
        the = ival ? extrapolate(the, tn) : 0.0;
      }
      publish_duals(phe, the);
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
    iter_no = j;
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
          z_cur = max_nn(z_cur, fabs(c));
          z_prev = max_nn(z_prev, fabs(o));
          z_del = max_nn(z_del, fabs(c - o));
          if (finite_checked && !pt_finite(c)) bad = 1.0;
        }
      };
      auto dual = [&](int off, int count, bool finite_checked) {
        for (int e = tid; e < count; e += T) {
          const double c = cur[off + e], o = prev[off + e];
          r_cur = max_nn(r_cur, fabs(c));
          r_prev = max_nn(r_prev, fabs(o));
          r_del = max_nn(r_del, fabs(c - o));
          if (finite_checked && !pt_finite(c)) bad = 1.0;
        }
      };
      primal(S.x, NXn, true);
      primal(S.u, NUn, true);
      primal(S.vp, NM, false);
      primal(S.vn, NM, false);
      dual(S.ph, NM, true);
      dual(S.th, mloc, false);
      z_cur = warp_max_nn(z_cur); z_prev = warp_max_nn(z_prev); z_del = warp_max_nn(z_del);
      r_cur = warp_max_nn(r_cur); r_prev = warp_max_nn(r_prev); r_del = warp_max_nn(r_del);
      bad = warp_max_nn(bad);
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
        for (int w = 0; w < kFastWarps; ++w) mx = max_nn(mx, w < nwarps ? red[w * 8 + q] : 0.0);
        v[q] = mx;
      }
      if constexpr (kCluster) {  // combine with the partner's maxima
        if (tid == 0) {
          double* rv = in_cta(red + kFastWarps * 8, cut.rank ^ 1);
#pragma unroll
          for (int q = 0; q < 7; ++q) rv[q] = v[q];
        }
        cg::this_cluster().sync();
#pragma unroll
        for (int q = 0; q < 7; ++q) v[q] = max_nn(v[q], red[kFastWarps * 8 + q]);
        cg::this_cluster().sync();  // red and the snapshots are rewritten later
      } else {
        __syncthreads();  // red and the snapshots are rewritten later
      }
      if (v[6] > 0.0) {
        diverged = true;
        break;
      }
      if (v[2] <= a.eps_abs + a.eps_rel * max_nn(v[0], v[1]) &&
          v[5] <= a.eps_abs + a.eps_rel * max_nn(v[3], v[4])) {
        converged = true;
        break;
      }
    }
  }

  if constexpr (kCluster) bx.recv_prev(iters);  // what rank 0 sent after the last iteration
  if (diverged) {  // SolverDiverged(j): the workspace is left untouched, pipg.hpp:478
    if (tid == 0 && cut.rank == 0) {
      if (a.status) a.status[b] = kStSolverDiverged;
      if (a.fail_index) a.fail_index[b] = iters;
      if (a.iterations) a.iterations[b] = iters;
      if (a.converged) a.converged[b] = 0;
      if (a.active) a.active[b] = 0;
    }
    if constexpr (kCluster) cg::this_cluster().sync();  // nobody leaves while the partner reads
    return;
  }
  // solution = the *_cur groups, pipg.hpp:490-495 (all threads passed a barrier after the last
  // snapshot write)
  const double* cur = snap0 + cur_set * S.total;
  for (int e = tid; e < NXn; e += T) a.ws.x[gx + e] = cur[S.x + e];
  for (int e = tid; e < NUn; e += T) a.ws.u[gu + e] = cur[S.u + e];
  for (int e = tid; e < NM; e += T) {
    a.ws.vc_pos[gm + e] = cur[S.vp + e];
    a.ws.vc_neg[gm + e] = cur[S.vn + e];
    a.ws.dyn_dual[gm + e] = cur[S.ph + e];
  }
  for (int e = tid; e < mloc; e += T) a.ws.relax_dual[gt + e] = cur[S.th + e];
  if (tid == 0 && cut.rank == 0) {
    if (a.iterations) a.iterations[b] = iters;
    if (a.converged) a.converged[b] = converged ? 1 : 0;
  }
  if constexpr (kCluster) cg::this_cluster().sync();  // nobody leaves while the partner reads
}

}  // namespace

bool solver_fast_supports(const SubShape& s, bool has_a_plus) {
  if (has_a_plus || s.nx != kNX || s.nu != kNU) return false;
  if (s.n < 2 || s.n > 2 * kFastMaxNodes) return false;
  for (int i = 0; i < kNX; ++i)
    if (s.e_y[i] != (i == kNX - 1 ? 1.0 : 0.0)) return false;
  return true;
}

bool solver_fast_can_split(const SubShape& s) { return s.n >= 4 && s.n <= 2 * kSplitMaxNodes; }

namespace {

constexpr size_t kPowerSmemFull = sizeof(double) * (size_t)fast_layout<kFastMaxNodes>(false).total;
constexpr size_t kPipgSmemFull = sizeof(double) * (size_t)fast_layout<kFastMaxNodes>(true).total;
constexpr size_t kPowerSmemSplit = sizeof(double) * (size_t)fast_layout<kSplitMaxNodes>(false).total;
constexpr size_t kPipgSmemSplit = sizeof(double) * (size_t)fast_layout<kSplitMaxNodes>(true).total;
// two co-resident CTAs: 228 KB per SM minus 1 KB reserved per CTA
static_assert(kPipgSmemSplit <= 113 * 1024, "two split CTAs must fit one SM");

bool use_split(const SubShape& s, bool split) { return split && solver_fast_can_split(s); }

/// One CTA per instance up to kFastMaxNodes nodes, a cluster of two above or when split.
bool needs_cluster(const SubShape& s, bool split) { return s.n > kFastMaxNodes || use_split(s, split); }

/// Just enough warps for five threads per (local) node; the kernels size their loops by blockDim.
int fast_threads(const SubShape& s, bool split) {
  const int nodes = needs_cluster(s, split) ? (s.n + 1) / 2 : s.n;
  return ((kG * nodes + 31) / 32) * 32;
}

template <class Args>
cudaError_t launch_fast(void (*single)(Args), void (*paired)(Args), void (*halves)(Args), const Args& a,
                        bool split, size_t smem, cudaStream_t stream) {
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3((unsigned)fast_threads(a.shape, split));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr{};
  if (needs_cluster(a.shape, split)) {
    cfg.gridDim = dim3(2u * (unsigned)a.batch);
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 2;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, use_split(a.shape, split) ? halves : paired, a);
  }
  cfg.gridDim = dim3((unsigned)a.batch);
  return cudaLaunchKernelEx(&cfg, single, a);
}

}  // namespace

size_t power_fast_smem(const SubShape& s, bool split) { return use_split(s, split) ? kPowerSmemSplit : kPowerSmemFull; }
size_t pipg_fast_smem(const SubShape& s, bool split) { return use_split(s, split) ? kPipgSmemSplit : kPipgSmemFull; }

cudaError_t configure_solver_fast(const SubShape&) {
  const auto opt_in = [](auto kernel, size_t bytes) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    // two split CTAs per SM need the largest shared-memory carveout
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e == cudaSuccess && getenv("PTOPT_DEBUG_OCCUPANCY")) {
      int blocks = -1;
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, kernel);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, 128, bytes);
      fprintf(stderr, "[ptopt] kernel regs=%d smem=%zu maxThreads=%d -> %d CTAs of 128 threads per SM\n",
              fa.numRegs, bytes, fa.maxThreadsPerBlock, blocks);
    }
    return e;
  };
  cudaError_t e = opt_in(power_fast_kernel<false, kFastMaxNodes>, kPowerSmemFull);
  if (e == cudaSuccess) e = opt_in(power_fast_kernel<true, kFastMaxNodes>, kPowerSmemFull);
  if (e == cudaSuccess) e = opt_in(power_fast_kernel<true, kSplitMaxNodes>, kPowerSmemSplit);
  if (e == cudaSuccess) e = opt_in(pipg_fast_kernel<false, kFastMaxNodes>, kPipgSmemFull);
  if (e == cudaSuccess) e = opt_in(pipg_fast_kernel<true, kFastMaxNodes>, kPipgSmemFull);
  if (e == cudaSuccess) e = opt_in(pipg_fast_kernel<true, kSplitMaxNodes>, kPipgSmemSplit);
  return e;
}

cudaError_t launch_power_fast(const PowerArgs& a, bool split, cudaStream_t stream) {
  return launch_fast<PowerArgs>(power_fast_kernel<false, kFastMaxNodes>, power_fast_kernel<true, kFastMaxNodes>,
                                power_fast_kernel<true, kSplitMaxNodes>, a, split,
                                power_fast_smem(a.shape, split), stream);
}

cudaError_t launch_pipg_fast(const PipgArgs& a, bool split, cudaStream_t stream) {
  return launch_fast<PipgArgs>(pipg_fast_kernel<false, kFastMaxNodes>, pipg_fast_kernel<true, kFastMaxNodes>,
                               pipg_fast_kernel<true, kSplitMaxNodes>, a, split,
                               pipg_fast_smem(a.shape, split), stream);
}

}  // namespace ptopt_b200
