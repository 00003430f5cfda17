// solver_lat.cu — latency mode of the power iteration and the customized PIPG for the rocket-shaped
// subproblem (n_x = 15, n_u = 7, A_plus = -I, e_y = unit vector of the last state): ONE instance
// spread over a thread-block cluster of up to eight CTAs, SIXTEEN threads per node.
//
// Why another mapping.  The throughput kernels (solver_fast.cu) give a node five threads with
// three operator rows each; one iteration is a dependent stream of ~550 instructions per warp and
// takes ~3 200 clk however few warps run (a lone instance uses one SM for ~215 ms at N = 50, and
// splitting it over two CTAs with the same mapping is slower still: the stream does not get
// shorter, the hand-off is added).  Latency needs a short per-thread stream instead:
//   * thread (rg, cq) of a node owns a 4 x 8 tile of the packed interval block [A- | B- | B+]
//     (rows 4rg..4rg+3; column segment cq: A- 0..7 | A- 8..14 | B- | B+): 32 operator doubles,
//     32 FMAs per product;
//   * forward product: the four partial row sums are reduce-scattered over the four cq lanes with
//     two shuffle hops, so lane cq ends up with dual row 4rg + cq complete and updates that row
//     alone (lane (3,3) owns the relaxation dual instead); the new duals are all-gathered back
//     with two hops;
//   * transposed product: eight partial column sums over the tile's rows, reduce-scattered over
//     the four rg lanes (two hops): every thread ends up owning two primal entries;
//   * register sets are rotated by the lane index (slot t <-> row 4rg + (cq ^ t), set s <-> column
//     pair rg ^ s), so every shuffle round sends a compile-time register — no selects;
//   * only neighbour-node coupling goes through shared memory (x_{k+1}, u_{k+1}, phi_{k-1},
//     B+^T phi_{k-1}), and across a CTA boundary through the mailboxes of mailbox.cuh.
// About 200 instructions per thread and iteration; the instance's FP64 work is spread over
// C SMs.
//
// Follows /root/reference/proj/include/ptopt/pipg.hpp:206-292 (power_iteration_custom), :307-326
// (stopping_custom), :335-340 (step_sizes), :350-497 (pipg_custom); per-entry arithmetic as in
// solver_fast.cu.  Row and column sums are added in butterfly order (rounding-only change).
#include <cooperative_groups.h>

#include "kernels.cuh"
#include "mailbox.cuh"

namespace ptopt_b200 {

namespace cg = cooperative_groups;

namespace {

constexpr int kLanes = 16;                    // threads per node
constexpr int kLatThreadsMax = kLanes * kLatMaxLocalNodes;
constexpr int kLatWarpsMax = kLatThreadsMax / 32;
constexpr int kSlots = kLatMaxLocalNodes + 3;  // node slots -1 .. kLatMaxLocalNodes + 1
constexpr int kXP = 16, kUP = 8;               // node pitch of the x / u arrays (entry 15 / 7 is a zero pad)

/// std::max(0.0, v) as the reference evaluates it (pipg.hpp:423-430).
__device__ __forceinline__ double clip0(double v) { return 0.0 < v ? v : 0.0; }

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
__device__ __forceinline__ double xor_get(double v, int mask) { return __shfl_xor_sync(0xffffffffu, v, mask); }

// Shared memory of one CTA.  Node arrays carry slot -1 in front (previous node: the zero guard of
// rank 0, or the last node of the previous rank, pushed by it) and two slots behind the local nodes
// (slot nloc: first node of the next rank, pushed by it; then scratch for the idle threads).
// `us` starts 4 doubles past a 16-double boundary: with that offset the four LDS.128 of a quarter
// warp (two row groups x four column segments) fall into eight different bank groups.
struct __align__(128) LatSmem {
  double xs[kSlots * kXP];       // primal x (power) / reflections (PIPG), [slot][16]
  double pad_[4];
  double us[kSlots * kUP + 4];   // [slot][8]
  double php[kSlots * kXP];      // dual rows of interval k: [0..14] dynamics dual, [15] relaxation dual
  double bps[kSlots * kUP];      // B+_k^T phi_k: the share of node k+1's control gradient
  double shares[kLatMaxRanks * 2 * kLatWarpsMax];  // power: norm shares [rank][parity][warp]
  double red[kLatWarpsMax * 8];  // PIPG stopping test: per-warp maxima
  double redc[kLatMaxRanks * 8];  //   ... and every rank's CTA maxima
  unsigned long long box[4];     // mailboxes: prev, next, norm (by trip parity)
};
enum { kBoxPrev = 0, kBoxNext = 1, kBoxNorm = 2 };
constexpr int kPrevBytes = 8 * (kXP + kUP);  // php row of the last node + its bps row
constexpr int kNextBytes = 8 * (kXP + kUP);  // xs row + us row of the first node

struct Cut {
  int ranks, rank, node0, nloc, nloc_prev;
  bool has_prev, has_next;
};

__device__ __forceinline__ Cut make_cut(int n) {
  Cut c;
  c.ranks = (int)cg::this_cluster().num_blocks();
  c.rank = (int)cg::this_cluster().block_rank();
  const int base = n / c.ranks, extra = n - base * c.ranks;
  c.nloc = base + (c.rank < extra ? 1 : 0);
  c.node0 = c.rank * base + min(c.rank, extra);
  c.nloc_prev = base + (c.rank - 1 < extra ? 1 : 0);
  c.has_prev = c.rank > 0;
  c.has_next = c.rank + 1 < c.ranks;
  return c;
}

/// Per-thread geometry shared by the two kernels.
struct Lane {
  int tid, lane, warp, nwarps;
  int p, pc, rg, cq;     // local node, its slot (idle threads: a scratch slot), row group, column segment
  int kg;                // global node
  bool node, ival;       // p is a node of this CTA / it has an interval behind it
  int row;               // dual row owned: 4rg + cq (15: the relaxation dual)
  bool row_alive, theta_lane;
  int c0;                // first of the two column entries owned inside the segment: 2rg
  bool push_prev, push_next;  // this thread's node is the CTA's last (feeds rank+1) / first (feeds rank-1)
  bool prev_warp, next_warp, prev_armer, next_armer;
};

__device__ __forceinline__ Lane make_lane(const Cut& cut, int m) {
  Lane t;
  t.tid = threadIdx.x;
  t.lane = t.tid & 31;
  t.warp = t.tid >> 5;
  t.nwarps = blockDim.x >> 5;
  t.p = t.tid >> 4;
  const int l = t.tid & 15;
  t.rg = l >> 2;
  t.cq = l & 3;
  t.node = t.p < cut.nloc;
  t.pc = t.node ? t.p : t.p + 1;  // slot nloc belongs to the next rank's first node
  t.kg = cut.node0 + t.p;
  t.ival = t.node && t.kg < m;
  t.row = 4 * t.rg + t.cq;
  t.row_alive = t.ival && t.row < kNX;
  t.theta_lane = t.row == kNX;
  t.c0 = 2 * t.rg;
  t.push_prev = cut.has_next && t.p == cut.nloc - 1;
  t.push_next = cut.has_prev && t.p == 0;
  t.prev_warp = cut.has_prev && t.warp == 0;
  t.next_warp = cut.has_next && t.warp == ((cut.nloc - 1) >> 1);
  t.prev_armer = cut.has_prev && t.tid == 0;
  t.next_armer = cut.has_next && t.tid == kLanes * (cut.nloc - 1);
  return t;
}

/// Loads the thread's 4 x 8 tile: a[t][s][e] = entry (row 4rg + (cq ^ t), column pair rg ^ s, e) of
/// its segment; rows >= 15 and the pad column of a segment are zero.
__device__ __forceinline__ void load_tile(const SubArrays& sp, size_t iv, const Lane& t, double (&a)[4][4][2]) {
#pragma unroll
  for (int tt = 0; tt < 4; ++tt) {
    const int i = 4 * t.rg + (t.cq ^ tt);
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 2 * (t.rg ^ s) + e;  // 0..7 inside the segment
        double v = 0.0;
        if (t.ival && i < kNX) {
          if (t.cq == 0) v = __ldg(sp.A_minus + (iv * kNX + i) * kNX + c);
          else if (t.cq == 1) v = c < 7 ? __ldg(sp.A_minus + (iv * kNX + i) * kNX + 8 + c) : 0.0;
          else if (t.cq == 2) v = c < 7 ? __ldg(sp.B_minus + (iv * kNX + i) * kNU + c) : 0.0;
          else v = c < 7 ? __ldg(sp.B_plus + (iv * kNX + i) * kNU + c) : 0.0;
        }
        a[tt][s][e] = v;
      }
  }
}

/// Forward product of the tile with its segment of the node vector, reduce-scattered over the four
/// cq lanes: returns dual row 4rg + cq of  A- x_k + B- u_k + B+ u_{k+1}.
__device__ __forceinline__ double forward_row(const double (&a)[4][4][2], const double* seg, int rg) {
  double v[4][2];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const double2 q = *reinterpret_cast<const double2*>(seg + 2 * (rg ^ s));
    v[s][0] = q.x;
    v[s][1] = q.y;
  }
  double r[4];
#pragma unroll
  for (int tt = 0; tt < 4; ++tt) {
    double lo = a[tt][0][0] * v[0][0], hi = a[tt][2][0] * v[2][0];
    lo = fma(a[tt][0][1], v[0][1], lo);
    hi = fma(a[tt][2][1], v[2][1], hi);
    lo = fma(a[tt][1][0], v[1][0], lo);
    hi = fma(a[tt][3][0], v[3][0], hi);
    lo = fma(a[tt][1][1], v[1][1], lo);
    hi = fma(a[tt][3][1], v[3][1], hi);
    r[tt] = lo + hi;
  }
  // slot t holds row (cq ^ t): the partner across bit 1 owns what I keep in slots 2, 3, ...
  r[0] += xor_get(r[2], 2);
  r[1] += xor_get(r[3], 2);
  r[0] += xor_get(r[1], 1);
  return r[0];
}

/// All-gather of the four cq lanes' dual values into rotated slots (slot t <-> row 4rg + (cq ^ t)).
__device__ __forceinline__ void gather_rows(double mine, double (&d)[4]) {
  d[0] = mine;
  d[1] = xor_get(mine, 1);
  d[2] = xor_get(d[0], 2);
  d[3] = xor_get(d[1], 2);
}

/// The gathered slot of "row 15" (row group 3) carries the relaxation dual, which is not a row of
/// the operator: zero it so that a non-finite value cannot leak through the zero tile entries.
__device__ __forceinline__ void drop_theta_slot(const Lane& t, double (&d)[4]) {
#pragma unroll
  for (int tt = 0; tt < 4; ++tt) d[tt] = (t.rg == 3 && (t.cq ^ tt) == 3) ? 0.0 : d[tt];
}

/// Transposed product of the tile with the gathered duals, reduce-scattered over the four rg lanes:
/// returns the two column sums (pair rg of the segment) this thread owns.
__device__ __forceinline__ void transposed_pair(const double (&a)[4][4][2], const double (&d)[4], double (&cs)[2]) {
  double q[4][2];
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double lo = a[0][s][e] * d[0], hi = a[2][s][e] * d[2];
      lo = fma(a[1][s][e], d[1], lo);
      hi = fma(a[3][s][e], d[3], hi);
      q[s][e] = lo + hi;
    }
  // rg sits in lane bits 2, 3
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    q[0][e] += xor_get(q[2][e], 8);
    q[1][e] += xor_get(q[3][e], 8);
    q[0][e] += xor_get(q[1][e], 4);
    cs[e] = q[0][e];
  }
}

struct Boxes {
  unsigned long long* local;
  unsigned to_next_prevbox, to_prev_nextbox;  // the neighbours' mailboxes this CTA sends to
};

/// Mailboxes: cleared shared memory first, then the barriers, then a cluster barrier so that every
/// CTA is running, cleared and initialised before any remote store.
__device__ __forceinline__ Boxes open_boxes(LatSmem* S, const Cut& cut, int tid) {
  for (int e = tid; e < (int)(sizeof(LatSmem) / sizeof(double)); e += blockDim.x)
    reinterpret_cast<double*>(S)[e] = 0.0;
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) mbar_init(S->box + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cg::this_cluster().sync();
  Boxes bx;
  bx.local = S->box;
  bx.to_next_prevbox = cut.has_next ? partner_u32(S->box + kBoxPrev, cut.rank + 1) : 0u;
  bx.to_prev_nextbox = cut.has_prev ? partner_u32(S->box + kBoxNext, cut.rank - 1) : 0u;
  return bx;
}

__device__ __forceinline__ void receive(const Boxes& bx, int which, bool mine, bool armer, int bytes, int phase) {
  if (!mine) return;
  if (armer) mbar_expect(bx.local + which, bytes);
  mbar_wait(bx.local + which, phase);
}

/// Publishes the duals of this thread's row (php) and — cq 3 — the B+ column sums (bps) in the
/// node's slot; the CTA's last node sends the same values into slot -1 of the next rank.
__device__ __forceinline__ void publish_duals(LatSmem* S, const Lane& t, const Cut& cut, const Boxes& bx, double d,
                                              const double (&cs)[2]) {
  S->php[(t.pc + 1) * kXP + t.row] = d;
  if (t.cq == 3) *reinterpret_cast<double2*>(S->bps + (t.pc + 1) * kUP + t.c0) = make_double2(cs[0], cs[1]);
  if (t.push_prev) {
    push_f64(partner_u32(S->php + t.row, cut.rank + 1), d, bx.to_next_prevbox);
    if (t.cq == 3) {
      const unsigned r = partner_u32(S->bps + t.c0, cut.rank + 1);
      push_f64(r, cs[0], bx.to_next_prevbox);
      push_f64(r + 8u, cs[1], bx.to_next_prevbox);
    }
  }
}

/// Stores the two primal entries (cq 0, 1: x; cq 2: u) into the node's slot; the CTA's first node
/// sends them into slot nloc of the previous rank as well.
__device__ __forceinline__ void publish_primal(LatSmem* S, const Lane& t, const Cut& cut, const Boxes& bx, double v0,
                                               double v1) {
  if (t.cq == 3) return;
  double* dst = t.cq == 2 ? S->us + (t.pc + 1) * kUP + t.c0 : S->xs + (t.pc + 1) * kXP + 8 * t.cq + t.c0;
  *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
  if (t.push_next) {
    const double* slot = t.cq == 2 ? S->us + (cut.nloc_prev + 1) * kUP + t.c0
                                   : S->xs + (cut.nloc_prev + 1) * kXP + 8 * t.cq + t.c0;
    const unsigned r = partner_u32(slot, cut.rank - 1);
    push_f64(r, v0, bx.to_prev_nextbox);
    push_f64(r + 8u, v1, bx.to_prev_nextbox);
  }
}

// ---------------------------------------------------------------------------------------------
// power iteration (pipg.hpp:206-292)
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kLatThreadsMax, 1) power_lat_kernel(PowerArgs a) {
  __shared__ LatSmem Sm;
  LatSmem* S = &Sm;
  const Cut cut = make_cut(a.shape.n);
  const int b = blockIdx.x / cut.ranks;
  if (a.active && !a.active[b]) return;  // every CTA of the cluster leaves together
  const int n = a.shape.n, m = n - 1;
  const Lane t = make_lane(cut, m);
  const Boxes bx = open_boxes(S, cut, t.tid);
  const double* seg = t.cq == 0   ? S->xs + (t.pc + 1) * kXP
                      : t.cq == 1 ? S->xs + (t.pc + 1) * kXP + 8
                      : t.cq == 2 ? S->us + (t.pc + 1) * kUP
                                  : S->us + (t.pc + 2) * kUP;
  const int rsel = t.theta_lane ? kNX - 1 : t.row;        // x entry this row owner reads from nodes k, k+1
  const double* x_next = S->xs + (t.pc + 2) * kXP + rsel;
  const double* x_cur = S->xs + (t.pc + 1) * kXP + rsel;
  // neighbour terms of the owned primal pair: x: phi_{k-1} (and theta_{k-1} behind row 14); u: B+^T phi_{k-1}
  const double* nb_ptr = t.cq == 2 ? S->bps + t.pc * kUP + t.c0 : S->php + t.pc * kXP + 8 * (t.cq & 1) + t.c0;
  const bool u_owner = t.cq == 2;
  const bool is14 = t.cq == 1 && t.rg == 3;  // entry 0 of this pair is x[14], entry 1 the pad
  const bool alive0 = t.node && t.cq < 3, alive1 = alive0 && t.rg < 3 + (t.cq == 0);
  const int unorm = 8 * t.nwarps * (cut.ranks - 1);  // bytes of the other ranks' norm shares per trip

  double aop[4][4][2];
  load_tile(a.sp, (size_t)b * m + (t.ival ? t.kg : 0), t, aop);

  // seed (pipg.hpp:213-230): x, u, vc+, vc-; sigma0 = ||seed||_2
  double acc = 0.0;
  {
    double v0 = 0.0, v1 = 0.0;
    if (alive0) {
      const double* src = u_owner ? a.seed_u + ((size_t)b * n + t.kg) * kNU + t.c0
                                  : a.seed_x + ((size_t)b * n + t.kg) * kNX + 8 * t.cq + t.c0;
      v0 = src[0];
      if (alive1) v1 = src[1];
    }
    publish_primal(S, t, cut, bx, v0, v1);  // the first node also reaches the previous rank: "next" phase 0
    acc = v0 * v0 + v1 * v1;
  }
  double vcd = 0.0;  // vc+ - vc-: the only combination of the two groups the forward map uses
  if (t.row_alive) {
    const double vp = a.seed_vcp[((size_t)b * m + t.kg) * kNX + t.row], vn = a.seed_vcn[((size_t)b * m + t.kg) * kNX + t.row];
    vcd = vp - vn;
    acc += vp * vp;
    acc += vn * vn;
  }
  auto send_share = [&](double share, int trip) {  // own slot, and the same slot in every other rank
    const int at = (cut.rank * 2 + (trip & 1)) * kLatWarpsMax + t.warp;
    S->shares[at] = share;
    for (int r = 0; r < cut.ranks; ++r)
      if (r != cut.rank)
        push_f64(partner_u32(S->shares + at, r), share, partner_u32(S->box + kBoxNorm + (trip & 1), r));
  };
  // two norm mailboxes by trip parity: a rank may run up to one trip ahead of another (see solver_fast.cu)
  auto recv_norm = [&](int trip) {
    if (cut.ranks > 1) receive(bx, kBoxNorm + (trip & 1), true, t.tid == 0, unorm, trip >> 1);
  };
  auto norm_sq = [&](int parity) {  // every rank adds the shares in the same order
    double s = 0.0;
    for (int r = 0; r < cut.ranks; ++r) {
      const double* sh = S->shares + (r * 2 + parity) * kLatWarpsMax;
      double sr = 0.0;
      for (int w = 0; w < t.nwarps; ++w) sr += sh[w];
      s += sr;
    }
    return s;
  };
  acc = warp_sum(acc);
  if (t.lane == 0) send_share(acc, 0);
  __syncthreads();
  recv_norm(0);
  double sigma = norm_sq(0);
  if (sigma == 0.0) {  // pipg.hpp:224-225
    if (t.tid == 0 && cut.rank == 0) {
      if (a.status) a.status[b] = kStSeedZero;
      a.sigma[b] = 0.0;
      if (a.trips) a.trips[(size_t)b * a.trips_stride + (a.trips_slot ? a.trips_slot[b] : 0)] = 0;
    }
    if (cut.has_next) receive(bx, kBoxNext, t.next_warp, t.next_armer, kNextBytes, 0);
    cg::this_cluster().sync();
    return;
  }
  double inv = rsqrt(sigma);
  sigma = sqrt(sigma);

  int trips = 0;
  bool done = false;
  for (int j = 1; j <= a.j_max; ++j) {
    // ---- forward map (pipg.hpp:234-245); the norm of trip j-1 arrives while the products run
    receive(bx, kBoxNext, t.next_warp, t.next_armer, kNextBytes, j - 1);  // the next rank's first node of trip j-1
    const double r = forward_row(aop, seg, t.rg);
    const double s = (r - x_next[0]) + vcd;
    const double dy = x_next[0] - x_cur[0];
    if (j > 1) {  // stopping test of trip j-1 (pipg.hpp:277-289)
      recv_norm(j - 1);
      const double ss = norm_sq((j - 1) & 1);
      const double sigma_star = sqrt(ss);
      inv = rsqrt(ss);
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
    const double phi = t.row_alive ? s * inv : 0.0;
    const double mine = t.theta_lane ? (t.ival ? dy * inv : 0.0) : phi;
    double d[4], cs[2];
    gather_rows(mine, d);
    drop_theta_slot(t, d);
    transposed_pair(aop, d, cs);
    publish_duals(S, t, cut, bx, mine, cs);
    vcd = 2.0 * phi;  // vc+ = phi, vc- = -phi (pipg.hpp:268-279)
    const double acc_d = vcd * phi;
    __syncthreads();
    // ---- adjoint map (pipg.hpp:247-275)
    receive(bx, kBoxPrev, t.prev_warp, t.prev_armer, kPrevBytes, j - 1);  // the previous rank's last interval
    const double2 nb = *reinterpret_cast<const double2*>(nb_ptr);
    double v0, v1;
    if (u_owner) {
      v0 = cs[0] + nb.x;
      v1 = cs[1] + nb.y;
    } else {
      v0 = cs[0] + -nb.x;
      v1 = cs[1] + -nb.y;
      if (is14) {  // -theta_k + theta_{k-1} on the last state (e_y)
        v0 += -S->php[(t.pc + 1) * kXP + kNX];
        v0 += nb.y;
      }
    }
    v0 = alive0 ? v0 : 0.0;
    v1 = alive1 ? v1 : 0.0;
    publish_primal(S, t, cut, bx, v0, v1);
    acc = fma(v0, v0, v1 * v1) + acc_d;
    acc = warp_sum(acc);
    if (t.lane == 0) send_share(acc, j);
    __syncthreads();
  }
  if (!done) {  // j_max trips without meeting the tolerance
    if (a.j_max >= 1) recv_norm(a.j_max);
    sigma = sqrt(norm_sq(a.j_max & 1));
  }
  // what the neighbours sent last is still on its way
  if (done) {
    // the loop was left after `receive next (trips)` but before `receive prev (trips)`: nothing pending
  } else if (a.j_max >= 1) {
    receive(bx, kBoxNext, t.next_warp, t.next_armer, kNextBytes, a.j_max);
  }
  if (t.tid == 0 && cut.rank == 0) {
    a.sigma[b] = (1.0 + a.eps_buff) * sigma;
    if (a.trips) a.trips[(size_t)b * a.trips_stride + (a.trips_slot ? a.trips_slot[b] : 0)] = trips;
  }
  cg::this_cluster().sync();  // nobody leaves while a neighbour may still write into it
}

// ---------------------------------------------------------------------------------------------
// customized PIPG (pipg.hpp:350-497)
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kLatThreadsMax, 1) pipg_lat_kernel(PipgArgs a) {
  __shared__ LatSmem Sm;
  LatSmem* S = &Sm;
  const Cut cut = make_cut(a.shape.n);
  const int b = blockIdx.x / cut.ranks;
  if (a.active && !a.active[b]) return;  // every CTA of the cluster leaves together
  const int n = a.shape.n, m = n - 1;
  const Lane t = make_lane(cut, m);
  const Boxes bx = open_boxes(S, cut, t.tid);
  const double* seg = t.cq == 0   ? S->xs + (t.pc + 1) * kXP
                      : t.cq == 1 ? S->xs + (t.pc + 1) * kXP + 8
                      : t.cq == 2 ? S->us + (t.pc + 1) * kUP
                                  : S->us + (t.pc + 2) * kUP;
  const int rsel = t.theta_lane ? kNX - 1 : t.row;
  const double* x_next = S->xs + (t.pc + 2) * kXP + rsel;
  const double* x_cur = S->xs + (t.pc + 1) * kXP + rsel;
  const double* nb_ptr = t.cq == 2 ? S->bps + t.pc * kUP + t.c0 : S->php + t.pc * kXP + 8 * (t.cq & 1) + t.c0;
  const bool u_owner = t.cq == 2;
  const bool is14 = t.cq == 1 && t.rg == 3;
  const bool alive0 = t.node && t.cq < 3, alive1 = alive0 && t.rg < 3 + (t.cq == 0);
  const bool last_node = t.node && t.kg == n - 1;

  double aop[4][4][2];
  load_tile(a.sp, (size_t)b * m + (t.ival ? t.kg : 0), t, aop);

  // ---- per-entry constants and the warm start (pipg.hpp:362-374): ex = cur = workspace
  // primal pair: entry index inside x / u, proximal-term extras, box or boundary value
  const int ce = u_owner ? t.c0 : 8 * t.cq + t.c0;
  double pe[2] = {0.0, 0.0}, lo[2], hi[2], fv[2] = {0.0, 0.0}, cost[2] = {0.0, 0.0};
  bool fixed[2] = {false, false};
  lo[0] = lo[1] = -INFINITY;
  hi[0] = hi[1] = INFINITY;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const bool alive = e == 0 ? alive0 : alive1;
    if (!alive) continue;
    if (u_owner) {
      const size_t g = ((size_t)b * n + t.kg) * kNU + ce + e;
      pe[e] = a.ws.u[g];
      lo[e] = a.sp.u_min[g];  // pipg.hpp:418-419
      hi[e] = a.sp.u_max[g];
    } else {
      pe[e] = a.ws.x[((size_t)b * n + t.kg) * kNX + ce + e];
      if (last_node) cost[e] = a.shape.w_cost * a.shape.e_cost[ce + e];
      // boundary rows (pipg.hpp:408-413); later entries override earlier ones, as the assignment loops do
      if (t.kg == 0)
        for (int i = 0; i < a.shape.n_init_fix; ++i)
          if (a.shape.init_fix_idx[i] == ce + e) {
            fixed[e] = true;
            fv[e] = a.sp.init_fix_val[(size_t)b * a.shape.n_init_fix + i];
          }
      if (last_node)
        for (int i = 0; i < a.shape.n_final_fix; ++i)
          if (a.shape.final_fix_idx[i] == ce + e) {
            fixed[e] = true;
            fv[e] = a.sp.final_fix_val[(size_t)b * a.shape.n_final_fix + i];
          }
    }
  }
  // dual row: dynamics dual + the two slack groups, or (lane (3,3)) the relaxation dual
  double phe = 0.0, vpe = 0.0, vne = 0.0, wrow = 0.0;
  if (t.row_alive) {
    const size_t g = ((size_t)b * m + t.kg) * kNX + t.row;
    phe = a.ws.dyn_dual[g];
    vpe = a.ws.vc_pos[g];
    vne = a.ws.vc_neg[g];
    wrow = a.sp.w[g];
  } else if (t.theta_lane && t.ival) {
    phe = a.ws.relax_dual[(size_t)b * m + t.kg];
    wrow = a.sp.eps_relax[(size_t)b * m + t.kg];
  }
  // materialised *_cur values of the last two iterations (pipg.hpp:490-495 returns the current ones)
  double cur_p[2] = {pe[0], pe[1]}, cur_d = phe, cur_vp = vpe, cur_vn = vne;
  double prv_p[2] = {pe[0], pe[1]}, prv_d = phe, prv_vp = vpe, prv_vn = vne;

  const double sigma = a.sigma[b];
  const double alpha = 2.0 / (a.shape.w_prox + sqrt(a.shape.w_prox * a.shape.w_prox + 4.0 * a.omega * sigma));
  const double beta = a.omega * alpha;
  auto extrapolate = [&](double ex, double cur) { return fma(a.rho, cur - ex, ex); };  // pipg.hpp:461-472

  double cs[2];
  {  // partial sums of H^T phi_ex of the warm start, for the first primal step
    double d[4];
    gather_rows(phe, d);
    drop_theta_slot(t, d);
    transposed_pair(aop, d, cs);
    publish_duals(S, t, cut, bx, phe, cs);
  }
  __syncthreads();

  int iters = 0;
  bool converged = false, diverged = false;
  int to_check = a.j_check;
  for (int j = 1; j <= a.j_max; ++j) {
    --to_check;
    const bool check = to_check == 0;
    if (check) to_check = a.j_check;
    // ---- primal projected-gradient step (pipg.hpp:388-420) by the owner of each entry
    receive(bx, kBoxPrev, t.prev_warp, t.prev_armer, kPrevBytes, j - 1);  // previous rank, after iteration j-1
    {
      const double2 nb = *reinterpret_cast<const double2*>(nb_ptr);
      const double nbv[2] = {nb.x, nb.y};
      double rf[2];
      prv_p[0] = cur_p[0];
      prv_p[1] = cur_p[1];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double x0 = pe[e];
        double xn;
        if (u_owner) {
          const double grad = x0 * a.shape.w_prox + (cs[e] + nbv[e]);
          xn = x0 + -alpha * grad;
          const double cl = (hi[e] < xn) ? hi[e] : xn;  // std::max(lo, std::min(hi, v))
          xn = (lo[e] < cl) ? cl : lo[e];
        } else {
          double base = x0 * a.shape.w_prox;
          base += cost[e];
          base += -nbv[e];
          if (e == 0 && is14) base += nb.y - S->php[(t.pc + 1) * kXP + kNX];
          const double grad = base + cs[e];
          xn = x0 + -alpha * grad;
          xn = fixed[e] ? fv[e] : xn;
        }
        const bool alive = e == 0 ? alive0 : alive1;
        xn = alive ? xn : 0.0;
        rf[e] = alive ? fma(2.0, xn, -x0) : 0.0;
        cur_p[e] = xn;
        pe[e] = alive ? extrapolate(x0, xn) : 0.0;
      }
      publish_primal(S, t, cut, bx, rf[0], rf[1]);
    }
    __syncthreads();
    receive(bx, kBoxNext, t.next_warp, t.next_armer, kNextBytes, j - 1);  // next rank's first node, this iteration
    // ---- slacks (pipg.hpp:423-430), PI feedback of the constraint violation (:433-458), extrapolation of
    //      the dual groups (:468-472) and the partial sums of H^T phi_ex for the next primal step
    {
      const double r = forward_row(aop, seg, t.rg);
      const double xn1 = x_next[0];
      prv_d = cur_d;
      prv_vp = cur_vp;
      prv_vn = cur_vn;
      if (t.theta_lane) {
        const double drift = xn1 - x_cur[0] - wrow;
        const double tn = clip0(phe + beta * drift);
        cur_d = t.ival ? tn : 0.0;
        phe = t.ival ? extrapolate(phe, tn) : 0.0;
      } else {
        double resid = r + -xn1;
        const double p0 = phe, vp0 = vpe, vn0 = vne;
        const double vp = clip0(vp0 - alpha * (a.shape.w_ep + p0));
        const double vn = clip0(vn0 - alpha * (a.shape.w_ep - p0));
        resid += (2.0 * vp - vp0) - (2.0 * vn - vn0) + wrow;
        const double pn = p0 + beta * resid;
        cur_d = t.row_alive ? pn : 0.0;
        cur_vp = t.row_alive ? vp : 0.0;
        cur_vn = t.row_alive ? vn : 0.0;
        phe = t.row_alive ? extrapolate(p0, pn) : 0.0;
        vpe = t.row_alive ? extrapolate(vp0, vp) : 0.0;
        vne = t.row_alive ? extrapolate(vn0, vn) : 0.0;
      }
      double d[4];
      gather_rows(phe, d);
      drop_theta_slot(t, d);
      transposed_pair(aop, d, cs);
      publish_duals(S, t, cut, bx, phe, cs);
    }
    iters = j;
    __syncthreads();
    if (check) {  // stopping_custom(cur, prev) and the divergence test, pipg.hpp:475-487
      double z_cur = 0.0, z_prev = 0.0, z_del = 0.0, r_cur = 0.0, r_prev = 0.0, r_del = 0.0, bad = 0.0;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        z_cur = fmax(z_cur, fabs(cur_p[e]));
        z_prev = fmax(z_prev, fabs(prv_p[e]));
        z_del = fmax(z_del, fabs(cur_p[e] - prv_p[e]));
        if (!pt_finite(cur_p[e])) bad = 1.0;
      }
      if (!t.theta_lane) {
        z_cur = fmax(z_cur, fmax(fabs(cur_vp), fabs(cur_vn)));
        z_prev = fmax(z_prev, fmax(fabs(prv_vp), fabs(prv_vn)));
        z_del = fmax(z_del, fmax(fabs(cur_vp - prv_vp), fabs(cur_vn - prv_vn)));
        if (!pt_finite(cur_d)) bad = 1.0;
      }
      r_cur = fabs(cur_d);
      r_prev = fabs(prv_d);
      r_del = fabs(cur_d - prv_d);
      double v[7] = {z_cur, z_prev, z_del, r_cur, r_prev, r_del, bad};
#pragma unroll
      for (int q = 0; q < 7; ++q) v[q] = warp_max(v[q]);
      if (t.lane == 0) {
#pragma unroll
        for (int q = 0; q < 7; ++q) S->red[t.warp * 8 + q] = v[q];
      }
      __syncthreads();
      if (t.tid < 7) {  // this CTA's maxima into every rank's table
        double mx = 0.0;
        for (int w = 0; w < t.nwarps; ++w) mx = fmax(mx, S->red[w * 8 + t.tid]);
        for (int r = 0; r < cut.ranks; ++r) *cg::this_cluster().map_shared_rank(S->redc + cut.rank * 8 + t.tid, r) = mx;
      }
      cg::this_cluster().sync();
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        double mx = 0.0;
        for (int r = 0; r < cut.ranks; ++r) mx = fmax(mx, S->redc[r * 8 + q]);
        v[q] = mx;
      }
      cg::this_cluster().sync();  // the tables are rewritten at the next check
      if (v[6] > 0.0) {
        diverged = true;
        break;
      }
      if (v[2] <= a.eps_abs + a.eps_rel * fmax(v[0], v[1]) && v[5] <= a.eps_abs + a.eps_rel * fmax(v[3], v[4])) {
        converged = true;
        break;
      }
    }
  }
  receive(bx, kBoxPrev, t.prev_warp, t.prev_armer, kPrevBytes, iters);  // what the previous rank sent last
  if (diverged) {  // SolverDiverged(j): the workspace is left untouched, pipg.hpp:478
    if (t.tid == 0 && cut.rank == 0) {
      if (a.status) a.status[b] = kStSolverDiverged;
      if (a.fail_index) a.fail_index[b] = iters;
      if (a.iterations) a.iterations[b] = iters;
      if (a.converged) a.converged[b] = 0;
      if (a.active) a.active[b] = 0;
    }
    cg::this_cluster().sync();
    return;
  }
  // solution = the *_cur groups (pipg.hpp:490-495), written by their owners
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const bool alive = e == 0 ? alive0 : alive1;
    if (!alive) continue;
    if (u_owner) a.ws.u[((size_t)b * n + t.kg) * kNU + ce + e] = cur_p[e];
    else a.ws.x[((size_t)b * n + t.kg) * kNX + ce + e] = cur_p[e];
  }
  if (t.row_alive) {
    const size_t g = ((size_t)b * m + t.kg) * kNX + t.row;
    a.ws.dyn_dual[g] = cur_d;
    a.ws.vc_pos[g] = cur_vp;
    a.ws.vc_neg[g] = cur_vn;
  } else if (t.theta_lane && t.ival) {
    a.ws.relax_dual[(size_t)b * m + t.kg] = cur_d;
  }
  if (t.tid == 0 && cut.rank == 0) {
    if (a.iterations) a.iterations[b] = iters;
    if (a.converged) a.converged[b] = converged ? 1 : 0;
  }
  cg::this_cluster().sync();  // nobody leaves while a neighbour may still write into it
}

template <class Args>
cudaError_t launch_lat(void (*kernel)(Args), const Args& a, int ranks, cudaStream_t stream) {
  const int nloc = (a.shape.n + ranks - 1) / ranks;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3((unsigned)((kLanes * nloc + 31) / 32 * 32));
  cfg.gridDim = dim3((unsigned)ranks * (unsigned)a.batch);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = (unsigned)ranks;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, a);
}

}  // namespace

int solver_lat_ranks(const SubShape& s, bool has_a_plus, int batch, int sm_count) {
  if (has_a_plus || s.nx != kNX || s.nu != kNU || s.n < 2) return 0;
  for (int i = 0; i < kNX; ++i)
    if (s.e_y[i] != (i == kNX - 1 ? 1.0 : 0.0)) return 0;
  // the largest cluster that still fits the whole batch on the chip in one wave (batch = 0: any)
  for (int ranks = kLatMaxRanks; ranks >= 2; ranks >>= 1) {
    if (ranks > s.n || (s.n + ranks - 1) / ranks > kLatMaxLocalNodes) continue;
    if (batch > 0 && (long long)batch * ranks > sm_count) continue;
    return ranks;
  }
  return 0;
}

cudaError_t launch_power_lat(const PowerArgs& a, int ranks, cudaStream_t stream) {
  return launch_lat<PowerArgs>(power_lat_kernel, a, ranks, stream);
}

cudaError_t launch_pipg_lat(const PipgArgs& a, int ranks, cudaStream_t stream) {
  return launch_lat<PipgArgs>(pipg_lat_kernel, a, ranks, stream);
}

}  // namespace ptopt_b200
