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

#include <cstdio>
#include <cstdlib>

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

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
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

/// Asynchronous remote store of a pair of doubles (16 bytes on the receiver's mailbox).
__device__ __forceinline__ void push_f64x2(unsigned dst, double v0, double v1, unsigned box) {
  asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(dst),
               "d"(v0), "d"(v1), "r"(box)
               : "memory");
}

/// Mailboxes: cleared shared memory first, then the barriers, then a cluster barrier so that every
/// CTA is running, cleared and initialised before any remote store.
__device__ __forceinline__ void open_boxes(LatSmem* S, int tid) {
  for (int e = tid; e < (int)(sizeof(LatSmem) / sizeof(double)); e += blockDim.x)
    reinterpret_cast<double*>(S)[e] = 0.0;
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) mbar_init(S->box + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cg::this_cluster().sync();
}

/// Where a thread's values go: its slots in this CTA's shared memory and — for the CTA's first /
/// last node — the matching guard slots of the neighbour rank (shared::cluster addresses, computed
/// once).  Loop-invariant, so the hot loops carry no address arithmetic.
struct Ports {
  double* dual_dst;    // php[node][row]
  double* bps_dst;     // bps[node][c0..c0+1]  (cq 3)
  double* prim_dst;    // xs / us [node][entry pair]  (cq 0..2)
  unsigned r_dual, r_bps, r_prim;  // the same slots inside the next (duals) / previous (primal) rank
  unsigned send_dual, send_bps, send_prim;  // 1 when this thread sends that value
  unsigned box_to_next, box_to_prev;
  const double* seg;     // this thread's segment of the node vector [x_k | u_k | u_{k+1}]
  const double* x_next;  // x_{k+1}[row] (row 15: entry 14), x_k[same]
  const double* x_cur;
  const double* nb;      // neighbour pair: phi_{k-1} (x owners; theta_{k-1} behind entry 14) / B+^T phi_{k-1} (u owners)
  const double* theta_k; // php[node][15]
  unsigned long long* box;
};

__device__ __forceinline__ Ports make_ports(LatSmem* S, const Lane& t, const Cut& cut) {
  Ports q;
  q.dual_dst = S->php + (t.pc + 1) * kXP + t.row;
  q.bps_dst = S->bps + (t.pc + 1) * kUP + t.c0;
  q.prim_dst = t.cq == 2 ? S->us + (t.pc + 1) * kUP + t.c0 : S->xs + (t.pc + 1) * kXP + 8 * (t.cq & 1) + t.c0;
  q.r_dual = q.r_bps = q.r_prim = q.box_to_next = q.box_to_prev = 0u;
  q.send_dual = t.push_prev ? 1u : 0u;
  q.send_bps = (t.push_prev && t.cq == 3) ? 1u : 0u;
  q.send_prim = (t.push_next && t.cq != 3) ? 1u : 0u;
  if (t.push_prev) {  // slot -1 of the next rank
    q.r_dual = partner_u32(S->php + t.row, cut.rank + 1);
    q.r_bps = partner_u32(S->bps + t.c0, cut.rank + 1);
    q.box_to_next = partner_u32(S->box + kBoxPrev, cut.rank + 1);
  }
  if (t.push_next) {  // slot nloc of the previous rank
    const double* slot = t.cq == 2 ? S->us + (cut.nloc_prev + 1) * kUP + t.c0
                                   : S->xs + (cut.nloc_prev + 1) * kXP + 8 * (t.cq & 1) + t.c0;
    q.r_prim = partner_u32(slot, cut.rank - 1);
    q.box_to_prev = partner_u32(S->box + kBoxNext, cut.rank - 1);
  }
  q.seg = t.cq == 0   ? S->xs + (t.pc + 1) * kXP
          : t.cq == 1 ? S->xs + (t.pc + 1) * kXP + 8
          : t.cq == 2 ? S->us + (t.pc + 1) * kUP
                      : S->us + (t.pc + 2) * kUP;
  const int rsel = t.theta_lane ? kNX - 1 : t.row;
  q.x_next = S->xs + (t.pc + 2) * kXP + rsel;
  q.x_cur = S->xs + (t.pc + 1) * kXP + rsel;
  q.nb = t.cq == 2 ? S->bps + t.pc * kUP + t.c0 : S->php + t.pc * kXP + 8 * (t.cq & 1) + t.c0;
  q.theta_k = S->php + (t.pc + 1) * kXP + kNX;
  q.box = S->box;
  return q;
}

// The hand-off code sits on the critical path of every warp, also of those it does not concern:
// a branch the compiler cannot prove warp-uniform costs a divergence frame (BSSY / BSYNC) on a loop
// that is one dependent chain.  So the sends are single predicated instructions (no branch), and
// the receive tests a vote result (provably uniform); `mine` is the same in all lanes of a warp.
__device__ __forceinline__ void push_f64_if(unsigned pred, unsigned dst, double v, unsigned box) {
  asm volatile(
      "{ .reg .pred p; setp.ne.u32 p, %3, 0;\n"
      "  @p st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2]; }" ::"r"(dst),
      "d"(v), "r"(box), "r"(pred)
      : "memory");
}
__device__ __forceinline__ void push_f64x2_if(unsigned pred, unsigned dst, double v0, double v1, unsigned box) {
  asm volatile(
      "{ .reg .pred p; setp.ne.u32 p, %4, 0;\n"
      "  @p st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3]; }" ::"r"(dst),
      "d"(v0), "d"(v1), "r"(box), "r"(pred)
      : "memory");
}
__device__ __forceinline__ void receive(const Ports& q, int which, bool mine, bool armer, int bytes, int phase) {
  if (!__any_sync(0xffffffffu, mine)) return;
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0;\n"
               "  @p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1; }" ::"r"(smem_u32(q.box + which)),
               "r"(bytes), "r"((unsigned)armer)
               : "memory");
  mbar_wait(q.box + which, phase);
}

/// Publishes the dual of this thread's row (php) and — cq 3 — the B+ column sums (bps) in the
/// node's slot; the CTA's last node sends the same values into slot -1 of the next rank.
template <bool kLone>
__device__ __forceinline__ void publish_duals(const Ports& q, const Lane& t, double d, const double (&cs)[2]) {
  *q.dual_dst = d;
  if (t.cq == 3) *reinterpret_cast<double2*>(q.bps_dst) = make_double2(cs[0], cs[1]);
  if constexpr (!kLone) {
    push_f64_if(q.send_dual, q.r_dual, d, q.box_to_next);
    push_f64x2_if(q.send_bps, q.r_bps, cs[0], cs[1], q.box_to_next);
  }
}

/// Stores the two primal entries (cq 0, 1: x; cq 2: u) into the node's slot; the CTA's first node
/// sends them into slot nloc of the previous rank as well.
template <bool kLone>
__device__ __forceinline__ void publish_primal(const Ports& q, const Lane& t, double v0, double v1) {
  if (t.cq != 3) *reinterpret_cast<double2*>(q.prim_dst) = make_double2(v0, v1);
  if constexpr (!kLone) push_f64x2_if(q.send_prim, q.r_prim, v0, v1, q.box_to_prev);
}

// ---------------------------------------------------------------------------------------------
// power iteration (pipg.hpp:206-292)
// ---------------------------------------------------------------------------------------------
// kLone: the cluster is a single CTA -- every hand-off (and its warp-uniform test) is compiled out.
template <bool kLone>
__global__ void __launch_bounds__(kLatThreadsMax, 1) power_lat_kernel(PowerArgs a) {
  __shared__ LatSmem Sm;
  LatSmem* S = &Sm;
  const Cut cut = make_cut(a.shape.n);
  const int b = blockIdx.x / cut.ranks;
  if (a.active && !a.active[b]) return;  // every CTA of the cluster leaves together
  const int n = a.shape.n, m = n - 1;
  const Lane t = make_lane(cut, m);
  open_boxes(S, t.tid);
  const Ports q = make_ports(S, t, cut);
  auto recv = [&](int which, bool mine, bool armer, int bytes, int phase) {
    if constexpr (!kLone) receive(q, which, mine, armer, bytes, phase);
  };
  const bool u_owner = t.cq == 2;
  const bool is14 = t.cq == 1 && t.rg == 3;  // entry 0 of this pair is x[14], entry 1 the pad
  const bool alive0 = t.node && t.cq < 3, alive1 = alive0 && t.rg < 3 + (t.cq == 0);
  const double sgn = u_owner ? 1.0 : -1.0;   // u: + B+^T phi_{k-1};  x: - phi_{k-1}  (A+ = -I)
  const double keep0 = alive0 ? 1.0 : 0.0, keep1 = alive1 ? 1.0 : 0.0;

  double aop[4][4][2];
  load_tile(a.sp, (size_t)b * m + (t.ival ? t.kg : 0), t, aop);

  // Squared norm of the iterate, two levels: every warp leaves its share in shared memory; after
  // the block barrier that ends the trip thread 0 adds the CTA's shares and sends the total to every
  // rank — its own included, so that one mailbox covers all of them — by trip parity (a rank may run
  // up to one trip ahead of another, see solver_fast.cu).  Every rank then adds the same eight
  // totals in the same order.
  double* shares = S->shares;                       // [parity][kLatWarpsMax]
  double* totals = S->shares + 2 * kLatWarpsMax;    // [parity][kLatMaxRanks]
  // lane r of warp 0 sends to rank r: one predicated store, no loop and no branch (every thread forms
  // the total -- four broadcast loads and three additions that overlap with what follows)
  unsigned tot_remote = 0u, box_remote = 0u, tot_send = 0u;
  if (!kLone && t.warp == 0 && t.lane < cut.ranks) {
    tot_remote = partner_u32(totals + cut.rank, t.lane);
    box_remote = partner_u32(S->box + kBoxNorm, t.lane);
    tot_send = 1u;
  }
  constexpr bool lone = kLone;  // a single CTA: the warps' shares are the whole norm, no mailbox
  auto send_total = [&](int trip) {  // after the block barrier behind the warps' shares
    static_assert(kLatWarpsMax == 8, "tree below");
    const double2* p = reinterpret_cast<const double2*>(shares + (trip & 1) * kLatWarpsMax);
    const double2 s0 = p[0], s1 = p[1], s2 = p[2], s3 = p[3];
    const double tot = ((s0.x + s0.y) + (s1.x + s1.y)) + ((s2.x + s2.y) + (s3.x + s3.y));
    push_f64_if(tot_send, tot_remote + 8u * (unsigned)((trip & 1) * kLatMaxRanks), tot, box_remote + 8u * (unsigned)(trip & 1));
  };
  auto norm_sq = [&](int trip) {  // waits for the totals of `trip`, then adds them (absent ranks: zero)
    static_assert(kLatMaxRanks == 8 && kLatWarpsMax == 8, "tree below");
    if (!lone) recv(kBoxNorm + (trip & 1), true, t.tid == 0, 8 * cut.ranks, trip >> 1);
    const double2* p = reinterpret_cast<const double2*>((lone ? shares : totals) + (trip & 1) * 8);
    const double2 s0 = p[0], s1 = p[1], s2 = p[2], s3 = p[3];
    return ((s0.x + s0.y) + (s1.x + s1.y)) + ((s2.x + s2.y) + (s3.x + s3.y));
  };

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
    publish_primal<kLone>(q, t, v0, v1);  // the first node also reaches the previous rank: "next" phase 0
    acc = v0 * v0 + v1 * v1;
  }
  double vcd = 0.0;  // vc+ - vc-: the only combination of the two groups the forward map uses
  if (t.row_alive) {
    const double vp = a.seed_vcp[((size_t)b * m + t.kg) * kNX + t.row], vn = a.seed_vcn[((size_t)b * m + t.kg) * kNX + t.row];
    vcd = vp - vn;
    acc += vp * vp;
    acc += vn * vn;
  }
  acc = warp_sum(acc);
  if (t.lane == 0) shares[t.warp] = acc;
  __syncthreads();
  if constexpr (!kLone) send_total(0);
  // The norm of trip j-1 (j = 1: the seed) is received and tested inside trip j, every trip alike --
  // no `if (j > 1)` block that would keep the norm -> rsqrt -> test chain out of the basic block of
  // the products it can overlap with.  The first test compares the seed's norm with a NaN, which no
  // tolerance accepts; a zero seed (pipg.hpp:224-225) is found there too.  Inside the loop sigma is
  // ss * rsqrt(ss) (1 ulp from sqrt: it only feeds the stopping test) and the scale 1 / sigma the
  // same rsqrt; the value returned is the correctly rounded sqrt of the last squared norm.
  // (A single CTA tests the seed in front of the loop as well: its norm needs no mailbox, and the
  // kernel measures 4 % faster that way.)
  double ss_last = 0.0, inv = 0.0;
  double sigma = __longlong_as_double(0x7ff8000000000000ll);
  bool seed_zero = false;
  if constexpr (kLone) {
    ss_last = norm_sq(0);
    if (ss_last == 0.0) {  // pipg.hpp:224-225
      if (t.tid == 0) {
        if (a.status) a.status[b] = kStSeedZero;
        a.sigma[b] = 0.0;
        if (a.trips) a.trips[(size_t)b * a.trips_stride + (a.trips_slot ? a.trips_slot[b] : 0)] = 0;
      }
      return;
    }
    inv = rsqrt(ss_last);
  }
  // row lanes scale (forward row - x_{k+1}[row]) + vcd; the relaxation-dual lane x_{k+1}[14] - x_k[14]
  const double live = (t.row_alive || (t.theta_lane && t.ival)) ? 1.0 : 0.0;

  int trips = 0;
  bool done = false;
  if constexpr (!kLone) {
    if (a.j_max < 1) {  // no trip at all: the seed's norm is the result
      ss_last = norm_sq(0);
      seed_zero = ss_last == 0.0;
      recv(kBoxNext, t.next_warp, t.next_armer, kNextBytes, 0);
      done = true;
    }
  }
  for (int j = 1; j <= a.j_max; ++j) {
    // ---- forward map (pipg.hpp:234-245); the norm of trip j-1 arrives while the products run
    recv(kBoxNext, t.next_warp, t.next_armer, kNextBytes, j - 1);  // the next rank's first node of trip j-1
    const double xn1 = q.x_next[0], xc = q.x_cur[0];
    const double r = forward_row(aop, q.seg, t.rg);
    const double s = t.theta_lane ? xn1 - xc : (r - xn1) + vcd;
    {  // stopping test of trip j-1 (pipg.hpp:277-289); j = 1: the seed against NaN, never met
      const double ss = norm_sq(j - 1);
      ss_last = ss;
      if (ss == 0.0) {  // a zero seed (pipg.hpp:224-225), or an iterate in the null space (:280-284)
        if constexpr (!kLone) seed_zero = j == 1;
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
    const double mine = live * (s * inv);  // phi_k[row], or theta_k on lane (3,3)
    double d[4], cs[2];
    gather_rows(mine, d);
    drop_theta_slot(t, d);
    transposed_pair(aop, d, cs);
    publish_duals<kLone>(q, t, mine, cs);
    const double phi = t.theta_lane ? 0.0 : mine;
    vcd = 2.0 * phi;  // vc+ = phi, vc- = -phi (pipg.hpp:268-279)
    const double acc_d = vcd * phi;
    __syncthreads();
    // ---- adjoint map (pipg.hpp:247-275)
    recv(kBoxPrev, t.prev_warp, t.prev_armer, kPrevBytes, j - 1);  // the previous rank's last interval
    const double2 nb = *reinterpret_cast<const double2*>(q.nb);
    const double extra = is14 ? nb.y - q.theta_k[0] : 0.0;  // -theta_k + theta_{k-1} on the last state (e_y)
    const double v0 = keep0 * (fma(sgn, nb.x, cs[0]) + extra);
    const double v1 = keep1 * fma(sgn, nb.y, cs[1]);
    publish_primal<kLone>(q, t, v0, v1);
    acc = fma(v0, v0, v1 * v1) + acc_d;
    acc = warp_sum(acc);
    if (t.lane == 0) shares[(j & 1) * kLatWarpsMax + t.warp] = acc;
    __syncthreads();
    if constexpr (!kLone) send_total(j);
  }
  if (!done) {  // j_max trips without meeting the tolerance
    if (a.j_max >= 1) ss_last = norm_sq(a.j_max);
    if (a.j_max >= 1) recv(kBoxNext, t.next_warp, t.next_armer, kNextBytes, a.j_max);  // still on its way
  }
  if (t.tid == 0 && cut.rank == 0) {
    if (seed_zero && a.status) a.status[b] = kStSeedZero;
    a.sigma[b] = (1.0 + a.eps_buff) * sqrt(ss_last);  // 0 for a zero seed
    if (a.trips) a.trips[(size_t)b * a.trips_stride + (a.trips_slot ? a.trips_slot[b] : 0)] = trips;
  }
  cg::this_cluster().sync();  // nobody leaves while a neighbour may still write into it
}

// ---------------------------------------------------------------------------------------------
// customized PIPG (pipg.hpp:350-497)
// ---------------------------------------------------------------------------------------------
template <bool kLone>
__global__ void __launch_bounds__(kLatThreadsMax, 1) pipg_lat_kernel(PipgArgs a) {
  __shared__ LatSmem Sm;
  LatSmem* S = &Sm;
  const Cut cut = make_cut(a.shape.n);
  const int b = blockIdx.x / cut.ranks;
  if (a.active && !a.active[b]) return;  // every CTA of the cluster leaves together
  const int n = a.shape.n, m = n - 1;
  const Lane t = make_lane(cut, m);
  open_boxes(S, t.tid);
  const Ports q = make_ports(S, t, cut);
  auto recv = [&](int which, bool mine, bool armer, int bytes, int phase) {
    if constexpr (!kLone) receive(q, which, mine, armer, bytes, phase);
  };
  const bool u_owner = t.cq == 2;
  const bool is14 = t.cq == 1 && t.rg == 3;
  const bool alive0 = t.node && t.cq < 3, alive1 = alive0 && t.rg < 3 + (t.cq == 0);
  const bool last_node = t.node && t.kg == n - 1;
  const double sgn = u_owner ? 1.0 : -1.0;

  double aop[4][4][2];
  load_tile(a.sp, (size_t)b * m + (t.ival ? t.kg : 0), t, aop);

  // ---- per-entry constants and the warm start (pipg.hpp:362-374): ex = cur = workspace.
  // One code path for every kind of entry: a control entry is clamped to its box (pipg.hpp:418-419),
  // a boundary row to [value, value] (:408-413), a free state to (-inf, inf), an entry that does
  // not exist (pads, idle threads, cq 3) to [0, 0].
  const int ce = u_owner ? t.c0 : 8 * t.cq + t.c0;
  double pe[2] = {0.0, 0.0}, lo[2] = {0.0, 0.0}, hi[2] = {0.0, 0.0}, cost[2] = {0.0, 0.0};
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const bool alive = e == 0 ? alive0 : alive1;
    if (!alive) continue;
    if (u_owner) {
      const size_t g = ((size_t)b * n + t.kg) * kNU + ce + e;
      pe[e] = a.ws.u[g];
      lo[e] = a.sp.u_min[g];
      hi[e] = a.sp.u_max[g];
    } else {
      pe[e] = a.ws.x[((size_t)b * n + t.kg) * kNX + ce + e];
      lo[e] = -INFINITY;
      hi[e] = INFINITY;
      if (last_node) cost[e] = a.shape.w_cost * a.shape.e_cost[ce + e];
      // later entries override earlier ones, as the assignment loops do
      if (t.kg == 0)
        for (int i = 0; i < a.shape.n_init_fix; ++i)
          if (a.shape.init_fix_idx[i] == ce + e) lo[e] = hi[e] = a.sp.init_fix_val[(size_t)b * a.shape.n_init_fix + i];
      if (last_node)
        for (int i = 0; i < a.shape.n_final_fix; ++i)
          if (a.shape.final_fix_idx[i] == ce + e) lo[e] = hi[e] = a.sp.final_fix_val[(size_t)b * a.shape.n_final_fix + i];
    }
  }
  // dual row: dynamics dual + the two slack groups, or (lane (3,3)) the relaxation dual.  Again one
  // code path: the relaxation lane has an infinite slack weight (its slacks stay 0) and clips its
  // dual at 0; a row that does not exist has a zero step (its dual stays 0).
  const bool theta_alive = t.theta_lane && t.ival;
  double phe = 0.0, vpe = 0.0, vne = 0.0, wrow = 0.0;
  if (t.row_alive) {
    const size_t g = ((size_t)b * m + t.kg) * kNX + t.row;
    phe = a.ws.dyn_dual[g];
    vpe = a.ws.vc_pos[g];
    vne = a.ws.vc_neg[g];
    wrow = a.sp.w[g];
  } else if (theta_alive) {
    phe = a.ws.relax_dual[(size_t)b * m + t.kg];
    wrow = -a.sp.eps_relax[(size_t)b * m + t.kg];
  }
  const double w_ep_lane = t.theta_lane ? INFINITY : a.shape.w_ep;
  // materialised *_cur values of the last two iterations (pipg.hpp:490-495 returns the current ones)
  double cur_p[2] = {pe[0], pe[1]}, cur_d = phe, cur_vp = vpe, cur_vn = vne;
  double prv_p[2] = {pe[0], pe[1]}, prv_d = phe, prv_vp = vpe, prv_vn = vne;

  const double sigma = a.sigma[b];
  const double alpha = 2.0 / (a.shape.w_prox + sqrt(a.shape.w_prox * a.shape.w_prox + 4.0 * a.omega * sigma));
  const double beta = a.omega * alpha;
  const double beta_lane = (t.row_alive || theta_alive) ? beta : 0.0;
  const double rho = a.rho, w_prox = a.shape.w_prox;

  double cs[2];
  {  // partial sums of H^T phi_ex of the warm start, for the first primal step
    double d[4];
    gather_rows(phe, d);
    drop_theta_slot(t, d);
    transposed_pair(aop, d, cs);
    publish_duals<kLone>(q, t, phe, cs);
  }
  __syncthreads();

  int iters = 0;
  bool converged = false, diverged = false;
  int to_check = a.j_check;
#ifdef PTOPT_LAT_PROFILE
  long long ph_clk[6] = {0, 0, 0, 0, 0, 0}, tc = clock64();
#define LAT_PHASE(i) { const long long tn = clock64(); ph_clk[i] += tn - tc; tc = tn; }
#else
#define LAT_PHASE(i)
#endif
  for (int j = 1; j <= a.j_max; ++j) {
    --to_check;
    const bool check = to_check == 0;
    if (check) {  // this iteration is compared with the one before it
      to_check = a.j_check;
      prv_p[0] = cur_p[0];
      prv_p[1] = cur_p[1];
      prv_d = cur_d;
      prv_vp = cur_vp;
      prv_vn = cur_vn;
    }
    // ---- primal projected-gradient step (pipg.hpp:388-420) by the owner of each entry
    recv(kBoxPrev, t.prev_warp, t.prev_armer, kPrevBytes, j - 1);  // previous rank, after iteration j-1
    {
      const double2 nb = *reinterpret_cast<const double2*>(q.nb);
      const double extra = is14 ? nb.y - q.theta_k[0] : 0.0;  // theta_{k-1} - theta_k on the last state
      const double nbv[2] = {nb.x, nb.y};
      double rf[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double x0 = pe[e];
        double base = x0 * w_prox;
        base += cost[e];
        base = fma(sgn, nbv[e], base);
        if (e == 0) base += extra;
        const double grad = base + cs[e];
        double xn = x0 + -alpha * grad;
        xn = clamp_box(lo[e], hi[e], xn);  // std::max(lo, std::min(hi, v))
        rf[e] = fma(2.0, xn, -x0);
        cur_p[e] = xn;
        pe[e] = fma(rho, xn - x0, x0);  // extrapolation, pipg.hpp:461-472
      }
      publish_primal<kLone>(q, t, rf[0], rf[1]);
    }
    LAT_PHASE(0)
    __syncthreads();
    LAT_PHASE(1)
    recv(kBoxNext, t.next_warp, t.next_armer, kNextBytes, j - 1);  // next rank's first node, this iteration
    LAT_PHASE(2)
    // ---- slacks (pipg.hpp:423-430), PI feedback of the constraint violation (:433-458), extrapolation of
    //      the dual groups (:468-472) and the partial sums of H^T phi_ex for the next primal step
    {
      const double xn1 = q.x_next[0], xc = q.x_cur[0];
      const double p0 = phe, vp0 = vpe, vn0 = vne;
      const double vp = clip0(vp0 - alpha * (w_ep_lane + p0));
      const double vn = clip0(vn0 - alpha * (w_ep_lane - p0));
      const double slack = ((2.0 * vp - vp0) - (2.0 * vn - vn0)) + wrow;
      const double r = forward_row(aop, q.seg, t.rg);
      // row lanes: (A- x + B- u + B+ u+)[row] - x_{k+1}[row];  relaxation lane: x_{k+1}[14] - x_k[14]
      const double lead = t.theta_lane ? xn1 : r, trail = t.theta_lane ? xc : xn1;
      const double resid = (lead - trail) + slack;
      double pn = fma(beta_lane, resid, p0);
      pn = t.theta_lane ? clip0(pn) : pn;
      cur_d = pn;
      cur_vp = vp;
      cur_vn = vn;
      phe = fma(rho, pn - p0, p0);
      vpe = fma(rho, vp - vp0, vp0);
      vne = fma(rho, vn - vn0, vn0);
      double d[4];
      gather_rows(phe, d);
      drop_theta_slot(t, d);
      transposed_pair(aop, d, cs);
      publish_duals<kLone>(q, t, phe, cs);
    }
    iters = j;
    LAT_PHASE(3)
    __syncthreads();
    LAT_PHASE(4)
    if (check) {  // stopping_custom(cur, prev) and the divergence test, pipg.hpp:475-487
      double z_cur = 0.0, z_prev = 0.0, z_del = 0.0, r_cur = 0.0, r_prev = 0.0, r_del = 0.0, bad = 0.0;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        z_cur = max_nn(z_cur, fabs(cur_p[e]));
        z_prev = max_nn(z_prev, fabs(prv_p[e]));
        z_del = max_nn(z_del, fabs(cur_p[e] - prv_p[e]));
        if (!pt_finite(cur_p[e])) bad = 1.0;
      }
      z_cur = max_nn(max_nn(z_cur, fabs(cur_vp)), fabs(cur_vn));
      z_prev = max_nn(max_nn(z_prev, fabs(prv_vp)), fabs(prv_vn));
      z_del = max_nn(max_nn(z_del, fabs(cur_vp - prv_vp)), fabs(cur_vn - prv_vn));
      if (!t.theta_lane && !pt_finite(cur_d)) bad = 1.0;
      r_cur = fabs(cur_d);
      r_prev = fabs(prv_d);
      r_del = fabs(cur_d - prv_d);
      double v[7] = {z_cur, z_prev, z_del, r_cur, r_prev, r_del, bad};
#pragma unroll
      for (int k = 0; k < 7; ++k) v[k] = warp_max_nn(v[k]);
      if (t.lane == 0) {
#pragma unroll
        for (int k = 0; k < 7; ++k) S->red[t.warp * 8 + k] = v[k];
      }
      __syncthreads();
      if (t.tid < 7) {  // this CTA's maxima into every rank's table
        double mx = 0.0;
        for (int w = 0; w < t.nwarps; ++w) mx = max_nn(mx, S->red[w * 8 + t.tid]);
        for (int r = 0; r < cut.ranks; ++r) *cg::this_cluster().map_shared_rank(S->redc + cut.rank * 8 + t.tid, r) = mx;
      }
      cg::this_cluster().sync();
#pragma unroll
      for (int k = 0; k < 7; ++k) {
        double mx = 0.0;
        for (int r = 0; r < cut.ranks; ++r) mx = max_nn(mx, S->redc[r * 8 + k]);
        v[k] = mx;
      }
      cg::this_cluster().sync();  // the tables are rewritten at the next check
      if (v[6] > 0.0) {
        diverged = true;
        break;
      }
      if (v[2] <= a.eps_abs + a.eps_rel * max_nn(v[0], v[1]) && v[5] <= a.eps_abs + a.eps_rel * max_nn(v[3], v[4])) {
        converged = true;
        break;
      }
    }
  }
#ifdef PTOPT_LAT_PROFILE
  if (t.lane == 0 && b == 0)
    printf("pipg_lat rank %d warp %d: primal %.0f  barrier %.0f  recv-next %.0f  dual %.0f  barrier %.0f clk/iter (%d iters)\n",
           cut.rank, t.warp, (double)ph_clk[0] / iters, (double)ph_clk[1] / iters, (double)ph_clk[2] / iters,
           (double)ph_clk[3] / iters, (double)ph_clk[4] / iters, iters);
#endif
  recv(kBoxPrev, t.prev_warp, t.prev_armer, kPrevBytes, iters);  // what the previous rank sent last
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
  } else if (theta_alive) {
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
  // Measured on B200 (single solve, full budget): N = 15 takes 134 ms in one CTA (no hand-off at all),
  // 141 / 151 / 163 ms over 2 / 4 / 8 CTAs; N = 50 takes 146 ms over 8 CTAs (one warp per scheduler) and
  // 159 ms over 4 (two warps per scheduler).  So: a single CTA whenever the instance fits one
  // (<= 16 nodes), else the largest cluster the batch leaves room for.  PTOPT_LAT_RANKS overrides.
  static const int forced = [] {
    const char* env = getenv("PTOPT_LAT_RANKS");
    return env ? atoi(env) : 0;
  }();
  const auto fits = [&](int ranks) {
    return ranks <= s.n && (s.n + ranks - 1) / ranks <= kLatMaxLocalNodes &&
           (batch <= 0 || (long long)batch * ranks <= sm_count);
  };
  if (forced > 0) return fits(forced) ? forced : 0;
  if (fits(1)) return 1;
  for (int ranks = kLatMaxRanks; ranks >= 2; ranks >>= 1)
    if (fits(ranks)) return ranks;
  return 0;
}

cudaError_t launch_power_lat(const PowerArgs& a, int ranks, cudaStream_t stream) {
  return launch_lat<PowerArgs>(ranks == 1 ? power_lat_kernel<true> : power_lat_kernel<false>, a, ranks, stream);
}

cudaError_t launch_pipg_lat(const PipgArgs& a, int ranks, cudaStream_t stream) {
  return launch_lat<PipgArgs>(ranks == 1 ? pipg_lat_kernel<true> : pipg_lat_kernel<false>, a, ranks, stream);
}

}  // namespace ptopt_b200
