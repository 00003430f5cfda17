// mailbox.cuh — one-way hand-off between the CTAs of a thread-block cluster without cluster
// barriers: every remote store is an asynchronous store that completes transaction bytes on an
// mbarrier in the RECEIVER's shared memory (`st.async ... mbarrier::complete_tx::bytes`); the
// receiver arms the barrier with the byte count of the phase and only the warps that read the
// received entries wait for it.  A release/acquire `cluster.sync` costs 450-530 clk on B200, this
// hand-off ~280 (tools/probes/cluster_sync_cost.cu).  Shared by the register-resident solver
// kernels (solver_fast.cu) and the latency-mode kernels (solver_lat.cu).
#pragma once

#include <cuda_runtime.h>

namespace ptopt_b200 {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
/// Shared-memory address of `local` inside CTA `rank` of the cluster (shared::cluster window).
__device__ __forceinline__ unsigned partner_u32(const void* local, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
  return r;
}
/// Asynchronous remote store of one double; completes 8 transaction bytes on the receiver's mailbox.
__device__ __forceinline__ void push_f64(unsigned dst, double v, unsigned box) {
  asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(dst), "d"(v),
               "r"(box)
               : "memory");
}
/// The same as one predicated instruction (no branch round the store).
__device__ __forceinline__ void push_f64_pred(unsigned pred, unsigned dst, double v, unsigned box) {
  asm volatile(
      "{ .reg .pred p; setp.ne.u32 p, %3, 0;\n"
      "  @p st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2]; }" ::"r"(dst),
      "d"(v), "r"(box), "r"(pred)
      : "memory");
}
/// Arms the mailbox at shared-memory address `bar` when `pred` is set (one predicated instruction).
__device__ __forceinline__ void mbar_expect_pred(unsigned pred, unsigned bar, int bytes) {
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0;\n"
               "  @p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1; }" ::"r"(bar),
               "r"(bytes), "r"(pred)
               : "memory");
}
/// mbar_wait on a shared-memory address.
__device__ __forceinline__ void mbar_wait_at(unsigned bar, unsigned parity) {
  unsigned ok, polls = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok)
                 : "r"(bar), "r"(parity & 1u)
                 : "memory");
  } while (!ok && ++polls < (1u << 26));
  if (!ok) __trap();
}
/// One non-blocking test of a mailbox phase (no memory clobber: ordinary loads and arithmetic may be
/// scheduled round it; other volatile asm statements -- the loads of the received entries -- stay
/// behind it).  Returns non-zero when the phase is complete.
__device__ __forceinline__ unsigned mbar_test_at(unsigned bar, unsigned parity) {
  unsigned ok;
  asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(ok)
               : "r"(bar), "r"(parity & 1u));
  return ok;
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long* bar, int bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
/// Waits for `phase` of a mailbox.  A wait normally ends within a microsecond; a protocol error
/// must surface as a failed launch, not as a hung device, so the poll gives up (trap) after
/// 2^26 attempts (seconds).
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, int phase) {
  unsigned ok, polls = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok)
                 : "r"(smem_u32(bar)), "r"((unsigned)(phase & 1))
                 : "memory");
  } while (!ok && ++polls < (1u << 26));
  if (!ok) __trap();
}

}  // namespace ptopt_b200
