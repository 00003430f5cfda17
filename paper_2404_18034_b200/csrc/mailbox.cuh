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
