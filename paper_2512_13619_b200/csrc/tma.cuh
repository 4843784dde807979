// mbarrier + 1D bulk-TMA (cp.async.bulk) helpers shared by the streaming kernels (k_stream_gemv.cu, k_orth.cu).
#pragma once
#include <cstdint>

namespace hdgb {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Consumer release of a TMA ring stage.  The stage's shared-memory reads must have COMPLETED before the arrive becomes
// visible to the producer, whose refill writes the stage through the async proxy.  An instruction that merely consumes
// the loaded registers (FMA, mma.sync) does not pin that order: ptxas is free to schedule the arrive ahead of those
// consumers, right behind the ISSUE of the loads (seen in SASS: SYNCS.ARRIVE between the last LDS batch and its DMMAs),
// and a refill from L2 can then land while loads are still queued -- observed as one corrupted 8 x 8 tile in ~3e5
// elements.  The cross-proxy fence orders this thread's prior generic-proxy accesses before later async-proxy writes.
// Every reading thread releases for itself (the empty barrier counts threads, not warps): no reliance on __syncwarp()
// to extend lane 0's release to the other lanes' reads -- compute-sanitizer's racecheck does not accept that extension
// (it reported the lanes 1..31 of every consumer warp against the refill), costs nothing measurable, and is the form
// racecheck verifies clean.
__device__ __forceinline__ void ring_release_all(uint64_t* empty_bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive(empty_bar);
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1D bulk TMA copy global -> shared (16-byte aligned addresses, size a multiple of 16), completion counted in bytes
// on the mbarrier.
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// The same copy with an L2 evict-first hint: a matrix that is streamed once per launch should not push the gathered
// vector (re-read by neighbouring rows, tens of MB at most) out of the L2.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
                 : "memory");
}

}  // namespace hdgb
