// TMA bulk copies (cp.async.bulk, SASS UBLKCP) with mbarrier completion:
// used to prefetch the next product's operand rows into shared memory while
// the current product is being transformed.
#pragma once
#include <cstdint>

// Race-stress builds (-DMC_RACE_CHECK; scripts/gpu_race_check.sh).  The
// pool's compute-sanitizer is closed, so synchronisation is checked by
// perturbation instead: after every CTA barrier and mbarrier wait, and before
// every shared-memory exchange, a pseudo-random eighth of the threads sleeps
// up to ~2 us.  A missing barrier, a buffer refilled while still being read,
// or an exchange read before its write then reads data of another stage and
// the bit-exact parity tests fail.  Normal builds compile this to nothing.
#ifdef MC_RACE_CHECK
__device__ __forceinline__ void mc_perturb() {
    unsigned h = (threadIdx.x + 1u) * 2654435761u ^ (blockIdx.x + 7u) * 40503u ^
                 (unsigned)clock();
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    if ((h & 7u) == 0u) __nanosleep((h >> 8) & 2047u);
}
#else
__device__ __forceinline__ void mc_perturb() {}
#endif

__device__ __forceinline__ void mc_sync() {
    __syncthreads();
    mc_perturb();
}

// Warp-scope barrier for the exchanges whose writers and readers share a warp
// (conv_small.cuh exch_local): orders the warp's shared-memory accesses.
__device__ __forceinline__ void mc_syncwarp() {
    __syncwarp();
    mc_perturb();
}

namespace mc {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Order this thread's earlier generic-proxy shared accesses before later
// async-proxy (TMA) writes to the same buffer.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *sdst, const void *gsrc, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
    mc_perturb();
}

// 3-D tensor tile load (cp.async.bulk.tensor, SASS UTMALDG): box at
// coordinates (c0, c1, c2) of the tensor described by *tmap.
__device__ __forceinline__ void tma_load_3d(void *sdst, const void *tmap, int c0, int c1, int c2,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(sdst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// Acquire load at system scope (a flag written by a copy stream's
// stream-memory operation), then order later async-proxy (bulk copy) reads
// after it.
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void fence_proxy_async_all() {
    asm volatile("fence.proxy.async;" ::: "memory");
}

// Bulk store shared -> global (cp.async.bulk, bulk-group completion): 16-byte
// aligned addresses on both sides, size a multiple of 16.  Used for product
// rows written straight to page-locked host memory (zero-copy host calls),
// where per-warp 128-byte stores reach only ~28 GB/s over PCIe.
__device__ __forceinline__ void bulk_s2g(void *gdst, const void *ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// the shared-memory sources of all committed bulk stores have been read
__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// all committed bulk stores are complete
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Bulk prefetch of a contiguous global range into L2 (no shared memory, no
// completion to wait for): 16-byte aligned address, size a multiple of 16.
__device__ __forceinline__ void bulk_prefetch_l2(const void *gsrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gsrc), "r"(bytes) : "memory");
}

}  // namespace mc
