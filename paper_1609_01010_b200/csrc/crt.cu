// Three-primes integer product over Z (config 5): per-prime products via
// the convolution engines (inputs reduced on load), then Garner CRT into
// 3 x 32-bit limbs.  No reference counterpart; see
// SURVEY.md section 8 a14 for the definition used here.
#include <cstdlib>
#include <cstring>

#include "crt.cuh"
#include "fourstep.cuh"
#include "runtime.h"

namespace mc {

static const u32 kP[3] = {kCrtP1, kCrtP2, kCrtP3};

// Garner: y2 = (r2 - r1) / p1 mod p2; x12 = r1 + p1*y2 (< p1*p2);
// y3 = (r3 - x12) / (p1*p2) mod p3; x = x12 + p1*p2*y3 (< 2^90).
// limbs[k * ls + i] for i < n; ls = n for the planar [3][n] layout, or the
// full length when a slice is written (the distributed CRT: residues and
// limbs may live in peer GPUs' memory, reached over NVLink by these loads
// and stores -- the gather is fused into the kernel).
__global__ void crt3_kernel(const u32 *__restrict__ r1, const u32 *__restrict__ r2,
                            const u32 *__restrict__ r3, u32 *__restrict__ limbs, long long n,
                            long long ls, const CrtConsts K) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const u32 a = __ldcs(r1 + i), b = __ldcs(r2 + i), c = __ldcs(r3 + i);
        u32 l0, l1, l2;
        garner_limbs(a, garner_y2(a, b, K), c, K, l0, l1, l2);
        __stcs(limbs + i, l0);
        __stcs(limbs + ls + i, l1);
        __stcs(limbs + 2 * ls + i, l2);
    }
}

static mc_status launch_crt(const u32 *r1, const u32 *r2, const u32 *r3, u32 *limbs, long long n,
                            cudaStream_t st, long long ls = -1) {
    if (n <= 0) return n == 0 ? MC_OK : fail(MC_EINVAL, "negative length");
    if (ls < 0) ls = n;
    const int thr = 256;
    long long blocks = std::min<long long>((n + thr - 1) / thr, (long long)sm_count() * 8);
    crt3_kernel<<<(unsigned)blocks, thr, 0, st>>>(r1, r2, r3, limbs, n, ls, crt_consts());
    note_launches(1);
    MC_CUDA_CHECK(cudaGetLastError());
    return MC_OK;
}

// three_primes.cu: the fused four-step path (K = 18..23)
bool three_primes_fused_ok(long long n);
long long three_primes_fused_scratch(long long n);
mc_status three_primes_fused(const u32 *a, int z1, const u32 *b, int z2, u32 *limbs,
                             u32 *scratch, cudaStream_t st, cudaStream_t fs[3],
                             cudaEvent_t fork_ev, cudaEvent_t done_ev[3]);

static bool fused_on() {  // MC_NO_FUSED_CRT=1: per-prime products + crt3 (A/B)
    static const bool on = [] { const char *e = getenv("MC_NO_FUSED_CRT"); return !(e && *e); }();
    return on;
}

// product mod kP[k] of arbitrary-word inputs (reduced on load)
mc_status conv_dispatch_reduced(const u32 *a, int z1, const u32 *b, int z2, u32 *r, u32 p,
                                cudaStream_t st);

}  // namespace mc

using namespace mc;

extern "C" {

mc_status mc_crt3(const uint32_t *r1, const uint32_t *r2, const uint32_t *r3, uint32_t *limbs,
                  int64_t n, void *stream) {
    if (n > 0 && (!r1 || !r2 || !r3 || !limbs)) return fail(MC_EINVAL, "null pointer");
    return launch_crt(r1, r2, r3, limbs, n, (cudaStream_t)stream);
}

mc_status mc_crt3_slice(const uint32_t *r1, const uint32_t *r2, const uint32_t *r3,
                        uint32_t *limbs, int64_t limb_stride, int64_t count, void *stream) {
    if (count < 0 || limb_stride < count) return fail(MC_EINVAL, "bad slice");
    if (count > 0 && (!r1 || !r2 || !r3 || !limbs)) return fail(MC_EINVAL, "null pointer");
    return launch_crt(r1, r2, r3, limbs, count, (cudaStream_t)stream, limb_stride);
}

// ---- peer memory for the distributed CRT (CUDA IPC; control plane only)
mc_status mc_ipc_alloc(int64_t bytes, void **dptr, uint8_t *handle) {
    if (bytes <= 0 || !dptr || !handle) return fail(MC_EINVAL, "bad arguments");
    MC_CUDA_CHECK(cudaMalloc(dptr, (size_t)bytes));
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, *dptr);
    if (e != cudaSuccess) {
        cudaFree(*dptr);
        *dptr = nullptr;
        return cuda_fail(e, "cudaIpcGetMemHandle");
    }
    memcpy(handle, &h, sizeof(h));
    return MC_OK;
}

mc_status mc_ipc_open(const uint8_t *handle, void **dptr) {
    if (!handle || !dptr) return fail(MC_EINVAL, "bad arguments");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    MC_CUDA_CHECK(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
    return MC_OK;
}

mc_status mc_ipc_close(void *dptr) {
    MC_CUDA_CHECK(cudaIpcCloseMemHandle(dptr));
    return MC_OK;
}

mc_status mc_ipc_free(void *dptr) {
    MC_CUDA_CHECK(cudaFree(dptr));
    return MC_OK;
}

mc_status mc_copy_device(void *dst, const void *src, int64_t bytes, void *stream) {
    if (bytes < 0 || (bytes > 0 && (!dst || !src))) return fail(MC_EINVAL, "bad arguments");
    if (bytes == 0) return MC_OK;
    MC_CUDA_CHECK(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice,
                                  (cudaStream_t)stream));
    return MC_OK;
}

int64_t mc_three_primes_scratch_words(int32_t z1, int32_t z2) {
    if (z1 < 1 || z2 < 1) return 0;
    const long long n = (long long)z1 + z2 - 1;
    if (fused_on() && three_primes_fused_ok(n)) return three_primes_fused_scratch(n);
    return 3ll * n;
}

mc_status mc_mul_mod_prime_k(const uint32_t *a, int32_t z1, const uint32_t *b, int32_t z2,
                             uint32_t *r, int k, void *stream) {
    if (k < 0 || k > 2) return fail(MC_EINVAL, "prime index must be 0, 1 or 2");
    if (z1 < 1 || z2 < 1) return fail(MC_EINVAL, "inputs must be nonempty");
    if (!a || !b || !r) return fail(MC_EINVAL, "null pointer");
    return conv_dispatch_reduced(a, z1, b, z2, r, kP[k], (cudaStream_t)stream);
}

mc_status mc_mul_three_primes(const uint32_t *a, int32_t z1, const uint32_t *b, int32_t z2,
                              uint32_t *limbs, uint32_t *scratch, void *stream) {
    if (z1 < 1 || z2 < 1) return fail(MC_EINVAL, "inputs must be nonempty");
    if (!a || !b || !limbs) return fail(MC_EINVAL, "null pointer");
    const long long n = (long long)z1 + z2 - 1;
    cudaStream_t st = (cudaStream_t)stream;
    // The three prime channels are independent: fork them onto three streams
    // so their kernels fill the GPU together, join for the CRT.
    static thread_local int dev_cached = -1;
    static thread_local cudaStream_t fs[3];
    static thread_local cudaEvent_t fork_ev, done_ev[3];
    const int dev = current_device();
    if (dev_cached != dev) {
        for (int k = 0; k < 3; ++k) {
            MC_CUDA_CHECK(cudaStreamCreateWithFlags(&fs[k], cudaStreamNonBlocking));
            MC_CUDA_CHECK(cudaEventCreateWithFlags(&done_ev[k], cudaEventDisableTiming));
        }
        MC_CUDA_CHECK(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
        dev_cached = dev;
    }
    if (fused_on() && three_primes_fused_ok(n))
        return three_primes_fused(a, z1, b, z2, limbs, scratch, st, fs, fork_ev, done_ev);
    uint32_t *res = scratch;
    bool own = false;
    if (!res) {
        keep_pool_memory();
        MC_CUDA_CHECK(cudaMallocAsync(&res, sizeof(uint32_t) * 3 * n, st));
        own = true;
    }
    MC_CUDA_CHECK(cudaEventRecord(fork_ev, st));
    mc_status s = MC_OK;
    for (int k = 0; k < 3; ++k) {
        MC_CUDA_CHECK(cudaStreamWaitEvent(fs[k], fork_ev, 0));
        if (s == MC_OK) s = conv_dispatch_reduced(a, z1, b, z2, res + k * n, kP[k], fs[k]);
        MC_CUDA_CHECK(cudaEventRecord(done_ev[k], fs[k]));
        MC_CUDA_CHECK(cudaStreamWaitEvent(st, done_ev[k], 0));
    }
    if (s == MC_OK) s = launch_crt(res, res + n, res + 2 * n, limbs, n, st);
    if (own) cudaFreeAsync(res, st);
    return s;
}

}  // extern "C"
