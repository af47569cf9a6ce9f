// Eq. 13 split engine on the GPU: a circular
// convolution of length 2n computed as one circular (mod x^n - 1) and one
// negacyclic (mod x^n + 1) convolution of length n, recombined with 1/2.
//   split_residues      convolve.py:214-219
//   recombine_residues  convolve.py:222-227
//   nega_conv           convolve.py:172-190 (twist by psi^j, psi = w_2n)
//   circ_conv_split     convolve.py:193-211
// The twist and the residue maps are fused into two elementwise kernels
// around the circular-convolution engine (conv_small / four-step).
#include "fourstep.cuh"
#include "runtime.h"

namespace mc {

mc_status get_twist_tables(u32 p, int K, const u32 **lo_f, const uint2 **hi_f, const u32 **lo_i,
                           const uint2 **hi_i);
mc_status circ_conv_dispatch(const u32 *u, const u32 *v, u32 *w, int log2L, long long batch,
                             u32 p, cudaStream_t st);

struct SplitParams {
    u32 p, pinv, r2;  // Montgomery constants (r2 = 2^64 mod p)
    Shoup inv2;       // (p + 1) / 2
    const u32 *lo_f, *lo_i;
    const uint2 *hi_f, *hi_i;
};

__device__ __forceinline__ u32 psi_pow(const SplitParams &S, u32 e, bool inv) {
    const u32 *lo = inv ? S.lo_i : S.lo_f;
    const uint2 *hi = inv ? S.hi_i : S.hi_f;
    const uint2 h = __ldg(hi + (e >> 12));
    return mul_shoup(__ldg(lo + (e & 4095)), h.x, h.y, S.p);
}

__device__ __forceinline__ u32 mulv(u32 x, u32 w, const SplitParams &S) {
    return mont_mul(mont_mul(x, w, S.p, S.pinv), S.r2, S.p, S.pinv);
}

// rows of u (length 2n) -> a (u_j + u_{j+n}) and b ((u_j - u_{j+n}) * psi^j
// when twist, else plain); n = 2^log2n.
__global__ void split_kernel(const u32 *u, long long ldu, u32 *a, u32 *b, int log2n,
                             long long batch, int twist, const SplitParams S) {
    const long long n = 1ll << log2n;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n * batch;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i >> log2n, j = i & (n - 1);
        const u32 x = u[r * ldu + j], y = u[r * ldu + j + n];
        a[r * n + j] = add_mod(x, y, S.p);
        const u32 d = sub_mod(x, y, S.p);
        b[r * n + j] = twist ? mulv(d, psi_pow(S, (u32)j, false), S) : d;
    }
}

// untwist (optional) the negacyclic half and recombine with 1/2
__global__ void recombine_kernel(const u32 *ca, const u32 *cb, u32 *w, long long ldw, int log2n,
                                 long long batch, int untwist, const SplitParams S) {
    const long long n = 1ll << log2n;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n * batch;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i >> log2n, j = i & (n - 1);
        const u32 x = ca[r * n + j];
        u32 y = cb[r * n + j];
        if (untwist) y = mulv(y, psi_pow(S, (u32)j, true), S);
        w[r * ldw + j] = mul_shoup(add_mod(x, y, S.p), S.inv2, S.p);
        w[r * ldw + j + n] = mul_shoup(sub_mod(x, y, S.p), S.inv2, S.p);
    }
}

// negacyclic: twist, circular convolution, untwist
__global__ void twist_kernel(const u32 *x, u32 *y, int log2n, long long batch, int inv,
                             const SplitParams S) {
    const long long n = 1ll << log2n;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n * batch;
         i += (long long)gridDim.x * blockDim.x) {
        const long long j = i & (n - 1);
        y[i] = mulv(x[i], psi_pow(S, (u32)j, inv != 0), S);
    }
}

static unsigned grid_for(long long work) {
    long long g = (work + 255) / 256, cap = (long long)sm_count() * 16;
    return (unsigned)std::max(1ll, std::min(g, cap));
}

// psi = w_{2n}: the twist tables of the 2n-point transform (psi^2 = w_n)
static mc_status split_setup(u32 p, int log2_2n, SplitParams *S) {
    const FieldTables *T;
    mc_status s = get_tables(p, log2_2n, &T);
    if (s != MC_OK) return s;
    if ((s = get_twist_tables(p, log2_2n, &S->lo_f, &S->hi_f, &S->lo_i, &S->hi_i)) != MC_OK)
        return s;
    S->p = p;
    S->pinv = T->pinv;
    const u64 r1 = (1ull << 32) % p;
    S->r2 = (u32)mulmod(r1, r1, p);
    S->inv2 = shoup((p + 1) >> 1, p);
    return MC_OK;
}

}  // namespace mc

using namespace mc;

extern "C" {

mc_status mc_split_residues(const uint32_t *u, uint32_t *a, uint32_t *b, int32_t log2n,
                            int64_t batch, uint32_t p, void *stream) {
    if (log2n < 0 || log2n > 29 || batch < 0) return fail(MC_EINVAL, "bad size");
    SplitParams S;
    memset(&S, 0, sizeof(S));
    mc_status s = check_field(p, 0);
    if (s != MC_OK) return s;
    S.p = p;
    if (batch == 0) return MC_OK;
    const long long n = 1ll << log2n;
    split_kernel<<<grid_for(n * batch), 256, 0, (cudaStream_t)stream>>>(u, 2 * n, a, b, log2n,
                                                                        batch, 0, S);
    note_launches(1);
    MC_CUDA_CHECK(cudaGetLastError());
    return MC_OK;
}

mc_status mc_recombine_residues(const uint32_t *a, const uint32_t *b, uint32_t *w,
                                int32_t log2n, int64_t batch, uint32_t p, void *stream) {
    if (log2n < 0 || log2n > 29 || batch < 0) return fail(MC_EINVAL, "bad size");
    SplitParams S;
    memset(&S, 0, sizeof(S));
    mc_status s = check_field(p, 0);
    if (s != MC_OK) return s;
    S.p = p;
    S.inv2 = shoup((p + 1) >> 1, p);
    if (batch == 0) return MC_OK;
    const long long n = 1ll << log2n;
    recombine_kernel<<<grid_for(n * batch), 256, 0, (cudaStream_t)stream>>>(a, b, w, 2 * n, log2n,
                                                                            batch, 0, S);
    note_launches(1);
    MC_CUDA_CHECK(cudaGetLastError());
    return MC_OK;
}

mc_status mc_nega_conv(const uint32_t *u, const uint32_t *v, uint32_t *w, int32_t log2n,
                       int64_t batch, uint32_t p, void *stream) {
    if (log2n < 0 || log2n > 29 || batch < 0) return fail(MC_EINVAL, "bad size");
    SplitParams S;
    memset(&S, 0, sizeof(S));
    mc_status s = split_setup(p, log2n + 1, &S);  // needs a root of order 2n
    if (s != MC_OK || batch == 0) return s;
    if (!u || !v || !w) return fail(MC_EINVAL, "null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    const long long n = 1ll << log2n;
    u32 *tmp = nullptr;
    keep_pool_memory();
    MC_CUDA_CHECK(cudaMallocAsync(&tmp, 4ull * 2 * n * batch, st));
    twist_kernel<<<grid_for(n * batch), 256, 0, st>>>(u, tmp, log2n, batch, 0, S);
    twist_kernel<<<grid_for(n * batch), 256, 0, st>>>(v, tmp + n * batch, log2n, batch, 0, S);
    s = circ_conv_dispatch(tmp, tmp + n * batch, w, log2n, batch, p, st);
    if (s == MC_OK) twist_kernel<<<grid_for(n * batch), 256, 0, st>>>(w, w, log2n, batch, 1, S);
    note_launches(3);
    cudaFreeAsync(tmp, st);
    MC_CUDA_CHECK(cudaGetLastError());
    return s;
}

mc_status mc_circ_conv_split(const uint32_t *u, const uint32_t *v, uint32_t *w, int32_t log2L,
                             int64_t batch, uint32_t p, void *stream) {
    if (log2L < 1 || log2L > 30 || batch < 0)
        return fail(MC_EINVAL, "length must be a power of two >= 2");
    SplitParams S;
    memset(&S, 0, sizeof(S));
    mc_status s = split_setup(p, log2L, &S);  // psi = w_L, L = 2n
    if (s != MC_OK || batch == 0) return s;
    if (!u || !v || !w) return fail(MC_EINVAL, "null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    const int log2n = log2L - 1;
    const long long n = 1ll << log2n;
    u32 *tmp = nullptr;
    keep_pool_memory();
    MC_CUDA_CHECK(cudaMallocAsync(&tmp, 4ull * 6 * n * batch, st));
    u32 *ua = tmp, *ub = ua + n * batch, *va = ub + n * batch, *vb = va + n * batch;
    u32 *ca = vb + n * batch, *cb = ca + n * batch;
    split_kernel<<<grid_for(n * batch), 256, 0, st>>>(u, 2 * n, ua, ub, log2n, batch, 1, S);
    split_kernel<<<grid_for(n * batch), 256, 0, st>>>(v, 2 * n, va, vb, log2n, batch, 1, S);
    s = circ_conv_dispatch(ua, va, ca, log2n, batch, p, st);  // mod x^n - 1
    if (s == MC_OK) s = circ_conv_dispatch(ub, vb, cb, log2n, batch, p, st);  // twisted: mod x^n + 1
    if (s == MC_OK)
        recombine_kernel<<<grid_for(n * batch), 256, 0, st>>>(ca, cb, w, 2 * n, log2n, batch, 1,
                                                              S);
    note_launches(3);
    cudaFreeAsync(tmp, st);
    MC_CUDA_CHECK(cudaGetLastError());
    return s;
}

}  // extern "C"
