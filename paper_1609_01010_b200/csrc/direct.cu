// Definition engine: convolution straight from its defining sum,
//   linear    c_k = sum_{i+j=k}        a_i b_j  mod p   (convolve.py:71-87 lin_conv_def,
//                                                       poly.py:90-105 schoolbook_raw)
//   circular  c_k = sum_{i+j=k mod n}  a_i b_j  mod p   (convolve.py:54-68 circ_conv_def)
// for any modulus 2 <= p < 2^31.  No roots of unity are involved, so this is
// the engine for products whose transform size exceeds the field's 2-adicity
// (the reference's "definition" engine keeps working there; e.g. p = 7,
// tests/test_convolve.py:62, or the p = 17 sweep rows of tests/test_cli.py:178).
//
// One thread per output coefficient, 256 outputs per CTA.  The operand a is
// staged 256 words at a time (read as a broadcast), b as the matching
// 511-word window (consecutive words across the warp), both zero outside
// their rows, so no thread needs its own summation bounds.  Products are
// accumulated exactly as two 64-bit sums of their low and high words
// (IMAD + IMAD.HI + two 64-bit adds) and reduced once at the end.
#include "runtime.h"
#include "tma.cuh"

namespace mc {

constexpr int kDirTile = 256;

__global__ void __launch_bounds__(kDirTile) direct_conv_kernel(
    const u32 *a, long long lda, int z1, const u32 *b, long long ldb, int z2, u32 *c,
    long long ldc, int n, int circ, u32 p, u32 r32) {
    __shared__ u32 sa[kDirTile];
    __shared__ u32 sb[2 * kDirTile];
    const long long row = blockIdx.y;
    const u32 *ar = a + row * lda, *br = b + row * ldb;
    const int k0 = blockIdx.x * kDirTile, t = threadIdx.x, k = k0 + t;
    // a-chunks that can meet an output of this tile
    int i_lo = 0, i_hi = z1;  // [i_lo, i_hi)
    if (!circ) {
        i_lo = max(0, k0 - (z2 - 1));
        i_hi = min(z1, k0 + kDirTile);
    }
    unsigned long long s_lo = 0, s_hi = 0;
    for (int i0 = i_lo; i0 < i_hi; i0 += kDirTile) {
        mc_sync();
        sa[t] = (i0 + t < i_hi) ? ar[i0 + t] : 0u;
        // sb[x] = b[k0 - i0 - (kDirTile - 1) + x]: output k = k0 + t and a index
        // i0 + ii meet b[k - i0 - ii] = sb[t - ii + kDirTile - 1]
        for (int x = t; x < 2 * kDirTile - 1; x += kDirTile) {
            long long j = (long long)k0 - i0 - (kDirTile - 1) + x;
            u32 w = 0;
            if (circ) {
                j %= n;
                if (j < 0) j += n;
                w = br[j];
            } else if (j >= 0 && j < z2) {
                w = br[j];
            }
            sb[x] = w;
        }
        mc_sync();
#pragma unroll 8
        for (int ii = 0; ii < kDirTile; ++ii) {
            const u32 x = sa[ii], y = sb[t - ii + kDirTile - 1];
            s_lo += (unsigned long long)(x * y);
            s_hi += (unsigned long long)__umulhi(x, y);
        }
    }
    if (k < n) {
        const unsigned long long r =
            ((s_hi % p) * (unsigned long long)r32 + s_lo % p) % p;
        c[row * ldc + k] = (u32)r;
    }
}

}  // namespace mc

using namespace mc;

extern "C" {

mc_status mc_conv_direct(const uint32_t *a, int64_t lda, int32_t z1, const uint32_t *b,
                         int64_t ldb, int32_t z2, uint32_t *c, int64_t ldc, int64_t batch,
                         uint32_t p, int32_t circ, void *stream) {
    if (z1 < 1 || z2 < 1) return fail(MC_EINVAL, "inputs must be nonempty");
    if (circ && z1 != z2) return fail(MC_EINVAL, "circular convolution needs equal lengths");
    if (p < 2 || p >= (1u << 31)) return fail(MC_EUNSUPPORTED, "modulus must be in [2, 2^31)");
    if (batch < 0 || batch > 65535) return fail(MC_EINVAL, "batch must be in [0, 65535]");
    const long long n = circ ? z1 : (long long)z1 + z2 - 1;
    if (n > 0x7fffffffll - kDirTile) return fail(MC_EINVAL, "product too long");
    if (lda < z1 || ldb < z2 || ldc < n) return fail(MC_EINVAL, "bad leading dimension");
    if (batch == 0) return MC_OK;
    if (!a || !b || !c) return fail(MC_EINVAL, "null pointer");
    const u32 r32 = (u32)((1ull << 32) % p);
    dim3 grid((unsigned)((n + kDirTile - 1) / kDirTile), (unsigned)batch);
    direct_conv_kernel<<<grid, kDirTile, 0, (cudaStream_t)stream>>>(
        a, lda, z1, b, ldb, z2, c, ldc, (int)n, circ ? 1 : 0, p, r32);
    note_launches(1);
    MC_CUDA_CHECK(cudaGetLastError());
    return MC_OK;
}

}  // extern "C"
