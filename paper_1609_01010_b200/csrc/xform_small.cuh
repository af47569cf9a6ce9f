// Fused single-CTA standalone transforms for 16 <= L = 2^K <= 8192
// (SURVEY.md 8f row 1): the register passes of conv_small.cuh on one operand.
//   MODE_NTT_FWD  moddft forward   (transform.py:167-196): natural in, natural out
//   MODE_NTT_INV  moddft inverse   (same, scaled by 1/L):  natural in, natural out
//   MODE_TFT      tft              (transform.py:421-448): first n values of the
//                 bit-reversed spectrum of the zero-extended input, n > L/2
// The DIF forward leaves position x holding X[rev_K(x)]; natural order is
// one shared-memory permutation away (stores stay coalesced).  The inverse
// permutes its natural input into bit-reversed positions and runs the DIT.
// itft keeps the level-scheduled kernels (transforms.cu): its exact
// truncation below the G-block needs the full-granularity recursion.
#pragma once
#include "conv_small.cuh"

namespace mc {

enum { MODE_NTT_FWD = 0, MODE_NTT_INV = 1, MODE_TFT = 2 };

struct XformParams {
    ConvSmallParams cs;  // p, stage tables, lowest-pass constants
    const u32 *x;
    long long ldx;
    u32 *y;
    long long ldy;
    int z, n;            // input words (zero-extended to L), output words
    long long batch;
    Shoup linv;          // 1/L (inverse)
    u32 red_wp;          // floor(2^32 / p): inputs reduced on load
};

template <int K>
__device__ __forceinline__ int brev_k(int x) {
    return (int)(__brev((unsigned)x) >> (32 - K));
}

template <int K, int MODE, int NT>
__global__ void __launch_bounds__(SmallCfg<K>::THREADS, SmallCfg<K>::MINB)
xform_small_kernel(const XformParams X) {
    using C = SmallCfg<K>;
    constexpr int L = C::L, T = C::T, G = L / 16;
    extern __shared__ uint4 smem_raw[];
    uint2 *tab = reinterpret_cast<uint2 *>(smem_raw);  // tf (forward) or ti (inverse)
    u32 *data = reinterpret_cast<u32 *>(tab + L);
    {
        const uint4 *g = reinterpret_cast<const uint4 *>(MODE == MODE_NTT_INV ? X.cs.ti : X.cs.tf);
        for (int i = threadIdx.x; i < L / 2; i += C::THREADS)
            reinterpret_cast<uint4 *>(tab)[i] = __ldg(g + i);
    }
    const Tw W{tab, tab};
    const int grp = threadIdx.x / T;
    const int t = threadIdx.x % T;
    u32 *buf = data + grp * L;
    const u32 p = X.cs.p;
    mc_sync();
    constexpr int SBL = last_sb<K>();
    for (long long base = (long long)blockIdx.x * C::PPC; base < X.batch;
         base += (long long)gridDim.x * C::PPC) {
        const long long row = base + grp;
        const bool valid = row < X.batch;
        const u32 *gx = X.x + (valid ? row : 0) * X.ldx;
        u32 *gy = X.y + (valid ? row : 0) * X.ldy;
        u32 v[16];
        if constexpr (MODE == MODE_NTT_INV) {
            // natural spectrum -> position rev(k) (the DIT's bit-reversed input)
            mc_sync();  // the previous row is done with buf
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                const int k = t + G * s;
                buf[swz_xf(brev_k<K>(k))] = valid ? mul_shoup(__ldcs(gx + k), 1u, X.red_wp, p) : 0u;
            }
            mc_sync();
#pragma unroll
            for (int s = 0; s < 16; ++s) v[s] = buf[swz_xf(slot_pos<SBL>(t, s))];
            inv_lower_chain1<K, Plan<K>::NP - 1, LayXf, 16>(buf, v, t, X.cs, W, LayXf());
            ItftTop<K, 16, 16, 0>::run(v, t, X.cs, W);
            if (valid) {
#pragma unroll
                for (int s = 0; s < 16; ++s) __stcs(gy + t + G * s, mul_shoup(v[s], X.linv, p));
            }
        } else {
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                const int x = t + G * s;
                v[s] = (valid && x < X.z) ? mul_shoup(__ldcs(gx + x), 1u, X.red_wp, p) : 0u;
            }
            fwd_top<K, NT>(v, X.z, t, X.cs, W);
            fwd_lower_chain1<K, 0, LayXf, NT>(buf, v, t, X.cs, W, LayXf());
            // v[s] = X[rev(x)] at x = slot_pos<SBL>(t, s); stage it for a coalesced store
            mc_sync();
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                const int x = slot_pos<SBL>(t, s);
                if (NT >= 16 || (x >> (K - 4)) < NT)
                    buf[swz_xf(MODE == MODE_NTT_FWD ? brev_k<K>(x) : x)] = v[s];
            }
            mc_sync();
            if (valid) {
#pragma unroll
                for (int s = 0; s < 16; ++s) {
                    const int x = t + G * s;
                    if (MODE == MODE_NTT_FWD || x < X.n) __stcs(gy + x, buf[swz_xf(x)]);
                }
            }
        }
    }
}

}  // namespace mc
