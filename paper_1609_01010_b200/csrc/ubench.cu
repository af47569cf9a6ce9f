// Integer-pipe microbenchmarks: the denominators of the integer roofline
// reported beside the HBM one (configs 1-3 are integer-pipe bound).
// Each kernel runs 8 independent dependency chains per thread of one
// instruction kind; rate = lanes * instructions / (cycles * SMs).
#include <cstdint>
#include <cstdio>

#include "modarith.cuh"
#include "runtime.h"

namespace mc {

// mul_f64q_lazy (modarith.cuh): the FP64-quotient Shoup product.

template <int KIND>
__global__ void __launch_bounds__(256) ubench_kernel(u32 *out, u32 seed, int iters, u32 p,
                                                     u32 wp) {
    u32 x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = seed * (threadIdx.x + 1) + i * 0x9E3779B9u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (KIND == 0) x[i] = x[i] * p + wp;                       // IMAD
                if (KIND == 1) x[i] = __umulhi(x[i], wp) ^ p;              // IMAD.HI (+LOP)
                if (KIND == 2) x[i] = __viaddmin_u32(x[i], wp, x[i] ^ p);  // VIADDMNMX (+LOP)
                if (KIND == 3) x[i] = x[i] + wp - p;                       // IADD3
                if (KIND == 4) x[i] = mul_shoup(x[i], p - 7, wp, p);       // Shoup mul + red
                if (KIND == 5) {                                           // DIT butterfly
                    u32 a = x[i], b = x[(i + 1) & 7];
                    bfly_dit(a, b, p - 7, wp, p);
                    x[i] = a ^ b;
                }
                if (KIND == 6) {                                           // DFMA chain
                    double d = __hiloint2double((int)wp, (int)x[i]);
                    d = fma(d, 1.0000001, 0.5);
                    x[i] = (u32)__double2loint(d);
                }
                if (KIND == 7) {                                           // f64-quotient mul
                    x[i] = red1(mul_f64q_lazy(x[i], p - 7, (double)(p - 7) / p, p), p);
                }
            }
        }
    }
    u32 acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc ^= x[i];
    if (acc == 0x12345678u) out[0] = acc;  // keep the work live
}

// Butterfly variants of the pass benchmark (MODE):
//   0  bfly_dif as shipped (canonical values, two VIADDMNMX)
//   1  canonical, conditional subtractions as IADD3 + IMNMX (ALU pipe)
//   2  lazy (Harvey): values in [0, 2p), one VIADDMNMX; needs p < 2^30
//   3  lazy, its reduction as IADD3 + IMNMX
template <int MODE>
__device__ __forceinline__ void bfly_variant(u32 &a, u32 &b, u32 w, u32 wp, u32 p) {
    if (MODE == 0) {
        bfly_dif(a, b, w, wp, p);
    } else if (MODE == 1) {
        const u32 s = a + b, d = a - b + p;
        const u32 r = mul_shoup_lazy(d, w, wp, p);
        a = min(s, s - p);
        b = min(r, r - p);
    } else if (MODE == 2) {
        const u32 s = __viaddmin_u32(a, b, a + b - 2 * p);
        b = mul_shoup_lazy(a - b + 2 * p, w, wp, p);
        a = s;
    } else if (MODE == 3) {
        const u32 s = a + b;
        b = mul_shoup_lazy(a - b + 2 * p, w, wp, p);
        a = min(s, s - 2 * p);
    } else {  // MODE 4: canonical, quotient on the FP64 pipe (wp holds an index)
        const u32 s = a + b;
        const u32 r = mul_f64q_lazy(a - b + p, w, __longlong_as_double(
            ((long long)wp << 32) | w), p);
        a = min(s, s - p);
        b = min(r, r - p);
    }
}

// A radix-16 DIF register pass on two operands (32 butterflies each, one
// LDS.64 twiddle per butterfly) repeated `iters` times with no exchange and
// no barrier: the butterfly stream of conv_small_kernel in isolation.
// MIX > 0: the MIX lowest levels of each pass take the FP64-quotient
// product (MODE 4), the others MODE: can the FP64 pipe relieve the
// FMA-heavy one for a share of the butterflies?
template <int MINB, int MODE, int MIX = 0>
__global__ void __launch_bounds__(256, MINB) pass_bench_kernel(const uint2 *tw_g, u32 *out,
                                                                int iters, u32 p) {
    __shared__ uint2 tw[4096];
    for (int i = threadIdx.x; i < 4096; i += 256) tw[i] = tw_g[i];
    __syncthreads();
    const int t = threadIdx.x;
    u32 va[16], vb[16];
#pragma unroll
    for (int s = 0; s < 16; ++s) {
        va[s] = (t * 2654435761u + s * 40503u) % p;
        vb[s] = (t * 2246822519u + s * 97u) % p;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int lv = 3; lv >= 0; --lv) {
            const int H = 1 << lv;
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                if (s & H) continue;
                const uint2 w = tw[(H * 256 + t + 16 * (s & (2 * H - 1))) & 4095];
                if (lv < MIX) {
                    bfly_variant<4>(va[s], va[s + H], w.x, w.y, p);
                    bfly_variant<4>(vb[s], vb[s + H], w.x, w.y, p);
                } else {
                    bfly_variant<MODE>(va[s], va[s + H], w.x, w.y, p);
                    bfly_variant<MODE>(vb[s], vb[s + H], w.x, w.y, p);
                }
            }
        }
    }
    u32 acc = 0;
#pragma unroll
    for (int s = 0; s < 16; ++s) acc ^= va[s] ^ vb[s];
    if (acc == 0x12345678u) out[0] = acc;
}

}  // namespace mc

extern "C" {

// Butterflies per clock per SM of the isolated register pass:
// rates[0] MODE 0 at 2 CTAs/SM, rates[1] MODE 0 at 4 CTAs/SM,
// rates[2..5] MODES 1..4 at 2 CTAs/SM (see bfly_variant), rates[6..8] MODE 0
// with the 1, 2 or 3 lowest levels of each pass on the FP64-quotient product.
mc_status mc_ubench_pass(double *rates) {
    using namespace mc;
    const int sms = sm_count();
    int dev = current_device(), clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    const u32 p = 998244353u;  // < 2^30: valid for the lazy modes too
    uint2 *tw = nullptr;
    u32 *out = nullptr;
    MC_CUDA_CHECK(cudaMalloc(&tw, 4096 * sizeof(uint2)));
    MC_CUDA_CHECK(cudaMalloc(&out, 4));
    {
        uint2 h[4096];
        for (int i = 0; i < 4096; ++i) {
            Shoup s = shoup((u32)((i * 7919ull + 1) % p), p);
            h[i] = make_uint2(s.w, s.wp);
        }
        MC_CUDA_CHECK(cudaMemcpy(tw, h, sizeof(h), cudaMemcpyHostToDevice));
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 200;
    for (int k = 0; k < 9; ++k) {
        const int per_sm = k == 1 ? 4 : 2;
        const int blocks = sms * per_sm;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            switch (k) {
                case 0: pass_bench_kernel<2, 0><<<blocks, 256>>>(tw, out, iters, p); break;
                case 1: pass_bench_kernel<4, 0><<<blocks, 256>>>(tw, out, iters, p); break;
                case 2: pass_bench_kernel<2, 1><<<blocks, 256>>>(tw, out, iters, p); break;
                case 3: pass_bench_kernel<2, 2><<<blocks, 256>>>(tw, out, iters, p); break;
                case 4: pass_bench_kernel<2, 3><<<blocks, 256>>>(tw, out, iters, p); break;
                case 5: pass_bench_kernel<2, 4><<<blocks, 256>>>(tw, out, iters, p); break;
                case 6: pass_bench_kernel<2, 0, 1><<<blocks, 256>>>(tw, out, iters, p); break;
                case 7: pass_bench_kernel<2, 0, 2><<<blocks, 256>>>(tw, out, iters, p); break;
                case 8: pass_bench_kernel<2, 0, 3><<<blocks, 256>>>(tw, out, iters, p); break;
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bf = (double)blocks * 256 * iters * 64;
        rates[k] = bf / (ms * 1e-3 * clk_khz * 1e3) / sms;
    }
    cudaFree(tw);
    cudaFree(out);
    MC_CUDA_CHECK(cudaGetLastError());
    return MC_OK;
}

// rates[k] = thread-level operations per clock per SM for kind k
// (0 IMAD, 1 IMAD.HI, 2 VIADDMNMX, 3 IADD3, 4 Shoup mul, 5 DIT butterfly),
// measured at the current SM clock (sm_mhz[0] receives the clock used).
mc_status mc_ubench_int_pipes(double *rates, int nkinds, double *sm_mhz) {
    using namespace mc;
    int dev = current_device();
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    const int sms = sm_count();
    u32 *out = nullptr;
    MC_CUDA_CHECK(cudaMalloc(&out, 4));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 512, blocks = sms * 8, threads = 256;
    const u32 p = 2013265921u;
    const u32 wp = (u32)(((u64)(p - 7) << 32) / p);
    for (int k = 0; k < nkinds && k < 8; ++k) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            switch (k) {
                case 0: ubench_kernel<0><<<blocks, threads>>>(out, 7, iters, p, wp); break;
                case 1: ubench_kernel<1><<<blocks, threads>>>(out, 7, iters, p, wp); break;
                case 2: ubench_kernel<2><<<blocks, threads>>>(out, 7, iters, p, wp); break;
                case 3: ubench_kernel<3><<<blocks, threads>>>(out, 7, iters, p, wp); break;
                case 4: ubench_kernel<4><<<blocks, threads>>>(out, 7, iters, p, wp); break;
                case 5: ubench_kernel<5><<<blocks, threads>>>(out, 7, iters, p, wp); break;
                case 6: ubench_kernel<6><<<blocks, threads>>>(out, 7, iters, p, wp); break;
                case 7: ubench_kernel<7><<<blocks, threads>>>(out, 7, iters, p, wp); break;
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = (double)blocks * threads * iters * 16 * 8;
        const double cycles = ms * 1e-3 * (clk_khz * 1e3);
        rates[k] = ops / cycles / sms;
    }
    if (sm_mhz) *sm_mhz = clk_khz / 1e3;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    MC_CUDA_CHECK(cudaGetLastError());
    return MC_OK;
}

}  // extern "C"
