// Probe: does IMAD.WIDE (32 x 32 + 64 -> 64) issue at the IMAD rate or at the
// IMAD.HI rate on sm_100a?  If a wide product cost one IMAD slot, Shoup's
// quotient could come from its upper half and the butterfly would need 3
// FMA-heavy slots instead of 4.  8 independent chains per thread, as in
// csrc/ubench.cu.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_wide ubench_wide.cu
#include <cstdint>
#include <cstdio>
typedef uint32_t u32;
typedef unsigned long long u64;

template <int KIND>
__global__ void __launch_bounds__(256) k(u32 *out, u32 seed, int iters, u32 p, u32 wp) {
    u32 x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = seed * (threadIdx.x + 1) + i * 0x9E3779B9u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (KIND == 0) x[i] = x[i] * p + wp;           // IMAD
                if (KIND == 1) x[i] = __umulhi(x[i], wp) ^ p;  // IMAD.HI + LOP3
                if (KIND == 2) {                                // IMAD.WIDE + LOP3 (both halves used)
                    u32 lo, hi;
                    asm volatile("{ .reg .b64 t; mul.wide.u32 t, %2, %3; mov.b64 {%0, %1}, t; }"
                                 : "=r"(lo), "=r"(hi) : "r"(x[i]), "r"(wp));
                    x[i] = lo ^ hi;
                }
                if (KIND == 3) {                                // IMAD.WIDE with 64-bit addend
                    u32 lo, hi;
                    asm volatile("{ .reg .b64 t, a; mov.b64 a, {%2, %3}; mad.wide.u32 t, %2, %4, a; "
                                 "mov.b64 {%0, %1}, t; }"
                                 : "=r"(lo), "=r"(hi) : "r"(x[i]), "r"(p), "r"(wp));
                    x[i] = lo ^ hi;
                }
            }
        }
    }
    u32 acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc ^= x[i];
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    int dev = 0, sms = 0, khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
    u32 *out;
    cudaMalloc(&out, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 512, blocks = sms * 8, threads = 256;
    const u32 p = 2013265921u, wp = 4294967281u;
    const char *names[4] = {"IMAD", "IMAD.HI+LOP3", "IMAD.WIDE+LOP3", "IMAD.WIDE(+64)+LOP3"};
    for (int kind = 0; kind < 4; ++kind) {
        float ms = 0;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            if (kind == 0) k<0><<<blocks, threads>>>(out, 7, iters, p, wp);
            if (kind == 1) k<1><<<blocks, threads>>>(out, 7, iters, p, wp);
            if (kind == 2) k<2><<<blocks, threads>>>(out, 7, iters, p, wp);
            if (kind == 3) k<3><<<blocks, threads>>>(out, 7, iters, p, wp);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        const double ops = (double)blocks * threads * iters * 16 * 8;
        printf("%-22s %.1f thread-ops/clk/SM\n", names[kind], ops / (ms * 1e-3 * khz * 1e3) / sms);
    }
    printf("cuda error: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
