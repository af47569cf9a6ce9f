// Instantiations of the fused small-L convolution kernel for one K
// (compiled once per K with -DMC_K=<K> so the 10 sizes build in parallel).
#include "conv_small.cuh"
#include "runtime.h"
#include "xform_small.cuh"

#ifndef MC_K
#error "compile with -DMC_K=<log2 L>"
#endif

namespace mc {

template <int NT, int AR, int FL>
static cudaError_t launch_nt_fl(const ConvSmallParams &P, cudaStream_t st) {
    using C = SmallCfg<MC_K>;
    auto kern = conv_small_kernel<MC_K, NT, AR, FL>;
    // dynamic shared memory: tables + data (+ TMA staging of both rows)
    const int smem = C::SMEM + (P.tma ? 16 + 4 * (P.za16 + P.zb16) : 0);
    struct Once { int attr_smem = 0, per_sm = 0, per_sm_smem = 0; };
    static PerDevice<Once> once;
    int &attr_smem = once.get().attr_smem, &per_sm = once.get().per_sm,
        &per_sm_smem = once.get().per_sm_smem;
    if (smem > attr_smem) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             smem);
        if (e != cudaSuccess) return e;
        attr_smem = smem;
    }
    if (per_sm_smem != smem) {
        int nb = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, C::THREADS, smem);
        if (e != cudaSuccess) return e;
        per_sm = nb > 0 ? nb : 1;
        per_sm_smem = smem;
    }
    // persistent grid: every resident CTA walks the batch with a grid stride
    long long grid = (P.batch + C::PPC - 1) / C::PPC;
    const long long cap = (long long)per_sm * sm_count();
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, C::THREADS, smem, st>>>(P);
    return cudaGetLastError();
}

// Feature flags: host I/O only where the bulk-copy paths exist (one product
// per CTA); the input reduction only on complete transforms (three primes).
template <int NT, int AR>
static cudaError_t launch_nt(const ConvSmallParams &P, cudaStream_t st) {
    constexpr bool one_per_cta = SmallCfg<MC_K>::PPC == 1;
    if (P.fold || P.wrap_m) {  // split truncated product: complete transforms, device rows
        if constexpr (NT == 16) {
            if (P.reduce || P.bulk_out || P.ready || (P.fold && P.wrap_m))
                return cudaErrorInvalidValue;
            if (P.twq_f) return launch_nt_fl<NT, AR, FL_TWIST>(P, st);
            return P.fold ? launch_nt_fl<NT, AR, FL_FOLD>(P, st)
                          : launch_nt_fl<NT, AR, FL_WRAP>(P, st);
        } else {
            return cudaErrorInvalidValue;
        }
    }
    if (P.reduce) {
        if constexpr (NT == 16) {
            if (P.bulk_out || P.ready) return cudaErrorInvalidValue;
            return launch_nt_fl<NT, AR, FL_REDUCE>(P, st);
        } else {
            return cudaErrorInvalidValue;
        }
    }
    if constexpr (one_per_cta) {
        if (P.bulk_out || P.ready) return launch_nt_fl<NT, AR, FL_HOST>(P, st);
    }
    return launch_nt_fl<NT, AR, 0>(P, st);
}

#define MC_CAT2(a, b) a##b
#define MC_CAT(a, b) MC_CAT2(a, b)

cudaError_t MC_CAT(launch_conv_small_k, MC_K)(const ConvSmallParams &P, int nt, cudaStream_t st) {
    // truncated transforms take the Harvey ranges too when p < 2^30 (P.ar = 1):
    // their pre-adds, cross butterflies and combines canonicalise their operands
    const bool lz = P.ar == 1;
    switch (nt) {
        case 9: return lz ? launch_nt<9, 1>(P, st) : launch_nt<9, 2>(P, st);
        case 10: return lz ? launch_nt<10, 1>(P, st) : launch_nt<10, 2>(P, st);
        case 11: return lz ? launch_nt<11, 1>(P, st) : launch_nt<11, 2>(P, st);
        case 12: return lz ? launch_nt<12, 1>(P, st) : launch_nt<12, 2>(P, st);
        case 13: return lz ? launch_nt<13, 1>(P, st) : launch_nt<13, 2>(P, st);
        case 14: return lz ? launch_nt<14, 1>(P, st) : launch_nt<14, 2>(P, st);
        case 15: return lz ? launch_nt<15, 1>(P, st) : launch_nt<15, 2>(P, st);
        case 16: return lz ? launch_nt<16, 1>(P, st) : launch_nt<16, 2>(P, st);
        default: return cudaErrorInvalidValue;
    }
}

// ---- standalone transforms (xform_small.cuh)
template <int MODE, int NT>
static cudaError_t launch_xf(const XformParams &X, cudaStream_t st) {
    using C = SmallCfg<MC_K>;
    auto kern = xform_small_kernel<MC_K, MODE, NT>;
    const int smem = C::L * 8 + C::PPC * C::L * 4;
    static PerDevice<int> per_sm_dev;
    int &per_sm = per_sm_dev.get();
    if (!per_sm) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        int nb = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, C::THREADS, smem);
        if (e != cudaSuccess) return e;
        per_sm = nb > 0 ? nb : 1;
    }
    long long grid = (X.batch + C::PPC - 1) / C::PPC;
    const long long cap = (long long)per_sm * sm_count();
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, C::THREADS, smem, st>>>(X);
    return cudaGetLastError();
}

cudaError_t MC_CAT(launch_xform_small_k, MC_K)(const XformParams &X, int mode, int nt,
                                               cudaStream_t st) {
    if (mode == MODE_NTT_FWD) return launch_xf<MODE_NTT_FWD, 16>(X, st);
    if (mode == MODE_NTT_INV) return launch_xf<MODE_NTT_INV, 16>(X, st);
    switch (nt) {
        case 9: return launch_xf<MODE_TFT, 9>(X, st);
        case 10: return launch_xf<MODE_TFT, 10>(X, st);
        case 11: return launch_xf<MODE_TFT, 11>(X, st);
        case 12: return launch_xf<MODE_TFT, 12>(X, st);
        case 13: return launch_xf<MODE_TFT, 13>(X, st);
        case 14: return launch_xf<MODE_TFT, 14>(X, st);
        case 15: return launch_xf<MODE_TFT, 15>(X, st);
        case 16: return launch_xf<MODE_TFT, 16>(X, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace mc
