// Internal definitions shared by the four-step compilation units
// (fourstep.cu: row pass + orchestration; fourstep_cols.cu: column passes,
// one unit per column size KR).
#pragma once
#include <cuda.h>

#include "conv_small.cuh"
#include "fourstep.cuh"

namespace mc {

// Twiddle powers w_L^e for any e < L: lo[e & 4095] (plain) times hi[e >> 12]
// (Shoup pair).  Forward (w) and inverse (w^-1) sets.
struct TwistTabs {
    const u32 *lo_f;
    const uint2 *hi_f;
    const u32 *lo_i;
    const uint2 *hi_i;
    double two32_over_p;  // 2^32 / p, for Shoup companions computed on the fly
};

struct FourParams {
    ConvSmallParams cs;  // p, pinv, linv_mont (for the full L), level constants
    const u32 *a;
    const u32 *b;
    u32 *c;
    long long lda, ldb, ldc;
    long long z1, z2, n;
    u32 *Ah;  // scratch: [chunk][L] transformed a, later the product spectrum
    u32 *Bh;  // scratch: [chunk][L] transformed b
    long long prod0;  // first product of this chunk
    int chunk;
    int reduce;  // inputs are arbitrary words: reduce mod p on load
    u32 red_wp;  // floor(2^32 / p)
    TwistTabs tw;
    const uint2 *col_tf, *col_ti;  // stage tables for the R-point column transforms
    const uint2 *row_tf, *row_ti;  // stage tables for the C-point row transforms
    const uint2 *row_tm;           // merged stage table of the row transforms (TwM)
    long long nrows;  // rows of each product the row pass transforms (NT * R/16)
    // twist tables [R][C] (row_conv_kernel<.., TT = true>): twf[r][x] =
    // w_L^(x * rev(r)), twi[r][x] = w_L^-(x * rev(r)) * L^-1 * 2^32, Shoup pairs
    const uint2 *twf, *twi;
    int row_prefetch;  // L2 bulk prefetch of the next row (the row pass's data exceeds L2)
    int fold;  // split truncated product head: operands longer than L fold x + L onto x
    // Column passes on 8K-word tiles, two columns per thread, two CTAs per SM
    // (kSmallColTile) instead of 16K-word tiles: chosen when a chunk's spectra
    // stay in L2, where the 16-byte row segments of the narrower tiles cost
    // nothing (config 5: 121.0 -> 117.0 us; config 4, DRAM-resident: 1.04 -> 1.44 ms)
    int small_tiles;
};

constexpr int kSmallColTile = 8192;

// Column rotation of the product spectrum.  The row pass writes spectrum
// column x of (global) product g to scratch column (x + rot) mod C with rot =
// the word offset of g's output row modulo 8; the inverse column pass then
// maps its tile columns back, so that the 8-word row segments of every tile
// but one start on a 32-byte sector of the output even when the rows are not
// 16-byte aligned (ld = n, odd).  Measured on config 4: sector-aligned output
// rows run the step 5% faster (scripts/out_layout_ab.py).
__device__ __forceinline__ int out_rot(const FourParams &P, long long g) {
    return P.c ? (int)((((unsigned long long)(uintptr_t)P.c >> 2) + (unsigned long long)g * P.ldc) & 7)
               : 0;
}

__device__ __forceinline__ u32 pow_w(const u32 *lo, const uint2 *hi, u32 e, u32 p) {
    const uint2 h = __ldg(hi + (e >> 12));
    return mul_shoup(__ldg(lo + (e & 4095)), h.x, h.y, p);
}

// floor(w * 2^32 / p) via a double estimate and one exact correction step.
__device__ __forceinline__ u32 shoup_comp(u32 w, u32 p, double two32_over_p) {
    u32 q = __double2uint_rz((double)w * two32_over_p);
    long long r = (long long)(((unsigned long long)w << 32) - (unsigned long long)q * p);
    if (r < 0) --q;
    else if (r >= (long long)p) ++q;
    return q;
}


#ifndef MC_COL_TILE
#define MC_COL_TILE 16384
#endif

// Column tile: R rows x TC columns = MC_COL_TILE words, one 16-slot column
// transform per R/16 threads.  16K-word tiles (1024 threads, 1 CTA/SM)
// measured faster than 8K tiles with 2 CTAs/SM (narrower row segments cost
// more than the load/compute overlap gained).
template <int KR, int TL = MC_COL_TILE>
struct ColCfg {
    static constexpr int R = 1 << KR;
    static constexpr int TILE = TL;
    static constexpr int TC = TILE >> KR;  // columns per tile
    static constexpr int THREADS = TILE / 16;
    static constexpr int G = R / 16;
    static constexpr int MINB = THREADS >= 1024 ? 1 : 2;
    // both column stage tables (the truncated inverse needs w and w^-1) + tile
    static constexpr int SMEM = 2 * R * 8 + TILE * 4;
};

// TMA path of the forward column pass: 3-D tensor maps over the operands
// ({C columns, z/C rows, batch}); rows beyond z/C are zero-filled by TMA.
struct ColTma {
    CUtensorMap ma, mb;
    int ok;  // 0: fall back to the load/store kernel
};

// Column passes for one KR; NT = active top blocks of the column transform
// (16 = full; < 16 = truncated: rows >= NT*R/16 are never formed).
cudaError_t launch_cols_kr4(const FourParams &P, int KC, int NT, bool fwd, cudaStream_t st,
                            const ColTma *tma = nullptr);
cudaError_t launch_cols_kr5(const FourParams &P, int KC, int NT, bool fwd, cudaStream_t st,
                             const ColTma *tma = nullptr);
cudaError_t launch_cols_kr6(const FourParams &P, int KC, int NT, bool fwd, cudaStream_t st,
                             const ColTma *tma = nullptr);
cudaError_t launch_cols_kr7(const FourParams &P, int KC, int NT, bool fwd, cudaStream_t st,
                             const ColTma *tma = nullptr);
cudaError_t launch_cols_kr8(const FourParams &P, int KC, int NT, bool fwd, cudaStream_t st,
                             const ColTma *tma = nullptr);
cudaError_t launch_cols_kr9(const FourParams &P, int KC, int NT, bool fwd, cudaStream_t st,
                             const ColTma *tma = nullptr);
cudaError_t launch_cols_kr10(const FourParams &P, int KC, int NT, bool fwd, cudaStream_t st,
                             const ColTma *tma = nullptr);
cudaError_t launch_cols_kr11(const FourParams &P, int KC, int NT, bool fwd, cudaStream_t st,
                             const ColTma *tma = nullptr);
cudaError_t launch_cols_kr12(const FourParams &P, int KC, int NT, bool fwd, cudaStream_t st,
                             const ColTma *tma = nullptr);
cudaError_t launch_cols_kr13(const FourParams &P, int KC, int NT, bool fwd, cudaStream_t st,
                             const ColTma *tma = nullptr);

// One four-step convolution set up for launching (fourstep.cu): tables,
// twists and constants for one prime; the caller provides the scratch
// (P.Ah, P.Bh: 2L words per product of a chunk).
struct FourPlan {
    FourParams P;
    int K = 0, KC = 0, KR = 0, NT = 16;
    long long L = 0, batch = 0;
    ColTma tma;
};

mc_status fourstep_plan(int engine, const u32 *a, long long lda, int z1, const u32 *b,
                        long long ldb, int z2, u32 *c, long long ldc, long long batch, u32 p,
                        int circ_log2L, bool reduce_inputs, FourPlan *F);
// forward column pass + fused row pass of products [p0, p0 + chunk)
cudaError_t fourstep_fwd_rows(FourPlan &F, long long p0, int chunk, cudaStream_t st);
// inverse column pass of the chunk last given to fourstep_fwd_rows
cudaError_t fourstep_inv_cols(FourPlan &F, cudaStream_t st);

template <class KF>
static cudaError_t prep_kernel(KF kern, int smem, int threads, int *per_sm) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (per_sm) {
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kern, threads, smem);
        if (*per_sm < 1) *per_sm = 1;
    }
    return e;
}

}  // namespace mc
