// Fused single-CTA convolution kernel for transform sizes 16 <= L <= 8192
// (configs 1-3): forward transform of both operands, pointwise product with
// L^-1 folded in, inverse transform, all in registers + shared memory, one
// HBM read of each operand and one HBM write of the product.
//
// Replaces, per product row:
//   fft_pad: convolve.py:160-169 -> :143-157 (moddft x3 + _pointwise)
//   tft:     convolve.py:230-253 (tft x2 + _pointwise + itft + scale)
//
// Layout.  L = 2^K, G = L/16.  A product is owned by T = G threads, each
// holding 16 "slots" per operand in registers.  Position bits are processed
// in passes of <= 4 bits (radix-16 register passes): the top pass owns bits
// [K-4, K) (thread t holds x = t + G*s), lower passes own 4-bit windows
// [SB, SB+4) of lower bits.  Between passes the slots go through shared
// memory under the XOR swizzle swz() that makes every pass's 32-lane access
// hit 32 distinct banks.  Global loads/stores happen in the top-pass layout:
// for each slot a warp touches 32 consecutive words (128 B).
//
// Transforms.  Forward = decimation in frequency (natural in, bit-reversed
// out, the order of the reference TFT, transform.py:379-418) with direct
// per-stage twiddles tf[h + j] = w_{2h}^j; inverse = decimation in time on
// bit-reversed input with ti[h + j] = w_{2h}^-j (transform.py:150-164 run on
// the bit-reversed spectrum).  No bit-reversal permutation is ever done.
//
// Truncation (tft engine, and zero padding in both engines).  The top pass
// prunes butterflies exactly as the reference recursion does (known-zero
// inputs: position offset within its block >= z; unneeded outputs: block
// start >= n').  Truncation is "relaxed" to the G-block: n' = NT*G with
// NT = ceil(n/G) in [9, 16]; G-blocks >= NT are skipped by every lower pass
// and their spectral values are never formed.  The inverse runs the complete
// inverse DIT on the NT active G-blocks (lower passes), then the
// van der Hoeven inverse truncated recursion (transform.py:451-489) over the
// top 4 levels with base case m == G, fully unrolled for the compile-time NT.
// The product is exact either way (u_j = 0 for j >= n >= ... ), so the
// output equals the reference's bit for bit; see tests/kernel_model.py for
// the position-level model checked against the oracle.
#pragma once
#include <type_traits>

#include "modarith.cuh"
#include "tma.cuh"

namespace mc {

// Largest transform size of the fused single-CTA kernels (L = 2^13).
constexpr int kSmallMaxK = 13;

struct ConvSmallParams {
    const u32 *a;
    const u32 *b;
    u32 *c;
    long long lda, ldb, ldc;
    int z1, z2, n;
    long long batch;
    u32 p, pinv;
    Shoup linv_mont;   // L^-1 * 2^32 mod p
    const uint2 *tf;   // forward stage twiddles
    const uint2 *ti;   // inverse stage twiddles
    Shoup mlev[5];     // [l] = (2^l * G) mod p, l = 1..4  (m of a top level)
    Shoup hinv[5];     // [l] = (2^(l-1) * G)^-1 mod p    (1/h of a top level)
    int reduce;        // inputs are arbitrary words: reduce mod p on load
    u32 red_wp;        // floor(2^32 / p)
    int tma;           // prefetch operand rows with cp.async.bulk (1 product per CTA,
                       // 16-byte aligned rows); staging follows the data buffers
    int za16, zb16;    // words of a / b rows covered by the bulk copies (multiple of 4)
    uint2 c16f[16];    // tf[1..15] / ti[1..15]: the thread-invariant twiddles of the
    uint2 c16i[16];    // lowest pass (h <= 8), read from the constant bank
    double c16fd[16];  // RD(w / p) of the same twiddles (FP64-quotient products, MC_F64Q)
    double c16id[16];
    int ar;            // arithmetic mode of the launch (modarith.cuh): 1 or 2
    int bulk_out;      // write product rows by bulk copies from shared memory (PPC == 1;
                       // zero-copy host output)
    const uint32_t *ready;  // streamed inputs (PPC == 1 with TMA): rows of chunk i are
    uint32_t epoch;         // resident once ready[i] == epoch (set by the copy stream)
    int ready_rows;         // products per chunk
    // Split truncated product (tft engine, n = L/2 + m with m <= L/8; capi.cu
    // conv_dispatch): the head launch (fold) forms c mod (x^(L/2) - 1) from
    // operands folded on load, the tail launch (wrap_m = m) forms the low
    // product and unwraps: c[x] = low[x], c[wrap_off + x] = c0[x] - low[x].
    int fold;      // FL_FOLD launch: rows longer than L fold x + L onto x
    int wrap_m;    // FL_WRAP / FL_TWIST launch: coefficients to unwrap (n - L'/2)
    int wrap_off;  // FL_WRAP / FL_TWIST launch: half length L'/2 of the full product transform
    // FL_TWIST launch (quarter piece, L = L'/4 of the full transform L'): the
    // operands' true lengths, w_L'^x / w_L'^-x (the full transform's top-stage
    // tables, entries L'/2 + x), i = w_L'^(L'/4) and 1/2
    int tz1, tz2;
    const uint2 *twq_f, *twq_i;
    Shoup qi, qhalf;
};

// Shared-memory swizzle of the exchanges: XOR of position bits [2,5) with
// bits 4-6 and 8, a permutation of every aligned 32-word row that keeps each
// aligned quad of positions together (bits 0-1 untouched).  Conflict-free
// for every exchange pattern of the register passes: scalar accesses with
// lanes -> position bits [0,5) (top-pass and SB = 8 layouts) or [0,4) + {8}
// (SB = 4), and 16-byte vector accesses in the SB = 0 layout, where a thread
// holds 16 consecutive positions (four LDS.128 / STS.128 instead of 16
// scalar ones; every quarter-warp hits 8 distinct 16-byte bank groups).
__device__ __forceinline__ int swz(int x) { return x ^ ((((x >> 4) & 7) << 2) ^ ((x >> 4) & 16)); }

// Scalar-only swizzle (XOR of bits [0,5) with bits 5-8): conflict-free for
// lanes -> bits [0,5), [4,9), [0,4) + {8} with scalar accesses, and for the
// bit-reversal permutations of the standalone transforms (xform_small.cuh).
__device__ __forceinline__ int swz_xf(int x) { return x ^ (((x >> 5) & 15) | ((x >> 4) & 16)); }

template <int SB>
__device__ __forceinline__ int slot_pos(int t, int s) {
    return ((t >> SB) << (SB + 4)) | (s << SB) | (t & ((1 << SB) - 1));
}

// Twiddles are read from the CTA's shared-memory copy of the stage tables:
// one LDS.64 [Rt + imm] per twiddle (Rt = 8*t precomputed).
__device__ __forceinline__ uint2 ldtw(const uint2 *tab, int i) { return tab[i]; }

struct Tw {
    const uint2 *tf;  // shared-memory copy of P.tf
    const uint2 *ti;  // shared-memory copy of P.ti
    static constexpr bool kNeg = false;
};

// Merged stage table (half the shared memory of tf + ti): stage h = 2^lg
// holds w_{2h}^k for k = 0..h at m[h + lg - 1 + k].  Forward twiddle
// w_{2h}^j = m[h + lg - 1 + j]; inverse twiddle w_{2h}^-j = -w_{2h}^(h-j) =
// -m[2h + lg - 1 - j] (j = 0 reads w_{2h}^h = -1), so the inverse butterflies
// take the mirrored entry and swap their outputs (bfly_dit_neg_t).  Lanes read
// consecutive (or reverse-consecutive) entries, so the accesses stay
// conflict-free.
struct TwM {
    const uint2 *m;
    static constexpr bool kNeg = true;
};

__device__ __forceinline__ uint2 tw_fwd(const Tw &W, int h, int, int j) { return W.tf[h + j]; }
__device__ __forceinline__ uint2 tw_fwd(const TwM &W, int h, int lg, int j) {
    return W.m[h + lg - 1 + j];
}
__device__ __forceinline__ uint2 tw_inv(const Tw &W, int h, int, int j) { return W.ti[h + j]; }
__device__ __forceinline__ uint2 tw_inv(const TwM &W, int h, int lg, int j) {
    return W.m[2 * h + lg - 1 - j];
}

template <int AR, class TW>
__device__ __forceinline__ void bfly_dit_tw(u32 &a, u32 &b, uint2 w, u32 p) {
    if constexpr (TW::kNeg) bfly_dit_neg_t<AR>(a, b, w.x, w.y, p);
    else bfly_dit_t<AR>(a, b, w.x, w.y, p);
}

// ---------------------------------------------------------------- top pass (forward)
// Stages with half-size h = H*G, H = 8, 4, 2, 1 on slots (s, s+H).  All
// pruning is compile-time: NT (needed output blocks) and ZS = ceil(z/G)
// rounded up to even (input slots that may hold non-zeros).  A slot
// offset >= ZS is zero for every lane, so its butterfly is skipped; an
// offset < ZS whose partner is >= ZS is a multiply-only butterfly.  The one
// boundary slot that is zero for some lanes only is computed in full (the
// zeros are real zeros in the registers, so the result is exact).  No
// runtime branch splits the unrolled butterflies, so ptxas can interleave
// the independent chains.
// SCALE: the operand is multiplied by L^-1 * 2^32 on its ZS possibly non-zero
// slots first (the product is linear in each operand), so the pointwise
// step is a bare Montgomery product.  The kernel always scales operand a,
// which the host makes the shorter one: at most 8 slots per thread against
// the >= 9 active slots of the pointwise step.
template <int K, int NT, int ZS, int AR = 0, bool SCALE = false, class TW = Tw>
__device__ __forceinline__ void fwd_top_zs(u32 (&v)[16], int t, const ConvSmallParams &P,
                                           const TW &W) {
    constexpr int G = 1 << (K - 4);
    const u32 p = P.p;
    if constexpr (SCALE) {
#pragma unroll
        for (int s = 0; s < ZS; ++s) v[s] = mul_t<AR>(v[s], P.linv_mont, p);
    }
#pragma unroll
    for (int lv = 3; lv >= 0; --lv) {
        const int H = 1 << lv;
        const int h = H * G;
#pragma unroll
        for (int s = 0; s < 16; ++s) {
            if (s & H) continue;
            const int sblk = s & ~(2 * H - 1);
            if (sblk >= NT) continue;                 // whole block unneeded
            const bool hi_needed = (sblk + H) < NT;
            const int so = s & (2 * H - 1);           // slot offset within the 2H block
            if (so >= ZS) continue;                   // both inputs zero
            const bool hi_zero = so + H >= ZS;
            if (!hi_zero) {
                if (hi_needed) {
                    const uint2 w = tw_fwd(W, h, lv + K - 4, t + G * so);
                    bfly_dif_t<AR>(v[s], v[s + H], w.x, w.y, p);
                } else {
                    v[s] = add_t<AR>(v[s], v[s + H], p);  // lo-only add (fold)
                }
            } else if (hi_needed) {
                const uint2 w = tw_fwd(W, h, lv + K - 4, t + G * so);
                v[s + H] = mul_t<AR>(v[s], w.x, w.y, p);  // hi input is zero
            }
        }
    }
}

// Granularity of the compile-time zero-pruning variants (in top slots):
// finer = more pruning, larger code (instruction-cache pressure).
#ifndef MC_ZS_STEP
#define MC_ZS_STEP 4
#endif

template <int K, int NT, int AR = 0, bool SCALE = false, class TW = Tw>
__device__ __forceinline__ void fwd_top(u32 (&v)[16], int z, int t, const ConvSmallParams &P,
                                        const TW &W) {
    constexpr int G = 1 << (K - 4);
    const int zs = (z + G - 1) / G;  // uniform across the launch
#if MC_ZS_STEP == 2
    if (zs <= 2) fwd_top_zs<K, NT, 2, AR, SCALE, TW>(v, t, P, W);
    else if (zs <= 4) fwd_top_zs<K, NT, 4, AR, SCALE, TW>(v, t, P, W);
    else if (zs <= 6) fwd_top_zs<K, NT, 6, AR, SCALE, TW>(v, t, P, W);
    else if (zs <= 8) fwd_top_zs<K, NT, 8, AR, SCALE, TW>(v, t, P, W);
    else if (zs <= 10) fwd_top_zs<K, NT, 10, AR, SCALE, TW>(v, t, P, W);
    else if (zs <= 12) fwd_top_zs<K, NT, 12, AR, SCALE, TW>(v, t, P, W);
    else if (zs <= 14) fwd_top_zs<K, NT, 14, AR, SCALE, TW>(v, t, P, W);
    else fwd_top_zs<K, NT, 16, AR, SCALE, TW>(v, t, P, W);
#elif MC_ZS_STEP == 4
    if (zs <= 4) fwd_top_zs<K, NT, 4, AR, SCALE, TW>(v, t, P, W);
    else if (zs <= 8) fwd_top_zs<K, NT, 8, AR, SCALE, TW>(v, t, P, W);
    else if (zs <= 12) fwd_top_zs<K, NT, 12, AR, SCALE, TW>(v, t, P, W);
    else fwd_top_zs<K, NT, 16, AR, SCALE, TW>(v, t, P, W);
#else
    if (zs <= 8) fwd_top_zs<K, NT, 8, AR, SCALE, TW>(v, t, P, W);
    else fwd_top_zs<K, NT, 16, AR, SCALE, TW>(v, t, P, W);
#endif
}

// L^-1 folded into operand a at the top pass (fwd_top_zs SCALE) instead of
// the pointwise step; MC_PRESCALE=0 restores the pointwise scaling (A/B).
#ifndef MC_PRESCALE
#define MC_PRESCALE 1
#endif

// ---------------------------------------------------------------- lower passes
// Levels h = 2^b of the lowest pass (SB = 0, constant twiddles) whose
// products take the FP64-quotient form (modarith.cuh mul_f64q_lazy): bit b
// of MC_F64Q.  Off: with h = 8 and 4 on FP64 (-DMC_F64Q=0xC) config 2 ran
// 122.9 vs 121.1 us and config 3 4.03 vs 3.91 ms, config 4 1.058 vs 1.062 ms
// (scripts/variant_ab.sh, two alternations on one box).  The fused kernel is
// bound by issue and latency more than by the FMA-heavy pipe, so the extra
// DADD / DFMA issue slots cost more than the freed IMAD.HI cycles; the
// isolated pass, which has no exchanges, gains 7% (profiles/r02/ubench_r02.json).
#ifndef MC_F64Q
#define MC_F64Q 0
#endif

template <int K, int LO, int HI, int SB, int AR = 0, class TW = Tw>
__device__ __forceinline__ void fwd_lower(u32 (&v)[16], int t, const ConvSmallParams &P,
                                          const TW &W) {
    const u32 p = P.p;
    const int tpos = slot_pos<SB>(t, 0);
#pragma unroll
    for (int b = HI - 1; b >= LO; --b) {
        const int h = 1 << b;
        const int sbit = b - SB;
#pragma unroll
        for (int s = 0; s < 16; ++s) {
            if ((s >> sbit) & 1) continue;
            if (SB == 0) {  // twiddle index is compile-time: w_{2h}^(s mod h)
                const int j = s & (h - 1);
                if (j == 0) {  // w = 1: no multiplication
                    bfly_dif1_t<AR>(v[s], v[s | (1 << sbit)], p);
                } else if ((MC_F64Q >> b) & 1) {
                    bfly_dif_q_t<AR>(v[s], v[s | (1 << sbit)], P.c16f[h + j].x, P.c16fd[h + j], p);
                } else {
                    const uint2 w = P.c16f[h + j];
                    bfly_dif_t<AR>(v[s], v[s | (1 << sbit)], w.x, w.y, p);
                }
                continue;
            }
            const int j = (tpos | (s << SB)) & (h - 1);
            const uint2 w = tw_fwd(W, h, b, j);
            bfly_dif_t<AR>(v[s], v[s | (1 << sbit)], w.x, w.y, p);
        }
    }
}

template <int K, int LO, int HI, int SB, int AR = 0, class TW = Tw>
__device__ __forceinline__ void inv_lower(u32 (&v)[16], int t, const ConvSmallParams &P,
                                          const TW &W) {
    const u32 p = P.p;
    const int tpos = slot_pos<SB>(t, 0);
#pragma unroll
    for (int b = LO; b < HI; ++b) {
        const int h = 1 << b;
        const int sbit = b - SB;
#pragma unroll
        for (int s = 0; s < 16; ++s) {
            if ((s >> sbit) & 1) continue;
            if (SB == 0) {
                const int j = s & (h - 1);
                if (j == 0) {  // w = 1
                    bfly_dit1_t<AR>(v[s], v[s | (1 << sbit)], p);
                } else if ((MC_F64Q >> b) & 1) {
                    bfly_dit_q_t<AR>(v[s], v[s | (1 << sbit)], P.c16i[h + j].x, P.c16id[h + j], p);
                } else {
                    const uint2 w = P.c16i[h + j];
                    bfly_dit_t<AR>(v[s], v[s | (1 << sbit)], w.x, w.y, p);
                }
                continue;
            }
            const int j = (tpos | (s << SB)) & (h - 1);
            const uint2 w = tw_inv(W, h, b, j);
            bfly_dit_tw<AR, TW>(v[s], v[s | (1 << sbit)], w, p);
        }
    }
}

// ---------------------------------------------------------------- top pass (inverse)
// transform.py:451-489 restricted to slot granularity.  M, N, OFF in slots;
// level index LV = log2 M (m = M*G elements).  In a lazy mode (AR != 0) the
// complete sub-transforms and the closing DIT butterflies run lazily; the
// truncation steps (pre-adds, cross butterflies, combines), whose modular
// sums need canonical operands, canonicalise exactly those operands first
// (Shoup products accept any word).  Outputs are in the mode's inverse range.
template <int K, int M, int N, int OFF, int AR = 0>
struct ItftTop {
    template <class TW>
    static __device__ __forceinline__ void run(u32 (&v)[16], int t, const ConvSmallParams &P,
                                               const TW &W) {
        constexpr int G = 1 << (K - 4);
        constexpr int H = M / 2;
        constexpr int LV = (M == 16) ? 4 : (M == 8) ? 3 : (M == 4) ? 2 : 1;
        const u32 p = P.p;
        if constexpr (M == 1 || N == 0) {
            return;
        } else if constexpr (N <= H) {
            // pre: time values of both halves folded into the first half
#pragma unroll
            for (int s = N; s < H; ++s)
                v[OFF + s] = add_mod(canon_t<AR>(v[OFF + s], p), canon_t<AR>(v[OFF + s + H], p), p);
            ItftTop<K, H, N, OFF, AR>::run(v, t, P, W);
            // combine: m*u_i = 2*(h*(u_i + u_{i+h})) - m*u_{i+h}
            const Shoup mm = P.mlev[LV];
#pragma unroll
            for (int s = 0; s < N; ++s) {
                const u32 a = canon_t<AR>(v[OFF + s], p);
                v[OFF + s] = sub_mod(add_mod(a, a, p), mul_shoup(v[OFF + s + H], mm, p), p);
            }
        } else {
            ItftTop<K, H, H, OFF, AR>::run(v, t, P, W);  // complete first half
            const Shoup mm = P.mlev[LV];
            const Shoup ih = P.hinv[LV];
            constexpr int h = H * G;
#pragma unroll
            for (int s = N - H; s < H; ++s) {  // cross butterflies
                const u32 a = canon_t<AR>(v[OFF + s], p), b = canon_t<AR>(v[OFF + s + H], p);
                const uint2 w = tw_fwd(W, h, LV - 1 + K - 4, t + G * s);
                u32 d = sub_mod(mul_shoup(a, ih, p), add_mod(b, b, p), p);
                v[OFF + s + H] = mul_shoup(d, w.x, w.y, p);
                v[OFF + s] = sub_mod(add_mod(a, a, p), mul_shoup(b, mm, p), p);
            }
            ItftTop<K, H, N - H, OFF + H, AR>::run(v, t, P, W);
#pragma unroll
            for (int s = 0; s < N - H; ++s) {  // inverse DIT butterflies
                const uint2 w = tw_inv(W, h, LV - 1 + K - 4, t + G * s);
                bfly_dit_tw<AR, TW>(v[OFF + s], v[OFF + s + H], w, p);
            }
        }
    }
};

// Inverse top pass (complete or truncated) in mode AR; outputs in the mode's
// inverse range (canon_t before storing).
template <int K, int NT, int AR, class TW = Tw>
__device__ __forceinline__ void inv_top(u32 (&v)[16], int t, const ConvSmallParams &P,
                                        const TW &W) {
    ItftTop<K, 16, NT, 0, AR>::run(v, t, P, W);
}

// ---------------------------------------------------------------- exchange
// Shared-memory address of transform position x.  LaySmall: one transform
// per buffer (swz).  LayCol<TC>: TC interleaved column transforms, element
// (x, c) in row x of a TC-wide tile; rows are XOR-permuted so that the
// 32/TC transform threads sharing a warp always hit distinct bank groups.
// kCols: interleaved transforms per tile (thread index = t * kCols + c);
// kThreads: threads of the CTA if its exchange groups may use named barriers
// (exch_sync), else 0.
struct LaySmall {
    static constexpr int kCols = 1, kThreads = 0;
    __device__ __forceinline__ int operator()(int x) const { return swz(x); }
};

struct LayXf {  // standalone transforms: scalar accesses only (swz_xf)
    static constexpr int kCols = 1, kThreads = 0;
    __device__ __forceinline__ int operator()(int x) const { return swz_xf(x); }
};

// CW: columns per thread (1, or 2: columns c and c + 1, c even, exchanged as
// 8-byte words; kCols counts thread columns).
template <int TC, int NTH = 0, int CW = 1>
struct LayCol {
    static constexpr int kCols = TC / CW, kThreads = NTH;
    int c;
    static constexpr int M = TC >= 32 ? 0 : 32 / TC - 1;
    __device__ __forceinline__ int operator()(int x) const { return (x ^ ((x >> 4) & M)) * TC + c; }
};

template <int SB, class Lay = LaySmall>
__device__ __forceinline__ void put(u32 *buf, const u32 (&v)[16], int t, Lay lay = Lay()) {
    mc_perturb();
    if constexpr (SB == 0 && std::is_same<Lay, LaySmall>::value) {
#pragma unroll
        for (int k = 0; k < 4; ++k)  // positions 16t + 4k .. +3: one aligned quad
            *reinterpret_cast<uint4 *>(buf + swz(16 * t + 4 * k)) =
                make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
    } else {
#pragma unroll
        for (int s = 0; s < 16; ++s) buf[lay(slot_pos<SB>(t, s))] = v[s];
    }
}

template <int SB, class Lay = LaySmall>
__device__ __forceinline__ void get(const u32 *buf, u32 (&v)[16], int t, Lay lay = Lay()) {
    mc_perturb();
    if constexpr (SB == 0 && std::is_same<Lay, LaySmall>::value) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint4 q = *reinterpret_cast<const uint4 *>(buf + swz(16 * t + 4 * k));
            v[4 * k] = q.x;
            v[4 * k + 1] = q.y;
            v[4 * k + 2] = q.z;
            v[4 * k + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int s = 0; s < 16; ++s) v[s] = buf[lay(slot_pos<SB>(t, s))];
    }
}

// Two interleaved column transforms per thread (LayCol with CW = 2): slot s of
// columns c and c + 1 travels as one 8-byte word.
template <int SB, class Lay>
__device__ __forceinline__ void put2(u32 *buf, const u32 (&v0)[16], const u32 (&v1)[16], int t,
                                     Lay lay) {
    mc_perturb();
#pragma unroll
    for (int s = 0; s < 16; ++s)
        *reinterpret_cast<uint2 *>(buf + lay(slot_pos<SB>(t, s))) = make_uint2(v0[s], v1[s]);
}

template <int SB, class Lay>
__device__ __forceinline__ void get2(const u32 *buf, u32 (&v0)[16], u32 (&v1)[16], int t, Lay lay) {
    mc_perturb();
#pragma unroll
    for (int s = 0; s < 16; ++s) {
        const uint2 q = *reinterpret_cast<const uint2 *>(buf + lay(slot_pos<SB>(t, s)));
        v0[s] = q.x;
        v1[s] = q.y;
    }
}

// Lower-pass plan for K: up to three passes (bits [8,KL), [4,8), [0,4) with
// KL = K - 4), each with its slot window base SB.
template <int K>
struct Plan {
    static constexpr int KL = K - 4;
    static constexpr int NP = KL == 0 ? 0 : KL <= 4 ? 1 : KL <= 8 ? 2 : 3;
    // pass i (0 = highest bits)
    static constexpr int lo(int i) { return NP == 3 ? (i == 0 ? 8 : i == 1 ? 4 : 0)
                                          : NP == 2 ? (i == 0 ? 4 : 0) : 0; }
    static constexpr int hi(int i) { return NP == 3 ? (i == 0 ? KL : i == 1 ? 8 : 4)
                                          : NP == 2 ? (i == 0 ? KL : 4) : KL; }
    static constexpr int sb(int i) { return lo(i); }
};

// Warp-level skipping of inactive G-blocks (truncated transforms).  A warp
// may skip a lower pass when the lowest G-block it touches -- lane 0, slot 0
// -- is inactive: every other slot/lane of the warp is then in a block at
// least as high.  can_skip<K, I, NT>() is false when even the last warp
// starts below NT (e.g. K = 12 with NT = 15, where a warp straddles two
// G-blocks): the branch is then compiled out, since it only fences ptxas
// from overlapping the exchange with the butterflies (measured -9%).
template <int K, int SB>
constexpr int gblock_const(int t) {
    return (((t >> SB) << (SB + 4)) | (t & ((1 << SB) - 1))) >> (K - 4);
}

template <int K, int I, int NT>
constexpr bool can_skip() {
    constexpr int T = (1 << K) / 16;
    return NT < 16 && T >= 32 && gblock_const<K, Plan<K>::sb(I)>(T - 32) >= NT;
}

template <int K, int I>
__device__ __forceinline__ int gblock_of_pass(int t) {
    return slot_pos<Plan<K>::sb(I)>(t, 0) >> (K - 4);
}

template <int K, int I, int NT>
__device__ __forceinline__ bool pass_active(int t) {
    if constexpr (!can_skip<K, I, NT>()) return true;
    else return gblock_of_pass<K, I>(t & ~31) < NT;  // warp-uniform
}

// Scope of an exchange between the layouts SBW (the wider one: higher slot
// window) and a lower one.  Thread t holds in layout SBW the positions with
// low bits t mod 2^SBW and high bits t >> SBW, and in any lower layout only
// positions of the block (t >> SBW) << (SBW + 4): every exchange stays inside
// aligned groups of 2^SBW transform threads (times the TC interleaved columns
// of a column tile), which are contiguous in threadIdx.  A group of GT <= 32
// threads lies in one warp and synchronises with a warp barrier (the 4 -> 0
// exchange of every row transform, every exchange of the sizes with T <= 32);
// a larger group that is a proper part of the CTA uses its own named barrier
// (bar.sync 1 + group, GT: the 8 -> 4 exchange at K = 13, the products of a
// multi-product CTA, the 4 -> 0 exchange of a column tile).  The groups then
// drift apart between the remaining CTA barriers, and one group's exchange
// overlaps the others' butterflies.  NTH = threads of the CTA (0: unknown,
// CTA barriers).  MC_WARP_EXCH=0: CTA barriers everywhere (A/B).
#ifndef MC_WARP_EXCH
#define MC_WARP_EXCH 1
#endif

// threads of a fused-kernel / row-pass CTA at transform size 2^K (SmallCfg, RowCfg)
template <int K>
constexpr int small_threads() { return (1 << K) / 16 >= 128 ? (1 << K) / 16 : 128; }

template <int GT, int NTH>
__device__ __forceinline__ void exch_sync() {
    if constexpr (MC_WARP_EXCH && GT <= 32) {
        mc_syncwarp();
    } else if constexpr (MC_WARP_EXCH && NTH > 0 && GT < NTH && GT % 32 == 0 && NTH / GT <= 15) {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)threadIdx.x / GT), "n"(GT) : "memory");
        mc_perturb();
    } else {
        mc_sync();
    }
}

// The barrier BEFORE an exchange's stores (write-after-read) is only needed
// when other threads may still be reading the locations a thread is about to
// write.  Inside a chain every put<SB> rewrites exactly the positions the same
// thread last read with get<SB> (the previous exchange of that buffer, or for
// the inverse chain's first exchange the forward chain's last), so no other
// thread ever read them since they were last written: these barriers are
// dropped (MC_WAR_SYNC=1 keeps them, A/B).  The first forward exchange stores
// the top-pass layout: bufA was last read in that layout by the previous
// product's inverse (own positions again), bufB by the previous product's
// forward chain, with the group barriers of the whole inverse chain in
// between; only a launch whose epilogue reuses bufA as a bulk-store staging
// area (FL_HOST) needs it (FS = true).
#ifndef MC_WAR_SYNC
#define MC_WAR_SYNC 0
#endif

template <int K, int NT, int I, int AR = 0, class TW = Tw, bool FS = true>
__device__ __forceinline__ void fwd_lower_chain(u32 *bufA, u32 *bufB, u32 (&va)[16], u32 (&vb)[16],
                                                int t, const ConvSmallParams &P, const TW &W) {
    if constexpr (I < Plan<K>::NP) {
        constexpr int SBprev = (I == 0) ? (K - 4) : Plan<K>::sb(I - 1);
        constexpr int SB = Plan<K>::sb(I);
        constexpr int GT = 1 << SBprev, NTH = small_threads<K>();
        if constexpr (MC_WAR_SYNC || (I == 0 && FS)) exch_sync<GT, NTH>();
        put<SBprev>(bufA, va, t);
        put<SBprev>(bufB, vb, t);
#ifndef MC_RACE_SELFTEST  // self-test of the race-stress build: this barrier removed must fail
        exch_sync<GT, NTH>();
#endif
        get<SB>(bufA, va, t);
        get<SB>(bufB, vb, t);
        // Inactive G-blocks (>= NT) are skipped per warp where possible;
        // otherwise transformed and discarded at the pointwise step.
        if (pass_active<K, I, NT>(t)) {
            fwd_lower<K, Plan<K>::lo(I), Plan<K>::hi(I), SB, AR, TW>(va, t, P, W);
            fwd_lower<K, Plan<K>::lo(I), Plan<K>::hi(I), SB, AR, TW>(vb, t, P, W);
        }
        fwd_lower_chain<K, NT, I + 1, AR, TW, FS>(bufA, bufB, va, vb, t, P, W);
    }
}

// Software-pipelined variant of fwd_lower_chain (MC_PIPE): the two operands'
// exchanges are staggered so that every barrier interval mixes one operand's
// shared-memory traffic with the other's butterflies, instead of running
// both operands' exchanges back to back while the integer pipes idle.
// Precondition: operand a's values for pass I are stored in bufA (not yet
// ordered by a barrier); operand b's are in registers in the layout of the
// previous pass.  Interval 1: get a, put b, pass I on a.  Interval 2: get b,
// put a for pass I+1, pass I on b.
template <int K, int NT, int I, int AR = 0, class TW = Tw>
__device__ __forceinline__ void fwd_lower_pipe(u32 *bufA, u32 *bufB, u32 (&va)[16], u32 (&vb)[16],
                                               int t, const ConvSmallParams &P, const TW &W) {
    if constexpr (I < Plan<K>::NP) {
        constexpr int SBprev = (I == 0) ? (K - 4) : Plan<K>::sb(I - 1);
        constexpr int SB = Plan<K>::sb(I);
        const bool act = pass_active<K, I, NT>(t);
        mc_sync();  // a's stores visible; every read of bufB done
        get<SB>(bufA, va, t);
        put<SBprev>(bufB, vb, t);
        if (act) fwd_lower<K, Plan<K>::lo(I), Plan<K>::hi(I), SB, AR, TW>(va, t, P, W);
        mc_sync();  // b's stores visible; every read of bufA done
        get<SB>(bufB, vb, t);
        if constexpr (I + 1 < Plan<K>::NP) put<SB>(bufA, va, t);
        if (act) fwd_lower<K, Plan<K>::lo(I), Plan<K>::hi(I), SB, AR, TW>(vb, t, P, W);
        fwd_lower_pipe<K, NT, I + 1, AR, TW>(bufA, bufB, va, vb, t, P, W);
    }
}

#ifndef MC_PIPE
#define MC_PIPE 0  // measured: cfg2 +1%, cfg3 0% (the pipes, not the exchanges, bound the kernel)
#endif

// Inverse lower passes in reverse order (lowest bits first); on exit the
// slots are in the top-pass layout.
template <int K, int NT, int I, int AR = 0, class TW = Tw>
__device__ __forceinline__ void inv_lower_chain(u32 *buf, u32 (&v)[16], int t,
                                                const ConvSmallParams &P, const TW &W) {
    if constexpr (I >= 0) {
        constexpr int SB = Plan<K>::sb(I);
        constexpr int SBnext = (I == 0) ? (K - 4) : Plan<K>::sb(I - 1);
        constexpr int GT = 1 << SBnext, NTH = small_threads<K>();
        if (pass_active<K, I, NT>(t))
            inv_lower<K, Plan<K>::lo(I), Plan<K>::hi(I), SB, AR, TW>(v, t, P, W);  // zeros stay zeros
        if constexpr (MC_WAR_SYNC) exch_sync<GT, NTH>();
        put<SB>(buf, v, t);
        exch_sync<GT, NTH>();
        get<SBnext>(buf, v, t);
        inv_lower_chain<K, NT, I - 1, AR, TW>(buf, v, t, P, W);
    }
}

// One operand, arbitrary layout: forward lower passes; on exit the slots
// are in the last lower pass's layout.
template <int K, int I, class Lay, int NT = 16, int AR = 0, class TW = Tw>
__device__ __forceinline__ void fwd_lower_chain1(u32 *buf, u32 (&v)[16], int t,
                                                 const ConvSmallParams &P, const TW &W, Lay lay) {
    if constexpr (I < Plan<K>::NP) {
        constexpr int SBprev = (I == 0) ? (K - 4) : Plan<K>::sb(I - 1);
        constexpr int SB = Plan<K>::sb(I);
        constexpr int GT = (1 << SBprev) * Lay::kCols;
        exch_sync<GT, Lay::kThreads>();
        put<SBprev>(buf, v, t, lay);
        exch_sync<GT, Lay::kThreads>();
        get<SB>(buf, v, t, lay);
        if (NT >= 16 || gblock_of_pass<K, I>(t) < NT)
            fwd_lower<K, Plan<K>::lo(I), Plan<K>::hi(I), SB, AR, TW>(v, t, P, W);
        fwd_lower_chain1<K, I + 1, Lay, NT, AR, TW>(buf, v, t, P, W, lay);
    }
}

template <int K, int I, class Lay, int NT = 16, int AR = 0, class TW = Tw>
__device__ __forceinline__ void inv_lower_chain1(u32 *buf, u32 (&v)[16], int t,
                                                 const ConvSmallParams &P, const TW &W, Lay lay) {
    if constexpr (I >= 0) {
        constexpr int SB = Plan<K>::sb(I);
        constexpr int SBnext = (I == 0) ? (K - 4) : Plan<K>::sb(I - 1);
        constexpr int GT = (1 << SBnext) * Lay::kCols;
        if (NT >= 16 || gblock_of_pass<K, I>(t) < NT)
            inv_lower<K, Plan<K>::lo(I), Plan<K>::hi(I), SB, AR, TW>(v, t, P, W);
        exch_sync<GT, Lay::kThreads>();
        put<SB>(buf, v, t, lay);
        exch_sync<GT, Lay::kThreads>();
        get<SBnext>(buf, v, t, lay);
        inv_lower_chain1<K, I - 1, Lay, NT, AR, TW>(buf, v, t, P, W, lay);
    }
}

// Two columns per thread: the same passes on v0 and v1 (one set of twiddle
// loads serves both), 8-byte exchanges.
template <int K, int I, class Lay, int NT = 16, int AR = 0, class TW = Tw>
__device__ __forceinline__ void fwd_lower_chain2(u32 *buf, u32 (&v0)[16], u32 (&v1)[16], int t,
                                                 const ConvSmallParams &P, const TW &W, Lay lay) {
    if constexpr (I < Plan<K>::NP) {
        constexpr int SBprev = (I == 0) ? (K - 4) : Plan<K>::sb(I - 1);
        constexpr int SB = Plan<K>::sb(I);
        constexpr int GT = (1 << SBprev) * Lay::kCols;
        exch_sync<GT, Lay::kThreads>();
        put2<SBprev>(buf, v0, v1, t, lay);
        exch_sync<GT, Lay::kThreads>();
        get2<SB>(buf, v0, v1, t, lay);
        if (NT >= 16 || gblock_of_pass<K, I>(t) < NT) {
            fwd_lower<K, Plan<K>::lo(I), Plan<K>::hi(I), SB, AR, TW>(v0, t, P, W);
            fwd_lower<K, Plan<K>::lo(I), Plan<K>::hi(I), SB, AR, TW>(v1, t, P, W);
        }
        fwd_lower_chain2<K, I + 1, Lay, NT, AR, TW>(buf, v0, v1, t, P, W, lay);
    }
}

template <int K, int I, class Lay, int NT = 16, int AR = 0, class TW = Tw>
__device__ __forceinline__ void inv_lower_chain2(u32 *buf, u32 (&v0)[16], u32 (&v1)[16], int t,
                                                 const ConvSmallParams &P, const TW &W, Lay lay) {
    if constexpr (I >= 0) {
        constexpr int SB = Plan<K>::sb(I);
        constexpr int SBnext = (I == 0) ? (K - 4) : Plan<K>::sb(I - 1);
        constexpr int GT = (1 << SBnext) * Lay::kCols;
        if (NT >= 16 || gblock_of_pass<K, I>(t) < NT) {
            inv_lower<K, Plan<K>::lo(I), Plan<K>::hi(I), SB, AR, TW>(v0, t, P, W);
            inv_lower<K, Plan<K>::lo(I), Plan<K>::hi(I), SB, AR, TW>(v1, t, P, W);
        }
        exch_sync<GT, Lay::kThreads>();
        put2<SB>(buf, v0, v1, t, lay);
        exch_sync<GT, Lay::kThreads>();
        get2<SBnext>(buf, v0, v1, t, lay);
        inv_lower_chain2<K, I - 1, Lay, NT, AR, TW>(buf, v0, v1, t, P, W, lay);
    }
}

template <int K>
constexpr int last_sb() { return Plan<K>::NP == 0 ? (K - 4) : Plan<K>::sb(Plan<K>::NP - 1); }

template <int K>
struct SmallCfg {
    static constexpr int L = 1 << K;
    static constexpr int T = L / 16;
    static constexpr int PPC = T >= 128 ? 1 : 128 / T;  // products per CTA
    static constexpr int THREADS = T * PPC;
    static_assert(THREADS == small_threads<K>(), "exch_sync group barriers assume this CTA size");
    static constexpr int MINB = THREADS >= 512 ? 1 : 2;  // CTAs per SM (register cap)
    // shared memory: forward + inverse stage tables, then 2 operand buffers
    // per product
    static constexpr int SMEM = 2 * L * 8 + PPC * 2 * L * 4;
};

// Compile-time feature flags of a launch (FL): the device-resident path
// (FL = 0) carries none of the host-I/O or input-reduction code, which costs
// registers and scheduling freedom in the butterfly stream.
constexpr int FL_HOST = 1;    // bulk-store epilogue / streamed-input ready flags (zero copy)
constexpr int FL_REDUCE = 2;  // operands are arbitrary words: reduce mod p on load
constexpr int FL_FOLD = 4;    // split truncated product, head: fold rows longer than L
constexpr int FL_WRAP = 8;    // split truncated product, tail: unwrap the head's result
constexpr int FL_TWIST = 16;  // split truncated product, twisted quarter piece (mod x^(L'/4) - i)

// Persistent kernel: each CTA copies the (p, L) stage tables into shared
// memory once and then walks the batch with a grid stride.
template <int K, int NT, int AR = 0, int FL = 0>
__global__ void __launch_bounds__(SmallCfg<K>::THREADS, SmallCfg<K>::MINB)
conv_small_kernel(const ConvSmallParams P) {
    using C = SmallCfg<K>;
    constexpr int L = C::L, T = C::T;
    extern __shared__ uint4 smem_raw[];
    uint2 *tf_s = reinterpret_cast<uint2 *>(smem_raw);
    uint2 *ti_s = tf_s + L;
    u32 *data = reinterpret_cast<u32 *>(ti_s + L);
    const bool tma = C::PPC == 1 && P.tma;
    if (!tma) {
        const uint4 *gf = reinterpret_cast<const uint4 *>(P.tf);
        const uint4 *gi = reinterpret_cast<const uint4 *>(P.ti);
        uint4 *sf = reinterpret_cast<uint4 *>(tf_s);
        uint4 *si = reinterpret_cast<uint4 *>(ti_s);
        for (int i = threadIdx.x; i < L / 2; i += C::THREADS) {
            sf[i] = __ldg(gf + i);
            si[i] = __ldg(gi + i);
        }
    }
    const Tw W{tf_s, ti_s};
    const int grp = threadIdx.x / T;
    const int t = threadIdx.x % T;
    u32 *bufA = data + grp * 2 * L;
    u32 *bufB = bufA + L;
    // TMA staging (PPC == 1 only): [mbarrier (16 B)][a row][b row]
    uint64_t *mbar = reinterpret_cast<uint64_t *>(data + C::PPC * 2 * L);
    u32 *stA = reinterpret_cast<u32 *>(mbar + 2);
    u32 *stB = stA + P.za16;
    auto prefetch = [&](long long r, u32 extra_bytes) {  // thread 0 only
        const u32 ba = 4u * P.za16, bb = 4u * P.zb16;
        if ((FL & FL_HOST) && P.ready) {  // inputs still streaming in: wait for this row's chunk
            const uint32_t *f = P.ready + r / P.ready_rows;
            while (ld_acquire_sys(f) != P.epoch) __nanosleep(64);
            fence_proxy_async_all();
        }
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(mbar, ba + bb + extra_bytes);
        if (ba) bulk_g2s(stA, P.a + r * P.lda, ba, mbar);
        if (bb) bulk_g2s(stB, P.b + r * P.ldb, bb, mbar);
    };
    if (tma && threadIdx.x == 0) {
        // one DRAM round trip for the prologue: the stage tables and the
        // first product's rows all land on the first mbarrier phase (the
        // grid never exceeds the batch, so every CTA owns a product)
        mbar_init(mbar, 1);
        fence_mbar_init();
        prefetch(blockIdx.x, 2u * L * 8u);
        bulk_g2s(tf_s, P.tf, L * 8u, mbar);
        bulk_g2s(ti_s, P.ti, L * 8u, mbar);
    }
    mc_sync();
    uint32_t phase = 0;

    for (long long base = (long long)blockIdx.x * C::PPC; base < P.batch;
         base += (long long)gridDim.x * C::PPC) {
        const long long row = base + grp;
        const bool valid = row < P.batch;
        u32 va[16], vb[16];
        const u32 *ga = P.a + (valid ? row : 0) * P.lda;
        const u32 *gb = P.b + (valid ? row : 0) * P.ldb;
        if (tma) {
            mbar_wait(mbar, phase);
            phase ^= 1;
#pragma unroll
            for (int s = 0; s < 16; ++s) {  // predicated LDS, no branches
                const int x = (s << (K - 4)) | t;
                va[s] = x < P.za16 ? stA[x] : 0u;
                vb[s] = x < P.zb16 ? stB[x] : 0u;
                if constexpr ((FL & FL_FOLD) != 0) {  // x + L wraps onto x mod (x^L - 1)
                    if (x + L < P.za16) va[s] = add_mod(va[s], stA[x + L], P.p);
                    if (x + L < P.zb16) vb[s] = add_mod(vb[s], stB[x + L], P.p);
                }
            }
            if (P.z1 != P.za16 || P.z2 != P.zb16) {  // uniform: rows not a multiple of 4
#pragma unroll
                for (int s = 0; s < 16; ++s) {
                    const int x = (s << (K - 4)) | t;
                    if (x >= P.za16 && x < P.z1) va[s] = __ldcs(ga + x);
                    if (x >= P.zb16 && x < P.z2) vb[s] = __ldcs(gb + x);
                    if constexpr ((FL & FL_FOLD) != 0) {
                        const int y = x + L;
                        if (y >= P.za16 && y < P.z1) va[s] = add_mod(va[s], __ldcs(ga + y), P.p);
                        if (y >= P.zb16 && y < P.z2) vb[s] = add_mod(vb[s], __ldcs(gb + y), P.p);
                    }
                }
            }
            mc_sync();  // staging consumed: refill it for the next product
            const long long nxt = base + (long long)gridDim.x * C::PPC;
            if (threadIdx.x == 0 && nxt < P.batch) prefetch(nxt, 0u);
        } else {
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                const int x = (s << (K - 4)) | t;
                if constexpr ((FL & FL_TWIST) != 0) {
                    // a mod (x^L - i) (quarters folded with i^k), twisted by w_L'^x
                    // into the ring of the cyclic L-point product
                    auto fold4 = [&](const u32 *g, int z) {
                        const u32 u0 = (valid && x < z) ? __ldcs(g + x) : 0u;
                        const u32 u1 = (valid && x + L < z) ? __ldcs(g + x + L) : 0u;
                        const u32 u2 = (valid && x + 2 * L < z) ? __ldcs(g + x + 2 * L) : 0u;
                        const u32 u3 = (valid && x + 3 * L < z) ? __ldcs(g + x + 3 * L) : 0u;
                        const u32 f = add_mod(sub_mod(u0, u2, P.p),
                                              mul_shoup(sub_mod(u1, u3, P.p), P.qi, P.p), P.p);
                        const uint2 w = __ldg(P.twq_f + x);
                        return mul_shoup(f, w.x, w.y, P.p);
                    };
                    va[s] = fold4(ga, P.tz1);
                    vb[s] = fold4(gb, P.tz2);
                } else {
                    va[s] = (valid && x < P.z1) ? __ldcs(ga + x) : 0u;
                    vb[s] = (valid && x < P.z2) ? __ldcs(gb + x) : 0u;
                }
                if constexpr ((FL & FL_FOLD) != 0) {
                    if (valid && x + L < P.z1) va[s] = add_mod(va[s], __ldcs(ga + x + L), P.p);
                    if (valid && x + L < P.z2) vb[s] = add_mod(vb[s], __ldcs(gb + x + L), P.p);
                }
            }
        }
        if ((FL & FL_REDUCE) && P.reduce) {  // three-primes inputs: any 32-bit word -> residue
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                if (!MC_PRESCALE) va[s] = mul_t<AR>(va[s], 1u, P.red_wp, P.p);  // else: scaling reduces
                vb[s] = mul_t<AR>(vb[s], 1u, P.red_wp, P.p);
            }
        }

        if constexpr (MC_PIPE && Plan<K>::NP >= 1) {
            fwd_top<K, NT, AR, MC_PRESCALE != 0>(va, P.z1, t, P, W);
            // the previous product's bulk store has read its staging, and every
            // thread is past its last read of bufA, before bufA is refilled
            if ((FL & FL_HOST) && C::PPC == 1 && P.bulk_out && threadIdx.x == 0)
                bulk_wait_read_all();
            mc_sync();
            put<K - 4>(bufA, va, t);
            fwd_top<K, NT, AR>(vb, P.z2, t, P, W);  // overlaps a's stores
            fwd_lower_pipe<K, NT, 0, AR>(bufA, bufB, va, vb, t, P, W);
        } else {
            fwd_top<K, NT, AR, MC_PRESCALE != 0>(va, P.z1, t, P, W);
            fwd_top<K, NT, AR>(vb, P.z2, t, P, W);
            // the previous product's bulk store has read its staging before the
            // first exchange (after the barrier inside the chain) reuses bufA
            if ((FL & FL_HOST) && C::PPC == 1 && P.bulk_out && threadIdx.x == 0)
                bulk_wait_read_all();
            fwd_lower_chain<K, NT, 0, AR, Tw, (FL & FL_HOST) != 0>(bufA, bufB, va, vb, t, P, W);
        }

        // pointwise product in the last pass's layout, L^-1 folded in
        {
            constexpr int LAST = Plan<K>::NP - 1;
            constexpr int SB = (Plan<K>::NP == 0) ? (K - 4) : Plan<K>::sb(LAST < 0 ? 0 : LAST);
            if constexpr (NT < 16 && SB + 4 <= K - 4) {
                // all 16 slots of a thread sit in one G-block: one predicate
                if ((slot_pos<SB>(t, 0) >> (K - 4)) < NT) {
#pragma unroll
                    for (int s = 0; s < 16; ++s)
                        va[s] = MC_PRESCALE ? mont_mul(va[s], vb[s], P.p, P.pinv)
                                            : mul_inv_t<AR>(mont_mul(va[s], vb[s], P.p, P.pinv),
                                                            P.linv_mont, P.p);
                } else {
#pragma unroll
                    for (int s = 0; s < 16; ++s) va[s] = 0u;  // inactive tail: u_j = 0
                }
            } else {
#pragma unroll
                for (int s = 0; s < 16; ++s) {
                    const int x = slot_pos<SB>(t, s);
                    if (NT >= 16 || (x >> (K - 4)) < NT)
                        va[s] = MC_PRESCALE ? mont_mul(va[s], vb[s], P.p, P.pinv)
                                            : mul_inv_t<AR>(mont_mul(va[s], vb[s], P.p, P.pinv),
                                                            P.linv_mont, P.p);
                    else
                        va[s] = 0u;  // time values of the inactive tail: u_j = 0
                }
            }
        }

        inv_lower_chain<K, NT, Plan<K>::NP - 1, AR>(bufA, va, t, P, W);
        inv_top<K, NT, AR>(va, t, P, W);

        if ((FL & FL_HOST) && C::PPC == 1 && P.bulk_out) {
            // Stage the row in bufA (idle after the last inverse exchange; up to
            // 3 words spill into bufB, idle too) at the destination's offset mod
            // 16 bytes, then one bulk store of the aligned interior; the <= 3
            // head and tail words go out as plain stores.
            u32 *gc = P.c + row * P.ldc;
            const int mis = (int)(((uintptr_t)gc >> 2) & 3);
            u32 *stg = bufA + mis;
            mc_sync();  // every thread is done reading bufA
#pragma unroll
            for (int s = 0; s < 16; ++s)
                stg[(s << (K - 4)) | t] = canon_t<AR>(va[s], P.p);
            fence_proxy_async_smem();
            mc_sync();
            const int head = min((4 - mis) & 3, P.n);
            const int nb = ((P.n - head) >> 2) << 2;  // words in the bulk part
            if (threadIdx.x == 0 && nb > 0) {
                bulk_s2g(gc + head, stg + head, 4u * nb);
                bulk_commit();
            }
            if (t < head) gc[t] = stg[t];
            if (head + nb + t < P.n) gc[head + nb + t] = stg[head + nb + t];
        } else if (valid) {
            u32 *gc = P.c + row * P.ldc;
            if constexpr ((FL & FL_TWIST) != 0) {
                // c1 = c mod (x^L - i) (untwisted); c0 = c mod (x^(2L) - 1) from
                // the head; c = c0 + (x^(2L) - 1) h with h = (c0 mod (x^L - i) - c1) / 2
                u32 c0l[16], c0h[16];  // all loads in flight before the first store
#pragma unroll
                for (int s = 0; s < 16; ++s) {
                    const int x = (s << (K - 4)) | t;
                    c0l[s] = __ldcs(gc + x);
                    c0h[s] = __ldcs(gc + x + L);
                }
#pragma unroll
                for (int s = 0; s < 16; ++s) {
                    const int x = (s << (K - 4)) | t;
                    const uint2 w = __ldg(P.twq_i + x);
                    const u32 c1 = mul_shoup(canon_t<AR>(va[s], P.p), w.x, w.y, P.p);
                    const u32 f = add_mod(c0l[s], mul_shoup(c0h[s], P.qi, P.p), P.p);
                    const u32 h = mul_shoup(sub_mod(f, c1, P.p), P.qhalf, P.p);
                    __stcs(gc + x, sub_mod(c0l[s], h, P.p));
                    if (x < P.wrap_m) __stcs(gc + P.wrap_off + x, h);
                }
            } else if constexpr ((FL & FL_WRAP) != 0) {
                // c0 = c mod (x^(L/2) - 1) from the head launch holds c[x] +
                // c[x + L/2] for x < m; the low product gives c[x]
                u32 c0[16];  // all loads in flight before the first store
#pragma unroll
                for (int s = 0; s < 16; ++s) {
                    const int x = (s << (K - 4)) | t;
                    c0[s] = x < P.wrap_m ? __ldcs(gc + x) : 0u;
                }
#pragma unroll
                for (int s = 0; s < 16; ++s) {
                    const int x = (s << (K - 4)) | t;
                    if (x < P.wrap_m) {
                        const u32 lo = canon_t<AR>(va[s], P.p);
                        __stcs(gc + x, lo);
                        __stcs(gc + P.wrap_off + x, sub_mod(c0[s], lo, P.p));
                    }
                }
            } else {
#pragma unroll
                for (int s = 0; s < 16; ++s) {
                    const int x = (s << (K - 4)) | t;
                    if (x < P.n) __stcs(gc + x, canon_t<AR>(va[s], P.p));
                }
            }
        }
    }
    if ((FL & FL_HOST) && C::PPC == 1 && P.bulk_out && threadIdx.x == 0) bulk_wait_all();
}

}  // namespace mc
