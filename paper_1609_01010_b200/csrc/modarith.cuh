// Word-size modular arithmetic on the sm_100a integer pipes.
//
// Residues are uint32 in [0, p), p < 2^31 (so 2p < 2^32 and every lazy sum
// below fits in a word).  Fixed operands (twiddles, scale constants) use
// Shoup's precomputed quotient: w' = floor(w * 2^32 / p), and
//   q = umulhi(x, w');  r = x*w - q*p      in [0, 2p) for ANY x < 2^32,
// i.e. IMAD.HI + IMUL + IMAD.  Variable x variable products (the pointwise
// spectral product) use Montgomery REDC with R = 2^32.
//
// The reference performs the same arithmetic with Python ints and `%`
// (transform.py:160-163 butterfly, convolve.py:123 pointwise); every helper
// here returns the canonical residue, so results are bit-identical.
#pragma once
#include <cstdint>

namespace mc {

typedef uint32_t u32;
typedef uint64_t u64;

struct Shoup {
    u32 w;   // multiplier in [0, p)
    u32 wp;  // floor(w * 2^32 / p)
};

// The conditional subtractions below are unsigned minima: if x < p then
// x - p wraps above x.  They are written with the DPX add-min intrinsic
// (__viaddmin_u32(a, b, c) = min(a + b, c), one VIADDMNMX on the ALU pipe)
// so the additions stay off the FMA pipe, which the Shoup products already
// saturate.

// [0, 2p) -> [0, p)
__device__ __forceinline__ u32 red1(u32 x, u32 p) { return __viaddmin_u32(x, 0u - p, x); }

// (a + b) mod p for a, b in [0, p): min(a + b, a + b - p)
__device__ __forceinline__ u32 add_mod(u32 a, u32 b, u32 p) {
    return __viaddmin_u32(a, b, a + b - p);
}

// (a - b) mod p for a, b in [0, p): min(a - b, a - b + p)
__device__ __forceinline__ u32 sub_mod(u32 a, u32 b, u32 p) {
    u32 d = a - b;
    return __viaddmin_u32(d, p, d);
}

// x * w mod p in [0, 2p), any 32-bit x.
__device__ __forceinline__ u32 mul_shoup_lazy(u32 x, u32 w, u32 wp, u32 p) {
    u32 q = __umulhi(x, wp);
    return x * w - q * p;
}

__device__ __forceinline__ u32 mul_shoup(u32 x, u32 w, u32 wp, u32 p) {
    return red1(mul_shoup_lazy(x, w, wp, p), p);
}

__device__ __forceinline__ u32 mul_shoup(u32 x, Shoup s, u32 p) {
    return mul_shoup(x, s.w, s.wp, p);
}

// Montgomery product a*b*2^-32 mod p, canonical.  pinv = p^-1 mod 2^32.
// a*b - m*p is divisible by 2^32 with m = lo*pinv, and its quotient
// hi - umulhi(m, p) lies in (-p, p).
__device__ __forceinline__ u32 mont_mul(u32 a, u32 b, u32 p, u32 pinv) {
    u32 lo = a * b;
    u32 hi = __umulhi(a, b);
    u32 m = lo * pinv;
    u32 r = hi - __umulhi(m, p);
    return min(r, r + p);
}

// Decimation-in-frequency butterfly (Gentleman-Sande):
//   lo = a + b,  hi = (a - b) * w          (transform.py:390-393)
// Both butterflies are written as plain sums followed by unsigned minima
// (rather than through add_mod/red1): ptxas then moves about a third of the
// additions to the FMA pipe as IMAD.IADD, balancing it against the ALU pipe
// that carries the minima (+7% in the isolated pass benchmark, +3% on
// config 4; profiles/r01/ubench_pipes.txt).
__device__ __forceinline__ void bfly_dif(u32 &a, u32 &b, u32 w, u32 wp, u32 p) {
    const u32 s = a + b;
    const u32 r = mul_shoup_lazy(a - b + p, w, wp, p);
    a = min(s, s - p);
    b = min(r, r - p);
}

// Decimation-in-time butterfly (Cooley-Tukey):
//   t = b * w, lo = a + t, hi = a - t      (transform.py:160-163)
__device__ __forceinline__ void bfly_dit(u32 &a, u32 &b, u32 w, u32 wp, u32 p) {
    const u32 r = mul_shoup_lazy(b, w, wp, p);
    const u32 t = min(r, r - p);
    const u32 s = a + t, d = a - t + p;
    a = min(s, s - p);
    b = min(d, d - p);
}

// ---------------------------------------------------------------- lazy ranges
// Arithmetic modes of the transform kernels (template parameter AR):
//   AR = 0  canonical residues everywhere (bfly_dif / bfly_dit above).
//   AR = 1  Harvey's lazy ranges, p < 2^30 (4p < 2^32): forward DIF values in
//           [0, 2p), inverse DIT values in [0, 4p).  DIF 6 instructions
//           instead of 7, DIT 6 instead of 8.  The Montgomery pointwise
//           product accepts [0, 2p) operands when 4p < 2^32.
//   AR = 2  any p < 2^31: canonical forward; inverse values in [0, 2p).  A
//           DIT butterfly reduces only its additive input instead of both
//           outputs (a multiplicand may be any 32-bit word): 7 instructions
//           instead of 8.
// Kernels canonicalise (canon_t) before every store of a final result.
// Building with -DMC_AR_CANON turns modes 1 and 2 into mode 0 (A/B runs).
#ifdef MC_AR_CANON
#define MC_AR(ar) 0
#else
#define MC_AR(ar) (ar)
#endif

// forward-side multiply (DIF twiddles, input reduction, forward twists)
template <int AR>
__device__ __forceinline__ u32 mul_t(u32 x, u32 w, u32 wp, u32 p) {
    const u32 r = mul_shoup_lazy(x, w, wp, p);
    return MC_AR(AR) == 1 ? r : min(r, r - p);
}

template <int AR>
__device__ __forceinline__ u32 mul_t(u32 x, Shoup s, u32 p) { return mul_t<AR>(x, s.w, s.wp, p); }

// inverse-side multiply (pointwise scale, inverse twists): lazy in modes 1, 2
template <int AR>
__device__ __forceinline__ u32 mul_inv_t(u32 x, u32 w, u32 wp, u32 p) {
    const u32 r = mul_shoup_lazy(x, w, wp, p);
    return MC_AR(AR) >= 1 ? r : min(r, r - p);
}

template <int AR>
__device__ __forceinline__ u32 mul_inv_t(u32 x, Shoup s, u32 p) {
    return mul_inv_t<AR>(x, s.w, s.wp, p);
}

// a + b of two forward-range values
template <int AR>
__device__ __forceinline__ u32 add_t(u32 a, u32 b, u32 p) {
    const u32 s = a + b, q = MC_AR(AR) == 1 ? 2 * p : p;
    return min(s, s - q);
}

template <int AR>
__device__ __forceinline__ void bfly_dif_t(u32 &a, u32 &b, u32 w, u32 wp, u32 p) {
    if constexpr (MC_AR(AR) == 1) {
        const u32 s = a + b;
        b = mul_shoup_lazy(a - b + 2 * p, w, wp, p);
        a = min(s, s - 2 * p);
    } else {
        bfly_dif(a, b, w, wp, p);
    }
}

// DIF butterfly with w = 1
template <int AR>
__device__ __forceinline__ void bfly_dif1_t(u32 &a, u32 &b, u32 p) {
    const u32 q = MC_AR(AR) == 1 ? 2 * p : p;
    const u32 s = a + b, d = a - b + q;
    a = min(s, s - q);
    b = min(d, d - q);
}

template <int AR>
__device__ __forceinline__ void bfly_dit_t(u32 &a, u32 &b, u32 w, u32 wp, u32 p) {
    if constexpr (MC_AR(AR) == 1) {  // [0, 4p) in and out
        const u32 x = min(a, a - 2 * p);
        const u32 t = mul_shoup_lazy(b, w, wp, p);
        a = x + t;
        b = x - t + 2 * p;
    } else if constexpr (MC_AR(AR) == 2) {  // [0, 2p) in and out
        const u32 x = min(a, a - p);
        const u32 r = mul_shoup_lazy(b, w, wp, p);
        const u32 t = min(r, r - p);
        a = x + t;
        b = x - t + p;
    } else {
        bfly_dit(a, b, w, wp, p);
    }
}

// DIT butterfly with the twiddle given NEGATED (w' = -w): the merged stage
// table stores w_{2h}^{h-j} = -w_{2h}^{-j} for the inverse twiddles, so the
// butterfly forms the same products and swaps its two outputs.
template <int AR>
__device__ __forceinline__ void bfly_dit_neg_t(u32 &a, u32 &b, u32 w, u32 wp, u32 p) {
    if constexpr (MC_AR(AR) == 1) {  // [0, 4p) in and out
        const u32 x = min(a, a - 2 * p);
        const u32 t = mul_shoup_lazy(b, w, wp, p);
        a = x - t + 2 * p;
        b = x + t;
    } else if constexpr (MC_AR(AR) == 2) {  // [0, 2p) in and out
        const u32 x = min(a, a - p);
        const u32 r = mul_shoup_lazy(b, w, wp, p);
        const u32 t = min(r, r - p);
        a = x - t + p;
        b = x + t;
    } else {
        const u32 r = mul_shoup_lazy(b, w, wp, p);
        const u32 t = min(r, r - p);
        const u32 s = a + t, d = a - t + p;
        a = min(d, d - p);
        b = min(s, s - p);
    }
}

// ---------------------------------------------------------------- FP64 quotient
// Shoup's product with the quotient estimated on the FP64 pipe instead of
// IMAD.HI: x is made exact in a double by one DADD (2^52 bias), one DFMA.RZ
// forms floor(x * wd) + 2^52 with wd = RD(w / p) <= w / p, so q is floor(x w / p)
// or one less and r = x*w - q*p lies in [0, 2p) exactly as with Shoup.  The
// FMA-heavy pipe, which the Shoup products keep busiest (IMAD.HI holds it two
// cycles), then carries two IMADs instead of four slots; the otherwise idle
// FP64 pipe takes the rest.  Measured on the isolated radix-16 pass
// (scripts/ubench.py): a quarter of the butterflies this way, 10.95 -> 11.73
// butterflies/clk/SM; all of them, 10.8 (the issue slots then bind).
__device__ __forceinline__ u32 mul_f64q_lazy(u32 x, u32 w, double wd, u32 p) {
    const double xd = __hiloint2double(0x43300000, (int)x) - 4503599627370496.0;
    const double qd = __fma_rz(xd, wd, 4503599627370496.0);
    return x * w - (u32)__double2loint(qd) * p;
}

template <int AR>
__device__ __forceinline__ void bfly_dif_q_t(u32 &a, u32 &b, u32 w, double wd, u32 p) {
    if constexpr (MC_AR(AR) == 1) {
        const u32 s = a + b;
        b = mul_f64q_lazy(a - b + 2 * p, w, wd, p);
        a = min(s, s - 2 * p);
    } else {
        const u32 s = a + b;
        const u32 r = mul_f64q_lazy(a - b + p, w, wd, p);
        a = min(s, s - p);
        b = min(r, r - p);
    }
}

template <int AR>
__device__ __forceinline__ void bfly_dit_q_t(u32 &a, u32 &b, u32 w, double wd, u32 p) {
    if constexpr (MC_AR(AR) == 1) {
        const u32 x = min(a, a - 2 * p);
        const u32 t = mul_f64q_lazy(b, w, wd, p);
        a = x + t;
        b = x - t + 2 * p;
    } else if constexpr (MC_AR(AR) == 2) {
        const u32 x = min(a, a - p);
        const u32 r = mul_f64q_lazy(b, w, wd, p);
        const u32 t = min(r, r - p);
        a = x + t;
        b = x - t + p;
    } else {
        const u32 r = mul_f64q_lazy(b, w, wd, p);
        const u32 t = min(r, r - p);
        const u32 s = a + t, d = a - t + p;
        a = min(s, s - p);
        b = min(d, d - p);
    }
}

// DIT butterfly with w = 1
template <int AR>
__device__ __forceinline__ void bfly_dit1_t(u32 &a, u32 &b, u32 p) {
    if constexpr (MC_AR(AR) >= 1) {
        const u32 q = MC_AR(AR) == 1 ? 2 * p : p;
        const u32 x = min(a, a - q), y = min(b, b - q);
        a = x + y;
        b = x - y + q;
    } else {
        const u32 s = a + b, d = a - b + p;
        a = min(s, s - p);
        b = min(d, d - p);
    }
}

// inverse-range value -> canonical residue
template <int AR>
__device__ __forceinline__ u32 canon_t(u32 x, u32 p) {
    if constexpr (MC_AR(AR) == 1) x = min(x, x - 2 * p);
    if constexpr (MC_AR(AR) >= 1) x = min(x, x - p);
    return x;
}

}  // namespace mc
