// Garner reconstruction shared by the standalone CRT kernel (crt.cu) and the
// fused inverse-column + CRT pass of the three-primes four-step product
// (three_primes.cu).  No reference counterpart.
#pragma once
#include "runtime.h"

namespace mc {

constexpr u32 kCrtP1 = 469762049u, kCrtP2 = 998244353u, kCrtP3 = 2013265921u;

struct CrtConsts {
    u32 p1, p2, p3;
    Shoup inv12;     // p1^-1 mod p2
    Shoup p1_mod3;   // p1 mod p3
    Shoup inv123;    // (p1*p2)^-1 mod p3
    unsigned long long p12;
};

inline CrtConsts crt_consts() {
    CrtConsts k;
    k.p1 = kCrtP1;
    k.p2 = kCrtP2;
    k.p3 = kCrtP3;
    k.inv12 = shoup(inv_mod(kCrtP1 % kCrtP2, kCrtP2), kCrtP2);
    k.p1_mod3 = shoup(kCrtP1 % kCrtP3, kCrtP3);
    const u64 p12 = (u64)kCrtP1 * kCrtP2;
    k.inv123 = shoup(inv_mod((u32)(p12 % kCrtP3), kCrtP3), kCrtP3);
    k.p12 = p12;
    return k;
}

// Garner, first step: y2 = (r2 - r1) / p1 mod p2 (r1 < p1 < p2, canonical).
__device__ __forceinline__ u32 garner_y2(u32 r1, u32 r2, const CrtConsts &K) {
    return mul_shoup(sub_mod(r2, r1, K.p2), K.inv12, K.p2);
}

// Garner, second step: x = x12 + p1*p2*y3 with x12 = r1 + p1*y2 and
// y3 = (r3 - x12) / (p1*p2) mod p3; x < p1*p2*p3 < 2^90 as three 32-bit
// limbs (l0 least significant).
__device__ __forceinline__ void garner_limbs(u32 r1, u32 y2, u32 r3, const CrtConsts &K,
                                             u32 &l0, u32 &l1, u32 &l2) {
    const u32 x12m3 = add_mod(r1, mul_shoup(y2, K.p1_mod3, K.p3), K.p3);
    const u32 y3 = mul_shoup(sub_mod(r3, x12m3, K.p3), K.inv123, K.p3);
    const unsigned long long x12 = (unsigned long long)r1 + (unsigned long long)K.p1 * y2;
    const unsigned long long lo = K.p12 * y3;
    const unsigned long long hi = __umul64hi(K.p12, (unsigned long long)y3);
    const unsigned long long s = lo + x12;
    l0 = (u32)s;
    l1 = (u32)(s >> 32);
    l2 = (u32)(hi + (s < lo ? 1ull : 0ull));
}

}  // namespace mc
