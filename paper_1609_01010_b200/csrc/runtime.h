// Host runtime shared by the kernels and the C ABI: field math, twiddle
// table cache, error reporting and kernel-launch bookkeeping.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/modconv_b200.h"
#include "modarith.cuh"

namespace mc {

// ----------------------------------------------------------------- errors
void set_error(const std::string &msg, int required_two_adicity = -1);
mc_status fail(mc_status st, const std::string &msg, int required_two_adicity = -1);
mc_status cuda_fail(cudaError_t e, const char *what);
void note_launches(int64_t n);

#define MC_CUDA_CHECK(expr)                                    \
    do {                                                       \
        cudaError_t _e = (expr);                               \
        if (_e != cudaSuccess) return ::mc::cuda_fail(_e, #expr); \
    } while (0)

// ----------------------------------------------------------------- field math
u64 mulmod(u64 a, u64 b, u64 p);
u64 powmod(u64 b, u64 e, u64 p);
bool is_prime_u32(u64 n);
int two_adicity(u64 p);
u32 smallest_primitive_root(u32 p);
// Generator behind the roots of unity for p on this thread: the one set by
// mc_use_generator(p, g), else the smallest primitive root (field.py:102-108).
u32 field_generator(u32 p);
Shoup shoup(u32 w, u32 p);
u32 inv_mod(u32 a, u32 p);

// Validates p (odd prime < 2^31) and log2L <= two-adicity.
mc_status check_field(u32 p, int log2L);

// ----------------------------------------------------------------- tables
// Per-(device, p, log2L) constant set.  tf[h + j] = {w_{2h}^j, shoup},
// ti[h + j] = {w_{2h}^-j, shoup} for 1 <= h < L, 0 <= j < h (the stage
// slices fwd_stages / inv_stages of transform.py:106-107, concatenated so
// that one stage's twiddles are contiguous).
struct FieldTables {
    u32 p = 0;
    int log2L = 0;
    u32 gen = 0;        // primitive root the tables are built from
    u32 root = 0;       // w_L = gen^((p-1)/L) (field.py:209-224)
    u32 pinv = 0;       // p^-1 mod 2^32 (Montgomery)
    Shoup linv;         // L^-1 mod p
    Shoup linv_mont;    // L^-1 * 2^32 mod p (undoes REDC's 2^-32)
    uint2 *tf = nullptr;
    uint2 *ti = nullptr;
    // merged stage table (conv_small.cuh TwM): stage h = 2^lg at
    // tm[h + lg - 1 + k] = w_{2h}^k, k = 0..h; tm_entries = its length
    uint2 *tm = nullptr;
    int tm_entries = 0;
    uint2 h16f[16] = {};  // host copies of tf[0..15] / ti[0..15]
    uint2 h16i[16] = {};
    double h16fd[16] = {};  // RD(w / p) of the same twiddles (FP64-quotient products)
    double h16id[16] = {};
    Shoup mlev[5] = {};   // fused-kernel top-level constants (see ConvSmallParams)
    Shoup hinv[5] = {};
};

// Stage tables (tf/ti) are only materialised up to this size; larger
// transforms go through the four-step path whose row/column sub-transforms
// use their own (small) tables.
constexpr int kMaxStageTableLog2 = 16;

// Thread-safe cached lookup (builds on first use; synchronous).
mc_status get_tables(u32 p, int log2L, const FieldTables **out);

int current_device();
// Launch-time state that belongs to one device: kernel attributes
// (cudaFuncSetAttribute) and occupancy figures live in the device's context,
// so a process that drives several GPUs needs them once per device.
// `static PerDevice<T> x;` at the launch site, `x.get()` = the slot of the
// calling thread's current device.  Races between threads are benign: every
// writer stores the same value after the same idempotent runtime calls.
constexpr int kMaxDevices = 64;
template <class T>
struct PerDevice {
    T v[kMaxDevices] = {};
    T &get() {
        const int d = current_device();
        return v[d >= 0 && d < kMaxDevices ? d : 0];
    }
};
void keep_pool_memory();
// Lazy-range arithmetic (modarith.cuh) is valid for p < 2^30; MC_NO_LAZY
// (non-empty) forces the canonical kernels for A/B runs.
bool lazy_ok(uint32_t p);
int sm_count();

}  // namespace mc
