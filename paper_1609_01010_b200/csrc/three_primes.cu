// Three-primes integer product at four-step sizes (config 5: L = 2^21):
// the per-prime forward column and row passes run on three forked streams,
// then ONE kernel runs the inverse column transforms of all three primes on
// each column tile and reconstructs the exact coefficients by Garner's CRT in
// its epilogue, writing the planar limbs.  The residues never round-trip
// through HBM and no separate CRT launch is needed.
//
// No reference counterpart: the reference lists three-primes integer
// multiplication as out of scope.  Per prime this is the
// reference's fft_pad product (convolve.py:160-169) on DensePoly.from_ints
// inputs (poly.py:46-49); the CRT is SURVEY.md section 8 a14.
#include <algorithm>

#include "crt.cuh"
#include "fourstep_int.cuh"

namespace mc {

// Inverse column tile of the fused pass: 4096 words per prime (R rows x TC
// columns), 256 threads, one column transform per R/16 threads, two CTAs
// per SM.  A quarter of the 16K-word tile of the single-prime pass, so that
// a 128-register budget holds the first two primes' results (r1, y2) of
// each slot while the third prime's column transform runs.
#ifndef MC_INV3_TILE  // words per prime of one column tile (A/B: 8192 = 512 threads, 1 CTA/SM;
                      // 2048 = 128 threads, 4 CTAs/SM: config 5 119 vs 112 us, 16-byte row chunks)
#define MC_INV3_TILE 4096
#endif

template <int KR>
struct Col3Cfg {
    static constexpr int R = 1 << KR;
    static constexpr int TILE = MC_INV3_TILE >= (4 << KR) ? MC_INV3_TILE : (4 << KR);
    static constexpr int TC = TILE >> KR;  // KR <= 11: >= 4 columns (16-byte rows)
    static constexpr int THREADS = TILE / 16;
    static constexpr int G = R / 16;
    // landing layout: row r at r*TC + (r/16)*PADW words; conflict-free first
    // read (rows 16t + s) for every TC
    static constexpr int PADW = TC < 32 ? TC : 8;
    static constexpr int BUFW = TILE + (R / 16) * PADW;
    static constexpr int SMEM = 3 * R * 8 + 2 * BUFW * 4;
    // 128 registers per thread either way (A/B: 2048-word tiles = 128 threads, 4 CTAs/SM)
    static constexpr int MINB = THREADS >= 512 ? 1 : THREADS >= 256 ? 2 : 4;
    __device__ static __forceinline__ int off(int row) { return row * TC + (row >> 4) * PADW; }
};

struct Inv3Params {
    ConvSmallParams cs[3];  // per prime: p, lowest-pass constants (c16i), arithmetic mode
    const uint2 *ti[3];     // per prime: inverse stage table of the R-point column transform
    const u32 *spec[3];     // per prime: [R][C] product spectrum after the row pass
    u32 *limbs;             // [3][ls] planar limbs
    long long n, ls;
    CrtConsts crt;
};

// Inverse column transform of prime K3 on the landed tile `buf` (the tile
// is then reused for the exchanges); canonical residues out.
template <int KR, int K3, int AR>
__device__ __forceinline__ void inv3_column(const Inv3Params &Q, u32 *buf, const uint2 *ti_s,
                                            u32 (&v)[16], int t, int c) {
    using C = Col3Cfg<KR>;
    constexpr int SB = last_sb<KR>();
#pragma unroll
    for (int s = 0; s < 16; ++s) v[s] = buf[C::off(slot_pos<SB>(t, s)) + c];
    const Tw W{ti_s, ti_s};  // complete transforms: the forward table is never read
    LayCol<C::TC, C::THREADS> lay{c};
    // Every thread has read its landed values before any exchange write: the
    // landing layout (padded rows) and the exchange layout place a block's rows
    // at different addresses, and the chain's first exchange only synchronises
    // its own thread group (exch_sync).
    mc_sync();
    inv_lower_chain1<KR, Plan<KR>::NP - 1, LayCol<C::TC, C::THREADS>, 16, AR>(buf, v, t, Q.cs[K3], W, lay);
    inv_top<KR, 16, AR>(v, t, Q.cs[K3], W);
#pragma unroll
    for (int s = 0; s < 16; ++s) v[s] = canon_t<AR>(v[s], Q.cs[K3].p);
}

// Persistent over column tiles; per tile the three primes' spectra arrive in
// turn by 16-byte cp.async into the other of two shared buffers while the
// current prime's column transform runs.  Garner's CRT runs in registers in
// the epilogue: r1 and y2 = (r2 - r1)/p1 mod p2 are kept per slot while the
// third prime's transform runs.
template <int KR, int KC, int AR0, int AR1>
__global__ void __launch_bounds__(Col3Cfg<KR>::THREADS, Col3Cfg<KR>::MINB)
col_inv3_crt_kernel(const Inv3Params Q, int ntiles) {
    using C = Col3Cfg<KR>;
    constexpr long long Ccols = 1ll << KC;
    constexpr int CHUNKS = C::TC / 4;
    extern __shared__ __align__(1024) uint4 smem_raw[];
    uint2 *ti_s = reinterpret_cast<uint2 *>(smem_raw);
    u32 *bufs = reinterpret_cast<u32 *>(ti_s + 3 * C::R);
    const int c = threadIdx.x % C::TC;
    const int t = threadIdx.x / C::TC;
    auto issue = [&](int tile, int k, int sel) {  // every thread: its share of the chunks
        const u32 *src = Q.spec[k] + (long long)tile * C::TC;
        u32 *dst = bufs + sel * C::BUFW;
        for (int q = threadIdx.x; q < C::R * CHUNKS; q += C::THREADS) {
            const int row = q / CHUNKS, ch = q % CHUNKS;
            const u32 *g = src + (long long)row * Ccols + 4 * ch;
            const u32 sa = smem_u32(dst + C::off(row) + 4 * ch);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // Wait for the landed buffer; after the barrier every thread is also past
    // its last access of the other buffer (the previous step's exchanges), so
    // the next step's copy may be queued into it.
    auto land = [&]() {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        mc_sync();
    };
    if ((int)blockIdx.x < ntiles) issue(blockIdx.x, 0, 0);
    // stage tables after the first copies are in flight (land()'s barrier orders
    // them before the first transform)
#pragma unroll
    for (int k = 0; k < 3; ++k)
        for (int i = threadIdx.x; i < C::R / 2; i += C::THREADS)
            reinterpret_cast<uint4 *>(ti_s + k * C::R)[i] =
                __ldg(reinterpret_cast<const uint4 *>(Q.ti[k]) + i);
    int sel = 0;  // three steps per tile over two buffers: the parity alternates
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        u32 r1[16], y2[16], v[16];
        land();
        issue(tile, 1, sel ^ 1);
        inv3_column<KR, 0, AR0>(Q, bufs + sel * C::BUFW, ti_s, v, t, c);
        sel ^= 1;
#pragma unroll
        for (int s = 0; s < 16; ++s) r1[s] = v[s];
        land();
        issue(tile, 2, sel ^ 1);
        inv3_column<KR, 1, AR1>(Q, bufs + sel * C::BUFW, ti_s + C::R, v, t, c);
        sel ^= 1;
#pragma unroll
        for (int s = 0; s < 16; ++s) y2[s] = garner_y2(r1[s], v[s], Q.crt);
        land();
        if (tile + (int)gridDim.x < ntiles) issue(tile + gridDim.x, 0, sel ^ 1);
        inv3_column<KR, 2, 2>(Q, bufs + sel * C::BUFW, ti_s + 2 * C::R, v, t, c);
        sel ^= 1;
        // epilogue: rows t + G*s of column col, three limb planes; only a tile
        // that reaches position n checks bounds per slot (tile-uniform branch)
        constexpr long long SLOT = (long long)C::G * Ccols;
        const long long col = (long long)tile * C::TC + c;
        const long long pos0 = (long long)t * Ccols + col;
        const bool full = 15 * SLOT + (long long)(C::G - 1) * Ccols +
                              (long long)tile * C::TC + C::TC - 1 < Q.n;
#pragma unroll
        for (int s = 0; s < 16; ++s) {
            const long long pos = pos0 + s * SLOT;
            u32 l0, l1, l2;
            garner_limbs(r1[s], y2[s], v[s], Q.crt, l0, l1, l2);
            if (full || pos < Q.n) {
                __stcs(Q.limbs + pos, l0);
                __stcs(Q.limbs + Q.ls + pos, l1);
                __stcs(Q.limbs + 2 * Q.ls + pos, l2);
            }
        }
    }
}

template <int KR, int AR0, int AR1>
static cudaError_t launch_inv3(const Inv3Params &Q, cudaStream_t st) {
    using C = Col3Cfg<KR>;
    static PerDevice<bool> ready_dev;
    bool &ready = ready_dev.get();
    if (!ready) {
        cudaError_t e = prep_kernel(col_inv3_crt_kernel<KR, 12, AR0, AR1>, C::SMEM, C::THREADS,
                                    nullptr);
        if (e != cudaSuccess) return e;
        ready = true;
    }
    const int ntiles = (int)((1ll << 12) / C::TC);
    const int grid = std::min(ntiles, C::MINB * sm_count());
    col_inv3_crt_kernel<KR, 12, AR0, AR1><<<grid, C::THREADS, C::SMEM, st>>>(Q, ntiles);
    return cudaGetLastError();
}

template <int KR>
static cudaError_t launch_inv3_ar(const Inv3Params &Q, cudaStream_t st) {
    if (Q.cs[0].ar == 1 && Q.cs[1].ar == 1) return launch_inv3<KR, 1, 1>(Q, st);
    return launch_inv3<KR, 2, 2>(Q, st);
}

// K range of the fused path: the TMA column kernel needs R >= 64 (K >= 18
// with 2^12-point rows); p2's 2-adicity caps every three-primes product at
// K = 23.
bool three_primes_fused_ok(long long n) {
    int K = 0;
    while ((1ll << K) < n) ++K;
    return K >= 18 && K <= 23;
}

long long three_primes_fused_scratch(long long n) {
    int K = 0;
    while ((1ll << K) < n) ++K;
    return 6ll << K;  // 2L words (both operands' spectra) per prime
}

// The fused path (three_primes_fused_ok(n) must hold).  scratch: at least
// three_primes_fused_scratch(n) words, or null (stream-ordered allocation).
mc_status three_primes_fused(const u32 *a, int z1, const u32 *b, int z2, u32 *limbs,
                             u32 *scratch, cudaStream_t st, cudaStream_t fs[3],
                             cudaEvent_t fork_ev, cudaEvent_t done_ev[3]) {
    const long long n = (long long)z1 + z2 - 1;
    FourPlan F[3];
    for (int k = 0; k < 3; ++k) {
        const u32 p = k == 0 ? kCrtP1 : k == 1 ? kCrtP2 : kCrtP3;
        mc_status s = fourstep_plan(0, a, z1, z1, b, z2, z2, nullptr, n, 1, p, -1, true, &F[k]);
        if (s != MC_OK) return s;
        if (F[k].KC != 12 || F[k].KR < 6 || F[k].KR > 11 || F[k].NT != 16)
            return fail(MC_EINVAL, "three-primes fused path: unsupported decomposition");
    }
    const long long L = F[0].L;
    u32 *res = scratch;
    if (!res) {
        keep_pool_memory();
        MC_CUDA_CHECK(cudaMallocAsync(&res, sizeof(u32) * 6 * L, st));
    }
    MC_CUDA_CHECK(cudaEventRecord(fork_ev, st));
    cudaError_t e = cudaSuccess;
    for (int k = 0; k < 3; ++k) {
        F[k].P.Ah = res + 2 * k * L;
        F[k].P.Bh = res + (2 * k + 1) * L;
        MC_CUDA_CHECK(cudaStreamWaitEvent(fs[k], fork_ev, 0));
        if (e == cudaSuccess) e = fourstep_fwd_rows(F[k], 0, 1, fs[k]);
        MC_CUDA_CHECK(cudaEventRecord(done_ev[k], fs[k]));
        MC_CUDA_CHECK(cudaStreamWaitEvent(st, done_ev[k], 0));
    }
    if (e == cudaSuccess) {
        Inv3Params Q;
        memset(&Q, 0, sizeof(Q));
        for (int k = 0; k < 3; ++k) {
            Q.cs[k] = F[k].P.cs;
            Q.ti[k] = F[k].P.col_ti;
            Q.spec[k] = F[k].P.Ah;
        }
        Q.limbs = limbs;
        Q.n = n;
        Q.ls = n;
        Q.crt = crt_consts();
        switch (F[0].KR) {
            case 6: e = launch_inv3_ar<6>(Q, st); break;
            case 7: e = launch_inv3_ar<7>(Q, st); break;
            case 8: e = launch_inv3_ar<8>(Q, st); break;
            case 9: e = launch_inv3_ar<9>(Q, st); break;
            case 10: e = launch_inv3_ar<10>(Q, st); break;
            default: e = launch_inv3_ar<11>(Q, st); break;
        }
        note_launches(1);
    }
    if (!scratch) cudaFreeAsync(res, st);
    if (e != cudaSuccess) return cuda_fail(e, "three-primes fused launch");
    return MC_OK;
}

}  // namespace mc
