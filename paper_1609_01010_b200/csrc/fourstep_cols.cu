// Column passes of the four-step path for one column size KR (compiled once
// per KR with -DMC_KR=<KR>); see fourstep.cuh for the decomposition.
#include <algorithm>
#include <cstdlib>

#include "fourstep_int.cuh"

#ifndef MC_KR
#error "compile with -DMC_KR=<log2 R>"
#endif

namespace mc {

// Forward: R-point DIF down each column of a TC-wide tile.  Truncated (NT <
// 16): top-pass outputs of blocks >= NT are pruned, lower passes skip those
// blocks and only rows < NT*R/16 are written.
// AR: arithmetic mode (modarith.cuh).
template <int KR, int KC, int NT, int AR = 0>
__global__ void __launch_bounds__(ColCfg<KR>::THREADS, ColCfg<KR>::MINB) col_fwd_kernel(const FourParams P) {
    using C = ColCfg<KR>;
    constexpr long long Ccols = 1ll << KC;
    extern __shared__ uint4 smem_raw[];
    uint2 *tf_s = reinterpret_cast<uint2 *>(smem_raw);
    u32 *tile = reinterpret_cast<u32 *>(tf_s + 2 * C::R);
    for (int i = threadIdx.x; i < C::R / 2; i += C::THREADS)
        reinterpret_cast<uint4 *>(tf_s)[i] = __ldg(reinterpret_cast<const uint4 *>(P.col_tf) + i);
    const Tw W{tf_s, tf_s};
    const int op = blockIdx.y;
    const long long prod = P.prod0 + blockIdx.z;
    const u32 *src = op ? P.b + prod * P.ldb : P.a + prod * P.lda;
    const long long z = op ? P.z2 : P.z1;
    u32 *dst = (op ? P.Bh : P.Ah) + (long long)blockIdx.z * (Ccols << KR);
    const int c = threadIdx.x % C::TC;
    const int t = threadIdx.x / C::TC;
    const long long col = (long long)blockIdx.x * C::TC + c;
    const u32 p = P.cs.p;
    mc_sync();

    u32 v[16];
#pragma unroll
    for (int s = 0; s < 16; ++s) {
        const long long idx = (long long)(t + C::G * s) * Ccols + col;
        u32 x = idx < z ? __ldcs(src + idx) : 0u;
        const long long L = Ccols << KR;
        if (P.fold && idx + L < z) x = add_mod(x, __ldcs(src + idx + L), p);
        if (P.reduce) x = mul_t<AR>(x, 1u, P.red_wp, p);
        v[s] = x;
    }
    const int zrows = (int)((z + Ccols - 1) / Ccols);
    fwd_top<KR, NT, AR>(v, zrows, t, P.cs, W);
    LayCol<C::TC, C::THREADS> lay{c};
    fwd_lower_chain1<KR, 0, LayCol<C::TC, C::THREADS>, NT, AR>(tile, v, t, P.cs, W, lay);
    constexpr int SB = last_sb<KR>();
#pragma unroll
    for (int s = 0; s < 16; ++s) {
        const int row = slot_pos<SB>(t, s);
        if (NT >= 16 || (row >> (KR - 4)) < NT) dst[(long long)row * Ccols + col] = v[s];
    }
}

// Final column store: rows t + G*s of column col (first n positions of the
// product).  Only a tile that reaches position n needs the per-slot bound
// check (tile-uniform branch); the others store through one base pointer.
template <int KR, int KC, int NT, int AR>
__device__ __forceinline__ void store_col(u32 *dst, const u32 (&v)[16], int t, long long col,
                                          long long tile_maxcol, const FourParams &P) {
    using C = ColCfg<KR>;
    constexpr long long Ccols = 1ll << KC;
    constexpr long long SLOT = (long long)C::G * Ccols;  // position stride of a slot
    u32 *base = dst + (long long)t * Ccols + col;
    if (15 * SLOT + (long long)(C::G - 1) * Ccols + tile_maxcol < P.n) {
#pragma unroll
        for (int s = 0; s < 16; ++s) __stcs(base + s * SLOT, canon_t<AR>(v[s], P.cs.p));
    } else {
        const long long idx0 = (long long)t * Ccols + col;
#pragma unroll
        for (int s = 0; s < 16; ++s)
            if (idx0 + s * SLOT < P.n) __stcs(base + s * SLOT, canon_t<AR>(v[s], P.cs.p));
    }
}

// Two adjacent columns per thread (col even, both below the wrap of the
// column rotation): 8-byte stores.  The output address of column col is
// congruent to the tile column modulo 8 words (out_rot), so it is 8-byte
// aligned.  A row's last position n - 1 may fall between the two columns.
template <int KR, int KC, int NT, int AR>
__device__ __forceinline__ void store_col2(u32 *dst, const u32 (&v0)[16], const u32 (&v1)[16],
                                           int t, long long col, long long tile_maxcol,
                                           const FourParams &P) {
    using C = ColCfg<KR>;
    constexpr long long Ccols = 1ll << KC;
    constexpr long long SLOT = (long long)C::G * Ccols;
    u32 *base = dst + (long long)t * Ccols + col;
    const u32 p = P.cs.p;
    if (15 * SLOT + (long long)(C::G - 1) * Ccols + tile_maxcol < P.n) {
#pragma unroll
        for (int s = 0; s < 16; ++s)
            __stcs(reinterpret_cast<uint2 *>(base + s * SLOT),
                   make_uint2(canon_t<AR>(v0[s], p), canon_t<AR>(v1[s], p)));
    } else {
        const long long idx0 = (long long)t * Ccols + col;
#pragma unroll
        for (int s = 0; s < 16; ++s) {
            if (idx0 + s * SLOT + 1 < P.n)
                __stcs(reinterpret_cast<uint2 *>(base + s * SLOT),
                       make_uint2(canon_t<AR>(v0[s], p), canon_t<AR>(v1[s], p)));
            else if (idx0 + s * SLOT < P.n)
                __stcs(base + s * SLOT, canon_t<AR>(v0[s], p));
        }
    }
}

// Inverse: R-point inverse DIT up each column; truncated (NT < 16): rows
// >= NT*R/16 hold the column time values, which are zero for a product of
// length <= NT*L/16, then the van der Hoeven top pass (ItftTop).
template <int KR, int KC, int NT, int AR = 0>
__global__ void __launch_bounds__(ColCfg<KR>::THREADS, ColCfg<KR>::MINB) col_inv_kernel(const FourParams P) {
    using C = ColCfg<KR>;
    constexpr long long Ccols = 1ll << KC;
    extern __shared__ uint4 smem_raw[];
    uint2 *tf_s = reinterpret_cast<uint2 *>(smem_raw);
    uint2 *ti_s = tf_s + C::R;
    u32 *tile = reinterpret_cast<u32 *>(tf_s + 2 * C::R);
    for (int i = threadIdx.x; i < C::R / 2; i += C::THREADS) {
        reinterpret_cast<uint4 *>(ti_s)[i] = __ldg(reinterpret_cast<const uint4 *>(P.col_ti) + i);
        if (NT < 16)
            reinterpret_cast<uint4 *>(tf_s)[i] =
                __ldg(reinterpret_cast<const uint4 *>(P.col_tf) + i);
    }
    const Tw W{tf_s, ti_s};
    const long long prod = P.prod0 + blockIdx.z;
    const u32 *src = P.Ah + (long long)blockIdx.z * (Ccols << KR);
    u32 *dst = P.c + prod * P.ldc;
    const int c = threadIdx.x % C::TC;
    const int t = threadIdx.x / C::TC;
    // scratch column j holds spectrum column (j - rot) mod C (out_rot)
    const int rot = out_rot(P, prod);
    const long long j0 = (long long)blockIdx.x * C::TC;
    const long long col = (j0 + c - rot) & (Ccols - 1);
    const long long maxcol = j0 >= rot ? j0 - rot + C::TC - 1 : Ccols - 1;
    mc_sync();

    u32 v[16];
    constexpr int SB = last_sb<KR>();
#pragma unroll
    for (int s = 0; s < 16; ++s) {
        const int row = slot_pos<SB>(t, s);
        v[s] = (NT >= 16 || (row >> (KR - 4)) < NT) ? src[(long long)row * Ccols + j0 + c] : 0u;
    }
    LayCol<C::TC, C::THREADS> lay{c};
    inv_lower_chain1<KR, Plan<KR>::NP - 1, LayCol<C::TC, C::THREADS>, NT, AR>(tile, v, t, P.cs, W, lay);
    inv_top<KR, NT, AR>(v, t, P.cs, W);
    store_col<KR, KC, NT, AR>(dst, v, t, col, maxcol, P);
}

// Forward column pass, TMA variant: persistent CTAs walk the (product,
// operand, column tile) list; each tile (R rows x TC columns) arrives by
// 3-D tensor-map bulk loads into one of two shared buffers while the
// previous tile is being transformed, so DRAM latency is off the critical
// path and the 16 strided scalar loads per thread disappear.
// CW = 2: every thread transforms two adjacent columns (half the threads):
// one set of twiddle loads and exchange addresses serves both, and the tile
// reads, exchanges and spectrum stores move 8-byte words.
#ifndef MC_COL_CW
#define MC_COL_CW 1
#endif

template <int KR, int KC, int NT, int AR = 0, int CW = 1, int TL = MC_COL_TILE>
__global__ void __launch_bounds__(ColCfg<KR, TL>::THREADS / CW, TL <= 8192 ? 2 : 1)
col_fwd_tma_kernel(const FourParams P, const __grid_constant__ CUtensorMap ta,
                   const __grid_constant__ CUtensorMap tb, int ntiles) {
    using C = ColCfg<KR, TL>;
    constexpr int THREADS = C::THREADS / CW;
    constexpr int BR = C::R < 256 ? C::R : 256;
    constexpr int NBOX = C::R / BR;
    constexpr long long Ccols = 1ll << KC;
    constexpr int CT = (1 << KC) / C::TC;  // column tiles per operand
    extern __shared__ __align__(1024) uint4 smem_raw[];
    uint2 *tf_s = reinterpret_cast<uint2 *>(smem_raw);
    u32 *buf0 = reinterpret_cast<u32 *>(tf_s + 2 * C::R);
    u32 *buf1 = buf0 + C::TILE;
    uint64_t *bar = reinterpret_cast<uint64_t *>(buf1 + C::TILE);
    const Tw W{tf_s, tf_s};
    const int c = CW * (threadIdx.x % (C::TC / CW));
    const int t = threadIdx.x / (C::TC / CW);
    const u32 p = P.cs.p;
    auto issue = [&](int tile, int k) {  // thread 0
        const int ct = tile % CT, op = (tile / CT) & 1, pc = tile / (2 * CT);
        u32 *dst = k ? buf1 : buf0;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(bar + k, (u32)(C::TILE * 4));
#pragma unroll
        for (int bx = 0; bx < NBOX; ++bx)
            tma_load_3d(dst + bx * BR * C::TC, op ? (const void *)&tb : (const void *)&ta,
                        ct * C::TC, bx * BR, (int)(P.prod0 + pc), bar + k);
    };
    // the first tile is requested before the stage table is read
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        fence_mbar_init();
        if ((int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    }
    for (int i = threadIdx.x; i < C::R / 2; i += THREADS)
        reinterpret_cast<uint4 *>(tf_s)[i] = __ldg(reinterpret_cast<const uint4 *>(P.col_tf) + i);
    mc_sync();
    uint32_t ph0 = 0, ph1 = 0;
    int k = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int ct = tile % CT, op = (tile / CT) & 1, pc = tile / (2 * CT);
        u32 *buf = k ? buf1 : buf0;
        if (k) {
            mbar_wait(bar + 1, ph1);
            ph1 ^= 1;
        } else {
            mbar_wait(bar, ph0);
            ph0 ^= 1;
        }
        const long long z = op ? P.z2 : P.z1;
        const int zrows = (int)((z + Ccols - 1) / Ccols);
        u32 *dst = (op ? P.Bh : P.Ah) + (long long)pc * (Ccols << KR);
        const long long col = (long long)ct * C::TC + c;
        constexpr int SB = last_sb<KR>();
        if constexpr (CW == 2) {
            u32 v0[16], v1[16];
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                const uint2 q = *reinterpret_cast<const uint2 *>(buf + (t + C::G * s) * C::TC + c);
                v0[s] = P.reduce ? mul_t<AR>(q.x, 1u, P.red_wp, p) : q.x;
                v1[s] = P.reduce ? mul_t<AR>(q.y, 1u, P.red_wp, p) : q.y;
            }
            mc_sync();  // tile consumed; the other buffer is free since last iteration
            if (threadIdx.x == 0 && tile + (int)gridDim.x < ntiles) issue(tile + gridDim.x, k ^ 1);
            fwd_top<KR, NT, AR>(v0, zrows, t, P.cs, W);
            fwd_top<KR, NT, AR>(v1, zrows, t, P.cs, W);
            LayCol<C::TC, THREADS, 2> lay{c};
            fwd_lower_chain2<KR, 0, LayCol<C::TC, THREADS, 2>, NT, AR>(buf, v0, v1, t, P.cs, W, lay);
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                const int row = slot_pos<SB>(t, s);
                if (NT >= 16 || (row >> (KR - 4)) < NT)
                    *reinterpret_cast<uint2 *>(dst + (long long)row * Ccols + col) =
                        make_uint2(v0[s], v1[s]);
            }
        } else {
            u32 v[16];
#pragma unroll
            for (int s = 0; s < 16; ++s) {  // plain row-major tile: conflict-free for this layout
                u32 x = buf[(t + C::G * s) * C::TC + c];
                if (P.reduce) x = mul_t<AR>(x, 1u, P.red_wp, p);
                v[s] = x;
            }
            mc_sync();  // tile consumed; the other buffer is free since last iteration
            if (threadIdx.x == 0 && tile + (int)gridDim.x < ntiles) issue(tile + gridDim.x, k ^ 1);
            fwd_top<KR, NT, AR>(v, zrows, t, P.cs, W);
            LayCol<C::TC, THREADS> lay{c};
            fwd_lower_chain1<KR, 0, LayCol<C::TC, THREADS>, NT, AR>(buf, v, t, P.cs, W, lay);
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                const int row = slot_pos<SB>(t, s);
                if (NT >= 16 || (row >> (KR - 4)) < NT) dst[(long long)row * Ccols + col] = v[s];
            }
        }
        k ^= 1;
    }
}

// Inverse column pass, async-copy variant: persistent CTAs; the next tile's
// rows arrive by 16-byte cp.async (LDGSTS.128, 4 per thread instead of 16
// scalar loads) into the other of two shared buffers while this tile is
// transformed.  Landing layout: row r at r*TC + (r/16)*8 words, which makes
// the first read (rows 16t + s, the last forward pass's layout) conflict-free.
template <int KR, int TL = MC_COL_TILE>
struct ColInvAsync {
    static constexpr int PADW = 8;  // words of padding per 16 rows
    static constexpr int BUFW = ColCfg<KR, TL>::TILE + (ColCfg<KR, TL>::R / 16) * PADW;
    static constexpr int SMEM = 2 * ColCfg<KR, TL>::R * 8 + 2 * BUFW * 4;
    __device__ static __forceinline__ int off(int row) {
        return row * ColCfg<KR, TL>::TC + (row >> 4) * PADW;
    }
};

template <int KR, int KC, int NT, int AR, int CW = 1, int TL = MC_COL_TILE>
__global__ void __launch_bounds__(ColCfg<KR, TL>::THREADS / CW, TL <= 8192 ? 2 : 1)
col_inv_async_kernel(const FourParams P, int ntiles) {
    using C = ColCfg<KR, TL>;
    using A = ColInvAsync<KR, TL>;
    constexpr int THREADS = C::THREADS / CW;
    constexpr long long Ccols = 1ll << KC;
    constexpr int CT = (1 << KC) / C::TC;
    constexpr int CHUNKS = C::TC / 4;     // 16-byte chunks per row
    constexpr int NR = NT * (C::R / 16);  // rows of the column spectrum that were formed
    extern __shared__ __align__(1024) uint4 smem_raw[];
    uint2 *tf_s = reinterpret_cast<uint2 *>(smem_raw);
    uint2 *ti_s = tf_s + C::R;
    u32 *bufs = reinterpret_cast<u32 *>(tf_s + 2 * C::R);
    const Tw W{tf_s, ti_s};
    const int c = CW * (threadIdx.x % (C::TC / CW));
    const int t = threadIdx.x / (C::TC / CW);
    auto issue = [&](int tile, int k) {  // every thread: its share of the tile's chunks
        const int ct = tile % CT, pc = tile / CT;
        const u32 *src = P.Ah + (long long)pc * (Ccols << KR) + (long long)ct * C::TC;
        u32 *dst = bufs + k * A::BUFW;
        for (int q = threadIdx.x; q < NR * CHUNKS; q += THREADS) {
            const int row = q / CHUNKS, ch = q % CHUNKS;
            const u32 *g = src + (long long)row * Ccols + 4 * ch;
            const u32 sa = smem_u32(dst + A::off(row) + 4 * ch);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if ((int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    // stage tables after the first tile's copies are in flight (the loop's first
    // barrier orders them before the transforms)
    for (int i = threadIdx.x; i < C::R / 2; i += THREADS) {
        reinterpret_cast<uint4 *>(ti_s)[i] = __ldg(reinterpret_cast<const uint4 *>(P.col_ti) + i);
        if (NT < 16)
            reinterpret_cast<uint4 *>(tf_s)[i] =
                __ldg(reinterpret_cast<const uint4 *>(P.col_tf) + i);
    }
    int k = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int ct = tile % CT, pc = tile / CT;
        u32 *buf = bufs + k * A::BUFW;
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        mc_sync();
        constexpr int SB = last_sb<KR>();
        u32 *dst = P.c + (P.prod0 + pc) * P.ldc;
        const int rot = out_rot(P, P.prod0 + pc);  // scratch column j = spectrum column j - rot
        const long long j0 = (long long)ct * C::TC;
        const long long col = (j0 + c - rot) & (Ccols - 1);
        const long long maxcol = j0 >= rot ? j0 - rot + C::TC - 1 : Ccols - 1;
        if constexpr (CW == 2) {
            u32 v0[16], v1[16];
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                const int row = slot_pos<SB>(t, s);
                const uint2 q = (NT >= 16 || (row >> (KR - 4)) < NT)
                                    ? *reinterpret_cast<const uint2 *>(buf + A::off(row) + c)
                                    : make_uint2(0u, 0u);
                v0[s] = q.x;
                v1[s] = q.y;
            }
            mc_sync();  // tile consumed; the other buffer is free
            if (tile + (int)gridDim.x < ntiles) issue(tile + gridDim.x, k ^ 1);
            LayCol<C::TC, THREADS, 2> lay{c};
            inv_lower_chain2<KR, Plan<KR>::NP - 1, LayCol<C::TC, THREADS, 2>, NT, AR>(buf, v0, v1, t,
                                                                                     P.cs, W, lay);
            inv_top<KR, NT, AR>(v0, t, P.cs, W);
            inv_top<KR, NT, AR>(v1, t, P.cs, W);
            if (j0 >= rot) {  // tile-uniform: the pair (col, col + 1) does not straddle the wrap
                store_col2<KR, KC, NT, AR>(dst, v0, v1, t, col, maxcol, P);
            } else {
                store_col<KR, KC, NT, AR>(dst, v0, t, col, maxcol, P);
                store_col<KR, KC, NT, AR>(dst, v1, t, (col + 1) & (Ccols - 1), maxcol, P);
            }
        } else {
            u32 v[16];
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                const int row = slot_pos<SB>(t, s);
                v[s] = (NT >= 16 || (row >> (KR - 4)) < NT) ? buf[A::off(row) + c] : 0u;
            }
            mc_sync();  // tile consumed; the other buffer is free
            if (tile + (int)gridDim.x < ntiles) issue(tile + gridDim.x, k ^ 1);
            LayCol<C::TC, THREADS> lay{c};
            inv_lower_chain1<KR, Plan<KR>::NP - 1, LayCol<C::TC, THREADS>, NT, AR>(buf, v, t, P.cs, W,
                                                                                  lay);
            inv_top<KR, NT, AR>(v, t, P.cs, W);
            store_col<KR, KC, NT, AR>(dst, v, t, col, maxcol, P);
        }
        k ^= 1;
    }
}

template <int KR, int KC, int NT, int AR, int CW = MC_COL_CW, int TL = MC_COL_TILE>
static cudaError_t launch_inv_async(const FourParams &P, cudaStream_t st) {
    using C = ColCfg<KR, TL>;
    static PerDevice<bool> ready_dev;
    bool &ready = ready_dev.get();
    if (!ready) {
        cudaError_t e = prep_kernel(col_inv_async_kernel<KR, KC, NT, AR, CW, TL>,
                                    ColInvAsync<KR, TL>::SMEM, C::THREADS / CW, nullptr);
        if (e != cudaSuccess) return e;
        ready = true;
    }
    const int ntiles = (int)((1ll << KC) / C::TC) * P.chunk;
    const int grid = std::min(ntiles, (C::TILE <= 8192 ? 2 : 1) * sm_count());
    col_inv_async_kernel<KR, KC, NT, AR, CW, TL>
        <<<grid, C::THREADS / CW, ColInvAsync<KR, TL>::SMEM, st>>>(P, ntiles);
    return cudaGetLastError();
}

// On by default (+1% on configs 4 and 5: the pass is bound by its instruction
// stream, not by the load latency this hides); MC_NO_COL_INV_ASYNC disables.
static bool col_inv_async_on() {
    static const bool on = [] { const char *e = getenv("MC_NO_COL_INV_ASYNC"); return !(e && *e); }();
    return on;
}

template <int KR, int KC, int NT, int AR, int CW = MC_COL_CW, int TL = MC_COL_TILE>
static cudaError_t launch_fwd_tma(const FourParams &P, const ColTma &M, cudaStream_t st) {
    using C = ColCfg<KR, TL>;
    constexpr int SMEM = 2 * C::R * 8 + 2 * C::TILE * 4 + 64;
    static PerDevice<bool> ready_dev;
    bool &ready = ready_dev.get();
    if (!ready) {
        cudaError_t e =
            prep_kernel(col_fwd_tma_kernel<KR, KC, NT, AR, CW, TL>, SMEM, C::THREADS / CW, nullptr);
        if (e != cudaSuccess) return e;
        ready = true;
    }
    const int ntiles = (int)((1ll << KC) / C::TC) * 2 * P.chunk;
    const int grid = std::min(ntiles, (C::TILE <= 8192 ? 2 : 1) * sm_count());
    col_fwd_tma_kernel<KR, KC, NT, AR, CW, TL>
        <<<grid, C::THREADS / CW, SMEM, st>>>(P, M.ma, M.mb, ntiles);
    return cudaGetLastError();
}

template <int KR, int KC, int NT, int AR = 0>
static cudaError_t launch_one(const FourParams &P, bool fwd, cudaStream_t st,
                              const ColTma *tma) {
    // bulk-copy / async variants need >= 16-byte tile rows (TC >= 4, KR <= 12)
    if constexpr (KR >= 6 && ColCfg<KR>::TILE >= 8192 && ColCfg<KR>::TC >= 4) {
        // complete transforms on L2-resident chunks: narrower tiles (FourParams::small_tiles)
        if constexpr (NT == 16 && ColCfg<KR, kSmallColTile>::TC >= 4) {
            if (P.small_tiles) {
                if (fwd && tma && tma->ok)
                    return launch_fwd_tma<KR, KC, NT, AR, 2, kSmallColTile>(P, *tma, st);
                if (!fwd && col_inv_async_on())
                    return launch_inv_async<KR, KC, NT, AR, 2, kSmallColTile>(P, st);
            }
        }
        if (fwd && tma && tma->ok) return launch_fwd_tma<KR, KC, NT, AR>(P, *tma, st);
        if (!fwd && col_inv_async_on()) return launch_inv_async<KR, KC, NT, AR>(P, st);
    }
    using C = ColCfg<KR>;
    static PerDevice<bool> ready_f_dev, ready_i_dev;
    bool &ready_f = ready_f_dev.get(), &ready_i = ready_i_dev.get();
    dim3 grid((unsigned)((1u << KC) / C::TC), fwd ? 2u : 1u, (unsigned)P.chunk);
    if (fwd) {
        if (!ready_f) {
            cudaError_t e =
                prep_kernel(col_fwd_kernel<KR, KC, NT, AR>, C::SMEM, C::THREADS, nullptr);
            if (e != cudaSuccess) return e;
            ready_f = true;
        }
        col_fwd_kernel<KR, KC, NT, AR><<<grid, C::THREADS, C::SMEM, st>>>(P);
    } else {
        if (!ready_i) {
            cudaError_t e =
                prep_kernel(col_inv_kernel<KR, KC, NT, AR>, C::SMEM, C::THREADS, nullptr);
            if (e != cudaSuccess) return e;
            ready_i = true;
        }
        col_inv_kernel<KR, KC, NT, AR><<<grid, C::THREADS, C::SMEM, st>>>(P);
    }
    return cudaGetLastError();
}

template <int KR, int KC>
static cudaError_t launch_nt(const FourParams &P, int NT, bool fwd, cudaStream_t st,
                             const ColTma *tma) {
    switch (NT) {
        case 9: return P.cs.ar == 1 ? launch_one<KR, KC, 9, 1>(P, fwd, st, tma)
                                 : launch_one<KR, KC, 9, 2>(P, fwd, st, tma);
        case 10: return P.cs.ar == 1 ? launch_one<KR, KC, 10, 1>(P, fwd, st, tma)
                                 : launch_one<KR, KC, 10, 2>(P, fwd, st, tma);
        case 11: return P.cs.ar == 1 ? launch_one<KR, KC, 11, 1>(P, fwd, st, tma)
                                 : launch_one<KR, KC, 11, 2>(P, fwd, st, tma);
        case 12: return P.cs.ar == 1 ? launch_one<KR, KC, 12, 1>(P, fwd, st, tma)
                                 : launch_one<KR, KC, 12, 2>(P, fwd, st, tma);
        case 13: return P.cs.ar == 1 ? launch_one<KR, KC, 13, 1>(P, fwd, st, tma)
                                 : launch_one<KR, KC, 13, 2>(P, fwd, st, tma);
        case 14: return P.cs.ar == 1 ? launch_one<KR, KC, 14, 1>(P, fwd, st, tma)
                                 : launch_one<KR, KC, 14, 2>(P, fwd, st, tma);
        case 15: return P.cs.ar == 1 ? launch_one<KR, KC, 15, 1>(P, fwd, st, tma)
                                 : launch_one<KR, KC, 15, 2>(P, fwd, st, tma);
        case 16:
            return P.cs.ar == 1 ? launch_one<KR, KC, 16, 1>(P, fwd, st, tma)
                                : launch_one<KR, KC, 16, 2>(P, fwd, st, tma);
        default: return cudaErrorInvalidValue;
    }
}

#define MC_CAT2(a, b) a##b
#define MC_CAT(a, b) MC_CAT2(a, b)

cudaError_t MC_CAT(launch_cols_kr, MC_KR)(const FourParams &P, int KC, int NT, bool fwd,
                                          cudaStream_t st, const ColTma *tma) {
#if MC_KR == 4
    switch (KC) {  // K = 14, 15, 16
        case 10: return launch_nt<4, 10>(P, NT, fwd, st, tma);
        case 11: return launch_nt<4, 11>(P, NT, fwd, st, tma);
        case 12: return launch_nt<4, 12>(P, NT, fwd, st, tma);
        default: return cudaErrorInvalidValue;
    }
#elif MC_KR >= 9 && MC_KR <= 12
    switch (KC) {  // K = 21..25 may use 2^13 rows (K = 25 always does)
        case 12: return launch_nt<MC_KR, 12>(P, NT, fwd, st, tma);
        case 13: return launch_nt<MC_KR, 13>(P, NT, fwd, st, tma);
        default: return cudaErrorInvalidValue;
    }
#elif MC_KR == 13
    if (KC != 13) return cudaErrorInvalidValue;  // K = 26
    return launch_nt<13, 13>(P, NT, fwd, st, tma);
#else
    if (KC != 12) return cudaErrorInvalidValue;
    return launch_nt<MC_KR, 12>(P, NT, fwd, st, tma);
#endif
}

}  // namespace mc
