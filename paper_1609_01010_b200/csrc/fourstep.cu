// Four-step large-transform convolution (see fourstep.cuh for the plan).
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include <cudaTypedefs.h>

#include "fourstep_int.cuh"

namespace mc {

// ---------------------------------------------------------------- row kernel
// The row transforms read one merged stage table (TwM: C - 1 + KC entries,
// half of separate forward and inverse tables), which leaves room for three
// 256-thread CTAs per SM at KC = 12 (80 registers, no spills).
#ifndef MC_ROW_TM  // 0: separate forward / inverse stage tables in the row pass (A/B)
#define MC_ROW_TM 1
#endif
#ifndef MC_ROW_MINB  // CTAs per SM of the 256-thread row pass (A/B: 3 measured slower)
#define MC_ROW_MINB 2
#endif
#ifndef MC_ROW_STAGE  // stage the next row pair in shared memory by bulk copies (A/B)
#define MC_ROW_STAGE 1
#endif

template <int KC>
struct RowCfg {
    static constexpr int C = 1 << KC;
    static constexpr int T = C / 16;
    static constexpr int PPC = T >= 128 ? 1 : 128 / T;
    static constexpr int THREADS = T * PPC;
    static_assert(THREADS == small_threads<KC>(), "exch_sync group barriers assume this CTA size");
    static constexpr int TM = (C - 1 + KC + 1) & ~1;  // merged-table entries (even)
    static constexpr int TABW = MC_ROW_TM ? TM : 2 * C;  // table entries in shared memory
    // with one row pair per CTA (PPC == 1) the next pair lands in a staging
    // area by bulk copies while the current one is transformed (TT path)
    static constexpr bool STAGE = MC_ROW_STAGE && PPC == 1;
    static constexpr int SMEM = TABW * 8 + PPC * (2 * C * 4 + 32 * 8) + (STAGE ? 2 * C * 4 + 16 : 0);
    static constexpr int MINB = THREADS >= 512 ? 1 : THREADS == 256 ? MC_ROW_MINB : 2;
};

// AR: arithmetic mode (modarith.cuh); inputs and outputs in [0, 2p).
// TT: twist factors read from the precomputed per-(p, L) tables P.twf / P.twi
// (one Shoup product per element and direction, L^-1 folded into the inverse
// table) instead of formed as alpha_t * beta_s (two products per element and
// direction plus the pointwise scale).  Work items are then row-major over
// the chunk's products (item = r * chunk + product), so the CTAs working on
// the same row r at the same time share its table row in L2.
// MC_ROW_PREFETCH: bulk-prefetch the next row's operand and twist-table rows
// into L2 while the current row is transformed (A/B with -DMC_ROW_PREFETCH=0).
#ifndef MC_ROW_PREFETCH
#define MC_ROW_PREFETCH 1
#endif

template <int KC, int AR = 0, bool TT = false>
__global__ void __launch_bounds__(RowCfg<KC>::THREADS, RowCfg<KC>::MINB)
row_conv_kernel(const FourParams P, int KR) {
    using RC = RowCfg<KC>;
    constexpr int Cn = RC::C, T = RC::T, G = Cn / 16;
    extern __shared__ uint4 smem_raw[];
    uint2 *tm_s = reinterpret_cast<uint2 *>(smem_raw);
    const int grp = threadIdx.x / T;
    const int t = threadIdx.x % T;
    u32 *bufA = reinterpret_cast<u32 *>(tm_s + RC::TABW) + grp * (2 * Cn + 64);
    u32 *bufB = bufA + Cn;
    uint2 *beta = reinterpret_cast<uint2 *>(bufB + Cn);  // [0,16) fwd, [16,32) inv
    const u32 p = P.cs.p;
    const long long R = 1ll << KR;
    const long long rows = P.nrows * P.chunk;  // truncated: only rows < nrows
    // staging of the next row pair (PPC == 1): [a row][b row][mbarrier]; the first
    // pair is requested before the stage table is read
    constexpr bool STG = RC::STAGE;  // both twist paths (row-major items with tables, else product-major)
    u32 *stA = reinterpret_cast<u32 *>(tm_s + RC::TABW) + RC::PPC * (2 * Cn + 64);
    u32 *stB = stA + Cn;
    uint64_t *mbar = reinterpret_cast<uint64_t *>(stB + Cn);
    auto stage = [&](long long g) {  // thread 0: bulk copies of work item g's rows
        const long long np = TT ? g % P.chunk : g / P.nrows;
        const long long nr = TT ? g / P.chunk : g % P.nrows;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(mbar, 8u * Cn);
        bulk_g2s(stA, P.Ah + np * (R << KC) + (nr << KC), 4u * Cn, mbar);
        bulk_g2s(stB, P.Bh + np * (R << KC) + (nr << KC), 4u * Cn, mbar);
    };
#if MC_ROW_TM
    if constexpr (STG) {
        // one round trip for the prologue: the merged stage table and the first
        // row pair land on the mbarrier's first phase (the grid never exceeds
        // the work items, so every CTA owns one)
        if (threadIdx.x == 0) {
            mbar_init(mbar, 1);
            fence_mbar_init();
            const long long g = blockIdx.x;
            const long long np = TT ? g % P.chunk : g / P.nrows;
            const long long nr = TT ? g / P.chunk : g % P.nrows;
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(mbar, 8u * Cn + 8u * RC::TM);
            bulk_g2s(stA, P.Ah + np * (R << KC) + (nr << KC), 4u * Cn, mbar);
            bulk_g2s(stB, P.Bh + np * (R << KC) + (nr << KC), 4u * Cn, mbar);
            bulk_g2s(tm_s, P.row_tm, 8u * RC::TM, mbar);
        }
    } else {
        const uint4 *gm = reinterpret_cast<const uint4 *>(P.row_tm);
        for (int i = threadIdx.x; i < RC::TM / 2; i += RC::THREADS)
            reinterpret_cast<uint4 *>(tm_s)[i] = __ldg(gm + i);
    }
    const TwM W{tm_s};
#else
    if (STG && threadIdx.x == 0) {
        mbar_init(mbar, 1);
        fence_mbar_init();
        if ((long long)blockIdx.x < rows) stage(blockIdx.x);
    }
    {
        const uint4 *gf = reinterpret_cast<const uint4 *>(P.row_tf);
        const uint4 *gi = reinterpret_cast<const uint4 *>(P.row_ti);
        for (int i = threadIdx.x; i < Cn / 2; i += RC::THREADS) {
            reinterpret_cast<uint4 *>(tm_s)[i] = __ldg(gf + i);
            reinterpret_cast<uint4 *>(tm_s + Cn)[i] = __ldg(gi + i);
        }
    }
    const Tw W{tm_s, tm_s + Cn};
#endif
    uint32_t phase = 0;
    mc_sync();

    for (long long base = (long long)blockIdx.x * RC::PPC; base < rows;
         base += (long long)gridDim.x * RC::PPC) {
        const long long gr = base + grp;
        const bool valid = gr < rows;
        if constexpr (TT) {
#if MC_ROW_PREFETCH
            // next rows of every row group: operand + twist rows into L2 (thread g
            // prefetches group g's next row)
            if (P.row_prefetch && threadIdx.x < RC::PPC) {
                const long long ng = base + (long long)gridDim.x * RC::PPC + threadIdx.x;
                if (ng < rows) {
                    const long long np = ng % P.chunk, nr = ng / P.chunk;
                    if (!STG) {
                        bulk_prefetch_l2(P.Ah + np * (R << KC) + (nr << KC), 4u * Cn);
                        bulk_prefetch_l2(P.Bh + np * (R << KC) + (nr << KC), 4u * Cn);
                    }
                    bulk_prefetch_l2(P.twf + (nr << KC), 8u * Cn);
                    bulk_prefetch_l2(P.twi + (nr << KC), 8u * Cn);
                }
            }
#endif
            const long long prod = valid ? gr % P.chunk : 0;
            const long long r = valid ? gr / P.chunk : 0;
            u32 *rowA = P.Ah + prod * (R << KC) + (r << KC);
            const u32 *rowB = P.Bh + prod * (R << KC) + (r << KC);
            const uint2 *twf = P.twf + (r << KC);
            const uint2 *twi = P.twi + (r << KC);
            u32 va[16], vb[16];
            if constexpr (STG) {  // the row pair landed in the staging area
                mbar_wait(mbar, phase);
                phase ^= 1;
#pragma unroll
                for (int s = 0; s < 16; ++s) {
                    const int x = t + G * s;
                    const uint2 w = __ldg(twf + x);
                    va[s] = mul_t<AR>(stA[x], w.x, w.y, p);
                    vb[s] = mul_t<AR>(stB[x], w.x, w.y, p);
                }
                mc_sync();  // staging consumed: bring in the next work item's rows
                const long long ng = base + (long long)gridDim.x;
                if (threadIdx.x == 0 && ng < rows) stage(ng);
            } else {
#pragma unroll
                for (int s = 0; s < 16; ++s) {
                    const int x = t + G * s;
                    const uint2 w = __ldg(twf + x);
                    va[s] = mul_t<AR>(valid ? rowA[x] : 0u, w.x, w.y, p);
                    vb[s] = mul_t<AR>(valid ? rowB[x] : 0u, w.x, w.y, p);
                }
            }
            fwd_top<KC, 16, AR>(va, Cn, t, P.cs, W);
            fwd_top<KC, 16, AR>(vb, Cn, t, P.cs, W);
            fwd_lower_chain<KC, 16, 0, AR, std::remove_const_t<decltype(W)>, false>(bufA, bufB, va, vb, t, P.cs, W);
#pragma unroll
            for (int s = 0; s < 16; ++s) va[s] = mont_mul(va[s], vb[s], p, P.cs.pinv);
            inv_lower_chain<KC, 16, Plan<KC>::NP - 1, AR>(bufA, va, t, P.cs, W);
            ItftTop<KC, 16, 16, 0, AR>::run(va, t, P.cs, W);
            if (valid) {
                const int rot = out_rot(P, P.prod0 + prod);
#pragma unroll
                for (int s = 0; s < 16; ++s) {
                    const int x = t + G * s;
                    const uint2 w = __ldg(twi + x);  // w^-(x f1) * L^-1 * 2^32
                    rowA[(x + rot) & (Cn - 1)] = mul_inv_t<AR>(va[s], w.x, w.y, p);
                }
            }
            mc_sync();
            continue;
        }
        const long long prod = valid ? gr / P.nrows : 0;
        const u32 r = valid ? (u32)(gr % P.nrows) : 0u;
        const u32 f1 = __brev(r) >> (32 - KR);
        if (t < 32) {  // per-row twist factors beta_s = w^(f1*G*s), and inverses
            const int s = t & 15;
            const u32 e = f1 * (u32)G * (u32)s;
            const u32 w = (t < 16) ? pow_w(P.tw.lo_f, P.tw.hi_f, e, p)
                                   : pow_w(P.tw.lo_i, P.tw.hi_i, e, p);
            beta[t] = make_uint2(w, shoup_comp(w, p, P.tw.two32_over_p));
        }
        // per-thread twist factors alpha_t = w^(f1*t), and inverse
        const u32 ea = f1 * (u32)t;
        const u32 af = pow_w(P.tw.lo_f, P.tw.hi_f, ea, p);
        const u32 ai = pow_w(P.tw.lo_i, P.tw.hi_i, ea, p);
        const u32 afp = shoup_comp(af, p, P.tw.two32_over_p);
        const u32 aip = shoup_comp(ai, p, P.tw.two32_over_p);
        u32 *rowA = P.Ah + prod * (R << KC) + ((long long)r << KC);
        const u32 *rowB = P.Bh + prod * (R << KC) + ((long long)r << KC);
        mc_sync();

        u32 va[16], vb[16];
        if constexpr (STG) {  // the row pair landed in the staging area
            mbar_wait(mbar, phase);
            phase ^= 1;
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                const int x = t + G * s;
                const uint2 bt = beta[s];
                va[s] = mul_t<AR>(mul_t<AR>(stA[x], af, afp, p), bt.x, bt.y, p);
                vb[s] = mul_t<AR>(mul_t<AR>(stB[x], af, afp, p), bt.x, bt.y, p);
            }
            mc_sync();  // staging consumed: bring in the next work item's rows
            const long long ng = base + (long long)gridDim.x;
            if (threadIdx.x == 0 && ng < rows) stage(ng);
        } else {
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                const int x = t + G * s;
                const uint2 bt = beta[s];
                va[s] = mul_t<AR>(mul_t<AR>(valid ? rowA[x] : 0u, af, afp, p), bt.x, bt.y, p);
                vb[s] = mul_t<AR>(mul_t<AR>(valid ? rowB[x] : 0u, af, afp, p), bt.x, bt.y, p);
            }
        }
        fwd_top<KC, 16, AR>(va, Cn, t, P.cs, W);
        fwd_top<KC, 16, AR>(vb, Cn, t, P.cs, W);
        fwd_lower_chain<KC, 16, 0, AR, std::remove_const_t<decltype(W)>, false>(bufA, bufB, va, vb, t, P.cs, W);
#pragma unroll
        for (int s = 0; s < 16; ++s)
            va[s] = mul_inv_t<AR>(mont_mul(va[s], vb[s], p, P.cs.pinv), P.cs.linv_mont, p);
        inv_lower_chain<KC, 16, Plan<KC>::NP - 1, AR>(bufA, va, t, P.cs, W);
        ItftTop<KC, 16, 16, 0, AR>::run(va, t, P.cs, W);
        if (valid) {
            const int rot = out_rot(P, P.prod0 + prod);
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                const uint2 bt = beta[16 + s];
                rowA[(t + G * s + rot) & (Cn - 1)] =
                    mul_inv_t<AR>(mul_inv_t<AR>(va[s], ai, aip, p), bt.x, bt.y, p);
            }
        }
        mc_sync();
    }
}

// ---------------------------------------------------------------- host side
struct TwistHost {
    u32 *lo_f = nullptr, *lo_i = nullptr;
    uint2 *hi_f = nullptr, *hi_i = nullptr;
};

static std::mutex g_tw_mu;
static std::map<std::tuple<int, u32, u32, int>, TwistHost> g_tw;  // (dev, p, w_L, K)

static mc_status get_twist(const FieldTables *T, TwistTabs *out) {
    const int K = T->log2L;
    const u32 p = T->p;
    const int dev = current_device();
    auto key = std::make_tuple(dev, p, T->root, K);
    std::lock_guard<std::mutex> lock(g_tw_mu);
    auto it = g_tw.find(key);
    if (it == g_tw.end()) {
        const u64 nlo = 4096, nhi = (K > 12) ? (1ull << (K - 12)) : 1;
        std::vector<u32> lf(nlo), li(nlo);
        std::vector<uint2> hf(nhi), hi(nhi);
        const u32 w = T->root, wi = inv_mod(w, p);
        u64 a = 1, ai = 1;
        for (u64 j = 0; j < nlo; ++j) {
            lf[j] = (u32)a;
            li[j] = (u32)ai;
            a = mulmod(a, w, p);
            ai = mulmod(ai, wi, p);
        }
        const u64 step = powmod(w, 4096, p), stepi = powmod(wi, 4096, p);
        a = ai = 1;
        for (u64 j = 0; j < nhi; ++j) {
            Shoup sf = shoup((u32)a, p), si = shoup((u32)ai, p);
            hf[j] = make_uint2(sf.w, sf.wp);
            hi[j] = make_uint2(si.w, si.wp);
            a = mulmod(a, step, p);
            ai = mulmod(ai, stepi, p);
        }
        TwistHost h;
        cudaError_t e = cudaMalloc(&h.lo_f, 4 * nlo);
        if (e == cudaSuccess) e = cudaMalloc(&h.lo_i, 4 * nlo);
        if (e == cudaSuccess) e = cudaMalloc(&h.hi_f, 8 * nhi);
        if (e == cudaSuccess) e = cudaMalloc(&h.hi_i, 8 * nhi);
        if (e == cudaSuccess) e = cudaMemcpy(h.lo_f, lf.data(), 4 * nlo, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(h.lo_i, li.data(), 4 * nlo, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(h.hi_f, hf.data(), 8 * nhi, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(h.hi_i, hi.data(), 8 * nhi, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cuda_fail(e, "twist table upload");
        it = g_tw.emplace(key, h).first;
    }
    out->lo_f = it->second.lo_f;
    out->lo_i = it->second.lo_i;
    out->hi_f = it->second.hi_f;
    out->hi_i = it->second.hi_i;
    out->two32_over_p = 4294967296.0 / (double)p;
    return MC_OK;
}

// Full twist tables for the row pass (FourParams::twf / twi), built on the
// device once per (device, p, K, KC) and kept: 16 B per transform position
// (128 MiB at L = 2^23).  Used up to L = 2^MC_TWIST_TABLE_MAX_K (default 24);
// MC_NO_TWIST_TABLE=1 forms the twists on the fly instead (A/B).
__global__ void twist_table_kernel(TwistTabs tw, int KR, int KC, u32 p, Shoup scale,
                                   uint2 *outf, uint2 *outi) {
    const long long L = 1ll << (KR + KC);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < L;
         i += (long long)gridDim.x * blockDim.x) {
        const u32 r = (u32)(i >> KC), x = (u32)(i & ((1ll << KC) - 1));
        const u32 e = x * (__brev(r) >> (32 - KR));  // < L <= 2^26
        const u32 wf = pow_w(tw.lo_f, tw.hi_f, e, p);
        const u32 wi = mul_shoup(pow_w(tw.lo_i, tw.hi_i, e, p), scale, p);
        outf[i] = make_uint2(wf, shoup_comp(wf, p, tw.two32_over_p));
        outi[i] = make_uint2(wi, shoup_comp(wi, p, tw.two32_over_p));
    }
}

struct FullTwist {
    uint2 *f = nullptr, *i = nullptr;
};
static std::map<std::tuple<int, u32, u32, int, int>, FullTwist> g_full_tw;

static bool twist_table_on(int K) {
    static const int max_k = [] {
        const char *e = getenv("MC_NO_TWIST_TABLE");
        if (e && *e) return 0;
        const char *m = getenv("MC_TWIST_TABLE_MAX_K");
        return m && *m ? atoi(m) : 24;
    }();
    return K <= max_k;
}

static mc_status get_full_twist(const FieldTables *T, const TwistTabs &tw, int KC,
                                const uint2 **f, const uint2 **i) {
    const int K = T->log2L, KR = K - KC;
    const int dev = current_device();
    auto key = std::make_tuple(dev, T->p, T->root, K, KC);
    std::lock_guard<std::mutex> lock(g_tw_mu);
    auto it = g_full_tw.find(key);
    if (it == g_full_tw.end()) {
        FullTwist h;
        const size_t bytes = sizeof(uint2) << K;
        cudaError_t e = cudaMalloc(&h.f, bytes);
        if (e == cudaSuccess) e = cudaMalloc(&h.i, bytes);
        if (e != cudaSuccess) {
            cudaFree(h.f);
            cudaGetLastError();
            return cuda_fail(e, "twist table allocation");
        }
        // L^-1 * 2^32 (the Montgomery pointwise product leaves a 2^-32)
        const Shoup scale = T->linv_mont;
        // built on a private stream and finished before the tables are
        // published: later calls on any stream may use them at once
        cudaStream_t bs = nullptr;
        e = cudaStreamCreateWithFlags(&bs, cudaStreamNonBlocking);
        if (e == cudaSuccess) {
            twist_table_kernel<<<4 * sm_count(), 256, 0, bs>>>(tw, KR, KC, T->p, scale, h.f, h.i);
            note_launches(1);
            e = cudaGetLastError();
            if (e == cudaSuccess) e = cudaStreamSynchronize(bs);
            cudaStreamDestroy(bs);
        }
        if (e != cudaSuccess) return cuda_fail(e, "twist table build");
        it = g_full_tw.emplace(key, h).first;
    }
    *f = it->second.f;
    *i = it->second.i;
    return MC_OK;
}

mc_status get_twist_tables(u32 p, int K, const u32 **lo_f, const uint2 **hi_f, const u32 **lo_i,
                           const uint2 **hi_i) {
    const FieldTables *T;
    mc_status s = get_tables(p, K, &T);
    if (s != MC_OK) return s;
    TwistTabs tw;
    if ((s = get_twist(T, &tw)) != MC_OK) return s;
    *lo_f = tw.lo_f;
    *hi_f = tw.hi_f;
    *lo_i = tw.lo_i;
    *hi_i = tw.hi_i;
    return MC_OK;
}

template <int KC, int AR, bool TT>
static cudaError_t launch_rows_lz(const FourParams &P, int KR, cudaStream_t st) {
    using RC = RowCfg<KC>;
    static PerDevice<int> per_sm_dev;
    int &per_sm = per_sm_dev.get();
    if (!per_sm) {
        cudaError_t e = prep_kernel(row_conv_kernel<KC, AR, TT>, RC::SMEM, RC::THREADS, &per_sm);
        if (e != cudaSuccess) return e;
    }
    long long work = (P.nrows * P.chunk + RC::PPC - 1) / RC::PPC;
    long long grid = std::min<long long>(work, (long long)per_sm * sm_count());
    row_conv_kernel<KC, AR, TT><<<(unsigned)grid, RC::THREADS, RC::SMEM, st>>>(P, KR);
    return cudaGetLastError();
}

template <int KC>
static cudaError_t launch_rows(const FourParams &P, int KR, cudaStream_t st) {
    if (P.twf)
        return P.cs.ar == 1 ? launch_rows_lz<KC, 1, true>(P, KR, st)
                            : launch_rows_lz<KC, 2, true>(P, KR, st);
    return P.cs.ar == 1 ? launch_rows_lz<KC, 1, false>(P, KR, st)
                        : launch_rows_lz<KC, 2, false>(P, KR, st);
}

static cudaError_t launch_cols_any(int KC, int KR, int NT, const FourParams &P, bool fwd,
                                   cudaStream_t st, const ColTma *tma = nullptr) {
    switch (KR) {
        case 4: return launch_cols_kr4(P, KC, NT, fwd, st, tma);
        case 5: return launch_cols_kr5(P, KC, NT, fwd, st, tma);
        case 6: return launch_cols_kr6(P, KC, NT, fwd, st, tma);
        case 7: return launch_cols_kr7(P, KC, NT, fwd, st, tma);
        case 8: return launch_cols_kr8(P, KC, NT, fwd, st, tma);
        case 9: return launch_cols_kr9(P, KC, NT, fwd, st, tma);
        case 10: return launch_cols_kr10(P, KC, NT, fwd, st, tma);
        case 11: return launch_cols_kr11(P, KC, NT, fwd, st, tma);
        case 12: return launch_cols_kr12(P, KC, NT, fwd, st, tma);
        case 13: return launch_cols_kr13(P, KC, NT, fwd, st, tma);
        default: return cudaErrorInvalidValue;
    }
}

// Tensor maps for the TMA forward column pass ({C, z/C, batch} per operand);
// ok = 0 when the operands do not fit the bulk-tensor constraints.
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}

static ColTma make_col_tma(const u32 *a, long long lda, long long z1, const u32 *b, long long ldb,
                          long long z2, long long batch, int KC, int KR, int tile) {
    ColTma M;
    memset(&M, 0, sizeof(M));
    static const bool off = [] { const char *e = getenv("MC_NO_COL_TMA"); return e && *e; }();
    const long long C = 1ll << KC;
    const int TC = tile >> KR;
    const int BR = std::min(1 << KR, 256);
    auto enc = tensor_map_encoder();
    if (off || !enc || KR < 6 || (z1 % C) || (z2 % C) || (lda % 4) || (ldb % 4) ||
        ((uintptr_t)a % 16) || ((uintptr_t)b % 16) || batch > 0x7fffffff)
        return M;
    auto one = [&](CUtensorMap *m, const u32 *base, long long ld, long long z) {
        cuuint64_t dims[3] = {(cuuint64_t)C, (cuuint64_t)(z / C), (cuuint64_t)batch};
        cuuint64_t strides[2] = {(cuuint64_t)C * 4, (cuuint64_t)ld * 4};
        cuuint32_t box[3] = {(cuuint32_t)TC, (cuuint32_t)BR, 1};
        cuuint32_t es[3] = {1, 1, 1};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, (void *)base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    M.ok = one(&M.ma, a, lda, z1) && one(&M.mb, b, ldb, z2);
    return M;
}

static cudaError_t launch_rows_any(int KC, int KR, const FourParams &P, cudaStream_t st) {
    switch (KC) {
        case 10: return launch_rows<10>(P, KR, st);
        case 11: return launch_rows<11>(P, KR, st);
        case 12: return launch_rows<12>(P, KR, st);
        case 13: return launch_rows<13>(P, KR, st);
        default: return cudaErrorInvalidValue;
    }
}

// scratch budget per chunk (default 512 MiB: bigger launches beat L2 residency,
// the four-step passes are integer-pipe bound; profiles/r01/README.md)
static long long scratch_budget_words() {
    static const long long budget_words = [] {
        const char *e = getenv("MC_FOURSTEP_SCRATCH_MB");
        return (e ? atoll(e) : 512ll) << 18;  // MiB -> 32-bit words
    }();
    return budget_words;
}

mc_status fourstep_plan(int engine, const u32 *a, long long lda, int z1, const u32 *b,
                        long long ldb, int z2, u32 *c, long long ldc, long long batch, u32 p,
                        int circ_log2L, bool reduce_inputs, FourPlan *F) {
    const bool circ = circ_log2L >= 0;
    const long long n = circ ? (1ll << circ_log2L) : (long long)z1 + z2 - 1;
    int K = 0;
    while ((1ll << K) < n) ++K;
    if (circ) K = circ_log2L;
    const FieldTables *TL, *TR, *TC;
    mc_status s = get_tables(p, K, &TL);  // the reference's 2-adicity check
    if (s != MC_OK) return s;
    F->K = K;
    if (K > kFourStepMaxK) return MC_OK;  // levels_conv territory (caller checks K)
    // Row length C = 2^KC: 2^12 (measured better than 2^13 at K = 23, whose
    // wider column tiles do not pay for the 1-CTA/SM K=13 row pass, and than
    // 2^11 at K = 21 and 23); MC_FOURSTEP_KC overrides for A/B runs.
    static const int kc_env = [] {
        const char *e = getenv("MC_FOURSTEP_KC");
        return e ? atoi(e) : 0;
    }();
    int KC = std::min(12, K - 4);
    if (K - KC > 12) KC = 13;  // K = 25, 26: 2^13-point rows, 2^12 / 2^13-point columns
    if (kc_env >= 10 && kc_env <= 13 && K - kc_env >= 4 && K - kc_env <= 12 &&
        (kc_env == 12 || kc_env == 13 || K - kc_env == 4))
        KC = kc_env;
    const int KR = K - KC;
    if ((s = get_tables(p, KR, &TR)) != MC_OK) return s;
    if ((s = get_tables(p, KC, &TC)) != MC_OK) return s;
    FourParams &P = F->P;
    memset(&P, 0, sizeof(P));
    if ((s = get_twist(TL, &P.tw)) != MC_OK) return s;
    // Full twist tables pay when several products share each table row (the
    // row items of a chunk are row-major over its products); a single product
    // reads every row once from DRAM, and forming the twists from the small
    // power tables is faster there (config 5, one product per prime: 123.8 ->
    // 121.2 us; config 4, 8 products: 1.063 ms with the tables, 1.166 without)
    static const bool tw_single = [] { const char *e = getenv("MC_TWIST_SINGLE"); return e && *e; }();
    if (twist_table_on(K) && (batch >= 2 || tw_single) &&
        (s = get_full_twist(TL, P.tw, KC, &P.twf, &P.twi)) != MC_OK)
        return s;
    P.cs.p = p;
    memcpy(P.cs.mlev, TR->mlev, sizeof(P.cs.mlev));  // column-level ITFT constants
    memcpy(P.cs.hinv, TR->hinv, sizeof(P.cs.hinv));
    // tf[h + j] = w_{2h}^j does not depend on L: the lowest-pass constants of
    // the column and row transforms are the same
    memcpy(P.cs.c16f, TR->h16f, sizeof(P.cs.c16f));
    memcpy(P.cs.c16fd, TR->h16fd, sizeof(P.cs.c16fd));
    memcpy(P.cs.c16id, TR->h16id, sizeof(P.cs.c16id));
    memcpy(P.cs.c16i, TR->h16i, sizeof(P.cs.c16i));
    P.cs.pinv = TL->pinv;
    P.cs.linv_mont = TL->linv_mont;  // 1/L for the whole transform
    P.a = a;
    P.b = b;
    P.c = c;
    P.lda = lda;
    P.ldb = ldb;
    P.ldc = ldc;
    P.z1 = circ ? n : z1;
    P.z2 = circ ? n : z2;
    P.n = n;
    P.reduce = reduce_inputs ? 1 : 0;
    P.red_wp = (u32)((1ull << 32) / p);
    P.col_tf = TR->tf;
    P.col_ti = TR->ti;
    P.row_tf = TC->tf;
    P.row_ti = TC->ti;
    P.row_tm = TC->tm;
    const long long L = 1ll << K;
    // Truncation (tft engine): relaxed to L/16 granularity like the fused
    // kernel; the column transforms are truncated at NT of their 16 top
    // blocks and the row pass only forms rows < NT * R/16.
    int NT = 16;
    if (engine == 1 && !circ) NT = (int)((n + (L >> 4) - 1) / (L >> 4));
    if (NT == 15 && lazy_ok(p)) NT = 16;  // as the fused path (capi.cu conv_dispatch)
    P.nrows = (long long)NT << (KR - 4);
    // Harvey ranges for p < 2^30 on every pass: the row transforms are complete
    // whatever NT, and the truncated column passes canonicalise the operands of
    // their van der Hoeven steps like the fused kernel's
    P.cs.ar = lazy_ok(p) ? 1 : 2;
    F->KC = KC;
    F->KR = KR;
    F->NT = NT;
    F->L = L;
    F->batch = batch;
    // narrower column tiles when one chunk's spectra (2L words per product)
    // stay in L2; MC_SMALL_COL_TILES=0/1 forces (A/B)
    {
        const long long chunk = std::max(1ll, std::min(batch, scratch_budget_words() / (2 * L)));
        P.small_tiles = NT == 16 && KR <= 11 && 8 * L * chunk <= (16ll << 20);
        if (const char *f = getenv("MC_SMALL_COL_TILES"))
            if (*f) P.small_tiles = atoi(f) && NT == 16 && KR <= 11;
    }
    F->tma = make_col_tma(a, lda, P.z1, b, ldb, P.z2, batch, KC, KR,
                          P.small_tiles ? kSmallColTile : MC_COL_TILE);
    return MC_OK;
}

cudaError_t fourstep_fwd_rows(FourPlan &F, long long p0, int chunk, cudaStream_t st) {
    FourParams &P = F.P;
    P.prod0 = p0;
    P.chunk = chunk;
    // operand rows + twist tables of one chunk: prefetching pays once they
    // cannot stay in the 126 MB L2 (config 4: -2.4%; config 5, 48 MB per
    // prime: +1.3% without this gate)
    P.row_prefetch = 8ll * F.L * P.chunk + 16ll * F.L > (96ll << 20) ? 1 : 0;
    if (const char *f = getenv("MC_ROW_PREFETCH"))  // 0/1: force (sanitizer / A/B runs)
        if (*f) P.row_prefetch = atoi(f) ? 1 : 0;
    cudaError_t e = launch_cols_any(F.KC, F.KR, F.NT, P, true, st, &F.tma);
    if (e == cudaSuccess) e = launch_rows_any(F.KC, F.KR, P, st);
    note_launches(2);
    return e;
}

cudaError_t fourstep_inv_cols(FourPlan &F, cudaStream_t st) {
    note_launches(1);
    return launch_cols_any(F.KC, F.KR, F.NT, F.P, false, st);
}

mc_status fourstep_conv(int engine, const u32 *a, long long lda, int z1, const u32 *b,
                        long long ldb, int z2, u32 *c, long long ldc, long long batch, u32 p,
                        cudaStream_t st, int circ_log2L, bool reduce_inputs, bool fold) {
    FourPlan F;
    mc_status s = fourstep_plan(engine, a, lda, z1, b, ldb, z2, c, ldc, batch, p, circ_log2L,
                                reduce_inputs, &F);
    if (s != MC_OK) return s;
    if (fold) {  // split truncated product head: circular product of the folded operands
        if (circ_log2L < 0 || F.K > kFourStepMaxK) return fail(MC_EINVAL, "fold needs a circular plan");
        F.P.z1 = z1;
        F.P.z2 = z2;
        F.P.fold = 1;
        F.tma.ok = 0;  // plain column loads (the tensor maps cover L words)
    }
    if (F.K > kFourStepMaxK)  // L = 2^27 (p3 only): level-scheduled transforms
        return levels_conv(a, lda, z1, b, ldb, z2, c, ldc, batch, p, F.K,
                           circ_log2L >= 0 ? (1ll << circ_log2L) : (long long)z1 + z2 - 1, st);
    const long long L = F.L;
    const long long chunk = std::max(1ll, std::min(batch, scratch_budget_words() / (2 * L)));
    u32 *scratch = nullptr;
    keep_pool_memory();
    MC_CUDA_CHECK(cudaMallocAsync(&scratch, sizeof(u32) * 2 * L * chunk, st));
    F.P.Ah = scratch;
    F.P.Bh = scratch + L * chunk;
    mc_status result = MC_OK;
    for (long long p0 = 0; p0 < batch && result == MC_OK; p0 += chunk) {
        cudaError_t e = fourstep_fwd_rows(F, p0, (int)std::min(chunk, batch - p0), st);
        if (e == cudaSuccess) e = fourstep_inv_cols(F, st);
        if (e != cudaSuccess) result = cuda_fail(e, "four-step launch");
    }
    cudaFreeAsync(scratch, st);
    return result;
}

}  // namespace mc
