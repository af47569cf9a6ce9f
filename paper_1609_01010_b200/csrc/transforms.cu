// Standalone transforms with the reference's exact semantics (API parity,
// SURVEY.md 8f row 1):
//   mc_ntt   transform.py:167-196  natural order in and out, inverse / L
//   mc_tft   transform.py:379-448  first n bit-reversed spectral values
//   mc_itft  transform.py:451-529  L * u_i, i < n, from n spectral values
//
// Three tiers: the fused register-pass kernels (xform_small.cuh) for moddft
// and tft with n > L/2 at 16 <= L <= 8192; row-resident shared-memory
// kernels (rows_kernel) for the exact truncated transforms (itft, tft with
// n <= L/2) at L <= 2^14; otherwise level-scheduled on global memory: one
// launch per butterfly level over all rows of the batch (any L up to 2^27,
// limited by the field).  Twiddles
// w_{2h}^j = w_L^(j*L/2h) come from the two-level power tables of the
// four-step path (lo[e & 4095] * hi[e >> 12]); the variable-twiddle
// products use Montgomery multiplication with the twiddle in Montgomery
// form.  These entry points exist for call-compatibility of
// moddft/tft/itft; the convolution hot path never uses them.
#include <algorithm>
#include <vector>

#include "fourstep.cuh"
#include "runtime.h"
#include "xform_small.cuh"

namespace mc {

struct TfmTabs {
    const u32 *lo_f;
    const uint2 *hi_f;
    const u32 *lo_i;
    const uint2 *hi_i;
};

// defined in fourstep.cu
mc_status get_twist_tables(u32 p, int K, const u32 **lo_f, const uint2 **hi_f, const u32 **lo_i,
                           const uint2 **hi_i);

struct TfmParams {
    u32 *w;           // work rows [batch][ldw]
    long long ldw;
    long long batch;
    int K;            // log2 L
    u32 p, pinv;
    u32 r2;           // 2^64 mod p (to enter Montgomery form)
    TfmTabs tb;
};

__device__ __forceinline__ u32 tw_pow(const u32 *lo, const uint2 *hi, u32 e, u32 p) {
    const uint2 h = __ldg(hi + (e >> 12));
    return mul_shoup(__ldg(lo + (e & 4095)), h.x, h.y, p);
}

// x * w mod p, w canonical (variable): Montgomery with an R^2 correction.
__device__ __forceinline__ u32 mulv(u32 x, u32 w, const TfmParams &P) {
    return mont_mul(mont_mul(x, w, P.p, P.pinv), P.r2, P.p, P.pinv);
}

// w_{2h}^j for the stage with half-size h (both directions)
__device__ __forceinline__ u32 stage_tw(const TfmParams &P, long long h, long long j, bool inv) {
    const u32 e = (u32)(j << (P.K - 1 - __ffsll(h) + 1));  // j * L / (2h)
    return inv ? tw_pow(P.tb.lo_i, P.tb.hi_i, e, P.p) : tw_pow(P.tb.lo_f, P.tb.hi_f, e, P.p);
}

// --- moddft -------------------------------------------------------------
__global__ void bitrev_copy_kernel(const u32 *x, u32 *w, long long ldw, long long batch, int K) {
    const long long L = 1ll << K;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < L * batch;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i >> K, j = i & (L - 1);
        const long long rj = K ? (long long)(__brevll((unsigned long long)j) >> (64 - K)) : 0;
        w[r * ldw + rj] = x[r * L + j];
    }
}

__global__ void dit_stage_kernel(TfmParams P, long long h, int inv) {
    const long long L = 1ll << P.K, half = L >> 1;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < half * P.batch;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / half, k = i % half;
        const long long j = k & (h - 1), blk = k / h;
        u32 *row = P.w + r * P.ldw;
        const long long lo = blk * 2 * h + j, hi = lo + h;
        const u32 t = mulv(row[hi], stage_tw(P, h, j, inv), P);
        const u32 u = row[lo];
        row[lo] = add_mod(u, t, P.p);
        row[hi] = sub_mod(u, t, P.p);
    }
}

__global__ void scale_copy_kernel(const u32 *w, long long ldw, u32 *y, long long n, long long ldy,
                                  long long batch, u32 s, u32 sp, u32 p, int do_scale) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n * batch;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / n, j = i % n;
        u32 v = w[r * ldw + j];
        if (do_scale) v = mul_shoup(v, s, sp, p);
        y[r * ldy + j] = v;
    }
}

// --- truncated forward ----------------------------------------------------
// One DIF level (block size m = 2h) of the reference recursion
// (transform.py:379-418), all computed blocks (start < n) at once.
__global__ void tft_level_kernel(TfmParams P, long long h, long long z, long long n) {
    const long long m = 2 * h;
    const long long nblk = (n + m - 1) / m;
    const long long per = nblk * h;
    const long long zz = z < m ? z : m;  // every computed block holds min(z, m) inputs
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < per * P.batch;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / per, k = i % per;
        const long long b = (k / h) * m, j = k % h;
        if (j >= zz) continue;  // both inputs known zero
        u32 *row = P.w + r * P.ldw;
        const bool b_zero = j + h >= zz;
        const bool hi_needed = b + h < n;
        const long long lo = b + j, hi = lo + h;
        if (hi_needed) {
            const u32 w = stage_tw(P, h, j, false);
            if (b_zero) {
                row[hi] = mulv(row[lo], w, P);
            } else {
                const u32 a = row[lo], c = row[hi];
                row[lo] = add_mod(a, c, P.p);
                row[hi] = mulv(sub_mod(a, c, P.p), w, P);
            }
        } else if (!b_zero) {
            row[lo] = add_mod(row[lo], row[hi], P.p);
        }
    }
}

__global__ void load_pad_kernel(const u32 *x, long long ldx, long long z, u32 *w, long long ldw,
                                long long L, long long batch, u32 p, u32 red_wp) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < L * batch;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / L, j = i % L;
        w[r * ldw + j] = j < z ? mul_shoup(x[r * ldx + j], 1u, red_wp, p) : 0u;
    }
}

// --- truncated inverse ----------------------------------------------------
// Chain of the van der Hoeven recursion (transform.py:451-489): complete
// sub-blocks are plain inverse DITs (done first, all at once); the partial
// path is walked top-down (cross / pre-add) and then bottom-up (DIT /
// combine).
struct Block {
    long long off, size;
};

constexpr int kMaxBlocks = 40;

struct BlockList {
    Block b[kMaxBlocks];
    long long pre[kMaxBlocks + 1];  // prefix sums of per-stage butterflies
    int nb;
};

__global__ void blocks_dit_stage_kernel(TfmParams P, BlockList BL, long long h) {
    const long long total = BL.pre[BL.nb];
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total * P.batch;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / total, k = i % total;
        int q = 0;
        while (k >= BL.pre[q + 1]) ++q;
        const long long kk = k - BL.pre[q];
        const long long j = kk & (h - 1), blk = kk / h;
        u32 *row = P.w + r * P.ldw + BL.b[q].off;
        const long long lo = blk * 2 * h + j, hi = lo + h;
        const u32 t = mulv(row[hi], stage_tw(P, h, j, true), P);
        const u32 u = row[lo];
        row[lo] = add_mod(u, t, P.p);
        row[hi] = sub_mod(u, t, P.p);
    }
}

// kind: 0 pre-add, 1 combine, 2 cross, 3 DIT; range [i0, i1) of offsets
__global__ void chain_op_kernel(TfmParams P, long long off, long long h, long long i0,
                                long long i1, int kind, Shoup m_mod, Shoup inv_h) {
    const long long cnt = i1 - i0;
    if (cnt <= 0) return;
    const u32 p = P.p;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < cnt * P.batch;
         t += (long long)gridDim.x * blockDim.x) {
        const long long r = t / cnt, i = i0 + t % cnt;
        u32 *row = P.w + r * P.ldw + off;
        const long long lo = i, hi = i + h;
        if (kind == 0) {
            row[lo] = add_mod(row[lo], row[hi], p);
        } else if (kind == 1) {
            const u32 a = row[lo];
            row[lo] = sub_mod(add_mod(a, a, p), mul_shoup(row[hi], m_mod, p), p);
        } else if (kind == 2) {
            const u32 a = row[lo], b = row[hi];
            const u32 d = sub_mod(mul_shoup(a, inv_h, p), add_mod(b, b, p), p);
            row[hi] = mulv(d, stage_tw(P, h, i, false), P);
            row[lo] = sub_mod(add_mod(a, a, p), mul_shoup(b, m_mod, p), p);
        } else {
            const u32 tt = mulv(row[hi], stage_tw(P, h, i, true), P);
            const u32 a = row[lo];
            row[lo] = add_mod(a, tt, p);
            row[hi] = sub_mod(a, tt, p);
        }
    }
}

// ---------------------------------------------------------------- host helpers
static unsigned grid_for(long long work) {
    long long g = (work + 255) / 256;
    long long cap = (long long)sm_count() * 16;
    if (g > cap) g = cap;
    return (unsigned)(g < 1 ? 1 : g);
}

static mc_status tfm_setup(u32 p, int K, TfmParams *P) {
    const FieldTables *T;
    mc_status s = get_tables(p, K, &T);
    if (s != MC_OK) return s;
    if ((s = get_twist_tables(p, K, &P->tb.lo_f, &P->tb.hi_f, &P->tb.lo_i, &P->tb.hi_i)) != MC_OK)
        return s;
    P->K = K;
    P->p = p;
    P->pinv = T->pinv;
    const u64 r1 = (1ull << 32) % p;
    P->r2 = (u32)mulmod(r1, r1, p);
    return MC_OK;
}

__global__ void pointwise_kernel(u32 *x, const u32 *y, long long L, TfmParams P) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < L;
         i += (long long)gridDim.x * blockDim.x)
        x[i] = mulv(x[i], y[i], P);
}

mc_status levels_conv(const u32 *a, long long lda, int z1, const u32 *b, long long ldb, int z2,
                      u32 *c, long long ldc, long long batch, u32 p, int K, long long n,
                      cudaStream_t st) {
    TfmParams P;
    memset(&P, 0, sizeof(P));
    mc_status s = tfm_setup(p, K, &P);
    if (s != MC_OK || batch == 0) return s;
    const long long L = 1ll << K;
    const u32 red_wp = (u32)((1ull << 32) / p);
    u32 *buf = nullptr;
    keep_pool_memory();
    MC_CUDA_CHECK(cudaMallocAsync(&buf, 4ull * 3 * L, st));
    u32 *wa = buf, *wb = buf + L, *tmp = buf + 2 * L;
    P.ldw = L;
    P.batch = 1;
    const FieldTables *T;
    get_tables(p, K, &T);
    auto forward = [&](const u32 *x, long long ldx, long long z, u32 *w) {
        // zero-padded, reduced copy, then the bit-reversed DIT = natural-order spectrum
        load_pad_kernel<<<grid_for(L), 256, 0, st>>>(x, ldx, z, tmp, L, L, 1, p, red_wp);
        bitrev_copy_kernel<<<grid_for(L), 256, 0, st>>>(tmp, w, L, 1, K);
        P.w = w;
        for (long long h = 1; h < L; h <<= 1)
            dit_stage_kernel<<<grid_for(L / 2), 256, 0, st>>>(P, h, 0);
    };
    for (long long r = 0; r < batch; ++r) {
        forward(a + r * lda, lda, z1, wa);
        forward(b + r * ldb, ldb, z2, wb);
        pointwise_kernel<<<grid_for(L), 256, 0, st>>>(wa, wb, L, P);
        bitrev_copy_kernel<<<grid_for(L), 256, 0, st>>>(wa, tmp, L, 1, K);
        P.w = tmp;
        for (long long h = 1; h < L; h <<= 1)
            dit_stage_kernel<<<grid_for(L / 2), 256, 0, st>>>(P, h, 1);
        scale_copy_kernel<<<grid_for(n), 256, 0, st>>>(tmp, L, c + r * ldc, n, ldc, 1, T->linv.w,
                                                       T->linv.wp, p, 1);
        note_launches(8 + 3 * K);
    }
    cudaFreeAsync(buf, st);
    MC_CUDA_CHECK(cudaGetLastError());
    return MC_OK;
}

// ---------------------------------------------------------------- row-resident (L <= 2^14)
// Exact truncated transforms with one CTA per row and the row resident in
// shared memory: every level of the reference recursion is one pass over
// the row between two barriers, twiddles are the Shoup stage tables
// (tf/ti, L2-resident).  Serves itft (every n) and tft with n <= L/2 (the
// fused register passes take n > L/2), replacing one launch per level on
// global memory.
constexpr int kRowsMaxK = 14;
constexpr int kChainMax = 16;

struct RowsParams {
    const u32 *x;
    long long ldx;
    u32 *y;
    long long ldy;
    long long batch;
    int K, z, n;
    u32 p, red_wp;
    const uint2 *tf;  // tf[h + j] = w_{2h}^j (Shoup pairs)
    const uint2 *ti;  // ti[h + j] = w_{2h}^-j
    // itft: the partial path of the van der Hoeven recursion, top-down
    int nc, nbig;  // chain nodes; the first nbig have h > 32 (CTA-wide), the rest run on one warp
    int c_off[kChainMax], c_h[kChainMax], c_n[kChainMax];
    Shoup c_mm[kChainMax], c_ih[kChainMax];  // m mod p, h^-1 mod p of each node
};

__device__ __forceinline__ u32 mul_tw(u32 x, uint2 w, u32 p) { return mul_shoup(x, w.x, w.y, p); }

// Row in shared memory, one pad word per 16 (position x at x + x/16): the
// stride-16 accesses of the register passes hit 32 distinct banks.
struct PadRow {
    u32 *s;
    int off;
    __device__ __forceinline__ u32 &operator[](int x) const {
        const int y = off + x;
        return s[y + (y >> 4)];
    }
};

// NB inverse DIT stages (h = S .. S 2^(NB-1)) in registers on each of the
// `full` aligned S 2^NB-chunks at the start of the row: item k = (chunk,
// offset o < S) holds the 2^NB elements chunk*S 2^NB + o + q S.
template <int NB>
__device__ __forceinline__ void dit_reg_pass(const PadRow &s, const uint2 *ti, int S, int lgS,
                                             int full, int tid, int nth, u32 p) {
    constexpr int E = 1 << NB;
    for (int k = tid; k < (full << lgS); k += nth) {
        const int o = k & (S - 1);
        const PadRow base{s.s, ((k >> lgS) << (lgS + NB)) + o};
        u32 v[E];
#pragma unroll
        for (int q = 0; q < E; ++q) v[q] = base[q * S];
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int hh = S << b;
#pragma unroll
            for (int q = 0; q < E; ++q) {
                if (q & (1 << b)) continue;
                const int j = (q & ((1 << b) - 1)) * S + o;
                const u32 t = mul_tw(v[q + (1 << b)], __ldg(ti + hh + j), p);
                const u32 a = v[q];
                v[q] = add_mod(a, t, p);
                v[q + (1 << b)] = sub_mod(a, t, p);
            }
        }
#pragma unroll
        for (int q = 0; q < E; ++q) base[q * S] = v[q];
    }
}

// MODE 0: tft (transform.py:379-418, levels top-down, pruned by z and n);
// MODE 1: itft (transform.py:451-489): the complete sub-blocks of the
// recursion are the aligned 2h-chunks inside [0, n) (the blocks are the
// binary decomposition of n), run as inverse DIT stages bottom-up; then the
// partial path top-down (cross / pre-add) and bottom-up (DIT / combine).
template <int MODE>
__global__ void __launch_bounds__(512) rows_kernel(const RowsParams P) {
    extern __shared__ uint4 smem_rows[];
    const PadRow s{reinterpret_cast<u32 *>(smem_rows), 0};
    const int L = 1 << P.K, n = P.n, NTH = blockDim.x, tid = threadIdx.x;
    const u32 p = P.p;
    for (long long r = blockIdx.x; r < P.batch; r += gridDim.x) {
        const u32 *xr = P.x + r * P.ldx;
        const int zin = MODE == 0 ? P.z : n;
        mc_sync();  // the previous row's stores have read s
        for (int i = tid; i < L; i += NTH) s[i] = i < zin ? mul_shoup(__ldcs(xr + i), 1u, P.red_wp, p) : 0u;
        mc_sync();
        if (MODE == 0) {
            for (int h = L >> 1; h >= 1; h >>= 1) {
                const int m = 2 * h, lgh = __ffs(h) - 1;
                const int nblk = (n + m - 1) / m;
                const int zz = P.z < m ? P.z : m;
                const int per = nblk * h;
                for (int k = tid; k < per; k += NTH) {
                    const int j = k & (h - 1);
                    if (j >= zz) continue;
                    const int lo = ((k >> lgh) << (lgh + 1)) + j, hi = lo + h;
                    const bool b_zero = j + h >= zz;
                    if (lo - j + h < n) {  // hi output needed
                        const uint2 w = __ldg(P.tf + h + j);
                        if (b_zero) {
                            s[hi] = mul_tw(s[lo], w, p);
                        } else {
                            const u32 a = s[lo], c = s[hi];
                            s[lo] = add_mod(a, c, p);
                            s[hi] = mul_tw(sub_mod(a, c, p), w, p);
                        }
                    } else if (!b_zero) {
                        s[lo] = add_mod(s[lo], s[hi], p);
                    }
                }
                mc_sync();
            }
        } else {
            // 1. complete blocks: inverse DIT, stage h over the aligned 2h-chunks
            // below n.  NB <= 4 stages at a time (h = S .. S 2^(NB-1)) run in
            // registers on the aligned S 2^NB-chunks below n (2^NB elements at
            // stride S per thread), NB the most stages that still have a
            // complete chunk; the tail [chunks, n) runs those stages one at a
            // time.  When no chunk of two stages' size fits, no stage is left.
            for (int h = 1; h < L;) {
                const int lgS = __ffs(h) - 1;
                int nb = min(4, P.K - lgS);
                while (nb > 0 && (n >> (lgS + nb)) == 0) --nb;
                if (nb == 0) break;
                const int full = n >> (lgS + nb);
                switch (nb) {
                    case 4: dit_reg_pass<4>(s, P.ti, h, lgS, full, tid, NTH, p); break;
                    case 3: dit_reg_pass<3>(s, P.ti, h, lgS, full, tid, NTH, p); break;
                    case 2: dit_reg_pass<2>(s, P.ti, h, lgS, full, tid, NTH, p); break;
                    default: dit_reg_pass<1>(s, P.ti, h, lgS, full, tid, NTH, p); break;
                }
                // tail stages (disjoint from the chunks above)
                for (int b = 0; b < nb; ++b) {
                    const int hh = h << b, lgh = lgS + b;
                    const int k0 = (full << (lgS + nb)) >> 1, per = (n >> (lgh + 1)) << lgh;
                    if (per > k0) {
                        for (int k = k0 + tid; k < per; k += NTH) {
                            const int j = k & (hh - 1);
                            const int lo = ((k >> lgh) << (lgh + 1)) + j, hi = lo + hh;
                            const u32 t = mul_tw(s[hi], __ldg(P.ti + hh + j), p);
                            const u32 a = s[lo];
                            s[lo] = add_mod(a, t, p);
                            s[hi] = sub_mod(a, t, p);
                        }
                        mc_sync();
                    }
                }
                mc_sync();
                h <<= nb;
            }
            // 2./3. the partial path: down (cross butterflies where n > h, else
            // pre-adds), then up (DIT butterflies / combines).  Nodes with
            // h > 32 run on the whole CTA, one barrier each; the small nodes at
            // the bottom of the path (a region of <= 64 elements) run on warp 0
            // between two warp barriers, down and back up without a CTA barrier.
            auto node_down = [&](int c, int first, int step) {
                const int off = P.c_off[c], h = P.c_h[c], nn = P.c_n[c];
                const PadRow row{s.s, off};
                if (nn > h) {
                    const Shoup mm = P.c_mm[c], ih = P.c_ih[c];
                    for (int i = nn - h + first; i < h; i += step) {
                        const u32 a = row[i], b = row[i + h];
                        const u32 d = sub_mod(mul_shoup(a, ih, p), add_mod(b, b, p), p);
                        row[i + h] = mul_tw(d, __ldg(P.tf + h + i), p);
                        row[i] = sub_mod(add_mod(a, a, p), mul_shoup(b, mm, p), p);
                    }
                } else {
                    for (int i = nn + first; i < h; i += step) row[i] = add_mod(row[i], row[i + h], p);
                }
            };
            auto node_up = [&](int c, int first, int step) {
                const int off = P.c_off[c], h = P.c_h[c], nn = P.c_n[c];
                const PadRow row{s.s, off};
                if (nn > h) {
                    for (int i = first; i < nn - h; i += step) {
                        const u32 t = mul_tw(row[i + h], __ldg(P.ti + h + i), p);
                        const u32 a = row[i];
                        row[i] = add_mod(a, t, p);
                        row[i + h] = sub_mod(a, t, p);
                    }
                } else {
                    const Shoup mm = P.c_mm[c];
                    for (int i = first; i < nn; i += step) {
                        const u32 a = row[i];
                        row[i] = sub_mod(add_mod(a, a, p), mul_shoup(row[i + h], mm, p), p);
                    }
                }
            };
            for (int c = 0; c < P.nbig; ++c) {
                node_down(c, tid, NTH);
                mc_sync();
            }
            if (P.nbig < P.nc) {
                if (tid < 32) {
                    for (int c = P.nbig; c < P.nc; ++c) {
                        node_down(c, tid, 32);
                        __syncwarp();
                        mc_perturb();
                    }
                    for (int c = P.nc - 1; c >= P.nbig; --c) {
                        node_up(c, tid, 32);
                        __syncwarp();
                        mc_perturb();
                    }
                }
                mc_sync();
            }
            for (int c = P.nbig - 1; c >= 0; --c) {
                node_up(c, tid, NTH);
                mc_sync();
            }
        }
        u32 *yr = P.y + r * P.ldy;
        for (int i = tid; i < n; i += NTH) __stcs(yr + i, s[i]);
    }
}

static mc_status rows_launch(int mode, const u32 *x, long long ldx, int z, u32 *y, long long ldy,
                             int n, int K, long long batch, u32 p, cudaStream_t st) {
    const FieldTables *T;
    mc_status s = get_tables(p, K, &T);
    if (s != MC_OK) return s;
    RowsParams R;
    memset(&R, 0, sizeof(R));
    R.x = x;
    R.ldx = ldx;
    R.y = y;
    R.ldy = ldy;
    R.batch = batch;
    R.K = K;
    R.z = z;
    R.n = n;
    R.p = p;
    R.red_wp = (u32)((1ull << 32) / p);
    R.tf = T->tf;
    R.ti = T->ti;
    if (mode == 1) {  // partial path of _itft_recurse (transform.py:451-489)
        long long off = 0, m = 1ll << K, nn = n;
        while (m > 1 && nn > 0 && nn < m) {
            const long long h = m >> 1;
            if (R.nc >= kChainMax) return fail(MC_EINVAL, "itft chain too long");
            R.c_off[R.nc] = (int)off;
            R.c_h[R.nc] = (int)h;
            R.c_n[R.nc] = (int)nn;
            R.c_mm[R.nc] = shoup((u32)(m % p), p);
            R.c_ih[R.nc] = shoup(inv_mod((u32)(h % p), p), p);
            ++R.nc;
            if (nn > h) {
                off += h;
                nn -= h;
            }
            m = h;
        }
        while (R.nbig < R.nc && R.c_h[R.nbig] > 32) ++R.nbig;
    }
    const int L = 1 << K;
    const int threads = std::max(32, std::min(512, L / 16));
    const size_t smem = 4ull * (L + L / 16 + 1);
    static PerDevice<bool> attr_dev;
    if (bool &attr = attr_dev.get(); !attr) {
        constexpr int max_dyn = 4 * ((1 << kRowsMaxK) + (1 << (kRowsMaxK - 4)) + 1);
        MC_CUDA_CHECK(cudaFuncSetAttribute(rows_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn));
        MC_CUDA_CHECK(cudaFuncSetAttribute(rows_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn));
        attr = true;
    }
    const int per_sm = std::max(1, std::min(2048 / threads, (int)((200u << 10) / smem)));
    const long long grid = std::min<long long>(batch, (long long)sm_count() * per_sm);
    if (mode == 0)
        rows_kernel<0><<<(unsigned)grid, threads, smem, st>>>(R);
    else
        rows_kernel<1><<<(unsigned)grid, threads, smem, st>>>(R);
    note_launches(1);
    MC_CUDA_CHECK(cudaGetLastError());
    return MC_OK;
}

// ---------------------------------------------------------------- fused (L <= 8192)
// MC_XFORM_LEVELS (non-empty) forces the level-scheduled kernels (A/B, parity).
static bool xform_levels_forced() {
    static const bool on = [] { const char *e = getenv("MC_XFORM_LEVELS"); return e && *e; }();
    return on;
}

cudaError_t launch_xform_small_k4(const XformParams &, int, int, cudaStream_t);
cudaError_t launch_xform_small_k5(const XformParams &, int, int, cudaStream_t);
cudaError_t launch_xform_small_k6(const XformParams &, int, int, cudaStream_t);
cudaError_t launch_xform_small_k7(const XformParams &, int, int, cudaStream_t);
cudaError_t launch_xform_small_k8(const XformParams &, int, int, cudaStream_t);
cudaError_t launch_xform_small_k9(const XformParams &, int, int, cudaStream_t);
cudaError_t launch_xform_small_k10(const XformParams &, int, int, cudaStream_t);
cudaError_t launch_xform_small_k11(const XformParams &, int, int, cudaStream_t);
cudaError_t launch_xform_small_k12(const XformParams &, int, int, cudaStream_t);
cudaError_t launch_xform_small_k13(const XformParams &, int, int, cudaStream_t);

// Fused single-CTA transform (xform_small.cuh); K in [4, kSmallMaxK].
static mc_status xform_small(int mode, const u32 *x, long long ldx, int z, u32 *y, long long ldy,
                             int n, int K, long long batch, u32 p, cudaStream_t st) {
    const FieldTables *T;
    mc_status s = get_tables(p, K, &T);
    if (s != MC_OK) return s;
    XformParams X;
    memset(&X, 0, sizeof(X));
    X.cs.p = p;
    X.cs.pinv = T->pinv;
    X.cs.tf = T->tf;
    X.cs.ti = T->ti;
    memcpy(X.cs.c16f, T->h16f, sizeof(X.cs.c16f));
    memcpy(X.cs.c16fd, T->h16fd, sizeof(X.cs.c16fd));
    memcpy(X.cs.c16id, T->h16id, sizeof(X.cs.c16id));
    memcpy(X.cs.c16i, T->h16i, sizeof(X.cs.c16i));
    memcpy(X.cs.mlev, T->mlev, sizeof(X.cs.mlev));
    memcpy(X.cs.hinv, T->hinv, sizeof(X.cs.hinv));
    X.x = x;
    X.ldx = ldx;
    X.y = y;
    X.ldy = ldy;
    X.z = z;
    X.n = n;
    X.batch = batch;
    X.linv = T->linv;
    X.red_wp = (u32)((1ull << 32) / p);
    const int G = 1 << (K - 4);
    const int nt = (n + G - 1) / G;
    cudaError_t e;
    switch (K) {
        case 4: e = launch_xform_small_k4(X, mode, nt, st); break;
        case 5: e = launch_xform_small_k5(X, mode, nt, st); break;
        case 6: e = launch_xform_small_k6(X, mode, nt, st); break;
        case 7: e = launch_xform_small_k7(X, mode, nt, st); break;
        case 8: e = launch_xform_small_k8(X, mode, nt, st); break;
        case 9: e = launch_xform_small_k9(X, mode, nt, st); break;
        case 10: e = launch_xform_small_k10(X, mode, nt, st); break;
        case 11: e = launch_xform_small_k11(X, mode, nt, st); break;
        case 12: e = launch_xform_small_k12(X, mode, nt, st); break;
        case 13: e = launch_xform_small_k13(X, mode, nt, st); break;
        default: return fail(MC_EINVAL, "fused transform size");
    }
    note_launches(1);
    if (e != cudaSuccess) return cuda_fail(e, "fused transform launch");
    return MC_OK;
}

}  // namespace mc

using namespace mc;

extern "C" {

mc_status mc_ntt(const uint32_t *x, uint32_t *y, int32_t log2L, int64_t batch, uint32_t p,
                 int inverse, void *stream) {
    if (log2L < 0 || log2L > 30) return fail(MC_EINVAL, "bad transform size");
    if (batch < 0) return fail(MC_EINVAL, "negative batch");
    TfmParams P;
    memset(&P, 0, sizeof(P));
    mc_status s = tfm_setup(p, log2L, &P);
    if (s != MC_OK || batch == 0) return s;
    if (!x || !y) return fail(MC_EINVAL, "null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    const long long L = 1ll << log2L;
    if (log2L >= 4 && log2L <= kSmallMaxK && !xform_levels_forced())
        return xform_small(inverse ? MODE_NTT_INV : MODE_NTT_FWD, x, L, (int)L, y, L, (int)L,
                           log2L, batch, p, st);
    u32 *w = nullptr;
    keep_pool_memory();
    MC_CUDA_CHECK(cudaMallocAsync(&w, 4ull * L * batch, st));
    P.w = w;
    P.ldw = L;
    P.batch = batch;
    bitrev_copy_kernel<<<grid_for(L * batch), 256, 0, st>>>(x, w, L, batch, log2L);
    for (long long h = 1; h < L; h <<= 1)
        dit_stage_kernel<<<grid_for(L / 2 * batch), 256, 0, st>>>(P, h, inverse ? 1 : 0);
    const FieldTables *T;
    get_tables(p, log2L, &T);
    scale_copy_kernel<<<grid_for(L * batch), 256, 0, st>>>(w, L, y, L, L, batch, T->linv.w,
                                                           T->linv.wp, p, inverse ? 1 : 0);
    note_launches(2 + log2L);
    cudaFreeAsync(w, st);
    MC_CUDA_CHECK(cudaGetLastError());
    return MC_OK;
}

mc_status mc_tft(const uint32_t *x, int32_t z, uint32_t *y, int32_t n, int32_t log2L,
                 int64_t batch, uint32_t p, void *stream) {
    if (log2L < 0 || log2L > 30) return fail(MC_EINVAL, "bad transform size");
    const long long L = 1ll << log2L;
    if (z < 1) return fail(MC_EINVAL, "input must be nonempty");
    if (z > n) return fail(MC_EINVAL, "input length exceeds output count");
    if (n > L) return fail(MC_EINVAL, "output count exceeds transform size");
    if (batch < 0) return fail(MC_EINVAL, "negative batch");
    TfmParams P;
    memset(&P, 0, sizeof(P));
    mc_status s = tfm_setup(p, log2L, &P);
    if (s != MC_OK || batch == 0) return s;
    if (!x || !y) return fail(MC_EINVAL, "null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    if (log2L >= 4 && log2L <= kSmallMaxK && 2ll * n > L && !xform_levels_forced())
        return xform_small(MODE_TFT, x, z, z, y, n, n, log2L, batch, p, st);
    if (log2L <= kRowsMaxK && !xform_levels_forced())
        return rows_launch(0, x, z, z, y, n, n, log2L, batch, p, st);
    u32 *w = nullptr;
    keep_pool_memory();
    MC_CUDA_CHECK(cudaMallocAsync(&w, 4ull * L * batch, st));
    P.w = w;
    P.ldw = L;
    P.batch = batch;
    load_pad_kernel<<<grid_for(L * batch), 256, 0, st>>>(x, z, z, w, L, L, batch, p,
                                                         (u32)((1ull << 32) / p));
    int launches = 2;
    for (long long h = L >> 1; h >= 1; h >>= 1) {
        const long long nblk = (n + 2 * h - 1) / (2 * h);
        tft_level_kernel<<<grid_for(nblk * h * batch), 256, 0, st>>>(P, h, z, n);
        ++launches;
    }
    scale_copy_kernel<<<grid_for((long long)n * batch), 256, 0, st>>>(w, L, y, n, n, batch, 0, 0,
                                                                      p, 0);
    note_launches(launches);
    cudaFreeAsync(w, st);
    MC_CUDA_CHECK(cudaGetLastError());
    return MC_OK;
}

mc_status mc_itft(const uint32_t *xhat, uint32_t *y, int32_t n, int32_t log2L, int64_t batch,
                  uint32_t p, void *stream) {
    if (log2L < 0 || log2L > 30) return fail(MC_EINVAL, "bad transform size");
    const long long L = 1ll << log2L;
    if (n < 1) return fail(MC_EINVAL, "spectral input must be nonempty");
    if (n > L) return fail(MC_EINVAL, "input length exceeds transform size");
    if (batch < 0) return fail(MC_EINVAL, "negative batch");
    TfmParams P;
    memset(&P, 0, sizeof(P));
    mc_status s = tfm_setup(p, log2L, &P);
    if (s != MC_OK || batch == 0) return s;
    if (!xhat || !y) return fail(MC_EINVAL, "null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    if (log2L <= kRowsMaxK && !xform_levels_forced())
        return rows_launch(1, xhat, n, n, y, n, n, log2L, batch, p, st);
    u32 *w = nullptr;
    keep_pool_memory();
    MC_CUDA_CHECK(cudaMallocAsync(&w, 4ull * L * batch, st));
    P.w = w;
    P.ldw = L;
    P.batch = batch;
    load_pad_kernel<<<grid_for(L * batch), 256, 0, st>>>(xhat, n, n, w, L, L, batch, p,
                                                         (u32)((1ull << 32) / p));
    int launches = 2;
    // Walk the partial path: nodes (off, m, n) with 0 < n < m.
    struct Node {
        long long off, m, n;
    };
    std::vector<Node> chain;
    BlockList BL;
    memset(&BL, 0, sizeof(BL));
    {
        long long off = 0, m = L, nn = n;
        while (m > 1 && nn > 0) {
            if (nn == m) {  // complete: plain inverse DIT of the whole block
                BL.b[BL.nb++] = Block{off, m};
                break;
            }
            const long long h = m >> 1;
            chain.push_back(Node{off, m, nn});
            if (nn <= h) {
                m = h;
            } else {
                BL.b[BL.nb++] = Block{off, h};  // complete first half
                off += h;
                nn -= h;
                m = h;
            }
        }
    }
    // 1. complete blocks, stage by stage (bottom-up)
    for (long long h = 1; h < L; h <<= 1) {
        BlockList sub;
        memset(&sub, 0, sizeof(sub));
        for (int q = 0; q < BL.nb; ++q)
            if (BL.b[q].size >= 2 * h) {
                sub.b[sub.nb] = BL.b[q];
                sub.pre[sub.nb + 1] = sub.pre[sub.nb] + BL.b[q].size / 2;
                ++sub.nb;
            }
        if (!sub.nb) break;
        blocks_dit_stage_kernel<<<grid_for(sub.pre[sub.nb] * batch), 256, 0, st>>>(P, sub, h);
        ++launches;
    }
    // 2. down the chain: cross (n > h) or pre-add (n <= h)
    for (const Node &nd : chain) {
        const long long h = nd.m >> 1;
        const Shoup mm = shoup((u32)(nd.m % p), p);
        const Shoup ih = shoup(inv_mod((u32)(h % p), p), p);
        if (nd.n > h)
            chain_op_kernel<<<grid_for((2 * h - nd.n) * batch), 256, 0, st>>>(
                P, nd.off, h, nd.n - h, h, 2, mm, ih);
        else
            chain_op_kernel<<<grid_for((h - nd.n) * batch), 256, 0, st>>>(P, nd.off, h, nd.n, h,
                                                                          0, mm, ih);
        ++launches;
    }
    // 3. up the chain: DIT (n > h) or combine (n <= h)
    for (auto it = chain.rbegin(); it != chain.rend(); ++it) {
        const Node &nd = *it;
        const long long h = nd.m >> 1;
        const Shoup mm = shoup((u32)(nd.m % p), p);
        const Shoup ih = shoup(inv_mod((u32)(h % p), p), p);
        if (nd.n > h)
            chain_op_kernel<<<grid_for((nd.n - h) * batch), 256, 0, st>>>(P, nd.off, h, 0,
                                                                          nd.n - h, 3, mm, ih);
        else
            chain_op_kernel<<<grid_for(nd.n * batch), 256, 0, st>>>(P, nd.off, h, 0, nd.n, 1, mm,
                                                                    ih);
        ++launches;
    }
    scale_copy_kernel<<<grid_for((long long)n * batch), 256, 0, st>>>(w, L, y, n, n, batch, 0, 0,
                                                                      p, 0);
    note_launches(launches);
    cudaFreeAsync(w, st);
    MC_CUDA_CHECK(cudaGetLastError());
    return MC_OK;
}

}  // extern "C"
