// C ABI entry points (include/modconv_b200.h): argument checking, table
// lookup, kernel selection.  No torch types cross this boundary.
#include <algorithm>
#include <cstdlib>

#include <cuda.h>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "conv_small.cuh"
#include "fourstep.cuh"
#include "runtime.h"

namespace mc {

cudaError_t launch_conv_small_k4(const ConvSmallParams &, int, cudaStream_t);
cudaError_t launch_conv_small_k5(const ConvSmallParams &, int, cudaStream_t);
cudaError_t launch_conv_small_k6(const ConvSmallParams &, int, cudaStream_t);
cudaError_t launch_conv_small_k7(const ConvSmallParams &, int, cudaStream_t);
cudaError_t launch_conv_small_k8(const ConvSmallParams &, int, cudaStream_t);
cudaError_t launch_conv_small_k9(const ConvSmallParams &, int, cudaStream_t);
cudaError_t launch_conv_small_k10(const ConvSmallParams &, int, cudaStream_t);
cudaError_t launch_conv_small_k11(const ConvSmallParams &, int, cudaStream_t);
cudaError_t launch_conv_small_k12(const ConvSmallParams &, int, cudaStream_t);
cudaError_t launch_conv_small_k13(const ConvSmallParams &, int, cudaStream_t);


// ---------------------------------------------------------------- tiny sizes
// L <= 8: one thread per product, direct convolution with 64-bit
// accumulation (exact; lin_conv_def semantics, convolve.py:71-87).
__global__ void conv_tiny_kernel(const u32 *a, long long lda, int z1, const u32 *b,
                                 long long ldb, int z2, u32 *c, long long ldc,
                                 long long batch, u32 p, int wrap_L) {
    long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= batch) return;
    const u32 *ar = a + r * lda;
    const u32 *br = b + r * ldb;
    u32 *cr = c + r * ldc;
    const int n = wrap_L ? wrap_L : z1 + z2 - 1;
    for (int k = 0; k < n; ++k) {
        unsigned long long acc = 0;
        for (int i = 0; i < z1; ++i) {
            for (int j = 0; j < z2; ++j) {
                int d = i + j;
                if (wrap_L) d &= wrap_L - 1;
                if (d == k) acc = (acc + (unsigned long long)ar[i] * br[j]) % p;
            }
        }
        cr[k] = (u32)acc;
    }
}

static int ceil_log2(long long n) {
    int k = 0;
    while ((1ll << k) < n) ++k;
    return k;
}

static ConvSmallParams make_params(const FieldTables *T, const u32 *a, long long lda, int z1,
                                   const u32 *b, long long ldb, int z2, u32 *c, long long ldc,
                                   int n, long long batch) {
    ConvSmallParams P;
    memset(&P, 0, sizeof(P));
    P.a = a;
    P.b = b;
    P.c = c;
    P.lda = lda;
    P.ldb = ldb;
    P.ldc = ldc;
    P.z1 = z1;
    P.z2 = z2;
    P.n = n;
    P.batch = batch;
    P.p = T->p;
    P.pinv = T->pinv;
    P.linv_mont = T->linv_mont;
    P.tf = T->tf;
    P.ti = T->ti;
    memcpy(P.c16f, T->h16f, sizeof(P.c16f));
    memcpy(P.c16fd, T->h16fd, sizeof(P.c16fd));
    memcpy(P.c16id, T->h16id, sizeof(P.c16id));
    memcpy(P.c16i, T->h16i, sizeof(P.c16i));
    memcpy(P.mlev, T->mlev, sizeof(P.mlev));
    memcpy(P.hinv, T->hinv, sizeof(P.hinv));
    return P;
}

// TMA row prefetch of the fused kernel: one product per CTA, 16-byte aligned
// rows, staging that fits in shared memory.
static void setup_tma(ConvSmallParams &P, int K, bool allow) {
    const bool one_per_cta = (1 << K) / 16 >= 128;
    const bool aligned = ((uintptr_t)P.a % 16 == 0) && ((uintptr_t)P.b % 16 == 0) &&
                         (P.lda % 4 == 0) && (P.ldb % 4 == 0);
    const int za16 = P.z1 & ~3, zb16 = P.z2 & ~3;
    const long long smem = 2ll * (1 << K) * 8 + 2ll * (1 << K) * 4 + 16 +
                           4ll * (za16 + zb16);  // upper bound (tables in smem)
    if (allow && one_per_cta && aligned && smem <= 227 * 1024 && P.batch > 0) {
        P.tma = 1;
        P.za16 = za16;
        P.zb16 = zb16;
    }
}

static cudaError_t launch_small(int K, const ConvSmallParams &P, int nt, cudaStream_t st) {
    switch (K) {
        case 4: return launch_conv_small_k4(P, nt, st);
        case 5: return launch_conv_small_k5(P, nt, st);
        case 6: return launch_conv_small_k6(P, nt, st);
        case 7: return launch_conv_small_k7(P, nt, st);
        case 8: return launch_conv_small_k8(P, nt, st);
        case 9: return launch_conv_small_k9(P, nt, st);
        case 10: return launch_conv_small_k10(P, nt, st);
        case 11: return launch_conv_small_k11(P, nt, st);
        case 12: return launch_conv_small_k12(P, nt, st);
        case 13: return launch_conv_small_k13(P, nt, st);
        default: return cudaErrorInvalidValue;
    }
}

// Inputs that a copy stream is still delivering when the kernel starts: the
// rows of chunk i (rows products each) are resident once flags[i] == epoch.
struct StreamIn {
    const uint32_t *flags;
    uint32_t epoch;
    int rows;
};

// Split truncated product (tft engine just past a power of two): n = L/2 + m
// with m <= L/8.  The relaxed truncated transform of the fused kernel keeps
// whole 16ths of the transform and idles the warps of the skipped blocks, so
// it gains little there (profiles/r01/sweep_fig3_*.csv).  Instead:
//   head: c0 = c mod (x^(L/2) - 1), the complete half of the truncated
//         transform, as an L/2-point cyclic convolution of the operands
//         folded on load (a_x + a_{x+L/2});
//   tail: low = the first m coefficients of a*b (operands truncated to m),
//         then c[x] = low[x], c[L/2 + x] = c0[x] - low[x] for x < m.
// Work ~ L/2 + 2m points instead of L; exact, so bit-identical to the
// reference's tft x2 + pointwise + itft (convolve.py:230-253).
// Twisted quarter tail (m in (L/8, L/4]): the L/4-point product mod
// (x^(L/4) - i) instead of a 2m-point low product.  Measured over whole
// octaves (profiles/r02/octave_*.csv): +6% at K = 13 and +31% at K = 14 (whose
// complete transform is four-step) over the complete transform, but -8..-10%
// at K = 12 (the extra folds, twists and global twiddle loads outweigh a
// quarter of a fast K = 12 product) and even with the relaxed four-step
// truncation at K = 15; so K = 13, 14 only.
static bool split_twist(int K, int m) {
    static const bool off = [] { const char *e = getenv("MC_NO_SPLIT_TWIST"); return e && *e; }();
    return !off && (K == 13 || K == 14) && m > (1 << K) / 8 && m <= (1 << K) / 4;
}

static bool split_tft_on(int K, int n, long long batch) {
    static const bool off = [] { const char *e = getenv("MC_NO_SPLIT_TFT"); return e && *e; }();
    if (off || K < 5 || K - 1 > kFourStepMaxK) return false;
    const int half = 1 << (K - 1), m = n - half;
    if (m < 1) return false;
    if (!split_twist(K, m)) {
        // low-product tail, a fused launch: 2m - 1 <= 2^13; up to K = 10 the
        // split pays only for m <= L/16 (octave sweeps, profiles/r02/octave_*.csv)
        if (m > (1 << K) / (K <= 10 ? 16 : 8) || 2 * m - 1 > (1 << kSmallMaxK)) return false;
    }
    // two launches: only where the kernels, not the launch latency, dominate
    return K >= 10 || batch * (1ll << K) >= (1ll << 20);
}

static mc_status split_tft(const u32 *a, long long lda, int z1, const u32 *b, long long ldb,
                           int z2, u32 *c, long long ldc, long long batch, u32 p, int K, int n,
                           cudaStream_t st, bool allow_tma) {
    if (z1 > z2) {  // the kernel folds L^-1 into operand a: make it the shorter one
        std::swap(a, b);
        std::swap(lda, ldb);
        std::swap(z1, z2);
    }
    const int half = 1 << (K - 1), m = n - half;
    const FieldTables *T1, *T2;
    mc_status s = get_tables(p, K - 1, &T1);
    if (s != MC_OK) return s;
    cudaError_t e;
    if (K - 1 <= kSmallMaxK) {
        ConvSmallParams H = make_params(T1, a, lda, z1, b, ldb, z2, c, ldc, half, batch);
        H.fold = 1;
        H.ar = lazy_ok(p) ? 1 : 2;
        setup_tma(H, K - 1, allow_tma);
        e = launch_small(K - 1, H, 16, st);
        note_launches(1);
        if (e != cudaSuccess) return cuda_fail(e, "split tft head launch");
    } else {  // four-step head: circular L/2-point product of the folded operands
        s = fourstep_conv(0, a, lda, z1, b, ldb, z2, c, ldc, batch, p, st, K - 1, false, true);
        if (s != MC_OK) return s;
    }
    if (split_twist(K, m)) {
        // c mod (x^(L/4) - i), i = w_L^(L/4): an L/4-point cyclic product of
        // the operands folded by quarters and twisted by w_L^x; then
        // c = c0 + (x^(L/2) - 1) h, h = (c0 mod (x^(L/4) - i) - c1) / 2
        const int K2 = K - 2, Lq = 1 << K2;
        const FieldTables *TK;
        if ((s = get_tables(p, K, &TK)) != MC_OK) return s;
        if ((s = get_tables(p, K2, &T2)) != MC_OK) return s;
        ConvSmallParams Q = make_params(T2, a, lda, Lq, b, ldb, Lq, c, ldc, Lq, batch);
        Q.tz1 = z1;
        Q.tz2 = z2;
        Q.twq_f = TK->tf + (1 << (K - 1));
        Q.twq_i = TK->ti + (1 << (K - 1));
        Q.qi = shoup((u32)powmod(TK->root, (u64)Lq, p), p);
        Q.qhalf = shoup((u32)((p + 1) / 2), p);
        Q.wrap_m = m;
        Q.wrap_off = half;
        Q.ar = lazy_ok(p) ? 1 : 2;
        e = launch_small(K2, Q, 16, st);
        note_launches(1);
        if (e != cudaSuccess) return cuda_fail(e, "split tft twisted tail launch");
        return MC_OK;
    }
    const int y1 = std::min(z1, m), y2 = std::min(z2, m);
    const int K2 = std::max(4, ceil_log2(y1 + y2 - 1));
    if ((s = get_tables(p, K2, &T2)) != MC_OK) return s;
    ConvSmallParams W = make_params(T2, a, lda, y1, b, ldb, y2, c, ldc, m, batch);
    W.wrap_m = m;
    W.wrap_off = half;
    W.ar = lazy_ok(p) ? 1 : 2;
    setup_tma(W, K2, allow_tma);
    e = launch_small(K2, W, 16, st);
    note_launches(1);
    if (e != cudaSuccess) return cuda_fail(e, "split tft tail launch");
    return MC_OK;
}

// Relaxed truncation limit of the fused kernel.  It truncates at whole 16ths
// (G-blocks); its lower passes skip only warps whose G-blocks are all
// inactive (two blocks per warp at K = 12), and the truncated inverse's
// van der Hoeven steps cost three products per cross butterfly.  Measured
// over whole octaves (profiles/r02/octave_*.csv, p2 and p3): with 11..15 of
// 16 blocks the truncated kernel ran 5-13% slower than the complete
// transform at K <= 12, and at K = 13 with 13..15 blocks, so the tft engine
// rounds NT up to 16 there (the relaxation's limit case: the product is the
// same); NT <= 10 takes the split product.  MC_TFT_KEEP_NT=1 keeps the
// truncated schedule (A/B, tests).
static int tft_full_from(int K) {
    const char *e = getenv("MC_TFT_KEEP_NT");
    if (e && *e && *e != '0') return 17;
    return K == 13 ? 13 : 11;
}

// engine 0 = fft_pad, 1 = tft; wrap != 0 => circular convolution of length L
static mc_status conv_dispatch(int engine, const u32 *a, long long lda, int z1, const u32 *b,
                               long long ldb, int z2, u32 *c, long long ldc, long long batch,
                               u32 p, cudaStream_t st, int circ_log2L = -1,
                               bool reduce = false, bool allow_tma = true,
                               bool host_out = false, const StreamIn *sin = nullptr) {
    if (z1 < 1 || z2 < 1) return fail(MC_EINVAL, "inputs must be nonempty");
    if (batch < 0) return fail(MC_EINVAL, "negative batch");
    if (lda < z1 || ldb < z2) return fail(MC_EINVAL, "leading dimension smaller than row length");
    const bool circ = circ_log2L >= 0;
    const int n = circ ? (1 << circ_log2L) : z1 + z2 - 1;
    if (ldc < n) return fail(MC_EINVAL, "output leading dimension smaller than product length");
    const int K = circ ? circ_log2L : ceil_log2(n);
    const FieldTables *T;
    mc_status s = get_tables(p, K, &T);
    if (s != MC_OK) return s;
    if (batch == 0) return MC_OK;
    if (!a || !b || !c) return fail(MC_EINVAL, "null pointer");
    if (K <= 3) {
        const int thr = 128;
        conv_tiny_kernel<<<(unsigned)((batch + thr - 1) / thr), thr, 0, st>>>(
            a, lda, z1, b, ldb, z2, c, ldc, batch, p, circ ? (1 << K) : 0);
        note_launches(1);
        MC_CUDA_CHECK(cudaGetLastError());
        return MC_OK;
    }
    if (engine == 1 && !circ && !reduce && !host_out && !sin && split_tft_on(K, n, batch))
        return split_tft(a, lda, z1, b, ldb, z2, c, ldc, batch, p, K, n, st, allow_tma);
    if (K <= kSmallMaxK) {
        if (z1 > z2) {  // the kernel folds L^-1 into operand a: make it the shorter one
            std::swap(a, b);
            std::swap(lda, ldb);
            std::swap(z1, z2);
        }
        ConvSmallParams P = make_params(T, a, lda, z1, b, ldb, z2, c, ldc, n, batch);
        P.reduce = reduce ? 1 : 0;
        P.red_wp = (u32)((1ull << 32) / p);
        setup_tma(P, K, allow_tma);
        if (sin) {  // streamed inputs: only the bulk-copy prefetch can wait for them
            if (!P.tma) return fail(MC_EINVAL, "streamed inputs need the bulk-copy path");
            P.ready = sin->flags;
            P.epoch = sin->epoch;
            P.ready_rows = sin->rows;
        }
        int nt = 16;
        if (engine == 1 && !circ) {
            const int G = 1 << (K - 4);
            nt = (n + G - 1) / G;
            if (nt >= tft_full_from(K)) nt = 16;
        }
        if (batch > 0x7fffffffll * SmallCfg<4>::PPC)
            return fail(MC_EINVAL, "batch too large for one launch");
        P.ar = lazy_ok(p) ? 1 : 2;
        {  // bulk-copy epilogue: host output (zero copy), or forced for A/B runs
            static const bool force = [] { const char *e = getenv("MC_BULK_OUT"); return e && *e; }();
            P.bulk_out = ((host_out || force) && (1 << K) / 16 >= 128) ? 1 : 0;
        }
        cudaError_t e = launch_small(K, P, nt, st);
        note_launches(1);
        if (e != cudaSuccess) return cuda_fail(e, "conv_small launch");
        return MC_OK;
    }
    return fourstep_conv(engine, a, lda, z1, b, ldb, z2, c, ldc, batch, p, st, circ_log2L,
                         reduce);
}

// Batched circular convolution of length 2^log2L (split engine building block).
mc_status circ_conv_dispatch(const u32 *u, const u32 *v, u32 *w, int log2L, long long batch,
                             u32 p, cudaStream_t st) {
    const long long L = 1ll << log2L;
    return conv_dispatch(0, u, L, (int)L, v, L, (int)L, w, L, batch, p, st, log2L);
}

// Product mod p of two arbitrary-word vectors (three-primes channels).
mc_status conv_dispatch_reduced(const u32 *a, int z1, const u32 *b, int z2, u32 *r, u32 p,
                                cudaStream_t st) {
    return conv_dispatch(0, a, z1, z1, b, z2, z2, r, (long long)z1 + z2 - 1, 1, p, st, -1, true);
}

}  // namespace mc

using namespace mc;

extern "C" {

mc_status mc_conv_fft_pad(const uint32_t *a, int64_t lda, int32_t z1, const uint32_t *b,
                          int64_t ldb, int32_t z2, uint32_t *c, int64_t ldc, int64_t batch,
                          uint32_t p, void *stream) {
    return conv_dispatch(0, a, lda, z1, b, ldb, z2, c, ldc, batch, p, (cudaStream_t)stream);
}

mc_status mc_conv_tft(const uint32_t *a, int64_t lda, int32_t z1, const uint32_t *b,
                      int64_t ldb, int32_t z2, uint32_t *c, int64_t ldc, int64_t batch,
                      uint32_t p, void *stream) {
    return conv_dispatch(1, a, lda, z1, b, ldb, z2, c, ldc, batch, p, (cudaStream_t)stream);
}

mc_status mc_circ_conv(const uint32_t *u, const uint32_t *v, uint32_t *w, int32_t log2L,
                       int64_t batch, uint32_t p, void *stream) {
    if (log2L < 0 || log2L > 30) return fail(MC_EINVAL, "bad transform size");
    const int64_t L = 1ll << log2L;
    return conv_dispatch(0, u, L, (int)L, v, L, (int)L, w, L, batch, p, (cudaStream_t)stream,
                         log2L);
}

// ---------------------------------------------------------------- host-buffer call
mc_status mc_conv_host(int engine, const uint32_t *a, int64_t lda, int32_t z1,
                       const uint32_t *b, int64_t ldb, int32_t z2, uint32_t *c, int64_t ldc,
                       int64_t batch, uint32_t p) {
    // the asynchronous host path on the legacy default stream, then a
    // synchronize: zero copy for page-locked buffers, the chunked copy
    // pipeline for pageable ones (a ctypes caller's arrays)
    mc_status s = mc_conv_host_async(engine, a, lda, z1, b, ldb, z2, c, ldc, batch, p, 0, nullptr);
    if (s != MC_OK) return s;
    MC_CUDA_CHECK(cudaStreamSynchronize(nullptr));
    return MC_OK;
}

// ---------------------------------------------------------------- pipelined host call
struct PipeState {
    int dev = -1;
    cudaStream_t s_in = nullptr, s_cmp = nullptr, s_out = nullptr;
    static constexpr int NBUF = 3;
    cudaEvent_t ev_in[NBUF] = {}, ev_cmp[NBUF] = {}, ev_out[NBUF] = {}, ev_start = nullptr;
    void *buf = nullptr;
    size_t bytes = 0;
    // streamed-input mode: whole-batch operand buffer + per-chunk ready flags
    static constexpr int MAX_CHUNKS = 1 << 16;
    void *in_buf = nullptr;
    size_t in_bytes = 0;
    uint32_t *flags = nullptr;
    uint32_t epoch = 0;
    cudaEvent_t ev_k = nullptr, ev_cp = nullptr;
    // copy-engine mode: whole-batch device buffers + per-chunk events
    void *ce_buf = nullptr;
    size_t ce_bytes = 0;
    std::vector<cudaEvent_t> ce_in, ce_cmp;
    // recorded on the caller's stream at the end of every call: the next call's
    // internal streams wait on it, so reused buffers are never overwritten
    // while an earlier call (possibly on another caller stream) still uses them
    cudaEvent_t ev_done = nullptr;
};

// cuStreamWriteValue32 through the runtime's driver entry point (no libcuda link)
typedef CUresult (*PFN_write_value32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PFN_write_value32 write_value32() {
    static PFN_write_value32 fn = [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_write_value32>(f);
    }();
    return fn;
}

static std::mutex g_pipe_mu;

// Host-memory modes for the fused single-pass kernel (every operand word
// read once, every product word written once), from measurements on B200
// (DESIGN.md section 7):
//   2  zero copy (the kernel reads and writes page-locked host memory):
//      calls under 8 MiB (latency bound), and one-product-per-CTA sizes
//      (L >= 2048, bulk-store epilogue) with under 512 MiB of operands;
//   3  copy engines both ways over whole-batch device buffers (ce_full_call):
//      one-product-per-CTA sizes with >= 512 MiB of operands, contiguous
//      rows (config 3: 1.39M products/s; streamed inputs 1.34M);
//   1  streamed inputs + zero-copy output (stream_in_call): the same sizes
//      when mode 3 does not apply (strided rows, > 8 GiB of buffers);
//   0  chunked copy pipeline (other sizes).
// Zero copy stays the default below 512 MiB: at config 2 sizes the
// copy-engine pipeline measured 2.06-2.36M products/s at 6-24 chunks against
// 2.61M (every chunk's operands must land before its products can leave).
// MC_HOST_MODE=zc|ce|in|pipe forces a mode where the size allows it (tests, A/B).
static int zero_copy_shape(int64_t n, int64_t z12, int64_t batch) {
    int K = 0;
    while ((1ll << K) < n) ++K;
    if (K < 4 || K > kSmallMaxK) return 0;
    const char *m = getenv("MC_HOST_MODE");  // read per call
    if (m && *m) {
        if (!strcmp(m, "zc")) return 2;
        if (!strcmp(m, "ce")) return 3;
        if (!strcmp(m, "in")) return K >= 11 ? 1 : 0;
        return 0;
    }
    if (8 * n * batch < (8ll << 20)) return 2;
    if (K < 11) return 0;
    const char *e = getenv("MC_STREAM_IN_MIN_MB");  // read per call (tests force the mode)
    const long long min_mb = e && *e ? atoll(e) : 512;
    return 4 * z12 * batch < (min_mb << 20) ? 2 : 3;
}

// Host memory the device can address directly (page-locked, mapped into the
// unified address space at the same pointer).  MC_NO_ZERO_COPY disables.
static bool zero_copy_ok(const void *ptr) {
    static const bool off = [] { const char *e = getenv("MC_NO_ZERO_COPY"); return e && *e; }();
    if (off) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost && at.devicePointer == ptr;
}

// Streamed inputs, page-locked output: the operand rows go H2D in chunks on a
// copy stream, each chunk followed by a stream-memory write of its ready
// flag; ONE persistent fused kernel, launched at once, waits per product for
// its chunk's flag before the bulk-copy prefetch and writes its products
// straight into host memory with bulk stores.  Copy-engine reads and
// kernel writes share PCIe (~44 GB/s each way measured), with no per-chunk
// kernel drain.  Returns 1 (not applicable) to fall back to the pipeline.
static int stream_in_call(PipeState &S, int engine, const uint32_t *a, int64_t lda, int32_t z1,
                          const uint32_t *b, int64_t ldb, int32_t z2, uint32_t *c, int64_t ldc,
                          int64_t batch, uint32_t p, cudaStream_t user, mc_status *out) {
    static const bool off = [] { const char *e = getenv("MC_NO_STREAM_IN"); return e && *e; }();
    auto wv = write_value32();
    if (off || !wv) return 1;
    const int64_t lda_d = (z1 + 3) & ~3ll, ldb_d = (z2 + 3) & ~3ll;  // 16-byte rows
    const size_t need = 4ull * batch * (lda_d + ldb_d);
    if (need > (4ull << 30)) return 1;
    // 32 uniform chunks: used only for >= 512 MiB of operands, so every copy
    // is large (a copy-engine call costs ~10-20 us; geometric chunk sizes were
    // measured worse: the kernel stalls on the last, largest chunk)
    const char *ce = getenv("MC_STREAM_IN_CHUNKS");  // A/B override of the chunk count
    const int64_t want = ce && *ce ? std::max(1, atoi(ce)) : 32;
    const int64_t rows = std::max<int64_t>(16, (batch + want - 1) / want);
    const int64_t nch = (batch + rows - 1) / rows;
    if (nch > PipeState::MAX_CHUNKS || rows > 0x7fffffff) return 1;
    auto fail_out = [&](mc_status st) { *out = st; return 0; };
    if (!S.flags) {
        if (cudaMalloc(&S.flags, 4ull * PipeState::MAX_CHUNKS) != cudaSuccess ||
            cudaMemset(S.flags, 0, 4ull * PipeState::MAX_CHUNKS) != cudaSuccess ||
            cudaEventCreateWithFlags(&S.ev_k, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&S.ev_cp, cudaEventDisableTiming) != cudaSuccess)
            return fail_out(cuda_fail(cudaGetLastError(), "stream-in state"));
    }
    if (S.in_bytes < need) {
        cudaDeviceSynchronize();  // the previous call's kernel may still read in_buf
        if (S.in_buf) cudaFree(S.in_buf);
        S.in_buf = nullptr;
        S.in_bytes = 0;
        if (cudaMalloc(&S.in_buf, need) != cudaSuccess)
            return fail_out(cuda_fail(cudaGetLastError(), "stream-in buffer"));
        S.in_bytes = need;
    }
    if (++S.epoch == 0) S.epoch = 1;
    uint32_t *da = (uint32_t *)S.in_buf, *db = da + batch * lda_d;
    // both streams start after prior work on the user's stream (this also
    // orders the copies after the previous call's kernel, which read in_buf)
    if (cudaEventRecord(S.ev_start, user) != cudaSuccess ||
        cudaStreamWaitEvent(S.s_in, S.ev_start, 0) != cudaSuccess ||
        cudaStreamWaitEvent(S.s_cmp, S.ev_start, 0) != cudaSuccess ||
        cudaStreamWaitEvent(S.s_in, S.ev_done, 0) != cudaSuccess)
        return fail_out(cuda_fail(cudaGetLastError(), "stream-in ordering"));
    for (int64_t i = 0; i < nch; ++i) {
        const int64_t r0 = i * rows, nr = std::min(rows, batch - r0);
        // one linear DMA per operand chunk when the rows are contiguous on both
        // sides (pitched copies of short rows run far below PCIe speed)
        auto copy = [&](uint32_t *dst, int64_t ldd, const uint32_t *src, int64_t lds, int32_t z) {
            if (lds == z && ldd == z)
                return cudaMemcpyAsync(dst + r0 * ldd, src + r0 * lds, 4ull * z * nr,
                                       cudaMemcpyHostToDevice, S.s_in);
            return cudaMemcpy2DAsync(dst + r0 * ldd, 4 * ldd, src + r0 * lds, 4 * lds, 4 * z, nr,
                                     cudaMemcpyHostToDevice, S.s_in);
        };
        if (copy(da, lda_d, a, lda, z1) != cudaSuccess || copy(db, ldb_d, b, ldb, z2) != cudaSuccess)
            return fail_out(cuda_fail(cudaGetLastError(), "stream-in copy"));
        if (wv((CUstream)S.s_in, (CUdeviceptr)(S.flags + i), S.epoch, CU_STREAM_WRITE_VALUE_DEFAULT) !=
            CUDA_SUCCESS) {
            // the kernel would wait forever: drain the copies, report
            cudaStreamSynchronize(S.s_in);
            return fail_out(fail(MC_ECUDA, "cuStreamWriteValue32 failed"));
        }
    }
    const StreamIn sin{S.flags, S.epoch, (int)rows};
    mc_status st = conv_dispatch(engine, da, lda_d, z1, db, ldb_d, z2, c, ldc, batch, p, S.s_cmp,
                                 -1, false, true, true, &sin);
    if (st != MC_OK) {
        cudaStreamSynchronize(S.s_in);
        return fail_out(st);
    }
    if (cudaEventRecord(S.ev_k, S.s_cmp) != cudaSuccess ||
        cudaEventRecord(S.ev_cp, S.s_in) != cudaSuccess ||
        cudaStreamWaitEvent(user, S.ev_k, 0) != cudaSuccess ||
        cudaStreamWaitEvent(user, S.ev_cp, 0) != cudaSuccess ||
        cudaEventRecord(S.ev_done, user) != cudaSuccess)
        return fail_out(cuda_fail(cudaGetLastError(), "stream-in join"));
    *out = MC_OK;
    return 0;
}

// Copy engines both ways, whole-batch device buffers: operand chunks go H2D
// back to back on one stream, each chunk's fused kernel runs on a second as
// soon as its rows land, its products go D2H on a third.  No buffer is
// reused inside a call, so the H2D stream never waits and both copy
// directions run concurrently (measured at cfg2 sizes: 59 MB each way in
// 1.20-1.24 ms with up to 8 chunks, ~96 GB/s together, against ~72 GB/s for
// kernel reads and writes of host memory; scripts/ce_gate_probe.py).
// Returns 1 (not applicable) to fall back.
static int ce_full_call(PipeState &S, int engine, const uint32_t *a, int64_t lda, int32_t z1,
                        const uint32_t *b, int64_t ldb, int32_t z2, uint32_t *c, int64_t ldc,
                        int64_t batch, uint32_t p, cudaStream_t user, mc_status *out) {
    const int64_t n = (int64_t)z1 + z2 - 1;
    if (lda != z1 || ldb != z2 || ldc != n) return 1;  // linear DMA per chunk only
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t sa = up(4ull * batch * z1), sb = up(4ull * batch * z2), sc = up(4ull * batch * n);
    if (sa + sb + sc > (8ull << 30)) return 1;
    auto fail_out = [&](mc_status st) { *out = st; return 0; };
    // chunk plan: equal chunks.  The products of a chunk leave only after its
    // operands have arrived, so the D2H stream trails the H2D stream by one
    // chunk: time ~ T (1 + 1/N) + N o, o the per-chunk cost of the copies and
    // the kernel launch.  32 chunks measured best on config 3 (4.3 GB moved:
    // 1.39M products/s vs 1.34M streamed inputs, 1.30M at 128 chunks);
    // MC_CE_CHUNKS overrides.
    const char *ce_env = getenv("MC_CE_CHUNKS");
    int64_t nchunk = ce_env && *ce_env ? std::max(1, atoi(ce_env)) : 32;
    nchunk = std::min<int64_t>(nchunk, batch);
    std::vector<int64_t> rows;
    const int64_t per = (batch + nchunk - 1) / nchunk;
    for (int64_t r = 0; r < batch; r += per) rows.push_back(std::min(per, batch - r));
    const size_t nch = rows.size();
    while (S.ce_in.size() < nch) {
        cudaEvent_t e1, e2;
        if (cudaEventCreateWithFlags(&e1, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&e2, cudaEventDisableTiming) != cudaSuccess)
            return fail_out(cuda_fail(cudaGetLastError(), "copy-engine events"));
        S.ce_in.push_back(e1);
        S.ce_cmp.push_back(e2);
    }
    if (!S.ev_k && cudaEventCreateWithFlags(&S.ev_k, cudaEventDisableTiming) != cudaSuccess)
        return fail_out(cuda_fail(cudaGetLastError(), "copy-engine events"));
    if (S.ce_bytes < sa + sb + sc) {
        cudaDeviceSynchronize();  // the previous call may still use ce_buf
        if (S.ce_buf) cudaFree(S.ce_buf);
        S.ce_buf = nullptr;
        S.ce_bytes = 0;
        if (cudaMalloc(&S.ce_buf, sa + sb + sc) != cudaSuccess)
            return fail_out(cuda_fail(cudaGetLastError(), "copy-engine buffer"));
        S.ce_bytes = sa + sb + sc;
    }
    uint32_t *da = (uint32_t *)S.ce_buf;
    uint32_t *db = (uint32_t *)((char *)S.ce_buf + sa);
    uint32_t *dc = (uint32_t *)((char *)S.ce_buf + sa + sb);
    // all three streams start after prior work on the caller's stream and
    // after the previous call (which used the same buffers) has finished
    if (cudaEventRecord(S.ev_start, user) != cudaSuccess ||
        cudaStreamWaitEvent(S.s_in, S.ev_start, 0) != cudaSuccess ||
        cudaStreamWaitEvent(S.s_in, S.ev_done, 0) != cudaSuccess ||
        cudaStreamWaitEvent(S.s_cmp, S.ev_start, 0) != cudaSuccess ||
        cudaStreamWaitEvent(S.s_out, S.ev_start, 0) != cudaSuccess)
        return fail_out(cuda_fail(cudaGetLastError(), "copy-engine ordering"));
    int64_t r0 = 0;
    for (size_t i = 0; i < nch; ++i) {
        const int64_t nr = rows[i];
        if (cudaMemcpyAsync(da + r0 * z1, a + r0 * z1, 4ull * z1 * nr, cudaMemcpyHostToDevice,
                            S.s_in) != cudaSuccess ||
            cudaMemcpyAsync(db + r0 * z2, b + r0 * z2, 4ull * z2 * nr, cudaMemcpyHostToDevice,
                            S.s_in) != cudaSuccess ||
            cudaEventRecord(S.ce_in[i], S.s_in) != cudaSuccess ||
            cudaStreamWaitEvent(S.s_cmp, S.ce_in[i], 0) != cudaSuccess)
            return fail_out(cuda_fail(cudaGetLastError(), "copy-engine H2D"));
        mc_status st = conv_dispatch(engine, da + r0 * z1, z1, z1, db + r0 * z2, z2, z2,
                                     dc + r0 * n, n, nr, p, S.s_cmp);
        if (st != MC_OK) return fail_out(st);
        if (cudaEventRecord(S.ce_cmp[i], S.s_cmp) != cudaSuccess ||
            cudaStreamWaitEvent(S.s_out, S.ce_cmp[i], 0) != cudaSuccess ||
            cudaMemcpyAsync(c + r0 * n, dc + r0 * n, 4ull * n * nr, cudaMemcpyDeviceToHost,
                            S.s_out) != cudaSuccess)
            return fail_out(cuda_fail(cudaGetLastError(), "copy-engine D2H"));
        r0 += nr;
    }
    if (cudaEventRecord(S.ev_k, S.s_out) != cudaSuccess ||
        cudaStreamWaitEvent(user, S.ev_k, 0) != cudaSuccess ||
        cudaEventRecord(S.ev_done, user) != cudaSuccess)
        return fail_out(cuda_fail(cudaGetLastError(), "copy-engine join"));
    *out = MC_OK;
    return 0;
}

mc_status mc_conv_host_async(int engine, const uint32_t *a, int64_t lda, int32_t z1,
                             const uint32_t *b, int64_t ldb, int32_t z2, uint32_t *c,
                             int64_t ldc, int64_t batch, uint32_t p, int64_t chunk_rows,
                             void *stream) {
    // one pipeline state per (thread, device): streams, events and buffers
    // belong to the device they were created on
    static thread_local std::map<int, PipeState> states;
    if (engine != 0 && engine != 1) return fail(MC_EINVAL, "engine must be 0 (fft_pad) or 1 (tft)");
    if (z1 < 1 || z2 < 1) return fail(MC_EINVAL, "inputs must be nonempty");
    const int64_t n = (int64_t)z1 + z2 - 1;
    if (lda < z1 || ldb < z2 || ldc < n) return fail(MC_EINVAL, "bad leading dimension");
    if (batch <= 0) return batch == 0 ? MC_OK : fail(MC_EINVAL, "negative batch");
    if (!a || !b || !c) return fail(MC_EINVAL, "null pointer");
    int K = 0;
    while ((1ll << K) < n) ++K;
    {  // validate the field / size up front (synchronous errors, nothing launched)
        const FieldTables *T;
        mc_status st = get_tables(p, K, &T);
        if (st != MC_OK) return st;
    }
    cudaStream_t user = (cudaStream_t)stream;
    const int zc = zero_copy_shape(n, (int64_t)z1 + z2, batch);
    const bool c_mapped = zc && zero_copy_ok(c);
    if (zc == 2 && c_mapped && zero_copy_ok(a) && zero_copy_ok(b)) {
        // Zero copy: page-locked host rows are device-addressable (UVA), so the
        // fused kernel reads the operands (bulk-copy prefetch) and writes the
        // products (bulk stores from shared memory) over PCIe itself -- no
        // copy-engine calls (~10-20 us each) and no pipeline start-up.
        return conv_dispatch(engine, a, lda, z1, b, ldb, z2, c, ldc, batch, p, user, -1, false,
                             true, true);
    }
    // Large calls with a page-locked output: streamed inputs (stream_in_call).
    // Measured on cfg2 shapes: copy-engine H2D alongside kernel bulk writes to
    // host reaches ~44 GB/s each way; kernel reads from host alongside any
    // host writes only ~36 (scripts/zc_probe{2,3,4}.py).
    const int dev = current_device();
    PipeState &S = states[dev];
    if (S.dev != dev) {
        std::lock_guard<std::mutex> lock(g_pipe_mu);
        MC_CUDA_CHECK(cudaStreamCreateWithFlags(&S.s_in, cudaStreamNonBlocking));
        MC_CUDA_CHECK(cudaStreamCreateWithFlags(&S.s_cmp, cudaStreamNonBlocking));
        MC_CUDA_CHECK(cudaStreamCreateWithFlags(&S.s_out, cudaStreamNonBlocking));
        for (int k = 0; k < PipeState::NBUF; ++k) {
            MC_CUDA_CHECK(cudaEventCreateWithFlags(&S.ev_in[k], cudaEventDisableTiming));
            MC_CUDA_CHECK(cudaEventCreateWithFlags(&S.ev_cmp[k], cudaEventDisableTiming));
            MC_CUDA_CHECK(cudaEventCreateWithFlags(&S.ev_out[k], cudaEventDisableTiming));
        }
        MC_CUDA_CHECK(cudaEventCreateWithFlags(&S.ev_start, cudaEventDisableTiming));
        MC_CUDA_CHECK(cudaEventCreateWithFlags(&S.ev_done, cudaEventDisableTiming));
        S.dev = dev;
        S.buf = nullptr;
        S.bytes = 0;
        S.in_buf = nullptr;
        S.in_bytes = 0;
        S.flags = nullptr;
    }
    if (zc == 3 && c_mapped && zero_copy_ok(a) && zero_copy_ok(b)) {
        mc_status st = MC_OK;
        if (ce_full_call(S, engine, a, lda, z1, b, ldb, z2, c, ldc, batch, p, user, &st) == 0)
            return st;
    }
    if ((zc == 1 || (zc == 3 && K >= 11)) && c_mapped) {  // streamed inputs (or mode 3 n/a)
        mc_status st = MC_OK;
        if (stream_in_call(S, engine, a, lda, z1, b, ldb, z2, c, ldc, batch, p, user, &st) == 0)
            return st;
    }
    if (chunk_rows <= 0) {  // ~8 chunks, at least 64 rows, at most ~16 MiB of operands
        chunk_rows = std::max<int64_t>(64, (batch + 7) / 8);
        const int64_t cap = std::max<int64_t>(1, (16ll << 20) / (4 * (z1 + z2 + n)));
        chunk_rows = std::min(chunk_rows, std::max<int64_t>(cap, 1));
    }
    chunk_rows = std::min(chunk_rows, batch);
    // every sub-buffer 256-byte aligned (TMA tensor maps need 16-byte bases)
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t sa = up(4ull * chunk_rows * z1), sb = up(4ull * chunk_rows * z2);
    const size_t per_buf = sa + sb + up(4ull * chunk_rows * n);
    if (S.bytes < per_buf * PipeState::NBUF) {
        MC_CUDA_CHECK(cudaStreamSynchronize(S.s_out));
        if (S.buf) cudaFree(S.buf);
        S.buf = nullptr;
        MC_CUDA_CHECK(cudaMalloc(&S.buf, per_buf * PipeState::NBUF));
        S.bytes = per_buf * PipeState::NBUF;
    }
    MC_CUDA_CHECK(cudaEventRecord(S.ev_start, user));
    MC_CUDA_CHECK(cudaStreamWaitEvent(S.s_in, S.ev_start, 0));
    MC_CUDA_CHECK(cudaStreamWaitEvent(S.s_in, S.ev_done, 0));
    const int64_t nch = (batch + chunk_rows - 1) / chunk_rows;
    for (int64_t i = 0; i < nch; ++i) {
        const int k = (int)(i % PipeState::NBUF);
        const int64_t r0 = i * chunk_rows, rows = std::min(chunk_rows, batch - r0);
        uint32_t *da = (uint32_t *)((char *)S.buf + per_buf * k);
        uint32_t *db = (uint32_t *)((char *)da + sa);
        uint32_t *dc = (uint32_t *)((char *)db + sb);
        if (i >= PipeState::NBUF) MC_CUDA_CHECK(cudaStreamWaitEvent(S.s_in, S.ev_out[k], 0));
        if (lda == z1)  // contiguous rows: one linear DMA per operand chunk
            MC_CUDA_CHECK(cudaMemcpyAsync(da, a + r0 * lda, 4ull * z1 * rows,
                                          cudaMemcpyHostToDevice, S.s_in));
        else
            MC_CUDA_CHECK(cudaMemcpy2DAsync(da, 4 * z1, a + r0 * lda, 4 * lda, 4 * z1, rows,
                                            cudaMemcpyHostToDevice, S.s_in));
        if (ldb == z2)
            MC_CUDA_CHECK(cudaMemcpyAsync(db, b + r0 * ldb, 4ull * z2 * rows,
                                          cudaMemcpyHostToDevice, S.s_in));
        else
            MC_CUDA_CHECK(cudaMemcpy2DAsync(db, 4 * z2, b + r0 * ldb, 4 * ldb, 4 * z2, rows,
                                            cudaMemcpyHostToDevice, S.s_in));
        MC_CUDA_CHECK(cudaEventRecord(S.ev_in[k], S.s_in));
        MC_CUDA_CHECK(cudaStreamWaitEvent(S.s_cmp, S.ev_in[k], 0));
        mc_status st = conv_dispatch(engine, da, z1, z1, db, z2, z2, dc, n, rows, p, S.s_cmp);
        if (st != MC_OK) return st;
        MC_CUDA_CHECK(cudaEventRecord(S.ev_cmp[k], S.s_cmp));
        MC_CUDA_CHECK(cudaStreamWaitEvent(S.s_out, S.ev_cmp[k], 0));
        if (ldc == n)
            MC_CUDA_CHECK(cudaMemcpyAsync(c + r0 * ldc, dc, 4ull * n * rows,
                                          cudaMemcpyDeviceToHost, S.s_out));
        else
            MC_CUDA_CHECK(cudaMemcpy2DAsync(c + r0 * ldc, 4 * ldc, dc, 4 * n, 4 * n, rows,
                                            cudaMemcpyDeviceToHost, S.s_out));
        MC_CUDA_CHECK(cudaEventRecord(S.ev_out[k], S.s_out));
    }
    // the user's stream continues after the last write of c
    const int last = (int)((nch - 1) % PipeState::NBUF);
    MC_CUDA_CHECK(cudaStreamWaitEvent(user, S.ev_out[last], 0));
    MC_CUDA_CHECK(cudaEventRecord(S.ev_done, user));
    return MC_OK;
}

// ---------------------------------------------------------------- generator
__device__ __forceinline__ unsigned long long sm64(unsigned long long x) {
    unsigned long long z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void gen_kernel(unsigned long long seed, unsigned long long sid,
                           unsigned long long row0, long long rows, long long len,
                           unsigned long long hi, uint32_t *out, long long ld) {
    const long long r = blockIdx.y + (long long)blockIdx.z * gridDim.y;
    if (r >= rows) return;
    const unsigned long long key = sm64(sm64(sm64(seed) ^ sid) ^ (row0 + r));
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < len;
         i += (long long)gridDim.x * blockDim.x) {
        unsigned long long v = sm64(key + (unsigned long long)i);
        out[r * ld + i] = (uint32_t)(((v >> 32) * hi) >> 32);
    }
}

mc_status mc_gen_u32(uint64_t seed, uint64_t sid, uint64_t row0, int64_t rows, int64_t len,
                     uint64_t hi, uint32_t *out, int64_t ld, void *stream) {
    if (rows < 0 || len < 0 || ld < len || hi == 0 || hi > (1ull << 32))
        return fail(MC_EINVAL, "bad generator arguments");
    if (rows == 0 || len == 0) return MC_OK;
    const int thr = 256;
    long long bx = std::min<long long>((len + thr - 1) / thr, 64);
    long long gy = std::min<long long>(rows, 65535);
    long long gz = (rows + gy - 1) / gy;
    gen_kernel<<<dim3((unsigned)bx, (unsigned)gy, (unsigned)gz), thr, 0, (cudaStream_t)stream>>>(
        seed, sid, row0, rows, len, hi, out, ld);
    note_launches(1);
    MC_CUDA_CHECK(cudaGetLastError());
    return MC_OK;
}

}  // extern "C"
