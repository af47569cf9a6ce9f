/*
 * modconv_b200.h -- C ABI of the B200-native modular polynomial
 * multiplication path (libmodconv_b200.so).
 *
 * The reference (arXiv 1609.01010's `modconv`, pure Python) has no FFI; its
 * "operator API" for this path is the engine functions selected through
 * ConvRequest.engine.  Each entry point below replaces one of them and
 * cites it (paths relative to /root/reference/pkg/src/modconv/).
 *
 * Conventions
 *  - Residues are uint32 in [0, p) for a prime p < 2^31 with
 *    log2(L) <= two_adicity(p).  Larger moduli return MC_EUNSUPPORTED
 *    (the reference admits p < 2^62; a GPU word kernel does not).
 *  - Unless a function says "host", every pointer is DEVICE memory owned by
 *    the caller; calls are asynchronous on `stream` (a cudaStream_t passed
 *    as void*; NULL = legacy default stream).  Argument errors are reported
 *    synchronously and nothing is launched.
 *  - Batched calls take row-major operands with leading dimensions (in
 *    elements); row r of the output receives the product of row r of a and
 *    row r of b.  Inputs are never modified (reference engines copy:
 *    transform.py:189,441,510; convolve.py:167-168).
 *  - The root of unity is the reference's: w_L = g^((p-1)/L) with g the
 *    smallest primitive root (field.py:102-108, 209-224).
 *  - Thread safety: every entry point is reentrant; twiddle tables are built
 *    once per (device, p, log2 L) under a mutex (transform.py:110-124).
 */
#ifndef MODCONV_B200_H
#define MODCONV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MC_OK = 0,
    MC_EINVAL = 1,        /* usage error -> ValueError                        */
    MC_EUNSUPPORTED = 2,  /* log2 L > 2-adicity (UnsupportedSizeError,
                             field.py:28-33 / transform.py:77-82), or p >= 2^31 */
    MC_ECUDA = 3,         /* CUDA runtime error (message in mc_last_error)    */
    MC_ENOMEM = 4         /* device allocation failed                         */
} mc_status;

/* Library version string. */
const char *mc_version(void);

/* Thread-local message describing the last non-OK status. */
const char *mc_last_error(void);

/* For MC_EUNSUPPORTED caused by a transform size: the 2-adicity the call
 * would have needed (UnsupportedSizeError.required_two_adicity); else -1. */
int mc_last_required_two_adicity(void);

/* Field descriptor (field.py:111-151 FourierPrime.from_modulus):
 * two-adicity and smallest primitive root of p.  Host-only, synchronous.
 * MC_EINVAL if p is not an odd prime. */
mc_status mc_field_info(uint32_t p, int *two_adicity, uint32_t *generator);

/* Principal 2^log2n-th root of unity (field.py:209-224 root_of_unity). */
mc_status mc_root_of_unity(uint32_t p, int log2n, uint32_t *root);

/* Select the primitive root g behind the roots of unity for p on the
 * calling thread (g = 0: back to the smallest primitive root).  The
 * reference's FourierPrime carries any valid generator
 * (field.py:111-131), and TwiddleTable takes w_L = g^((p-1)/L) from it
 * (transform.py:83, field.py:209-224); the transforms (mc_ntt, mc_tft,
 * mc_itft) then match the reference for that generator.  Convolutions do
 * not depend on the choice.  MC_EINVAL if g is not a primitive root mod p. */
mc_status mc_use_generator(uint32_t p, uint32_t g);

/* Build (or find cached) the twiddle tables for (device, p, log2L)
 * (transform.py:73-124 TwiddleTable/get_table).  Optional: every compute
 * call prepares what it needs; calling this up front keeps table
 * construction out of timed regions.  Synchronous. */
mc_status mc_field_prepare(uint32_t p, int log2L, int device);

/* Batched linear convolution by zero-padding to L = next_pow2(z1+z2-1)
 * (convolve.py:160-169 lin_conv_fft_pad -> :143-157 circ_conv_fft).
 * Writes n = z1+z2-1 residues per row of c (not normalized, like the engine
 * function).  Replaces: lin_conv_fft_pad(u, v, req) for each row. */
mc_status mc_conv_fft_pad(const uint32_t *a, int64_t lda, int32_t z1,
                          const uint32_t *b, int64_t ldb, int32_t z2,
                          uint32_t *c, int64_t ldc, int64_t batch,
                          uint32_t p, void *stream);

/* Batched linear convolution by truncated transforms
 * (convolve.py:230-253 conv_tft): n spectral values per operand,
 * n pointwise products, inverse truncated transform, times L^-1.
 * Same layout and output as mc_conv_fft_pad. */
mc_status mc_conv_tft(const uint32_t *a, int64_t lda, int32_t z1,
                      const uint32_t *b, int64_t ldb, int32_t z2,
                      uint32_t *c, int64_t ldc, int64_t batch,
                      uint32_t p, void *stream);

/* Batched circular convolution of length L (power of two)
 * (convolve.py:143-157 circ_conv_fft).  u, v, w: [batch][L] contiguous. */
mc_status mc_circ_conv(const uint32_t *u, const uint32_t *v, uint32_t *w,
                       int32_t log2L, int64_t batch, uint32_t p, void *stream);

/* Definition engine: batched convolution straight from its defining sum,
 * for any modulus 2 <= p < 2^31 (no roots of unity, so any length).
 * circ == 0: linear, c[k] = sum_{i+j=k} a_i b_j, n = z1 + z2 - 1 per row
 *   (convolve.py:71-87 lin_conv_def; poly.py:90-105 schoolbook_raw behind
 *   mul_schoolbook / mul_karatsuba, poly.py:100-169);
 * circ != 0: circular of length n = z1 == z2, c[k] = sum_{i+j=k mod n}
 *   (convolve.py:54-68 circ_conv_def).
 * Rows with leading dimensions lda/ldb/ldc; batch <= 65535.  Inputs may be
 * any 32-bit words (reduced exactly); outputs canonical. */
mc_status mc_conv_direct(const uint32_t *a, int64_t lda, int32_t z1,
                         const uint32_t *b, int64_t ldb, int32_t z2,
                         uint32_t *c, int64_t ldc, int64_t batch,
                         uint32_t p, int32_t circ, void *stream);

/* Eq. 13 split engine.  Residues of each row u (length
 * 2n) mod x^n - 1 and mod x^n + 1: a_j = u_j + u_{j+n}, b_j = u_j - u_{j+n}
 * (convolve.py:214-219 split_residues); u: [batch][2n], a, b: [batch][n]. */
mc_status mc_split_residues(const uint32_t *u, uint32_t *a, uint32_t *b, int32_t log2n,
                            int64_t batch, uint32_t p, void *stream);

/* Inverse of mc_split_residues: w_j = (a_j + b_j)/2, w_{j+n} = (a_j - b_j)/2
 * (convolve.py:222-227 recombine_residues). */
mc_status mc_recombine_residues(const uint32_t *a, const uint32_t *b, uint32_t *w,
                                int32_t log2n, int64_t batch, uint32_t p, void *stream);

/* Batched negacyclic convolution of length n (product mod x^n + 1) by
 * twisting with psi = w_2n (convolve.py:172-190 nega_conv); needs
 * log2(2n) <= two_adicity(p). */
mc_status mc_nega_conv(const uint32_t *u, const uint32_t *v, uint32_t *w, int32_t log2n,
                       int64_t batch, uint32_t p, void *stream);

/* Batched circular convolution of length L = 2n through the split into a
 * circular and a negacyclic half (convolve.py:193-211 circ_conv_split). */
mc_status mc_circ_conv_split(const uint32_t *u, const uint32_t *v, uint32_t *w, int32_t log2L,
                             int64_t batch, uint32_t p, void *stream);

/* Batched full transform, natural order in and out; inverse applies the
 * 1/L scale (transform.py:167-196 moddft).  x, y: [batch][L]. */
mc_status mc_ntt(const uint32_t *x, uint32_t *y, int32_t log2L, int64_t batch,
                 uint32_t p, int inverse, void *stream);

/* Batched truncated transform: first n values, bit-reversed order, of the
 * L-point DFT of x zero-extended from z (transform.py:421-448 tft).
 * Requires 1 <= z <= n <= L.  x: [batch][z] (leading dim z),
 * y: [batch][n]. */
mc_status mc_tft(const uint32_t *x, int32_t z, uint32_t *y, int32_t n,
                 int32_t log2L, int64_t batch, uint32_t p, void *stream);

/* Batched inverse truncated transform: from the first n bit-reversed
 * spectral values recover L*u_i, i < n, assuming u_j = 0 for j >= n
 * (transform.py:492-529 itft).  xhat, y: [batch][n]. */
mc_status mc_itft(const uint32_t *xhat, uint32_t *y, int32_t n, int32_t log2L,
                  int64_t batch, uint32_t p, void *stream);

/* Three-primes CRT (no reference counterpart: SPEC.md:15,402 put it out of
 * the reference's scope).  Garner reconstruction of residues mod
 * p1 = 469762049, p2 = 998244353, p3 = 2013265921 into the exact integer
 * x < p1*p2*p3 < 2^90, written as 3 little-endian 32-bit limbs, planar:
 * limbs[k*n + i] = bits [32k, 32k+32) of x_i. */
mc_status mc_crt3(const uint32_t *r1, const uint32_t *r2, const uint32_t *r3,
                  uint32_t *limbs, int64_t n, void *stream);

/* A slice of the CRT: count coefficients, limbs[k*limb_stride + i].  Any
 * pointer may address a peer GPU's memory (CUDA IPC, NVLink): the
 * distributed three-primes path runs one slice per rank, each reading the
 * residue vectors where they were computed and writing its limbs straight
 * into the destination rank's buffer -- the gather fused into the kernel. */
mc_status mc_crt3_slice(const uint32_t *r1, const uint32_t *r2, const uint32_t *r3,
                        uint32_t *limbs, int64_t limb_stride, int64_t count, void *stream);

/* Peer memory for the distributed CRT (control plane): device allocation
 * with its 64-byte IPC handle; open / close a peer's handle; free. */
mc_status mc_ipc_alloc(int64_t bytes, void **dptr, uint8_t *handle);
mc_status mc_ipc_open(const uint8_t *handle, void **dptr);
mc_status mc_ipc_close(void *dptr);
mc_status mc_ipc_free(void *dptr);
/* Device-to-device copy on `stream` (the destination rank copies the limbs
 * out of its IPC-shared buffer into the caller's tensor). */
mc_status mc_copy_device(void *dst, const void *src, int64_t bytes, void *stream);

/* Three-primes integer product over Z: a (z1 words) and b (z2 words) are
 * non-negative integers < 2^32 (any width; reduced mod each prime on the
 * fly, poly.py:46-49 from_ints semantics); the exact product coefficients
 * (valid while min(z1,z2) * max(a) * max(b) < p1*p2*p3) are written as
 * planar limbs [3][n], n = z1+z2-1.  `scratch` may be NULL (allocated
 * internally, cached per device) or a device buffer of
 * mc_three_primes_scratch_words(z1, z2) words. */
mc_status mc_mul_three_primes(const uint32_t *a, int32_t z1, const uint32_t *b,
                              int32_t z2, uint32_t *limbs, uint32_t *scratch,
                              void *stream);
int64_t mc_three_primes_scratch_words(int32_t z1, int32_t z2);

/* One residue channel of the three-primes product (used when the primes
 * are spread over GPUs): the product mod primes[k] of the reduced inputs,
 * n words written to r.  k in {0,1,2}. */
mc_status mc_mul_mod_prime_k(const uint32_t *a, int32_t z1, const uint32_t *b,
                             int32_t z2, uint32_t *r, int k, void *stream);

/* Host-buffer convenience (synchronous): copies host operands to the
 * current device, runs mc_conv_fft_pad (engine 0) or mc_conv_tft
 * (engine 1) and copies the result back.  Device buffers are cached per
 * thread.  This is the call a C/ctypes caller of the reference's
 * poly-multiply makes without managing device memory. */
mc_status mc_conv_host(int engine, const uint32_t *a, int64_t lda, int32_t z1,
                       const uint32_t *b, int64_t ldb, int32_t z2, uint32_t *c,
                       int64_t ldc, int64_t batch, uint32_t p);

/* Host-buffer batched call, asynchronous.  When a, b and c are page-locked
 * host memory mapped into the unified address space (cudaHostAlloc, torch
 * pin_memory) and the product fits the fused kernel (L <= 8192), the kernel
 * reads the operand rows and writes the products over PCIe itself (zero
 * copy: bulk-copy prefetch in, bulk stores out; MC_NO_ZERO_COPY disables).
 * Otherwise the batch is cut into chunks of `chunk_rows` products
 * (0 = automatic); for each chunk the H2D copy of its operand rows, the
 * convolution kernel and the D2H copy of its products run on three internal
 * streams, so copies in both directions overlap each other and the kernels.
 * The call is ordered after prior work on `stream` and `stream` waits for the
 * last write of c before later work.  The caller must not touch c before
 * synchronizing `stream`. */
mc_status mc_conv_host_async(int engine, const uint32_t *a, int64_t lda, int32_t z1,
                             const uint32_t *b, int64_t ldb, int32_t z2, uint32_t *c,
                             int64_t ldc, int64_t batch, uint32_t p, int64_t chunk_rows,
                             void *stream);

/* Seeded input generator (splitmix64, see oracle/modconv_oracle.c):
 * out[r*ld + i] = gen(seed, stream, row0 + r, i) mod-scaled to [0, hi). */
mc_status mc_gen_u32(uint64_t seed, uint64_t stream_id, uint64_t row0,
                     int64_t rows, int64_t len, uint64_t hi, uint32_t *out,
                     int64_t ld, void *stream);

/* Number of kernels this library has launched in this process (for the
 * bench's gpu_launches accounting). */
int64_t mc_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* MODCONV_B200_H */
