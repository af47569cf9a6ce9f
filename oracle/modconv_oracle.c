/*
 * modconv_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference `modconv` hot path (pure Python in
 * /root/reference/pkg/src/modconv), used as the parity checker for the CUDA
 * kernels and as the `cpu_baseline` / `--impl reference` arm of bench.py.
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
 * load this library; the product path (paper_1609_01010_b200) never does.
 *
 * Every function cites the reference lines it restates.  Arithmetic is the
 * reference's: canonical residues in [0, p), products reduced with `%` in
 * 64-bit (all supported moduli are < 2^31, so a*b < 2^62 fits).  The
 * algorithms (bit-reversal + iterative radix-2 DIT, the recursive truncated
 * DIF and the van der Hoeven inverse) follow the reference step for step, so
 * the butterfly counts returned here equal the reference OpCounters.
 *
 * Pinned against fixtures produced by the reference itself
 * (tests/golden/make_golden.py writes the tests/golden JSON files; see
 * tests/test_oracle_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

typedef uint64_t u64;
typedef uint32_t u32;
typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------
 * Seeded input generator shared by the oracle, the Python tests, bench.py
 * and the CUDA generator kernel: value i of (seed, stream, row) is
 *   key  = sm64(sm64(sm64(seed) ^ stream) ^ row)
 *   v    = sm64(key + i)
 *   out  = ((v >> 32) * hi) >> 32          (uniform in [0, hi), hi <= 2^32)
 * where sm64 is splitmix64.  Index-addressable, so any product of a batch can
 * be regenerated on its own.
 * ---------------------------------------------------------------------- */
static inline u64 sm64(u64 x) {
    u64 z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

u64 orc_gen_key(u64 seed, u64 stream, u64 row) {
    return sm64(sm64(sm64(seed) ^ stream) ^ row);
}

void orc_gen_u32(u64 seed, u64 stream, u64 row0, int64_t rows, int64_t len,
                 u64 hi, u32 *out, int64_t ld) {
    for (int64_t r = 0; r < rows; ++r) {
        u64 key = orc_gen_key(seed, stream, row0 + (u64)r);
        u32 *o = out + r * ld;
        for (int64_t i = 0; i < len; ++i) {
            u64 v = sm64(key + (u64)i);
            o[i] = (u32)(((v >> 32) * hi) >> 32);
        }
    }
}

/* ------------------------------------------------------------------------
 * Field: reference src/modconv/field.py
 * ---------------------------------------------------------------------- */
static u64 powmod(u64 b, u64 e, u64 p) {
    u64 r = 1 % p;
    b %= p;
    while (e) {
        if (e & 1) r = (u64)((u128)r * b % p);
        b = (u64)((u128)b * b % p);
        e >>= 1;
    }
    return r;
}

/* field.py:98-99 */
int orc_two_adicity(u64 p) {
    u64 n = p - 1;
    int k = 0;
    while (n && !(n & 1)) { n >>= 1; ++k; }
    return k;
}

/* field.py:102-108 (smallest primitive root; factorize by trial division,
 * which is exact for the < 2^62 moduli the reference admits at the sizes
 * tested here) */
u64 orc_primitive_root(u64 p) {
    u64 f[64];
    int nf = 0;
    u64 m = p - 1;
    for (u64 q = 2; q * q <= m; q += (q == 2 ? 1 : 2)) {
        if (m % q == 0) {
            f[nf++] = q;
            while (m % q == 0) m /= q;
        }
    }
    if (m > 1) f[nf++] = m;
    for (u64 g = 2;; ++g) {
        int ok = 1;
        for (int i = 0; i < nf; ++i)
            if (powmod(g, (p - 1) / f[i], p) == 1) { ok = 0; break; }
        if (ok) return g;
    }
}

/* field.py:209-224: w = g^((p-1) >> log2 n), g the smallest primitive root */
u64 orc_root_of_unity(u64 p, int log2n) {
    return powmod(orc_primitive_root(p), (p - 1) >> log2n, p);
}

/* ------------------------------------------------------------------------
 * Twiddle table: transform.py:73-107
 * ---------------------------------------------------------------------- */
typedef struct {
    u64 p;
    int64_t size;
    int log2;
    u64 root;
    u64 *powers;      /* w^j, j < size           (:85-89)  */
    u64 *inv_powers;  /* [1] + powers[:0:-1]     (:91)     */
    u64 inv_size;     /* size^-1                 (:98)     */
    u64 pow2[64];     /* 2^k mod p, k <= log2    (:99)     */
    u64 inv_pow2[64]; /* 2^-k mod p              (:100-101)*/
} orc_table;

static int table_init(orc_table *t, u64 p, int log2) {
    int64_t size = (int64_t)1 << log2;
    if (log2 > orc_two_adicity(p)) return -1; /* UnsupportedSizeError :77-82 */
    t->p = p;
    t->size = size;
    t->log2 = log2;
    t->root = orc_root_of_unity(p, log2);
    t->powers = (u64 *)malloc(sizeof(u64) * size);
    t->inv_powers = (u64 *)malloc(sizeof(u64) * size);
    u64 acc = 1;
    t->powers[0] = 1;
    for (int64_t j = 1; j < size; ++j) {
        acc = acc * t->root % p;
        t->powers[j] = acc;
    }
    t->inv_powers[0] = 1;
    for (int64_t j = 1; j < size; ++j) t->inv_powers[j] = t->powers[size - j];
    t->inv_size = powmod((u64)size % p, p - 2, p);
    u64 inv2 = (p + 1) >> 1;
    for (int k = 0; k <= log2; ++k) {
        t->pow2[k] = powmod(2, k, p);
        t->inv_pow2[k] = powmod(inv2, k, p);
    }
    return 0;
}

static void table_free(orc_table *t) {
    free(t->powers);
    free(t->inv_powers);
}

/* ------------------------------------------------------------------------
 * Full transform: transform.py:127-196
 * ---------------------------------------------------------------------- */
static void dit_inplace(u64 *vec, int64_t n, const u64 *pw, u64 p) {
    /* transform.py:150-164; stage with half-size h uses pw[j * (n/2h)],
     * i.e. fwd_stages[s] = powers[: n/2 : n >> (s+1)] (:106-107) */
    for (int64_t h = 1; h < n; h <<= 1) {
        int64_t step = h << 1, stride = n / step;
        for (int64_t base = 0; base < n; base += step) {
            for (int64_t j = 0; j < h; ++j) {
                int64_t lo = base + j, hi = lo + h;
                u64 t = vec[hi] * pw[j * stride] % p;
                u64 u = vec[lo];
                vec[lo] = (u + t) % p;
                vec[hi] = (u + p - t) % p;
            }
        }
    }
}

static void moddft_t(const orc_table *t, const u64 *x, u64 *y, int inverse) {
    /* transform.py:167-196 */
    int64_t n = t->size;
    int bits = t->log2;
    for (int64_t i = 0; i < n; ++i) {
        int64_t r = 0;
        for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
        y[i] = x[r];
    }
    dit_inplace(y, n, inverse ? t->inv_powers : t->powers, t->p);
    if (inverse)
        for (int64_t i = 0; i < n; ++i) y[i] = y[i] * t->inv_size % t->p;
}

/* ------------------------------------------------------------------------
 * Truncated transforms: transform.py:379-529
 * ---------------------------------------------------------------------- */
static int64_t tft_recurse(u64 *c, int64_t off, int64_t m, int64_t z, int64_t n,
                           int64_t stride, const u64 *pw, u64 p) {
    /* transform.py:379-418 */
    if (n == 0 || m == 1) return 0;
    int64_t h = m >> 1, count, zz;
    if (n > h) {
        if (z > h) {
            for (int64_t i = 0; i < z - h; ++i) {
                int64_t lo = off + i, hi = lo + h;
                u64 a = c[lo], b = c[hi];
                c[lo] = (a + b) % p;
                c[hi] = (a + p - b) % p * pw[i * stride] % p;
            }
            for (int64_t i = z - h; i < h; ++i) {
                int64_t lo = off + i;
                c[lo + h] = c[lo] * pw[i * stride] % p;
            }
            count = h;
            zz = h;
        } else {
            for (int64_t i = 0; i < z; ++i) {
                int64_t lo = off + i;
                c[lo + h] = c[lo] * pw[i * stride] % p;
            }
            count = z;
            zz = z;
        }
        int64_t s2 = stride << 1;
        count += tft_recurse(c, off, h, zz, h, s2, pw, p);
        count += tft_recurse(c, off + h, h, zz, n - h, s2, pw, p);
        return count;
    }
    if (z > h) {
        for (int64_t i = 0; i < z - h; ++i) {
            int64_t lo = off + i;
            c[lo] = (c[lo] + c[lo + h]) % p;
        }
        count = z - h;
        zz = h;
    } else {
        count = 0;
        zz = z;
    }
    return count + tft_recurse(c, off, h, zz, n, stride << 1, pw, p);
}

static int64_t itft_recurse(u64 *c, int64_t off, int64_t m, int64_t n,
                            int64_t stride, const orc_table *t, int mlog) {
    /* transform.py:451-489 */
    if (m == 1 || n == 0) return 0;
    u64 p = t->p;
    int64_t h = m >> 1, s2 = stride << 1, count;
    if (n <= h) {
        for (int64_t j = n; j < h; ++j) {
            int64_t lo = off + j;
            c[lo] = (c[lo] + c[lo + h]) % p;
        }
        count = h - n;
        count += itft_recurse(c, off, h, n, s2, t, mlog - 1);
        u64 m_mod = t->pow2[mlog];
        for (int64_t i = 0; i < n; ++i) {
            int64_t lo = off + i;
            c[lo] = (2 * c[lo] % p + p - m_mod * c[lo + h] % p) % p;
        }
        return count + n;
    }
    count = itft_recurse(c, off, h, h, s2, t, mlog - 1);
    u64 m_mod = t->pow2[mlog];
    u64 inv_h = t->inv_pow2[mlog - 1];
    for (int64_t i = n - h; i < h; ++i) {
        int64_t lo = off + i, hi = lo + h;
        u64 a = c[lo], b = c[hi];
        u64 d = (a * inv_h % p + 2 * (p - b)) % p;
        c[hi] = d * t->powers[i * stride] % p;
        c[lo] = (2 * a % p + p - m_mod * b % p) % p;
    }
    count += h - (n - h);
    count += itft_recurse(c, off + h, h, n - h, s2, t, mlog - 1);
    for (int64_t i = 0; i < n - h; ++i) {
        int64_t lo = off + i, hi = lo + h;
        u64 tt = c[hi] * t->inv_powers[i * stride] % p;
        u64 a = c[lo];
        c[lo] = (a + tt) % p;
        c[hi] = (a + p - tt) % p;
    }
    return count + n - h;
}

/* ------------------------------------------------------------------------
 * Public oracle entry points (u32 residues in, u32 residues out).
 * Return value: butterflies spent (>= 0) or a negative error code:
 *   -1 unsupported size (log2 L > 2-adicity; UnsupportedSizeError)
 *   -2 usage error (ValueError)
 * ---------------------------------------------------------------------- */
static int ilog2_ceil(int64_t n) {
    /* convolve.py:50-51 (_next_pow2) as an exponent */
    int k = 0;
    while (((int64_t)1 << k) < n) ++k;
    return k;
}

/* transform.py:167-196 (moddft) */
int64_t orc_moddft(u32 p, int log2L, const u32 *x, u32 *y, int inverse) {
    orc_table t;
    if (table_init(&t, p, log2L)) return -1;
    int64_t L = t.size;
    u64 *in = (u64 *)calloc((size_t)L, 8), *out = (u64 *)malloc(8 * L);
    if (!in || !out) {
        free(in);
        free(out);
        table_free(&t);
        return -2;
    }
    for (int64_t i = 0; i < L; ++i) in[i] = x[i];
    moddft_t(&t, in, out, inverse);
    for (int64_t i = 0; i < L; ++i) y[i] = (u32)out[i];
    free(in);
    free(out);
    table_free(&t);
    return (L >> 1) * log2L;
}

/* transform.py:421-448 (tft): first n bit-reversed spectral values */
int64_t orc_tft(u32 p, int log2L, const u32 *x, int64_t z, u32 *y, int64_t n) {
    int64_t L = (int64_t)1 << log2L;
    if (z < 1 || z > n || n > L) return -2;
    orc_table t;
    if (table_init(&t, p, log2L)) return -1;
    u64 *c = (u64 *)calloc(L, 8);
    for (int64_t i = 0; i < z; ++i) c[i] = x[i];
    int64_t used = tft_recurse(c, 0, L, z, n, 1, t.powers, p);
    for (int64_t i = 0; i < n; ++i) y[i] = (u32)c[i];
    free(c);
    table_free(&t);
    return used;
}

/* transform.py:492-529 (itft): returns L * u_i for i < n */
int64_t orc_itft(u32 p, int log2L, const u32 *xhat, int64_t n, u32 *y) {
    int64_t L = (int64_t)1 << log2L;
    if (n < 1 || n > L) return -2;
    orc_table t;
    if (table_init(&t, p, log2L)) return -1;
    u64 *c = (u64 *)calloc(L, 8);
    for (int64_t i = 0; i < n; ++i) c[i] = xhat[i];
    int64_t used = itft_recurse(c, 0, L, n, 1, &t, log2L);
    for (int64_t i = 0; i < n; ++i) y[i] = (u32)c[i];
    free(c);
    table_free(&t);
    return used;
}

/* One product with a prepared table.  engine 0 = fft_pad
 * (convolve.py:160-169 -> circ_conv_fft :143-157), engine 1 = tft
 * (convolve.py:230-253).  Writes n = z1 + z2 - 1 coefficients (not
 * normalized, like the engine functions).  Returns butterflies. */
static int64_t conv_one(const orc_table *t, int engine, const u32 *u, int64_t z1,
                        const u32 *v, int64_t z2, u32 *out, u64 *w0, u64 *w1,
                        u64 *w2, int64_t *pointwise) {
    u64 p = t->p;
    int64_t L = t->size, n = z1 + z2 - 1, bf;
    if (engine == 0) {
        memset(w0, 0, 8 * L);
        memset(w1, 0, 8 * L);
        for (int64_t i = 0; i < z1; ++i) w0[i] = u[i];
        for (int64_t i = 0; i < z2; ++i) w1[i] = v[i];
        moddft_t(t, w0, w2, 0);
        moddft_t(t, w1, w0, 0);
        for (int64_t i = 0; i < L; ++i) w1[i] = w2[i] * w0[i] % p; /* :117-140 */
        moddft_t(t, w1, w2, 1);
        for (int64_t i = 0; i < n; ++i) out[i] = (u32)w2[i];
        bf = 3 * (L >> 1) * t->log2;
        *pointwise = L;
    } else {
        memset(w0, 0, 8 * L);
        memset(w1, 0, 8 * L);
        for (int64_t i = 0; i < z1; ++i) w0[i] = u[i];
        for (int64_t i = 0; i < z2; ++i) w1[i] = v[i];
        bf = tft_recurse(w0, 0, L, z1, n, 1, t->powers, p);
        bf += tft_recurse(w1, 0, L, z2, n, 1, t->powers, p);
        memset(w2, 0, 8 * L);
        for (int64_t i = 0; i < n; ++i) w2[i] = w0[i] * w1[i] % p;
        bf += itft_recurse(w2, 0, L, n, 1, t, t->log2);
        for (int64_t i = 0; i < n; ++i) out[i] = (u32)(w2[i] * t->inv_size % p);
        *pointwise = n;
    }
    return bf;
}

typedef struct {
    const orc_table *t;
    int engine;
    const u32 *a, *b;
    int64_t lda, ldb, ldc, z1, z2;
    u32 *c;
    int64_t r0, r1;
    int64_t bf, pw;
} conv_job;

static void *conv_worker(void *arg) {
    conv_job *j = (conv_job *)arg;
    int64_t L = j->t->size;
    u64 *w = (u64 *)malloc(24 * L);
    j->bf = 0;
    j->pw = 0;
    for (int64_t r = j->r0; r < j->r1; ++r) {
        int64_t pw;
        j->bf += conv_one(j->t, j->engine, j->a + r * j->lda, j->z1, j->b + r * j->ldb,
                          j->z2, j->c + r * j->ldc, w, w + L, w + 2 * L, &pw);
        j->pw += pw;
    }
    free(w);
    return NULL;
}

/* Batched engine call: rows r of a (length z1, leading dim lda) times rows of
 * b, written to rows of c (n = z1+z2-1 values).  `threads` host threads.
 * counters[0] += butterflies, counters[1] += pointwise products (the
 * reference OpCounters semantics, transform.py:23-49).  Returns 0 / -1 / -2. */
int orc_conv_batch(u32 p, int engine, const u32 *a, int64_t lda, int64_t z1,
                   const u32 *b, int64_t ldb, int64_t z2, u32 *c, int64_t ldc,
                   int64_t batch, int threads, int64_t *counters) {
    if (z1 < 1 || z2 < 1 || (engine != 0 && engine != 1)) return -2;
    int64_t n = z1 + z2 - 1;
    int log2L = ilog2_ceil(n);
    orc_table t;
    if (table_init(&t, p, log2L)) return -1;
    if (threads < 1) threads = 1;
    if (threads > batch) threads = (int)(batch > 0 ? batch : 1);
    conv_job *jobs = (conv_job *)calloc(threads, sizeof(conv_job));
    pthread_t *th = (pthread_t *)calloc(threads, sizeof(pthread_t));
    for (int i = 0; i < threads; ++i) {
        conv_job *j = &jobs[i];
        j->t = &t;
        j->engine = engine;
        j->a = a;
        j->b = b;
        j->c = c;
        j->lda = lda;
        j->ldb = ldb;
        j->ldc = ldc;
        j->z1 = z1;
        j->z2 = z2;
        j->r0 = batch * i / threads;
        j->r1 = batch * (i + 1) / threads;
        if (threads > 1) pthread_create(&th[i], NULL, conv_worker, j);
        else conv_worker(j);
    }
    int64_t bf = 0, pw = 0;
    for (int i = 0; i < threads; ++i) {
        if (threads > 1) pthread_join(th[i], NULL);
        bf += jobs[i].bf;
        pw += jobs[i].pw;
    }
    if (counters) {
        counters[0] += bf;
        counters[1] += pw;
    }
    free(jobs);
    free(th);
    table_free(&t);
    return 0;
}

/* ------------------------------------------------------------------------
 * Three-primes CRT (no reference counterpart: SPEC.md:15,402 list it as out
 * of the reference's scope; SURVEY.md section 8 a14 defines it).  Garner:
 *   y2 = (r2 - r1) * p1^-1 mod p2
 *   x12 = r1 + p1*y2                      (< p1*p2)
 *   y3 = (r3 - x12) * (p1*p2)^-1 mod p3
 *   x  = x12 + p1*p2*y3                   (< p1*p2*p3 < 2^90)
 * limbs: planar [3][n], little-endian 32-bit words of x.
 * ---------------------------------------------------------------------- */
void orc_crt3(u32 p1, u32 p2, u32 p3, const u32 *r1, const u32 *r2, const u32 *r3,
              int64_t n, u32 *limbs) {
    u64 i12 = powmod(p1 % p2, p2 - 2, p2);
    u64 p12 = (u64)p1 * p2;
    u64 i123 = powmod(p12 % p3, p3 - 2, p3);
    for (int64_t i = 0; i < n; ++i) {
        u64 a = r1[i], b = r2[i], c = r3[i];
        u64 y2 = (b + p2 - a % p2) % p2 * i12 % p2;
        u64 x12 = a + (u64)p1 * y2;
        u64 y3 = (c + p3 - x12 % p3) % p3 * i123 % p3;
        u128 x = (u128)x12 + (u128)p12 * y3;
        limbs[i] = (u32)x;
        limbs[n + i] = (u32)(x >> 32);
        limbs[2 * n + i] = (u32)(x >> 64);
    }
}

/* Full three-primes multiply over Z (oracle): integer inputs < 2^32 reduced
 * mod each prime (poly.py:46-49 from_ints), fft_pad per prime, then Garner.
 * threads >= 3 runs the three primes concurrently (one process
 * per prime); the Garner step is serial. */
typedef struct {
    u32 p;
    const u32 *a, *b;
    int64_t z1, z2, n;
    u32 *res;
    int rc;
} prime_job;

static void *prime_worker(void *arg) {
    prime_job *j = (prime_job *)arg;
    u32 *ra = (u32 *)malloc(4 * j->z1), *rb = (u32 *)malloc(4 * j->z2);
    if (!ra || !rb) {
        free(ra);
        free(rb);
        j->rc = 1;
        return NULL;
    }
    for (int64_t i = 0; i < j->z1; ++i) ra[i] = j->a[i] % j->p;
    for (int64_t i = 0; i < j->z2; ++i) rb[i] = j->b[i] % j->p;
    j->rc = orc_conv_batch(j->p, 0, ra, j->z1, j->z1, rb, j->z2, j->z2, j->res, j->n, 1, 1, NULL);
    free(ra);
    free(rb);
    return NULL;
}

int orc_mul_three_primes(const u32 *a, int64_t z1, const u32 *b, int64_t z2,
                         u32 *limbs, int threads) {
    static const u32 P[3] = {469762049u, 998244353u, 2013265921u};
    int64_t n = z1 + z2 - 1;
    u32 *res = (u32 *)malloc(4 * 3 * n);
    if (!res) return 1;
    prime_job jobs[3];
    pthread_t th[3];
    int started[3] = {0, 0, 0};
    for (int k = 0; k < 3; ++k) {
        prime_job j = {P[k], a, b, z1, z2, n, res + k * n, 0};
        jobs[k] = j;
        if (threads >= 3 && pthread_create(&th[k], NULL, prime_worker, &jobs[k]) == 0)
            started[k] = 1;
        else
            prime_worker(&jobs[k]);
    }
    int rc = 0;
    for (int k = 0; k < 3; ++k) {
        if (started[k]) pthread_join(th[k], NULL);
        if (jobs[k].rc) rc = jobs[k].rc;
    }
    if (!rc) orc_crt3(P[0], P[1], P[2], res, res + n, res + 2 * n, n, limbs);
    free(res);
    return rc;
}

/* Op counts of the reference recursions without doing arithmetic
 * (transform.py:379-418 / :451-489 shapes), used to check the host-side
 * analytic OpCounters of the product package. */
static int64_t tft_count(int64_t m, int64_t z, int64_t n) {
    if (n == 0 || m == 1) return 0;
    int64_t h = m >> 1;
    if (n > h) {
        int64_t c = z > h ? h : z, zz = z > h ? h : z;
        return c + tft_count(h, zz, h) + tft_count(h, zz, n - h);
    }
    if (z > h) return (z - h) + tft_count(h, h, n);
    return tft_count(h, z, n);
}

static int64_t itft_count(int64_t m, int64_t n) {
    if (m == 1 || n == 0) return 0;
    int64_t h = m >> 1;
    if (n == m) { /* complete block: plain inverse DIT, (m/2) log2 m */
        int k = 0;
        while (((int64_t)1 << k) < m) ++k;
        return h * k;
    }
    if (n <= h) return (h - n) + itft_count(h, n) + n;
    return itft_count(h, h) + (h - (n - h)) + itft_count(h, n - h) + (n - h);
}

int64_t orc_tft_count(int log2L, int64_t z, int64_t n) {
    return tft_count((int64_t)1 << log2L, z, n);
}

int64_t orc_itft_count(int log2L, int64_t n) {
    return itft_count((int64_t)1 << log2L, n);
}
