// Host runtime: field arithmetic, twiddle-table cache, error state.
#include <cmath>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "runtime.h"

namespace mc {

// ----------------------------------------------------------------- errors
static thread_local std::string g_err;
static thread_local int g_req_adicity = -1;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string &msg, int req) {
    g_err = msg;
    g_req_adicity = req;
}

mc_status fail(mc_status st, const std::string &msg, int req) {
    set_error(msg, req);
    return st;
}

mc_status cuda_fail(cudaError_t e, const char *what) {
    set_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? MC_ENOMEM : MC_ECUDA;
}

void note_launches(int64_t n) { g_launches += n; }

// ----------------------------------------------------------------- field math
u64 mulmod(u64 a, u64 b, u64 p) { return (u64)((unsigned __int128)a * b % p); }

u64 powmod(u64 b, u64 e, u64 p) {
    u64 r = 1 % p;
    b %= p;
    while (e) {
        if (e & 1) r = mulmod(r, b, p);
        b = mulmod(b, b, p);
        e >>= 1;
    }
    return r;
}

// Deterministic Miller-Rabin for n < 2^32 (bases 2, 7, 61); the reference
// uses a larger witness set valid to 3.3e24 (field.py:18-58).
bool is_prime_u32(u64 n) {
    if (n < 2) return false;
    for (u64 q : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 61ull})
        if (n % q == 0) return n == q;
    u64 d = n - 1;
    int r = 0;
    while (!(d & 1)) {
        d >>= 1;
        ++r;
    }
    for (u64 a : {2ull, 7ull, 61ull}) {
        u64 x = powmod(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int i = 1; i < r; ++i) {
            x = mulmod(x, x, n);
            if (x == n - 1) {
                comp = false;
                break;
            }
        }
        if (comp) return false;
    }
    return true;
}

int two_adicity(u64 p) {
    u64 n = p - 1;
    int k = 0;
    while (n && !(n & 1)) {
        n >>= 1;
        ++k;
    }
    return k;
}

// field.py:102-108: smallest g with g^((p-1)/q) != 1 for every prime q | p-1.
u32 smallest_primitive_root(u32 p) {
    std::vector<u64> f;
    u64 m = p - 1;
    for (u64 q = 2; q * q <= m; ++q) {
        if (m % q == 0) {
            f.push_back(q);
            while (m % q == 0) m /= q;
        }
    }
    if (m > 1) f.push_back(m);
    for (u64 g = 2;; ++g) {
        bool ok = true;
        for (u64 q : f)
            if (powmod(g, (p - 1) / q, p) == 1) {
                ok = false;
                break;
            }
        if (ok) return (u32)g;
    }
}

static thread_local u32 g_gen_p = 0, g_gen_g = 0;

u32 field_generator(u32 p) {
    if (g_gen_p == p && g_gen_g) return g_gen_g;
    static std::mutex mu;
    static std::map<u32, u32> smallest;
    std::lock_guard<std::mutex> lock(mu);
    auto it = smallest.find(p);
    if (it == smallest.end()) it = smallest.emplace(p, smallest_primitive_root(p)).first;
    return it->second;
}

static bool is_primitive_root(u32 g, u32 p) {
    if (g < 2 || g >= p) return false;
    u64 m = p - 1;
    for (u64 q = 2; q * q <= m; ++q) {
        if (m % q) continue;
        if (powmod(g, (p - 1) / q, p) == 1) return false;
        while (m % q == 0) m /= q;
    }
    return m == 1 || powmod(g, (p - 1) / m, p) != 1;
}

Shoup shoup(u32 w, u32 p) {
    Shoup s;
    s.w = w;
    s.wp = (u32)(((u64)w << 32) / p);
    return s;
}

u32 inv_mod(u32 a, u32 p) { return (u32)powmod(a, p - 2, p); }

mc_status check_field(u32 p, int log2L) {
    if (p < 3 || !(p & 1) || !is_prime_u32(p))
        return fail(MC_EINVAL, "modulus must be an odd prime: " + std::to_string(p));
    if (p >= (1u << 31))
        return fail(MC_EUNSUPPORTED,
                    "modulus " + std::to_string(p) + " >= 2^31 is not supported by the GPU path");
    if (log2L < 0) return fail(MC_EINVAL, "negative transform size");
    int a = two_adicity(p);
    if (log2L > a)
        return fail(MC_EUNSUPPORTED,
                    "size " + std::to_string(1ull << log2L) + " needs 2-adicity " +
                        std::to_string(log2L) + ", field p=" + std::to_string(p) + " has " +
                        std::to_string(a),
                    log2L);
    return MC_OK;
}

// ----------------------------------------------------------------- tables
static std::mutex g_tab_mu;
static std::map<std::tuple<int, u32, u32, int>, FieldTables *> g_tabs;

int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

// Keep stream-ordered scratch (cudaMallocAsync) in the device's default pool
// across synchronizations instead of unmapping it each time.
bool lazy_ok(uint32_t p) {
    static const bool off = [] { const char *e = getenv("MC_NO_LAZY"); return e && *e; }();
    return !off && p < (1u << 30);
}

void keep_pool_memory() {
    static bool done[64] = {false};
    const int d = current_device();
    if (d < 64 && done[d]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) {
        unsigned long long thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    if (d < 64) done[d] = true;
}

int sm_count() {
    static int cached[64] = {0};
    int d = current_device();
    if (d < 64 && cached[d]) return cached[d];
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    if (d < 64) cached[d] = n;
    return n;
}

mc_status get_tables(u32 p, int log2L, const FieldTables **out) {
    mc_status st = check_field(p, log2L);
    if (st != MC_OK) return st;
    int dev = current_device();
    const u32 g = field_generator(p);
    auto key = std::make_tuple(dev, p, g, log2L);
    std::lock_guard<std::mutex> lock(g_tab_mu);
    auto it = g_tabs.find(key);
    if (it != g_tabs.end()) {
        *out = it->second;
        return MC_OK;
    }
    FieldTables *T = new FieldTables();
    const u64 L = 1ull << log2L;
    T->p = p;
    T->log2L = log2L;
    T->gen = g;
    T->root = (u32)powmod(g, (p - 1) >> log2L, p);
    // Montgomery inverse p^-1 mod 2^32 (Newton iteration)
    u32 inv = p;
    for (int i = 0; i < 5; ++i) inv *= 2 - p * inv;
    T->pinv = inv;
    u32 li = inv_mod((u32)(L % p), p);
    T->linv = shoup(li, p);
    T->linv_mont = shoup((u32)mulmod(li, (1ull << 32) % p, p), p);
    if (log2L >= 4) {  // level constants of the fused kernel's top pass
        const u64 G = 1ull << (log2L - 4);
        for (int l = 1; l <= 4; ++l) {
            T->mlev[l] = shoup((u32)((G << l) % p), p);
            T->hinv[l] = shoup(inv_mod((u32)((G << (l - 1)) % p), p), p);
        }
    }
    if (log2L > kMaxStageTableLog2) {  // large L: four-step sub-tables only
        g_tabs[key] = T;
        *out = T;
        return MC_OK;
    }
    std::vector<uint2> hf(L > 1 ? L : 2), hi(L > 1 ? L : 2);
    hf[0] = make_uint2(1, (u32)((1ull << 32) / p));
    hi[0] = hf[0];
    for (u64 h = 1; h < L; h <<= 1) {
        u32 w = (u32)powmod(T->root, L / (2 * h), p);  // w_{2h}
        u32 wi = inv_mod(w, p);
        u64 acc = 1, acci = 1;
        for (u64 j = 0; j < h; ++j) {
            Shoup a = shoup((u32)acc, p), b = shoup((u32)acci, p);
            hf[h + j] = make_uint2(a.w, a.wp);
            hi[h + j] = make_uint2(b.w, b.wp);
            acc = mulmod(acc, w, p);
            acci = mulmod(acci, wi, p);
        }
    }
    for (u64 i = 0; i < 16 && i < hf.size(); ++i) {
        T->h16f[i] = hf[i];
        T->h16i[i] = hi[i];
        // RD(w / p): the round-to-nearest quotient stepped down one ulp is <= w / p
        T->h16fd[i] = std::nextafter((double)hf[i].x / (double)p, 0.0);
        T->h16id[i] = std::nextafter((double)hi[i].x / (double)p, 0.0);
    }
    // merged table: L - 1 + log2 L entries, padded to a multiple of 2 (uint4 copies)
    std::vector<uint2> hm;
    for (u64 h = 1; h < L; h <<= 1) {
        const u32 w = (u32)powmod(T->root, L / (2 * h), p);
        u64 acc = 1;
        for (u64 k = 0; k <= h; ++k) {
            Shoup a = shoup((u32)acc, p);
            hm.push_back(make_uint2(a.w, a.wp));
            acc = mulmod(acc, w, p);
        }
    }
    while (hm.size() % 2 || hm.size() < 2) hm.push_back(make_uint2(0, 0));
    T->tm_entries = (int)hm.size();
    size_t bytes = sizeof(uint2) * hf.size();
    cudaError_t e = cudaMalloc(&T->tf, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&T->ti, bytes);
    if (e == cudaSuccess) e = cudaMemcpy(T->tf, hf.data(), bytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(T->ti, hi.data(), bytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&T->tm, sizeof(uint2) * hm.size());
    if (e == cudaSuccess)
        e = cudaMemcpy(T->tm, hm.data(), sizeof(uint2) * hm.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(T->tf);
        cudaFree(T->ti);
        cudaFree(T->tm);
        delete T;
        return cuda_fail(e, "twiddle table upload");
    }
    g_tabs[key] = T;
    *out = T;
    return MC_OK;
}

}  // namespace mc

extern "C" {

const char *mc_version(void) { return "modconv_b200 0.1.0 (sm_100a)"; }

const char *mc_last_error(void) { return mc::g_err.c_str(); }

int mc_last_required_two_adicity(void) { return mc::g_req_adicity; }

int64_t mc_launch_count(void) { return mc::g_launches.load(); }

mc_status mc_field_info(uint32_t p, int *two_adicity, uint32_t *generator) {
    if (p < 3 || !(p & 1) || !mc::is_prime_u32(p))
        return mc::fail(MC_EINVAL, "modulus must be an odd prime: " + std::to_string(p));
    if (two_adicity) *two_adicity = mc::two_adicity(p);
    if (generator) *generator = mc::smallest_primitive_root(p);
    return MC_OK;
}

mc_status mc_root_of_unity(uint32_t p, int log2n, uint32_t *root) {
    if (p < 3 || !(p & 1) || !mc::is_prime_u32(p))
        return mc::fail(MC_EINVAL, "modulus must be an odd prime: " + std::to_string(p));
    if (log2n < 0) return mc::fail(MC_EINVAL, "order must be a power of two");
    int a = mc::two_adicity(p);
    if (log2n > a)
        return mc::fail(MC_EUNSUPPORTED,
                        "order " + std::to_string(1ull << log2n) + " needs 2-adicity " +
                            std::to_string(log2n) + ", field p=" + std::to_string(p) +
                            " has " + std::to_string(a),
                        log2n);
    uint32_t g = mc::field_generator(p);
    if (root) *root = (uint32_t)mc::powmod(g, (uint64_t)(p - 1) >> log2n, p);
    return MC_OK;
}

mc_status mc_use_generator(uint32_t p, uint32_t g) {
    if (g == 0) {
        if (mc::g_gen_p == p) mc::g_gen_p = mc::g_gen_g = 0;
        return MC_OK;
    }
    if (p < 3 || !(p & 1) || !mc::is_prime_u32(p))
        return mc::fail(MC_EINVAL, "modulus must be an odd prime: " + std::to_string(p));
    if (!mc::is_primitive_root(g, p))
        return mc::fail(MC_EINVAL, std::to_string(g) + " is not a primitive root mod " +
                                       std::to_string(p));
    mc::g_gen_p = p;
    mc::g_gen_g = g;
    return MC_OK;
}

mc_status mc_field_prepare(uint32_t p, int log2L, int device) {
    int prev = mc::current_device();
    if (device >= 0 && device != prev) MC_CUDA_CHECK(cudaSetDevice(device));
    const mc::FieldTables *T;
    mc_status st = mc::get_tables(p, log2L, &T);
    if (device >= 0 && device != prev) cudaSetDevice(prev);
    return st;
}

}  // extern "C"
