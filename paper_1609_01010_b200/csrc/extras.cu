// Standalone transforms and the three-primes CRT path.
#include "runtime.h"

using namespace mc;

extern "C" {

mc_status mc_ntt(const uint32_t *, uint32_t *, int32_t, int64_t, uint32_t, int, void *) {
    return fail(MC_EUNSUPPORTED, "mc_ntt not implemented yet");
}
mc_status mc_tft(const uint32_t *, int32_t, uint32_t *, int32_t, int32_t, int64_t, uint32_t,
                 void *) {
    return fail(MC_EUNSUPPORTED, "mc_tft not implemented yet");
}
mc_status mc_itft(const uint32_t *, uint32_t *, int32_t, int32_t, int64_t, uint32_t, void *) {
    return fail(MC_EUNSUPPORTED, "mc_itft not implemented yet");
}
mc_status mc_crt3(const uint32_t *, const uint32_t *, const uint32_t *, uint32_t *, int64_t,
                  void *) {
    return fail(MC_EUNSUPPORTED, "mc_crt3 not implemented yet");
}
mc_status mc_mul_three_primes(const uint32_t *, int32_t, const uint32_t *, int32_t, uint32_t *,
                              uint32_t *, void *) {
    return fail(MC_EUNSUPPORTED, "not implemented yet");
}
int64_t mc_three_primes_scratch_words(int32_t, int32_t) { return 0; }
mc_status mc_mul_mod_prime_k(const uint32_t *, int32_t, const uint32_t *, int32_t, uint32_t *,
                             int, void *) {
    return fail(MC_EUNSUPPORTED, "not implemented yet");
}

}  // extern "C"
