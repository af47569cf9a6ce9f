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
}  // extern "C"
