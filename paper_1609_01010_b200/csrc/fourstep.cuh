// Large transforms (L > 8192): four-step decomposition staged through HBM.
#pragma once
#include "runtime.h"

namespace mc {

mc_status fourstep_conv(int engine, const u32 *a, long long lda, int z1, const u32 *b,
                        long long ldb, int z2, u32 *c, long long ldc, long long batch, u32 p,
                        cudaStream_t st, int circ_log2L);

}  // namespace mc
