// Large transforms (L = 2^K > 8192, configs 4 and 5): four-step
// decomposition L = R x C staged through HBM.
//
//   position x = x_hi * C + x_lo   (x_hi < R = 2^KR, x_lo < C = 2^KC)
//
//   col_fwd  (per operand): R-point DIF down every column (natural x_hi ->
//            bit-reversed row r), only the z non-zero inputs are read.
//   row_conv (fused):       per row r (frequency f1 = rev_KR(r)): twist both
//            rows by w_L^(x_lo*f1), C-point DIF of both, pointwise product
//            times L^-1, C-point inverse DIT, inverse twist, write back.
//   col_inv:                R-point inverse DIT up every column
//            (bit-reversed -> natural), write the first n positions.
//
// Position r*C + c' after the forward passes holds X[rev_K(r*C + c')]: the
// same bit-reversed spectrum as the fused small kernel, so both paths share
// the transform conventions of the reference (transform.py).  The row and
// column transforms reuse the fused kernel's register passes
// (conv_small.cuh) with their own stage tables (root w_L^R resp. w_L^C).
#pragma once
#include "runtime.h"

namespace mc {

// Largest K handled by the two-level (R x C) decomposition.
constexpr int kFourStepMaxK = 26;

// Products beyond the four-step limit (L = 2^27 with p3, whose 2-adicity is
// 27): level-scheduled transforms on global memory (transforms.cu), one
// product at a time.  Correct, not fast (~27 global passes per transform).
mc_status levels_conv(const u32 *a, long long lda, int z1, const u32 *b, long long ldb, int z2,
                      u32 *c, long long ldc, long long batch, u32 p, int K, long long n,
                      cudaStream_t st);

mc_status fourstep_conv(int engine, const u32 *a, long long lda, int z1, const u32 *b,
                        long long ldb, int z2, u32 *c, long long ldc, long long batch, u32 p,
                        cudaStream_t st, int circ_log2L, bool reduce_inputs = false,
                        bool fold = false);

}  // namespace mc
