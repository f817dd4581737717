// chol_q6.cu -- the factorization kernels (chol.cu) compiled a second time
// with six digits per factor entry and pairs a + b <= 7 (21 digit-pair
// products and six sevenths of the operand bytes of the default 34 / seven):
// 47 bits below each row's scale, truncated.  Contexts that use it (large dual
// systems, where the factorization stream is the bound and the x-chain has
// room) correct w by one step of iterative refinement against the fp64 Gram
// ring (capi.cu: enqueue_x_chain, k_gram_apply), which restores fp64-level
// iterates.  Everything lands in namespace slim::q6.
#define SLIM_QD 6
#define SLIM_QX 0
#define SLIM_CHOL_VARIANT q6
// Six digits make a TMA stage 72 KB, so a THREE-stage operand ring fits an SM
// (217 KB; seven digits: 3 x 84 KB does not).  Measured with two stages:
// configs[2] 145.3 it/s, configs[3] 158.2; with three: 154.1 and 171.6, same
// bits (profiles/chol_q6_stages_r02.txt) -- the operand bytes in flight per SM
// were what held the two-stage kernel.  SLIM_Q6_NST=2 rebuilds the two-stage ring.
#ifndef SLIM_Q6_NST
#define SLIM_Q6_NST 3
#endif
#define SLIM_OZ_NST SLIM_Q6_NST
#include "chol.cu"
