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
#include "chol.cu"
