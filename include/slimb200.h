/*
 * slimb200.h -- C-ABI of the B200-native slimLS hot path.
 *
 * Drop-in boundary for the reference's solver entry point
 *   slimsolve.solvers.run("slimls", op, sampler, schedule, *, epochs, r, ...)
 *   (reference pkg/src/slimsolve/solvers.py:480-588)
 * and its secondary kernel-level seam
 *   slimsolve.innersolve.solve_step(..., method="dual") -> dual_step
 *   (reference pkg/src/slimsolve/innersolve.py:305-321, 359-381).
 *
 * Plain C types only: pointers, sizes, status codes.  Host pointers are
 * borrowed for the duration of a call; all device memory is owned by the
 * opaque context.  One context drives one device from one host thread
 * (reference SPEC.md:309: one run owns one state, single-threaded).
 *
 * Status codes map onto the reference's Python exceptions:
 *   SLIM_OK 0
 *   SLIM_EINVAL  -> ValueError       (solvers.py:504-528, linops.py:64-72)
 *   SLIM_ERANGE  -> IndexError       (linops.py:90-94)
 *   SLIM_ENOTSPD -> LinAlgError      (innersolve.py:289-295)
 *   SLIM_ECUDA / SLIM_ENCCL / SLIM_ESTATE -> RuntimeError
 * The message of the last failure is available from slim_last_error().
 */
#ifndef SLIMB200_H
#define SLIMB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SLIM_ABI_VERSION 1

enum slim_status {
  SLIM_OK = 0,
  SLIM_EINVAL = 1,
  SLIM_ERANGE = 2,
  SLIM_ENOTSPD = 3,
  SLIM_ECUDA = 4,
  SLIM_ENCCL = 5,
  SLIM_ESTATE = 6,
  SLIM_ENOMEM = 7
};

/* value dtype of the stored operator (products are always fp64) */
enum slim_dtype { SLIM_F64 = 0, SLIM_F32 = 1 };

/* operator storage layout */
enum slim_layout {
  SLIM_DENSE_ROWMAJOR = 0,   /* DenseBlockOperator (linops.py:142-206)      */
  SLIM_CSR_PERBLOCK = 1,     /* SparseBlockOperator (linops.py:209-299)     */
  SLIM_GEN_SPLITMIX64 = 2    /* generated rows, never stored (configs[4])   */
};

/* step rule of slim_run (slim_set_method) */
enum slim_method {
  SLIM_METHOD_SLIMLS = 0,    /* slimls_step, dual solve (solvers.py:213-242) */
  SLIM_METHOD_SG = 1         /* sg_step: x - alpha A_k^T r (solvers.py:245-250);
                                needs memory_r = 0                           */
};

typedef struct slim_ctx slim_ctx;

/* slim_desc.flags: factor the dual systems with the fp64 DMMA kernel instead of
 * the int8 digit-slice kernel (like SLIM_CHOL=dmma, per context).         */
#define SLIM_FLAG_FP64_FACTOR 1

typedef struct slim_desc {
  int64_t n_rows;      /* m                                                */
  int64_t n_cols;      /* n (columns owned by this context)                */
  int64_t block_rows;  /* ell; m must be divisible (linops.py:64-72)       */
  int64_t memory_r;    /* r >= 0; window holds r+1 blocks (solvers.py:67)  */
  int32_t value_dtype; /* enum slim_dtype                                  */
  int32_t layout;      /* enum slim_layout                                 */
  int32_t device;      /* CUDA device ordinal                              */
  int32_t flags;       /* 0, or SLIM_FLAG_* bits                           */
  uint64_t gen_seed;   /* SLIM_GEN_SPLITMIX64 only                         */
  int64_t gen_n_total; /* generator row length (global n) for GEN layout   */
  int64_t col_offset;  /* first global column of this context's shard      */
} slim_desc;

/* ---- lifetime -------------------------------------------------------- */
int slim_create(slim_ctx** out, const slim_desc* desc);
void slim_destroy(slim_ctx* ctx);
const char* slim_last_error(const slim_ctx* ctx); /* ctx may be NULL */
int slim_abi_version(void);

/* ---- operator upload (replaces RowBlockOperator.fetch_block's storage,
 *      linops.py:192-206 dense views and 270-279 per-fetch densify) ---- */
/* Dense row-major A (n_rows x n_cols, dtype per desc) and b (n_rows).     */
int slim_upload_dense(slim_ctx* ctx, const void* a_rowmajor, const double* b);
/* One CSR block (1-based index): rowptr has ell+1 entries relative to the
 * block, col/val hold rowptr[ell] entries, b_block has ell entries.      */
int slim_upload_csr_block(slim_ctx* ctx, int64_t block, const int64_t* rowptr,
                          const int32_t* col, const void* val, const double* b_block);
/* every block at once (block i + 1 = rowptrs[i], cols[i], vals[i]; b is the
 * whole right-hand side): one call instead of n_blocks                    */
int slim_upload_csr_blocks(slim_ctx* ctx, int64_t count, const int64_t* const* rowptrs,
                           const int32_t* const* cols, const void* const* vals, const double* b);
/* All CSR blocks at once: global rowptr (n_rows+1 entries, int64).       */
int slim_upload_csr(slim_ctx* ctx, const int64_t* rowptr, const int32_t* col,
                    const void* val, const double* b);
/* finalize the uploaded operator (builds per-block CSC for the Gram and
 * the transposed product); must be called before slim_run               */
int slim_finalize_operator(slim_ctx* ctx);
/* right-hand side for the generated layout (n_rows entries)              */
int slim_set_rhs(slim_ctx* ctx, const double* b);
/* generated layout, problem setup: out = A x over all n_rows rows, fp64
 * accumulation of the generated fp32 entries (x has n_cols entries)      */
int slim_gen_apply(slim_ctx* ctx, const double* x, double* out);

/* ---- run state -------------------------------------------------------- */
int slim_set_x(slim_ctx* ctx, const double* x0);          /* n_cols      */
int slim_get_x(slim_ctx* ctx, double* x_out);             /* n_cols      */
/* error references for the history (solvers.py:532-536, 550-552)       */
int slim_set_references(slim_ctx* ctx, int32_t count, const double* const* refs);
/* divergence threshold 1e12 (1 + ||x0||) (solvers.py:144-146)          */
int slim_set_divergence_limit(slim_ctx* ctx, double limit);

/* History row layout written by slim_run, SLIM_HIST_FIXED + n_refs doubles:
 *   [0] k  [1] alpha_k  [2] ||r_k||  [3] device timestamp (ns)
 *   [4] status (0 ok, 1 diverged)  [5..] ||x - ref_q|| (unnormalised)   */
#define SLIM_HIST_FIXED 5

/* Run K slimLS steps over a precomputed 1-based block index trace and
 * alpha_k sequence (Sampler.next_index / Schedule.alpha_at, replaced by a
 * host-side precompute).  Rows are recorded at every step with
 * k % record_every == 0, at k == K, and at a divergence step.
 * hist must hold (K / record_every + 2) * (SLIM_HIST_FIXED + n_refs)
 * doubles; *n_rows receives the count written.  Row k = 0 is NOT written
 * (the host records it, solvers.py:558).  iterates (nullable) receives
 * a copy of x at every recorded row (store_iterates, solvers.py:553).  */
int slim_run(slim_ctx* ctx, const int64_t* block_idx, const double* alphas, int64_t K,
             int64_t record_every, double* hist, int64_t* n_rows, int32_t* status,
             int64_t* diverged_at, double* iterates);

/* Host streaming (replaces the per-step fetch_block of a
 * host operator, linops.py:192-206, 270-279).  Call before uploading: with
 * enable = 1, slim_upload_dense / slim_upload_csr_block only REGISTER the
 * host pointers (they must stay valid while the context may still copy
 * them); slim_finalize_operator sizes the device arrays; slim_run copies
 * each block to HBM on its own stream right before the batch that first
 * samples it (per-block CSC built there), overlapped with earlier device
 * work.  Column indices are validated when a block is copied (SLIM_EINVAL).
 * Results are bit-identical to an operator uploaded up front.  Not for the
 * generated layout or sharded contexts.                                  */
int slim_set_host_streaming(slim_ctx* ctx, int32_t enable);

/* Single-pass .slim stream file as the operator (replaces the reference's
 * FileStreamOperator.fetch_block, linops.py:374-415).  Layout: "SLIM1",
 * then m, n, M, ell as little-endian uint64, then M records of ell*n fp64
 * block rows followed by the block's ell fp64 rhs entries.  The header must
 * match the (dense, fp64) context; the file stays open and slim_run reads
 * each record once, when its block is first sampled, through the pinned
 * ring straight into HBM -- no host copy of the matrix.  SLIM_EINVAL
 * (ValueError) for a bad magic, an inconsistent header or a truncated
 * record, with the reference's messages.  Implies host streaming.        */
int slim_attach_stream_file(slim_ctx* ctx, const char* path);

/* ---- column sharding -------------------------------------
 * Each rank's context holds the columns [col_offset, col_offset + n_cols)
 * of A (and the matching slice of x and of every reference).  Per step the
 * shards exchange, by in-place sum-allreduce: the new Gram panel (on the
 * x-independent stream), the residual partials A_k x_p (rank 0 subtracts
 * b_k) and the norm partials; the factorization is replicated (identical
 * inputs, deterministic kernels), s = alpha M_k^T w and the x update stay
 * local.                                                                  */
/* NCCL over NVLink: 128-byte unique id created on rank 0 with
 * slim_nccl_unique_id and broadcast by the host runtime.                 */
int slim_nccl_unique_id(void* out_128_bytes);
int slim_comm_init(slim_ctx* ctx, const void* nccl_unique_id, int32_t nranks, int32_t rank);
/* In-process group of up to 8 shards on one device, one host thread per
 * shard (test and single-GPU emulation; no kernel waits on another).    */
void* slim_local_group_create(int32_t nranks);
void slim_local_group_destroy(void* group);
int slim_comm_init_local(slim_ctx* ctx, void* group, int32_t rank);
/* column shards only: the batched factorization of batch B
 * runs on rank B mod P alone; that rank's triangular solves give w and the
 * other ranks add zeros in an allreduce of w (N doubles per step), so the
 * replicated factorization cost is divided by P. Results are bit-identical
 * to the replicated mode except for the first system of each batch, which
 * is factored without the previous batch's tiles (same arithmetic).       */
int slim_set_factor_round_robin(slim_ctx* ctx, int32_t enable);
/* step rule of the following slim_run calls (enum slim_method)           */
int slim_set_method(slim_ctx* ctx, int32_t method);

/* ---- secondary seam and kernel-level entry points -------------------- */
/* innersolve.dual_step (innersolve.py:305-321): stacked dense window
 * M (rows x n, row-major fp64, oldest block first), residual of the
 * newest ell rows, alpha.  s_out has n entries.                         */
int slim_dual_step(int32_t device, const double* M, int64_t rows, int64_t n,
                   const double* residual, int64_t ell, double alpha, double* s_out);
/* fp64 Cholesky of an SPD matrix (lower), N x N row-major in/out.       */
int slim_potrf(int32_t device, const double* G, int64_t N, double* L_out);
/* debug variant: per-tile globaltimer trace (4 stamps per ticket: start,
 * accumulation done, dependency ready, published) and the event time     */
int slim_potrf_traced(int32_t device, const double* G, int64_t N, double* L_out,
                      unsigned long long* trace_out, double* ms_out);
/* residual r = A_k x - b_k of one block and its norm (solvers.py:180)   */
int slim_block_residual(slim_ctx* ctx, int64_t block, const double* x, double* r_out,
                        double* norm_out);

/* ---- timing introspection for bench.py -------------------------------- */
/* per-kernel-class device time accumulated over the last slim_run
 * (CUDA events on the launching streams), in milliseconds.
 * which: 0 gram, 1 cholesky, 2 x-chain, 3 whole run (events on sx);
 * which = 5 returns instead the algorithmic fp64 flops of the profiled
 * factorization launches (the tiles they factor; (64 T)^3 / 3 for a
 * from-scratch system) in *ms_out and their count in *launches_out;
 * which = 6 the int8 tensor-core ops of their tile updates (QD (QD + 1) / 2
 * digit-pair products of 2 * 64^3 per 64x64x64 update; 0 with
 * SLIM_CHOL=dmma); which = 7 the digit layout of those updates: the digit
 * count QD in *ms_out and the trailing-digit width in bits in
 * *launches_out (compile-time SLIM_QD / SLIM_DBITS); which = 8 the operator
 * bytes copied host -> device since the operator was registered (block
 * values and columns, row pointers, b; host streaming counts only the
 * blocks a run actually sampled) in *ms_out; which = 9 the digit-pair
 * products per 64^3 tile update in *ms_out and the extra pair order QX
 * (compile-time SLIM_QX) in *launches_out.                               */
int slim_timing(slim_ctx* ctx, int32_t which, double* ms_out, int64_t* launches_out);
int slim_set_profiling(slim_ctx* ctx, int32_t enable);
/* time only steps k0..K of the next slim_run (which = 3 in slim_timing):
 * from the end of step k0-1's x-chain to the end of the run; which = 4
 * returns the number of kernels launched inside that window.           */
int slim_set_timing_start(slim_ctx* ctx, int64_t k0);
/* streaming-kernel probe: `reps` launches of one operator-streaming kernel
 * (0: residual A_k x - b_k, 1: M_k^T w, 2: the new Gram panel A_k M_k^T;
 * 2 is not defined for generated blocks), each on a different window of
 * resident blocks with the L2 flushed in between; returns the mean launch
 * time (us, CUDA events on the x-chain stream) and the algorithmic bytes
 * per launch. Scratch only: the solver state (x, panels, factors) is kept. */
int slim_probe_stream(slim_ctx* ctx, int32_t kernel, int32_t reps, double* us_out,
                      double* bytes_out);

/* ---- problem setup helpers (host side, not the hot path) ------------- */
/* Siddon parallel-beam 2D view block (restates tomo.py:219-273): counts
 * nnz per row when col/val are NULL, otherwise fills them.               */
int slim_siddon2d_view(double angle_deg, int64_t grid, int64_t rays, double spacing,
                       int64_t* rowptr, int32_t* col, double* val);
int slim_siddon3d_view(const double* direction, int64_t grid, int64_t side, double spacing,
                       int64_t* rowptr, int32_t* col, double* val);

/* ---- device projector (tomo.py:304-320) --------------- */
/* Trace the parallel-beam operator on the GPU into a CSR context (no host
 * copy of the matrix). dims 2: `views` = n_views angles in degrees, `rays`
 * rays per view (tomo.py:259-273); dims 3: `views` = n_views x 3 unit
 * directions, `rays` = detector side, rows per view = side^2 (tomo.py:
 * 285-301). Row i of view v is ray ray_of_row[v * rows_per_view + i] of the
 * view (NULL = identity; configs[3]'s permuted sub-blocks). Bit-identical to
 * slim_siddon2d_view / slim_siddon3d_view. Follow with slim_set_rhs and
 * slim_finalize_operator.                                                 */
int slim_build_projector(slim_ctx* ctx, int32_t dims, int64_t grid, int64_t rays, int64_t n_views,
                         const double* views, double spacing, const int32_t* ray_of_row);
/* stored nonzeros of the context's CSR operator (0 for other layouts)   */
int slim_nnz(slim_ctx* ctx, int64_t* nnz_out);
/* out = A x over all rows of a resident CSR operator (or the generated one) */
int slim_apply(slim_ctx* ctx, const double* x, double* out);
/* one resident CSR block back to the host: rowptr_out (ell + 1, relative),
 * then, when non-NULL, its columns and values (the context's value type)  */
int slim_get_csr_block(slim_ctx* ctx, int64_t block, int64_t* rowptr_out, int32_t* col_out,
                       void* val_out);

#ifdef __cplusplus
}
#endif
#endif /* SLIMB200_H */
