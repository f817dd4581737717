// ops.h -- launchers for the streaming kernels in ops.cu.
#pragma once
#include "kernels.h"

namespace slim {

constexpr int SLIM_HIST_FIXED_DEV = 5;  // must equal SLIM_HIST_FIXED in slimb200.h

struct FinishParams {
  double* x;
  const double* s_parts;  // nsplit x n partial sums of M^T w
  int nsplit;
  int n;
  double alpha;
  const double* refs[MAX_REFS];
  int nref;
  Ctl* ctl;
  double* part;           // grid x (1 + nref) block partials
  double* hist;
  int64_t k;
  int record;
  const double* r;        // residual (ell) for ||r||
  int ell;
  // sharded mode: write the block-reduced partial norms to `norms` and stop;
  // the host allreduces them and k_record takes the decision
  int split;
  double* norms;          // 1 + nref
};

struct RecordParams {
  Ctl* ctl;
  const double* norms;    // ||x||^2, ||x - ref_q||^2 (allreduced)
  const double* r;
  int ell;
  double* hist;
  int64_t k;
  double alpha;
  int record, nref;
};
void launch_record(const RecordParams& R, cudaStream_t s);
// out[i] = sum_q in[q][i] in rank order (in-process shard group)
void launch_group_sum(double* out, const double* const* in, int nin, int64_t count, cudaStream_t s);

// scratch of a column-split row-dot launch: nch partials per row and a
// per-row arrival counter (zero between launches)
struct RowSplit {
  double* part;  // ell x nch
  int* cnt;      // ell
  int nch;
  int vec;       // set by the launcher: 16-byte loads
};
int rowdot_chunks(int ell, int64_t n);
template <typename T>
void launch_residual_dense(double* r, const T* A, int64_t lda, int64_t row0, int64_t brow0,
                           int ell, int n, const double* x, const double* b, const Ctl* ctl,
                           RowSplit rs, cudaStream_t s);
void launch_gen_block(float* dst, float* hi, float* lo, uint64_t seed, int64_t row0, int ell,
                      int n_local, int64_t n_total, int64_t col0, cudaStream_t s);
void launch_gen_apply(double* out, uint64_t seed, int64_t m, int n_local, int64_t n_total,
                      int64_t col0, const double* x, cudaStream_t s);
template <typename T>
void launch_residual_csr(double* r, const int64_t* rowptr, const int* col, const T* val,
                         int64_t row0, int64_t brow0, int ell, const double* x, const double* b,
                         const Ctl* ctl, cudaStream_t s);
// `lut`: scratch of gram_lut_bytes(n, ell) for the per-column records and row
// exponents of the new block (k_gram_rowexp + k_gram_lut + k_gram_csr_fx:
// one gather per nonzero, exact fixed-point sums); nullptr runs the
// pointer-chasing fp64 k_gram_csr.
size_t gram_lut_bytes(int n, int ell);
bool gram_csr_variant(double nnz_per_block);  // true: k_gram_csr_fx
template <typename T>
void launch_gram_csr(double* panel, const Window& W, const int64_t* rowptr, const int* col,
                     const T* val, const int* colptr_new, const int* cscrow, const T* cscval,
                     int64_t base_new, cudaStream_t s, void* lut, int n);
template <typename T>
void launch_gram_dense(double* panel, double* part, int nsplit, const Window& W, const T* A,
                       int64_t lda, int64_t newrow0, int n, cudaStream_t s);
template <typename T>
void launch_mtw_dense(double* part, int nsplit, const Window& W, const T* A, int64_t lda, int n,
                      const double* w, const Ctl* ctl, cudaStream_t s);
template <typename T>
void launch_mtw_csc(double* s_out, const Window& W, const int* colptr, int n, const int* cscrow,
                    const T* cscval, const int64_t* blkbase, const double* w, const Ctl* ctl,
                    cudaStream_t s, int quad = 0);
// M^T w kernel variant for a CSR operator: 0 = one column per thread, 3 =
// four columns per thread with eight entries per block prefetched (dense
// enough columns, n large enough to fill the GPU at n / 4 threads);
// SLIM_MTW_QUAD=<v> overrides
int mtw_variant(int64_t n, double nnz_per_block);
// block list for the batched per-block CSC build of a streamed batch
struct BlkList {
  int n;
  int id[MAX_BATCH];
};
template <typename T>
void launch_build_csc_list(int* colptr, int* cscrow, T* cscval, const int64_t* rowptr, const int* col,
                           const T* val, const int64_t* blkbase, int ell, int n, const BlkList& L,
                           cudaStream_t s);
template <typename T>
void launch_build_csc(int* colptr, int* cscrow, T* cscval, const int64_t* rowptr, const int* col,
                      const T* val, const int64_t* blkbase, int64_t m, int ell, int n,
                      int64_t nblocks, cudaStream_t s, int64_t blk0 = 0, int64_t nblk = -1);
void launch_finish(const FinishParams& F, cudaStream_t s);
// CSC M^T w and the finish in one kernel (s never leaves registers)
template <typename T>
void launch_mtw_finish_csc(const FinishParams& F, const Window& W, const int* colptr,
                           const int* cscrow, const T* cscval, const int64_t* blkbase,
                           const double* w, cudaStream_t s, int quad = 0);
void launch_gram_reduce(double* panel, const Window& W, const double* part, int nsplit,
                        cudaStream_t s);
void launch_gram_diag_fp64(double* panel_diag, int64_t ld, const float* A, int ell, int n,
                           RowSplit rs, cudaStream_t s);
int finish_grid(int n);
// res = y - (I + alpha ring) w in slot order (iterative refinement of w); part:
// nw x ldp partial sums, res: npad entries (the solve's padded length)
struct GramApplyParams {
  const double* panels;
  int64_t panel_stride;
  int ell, nw, newp, npad;
  int slot[MAX_WINDOW], age[MAX_WINDOW];
  double alpha;
  const double* w;   // current solution (nw ell)
  const double* r;   // residual of the new block (ell): y = r on its rows
  double* part;
  int64_t ldp;
  double* res;
  const Ctl* ctl;
};
void launch_gram_apply(const GramApplyParams& G, cudaStream_t s);
void launch_add_inplace(double* w, const double* dw, int count, const Ctl* ctl, cudaStream_t s);
void launch_stamp_start(Ctl* ctl, cudaStream_t s);
void launch_flush_read(const void* buf, size_t bytes, unsigned* sink, cudaStream_t s);

}  // namespace slim
