// kernels.h -- parameter blocks and launch declarations shared by the
// slimLS kernels and the C-ABI driver.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace slim {

// Device-resident run control (one per context).
struct Ctl {
  double rnorm2;          // ||r_k||^2 of the current step
  double div_limit_sq;    // (1e12 (1 + ||x0||))^2, solvers.py:144-146
  int64_t diverged_at;    // 0 = ok, else first diverged step k
  int64_t nrows;          // history rows written
  uint64_t t_start_ns;    // globaltimer at run start
  unsigned int done;      // last-block-done counter for k_finish
  int pad;
};

// one system of a batched factorization
struct CholMat {
  CUtensorMap map;      // TMA view of L: (tiles * 64) x 64 fp64, box 16 x 64, SW128
  double* L;            // lower tiles, tile_off(i, j)
  double* Dinv;         // T x 512: inverses of the 8x8 diagonal blocks of L_jj
  double* Linv;         // T x 4096: inverses of the diagonal tiles (k_diag_inv)
  // int8 digit slices of L for the tensor-core updates (chol.cu, k_chol_i8),
  // by tile column: [k][k half][digit][tile row i < qT][64 rows][32 B], so the
  // A operand of a task (tile rows i, i + 1, all QD digits) is one 3D TMA box;
  // qmapA boxes 128 rows x QD digits, qmapB 64 rows x QD digits (SWIZZLE_32B)
  int8_t* Q;
  CUtensorMap qmapA, qmapB;
  int qT;               // tile rows per column in Q (the buffer's Tmax)
  int* rexp;            // T * 64: row scale exponents, 2^rexp >= sqrt(G_rr)
  int* flags;           // T (T + 1) / 2 epoch flags
  int N, T, nw, epoch;
  double alpha;
  // window positions are fixed slots: the block of step k sits at position
  // (k - 1) mod (r + 1), so consecutive systems differ in one block row
  int pnew;              // position of this step's new block
  int full;              // 1: every tile is recomputed (first step, alpha changed)
  int slot[MAX_WINDOW];  // window position -> ring slot
  int age[MAX_WINDOW];   // window position -> steps since its block arrived (0 = new)
};

struct CholParams {
  CholMat m[MAX_BATCH];
  int nb;               // systems in this launch
  int ntasks;
  const int2* map;      // ticket -> (system, (i << 16) | j); i == j marks a pair task
  int* ticket;          // zeroed before each launch
  int* error;           // set to 1 on a non-positive pivot
  // ring mode: initial tiles gathered from the incremental Gram panels
  const double* panels;
  int64_t panel_stride;  // (r + 1) * ell * ell: one product block per window position
  int ell, S;
  int W;                 // window positions (r + 1)
  int i8;                // 1: k_chol_i8 (int8 tensor-core updates), 0: k_chol_tiles (fp64 DMMA)
  // tiles a system shares with the previous batch's last system (step
  // k0 - 1) are copied from its factor buffer by k_assemble
  const double* prevL;
  const double* prevDinv;
  const int8_t* prevQ;   // digit slices of the previous batch's last system
  // dense mode (panels == nullptr, nb == 1): G is the full SPD matrix, row-major
  const double* G;
  int64_t ldg;
  // optional timeline (debug): 4 globaltimer stamps per ticket
  unsigned long long* trace;
  // k_assemble: first CTA of each system (tile counts prefix-summed)
  int tile_base[MAX_BATCH + 1];
};

struct TrsvParams {
  const double* L;     // factor tiles, tile_off(i, j)
  const double* Linv;  // T x 64 x 64: inverses of the diagonal tiles (row-major)
  int N, T, i0, rstart, rend;  // y = r on rows [rstart, rend), zero elsewhere;
                               // t is zero above tile row i0
  const double* r;     // newest-block residual (ell)
  double* w;           // T * 64 result w = G^{-1} y (window order)
  const Ctl* ctl;      // nullable; skip when diverged
  int C;               // cluster size = grid (tile row i belongs to CTA i mod C)
  int rs;              // bulk-copy ring slots (1..3)
};

// window description shared by the x-chain / Gram kernels
struct Window {
  int nw;                     // blocks in the window
  int ell;
  int blk[MAX_WINDOW];        // storage block of window position (row block of A,
                              // or the generated-block ring slot)
  int slot[MAX_WINDOW];       // ring slot at window position
  int age[MAX_WINDOW];        // steps since the block at the position arrived
  int newp;                   // position of the newest block
};

// batch shape of one system, for the (cached) ticket order
struct SysShape {
  int T, pnew, full;
  bool operator<(const SysShape& o) const {
    return T != o.T ? T < o.T : (pnew != o.pnew ? pnew < o.pnew : full < o.full);
  }
};

// Does step k recompute tile (i, j)?  Only tiles whose rows or columns reach
// the new block's position (or everything, on a full step); the others are
// bit-identical to step k - 1's.
__host__ __device__ inline bool tile_fresh(int full, int pnew, int W, int ell, int i, int j) {
  if (full) return true;
  int pj = (TB * j + TB - 1) / ell;  // last position touched by tile column j
  if (pj > W - 1) pj = W - 1;
  if (pnew <= pj) return true;
  const int s0 = (TB * i) / ell;
  int s1 = (TB * i + TB - 1) / ell;
  if (s1 > W - 1) s1 = W - 1;
  return pnew >= s0 && pnew <= s1;
}

// ---- launchers (ops.cu / chol.cu) ----
void launch_chol(const CholParams& P, cudaStream_t s);
// G tiles of every system of the batch into its factor buffer
// (P.tile_base[b] = first CTA of system b, P.tile_base[nb] = total)
void launch_assemble(const CholParams& P, cudaStream_t s);
// ticket order of one batched factorization launch; cols >= 2 selects the
// banded order (C columns per group, `band` tile rows per band), cols < 2
// the column-by-column order; -1 = SLIM_CHOL_COLS / SLIM_CHOL_BAND or the
// defaults below
constexpr int CHOL_COLS_DEFAULT = 1;
constexpr int CHOL_BAND_DEFAULT = 32;
std::vector<int2> chol_task_map(const SysShape* sh, int nb, int W, int ell, int cols = -1,
                                int band = -1);
// inverses of the diagonal tiles of every system of the batch (after launch_chol)
void launch_diag_inv(const CholParams& P, cudaStream_t s);
// one cluster of P.C CTAs (trsv_cluster_size(T))
cudaError_t launch_trsv(const TrsvParams& P, cudaStream_t s);
int trsv_cluster_size(int T);
size_t trsv_smem_bytes(int T, int C, int rs = 3);


// chol.cu is compiled once per digit layout of the int8 factorization (the
// digit count shapes the TMA boxes, the MMA table and the TMEM accumulators at
// compile time): the default layout in namespace slim, and through
// chol_q6.cu a six-digit layout in namespace slim::q6 whose factors are
// corrected by one step of iterative refinement on the x-chain (capi.cu picks
// one per context).  A translation unit describes itself in `chol_table`.
struct CholVariant {
  int qd, qx, dbits, pairs, tmax;  // digits, extra pair order, digit bits, digit pairs, tile-row limit
  size_t (*q_bytes)(int qT);
  void (*launch_assemble)(const CholParams&, cudaStream_t);
  void (*launch_chol)(const CholParams&, cudaStream_t);
};
extern const CholVariant chol_table;
namespace q6 {
extern const CholVariant chol_table;
}

size_t chol_smem_bytes();
// factorization kernel: true = int8 tensor-core updates (default), false =
// fp64 DMMA updates (SLIM_CHOL=dmma, kept for A/B measurements)
bool chol_use_i8();
// kernel for a system of T tile rows: int8 unless disabled or T exceeds
// CHOL_I8_TMAX (the exact int32 digit-product bound), then fp64 DMMA
bool chol_i8_for(int T);
// signed digits per factor entry in the int8 tensor-core updates
// (k_chol_i8): a leading digit in [-127, 127] (7 bits) and QD - 1 balanced
// digits of DBITS bits each, so 7 + DBITS (QD - 1) bits below each row's scale
#ifndef SLIM_QD
#define SLIM_QD 7
#endif
#ifndef SLIM_DBITS
#define SLIM_DBITS 8
#endif
// SLIM_QX: digit-pair products are kept for a + b <= QD + 1 + QX.  QX = 0
// drops the order a + b = QD + 2 (weight ~2^-53 of the row scales per k
// term, and not random: the iterate error at configs[1] grew to 2.6e-10 of
// the reference's after one epoch); QX = 1 (default) keeps it -- QD - 1 more
// products into an eighth TMEM accumulator, 34 instead of 28 pairs in 12
// instead of 10 MMAs per stage -- for 3% of the factorization's speed
// (operand-bandwidth bound) and a 26x smaller one-epoch error (9.9e-12)
#ifndef SLIM_QX
#define SLIM_QX 1
#endif
constexpr int QD = SLIM_QD;
constexpr int DBITS = SLIM_DBITS;
constexpr int QX = SLIM_QX;
constexpr int QACC = QD + QX;  // TMEM accumulators of 64 columns (t = a + b - 2)
static_assert(QD >= 5 && QD <= 8, "digit count");
static_assert(DBITS == 7 || DBITS == 8, "digit width");
static_assert(QX >= 0 && QACC <= 8, "TMEM holds at most 8 accumulators of 64 columns");
static_assert(QX <= 1, "one extra accumulator: its first writer is the MMA (a = 2, b = QD)");
// B digits multiplied with A digit a (1-based) and the digit-pair count
static __host__ __device__ constexpr int q_nb(int a) { return QD < QD + 1 + QX - a ? QD : QD + 1 + QX - a; }
static __host__ __device__ constexpr int q_pairs(int a = 1) { return a > QD ? 0 : q_nb(a) + q_pairs(a + 1); }
constexpr int QPAIRS = q_pairs();
// int8 updates: |P_t| <= (2 * 127 * H + (QD - 2) * H^2) * 64 T < 2^31 with
// H = 2^(DBITS - 1) the largest trailing digit magnitude
constexpr long long CHOL_I8_PAIRMAX =
    (2LL * 127 * (1 << (DBITS - 1)) + (QD - 2) * (1LL << (2 * (DBITS - 1)))) * 64;
constexpr int CHOL_I8_TMAX =
    (int)(((1LL << 31) - 1) / CHOL_I8_PAIRMAX < 800 ? ((1LL << 31) - 1) / CHOL_I8_PAIRMAX : 800);
// Row width of the digit slices in bytes (SLIM_OZ_SW): 64 = one k tile per
// row, a TMA stage is one k tile under SWIZZLE_64B (default); 32 = the round-1
// layout, one k half per row under SWIZZLE_32B.  A TMA box of 32-byte rows
// delivers at most ~53 GB/s per SM from L2 on B200, 64-byte rows ~99 GB/s
// (tools/microbench/tma_rows.cu, profiles/tma_row_width_r02.txt).
#ifndef SLIM_OZ_SW
#define SLIM_OZ_SW 64
#endif
constexpr int QROW = SLIM_OZ_SW;
static_assert(QROW == 32 || QROW == 64, "digit-slice row width");
// TMA views of a sliced factor buffer with qT tile rows per column (box
// rows = 128 for the A operand, 64 for B; QD digits per box)
bool tma_map_q(CUtensorMap* m, const int8_t* base, int qT, int box_rows, int qd);
// bytes of a sliced factor buffer (the same for both layouts):
//   QROW 32: [k][k half][digit][tile row][64 rows][32 B]
//   QROW 64: [k][digit][tile row][64 rows][64 B]
static inline size_t q_bytes(int qT, int qd = QD) { return (size_t)qT * qT * 2 * qd * 64 * 32; }
// byte offset of row r, k half kh (32 bytes) of digit a (0-based) of the
// sliced tile (i, k)
static __host__ __device__ __forceinline__ int64_t q_off(int qT, int i, int k, int kh, int a, int r) {
  if (QROW == 32) return ((((int64_t)k * 2 * QD + kh * QD + a) * qT + i) * 64 + r) * 32;
  return ((((int64_t)k * QD + a) * qT + i) * 64 + r) * 64 + 32 * kh;
}

}  // namespace slim
