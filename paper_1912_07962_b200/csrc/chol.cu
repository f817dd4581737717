// chol.cu -- fp64 tile-DAG Cholesky of the slimLS dual system and the
// triangular solves that apply its inverse.
//
// Replaces the reference's per-step
//     G = alpha * (M M^T) + I              (innersolve.py:298-302)
//     w = scipy.linalg.solve(G, y, assume_a="pos")   (innersolve.py:320)
// where y = [0 .. 0; r] (innersolve.py:317-319).
//
// Design (B200): one launch factors the whole (N x N) system.  The lower
// triangle is cut into 64x64 fp64 tiles stored tile-major; each CTA takes
// one tile from an atomic ticket in column-major order and runs the
// left-looking update
//     C_ij = G_ij - sum_{k<j} L_ik L_jk^T        (DMMA m8n8k4, fp64)
// then POTRF (diagonal) or TRSM against L_jj (off-diagonal), and publishes
// the tile with a release flag.  Every dependency of ticket t has a smaller
// ticket, handed to a CTA that is already resident, so spinning on acquire
// flags cannot deadlock.  G is never assembled: the initial C_ij is
// gathered straight from the ring of incremental Gram panels (alpha
// scaling and +I fused).
//
// The factorization is critical-path bound (64 dependent pivots per tile
// column), so the finalize steps are built for latency: POTRF works on
// 8-wide panels (one warp factors the panel with shuffles, DMMA applies
// the trailing update, 16 barriers per tile instead of 64), and it also
// stores the inverses of the eight 8x8 diagonal blocks of L_jj.  The
// off-diagonal TRSM is then warp-local -- each warp owns 8 rows of X and
// solves X L^T = C block by block with DMMA (no CTA barrier) -- and the
// triangular solves of the x-chain reuse the same small inverses.  Only
// 8x8 blocks are inverted, so the backward error stays that of a
// substitution (the 8x8 blocks of a Cholesky factor are well conditioned).
#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace slim {
#ifdef SLIM_CHOL_VARIANT
namespace SLIM_CHOL_VARIANT {  // a second digit layout (chol_q6.cu)
#endif

constexpr unsigned FULL = 0xffffffffu;


// per-CTA view of its system, in registers (indexing the kernel-parameter
// array with the runtime system id would turn every field access into a
// dynamically indexed constant load)
struct MatRT {
  const CUtensorMap* map;  // kernel-parameter (grid-constant) TMA view of L
  double* L;
  double* Dinv;
  int* flags;
  int N, T, epoch;
  double alpha;
};

__device__ __forceinline__ void load_tile_async(double* s, const double* g, int tid) {
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int c = tid + it * 256;  // 2048 16-byte chunks
    const int row = c >> 5, cc = (c & 31) * 2;
    cp_async16(s + row * TS + cc, g + row * TB + cc);
  }
}

__device__ __forceinline__ void load_dinv_async(double* s, const double* g, int tid) {
  if (tid < 256) cp_async16(s + 2 * tid, g + 2 * tid);  // 512 doubles
}

__device__ __forceinline__ void store_tile(double* g, const double* s, int tid) {
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int c = tid + it * 256;
    const int row = c >> 5, cc = (c & 31) * 2;
    const double2 v = *reinterpret_cast<const double2*>(s + row * TS + cc);
    *reinterpret_cast<double2*>(g + row * TB + cc) = v;
  }
}

// fp64 1/sqrt(x): MUFU.RSQ64H seed + two Newton steps (~1 ulp), so the
// pivot chain pays ~50 cycles per column instead of a sqrt and a divide
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  double e = fma(-h * y, y, 0.5);
  y = fma(y, e, y);
  e = fma(-h * y, y, 0.5);
  return fma(y, e, y);
}

// ---------------------------------------------------------------------------
// POTRF of the 64x64 tile in S (lower part valid), plus the inverses of its
// eight 8x8 diagonal blocks into Dv[q * 64 + i * 8 + k] (lower, row-major).
// Panels of 8 columns: warp 0 factors the panel in registers; the lane that
// owns the next pivot row computes that pivot's reciprocal square root
// before the rest of the rank-1 update, so the serial chain per column is
// one shuffle, one multiply, one FMA and one rsqrt.
// ---------------------------------------------------------------------------
__device__ void potrf_tile_blocked(double* S, double* Dv, double* rdiag, int tid, int* error) {
  const int warp = tid >> 5, lane = tid & 31;
  for (int p = 0; p < 8; ++p) {
    const int c0 = 8 * p;
    if (warp == 0) {
      const int r0 = c0 + lane, r1 = r0 + 32;
      double v0[8], v1[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        v0[c] = (r0 < TB) ? S[r0 * TS + c0 + c] : 0.0;
        v1[c] = (r1 < TB) ? S[r1 * TS + c0 + c] : 0.0;
      }
      bool bad = (lane == 0) && !(v0[0] > 0.0);
      double myinv = rsqrt_nr(v0[0]);  // meaningful on lane 0 only
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double inv = __shfl_sync(FULL, myinv, c);
        const double l0 = v0[c] * inv, l1 = v1[c] * inv;
        if (c < 7) {
          // next pivot, on the lane that owns row c0 + c + 1
          const double dn = fma(-l0, l0, v0[c + 1]);
          if (lane == c + 1) {
            bad |= !(dn > 0.0);
            myinv = rsqrt_nr(dn);
          }
        }
#pragma unroll
        for (int j = c + 1; j < 8; ++j) {
          const double ljc = __shfl_sync(FULL, l0, j);
          v0[j] = fma(-l0, ljc, v0[j]);
          v1[j] = fma(-l1, ljc, v1[j]);
        }
        v0[c] = l0;
        v1[c] = l1;
        if (lane == c) rdiag[c0 + c] = inv;
      }
      if (__any_sync(FULL, bad) && lane == 0) atomicExch(error, 1);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (r0 < TB) S[r0 * TS + c0 + c] = (lane >= c) ? v0[c] : 0.0;
        if (r1 < TB) S[r1 * TS + c0 + c] = v1[c];
      }
    }
    __syncthreads();
    // trailing update of 8x8 blocks (bi, bj), p < bj <= bi <= 7, via DMMA
    const int nb = 7 - p;
    const int nblk = nb * (nb + 1) / 2;
    // up to 4 blocks per warp, two independent chains at a time
#pragma unroll 1
    for (int u0 = 0; u0 < 4; u0 += 2) {
      double acc[2][2], a[2][2], b[2][2];
      int off[2];
      bool on[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int e = warp + 8 * (u0 + u);
        on[u] = e < nblk;
        int bi = p + 1, rem = on[u] ? e : 0;
        while (rem > bi - (p + 1)) {
          rem -= bi - p;
          ++bi;
        }
        const int bj = p + 1 + rem;
        off[u] = (8 * bi + (lane >> 2)) * TS + 8 * bj + 2 * (lane & 3);
        if (on[u]) {
          acc[u][0] = S[off[u]];
          acc[u][1] = S[off[u] + 1];
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            a[u][ks] = -S[(8 * bi + (lane >> 2)) * TS + c0 + 4 * ks + (lane & 3)];
            b[u][ks] = S[(8 * bj + (lane >> 2)) * TS + c0 + 4 * ks + (lane & 3)];
          }
        }
      }
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int u = 0; u < 2; ++u)
          if (on[u]) dmma8x8x4(acc[u], a[u][ks], b[u][ks]);
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (on[u]) {
          S[off[u]] = acc[u][0];
          S[off[u] + 1] = acc[u][1];
        }
    }
    __syncthreads();
  }
  // zero the strict upper triangle of the off-diagonal 8x8 blocks
  for (int e = tid; e < TB * TB; e += 256) {
    const int r = e >> 6, c = e & 63;
    if ((c >> 3) > (r >> 3)) S[r * TS + c] = 0.0;
  }
  // inverses of the diagonal 8x8 blocks: warp q, lane c < 8 solves column c
  if (lane < 8) {
    const int q = warp, c = lane;
    const double* L = S + (8 * q) * TS + 8 * q;
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < i; ++k) s -= L[i * TS + k] * x[k];
      x[i] = s * rdiag[8 * q + i];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) Dv[q * 64 + i * 8 + c] = x[i];
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// X L^T = C (X, C: 64x64 in X (stride TS); L = L_jj in Lj; Dv = inverses of
// its 8x8 diagonal blocks).  Warp w owns rows 8w..8w+7 and never waits on
// another warp: column block q is X_q = (C_q - sum_{p<q} X_p L_qp^T) Dinv_q^T.
// ---------------------------------------------------------------------------
__device__ void trsm_tile_warp(double* As, const double* Bs, const double* Dv, int warp,
                               int lane) {
  const int rowA = (8 * warp + (lane >> 2)) * TS;
  const int rowB = lane >> 2, colk = lane & 3;
#pragma unroll 1
  for (int q = 0; q < 8; ++q) {
    double* cp = As + rowA + 8 * q + 2 * colk;
    double acc[2] = {cp[0], cp[1]};
    for (int p = 0; p < q; ++p) {
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const double a = -As[rowA + 8 * p + 4 * ks + colk];
        const double b = Bs[(8 * q + rowB) * TS + 8 * p + 4 * ks + colk];
        dmma8x8x4(acc, a, b);
      }
    }
    __syncwarp();
    cp[0] = acc[0];
    cp[1] = acc[1];
    __syncwarp();
    double x2[2] = {0.0, 0.0};
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const double a = As[rowA + 8 * q + 4 * ks + colk];
      const double b = Dv[q * 64 + rowB * 8 + 4 * ks + colk];
      dmma8x8x4(x2, a, b);
    }
    __syncwarp();
    cp[0] = x2[0];
    cp[1] = x2[1];
    __syncwarp();
  }
}

// the same for two right-hand tiles X1, X2 at once: two independent DMMA
// chains per warp
__device__ void trsm_tile_warp2(double* A1, double* A2, const double* Bs, const double* Dv, int warp,
                                int lane) {
  const int rowA = (8 * warp + (lane >> 2)) * TS;
  const int rowB = lane >> 2, colk = lane & 3;
#pragma unroll 1
  for (int q = 0; q < 8; ++q) {
    double* c1 = A1 + rowA + 8 * q + 2 * colk;
    double* c2 = A2 + rowA + 8 * q + 2 * colk;
    double acc1[2] = {c1[0], c1[1]}, acc2[2] = {c2[0], c2[1]};
    for (int p = 0; p < q; ++p) {
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const double b = Bs[(8 * q + rowB) * TS + 8 * p + 4 * ks + colk];
        dmma8x8x4(acc1, -A1[rowA + 8 * p + 4 * ks + colk], b);
        dmma8x8x4(acc2, -A2[rowA + 8 * p + 4 * ks + colk], b);
      }
    }
    __syncwarp();
    c1[0] = acc1[0];
    c1[1] = acc1[1];
    c2[0] = acc2[0];
    c2[1] = acc2[1];
    __syncwarp();
    double x1[2] = {0.0, 0.0}, x2[2] = {0.0, 0.0};
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const double b = Dv[q * 64 + rowB * 8 + 4 * ks + colk];
      dmma8x8x4(x1, A1[rowA + 8 * q + 4 * ks + colk], b);
      dmma8x8x4(x2, A2[rowA + 8 * q + 4 * ks + colk], b);
    }
    __syncwarp();
    c1[0] = x1[0];
    c1[1] = x1[1];
    c2[0] = x2[0];
    c2[1] = x2[1];
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// tile Cholesky kernel
// ---------------------------------------------------------------------------
// K chunks of 16 fp64 (one 128-byte swizzle row per tile row) stream through a
// 3-stage TMA ring: a stage holds the 64x16 slices of up to three operand
// tiles (A, B, and the second A of a dual task).
constexpr int KC = 16;
constexpr int NSTAGE = 3;
constexpr int BOX_BYTES = TB * KC * 8;         // 8 KB
constexpr int STAGE_BYTES = 3 * BOX_BYTES;     // 24 KB

// dynamic shared layout (bytes, from a 1024-aligned base):
//   stage ring [NSTAGE][STAGE_BYTES] | Sg[TB*TS] | Dv[512] | rdiag[64]
// the 64 x TS work tiles X (two for a dual task) overlay the stage ring once
// the operands are consumed; two CTAs fit an SM (2 x 112 KB)
constexpr int SMB_ST = 0;
constexpr int SMB_SG = NSTAGE * STAGE_BYTES;
constexpr int SMB_DV = SMB_SG + TB * TS * 8;
constexpr int SMB_RD = SMB_DV + 512 * 8;
constexpr int SMB_TOTAL = SMB_RD + 64 * 8 + 1024;  // + alignment slack
static_assert(2 * TB * TS * 8 <= SMB_SG, "two work tiles must fit over the stage ring");

// the tile (i, j) of G was assembled in place by k_assemble (tile-major)
__device__ __forceinline__ void init_acc(const CholParams& P, const MatRT& M, int i, int j,
                                         int warp, int lane, double (&acc)[8][2]) {
  // warp tile: rows 16 (warp >> 1) .. +15, columns 32 (warp & 1) .. +31;
  // accumulator f = rb * 4 + cb holds the 8x8 block (rb, cb) of it
  (void)P;
  const double* t = M.L + tile_off(i, j);
#pragma unroll
  for (int f = 0; f < 8; ++f) {
    const int r = 16 * (warp >> 1) + 8 * (f >> 2) + (lane >> 2);
    const int c = 32 * (warp & 1) + 8 * (f & 3) + 2 * (lane & 3);
    const double2 v = __ldcg(reinterpret_cast<const double2*>(t + r * TB + c));
    acc[f][0] = v.x;
    acc[f][1] = v.y;
  }
}

// G = alpha * (Gram ring) + I, identity padding, written tile-major into the
// factor buffers (one CTA per 64x64 tile of every system of the batch).
// Entry (p, q) is the product of two window blocks; the ring keeps it in the
// panel of the newer of the two (ring slot), at the older one's window
// position (fixed for a block's lifetime), newer block's rows contiguous.
// Pass 1 reads the entries whose row block is the newer one with threads
// along p, pass 2 the others with threads along q (both coalesced); the
// tile is transposed through shared memory into row-major order.
// Tiles that are not fresh for this step are either produced by an earlier
// system of the batch (its tile task stores them here) or, when no system of
// the batch recomputes them, copied from the previous batch's last system.
__global__ void __launch_bounds__(256) k_assemble(CholParams P) {
  __shared__ double sh[TB][TB + 1];
  // locate (system, tile) of this CTA
  int b = 0;
  while (b + 1 < P.nb && (int)blockIdx.x >= P.tile_base[b + 1]) ++b;
  const CholMat& Mp = P.m[b];
  int t = blockIdx.x - P.tile_base[b];
  int I = 0;
  while (t > I) {
    t -= I + 1;
    ++I;
  }
  const int J = t;
  const int N = Mp.N, ell = P.ell;
  const int tid = threadIdx.x;
  const int64_t toff = tile_off(I, J);
  if (I == J && Mp.rexp != nullptr && tid < TB) {
    // row scales of the int8 digit slices: 2^e >= sqrt(G_pp) >= |L_pk|
    // (every system, fresh or not: the same G_pp gives the same exponent)
    const int p = I * TB + tid;
    double gpp = 1.0;
    if (p < N) {
      if (P.panels != nullptr) {
        const int pb = p / ell, a = p - pb * ell;
        const double* pan = P.panels + (int64_t)Mp.slot[pb] * P.panel_stride;
        gpp = Mp.alpha * pan[((int64_t)pb * ell + a) * ell + a] + 1.0;
      } else {
        gpp = P.G[(int64_t)p * P.ldg + p];
      }
    }
    // 2^e >= 1.004 sqrt(gpp): |L_pk| 2^(7 - e) < 127.5, so the leading digit
    // rounds into [-127, 127]
    int e = 0;
    frexp(1.004 * sqrt(fmax(gpp, 1e-300)), &e);
    Mp.rexp[p] = e;
  }
  if (!tile_fresh(Mp.full, Mp.pnew, P.W, ell, I, J)) {
    for (int bb = b - 1; bb >= 0; --bb)
      if (tile_fresh(P.m[bb].full, P.m[bb].pnew, P.W, ell, I, J)) return;  // produced in-batch
    const double2* src = reinterpret_cast<const double2*>(P.prevL + toff);
    double2* dst = reinterpret_cast<double2*>(Mp.L + toff);
    for (int e = tid; e < TB * TB / 2; e += 256) dst[e] = __ldcg(src + e);
    if (Mp.Q != nullptr && P.prevQ != nullptr && I != J) {  // 2 QD contiguous runs of 2 KB
      for (int e = tid; e < 2 * QD * 128; e += 256) {
        const int blk = e >> 7;  // QROW 32: (k half, digit); 64: (digit, half of its 4 KB)
        const int64_t off = (QROW == 32 ? q_off(Mp.qT, I, J, blk / QD, blk % QD, 0)
                                        : q_off(Mp.qT, I, J, 0, blk >> 1, 0) + (blk & 1) * 2048) +
                            (int64_t)(e & 127) * 16;
        *reinterpret_cast<uint4*>(Mp.Q + off) = __ldcg(reinterpret_cast<const uint4*>(P.prevQ + off));
      }
    }
    if (I == J)
      for (int e = tid; e < 512; e += 256) Mp.Dinv[(int64_t)J * 512 + e] = __ldcg(P.prevDinv + (int64_t)J * 512 + e);
    if (tid == 0) Mp.flags[I * (I + 1) / 2 + J] = Mp.epoch;  // next kernel: stream-ordered
    return;
  }
  const double alpha = Mp.alpha;
  const int ll = tid & 63;
  // pass 1: threads along p
  {
    const int p = I * TB + ll;
    const bool prow = p < N;
    const int pb = prow ? p / ell : 0, a = p - pb * ell;
    for (int qs = tid >> 6; qs < TB; qs += 4) {
      const int q = J * TB + qs;
      double v;
      if (!prow || q >= N) v = (p == q) ? 1.0 : 0.0;
      else if (q > p) v = 0.0;
      else if (P.panels != nullptr) {
        const int qb = q / ell, c = q - qb * ell;
        if (Mp.age[qb] < Mp.age[pb]) continue;  // column block newer: pass 2
        const double* pan = P.panels + (int64_t)Mp.slot[pb] * P.panel_stride;
        v = alpha * pan[((int64_t)qb * ell + c) * ell + a] + (p == q ? 1.0 : 0.0);
      } else {
        v = P.G[(int64_t)p * P.ldg + q];
      }
      sh[ll][qs] = v;
    }
  }
  // pass 2: threads along q, entries whose column block is the newer one
  if (P.panels != nullptr) {
    const int q = J * TB + ll;
    if (q < N) {
      const int qb = q / ell, c = q - qb * ell;
      const double* pan = P.panels + (int64_t)Mp.slot[qb] * P.panel_stride;
      for (int ps = tid >> 6; ps < TB; ps += 4) {
        const int p = I * TB + ps;
        if (p >= N || q > p) continue;
        const int pb = p / ell, a = p - pb * ell;
        if (!(Mp.age[qb] < Mp.age[pb])) continue;
        sh[ps][ll] = alpha * pan[((int64_t)pb * ell + a) * ell + c];
      }
    }
  }
  __syncthreads();
  double* dst = Mp.L + toff;
  for (int e = tid; e < TB * TB; e += 256) dst[e] = sh[e >> 6][e & 63];
}

// ---- TMA + mbarrier pipeline helpers ----
struct Pipe {
  uint64_t* full;    // NSTAGE, tx-count barriers (one arrival: the producer)
  uint64_t* empty;   // NSTAGE, one arrival per consumer warp
  uint32_t seq;      // chunks consumed so far by this CTA (uniform)
};

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(dst)),
      "l"(map), "r"(su32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(dst)),
      "l"(map), "r"(su32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}
// the same with an L2 eviction-priority hint (CUTLASS's CacheHintSm90 values)
__device__ __forceinline__ void tma3d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                           int z, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(su32(dst)),
      "l"(map), "r"(su32(bar)), "r"(x), "r"(y), "r"(z), "l"(policy)
      : "memory");
}
constexpr uint64_t L2_EVICT_FIRST = 0x12F0000000000000ull, L2_EVICT_LAST = 0x14F0000000000000ull;
// generic-proxy writes of other CTAs (acquired through a flag) made visible
// to this thread's subsequent async-proxy (TMA) reads
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}


// C_(ra, j) -= sum_{k in [kb, ke)} L_(ra,k) L_(j,k)^T into accA, and
//   MODE 1 (pair): also C_(j,j)    -= L_(j,k)    L_(j,k)^T into accB,
//   MODE 2 (dual): also C_(ra+1,j) -= L_(ra+1,k) L_(j,k)^T into accB
// (the B operand L_(j,k) shared: 16 independent DMMAs per 8 fragment loads).
// Thread 0 issues one 2D TMA box per operand per K chunk (64 rows x 16 fp64,
// SWIZZLE_128B) two chunks ahead; every warp releases a stage with one
// mbarrier arrival, so there is no CTA-wide barrier in the loop.  Dependency
// flags are probed once; only k-steps past the ready prefix make thread 0 wait.
template <int MODE>
__device__ void accumulate(const MatRT& P, int ra, int j, int kb, int ke, uint8_t* stage,
                           Pipe& pipe, double (&accA)[8][2], double (&accB)[8][2], int tid) {
  constexpr bool TWO = MODE != 0;
  constexpr int NBOX = MODE == 2 ? 3 : 2;
  const int warp = tid >> 5, lane = tid & 31;
  const int nchunk = (TB / KC) * (ke - kb);
  if (nchunk <= 0) return;
  // Thread 0 -- the TMA issuer -- probes every dependency flag of the task
  // once with relaxed loads, then one acquire fence and one proxy fence make
  // all the ready tiles visible to its async-proxy (TMA) reads.
  int kready = ke;
  if (tid == 0) {
    const int* fa = P.flags + ra * (ra + 1) / 2;
    const int* fb = P.flags + j * (j + 1) / 2;
    const int* fc = P.flags + (ra + 1) * (ra + 2) / 2;
    for (int k = kb; k < ke; ++k) {
      int va, vb, vc = P.epoch;
      asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(va) : "l"(fa + k) : "memory");
      asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(vb) : "l"(fb + k) : "memory");
      if (MODE == 2) asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(vc) : "l"(fc + k) : "memory");
      if (va < P.epoch || vb < P.epoch || vc < P.epoch) {
        kready = k;
        break;
      }
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    fence_proxy_async();
  }
  auto issue = [&](int u) {  // thread 0 only
    const uint32_t q = pipe.seq + u;
    const int st = q % NSTAGE;
    bar_wait(&pipe.empty[st], ((q / NSTAGE) & 1) ^ 1);
    const int k = kb + u / (TB / KC), c = u % (TB / KC);
    if (c == 0 && k >= kready) {
      wait_flag(P.flags + (ra * (ra + 1) / 2 + k), P.epoch);
      wait_flag(P.flags + (j * (j + 1) / 2 + k), P.epoch);
      if (MODE == 2) wait_flag(P.flags + ((ra + 1) * (ra + 2) / 2 + k), P.epoch);
      fence_proxy_async();
    }
    uint8_t* dst = stage + st * STAGE_BYTES;
    bar_expect(&pipe.full[st], NBOX * BOX_BYTES);
    tma2d(dst, P.map, &pipe.full[st], KC * c, (ra * (ra + 1) / 2 + k) * TB);
    tma2d(dst + BOX_BYTES, P.map, &pipe.full[st], KC * c, (j * (j + 1) / 2 + k) * TB);
    if (MODE == 2)
      tma2d(dst + 2 * BOX_BYTES, P.map, &pipe.full[st], KC * c, ((ra + 1) * (ra + 2) / 2 + k) * TB);
  };
  if (tid == 0)
    for (int u = 0; u < NSTAGE - 1 && u < nchunk; ++u) issue(u);
  // swizzled fragment offsets: row r of a box is 128 B, the 16-byte chunk
  // holding columns (2 m, 2 m + 1) sits at position m ^ (r & 7); every
  // fragment row base is a multiple of 8, so r & 7 = lane >> 2
  const int sw = lane >> 2;
  uint32_t colofs[KC / 4];
#pragma unroll
  for (int k4 = 0; k4 < KC / 4; ++k4)
    colofs[k4] = (uint32_t)((((2 * k4 + ((lane & 3) >> 1)) ^ sw) << 4) + ((lane & 1) << 3));
  const uint32_t arow = (uint32_t)(16 * (warp >> 1) + (lane >> 2)) * 128u;
  const uint32_t brow = (uint32_t)(32 * (warp & 1) + (lane >> 2)) * 128u;
  for (int u = 0; u < nchunk; ++u) {
    if (tid == 0 && u + NSTAGE - 1 < nchunk) issue(u + NSTAGE - 1);
    const uint32_t q = pipe.seq + u;
    const int st = q % NSTAGE;
    bar_wait(&pipe.full[st], (q / NSTAGE) & 1);
    __syncwarp();
    const uint8_t* sa = stage + st * STAGE_BYTES;
    const uint8_t* sb = sa + BOX_BYTES;
    const uint8_t* sd = MODE == 2 ? sa + 2 * BOX_BYTES : sb;  // second A operand
#pragma unroll
    for (int k4 = 0; k4 < KC / 4; ++k4) {
      double a[2], ad[2], b[4];
#pragma unroll
      for (int rb = 0; rb < 2; ++rb) {
        a[rb] = -*reinterpret_cast<const double*>(sa + arow + rb * 8 * 128 + colofs[k4]);
        if (TWO) ad[rb] = -*reinterpret_cast<const double*>(sd + arow + rb * 8 * 128 + colofs[k4]);
      }
#pragma unroll
      for (int cb = 0; cb < 4; ++cb)
        b[cb] = *reinterpret_cast<const double*>(sb + brow + cb * 8 * 128 + colofs[k4]);
#pragma unroll
      for (int f = 0; f < 8; ++f) {
        dmma8x8x4(accA[f], a[f >> 2], b[f & 3]);
        if (TWO) dmma8x8x4(accB[f], ad[f >> 2], b[f & 3]);
      }
    }
    // the next TMA into this stage is an async-proxy write: the warp's
    // generic reads of the stage are ordered before it by the warp barrier
    // plus one proxy fence ahead of the release (without the fence the TMA
    // can overwrite a stage that is still being read -- observed on B200)
    __syncwarp();
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bar_arrive(&pipe.empty[st]);
    }
  }
  pipe.seq += nchunk;
}

__device__ __forceinline__ void acc_to_smem(double* X, const double (&acc)[8][2], int warp, int lane) {
#pragma unroll
  for (int f = 0; f < 8; ++f) {
    double* dst = X + (16 * (warp >> 1) + 8 * (f >> 2) + (lane >> 2)) * TS + 32 * (warp & 1) +
                  8 * (f & 3) + 2 * (lane & 3);
    dst[0] = acc[f][0];
    dst[1] = acc[f][1];
  }
}

// Every thread that stored part of the tile makes its generic-proxy writes
// visible to the async proxy (consumers read tiles with TMA), then thread 0
// releases the flag.
__device__ __forceinline__ void publish(const MatRT& P, int i, int j, int tid) {
  fence_proxy_async();
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    st_release(P.flags + (i * (i + 1) / 2 + j), P.epoch);
  }
}

// Later systems of the batch that do not recompute tile (i, j) hold the
// same tile bit for bit: store this system's copy (and, for a diagonal
// tile, its 8x8 inverses) into their buffers and publish it there.
__device__ void forward_tile(const CholParams& P, int b, int i, int j, const double* S,
                             const double* Dv, int tid) {
  for (int bb = b + 1; bb < P.nb; ++bb) {
    const CholMat& M2 = P.m[bb];
    if (tile_fresh(M2.full, M2.pnew, P.W, P.ell, i, j)) break;  // recomputed from here on
    store_tile(M2.L + tile_off(i, j), S, tid);
    if (Dv != nullptr) {
      const double2 v = *reinterpret_cast<const double2*>(Dv + 2 * tid);
      *reinterpret_cast<double2*>(M2.Dinv + (int64_t)j * 512 + 2 * tid) = v;
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release(M2.flags + (i * (i + 1) / 2 + j), M2.epoch);
    }
  }
}

// Task order (host-built map, see chol_task_map): per column, the PAIR task
// (diagonal (j, j) plus the first sub-diagonal (j + 1, j), so the critical
// TRSM reuses L_jj straight from shared memory) is placed right after the
// first off-diagonal tile of column j - 1 it depends on -- one column ahead
// of the bulk tiles.  Only the tiles a step recomputes are tasks; shared
// tiles arrive through forward_tile or k_assemble.  Every task's
// dependencies carry smaller tickets, so spinning on them cannot deadlock.
__global__ void __launch_bounds__(256, 2) k_chol_tiles(const __grid_constant__ CholParams P) {
  extern __shared__ __align__(16) uint8_t smem_raw[];  // 1024-aligned by hand below
  // 1024-byte alignment for the SW128 TMA boxes by pointer arithmetic on the
  // shared array (a round trip through an integer would make every fragment
  // load a generic LD instead of LDS)
  uint8_t* base = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stage = base + SMB_ST;
  double* Sg = reinterpret_cast<double*>(base + SMB_SG);
  double* Dv = reinterpret_cast<double*>(base + SMB_DV);
  double* rdiag = reinterpret_cast<double*>(base + SMB_RD);
  double* X = reinterpret_cast<double*>(stage);  // work tile, once the stages are drained
  __shared__ int s_task;
  __shared__ __align__(8) uint64_t s_full[NSTAGE], s_empty[NSTAGE];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    s_task = atomicAdd(P.ticket, 1);
    for (int q = 0; q < NSTAGE; ++q) {
      bar_init(&s_full[q], 1);
      bar_init(&s_empty[q], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (s_task >= P.ntasks) return;
  const int2 e = P.map[s_task];
  const CholMat& Mp = P.m[e.x];
  MatRT M;
  M.map = &Mp.map;
  M.L = Mp.L;
  M.Dinv = Mp.Dinv;
  M.flags = Mp.flags;
  M.N = Mp.N;
  M.T = Mp.T;
  M.epoch = Mp.epoch;
  M.alpha = Mp.alpha;
  if (tid == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(M.map) : "memory");
  __syncthreads();
  Pipe pipe{s_full, s_empty, 0u};
  const int i = e.y >> 16, j = e.y & 0x7fff;
  const bool dual = (e.y & 0x8000) != 0;  // off-diagonal rows i and i + 1 of column j
  const int T = M.T;
  unsigned long long* tr = (P.trace != nullptr && tid == 0) ? P.trace + 8 * (int64_t)s_task : nullptr;
  if (tr) tr[0] = globaltimer_ns();
  double accA[8][2], accB[8][2];

  if (i == j) {
    // ---------------- pair task: (j, j) and (j + 1, j) ----------------
    const bool has_sub = j + 1 < T;
    init_acc(P, M, j, j, warp, lane, accB);
    if (has_sub) {
      init_acc(P, M, j + 1, j, warp, lane, accA);
      accumulate<1>(M, j + 1, j, 0, j - 1 > 0 ? j - 1 : 0, stage, pipe, accA, accB, tid);
    }
    // last update of the diagonal alone, then factor it right away
    if (j >= 1) accumulate<0>(M, j, j, has_sub ? j - 1 : 0, j, stage, pipe, accB, accB, tid);
    if (tr) tr[1] = globaltimer_ns();
    acc_to_smem(Sg, accB, warp, lane);
    __syncthreads();
    potrf_tile_blocked(Sg, Dv, rdiag, tid, P.error);
    if (tr) tr[2] = globaltimer_ns();
    store_tile(M.L + tile_off(j, j), Sg, tid);
    {
      double2 v = *reinterpret_cast<const double2*>(Dv + 2 * tid);
      *reinterpret_cast<double2*>(M.Dinv + (int64_t)j * 512 + 2 * tid) = v;
    }
    publish(M, j, j, tid);
    if (has_sub) {
      if (j >= 1) accumulate<0>(M, j + 1, j, j - 1, j, stage, pipe, accA, accA, tid);
      __syncthreads();  // every warp is done reading the stages X overlays
      acc_to_smem(X, accA, warp, lane);
      __syncthreads();
      trsm_tile_warp(X, Sg, Dv, warp, lane);
      __syncthreads();
      store_tile(M.L + tile_off(j + 1, j), X, tid);
      publish(M, j + 1, j, tid);
      forward_tile(P, e.x, j + 1, j, X, nullptr, tid);
    }
    forward_tile(P, e.x, j, j, Sg, Dv, tid);
  } else if (dual) {
    // ---------------- off-diagonal tiles (i, j) and (i + 1, j) ----------
    double* X2 = X + TB * TS;  // second work tile, also over the drained stages
    init_acc(P, M, i, j, warp, lane, accA);
    init_acc(P, M, i + 1, j, warp, lane, accB);
    accumulate<2>(M, i, j, 0, j, stage, pipe, accA, accB, tid);
    if (tr) tr[1] = globaltimer_ns();
    if (tid == 0) wait_flag(M.flags + (j * (j + 1) / 2 + j), M.epoch);
    if (tr) tr[2] = globaltimer_ns();
    __syncthreads();
    load_tile_async(Sg, M.L + tile_off(j, j), tid);
    load_dinv_async(Dv, M.Dinv + (int64_t)j * 512, tid);
    cp_async_commit();
    acc_to_smem(X, accA, warp, lane);
    acc_to_smem(X2, accB, warp, lane);
    cp_async_wait_all();
    __syncthreads();
    trsm_tile_warp(X, Sg, Dv, warp, lane);
    trsm_tile_warp(X2, Sg, Dv, warp, lane);
    __syncthreads();
    store_tile(M.L + tile_off(i, j), X, tid);
    store_tile(M.L + tile_off(i + 1, j), X2, tid);
    publish(M, i, j, tid);
    if (tid == 0) st_release(M.flags + ((i + 1) * (i + 2) / 2 + j), M.epoch);  // fenced by publish
    forward_tile(P, e.x, i, j, X, nullptr, tid);
    forward_tile(P, e.x, i + 1, j, X2, nullptr, tid);
  } else {
    // ---------------- off-diagonal tile (i, j), i > j -----------------
    init_acc(P, M, i, j, warp, lane, accA);
    accumulate<0>(M, i, j, 0, j, stage, pipe, accA, accA, tid);
    if (tr) tr[1] = globaltimer_ns();
    if (tid == 0) wait_flag(M.flags + (j * (j + 1) / 2 + j), M.epoch);
    if (tr) tr[2] = globaltimer_ns();
    __syncthreads();
    load_tile_async(Sg, M.L + tile_off(j, j), tid);
    load_dinv_async(Dv, M.Dinv + (int64_t)j * 512, tid);
    cp_async_commit();
    acc_to_smem(X, accA, warp, lane);
    cp_async_wait_all();
    __syncthreads();
    trsm_tile_warp(X, Sg, Dv, warp, lane);
    __syncthreads();
    store_tile(M.L + tile_off(i, j), X, tid);
    publish(M, i, j, tid);
    forward_tile(P, e.x, i, j, X, nullptr, tid);
  }
  if (tr) tr[3] = globaltimer_ns();
}

// ===========================================================================
// Tile updates on the 5th-generation tensor cores (tcgen05 kind::i8).
//
// The left-looking update C = G_ij - sum_k L_ik L_jk^T dominates the
// factorization (all but O(T^2) of its flops).  tcgen05 has no fp64 kind, so
// the update is computed in integer arithmetic from digit slices: every
// entry of L row p is written with QD signed digits (kernels.h: SLIM_QD, 7 in
// this translation unit by default, 6 in chol_q6.cu), a 7-bit leading digit
// and balanced DBITS = 8-bit digits after it,
//     L_pk = 2^(e_p - 7) sum_{a=1..QD} d_a 2^(-8 (a-1)),
// d_1 in [-127, 127], d_a in [-128, 127] for a > 1, with 2^(e_p) >= 1.004
// sqrt(G_pp) >= 1.004 |L_pk| (row scales known before the factorization
// starts, k_assemble): 7 + 8 (QD - 1) bits below each row's scale.
// Then
//     sum_k L_ik L_jk = 2^(e_i + e_j - 14) sum_t 2^(-8 t) P_t,
//     P_t = sum_{a + b = t + 2} D_a(i) D_b(j)^T        (int32, exact)
// where the digit products with a + b <= QD + 1 + QX are kept (34 pairs for
// QD = 7, QX = 1; 21 for QD = 6, QX = 0, whose truncation the x-chain's
// refinement step removes).  The Cholesky backward-error bound
// is componentwise in sqrt(G_ii G_jj), so this row scaling is the natural one.
// Each P_t is one TMEM accumulator (M = 128 rows of two output tiles x N = 64;
// QACC = QD + QX of them, at most 8 x 64 = all 512 columns), the int32 sums
// are exact for T <= CHOL_I8_TMAX tile rows (checked at context creation), and
// the accumulators are combined in fp64 once per task.  POTRF, TRSM and the
// 8x8 inverses stay in fp64 (DMMA), on O(T^2) tiles.
//
// A sliced tile (QD x 4 KB) is stored by tile column in 64-byte rows,
// [k][digit][tile row][64 rows][64 B] (q_off, kernels.h), so a task's A operand
// (tile rows i, i + 1, all digits of one k tile) is one 3D TMA box under
// SWIZZLE_64B and its B operand (tile row j) another.
// ===========================================================================
#ifndef SLIM_ACC_SLEEP_NS
#define SLIM_ACC_SLEEP_NS 500  // 2000 -> 500: +0.4% at configs[1]
#endif
namespace oz {
constexpr int DIG_A = 128 * QROW;        // one digit of the A operand: 128 rows x QROW B
constexpr int DIG_B = 64 * QROW;         // one digit of B: 64 rows x QROW B
constexpr int ST_A = QD * DIG_A;         // [digit][rows of tiles i, i + 1][QROW B]
constexpr int ST_B = QD * DIG_B;         // [digit][64 rows][QROW B]
constexpr int STAGE = ST_A + ST_B;       // QROW / 32 k halves of three tiles
constexpr int KSTEPS = QROW / 32;        // K = 32 MMA steps per stage
#ifndef SLIM_OZ_NST
#define SLIM_OZ_NST (SLIM_OZ_SW == 64 ? 2 : 3)  // 2 x 84 KB or 3 x 42 KB in flight
#endif
#ifndef SLIM_OZ_HINT
#define SLIM_OZ_HINT 1  // L2 hints on the operand loads: +0.5% at configs[1]
#endif
// TMA stage ring depth (48 KB per stage): three stages (145 KB) leave a
// third of each SM's shared memory to the x-chain kernels running beside
// the factorization; measured +0.8% at configs[1] over four, equal at [2]
constexpr int NST = SLIM_OZ_NST;
constexpr int SMEM = NST * STAGE + 1024;
// work tiles over the drained stage ring
constexpr int W_X = 0;                               // 128 x TS fp64
constexpr int W_SG = W_X + 2 * TB * TS * 8;          // L_jj, 64 x TS fp64
constexpr int W_DV = W_SG + TB * TS * 8;             // 8x8 inverses (512)
constexpr int W_RD = W_DV + 512 * 8;                 // 64 reciprocal pivots
static_assert(W_RD + 64 * 8 <= NST * STAGE, "work tiles must fit over the stage ring");
// kind::i8, S32 accumulate, signed A and B, M = 128, N = 64 n
__host__ __device__ constexpr uint32_t idesc(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(8 * n) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// K-major swizzled operand: rows of QROW bytes, 8-row groups 8 QROW apart;
// layout type SWIZZLE_32B (6) or SWIZZLE_64B (4).  With 64-byte rows the
// second K = 32 step of a stage starts 32 bytes into the swizzle atom.
__device__ __forceinline__ uint64_t sw_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) |
         ((uint64_t)((8 * QROW) >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)(QROW == 32 ? 6 : 4) << 61);
}
// One MMA per (A digit a, run of up to four B digits b0 .. b0 + n - 1): the
// B digits are stacked along N (64 rows each), and D starts at accumulator
// t = a + b0 - 2, so the product with B digit b lands in TMEM column block
// a + b - 2 -- its own accumulator.  With the default seven digits that is
// 10 MMAs (N up to 256) per stage instead of 28 with N = 64 (which cap at 2/3
// of the tensor peak); the MMAs of one A digit share it through the A-operand
// collector.
// The digit-pair MMAs of one stage: A digit a times the run of B digits
// b0 .. b0 + n - 1 (n <= 4, stacked along N) into accumulators
// t = a + b0 - 2 .. + n - 1.  One MMA carries one overwrite flag, so on the
// first stage a run is split where it would reach both accumulators written
// by an earlier MMA and fresh ones (with QX = 1 that is the run of a = 2
// reaching t = QD, first written by (a = 2, b = QD)).  coll: the A-operand
// collector (0 none, 1 fill, 2 use, 3 lastuse) across the MMAs of one A digit.
struct MmaGroup {
  int a, b0, n, coll;
  bool first;  // overwrites its accumulators on the first stage
};
struct MmaTable {
  MmaGroup g[32];
  int count;
};
constexpr MmaTable make_groups() {
  MmaTable t{};
  bool written[8] = {};
  int cnt = 0;
  for (int a = 1; a <= QD; ++a) {
    const int nbd = q_nb(a);
    const int first = cnt;
    for (int b0 = 1; b0 <= nbd;) {
      int n = nbd + 1 - b0 < 4 ? nbd + 1 - b0 : 4;
      const int t0 = a + b0 - 2;
      for (int q = 1; q < n; ++q)
        if (written[t0 + q] != written[t0]) {
          n = q;
          break;
        }
      t.g[cnt] = MmaGroup{a, b0, n, 2, !written[t0]};
      for (int q = 0; q < n; ++q) written[t0 + q] = true;
      ++cnt;
      b0 += n;
    }
    if (cnt - first == 1) {
      t.g[first].coll = 0;
    } else {
      t.g[first].coll = 1;
      t.g[cnt - 1].coll = 3;
    }
  }
  t.count = cnt;
  return t;
}
constexpr int NMMA = make_groups().count;

template <int COLL>  // 0 plain, 1 fill, 2 use, 3 lastuse
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idsc,
                                       uint32_t acc) {
  if (COLL == 2)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::use [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
                 "l"(adesc), "l"(bdesc), "r"(idsc), "r"(acc) : "memory");
  else if (COLL == 1)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::fill [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
                 "l"(adesc), "l"(bdesc), "r"(idsc), "r"(acc) : "memory");
  else if (COLL == 3)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::lastuse [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
                 "l"(adesc), "l"(bdesc), "r"(idsc), "r"(acc) : "memory");
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
                 "l"(adesc), "l"(bdesc), "r"(idsc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ double pow2(int e) {  // exact 2^e, |e| < 1000
  return __longlong_as_double((long long)(e + 1023) << 52);
}
}  // namespace oz

// digit slices of the 64x64 fp64 tile X (smem, stride TS) with row
// exponents rex[0..63]: thread = (row, 16 consecutive k); v = L 2^(7 - e)
// lies in (-127.5, 127.5); the integer I = rint(v 2^(DBITS (QD - 1))) is cut
// into a 7-bit leading digit and QD - 1 balanced DBITS-bit digits
struct Digits {
  uint4 w[QD];  // digit a of the thread's 16 entries, one byte each
};
__device__ __forceinline__ void slice_tile(const double* X, const int* rex, int tid, Digits& D) {
  const int r = tid >> 2, kq = tid & 3;
  // I = rint(L 2^(7 QD - e)) = rint(v 2^(7 (QD - 1))): |I| < 127.5 2^(7 (QD - 1)),
  // exact in fp64 and int64; balanced base-128 digits peeled off from the
  // bottom in integer arithmetic, the remaining top digit in [-127, 127]
  // (DBITS = 8: base-256 digits in [-128, 127], same argument)
  const double sc = oz::pow2(7 + DBITS * (QD - 1) - __ldcg(rex + r));
  uint32_t w[QD][4];
#pragma unroll
  for (int a = 0; a < QD; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q) w[a][q] = 0u;
#pragma unroll
  for (int cc = 0; cc < 16; ++cc) {
    long long I = __double2ll_rn(X[r * TS + 16 * kq + cc] * sc);
#pragma unroll
    for (int a = QD - 1; a >= 1; --a) {
      constexpr int H = 1 << (DBITS - 1);
      const int d = (((int)I + H) & (2 * H - 1)) - H;
      I = (I - d) >> DBITS;
      w[a][cc >> 2] |= ((uint32_t)d & 0xffu) << (8 * (cc & 3));
    }
    w[0][cc >> 2] |= ((uint32_t)(int)I & 0xffu) << (8 * (cc & 3));
  }
#pragma unroll
  for (int a = 0; a < QD; ++a) D.w[a] = make_uint4(w[a][0], w[a][1], w[a][2], w[a][3]);
}
// digit a of the thread's 16 entries (row r, k = 16 kq ..) into sliced tile (i, k)
__device__ __forceinline__ void store_digits(const CholMat& M, int i, int k, const Digits& D, int tid) {
  const int r = tid >> 2, kq = tid & 3, kh = kq >> 1, kk0 = (kq & 1) * 16;
#pragma unroll
  for (int a = 0; a < QD; ++a)
    *reinterpret_cast<uint4*>(M.Q + q_off(M.qT, i, k, kh, a, r) + kk0) = D.w[a];
}

// Store tile (i, j) -- fp64, digit slices (off-diagonal tiles: the only
// update operands) and, for a diagonal tile, its 8x8 inverses -- into system
// b and every later system of the batch that shares it bit for bit, then
// publish all copies behind one fence.
__device__ void store_publish_i8(const CholParams& P, int b, int i, int j, const double* X,
                                 const double* Dv, int tid, unsigned long long* tr = nullptr) {
  Digits D;
  const unsigned long long s0 = tr ? globaltimer_ns() : 0;
  if (i != j) slice_tile(X, P.m[b].rexp + i * TB, tid, D);
  if (tr) tr[6] += globaltimer_ns() - s0;
  const unsigned long long s1 = tr ? globaltimer_ns() : 0;
  int last = b;
  for (int bb = b; bb < P.nb; ++bb) {
    const CholMat& M2 = P.m[bb];
    if (bb > b && tile_fresh(M2.full, M2.pnew, P.W, P.ell, i, j)) break;  // recomputed from here on
    last = bb;
    store_tile(M2.L + tile_off(i, j), X, tid);
    if (i != j) store_digits(M2, i, j, D, tid);
    if (Dv != nullptr) {
      const double2 v = *reinterpret_cast<const double2*>(Dv + 2 * tid);
      *reinterpret_cast<double2*>(M2.Dinv + (int64_t)j * 512 + 2 * tid) = v;
    }
  }
  fence_proxy_async();  // consumers read the slices with TMA (async proxy)
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    for (int bb = b; bb <= last; ++bb) st_release(P.m[bb].flags + (i * (i + 1) / 2 + j), P.m[bb].epoch);
  }
  if (tr) tr[7] += globaltimer_ns() - s1;
}

// One task per CTA (same ticket map as k_chol_tiles): output rows ra (and
// ra + 1 for pair / dual tasks) of tile column j.  Warp 0 lane 0 streams the
// digit slices of L_(ra, k), L_(ra+1, k), L_(j, k) for k < j through an
// NST-stage TMA ring (one k tile per stage: 2 x 84 KB with seven digits, 3 x 72 KB
// with six); warp 1 lane 0 issues the stage's digit-pair MMAs (make_groups) into
// the QACC TMEM accumulators; then all eight warps combine the accumulators
// with G in fp64 and finish the tiles (POTRF / TRSM, DMMA).
__global__ void __launch_bounds__(256, 1) k_chol_i8(const __grid_constant__ CholParams P) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stage = base;
  double* X = reinterpret_cast<double*>(base + oz::W_X);
  double* X2 = X + TB * TS;
  double* Sg = reinterpret_cast<double*>(base + oz::W_SG);
  double* Dv = reinterpret_cast<double*>(base + oz::W_DV);
  double* rdiag = reinterpret_cast<double*>(base + oz::W_RD);
  __shared__ int s_task;
  __shared__ uint32_t s_tmem;
  __shared__ int s_ecol[TB];
  __shared__ __align__(8) uint64_t s_full[oz::NST], s_empty[oz::NST], s_accf;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    s_task = atomicAdd(P.ticket, 1);
    for (int q = 0; q < oz::NST; ++q) {
      bar_init(&s_full[q], 1);
      bar_init(&s_empty[q], 1);
    }
    bar_init(&s_accf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (s_task >= P.ntasks) return;
  const int2 e = P.map[s_task];
  const CholMat& M = P.m[e.x];
  const int i = e.y >> 16, j = e.y & 0x7fff;
  const bool pair = i == j;
  const int T = M.T;
  const bool two = pair ? (j + 1 < T) : ((e.y & 0x8000) != 0);
  const int ra = i;  // first output row tile (the diagonal for a pair task)
  unsigned long long* tr = (P.trace != nullptr && tid == 0) ? P.trace + 8 * (int64_t)s_task : nullptr;
  if (tr) tr[0] = globaltimer_ns();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        su32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid < TB) s_ecol[tid] = __ldcg(M.rexp + j * TB + tid);
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&M.qmapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&M.qmapB) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  const int nchunk = oz::KSTEPS == 2 ? j : 2 * j;  // stages: k tiles 0 .. j-1 (or their halves)

  if (tid == 0 && nchunk > 0) {
    // ---------------- TMA producer ----------------
    const int* fa = M.flags + ra * (ra + 1) / 2;
    const int* fa2 = M.flags + (ra + 1) * (ra + 2) / 2;
    const int* fb = M.flags + j * (j + 1) / 2;
    int kready = j;
    for (int k = 0; k < j; ++k) {
      int va, vb = M.epoch, vc = M.epoch;
      asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(va) : "l"(fa + k) : "memory");
      if (two) asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(vb) : "l"(fa2 + k) : "memory");
      if (!pair) asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(vc) : "l"(fb + k) : "memory");
      if (va < M.epoch || vb < M.epoch || vc < M.epoch) {
        kready = k;
        break;
      }
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    fence_proxy_async();
    unsigned long long t_dep = 0, t_ring = 0;  // trace: producer stall time
    for (int u = 0; u < nchunk; ++u) {
      const int st = u % oz::NST;
      const unsigned long long w0 = tr ? globaltimer_ns() : 0;
      bar_wait(&s_empty[st], ((u / oz::NST) & 1) ^ 1);
      const unsigned long long w1 = tr ? globaltimer_ns() : 0;
      t_ring += w1 - w0;
      const int k = oz::KSTEPS == 2 ? u : (u >> 1), kh = oz::KSTEPS == 2 ? 0 : (u & 1);
      if (kh == 0 && k >= kready) {
        wait_flag(fa + k, M.epoch);
        if (two) wait_flag(fa2 + k, M.epoch);
        if (!pair) wait_flag(fb + k, M.epoch);
        fence_proxy_async();
        if (tr) t_dep += globaltimer_ns() - w1;
      }
      uint8_t* dst = stage + st * oz::STAGE;
      bar_expect(&s_full[st], oz::STAGE);
      const int zc = oz::KSTEPS == 2 ? k * QD : (k * 2 + kh) * QD;  // first digit block of the stage
      // A: tile rows ra, ra + 1, all QD digits (a single task's spare row is
      // loaded and ignored); B: tile row j
#if SLIM_OZ_HINT
      // A (this task's row pair) is streamed once; B (row j) is shared by
      // every task of the column
      tma3d_hint(dst, &M.qmapA, &s_full[st], 0, ra * TB, zc, L2_EVICT_FIRST);
      tma3d_hint(dst + oz::ST_A, &M.qmapB, &s_full[st], 0, j * TB, zc, L2_EVICT_LAST);
#else
      tma3d(dst, &M.qmapA, &s_full[st], 0, ra * TB, zc);
      tma3d(dst + oz::ST_A, &M.qmapB, &s_full[st], 0, j * TB, zc);
#endif
    }
    if (tr) tr[4] = t_dep;
    (void)t_ring;
  } else if (warp == 1 && lane == 0 && nchunk > 0) {
    // ---------------- MMA issuer ----------------
    unsigned long long* trm = P.trace != nullptr ? P.trace + 8 * (int64_t)s_task : nullptr;
    unsigned long long t_data = 0;  // trace: waiting for operand stages
    for (int u = 0; u < nchunk; ++u) {
      const int st = u % oz::NST;
      const unsigned long long w0 = trm ? globaltimer_ns() : 0;
      bar_wait(&s_full[st], (u / oz::NST) & 1);
      if (trm) t_data += globaltimer_ns() - w0;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a0 = su32(stage + st * oz::STAGE);
#pragma unroll
      for (int ks = 0; ks < oz::KSTEPS; ++ks) {
      const uint64_t ad = oz::sw_desc(a0 + 32 * ks), bd = oz::sw_desc(a0 + oz::ST_A + 32 * ks);
      // accumulators are first touched by the a = 1 MMAs: only they may
      // overwrite (first stage)
      constexpr oz::MmaTable groups = oz::make_groups();
#pragma unroll
      for (int g = 0; g < oz::NMMA; ++g) {
        const oz::MmaGroup m = groups.g[g];
        const uint64_t A = ad + (((m.a - 1) * oz::DIG_A) >> 4);
        const uint64_t B = bd + (((m.b0 - 1) * oz::DIG_B) >> 4);
        const uint32_t acc = (u > 0 || ks > 0 || !m.first) ? 1u : 0u;
        const uint32_t d = tmem + 64 * (m.a + m.b0 - 2);
        if (m.coll == 0)
          oz::mma_i8<0>(d, A, B, oz::idesc(m.n), acc);
        else if (m.coll == 1)
          oz::mma_i8<1>(d, A, B, oz::idesc(m.n), acc);
        else if (m.coll == 2)
          oz::mma_i8<2>(d, A, B, oz::idesc(m.n), acc);
        else
          oz::mma_i8<3>(d, A, B, oz::idesc(m.n), acc);
      }
      }  // K steps of the stage
      oz::mma_commit(&s_empty[st]);
    }
    oz::mma_commit(&s_accf);
    if (trm) trm[5] = t_data;
  }
  __syncwarp();

  // ------- combine: X = G - 2^(e_r + e_c - 14) sum_t 2^(-DBITS t) P_t -------
  {
    if (nchunk > 0) {
      // idle warps poll with back-off: a tight try_wait loop of 250 threads
      // competes with the tensor core for shared-memory bandwidth
      const uint32_t a = su32(&s_accf);
      uint32_t done = 0;
      while (true) {
        asm volatile("{\n.reg .pred P1;\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], 0;\n"
                     "selp.u32 %0, 1, 0, P1;\n}\n"
                     : "=r"(done)
                     : "r"(a)
                     : "memory");
        if (done) break;
        __nanosleep(SLIM_ACC_SLEEP_NS);
      }
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp & 3, h = warp >> 2;
    const int R = 32 * q + lane, sel = R >> 6, r = R & 63;
    double s[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) s[c] = 0.0;
    if (nchunk > 0) {
#pragma unroll 1
      for (int t = QACC - 1; t >= 0; --t) {
        int v[32];
        oz::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + 64 * t + 32 * h, v);
#pragma unroll
        for (int c = 0; c < 32; ++c) s[c] = fma(s[c], 1.0 / (1 << DBITS), (double)v[c]);
      }
    }
    if (sel == 0 || two) {
      const int er = __ldcg(M.rexp + (ra + sel) * TB + r);
      const double* g = M.L + tile_off(ra + sel, j) + r * TB + 32 * h;
      double* x = X + R * TS + 32 * h;
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        const double2 gv = __ldcg(reinterpret_cast<const double2*>(g + c));
        x[c] = gv.x - s[c] * oz::pow2(er + s_ecol[32 * h + c] - 14);
        x[c + 1] = gv.y - s[c + 1] * oz::pow2(er + s_ecol[32 * h + c + 1] - 14);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  if (tr) tr[1] = globaltimer_ns();

  if (pair) {
    potrf_tile_blocked(X, Dv, rdiag, tid, P.error);
    if (tr) tr[2] = globaltimer_ns();
    store_publish_i8(P, e.x, j, j, X, Dv, tid, tr);
    if (two) {
      trsm_tile_warp(X2, X, Dv, warp, lane);
      __syncthreads();
      store_publish_i8(P, e.x, j + 1, j, X2, nullptr, tid, tr);
    }
  } else {
    if (tid == 0) wait_flag(M.flags + (j * (j + 1) / 2 + j), M.epoch);
    __syncthreads();
    load_tile_async(Sg, M.L + tile_off(j, j), tid);
    load_dinv_async(Dv, M.Dinv + (int64_t)j * 512, tid);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    if (two)
      trsm_tile_warp2(X, X2, Sg, Dv, warp, lane);
    else
      trsm_tile_warp(X, Sg, Dv, warp, lane);
    __syncthreads();
    if (tr) tr[2] = globaltimer_ns();  // wait + L_jj load + TRSM
    store_publish_i8(P, e.x, ra, j, X, nullptr, tid, tr);
    if (two) store_publish_i8(P, e.x, ra + 1, j, X2, nullptr, tid, tr);
  }
  if (tr) tr[3] = globaltimer_ns();
}

bool chol_use_i8() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SLIM_CHOL");
    v = (e != nullptr && std::string(e) == "dmma") ? 0 : 1;
  }
  return v == 1;
}

bool chol_i8_for(int T) { return chol_use_i8() && T <= CHOL_I8_TMAX; }

size_t chol_smem_bytes() { return chol_use_i8() ? (size_t)oz::SMEM : (size_t)SMB_TOTAL; }

// Ticket order.  A system's tasks are its fresh tiles (tile_fresh), grouped
// by column: pair(0) opens group -1; group j holds, in this order, the
// stand-alone (j + 1, j) (column j not fresh but that row is), the first
// off-diagonal tile (j + 2, j), the pair of column j + 1 (one column ahead
// of the bulk, so the critical diagonal chain is never queued behind it) and
// the rest of column j, consecutive fresh rows paired into dual tasks.
// Encoded as (i << 16) | j with i == j for pair tasks; bit 15 of the low half
// marks a dual task (rows i and i + 1).
// The batch is merged group-major, system-minor: a tile a system shares
// with an earlier system of the batch is produced by that system's task in
// the same or an earlier group, so every dependency holds a smaller ticket
// and spinning on it cannot deadlock.
// Banded order (cols = C >= 2): the columns are taken C at a time.  Each
// group first emits, column by column and system-minor, the tasks whose
// rows reach no further than J + C + 1 (the diagonal chain: stand-alone,
// first off-diagonal and pair tasks, as above); then the rest of the C
// columns in bands of `band` tile rows, each band system by system, rows
// ascending and, for one row pair, the C columns back to back.  Dual tasks
// pair rows (i, i + 1) with i EVEN in every column, so the tasks of one row
// pair in consecutive columns stream the same A panel (tile rows i, i + 1,
// k = 0 ..) at the same time: the second read hits L2 instead of DRAM.  A
// task whose first row is in the group's diagonal block goes to the head;
// the others are keyed by their aligned row pair (last row | 1), so every
// dependency (rows of the same or an earlier row pair in earlier columns,
// the diagonal chain) holds a smaller ticket and spinning on it cannot
// deadlock (checked for the configuration shapes by tools/taskmap_check.cu).
static std::vector<int2> chol_task_map_banded(const SysShape* sh, int nb, int W, int ell, int C,
                                              int band) {
  int Tmax = 0;
  for (int b = 0; b < nb; ++b) Tmax = std::max(Tmax, sh[b].T);
  auto fresh = [&](int b, int i, int j) { return tile_fresh(sh[b].full, sh[b].pnew, W, ell, i, j); };
  struct Task {
    int first, last, code;
  };
  // tasks of column j of system b, in the diagonal-chain order of chol_task_map
  auto column = [&](int b, int j, std::vector<Task>& out) {
    out.clear();
    const int T = sh[b].T;
    if (j >= T) return;
    if (!fresh(b, j, j) && j + 1 < T && fresh(b, j + 1, j))
      out.push_back({j + 1, j + 1, ((j + 1) << 16) | j});
    if (j + 2 < T && fresh(b, j + 2, j)) out.push_back({j + 2, j + 2, ((j + 2) << 16) | j});
    if (j + 1 < T && fresh(b, j + 1, j + 1))
      out.push_back({j + 1, std::min(j + 2, T - 1), ((j + 1) << 16) | (j + 1)});
    for (int i = j + 3; i < T; ++i) {
      if (!fresh(b, i, j)) continue;
      if ((i & 1) == 0 && i + 1 < T && fresh(b, i + 1, j)) {
        out.push_back({i, i + 1, (i << 16) | 0x8000 | j});
        ++i;
      } else {
        out.push_back({i, i, (i << 16) | j});
      }
    }
  };
  std::vector<int2> out;
  for (int b = 0; b < nb; ++b)
    if (fresh(b, 0, 0)) out.push_back(make_int2(b, 0));
  std::vector<Task> col;
  struct Body {
    int b, last, c, code;
  };
  std::vector<Body> body;
  for (int J = 0; J < Tmax; J += C) {
    const int Jend = std::min(J + C, Tmax), head = J + C + 1;
    body.clear();
    for (int c = J; c < Jend; ++c)
      for (int b = 0; b < nb; ++b) {
        column(b, c, col);
        for (const Task& t : col) {
          if (t.first <= head) out.push_back(make_int2(b, t.code));
          else body.push_back({b, t.last | 1, c, t.code});  // keyed by its aligned row pair
        }
      }
    // bands of `band` rows after the head; inside a band: system, row pair, column
    std::stable_sort(body.begin(), body.end(), [&](const Body& x, const Body& y) {
      const int bx = (x.last - head - 1) / band, by = (y.last - head - 1) / band;
      if (bx != by) return bx < by;
      if (x.b != y.b) return x.b < y.b;
      if (x.last != y.last) return x.last < y.last;
      return x.c < y.c;
    });
    for (const Body& t : body) out.push_back(make_int2(t.b, t.code));
  }
  return out;
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

std::vector<int2> chol_task_map(const SysShape* sh, int nb, int W, int ell, int cols, int band) {
  if (cols < 0) cols = env_int("SLIM_CHOL_COLS", CHOL_COLS_DEFAULT);
  if (band < 0) band = env_int("SLIM_CHOL_BAND", CHOL_BAND_DEFAULT);
  if (cols >= 2) return chol_task_map_banded(sh, nb, W, ell, cols, std::max(2, band));
  int Tmax = 0;
  for (int b = 0; b < nb; ++b) Tmax = std::max(Tmax, sh[b].T);
  std::vector<int2> out;
  auto fresh = [&](int b, int i, int j) {
    return tile_fresh(sh[b].full, sh[b].pnew, W, ell, i, j);
  };
  for (int g = -1; g < Tmax; ++g) {
    for (int b = 0; b < nb; ++b) {
      const int T = sh[b].T;
      if (g >= T) continue;
      if (g < 0) {
        if (fresh(b, 0, 0)) out.push_back(make_int2(b, 0));
        continue;
      }
      const int j = g;
      const bool col_fresh = fresh(b, j, j);  // the whole column then is
      if (!col_fresh && j + 1 < T && fresh(b, j + 1, j)) out.push_back(make_int2(b, ((j + 1) << 16) | j));
      if (j + 2 < T && fresh(b, j + 2, j)) out.push_back(make_int2(b, ((j + 2) << 16) | j));
      if (j + 1 < T && fresh(b, j + 1, j + 1)) out.push_back(make_int2(b, ((j + 1) << 16) | (j + 1)));
      // the rest of column j, fresh rows in consecutive pairs (dual tasks)
      for (int i = j + 3; i < T; ++i) {
        if (!fresh(b, i, j)) continue;
        if (i + 1 < T && fresh(b, i + 1, j)) {
          out.push_back(make_int2(b, (i << 16) | 0x8000 | j));
          ++i;
        } else {
          out.push_back(make_int2(b, (i << 16) | j));
        }
      }
    }
  }
  return out;
}

void launch_assemble(const CholParams& P, cudaStream_t s) {
  k_assemble<<<P.tile_base[P.nb], 256, 0, s>>>(P);
}

void launch_chol(const CholParams& P, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_chol_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMB_TOTAL);
    cudaFuncSetAttribute(k_chol_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)oz::SMEM);
    configured = true;
  }
  if (P.i8)
    k_chol_i8<<<P.ntasks, 256, oz::SMEM, s>>>(P);
  else
    k_chol_tiles<<<P.ntasks, 256, SMB_TOTAL, s>>>(P);
}

static size_t table_q_bytes(int qT) { return q_bytes(qT); }
extern const CholVariant chol_table = {QD,           QX,      DBITS, QPAIRS, CHOL_I8_TMAX, &table_q_bytes,
                                       &launch_assemble, &launch_chol};

#ifdef SLIM_CHOL_VARIANT
}  // namespace SLIM_CHOL_VARIANT
#endif
}  // namespace slim
