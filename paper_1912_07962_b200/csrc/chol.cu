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
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace slim {

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
  if (!tile_fresh(Mp.full, Mp.pnew, P.W, ell, I, J)) {
    for (int bb = b - 1; bb >= 0; --bb)
      if (tile_fresh(P.m[bb].full, P.m[bb].pnew, P.W, ell, I, J)) return;  // produced in-batch
    const double2* src = reinterpret_cast<const double2*>(P.prevL + toff);
    double2* dst = reinterpret_cast<double2*>(Mp.L + toff);
    for (int e = tid; e < TB * TB / 2; e += 256) dst[e] = __ldcg(src + e);
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
  unsigned long long* tr = (P.trace != nullptr && tid == 0) ? P.trace + 4 * (int64_t)s_task : nullptr;
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

size_t chol_smem_bytes() { return (size_t)SMB_TOTAL; }

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
std::vector<int2> chol_task_map(const SysShape* sh, int nb, int W, int ell) {
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
    cudaFuncSetAttribute(k_chol_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)chol_smem_bytes());
    configured = true;
  }
  k_chol_tiles<<<P.ntasks, 256, chol_smem_bytes(), s>>>(P);
}

}  // namespace slim
