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
#include "common.cuh"
#include "kernels.h"

namespace slim {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double chol_g_elem(const CholParams& P, int p, int q) {
  // requires q <= p < N
  if (P.panels != nullptr) {
    const int pb = p / P.ell, a = p - pb * P.ell;
    const int qb = q / P.ell, c = q - qb * P.ell;
    // product A_P[a] . A_Q[c] was stored when block P (the newer) was pushed:
    // panel[slot(P)] row (slot(Q) * ell + c), column a
    const double* pan = P.panels + (int64_t)P.slot[pb] * P.panel_stride;
    const double v = pan[((int64_t)P.slot[qb] * P.ell + c) * P.ell + a];
    return P.alpha * v + (p == q ? 1.0 : 0.0);
  }
  return P.G[(int64_t)p * P.ldg + q];
}

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

// ---------------------------------------------------------------------------
// POTRF of the 64x64 tile in S (lower part valid), plus the inverses of its
// eight 8x8 diagonal blocks into Dv[q * 64 + i * 8 + k] (lower, row-major).
// ---------------------------------------------------------------------------
__device__ void potrf_tile_blocked(double* S, double* Dv, int tid, int* error) {
  const int warp = tid >> 5, lane = tid & 31;
  for (int p = 0; p < 8; ++p) {
    const int c0 = 8 * p;
    if (warp == 0) {
      // panel rows c0 .. 63: lane owns rows r0 = c0 + lane, r1 = r0 + 32
      const int r0 = c0 + lane, r1 = r0 + 32;
      double v0[8], v1[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        v0[c] = (r0 < TB) ? S[r0 * TS + c0 + c] : 0.0;
        v1[c] = (r1 < TB) ? S[r1 * TS + c0 + c] : 0.0;
      }
      bool bad = false;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double d = __shfl_sync(FULL, v0[c], c);
        bad |= !(d > 0.0);
        const double inv = rsqrt(d);
        v0[c] = (lane > c) ? v0[c] * inv : ((lane == c) ? d * inv : 0.0);
        v1[c] = v1[c] * inv;
#pragma unroll
        for (int j = c + 1; j < 8; ++j) {
          const double ljc = __shfl_sync(FULL, v0[c], j);
          v0[j] -= v0[c] * ljc;
          v1[j] -= v1[c] * ljc;
        }
      }
      if (lane == 0 && bad) atomicExch(error, 1);
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
    for (int e = warp; e < nblk; e += 8) {
      int bi = p + 1, rem = e;
      while (rem > bi - (p + 1)) {
        rem -= bi - p;
        ++bi;
      }
      const int bj = p + 1 + rem;
      double* cp = S + (8 * bi + (lane >> 2)) * TS + 8 * bj + 2 * (lane & 3);
      double acc[2] = {cp[0], cp[1]};
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const double a = -S[(8 * bi + (lane >> 2)) * TS + c0 + 4 * ks + (lane & 3)];
        const double b = S[(8 * bj + (lane >> 2)) * TS + c0 + 4 * ks + (lane & 3)];
        dmma8x8x4(acc, a, b);
      }
      cp[0] = acc[0];
      cp[1] = acc[1];
    }
    __syncthreads();
  }
  // zero the strict upper triangle outside the (already clean) panel writes
  for (int e = tid; e < TB * TB; e += 256) {
    const int r = e >> 6, c = e & 63;
    if (c > r) S[r * TS + c] = 0.0;
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
      x[i] = s / L[i * TS + i];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) Dv[q * 64 + i * 8 + c] = x[i];
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// X L^T = C (X, C: 64x64 in As; L = L_jj in Bs; Dv = inverses of its 8x8
// diagonal blocks).  Warp w owns rows 8w..8w+7 and never waits on another
// warp: column block q is  X_q = (C_q - sum_{p<q} X_p L_qp^T) Dinv_q^T.
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

__global__ void __launch_bounds__(256, 3) k_chol_tiles(CholParams P) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + TB * TS;
  double* Dv = Bs + TB * TS;  // 512 doubles
  __shared__ int s_task;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_task = atomicAdd(P.ticket, 1);
  __syncthreads();
  int rem = s_task;
  const int T = P.T;
  if (rem >= T * (T + 1) / 2) return;
  int j = 0;
  while (rem >= T - j) {
    rem -= T - j;
    ++j;
  }
  const int i = j + rem;

  // ---- fused assembly: C = alpha * Gram + I (lower), identity padding ----
  double acc[8][2];
  const int p = i * TB + warp * 8 + (lane >> 2);
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int q = j * TB + nt * 8 + 2 * (lane & 3) + e;
      double v;
      if (p >= P.N || q >= P.N) v = (p == q) ? 1.0 : 0.0;
      else if (q > p) v = 0.0;
      else v = chol_g_elem(P, p, q);
      acc[nt][e] = v;
    }
  }

  // ---- left-looking update over the finished tiles of columns k < j ----
  const int arow = (warp * 8 + (lane >> 2)) * TS + (lane & 3);
  for (int k = 0; k < j; ++k) {
    if (tid == 0) {
      wait_flag(P.flags + (i * (i + 1) / 2 + k), P.epoch);
      wait_flag(P.flags + (j * (j + 1) / 2 + k), P.epoch);
    }
    __syncthreads();
    load_tile_async(As, P.L + tile_off(i, k), tid);
    load_tile_async(Bs, P.L + tile_off(j, k), tid);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
#pragma unroll 4
    for (int k4 = 0; k4 < TB / 4; ++k4) {
      const double a = -As[arow + 4 * k4];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const double b = Bs[(nt * 8 + (lane >> 2)) * TS + 4 * k4 + (lane & 3)];
        dmma8x8x4(acc[nt], a, b);
      }
    }
    __syncthreads();
  }

  // ---- finalize: POTRF on the diagonal, TRSM against L_jj below it ----
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    As[(warp * 8 + (lane >> 2)) * TS + nt * 8 + 2 * (lane & 3)] = acc[nt][0];
    As[(warp * 8 + (lane >> 2)) * TS + nt * 8 + 2 * (lane & 3) + 1] = acc[nt][1];
  }
  if (i == j) {
    __syncthreads();
    potrf_tile_blocked(As, Dv, tid, P.error);
    // publish the small inverses with the tile
    if (tid < 256) {
      double2 v = *reinterpret_cast<const double2*>(Dv + 2 * tid);
      *reinterpret_cast<double2*>(P.Dinv + (int64_t)j * 512 + 2 * tid) = v;
    }
  } else {
    if (tid == 0) wait_flag(P.flags + (j * (j + 1) / 2 + j), P.epoch);
    __syncthreads();
    load_tile_async(Bs, P.L + tile_off(j, j), tid);
    load_dinv_async(Dv, P.Dinv + (int64_t)j * 512, tid);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    trsm_tile_warp(As, Bs, Dv, warp, lane);
    __syncthreads();
  }
  store_tile(P.L + tile_off(i, j), As, tid);
  __threadfence();
  __syncthreads();
  if (tid == 0) st_release(P.flags + (i * (i + 1) / 2 + j), P.epoch);
}

// ---------------------------------------------------------------------------
// Triangular solves  t = L^{-1} y  (y zero above row N - ell),  w = L^{-T} t.
// One launch; tickets 0..nf-1 run the forward tile rows i0..T-1 in order,
// the rest run the backward tile rows T-1..0.  Every tile the task needs is
// already final (the factorization finished before this launch), so it is
// prefetched into shared memory while the task waits for the solved
// segment it multiplies; the critical path per tile row is one flag hop,
// one 64x64 product from shared memory and the blocked diagonal solve.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void load_vec_cg(double* s, const double* g, int tid) {
  if (tid < TB) s[tid] = __ldcg(g + tid);
}

// forward diagonal solve in place: v <- L_ii^{-1} v (blocked by 8)
__device__ void diag_solve_fwd(double* v, const double* Ld, const double* Dv, double* u, int tid) {
  const int warp = tid >> 5, lane = tid & 31;
  for (int q = 0; q < 8; ++q) {
    // warp i computes u_i = v[8q+i] - sum_{k < 8q} L[8q+i][k] v[k]
    const int row = 8 * q + warp;
    double s = 0.0;
    for (int k = lane; k < 8 * q; k += 32) s += Ld[row * TS + k] * v[k];
    s = warp_sum(s);
    if (lane == 0) u[warp] = v[row] - s;
    __syncthreads();
    if (tid < 8) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) t += Dv[q * 64 + tid * 8 + k] * u[k];
      v[8 * q + tid] = t;
    }
    __syncthreads();
  }
}

// backward diagonal solve in place: v <- L_ii^{-T} v
__device__ void diag_solve_bwd(double* v, const double* Ld, const double* Dv, double* u, int tid) {
  const int warp = tid >> 5, lane = tid & 31;
  for (int q = 7; q >= 0; --q) {
    const int col = 8 * q + warp;
    double s = 0.0;
    for (int k = 8 * q + 8 + lane; k < TB; k += 32) s += Ld[k * TS + col] * v[k];
    s = warp_sum(s);
    if (lane == 0) u[warp] = v[col] - s;
    __syncthreads();
    if (tid < 8) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) t += Dv[q * 64 + k * 8 + tid] * u[k];
      v[8 * q + tid] = t;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256, 2) k_trsv(TrsvParams P) {
  extern __shared__ __align__(16) double smem[];
  double* Ld = smem;                   // diagonal tile
  double* Lb0 = Ld + TB * TS;          // off-diagonal tile, double-buffered
  double* Lb1 = Lb0 + TB * TS;
  double* Dv = Lb1 + TB * TS;          // 512
  double* vec = Dv + 512;              // 64 accumulator
  double* tv = vec + TB;               // 64 incoming segment
  double* part = tv + TB;              // 4 x 64 partial sums
  double* u = part + 4 * TB;           // 8 scratch
  __shared__ int s_task;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (P.ctl != nullptr && P.ctl->diverged_at != 0) return;
  if (tid == 0) s_task = atomicAdd(P.ticket, 1);
  __syncthreads();
  const int T = P.T, i0 = P.i0, nf = T - i0;
  const int t = s_task;
  if (t >= nf + T) return;
  const bool fwd = t < nf;
  const int i = fwd ? i0 + t : T - 1 - (t - nf);
  int* fflag = P.flags;
  int* bflag = P.flags + T;

  // prefetch the diagonal tile and its small inverses (group 0)
  load_tile_async(Ld, P.L + tile_off(i, i), tid);
  load_dinv_async(Dv, P.Dinv + (int64_t)i * 512, tid);
  cp_async_commit();
  // the contributing tiles, in the order their solved segments arrive
  const int jfirst = fwd ? i0 : T - 1;
  const int jcount = fwd ? (i - i0) : (T - 1 - i);
  auto tile_of = [&](int jj) { return fwd ? tile_off(i, jj) : tile_off(jj, i); };
  if (jcount > 0) load_tile_async(Lb0, P.L + tile_of(jfirst), tid);
  cp_async_commit();

  if (fwd) {
    if (tid < TB) {
      const int pr = i * TB + tid;
      vec[tid] = (pr >= P.rstart && pr < P.N) ? P.r[pr - P.rstart] : 0.0;
    }
  } else {
    if (i >= i0) {
      if (tid == 0) wait_flag(fflag + i, P.epoch);
      __syncthreads();
      load_vec_cg(vec, P.t + (int64_t)i * TB, tid);
    } else if (tid < TB) {
      vec[tid] = 0.0;
    }
  }
  for (int s = 0; s < jcount; ++s) {
    const int jj = fwd ? jfirst + s : jfirst - s;
    double* cur = (s & 1) ? Lb1 : Lb0;
    double* nxt = (s & 1) ? Lb0 : Lb1;
    if (s + 1 < jcount) {
      const int jn = fwd ? jj + 1 : jj - 1;
      load_tile_async(nxt, P.L + tile_of(jn), tid);
    }
    cp_async_commit();
    if (tid == 0) wait_flag((fwd ? fflag : bflag) + jj, P.epoch);
    __syncthreads();
    load_vec_cg(tv, (fwd ? P.t : P.w) + (int64_t)jj * TB, tid);
    cp_async_wait_1();  // everything but the newest prefetch has landed
    __syncthreads();
    if (fwd) {
      // vec[a] -= sum_b L_ij[a][b] t_j[b]; warp w owns rows 8w..8w+7
      const double t0 = tv[2 * lane], t1 = tv[2 * lane + 1];
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) {
        const int a = warp * 8 + rr;
        const double2 lv = *reinterpret_cast<const double2*>(cur + a * TS + 2 * lane);
        const double d = warp_sum(lv.x * t0 + lv.y * t1);
        if (lane == 0) vec[a] -= d;
      }
    } else {
      // vec[a] -= sum_b L_ji[b][a] w_j[b]
      const int g = tid >> 6, a = tid & 63;
      double sacc = 0.0;
#pragma unroll
      for (int b = 0; b < 16; ++b) sacc += cur[(16 * g + b) * TS + a] * tv[16 * g + b];
      part[g * TB + a] = sacc;
      __syncthreads();
      if (tid < TB)
        vec[tid] -= ((part[tid] + part[TB + tid]) + (part[2 * TB + tid] + part[3 * TB + tid]));
    }
    __syncthreads();
  }
  cp_async_wait_all();
  __syncthreads();
  if (fwd) diag_solve_fwd(vec, Ld, Dv, u, tid);
  else diag_solve_bwd(vec, Ld, Dv, u, tid);
  if (tid < TB) (fwd ? P.t : P.w)[(int64_t)i * TB + tid] = vec[tid];
  __threadfence();
  __syncthreads();
  if (tid == 0) st_release((fwd ? fflag : bflag) + i, P.epoch);
}

size_t chol_smem_bytes() { return (size_t)(2 * TB * TS + 512) * sizeof(double); }
size_t trsv_smem_bytes() { return (size_t)(3 * TB * TS + 512 + 2 * TB + 4 * TB + 8) * sizeof(double); }

void launch_chol(const CholParams& P, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_chol_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)chol_smem_bytes());
    cudaFuncSetAttribute(k_trsv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)trsv_smem_bytes());
    configured = true;
  }
  const int ntiles = P.T * (P.T + 1) / 2;
  k_chol_tiles<<<ntiles, 256, chol_smem_bytes(), s>>>(P);
}

void launch_trsv(const TrsvParams& P, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_trsv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)trsv_smem_bytes());
    configured = true;
  }
  const int ntask = (P.T - P.i0) + P.T;
  k_trsv<<<ntask, 256, trsv_smem_bytes(), s>>>(P);
}

}  // namespace slim
