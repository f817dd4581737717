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
// then POTRF (diagonal) or TRSM against L_jj (off-diagonal) in shared
// memory, and publishes the tile with a release flag.  Every dependency of
// ticket t has a smaller ticket, handed to a CTA that is already resident,
// so spinning on acquire flags cannot deadlock.  G is never assembled:
// the initial C_ij is gathered straight from the ring of incremental Gram
// panels (alpha scaling and +I fused), so the only N^2 pass is the read.
#include "common.cuh"
#include "kernels.h"

namespace slim {

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

__device__ __forceinline__ void store_tile(double* g, const double* s, int tid) {
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int c = tid + it * 256;
    const int row = c >> 5, cc = (c & 31) * 2;
    const double2 v = *reinterpret_cast<const double2*>(s + row * TS + cc);
    *reinterpret_cast<double2*>(g + row * TB + cc) = v;
  }
}

// In-place Cholesky of the 64x64 tile in shared memory (lower part valid).
// One barrier per column: the Schur update uses the unscaled pivot column
// (S_ij -= S_ic S_jc / S_cc), the final pass scales by sqrt of the pivots.
__device__ void potrf_tile_smem(double* S, int tid, int* error) {
  const int r = tid >> 2, c0 = tid & 3;
  for (int c = 0; c < TB - 1; ++c) {
    if (r > c) {
      const double f = S[r * TS + c] / S[c * TS + c];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int j = c0 + 4 * q;
        if (j > c && j <= r) S[r * TS + j] -= f * S[j * TS + c];
      }
    }
    __syncthreads();
  }
  double out[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int j = c0 + 4 * q;
    const double d = S[j * TS + j];
    if (j < r) out[q] = S[r * TS + j] / sqrt(d);
    else if (j == r) out[q] = sqrt(d);
    else out[q] = 0.0;
    if (j == r && !(d > 0.0)) atomicExch(error, 1);
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 16; ++q) S[r * TS + c0 + 4 * q] = out[q];
  __syncthreads();
}

// X L^T = C for X (64x64), L lower (64x64) in shared memory; X overwrites C.
__device__ void trsm_tile_smem(double* X, const double* Lt, double* sinv, int tid) {
  const int r = tid >> 2, c0 = tid & 3;
  if (tid < TB) sinv[tid] = 1.0 / Lt[tid * TS + tid];
  __syncthreads();
  for (int c = 0; c < TB - 1; ++c) {
    const double x = X[r * TS + c] * sinv[c];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int j = c0 + 4 * q;
      if (j > c) X[r * TS + j] -= x * Lt[j * TS + c];
    }
    __syncthreads();
  }
  double out[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) out[q] = X[r * TS + c0 + 4 * q] * sinv[c0 + 4 * q];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 16; ++q) X[r * TS + c0 + 4 * q] = out[q];
  __syncthreads();
}

__global__ void __launch_bounds__(256, 3) k_chol_tiles(CholParams P) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + TB * TS;
  __shared__ int s_task;
  __shared__ double s_inv[TB];
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
    potrf_tile_smem(As, tid, P.error);
  } else {
    if (tid == 0) wait_flag(P.flags + (j * (j + 1) / 2 + j), P.epoch);
    __syncthreads();
    load_tile_async(Bs, P.L + tile_off(j, j), tid);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    trsm_tile_smem(As, Bs, s_inv, tid);
  }
  store_tile(P.L + tile_off(i, j), As, tid);
  __threadfence();
  __syncthreads();
  if (tid == 0) st_release(P.flags + (i * (i + 1) / 2 + j), P.epoch);
}

// ---------------------------------------------------------------------------
// Triangular solves  t = L^{-1} y  (y zero above row N - ell),  w = L^{-T} t.
// One launch; tickets 0..nf-1 run the forward tile rows i0..T-1 in order,
// the rest run the backward tile rows T-1..0.  Each task accumulates the
// off-diagonal products as the producing tiles publish, then one warp does
// the 64-row substitution with shuffles.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void load_vec_cg(double* s, const double* g, int tid) {
  if (tid < TB) s[tid] = __ldcg(g + tid);
}

__global__ void __launch_bounds__(256) k_trsv(TrsvParams P) {
  extern __shared__ __align__(16) double smem[];
  double* Ls = smem;                 // 64 x TS diagonal tile
  double* vec = smem + TB * TS;      // 64 accumulator
  double* tv = vec + TB;             // 64 incoming solved segment
  double* part = tv + TB;            // 4 x 64 partial sums
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

  if (fwd) {
    if (tid < TB) {
      const int pr = i * TB + tid;
      vec[tid] = (pr >= P.rstart && pr < P.N) ? P.r[pr - P.rstart] : 0.0;
    }
    __syncthreads();
    for (int jj = i0; jj < i; ++jj) {
      if (tid == 0) wait_flag(fflag + jj, P.epoch);
      __syncthreads();
      load_vec_cg(tv, P.t + (int64_t)jj * TB, tid);
      __syncthreads();
      const double* Lij = P.L + tile_off(i, jj);
      // warp w owns rows 8w .. 8w+7; lanes split the 64 columns in pairs
      const double t0 = tv[2 * lane], t1 = tv[2 * lane + 1];
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) {
        const int a = warp * 8 + rr;
        const double2 lv = *reinterpret_cast<const double2*>(Lij + a * TB + 2 * lane);
        const double d = warp_sum(lv.x * t0 + lv.y * t1);
        if (lane == 0) vec[a] -= d;
      }
      __syncthreads();
    }
  } else {
    if (i >= i0) {
      if (tid == 0) wait_flag(fflag + i, P.epoch);
      __syncthreads();
      load_vec_cg(vec, P.t + (int64_t)i * TB, tid);
    } else if (tid < TB) {
      vec[tid] = 0.0;
    }
    __syncthreads();
    for (int jj = T - 1; jj > i; --jj) {
      if (tid == 0) wait_flag(bflag + jj, P.epoch);
      __syncthreads();
      load_vec_cg(tv, P.w + (int64_t)jj * TB, tid);
      __syncthreads();
      const double* Lji = P.L + tile_off(jj, i);
      // acc[a] -= sum_b L_ji[b][a] w_j[b]; thread (g, a) sums rows 16g..16g+15
      const int g = tid >> 6, a = tid & 63;
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < 16; ++b) s += Lji[(16 * g + b) * TB + a] * tv[16 * g + b];
      part[g * TB + a] = s;
      __syncthreads();
      if (tid < TB) vec[tid] -= ((part[tid] + part[TB + tid]) + (part[2 * TB + tid] + part[3 * TB + tid]));
      __syncthreads();
    }
  }

  // diagonal tile substitution by warp 0
  load_tile_async(Ls, P.L + tile_off(i, i), tid);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  if (warp == 0) {
    double v0 = vec[lane], v1 = vec[lane + 32];
    if (fwd) {
      for (int c = 0; c < TB; ++c) {
        const double src = (c < 32) ? v0 : v1;
        const double x = __shfl_sync(0xffffffffu, src, c & 31) / Ls[c * TS + c];
        if (c < 32) { if (lane == c) v0 = x; } else { if (lane == c - 32) v1 = x; }
        if (lane > c) v0 -= Ls[lane * TS + c] * x;
        if (lane + 32 > c) v1 -= Ls[(lane + 32) * TS + c] * x;
      }
      double* out = P.t + (int64_t)i * TB;
      out[lane] = v0;
      out[lane + 32] = v1;
    } else {
      for (int c = TB - 1; c >= 0; --c) {
        const double src = (c < 32) ? v0 : v1;
        const double x = __shfl_sync(0xffffffffu, src, c & 31) / Ls[c * TS + c];
        if (c < 32) { if (lane == c) v0 = x; } else { if (lane == c - 32) v1 = x; }
        if (lane < c) v0 -= Ls[c * TS + lane] * x;
        if (lane + 32 < c) v1 -= Ls[c * TS + lane + 32] * x;
      }
      double* out = P.w + (int64_t)i * TB;
      out[lane] = v0;
      out[lane + 32] = v1;
    }
    __threadfence();
  }
  __syncthreads();
  if (tid == 0) st_release((fwd ? fflag : bflag) + i, P.epoch);
}

}  // namespace slim

namespace slim {

size_t chol_smem_bytes() { return (size_t)2 * TB * TS * sizeof(double); }
size_t trsv_smem_bytes() { return (size_t)(TB * TS + 2 * TB + 4 * TB) * sizeof(double); }

void launch_chol(const CholParams& P, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_chol_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)chol_smem_bytes());
    configured = true;
  }
  const int ntiles = P.T * (P.T + 1) / 2;
  k_chol_tiles<<<ntiles, 256, chol_smem_bytes(), s>>>(P);
}

void launch_trsv(const TrsvParams& P, cudaStream_t s) {
  const int ntask = (P.T - P.i0) + P.T;
  k_trsv<<<ntask, 256, trsv_smem_bytes(), s>>>(P);
}

}  // namespace slim
