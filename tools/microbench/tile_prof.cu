// Cycle counts of the Cholesky tile routines in isolation (one CTA).
#include <cstdio>
#include <vector>
#include <cmath>
#include "../../paper_1912_07962_b200/csrc/chol.cu"

using namespace slim;
namespace slim {
__device__ void potrf_prof(double* S, double* Dv, double* rdiag, int tid, int* error, long long* pc) {
  const int warp = tid >> 5, lane = tid & 31;
  for (int p = 0; p < 8; ++p) {
    const int c0 = 8 * p;
    long long tp0 = clock64();
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
    long long tp1 = clock64();
    if (tid == 0) pc[4 + p] += tp1 - tp0;
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
    if (tid == 0) pc[12 + p] += clock64() - tp1;
  }
  long long tz = clock64();
  // zero the strict upper triangle of the off-diagonal 8x8 blocks
  for (int e = tid; e < TB * TB; e += 256) {
    const int r = e >> 6, c = e & 63;
    if ((c >> 3) > (r >> 3)) S[r * TS + c] = 0.0;
  }
  __syncthreads();
  if (tid == 0) pc[20] += clock64() - tz;
  tz = clock64();
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
  if (tid == 0) pc[21] += clock64() - tz;
}

}


__global__ void k_bench(const double* G, double* Lout, long long* cyc, int* err) {
  extern __shared__ __align__(16) double sm[];
  double* S = sm;
  double* X = S + TB * TS;
  double* Dv = X + TB * TS;
  double* rd = Dv + 512;
  int tid = threadIdx.x;
  for (int e = tid; e < TB * TB; e += 256) S[(e / TB) * TS + e % TB] = G[e];
  __syncthreads();
  long long t0 = clock64();
  potrf_prof(S, Dv, rd, tid, err, cyc + 4);
  long long t1 = clock64();
  // TRSM of a random tile against the factor
  for (int e = tid; e < TB * TB; e += 256) X[(e / TB) * TS + e % TB] = G[e] * 0.5;
  __syncthreads();
  long long t2 = clock64();
  trsm_tile_warp(X, S, Dv, tid >> 5, tid & 31);
  __syncthreads();
  long long t3 = clock64();
  // one 64x64x64 tile GEMM step from shared memory (8 warps, DMMA)
  double acc[8][2] = {};
  const int warp = tid >> 5, lane = tid & 31;
  const int arow = (warp * 8 + (lane >> 2)) * TS + (lane & 3);
  __syncthreads();
  long long t4 = clock64();
#pragma unroll 4
  for (int k4 = 0; k4 < TB / 4; ++k4) {
    const double a = -S[arow + 4 * k4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const double b = X[(nt * 8 + (lane >> 2)) * TS + 4 * k4 + (lane & 3)];
      dmma8x8x4(acc[nt], a, b);
    }
  }
  __syncthreads();
  long long t5 = clock64();
  if (tid == 0) { cyc[0] = t1 - t0; cyc[1] = t3 - t2; cyc[2] = t5 - t4; }
  double s = 0; for (int nt = 0; nt < 8; ++nt) s += acc[nt][0] + acc[nt][1];
  if (s == 12345.0) cyc[3] = 1;
  for (int e = tid; e < TB * TB; e += 256) Lout[e] = S[(e / TB) * TS + e % TB];
}

int main() {
  const int n = 64;
  std::vector<double> g(n * n), a(n * (n + 8));
  srand(1);
  for (auto& v : a) v = (rand() / (double)RAND_MAX) - 0.5;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0; for (int k = 0; k < n + 8; ++k) s += a[i * (n + 8) + k] * a[j * (n + 8) + k];
      g[i * n + j] = s + (i == j ? 1.0 : 0.0);
    }
  double *dG, *dL; long long* dc; int* de;
  cudaMalloc(&dG, 8 * n * n); cudaMalloc(&dL, 8 * n * n); cudaMalloc(&dc, 8 * 32); cudaMemset(dc, 0, 8 * 32); cudaMalloc(&de, 4);
  cudaMemcpy(dG, g.data(), 8 * n * n, cudaMemcpyHostToDevice); cudaMemset(de, 0, 4);
  size_t smem = (2 * TB * TS + 512 + 64) * 8;
  cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  long long c[32];
  for (int rep = 0; rep < 3; ++rep) {
    k_bench<<<1, 256, smem>>>(dG, dL, dc, de);
    cudaDeviceSynchronize();
    cudaMemset(dc, 0, 8 * 32);
    k_bench<<<1, 256, smem>>>(dG, dL, dc, de);
    cudaDeviceSynchronize();
    cudaMemcpy(c, dc, 8 * 32, cudaMemcpyDeviceToHost);
    printf("potrf %lld cyc  trsm %lld cyc  gemm64 %lld cyc\n", c[0], c[1], c[2]);
    printf("  panels:"); for (int p = 0; p < 8; ++p) printf(" %lld", c[8 + p]); printf("\n");
    printf("  updates:"); for (int p = 0; p < 8; ++p) printf(" %lld", c[16 + p]); printf("\n");
    printf("  zero %lld  inverse %lld\n", c[24], c[25]);
  }
  std::vector<double> L(n * n);
  cudaMemcpy(L.data(), dL, 8 * n * n, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < n; ++i) for (int j = 0; j <= i; ++j) {
    double s = 0; for (int k = 0; k <= j; ++k) s += L[i * n + k] * L[j * n + k];
    err = fmax(err, fabs(s - g[i * n + j]));
  }
  printf("max |LL^T - G| = %.3e  (%s)\n", err, cudaGetErrorString(cudaGetLastError()));
}
