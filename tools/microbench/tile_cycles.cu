// Cycle counts of the Cholesky tile routines in isolation (one CTA).
#include <cstdio>
#include <vector>
#include <cmath>
#include "../../paper_1912_07962_b200/csrc/chol.cu"

using namespace slim;

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
  potrf_tile_blocked(S, Dv, rd, tid, err);
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
  cudaMalloc(&dG, 8 * n * n); cudaMalloc(&dL, 8 * n * n); cudaMalloc(&dc, 64); cudaMalloc(&de, 4);
  cudaMemcpy(dG, g.data(), 8 * n * n, cudaMemcpyHostToDevice); cudaMemset(de, 0, 4);
  size_t smem = (2 * TB * TS + 512 + 64) * 8;
  cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  long long c[4];
  for (int rep = 0; rep < 3; ++rep) {
    k_bench<<<1, 256, smem>>>(dG, dL, dc, de);
    cudaDeviceSynchronize();
    cudaMemcpy(c, dc, 32, cudaMemcpyDeviceToHost);
    printf("potrf %lld cyc  trsm %lld cyc  gemm64 %lld cyc\n", c[0], c[1], c[2]);
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
