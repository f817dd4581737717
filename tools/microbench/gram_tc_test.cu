// Standalone check + timing of the tcgen05 3xTF32 Gram kernel.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "gram_tc.h"
using namespace slim;

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atol(argv[1]) : 65536;
  const int nwin = argc > 2 ? atoi(argv[2]) : 5376;
  const int ell = 256;
  const int64_t rows = nwin + ell;
  std::vector<float> h((size_t)rows * n);
  srand(3);
  for (auto& v : h) v = ((rand() / (float)RAND_MAX) - 0.5f) / 128.f;
  float *x, *hi, *lo; double* out;
  cudaMalloc(&x, h.size() * 4); cudaMalloc(&hi, h.size() * 4); cudaMalloc(&lo, h.size() * 4);
  cudaMemcpy(x, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  launch_split_tf32(x, hi, lo, (int64_t)h.size(), 0);
  const int mtiles = nwin / 128;
  const int kchunk = gram_tc_kchunk(n, mtiles);
  const int kcs = (int)(n / kchunk);
  cudaMalloc(&out, sizeof(double) * kcs * nwin * ell);
  GramTcParams P{};
  P.out = out; P.nwin = nwin; P.ell = ell; P.kchunk = kchunk; P.brow = nwin;
  for (int t = 0; t < mtiles; ++t) P.arow[t] = t * 128;
  printf("supported=%d mtiles=%d kchunk=%d kcs=%d smem=%zu\n", (int)gram_tc_supported(ell, n), mtiles, kchunk, kcs, gram_tc_smem_bytes());
  cudaError_t e = launch_gram_tf32x3(hi, lo, rows, n, P, mtiles, kcs, 0);
  printf("launch: %s\n", cudaGetErrorString(e));
  e = cudaDeviceSynchronize();
  printf("sync: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) launch_gram_tf32x3(hi, lo, rows, n, P, mtiles, kcs, 0);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
  double flops = 2.0 * nwin * ell * n;
  printf("time %.3f ms  %.1f TFLOP/s (fp32-equivalent), %.1f TFLOP/s tf32 issued\n", ms, flops / ms / 1e9, 3 * flops / ms / 1e9);
  std::vector<double> part((size_t)kcs * nwin * ell);
  cudaMemcpy(part.data(), out, part.size() * 8, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  for (int p = 0; p < nwin; p += 97) for (int j = 0; j < ell; j += 13) {
    double s = 0; for (int q = 0; q < kcs; ++q) s += part[((size_t)q * nwin + p) * ell + j];
    double ref = 0; const float* ra = &h[(size_t)p * n]; const float* rb = &h[(size_t)(nwin + j) * n];
    for (int64_t k = 0; k < n; ++k) ref += (double)ra[k] * (double)rb[k];
    maxerr = fmax(maxerr, fabs(s - ref)); maxref = fmax(maxref, fabs(ref));
  }
  printf("max abs err %.3e  (max |ref| %.3e, rel %.3e)\n", maxerr, maxref, maxerr / maxref);
  return 0;
}
