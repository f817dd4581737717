// Microbenchmark: FP64 DFMA vs DMMA (mma.sync m8n8k4 f64) issue rates on B200.
// Used once to choose the instruction path for the Cholesky trailing update.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 0.999999, c = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void copy_k(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  double* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    int blocks = sms * (2048 / threads);
    int iters = 4000;
    dfma_loop<<<blocks, threads>>>(out, 10);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * (double)blocks * threads;
    printf("DFMA threads=%d blocks=%d: %.2f TFLOP/s\n", threads, blocks, flops / ms / 1e9);
    dmma_loop<<<blocks, threads>>>(out, 10);
    cudaEventRecord(e0);
    dmma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 8 * 256 * iters * (double)blocks * (threads / 32);
    printf("DMMA threads=%d blocks=%d: %.2f TFLOP/s\n", threads, blocks, flops / ms / 1e9);
  }
  size_t n = (size_t)1 << 27;  // 4 GiB per buffer in double4 units? 2^27*32B = 4 GiB
  double4 *a, *b; cudaMalloc(&a, n * 32); cudaMalloc(&b, n * 32);
  cudaMemset(a, 0, n * 32);
  copy_k<<<sms * 8, 512>>>(a, b, n);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) copy_k<<<sms * 8, 512>>>(a, b, n);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("copy: %.1f GB/s\n", 5.0 * 2 * n * 32 / ms / 1e6);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
