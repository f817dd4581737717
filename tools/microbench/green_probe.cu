// Probe: green-context SM partitions with runtime-API launches (B200).
// nvcc -gencode arch=compute_100a,code=sm_100a -o green_probe green_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>
#include <vector>

__global__ void k_smid(int* out, int spin) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
  long long t0 = clock64();
  while (clock64() - t0 < spin) {
  }
}
__global__ void k_smid_cluster(int* out) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
}

#define CKD(x)                                                              \
  do {                                                                      \
    CUresult r = (x);                                                       \
    if (r != CUDA_SUCCESS) {                                                \
      const char* m = nullptr;                                              \
      cuGetErrorString(r, &m);                                              \
      printf("FAIL %s: %s (line %d)\n", #x, m ? m : "?", __LINE__);         \
      return 1;                                                             \
    }                                                                       \
  } while (0)

int main(int argc, char** argv) {
  const int xs = argc > 1 ? atoi(argv[1]) : 16;
  cudaFree(0);
  CUdevice dev;
  CKD(cuDeviceGet(&dev, 0));
  CUdevResource all;
  CKD(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs %u\n", all.sm.smCount);
  CUdevResource grp[1], rest;
  unsigned n = 1;
  CKD(cuDevSmResourceSplitByCount(grp, &n, &all, &rest, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE, xs));
  printf("groups %u: x %u SMs, rest %u SMs\n", n, grp[0].sm.smCount, rest.sm.smCount);
  CUdevResourceDesc dx, dr;
  CKD(cuDevResourceGenerateDesc(&dx, grp, 1));
  CKD(cuDevResourceGenerateDesc(&dr, &rest, 1));
  CUgreenCtx gx, gr;
  CKD(cuGreenCtxCreate(&gx, dx, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CKD(cuGreenCtxCreate(&gr, dr, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sx, sr;
  CKD(cuGreenCtxStreamCreate(&sx, gx, CU_STREAM_NON_BLOCKING, -1));
  CKD(cuGreenCtxStreamCreate(&sr, gr, CU_STREAM_NON_BLOCKING, 0));
  int* d = nullptr;
  cudaMalloc(&d, sizeof(int) * 4096);  // primary context allocation
  // plain runtime launches into green streams, primary context current
  k_smid<<<1024, 128, 0, (cudaStream_t)sr>>>(d, 200000);
  k_smid<<<256, 128, 0, (cudaStream_t)sx>>>(d + 2048, 200000);
  cudaError_t e = cudaDeviceSynchronize();
  printf("launch into green streams: %s / %s\n", cudaGetErrorString(cudaGetLastError()), cudaGetErrorString(e));
  std::vector<int> h(4096);
  cudaMemcpy(h.data(), d, sizeof(int) * 4096, cudaMemcpyDeviceToHost);
  std::set<int> a(h.begin(), h.begin() + 1024), b(h.begin() + 2048, h.begin() + 2048 + 256);
  int inter = 0;
  for (int v : b) inter += a.count(v);
  printf("rest kernel SMs %zu, x kernel SMs %zu, overlap %d\n", a.size(), b.size(), inter);
  cudaFuncSetAttribute(k_smid_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int C : {16, 8, 4}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C, 1, 1);
    cfg.blockDim = dim3(128, 1, 1);
    cfg.stream = (cudaStream_t)sx;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int maxc = -1;
    cudaError_t eq = cudaOccupancyMaxPotentialClusterSize(&maxc, k_smid_cluster, &cfg);
    cudaMemset(d + 3000, 0xff, sizeof(int) * 16);
    cudaError_t el = cudaLaunchKernelEx(&cfg, k_smid_cluster, d + 3000);
    e = cudaStreamSynchronize((cudaStream_t)sx);
    cudaMemcpy(h.data(), d, sizeof(int) * 4096, cudaMemcpyDeviceToHost);
    std::set<int> c(h.begin() + 3000, h.begin() + 3000 + C);
    int inx = 0;
    for (int v : c) inx += b.count(v);
    printf("cluster %d in x partition: max potential %d (%s), launch %s / %s, SMs %zu inside x %d\n", C, maxc,
           cudaGetErrorString(eq), cudaGetErrorString(el), cudaGetErrorString(e), c.size(), inx);
  }
  // events across green streams
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  k_smid<<<64, 128, 0, (cudaStream_t)sr>>>(d, 1000);
  cudaEventRecord(ev, (cudaStream_t)sr);
  cudaStreamWaitEvent((cudaStream_t)sx, ev, 0);
  k_smid<<<64, 128, 0, (cudaStream_t)sx>>>(d, 1000);
  e = cudaDeviceSynchronize();
  printf("cross-partition event: %s\n", cudaGetErrorString(e));
  // timing events on a green stream
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  cudaEventRecord(t0, (cudaStream_t)sx);
  k_smid<<<16, 128, 0, (cudaStream_t)sx>>>(d, 100000);
  cudaEventRecord(t1, (cudaStream_t)sx);
  e = cudaEventSynchronize(t1);
  float ms = 0;
  cudaEventElapsedTime(&ms, t0, t1);
  printf("timing events: %s %.3f ms\n", cudaGetErrorString(e), ms);
  return 0;
}
