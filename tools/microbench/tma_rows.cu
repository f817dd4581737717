// Microbenchmark: TMA delivery rate into shared memory as a function of the
// box's row width (SWIZZLE_32B rows of 32 B -- the factorization's digit-slice
// operands -- vs 64 B and 128 B rows), one CTA per SM, a 3-stage mbarrier
// ring, no compute: the consumer releases each stage as soon as it lands.
// Sources: an L2-resident buffer (64 MB) and an HBM-resident one (4 GB).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tma_rows tma_rows.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NST>
__global__ void __launch_bounds__(64, 1) stream_boxes(const __grid_constant__ CUtensorMap map, int box_bytes,
                                                      int nblocks_z, int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  if (threadIdx.x == 0) {
    for (int q = 0; q < NST; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[q])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[q])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int per_z = 1;  // one box = all digits of one (column, row block)
  if (threadIdx.x == 0) {
    for (int u = 0; u < iters; ++u) {
      const int st = u % NST;
      asm volatile(
          "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
              su32(&empty[st])),
          "r"(((u / NST) & 1) ^ 1)
          : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(box_bytes)
                   : "memory");
      // walk the source: a different row block per (CTA, iteration)
      const int y = ((blockIdx.x * 7 + u * 13) % 64) * 128;
      const int z = ((blockIdx.x + u * 148) % (nblocks_z / 7)) * 7 * per_z;
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
              su32(sm + st * box_bytes)),
          "l"(&map), "r"(su32(&full[st])), "r"(0), "r"(y), "r"(z)
          : "memory");
    }
  } else if (threadIdx.x == 32) {
    for (int u = 0; u < iters; ++u) {
      const int st = u % NST;
      asm volatile(
          "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
              su32(&full[st])),
          "r"((u / NST) & 1)
          : "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[st])) : "memory");
    }
    sink[blockIdx.x] = sm[threadIdx.x];
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) {
    printf("no cuTensorMapEncodeTiled\n");
    return 1;
  }
  struct Case {
    const char* name;
    int row_bytes, rows;
    CUtensorMapSwizzle sw;
  } cases[] = {{"SW32  rows 32 B x 128 x 7 digits (28 KB, the factorization's A box)", 32, 128,
                CU_TENSOR_MAP_SWIZZLE_32B},
               {"SW64  rows 64 B x 128 x 7 digits (56 KB)", 64, 128, CU_TENSOR_MAP_SWIZZLE_64B},
               {"SW128 rows 128 B x 64 x 7 digits (56 KB)", 128, 64, CU_TENSOR_MAP_SWIZZLE_128B},
               {"SW32  rows 32 B x 64 x 7 digits (14 KB, B box)", 32, 64, CU_TENSOR_MAP_SWIZZLE_32B}};
  unsigned long long* sink;
  cudaMalloc(&sink, 148 * 8);
  for (size_t src_bytes : {(size_t)64 << 20, (size_t)4 << 30}) {
    uint8_t* buf;
    if (cudaMalloc(&buf, src_bytes) != cudaSuccess) return 1;
    cudaMemset(buf, 1, src_bytes);
    for (const Case& c : cases) {
      // dims: {row bytes, 64 tile rows x 64 rows... = 8192 rows, z blocks}
      const cuuint64_t rows_total = 8192;
      const cuuint64_t zdim = src_bytes / (c.row_bytes * rows_total);
      cuuint64_t dims[3] = {(cuuint64_t)c.row_bytes, rows_total, zdim};
      cuuint64_t strides[2] = {(cuuint64_t)c.row_bytes, (cuuint64_t)c.row_bytes * rows_total};
      cuuint32_t box[3] = {(cuuint32_t)c.row_bytes, (cuuint32_t)c.rows, 7};
      cuuint32_t es[3] = {1, 1, 1};
      CUtensorMap map;
      if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              c.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed for %s\n", c.name);
        continue;
      }
      const int box_bytes = c.row_bytes * c.rows * 7;
      const int smem = 3 * box_bytes + 1024;
      cudaFuncSetAttribute(stream_boxes<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      const int iters = 4000;
      stream_boxes<3><<<148, 64, smem>>>(map, box_bytes, (int)zdim, 200, sink);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      stream_boxes<3><<<148, 64, smem>>>(map, box_bytes, (int)zdim, iters, sink);
      cudaEventRecord(b);
      cudaError_t e = cudaEventSynchronize(b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = 148.0 * iters * box_bytes;
      printf("%-70s src %5zu MB: %7.2f TB/s total, %6.1f GB/s per SM (%s)\n", c.name, src_bytes >> 20,
             bytes / (ms * 1e-3) / 1e12, bytes / 148 / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
    }
    cudaFree(buf);
  }
  return 0;
}
