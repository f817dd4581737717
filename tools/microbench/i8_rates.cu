// Microbenchmark: tcgen05 kind::i8 MMA issue rate on B200 (one CTA per SM,
// operands resident in shared memory, accumulators in TMEM, no loads in the
// loop).  N = 256 is the best case (the measured int8 tensor peak, the
// roofline denominator); N = 64 is the shape of the Cholesky tile update
// (M = 128 rows of two output tiles x N = 64), whose smaller B operand per A
// read makes it shared-memory bound.
// nvcc -gencode arch=compute_100a,code=sm_100a -o i8_rates i8_rates.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

template <int N, bool REUSE>
__global__ void __launch_bounds__(128, 1) mma_loop(int* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar;
  constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  for (int i = threadIdx.x; i < (128 + N) * 128 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  if (threadIdx.x == 0) {
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sm);
    const uint64_t ad = sw128_desc(a0), bd = sw128_desc(a0 + 128 * 128);
    for (int it = 0; it < iters; ++it) {
      if (!REUSE) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t d = tmem + (uint32_t)((it & 1) * N) % 512;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                       "l"(ad + 2 * k), "l"(bd + 2 * k), "r"(IDESC), "r"(1u)
                       : "memory");
        }
      } else {
        // the Cholesky pattern: one A slice, four B slices (collector reuse)
        const uint32_t d = tmem + (uint32_t)((it & 1) * N) % 512;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::i8.collector::a::fill [%0], %1, %2, %3, p;\n"
                     "tcgen05.mma.cta_group::1.kind::i8.collector::a::use [%0], %1, %5, %3, p;\n"
                     "tcgen05.mma.cta_group::1.kind::i8.collector::a::use [%0], %1, %6, %3, p;\n"
                     "tcgen05.mma.cta_group::1.kind::i8.collector::a::lastuse [%0], %1, %7, %3, p;\n}\n" ::"r"(d),
                     "l"(ad), "l"(bd), "r"(IDESC), "r"(1u), "l"(bd + 2), "l"(bd + 4), "l"(bd + 6)
                     : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&bar))
                 : "memory");
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&bar))
                 : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  if (threadIdx.x == 0 && iters < 0) out[0] = 1;
}


// The Cholesky tile-update stage pattern: 4 stages of [A 2 dq x 16 KB | B 2 dq x
// 8 KB], 36 digit-pair MMAs per stage into 8 accumulators t = a + b - 2
// (ORDER 0: by accumulator, 1: by A digit with collector reuse, 2: by A digit
// without collector), commit per stage like the kernel's stage release.
template <int ORDER, bool RING = false, bool WRITES = false, int DEPTH = 4>
__global__ void __launch_bounds__(256, 1) chol_pattern(int* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar, ring[16];
  __shared__ volatile int s_stop;
  constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 0) s_stop = 0;
  for (int i = threadIdx.x; i < 4 * 49152 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x01fe03fdu * (i + 1), 0x7f80017fu ^ i, 0x11223344u + i, 0x55667788u - i);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    for (int q = 0; q < 16; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&ring[q])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  if (WRITES && threadIdx.x >= 128) {
    // stand-in for the TMA fills: 48 KB of shared stores per ~1.3 us into a
    // scratch region the MMAs do not read (the tail of stage 3's B area)
    uint4* dst = reinterpret_cast<uint4*>(sm + 3 * 49152 + 40960);
    long long t = clock64();
    int n = 0;
    while (!s_stop) {
      for (int i = threadIdx.x - 128; i < 512; i += 128) dst[i] = make_uint4(n, n + 1, n + 2, n + 3);
      ++n;
      while (clock64() - t < 480LL * n) {  // 8 KB per 480 clk ~ the TMA fill rate (48 KB per stage)
      }
    }
  }
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
      if (RING && it >= DEPTH)
        asm volatile("{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W2;\n}\n" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&ring[it % DEPTH])), "r"(((it / DEPTH) - 1) & 1)
                     : "memory");
      if (RING) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sm + (it & 3) * 49152);
      const uint64_t ad = sw128_desc(a0), bd = sw128_desc(a0 + 32768);
#define MMA_(Q, T, AO, BO)                                                                          \
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"                                        \
               "tcgen05.mma.cta_group::1.kind::i8" Q " [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + 64 * (T)), \
               "l"(ad + ((AO) >> 4)), "l"(bd + ((BO) >> 4)), "r"(IDESC), "r"(1u)                  \
               : "memory")
      if (ORDER == 0) {
#pragma unroll
        for (int t = 0; t < 8; ++t)
#pragma unroll
          for (int a = 1; a <= t + 1; ++a) {
            const int b = t + 2 - a;
            MMA_("", t, ((a - 1) >> 2) * 16384 + ((a - 1) & 3) * 32, ((b - 1) >> 2) * 8192 + ((b - 1) & 3) * 32);
          }
      } else {
#pragma unroll
        for (int a = 1; a <= 8; ++a)
#pragma unroll
          for (int b = 1; b <= 9 - a; ++b) {
            const int t = a + b - 2;
            const uint32_t ao = ((a - 1) >> 2) * 16384 + ((a - 1) & 3) * 32, bo = ((b - 1) >> 2) * 8192 + ((b - 1) & 3) * 32;
            if (ORDER == 2 || a == 8) MMA_("", t, ao, bo);
            else if (b == 1) MMA_(".collector::a::fill", t, ao, bo);
            else if (b == 9 - a) MMA_(".collector::a::lastuse", t, ao, bo);
            else MMA_(".collector::a::use", t, ao, bo);
          }
      }
#undef MMA_
      if (RING)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&ring[it % DEPTH])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&bar))
                 : "memory");
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&bar))
                 : "memory");
  }
  if (threadIdx.x == 0) s_stop = 1;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  if (threadIdx.x == 0 && iters < 0) out[0] = 1;
}

template <int ORDER, bool RING = false, bool WRITES = false, int DEPTH = 4>
void run_chol(int sms) {
#define KER chol_pattern<ORDER, RING, WRITES, DEPTH>
  const int iters = 4000;
  const size_t smem = 4 * 49152 + 1024;
  cudaFuncSetAttribute(KER, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int* d;
  cudaMalloc(&d, 4);
  KER<<<sms, 256, smem>>>(d, 10);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    KER<<<sms, 256, smem>>>(d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double ops = 2.0 * 128 * 64 * 32 * 36.0 * iters * sms;
  printf("Cholesky stage pattern (36 MMAs, 8 accumulators, order %d%s%s): %8.1f TOPS, %.3f us per k-tile (72 MMAs)  %s\n",
         ORDER, RING ? (DEPTH == 4 ? ", ring commit/wait depth 4" : (DEPTH == 8 ? ", ring commit/wait depth 8" : ", ring commit/wait depth 2")) : "", WRITES ? ", concurrent smem stores" : "", ops / best / 1e9, best * 1e3 / iters * 2, cudaGetErrorString(cudaGetLastError()));
}

// The kernel's operand pipeline without dependencies: one producer thread
// TMA-loads 6 boxes (48 KB) per stage from an L2-resident buffer into a
// 4-stage ring (full barriers with tx count); the MMA thread waits on full,
// issues the 36 MMAs and releases the stage with one commit every CPS stages.
#include <cuda.h>
#include <cudaTypedefs.h>
template <int CPS, bool FENCE = true, bool PAIRWAIT = false>
__global__ void __launch_bounds__(128, 1) pipe_kernel(const __grid_constant__ CUtensorMap map, int* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t full[4], empty[4], done;
  constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int q = 0; q < 4; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&full[q])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&empty[q])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  auto wait = [](uint64_t* b, uint32_t par) {
    asm volatile("{\n.reg .pred P1;\nW3:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W3;\n}\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(b)), "r"(par) : "memory");
  };
  if (threadIdx.x == 0) {
    for (int u = 0; u < iters; ++u) {
      const int st = u & 3;
      // a stage is released when its commit group completes (every CPS stages)
      if (CPS == 1 && u >= 4) wait(&empty[st], ((u >> 2) - 1) & 1);
      if (CPS >= 2 && u >= 4 && (u & 1) == 0) wait(&empty[(u >> 1) & 1], ((u >> 2) - 1) & 1);
      uint8_t* dst = sm + st * 49152;
      uint64_t* fb = CPS == 3 ? &full[(u >> 1) & 1] : &full[st];
      if (CPS != 3 || (u & 1) == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(fb)), "r"(CPS == 3 ? 98304 : 49152) : "memory");
      const int y0 = ((blockIdx.x * 7 + u) % 128) * 384;
      for (int q = 0; q < 6; ++q)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(dst + q * 8192)), "l"(&map),
                     "r"((uint32_t)__cvta_generic_to_shared(fb)), "r"(0), "r"(y0 + 64 * q) : "memory");
    }
  } else if (threadIdx.x == 32) {
    for (int u = 0; u < iters; ++u) {
      const int st = u & 3;
      if (CPS == 3) {
        if ((u & 1) == 0) wait(&full[(u >> 1) & 1], (u >> 2) & 1);
      } else if (!PAIRWAIT) wait(&full[st], (u >> 2) & 1);
      else if ((u & 1) == 0) {  // both stages of a k-tile at once
        wait(&full[st], (u >> 2) & 1);
        wait(&full[st + 1], (u >> 2) & 1);
      }
      if (FENCE) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sm + st * 49152);
      const uint64_t ad = sw128_desc(a0), bd = sw128_desc(a0 + 32768);
#pragma unroll
      for (int a = 1; a <= 8; ++a)
#pragma unroll
        for (int b = 1; b <= 9 - a; ++b) {
          const int t = a + b - 2;
          const uint32_t ao = ((a - 1) >> 2) * 16384 + ((a - 1) & 3) * 32, bo = ((b - 1) >> 2) * 8192 + ((b - 1) & 3) * 32;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + 64 * t),
                       "l"(ad + (ao >> 4)), "l"(bd + (bo >> 4)), "r"(IDESC), "r"(1u) : "memory");
        }
      if (CPS == 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&empty[st])) : "memory");
      else if ((u & 1) == 1)  // one commit releases both stages of the k-tile (CPS 2, 3)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&empty[(u >> 1) & 1])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&done)) : "memory");
    wait(&done, 0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  if (threadIdx.x == 0 && iters < 0) out[0] = 1;
}

template <int CPS, bool FENCE = true, bool PAIRWAIT = false>
void run_pipe(int sms, size_t buf_mb) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const size_t rows = buf_mb * 1024 * 1024 / 128;
  void* buf;
  cudaMalloc(&buf, rows * 128);
  cudaMemset(buf, 3, rows * 128);
  CUtensorMap map;
  cuuint64_t dims[2] = {128, (cuuint64_t)rows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {128, 64};
  cuuint32_t estr[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const size_t smem = 4 * 49152 + 1024;
  cudaFuncSetAttribute(pipe_kernel<CPS, FENCE, PAIRWAIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int* d;
  cudaMalloc(&d, 4);
  const int iters = 4000;
  pipe_kernel<CPS, FENCE, PAIRWAIT><<<sms, 128, smem>>>(map, d, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    pipe_kernel<CPS, FENCE, PAIRWAIT><<<sms, 128, smem>>>(map, d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double ops = 2.0 * 128 * 64 * 32 * 36.0 * iters * sms;
  printf("TMA pipeline (4 x 48 KB stages, mode %d (3: one full + one empty barrier per 2 stages), %zu MB source%s): %8.1f TOPS, %.3f us per k-tile  %s\n",
         CPS, buf_mb, FENCE ? (PAIRWAIT ? ", stages awaited in pairs" : "") : ", no tcgen05 fence after the full wait", ops / best / 1e9, best * 1e3 / iters * 2, cudaGetErrorString(cudaGetLastError()));
  cudaFree(buf);
}

// K-major SWIZZLE_32B descriptor: rows of 32 B (one K = 32 int8 chunk), 8-row
// core groups 256 B apart
__device__ __forceinline__ uint64_t sw32_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}
__device__ __forceinline__ constexpr uint32_t idesc_n(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
// Digit-stacked stage: A [digit][128 rows][32 B] (32 KB), B [digit][64 rows][32 B]
// (16 KB); per A digit a, ONE MMA against B digits b0..b0+n-1 stacked along N
// (N = 64 n <= 256) writes their products straight into accumulators
// t = a + b0 - 2 .. (D column offset 64 t): 12 MMAs per stage instead of 36.
// STACK=false: the same SW32 layout with the 36 N=64 MMAs (layout control).
template <bool STACK, bool RING>
__global__ void __launch_bounds__(128, 1) stacked_pattern(int* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar, ring[4];
  for (int i = threadIdx.x; i < 4 * 49152 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x01fe03fdu * (i + 1), 0x7f80017fu ^ i, 0x11223344u + i, 0x55667788u - i);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    for (int q = 0; q < 4; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&ring[q])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
      if (RING && it >= 4)
        asm volatile("{\n.reg .pred P1;\nW4:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W4;\n}\n" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&ring[it & 3])), "r"(((it >> 2) - 1) & 1)
                     : "memory");
      const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sm + (it & 3) * 49152);
      const uint64_t ad = sw32_desc(a0), bd = sw32_desc(a0 + 32768);
#define SMMA(N, T, AO, BO)                                                                           \
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"                                         \
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + 64 * (T)), \
               "l"(ad + ((AO) >> 4)), "l"(bd + ((BO) >> 4)), "r"(idesc_n(N)), "r"(1u)             \
               : "memory")
      if (STACK) {
#pragma unroll
        for (int a = 1; a <= 8; ++a)
#pragma unroll
          for (int b0 = 1; b0 <= 9 - a; b0 += 4) {
            const int n = (9 - a - b0 + 1) < 4 ? (9 - a - b0 + 1) : 4;
            SMMA(64 * n, a + b0 - 2, (a - 1) * 4096, (b0 - 1) * 2048);
          }
      } else {
#pragma unroll
        for (int a = 1; a <= 8; ++a)
#pragma unroll
          for (int b = 1; b <= 9 - a; ++b) SMMA(64, a + b - 2, (a - 1) * 4096, (b - 1) * 2048);
      }
#undef SMMA
      if (RING)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&ring[it & 3])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
    asm volatile("{\n.reg .pred P1;\nW5:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W5;\n}\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  if (threadIdx.x == 0 && iters < 0) out[0] = 1;
}

template <bool STACK, bool RING>
void run_stacked(int sms) {
  const int iters = 4000;
  const size_t smem = 4 * 49152 + 1024;
  cudaFuncSetAttribute(stacked_pattern<STACK, RING>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int* d;
  cudaMalloc(&d, 4);
  stacked_pattern<STACK, RING><<<sms, 128, smem>>>(d, 10);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    stacked_pattern<STACK, RING><<<sms, 128, smem>>>(d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double ops = 2.0 * 128 * 64 * 32 * 36.0 * iters * sms;
  printf("SW32 digit layout, %s%s: %8.1f TOPS (digit-pair ops), %.3f us per k-tile  %s\n",
         STACK ? "12 digit-stacked MMAs (N up to 256)" : "36 N=64 MMAs", RING ? ", ring commit/wait" : "",
         ops / best / 1e9, best * 1e3 / iters * 2, cudaGetErrorString(cudaGetLastError()));
}

template <int N, bool REUSE = false>
void run(int sms) {
  const int iters = 20000;
  const size_t smem = (128 + N) * 128 + 1024;
  cudaFuncSetAttribute(mma_loop<N, REUSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int* d;
  cudaMalloc(&d, 4);
  mma_loop<N, REUSE><<<sms, 128, smem>>>(d, 100);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    mma_loop<N, REUSE><<<sms, 128, smem>>>(d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double ops = 2.0 * 128 * N * 32 * 4.0 * iters * sms;
  printf("kind::i8 M=128 N=%3d K=32 (SS, smem operands%s): %8.1f TOPS  %s\n", N,
         REUSE ? ", A reused x4 via collector" : "", ops / best / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64>(sms);
  run<128>(sms);
  run<256>(sms);
  run<64, true>(sms);
  run_chol<0>(sms);
  run_chol<1>(sms);
  run_chol<2>(sms);
  run_chol<1, true, false, 2>(sms);
  run_chol<1, true>(sms);
  run_chol<1, true, false, 8>(sms);
  run_chol<1, false, true>(sms);
  run_chol<1, true, true>(sms);
  run_pipe<1>(sms, 48);
  run_pipe<2>(sms, 48);
  run_pipe<1>(sms, 4096);
  run_pipe<1, false>(sms, 48);
  run_pipe<2, true, true>(sms, 48);
  run_pipe<2>(sms, 4096);
  run_pipe<3>(sms, 48);
  run_stacked<false, false>(sms);
  run_stacked<true, false>(sms);
  run_stacked<false, true>(sms);
  run_stacked<true, true>(sms);
  return 0;
}
