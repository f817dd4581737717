// gram_tc.cu -- dense Gram panel on the 5th-generation tensor cores.
//
// For generated (configs[4]) / dense fp32 operators the new Gram panel
//     C = M_k A_k^T      (N_win x ell, K = n = 65,536)
// is 180 GFLOP per step.  It runs as a 3xTF32 product on tcgen05: every fp32
// operand x is stored as x_hi = tf32(x) and x_lo = x - x_hi (both exact in
// fp32), and C = A_hi B_hi^T + A_hi B_lo^T + A_lo B_hi^T is accumulated in
// fp32 in TMEM over K chunks; the chunk partials are written as fp64 and
// summed in a fixed order (k_gram_reduce), so the accuracy is that of an
// fp32 product with short fp32 accumulation runs -- well inside the 1e-4
// bar for fp32-matrix configs (plain TF32 fails it, 3xTF32 and
// fp32 pass).
//
// Kernel anatomy (one CTA per (128-row window tile, K chunk), 128 threads):
//   warp 0 lane 0   TMA producer: 4 boxes per stage (A_hi, A_lo 128x32 fp32,
//                   B_hi, B_lo 256x32 fp32), SWIZZLE_128B, mbarrier tx count
//   warp 1 lane 0   MMA issuer: tcgen05.mma.cta_group::1.kind::tf32,
//                   M=128 N=256 K=8, 3 products x 4 K-steps per stage,
//                   tcgen05.commit frees the stage
//   warps 0-3       epilogue: tcgen05.ld 32x32b.x32 -> fp64 partial rows
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "common.cuh"
#include "gram_tc.h"
#include "kernels.h"

namespace slim {

namespace tc {

constexpr int BM = 128;     // window rows per CTA (UMMA M)
constexpr int BN = 256;     // new-block rows (UMMA N)
constexpr int BK = 32;      // fp32 elements per 128-byte swizzle row
constexpr int STAGES = 2;
constexpr int A_BYTES = BM * BK * 4;   // 16 KB
constexpr int B_BYTES = BN * BK * 4;   // 32 KB
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // 96 KB
constexpr uint32_t IDESC =            // kind::tf32, fp32 accumulate, K-major A and B
    (1u << 4) |                       // c_format F32
    (2u << 7) |                       // a_format TF32
    (2u << 10) |                      // b_format TF32
    ((uint32_t)(BN >> 3) << 17) |     // N
    ((uint32_t)(BM >> 4) << 24);      // M

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

// K-major SWIZZLE_128B smem matrix descriptor (SBO = 8 rows x 128 B)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

}  // namespace tc

// out[kc][p][j] (fp64) = sum over the kc-th K chunk of M[p][:] A[j][:]
// (hi/lo split rings, window tile rows arow[mt] in the ring)
__global__ void __launch_bounds__(128, 1)
    k_gram_tf32x3(const __grid_constant__ CUtensorMap map_a_hi,
                  const __grid_constant__ CUtensorMap map_a_lo,
                  const __grid_constant__ CUtensorMap map_b_hi,
                  const __grid_constant__ CUtensorMap map_b_lo, GramTcParams P) {
  using namespace tc;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the swizzled tiles
  // 1024-byte alignment by pointer arithmetic (keeps the shared address space)
  uint8_t* smem = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES], tmem_full;
  __shared__ uint32_t tmem_base_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = blockIdx.x, kc = blockIdx.y;
  const int arow = P.arow[mt];
  const int k0 = kc * P.kchunk;
  const int iters = P.kchunk / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full_bar[s], 1);
      tc::mbar_init(&empty_bar[s], 1);
    }
    tc::mbar_init(&tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a_hi) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b_hi) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(&tmem_base_sh)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    for (int it = 0; it < iters; ++it) {
      const int s = it % STAGES;
      const uint32_t ph = (it / STAGES) & 1;
      tc::mbar_wait(&empty_bar[s], ph ^ 1);
      uint8_t* st = smem + s * STAGE_BYTES;
      tc::mbar_expect_tx(&full_bar[s], STAGE_BYTES);
      const int x = k0 + it * BK;
      tc::tma_load_2d(st, &map_a_hi, &full_bar[s], x, arow);
      tc::tma_load_2d(st + A_BYTES, &map_a_lo, &full_bar[s], x, arow);
      tc::tma_load_2d(st + 2 * A_BYTES, &map_b_hi, &full_bar[s], x, P.brow);
      tc::tma_load_2d(st + 2 * A_BYTES + B_BYTES, &map_b_lo, &full_bar[s], x, P.brow);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    for (int it = 0; it < iters; ++it) {
      const int s = it % STAGES;
      const uint32_t ph = (it / STAGES) & 1;
      tc::mbar_wait(&full_bar[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t base = tc::smem_u32(smem + s * STAGE_BYTES);
      const uint32_t a_hi = base, a_lo = base + A_BYTES;
      const uint32_t b_hi = base + 2 * A_BYTES, b_lo = base + 2 * A_BYTES + B_BYTES;
#pragma unroll
      for (int kk = 0; kk < BK / 8; ++kk) {
        const uint32_t off = kk * 32;  // 8 tf32 = 32 bytes along the swizzle row
        const uint32_t acc = (it > 0 || kk > 0) ? 1u : 0u;
        tc::mma_tf32(tmem, tc::sw128_desc(a_hi + off), tc::sw128_desc(b_hi + off), acc);
        tc::mma_tf32(tmem, tc::sw128_desc(a_hi + off), tc::sw128_desc(b_lo + off), 1u);
        tc::mma_tf32(tmem, tc::sw128_desc(a_lo + off), tc::sw128_desc(b_hi + off), 1u);
      }
      tc::mma_commit(&empty_bar[s]);  // stage reusable once these MMAs retire
    }
    tc::mma_commit(&tmem_full);
  }
  __syncwarp();

  // ---------------- epilogue: TMEM -> fp64 partial rows ----------------
  tc::mbar_wait(&tmem_full, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + lane;  // TMEM lane = output row within the tile
  double* out = P.out + ((int64_t)kc * P.nwin + (int64_t)mt * BM + row) * P.ell;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (c0 < P.ell) {
#pragma unroll
      for (int q = 0; q < 32; q += 2) {
        double2 d2;
        d2.x = (double)__uint_as_float(v[q]);
        d2.y = (double)__uint_as_float(v[q + 1]);
        *reinterpret_cast<double2*>(out + c0 + q) = d2;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
}

// split fp32 -> (tf32 hi, tf32 lo), both rounded to nearest so the
// residual |x - hi - lo| <= 2^-23 |x| is unbiased
__global__ void k_split_tf32(const float* __restrict__ x, float* __restrict__ hi,
                             float* __restrict__ lo, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    float h, l;
    split_tf32(x[i], h, l);
    hi[i] = h;
    lo[i] = l;
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// 2D fp32 map over rows x n (row-major, K = n innermost), box (32, box_rows), SW128
static bool make_map(CUtensorMap* m, const float* base, int64_t rows, int64_t n, int box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(n * sizeof(float))};
  cuuint32_t box[2] = {(cuuint32_t)tc::BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool tma_map_f64_sw128(CUtensorMap* m, const double* base, int64_t rows, int64_t cols,
                       int box_cols, int box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(cols * sizeof(double))};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool tma_map_q(CUtensorMap* m, const int8_t* base, int qT, int box_rows, int qd) {
  auto enc = get_encode();
  if (!enc) return false;
  // dim0: QROW bytes of one digit (K = QROW int8), dim1: rows over all tile
  // rows of a column (qT * 64), dim2: (column[, k half], digit) blocks
  const cuuint64_t zblocks = (cuuint64_t)qT * (64 / QROW) * qd;
  cuuint64_t dims[3] = {(cuuint64_t)QROW, (cuuint64_t)qT * 64, zblocks};
  cuuint64_t strides[2] = {(cuuint64_t)QROW, (cuuint64_t)qT * 64 * QROW};
  cuuint32_t box[3] = {(cuuint32_t)QROW, (cuuint32_t)box_rows, (cuuint32_t)qd};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   QROW == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool gram_tc_supported(int ell, int64_t n) {
  return ell == tc::BN && n % tc::BK == 0 && get_encode() != nullptr;
}

size_t gram_tc_smem_bytes() { return (size_t)tc::STAGES * tc::STAGE_BYTES + 1024; }

int gram_tc_kchunk(int64_t n, int mtiles) {
  // The tensor core's fp32 accumulation truncates, so its error grows
  // linearly with the run length: chunks of <= 2048 K-elements keep each
  // fp32 run short (fp64 across chunks) and give enough CTAs to fill the GPU.
  (void)mtiles;
  int64_t kc = 2048;
  while (kc > tc::BK && n % kc != 0) kc /= 2;
  return (int)kc;
}

cudaError_t launch_gram_tf32x3(const float* ring_hi, const float* ring_lo, int64_t ring_rows,
                               int64_t n, const GramTcParams& P, int mtiles, int kchunks,
                               cudaStream_t s) {
  CUtensorMap mah, mal, mbh, mbl;
  if (!make_map(&mah, ring_hi, ring_rows, n, tc::BM) || !make_map(&mal, ring_lo, ring_rows, n, tc::BM) ||
      !make_map(&mbh, ring_hi, ring_rows, n, tc::BN) || !make_map(&mbl, ring_lo, ring_rows, n, tc::BN))
    return cudaErrorInvalidValue;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_gram_tf32x3, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)gram_tc_smem_bytes());
    configured = true;
  }
  dim3 grid(mtiles, kchunks);
  k_gram_tf32x3<<<grid, 128, gram_tc_smem_bytes(), s>>>(mah, mal, mbh, mbl, P);
  return cudaGetLastError();
}

void launch_split_tf32(const float* x, float* hi, float* lo, int64_t count, cudaStream_t s) {
  const int64_t blocks = (count + 255) / 256;
  k_split_tf32<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, s>>>(x, hi, lo, count);
}

}  // namespace slim
