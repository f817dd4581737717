// common.cuh -- shared device helpers for the slimLS B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace slim {

// Cholesky / triangular-solve tile edge (fp64): 64x64 = 32 KB per tile.
constexpr int TB = 64;
// shared-memory row stride (doubles) for a 64-wide tile: 68 * 8 B = 544 B,
// so the 8 rows touched by one DMMA fragment load fall on 4 distinct
// 32-byte bank groups -> 2 wavefronts per 256-byte warp load (optimal).
constexpr int TS = 68;
constexpr int MAX_WINDOW = 32;   // r + 1 limit carried in kernel params
constexpr int MAX_BATCH = 16;    // systems factored by one interleaved launch
constexpr int MAX_REFS = 8;      // error references tracked on device

// ---- DMMA: D(8x8) += A(8x4, row) * B(4x8, col), fp64, IEEE FMA semantics ----
// per-block CSC column pointers: n + 1 entries padded to a multiple of 4, so
// every block's array starts 16-byte aligned (int4 loads of 4 columns)
__host__ __device__ __forceinline__ int64_t csc_stride(int n) { return ((int64_t)n + 4) & ~(int64_t)3; }

__device__ __forceinline__ void dmma8x8x4(double (&d)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// ---- acquire / release flags (tile DAG scheduling inside one launch) ----
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// spin until *p >= want (epoch-valued flags; one thread spins, CTA then
// syncs).  Tight spin: the producer is resident and the flag sits in L2,
// so any sleep only adds latency to the factorization's critical path.
__device__ __forceinline__ void wait_flag(const int* p, int want) {
  while (ld_acquire(p) < want) {
  }
}

// ---- cp.async (LDGSTS, L2-only .cg: never serves stale L1 lines) ----
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
// 4- and 8-byte copies (.ca: the only variant for sizes < 16)
template <int BYTES>
__device__ __forceinline__ void cp_async_small(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// L2-coherent scalar loads for data produced earlier in the same launch
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <typename T>
__device__ __forceinline__ double to_f64(T v) { return static_cast<double>(v); }

// 3xTF32 operand split: x ~= hi + lo, both exact TF32 (round to nearest)
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  uint32_t h, l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  const float r = x - __uint_as_float(h);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(r));
  hi = __uint_as_float(h);
  lo = __uint_as_float(l);
}

// splitmix64 (configs[4] generator): z += golden; z = (z ^ z>>30) * c1;
// z = (z ^ z>>27) * c2; z ^= z>>31
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// lower-triangular tile storage: tile (i, j), i >= j, row-major inside the
// tile, tiles laid out row by row: offset (i (i + 1) / 2 + j) * TB * TB
__host__ __device__ __forceinline__ int64_t tile_off(int i, int j) {
  return ((int64_t)i * (i + 1) / 2 + j) * (int64_t)(TB * TB);
}

}  // namespace slim
