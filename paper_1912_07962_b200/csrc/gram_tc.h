// gram_tc.h -- tcgen05 3xTF32 Gram panel (see gram_tc.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace slim {

constexpr int GRAM_TC_MAX_MTILES = 256;

struct GramTcParams {
  double* out;      // kchunks x nwin x ell fp64 partials
  int64_t nwin;     // window rows (multiple of 128)
  int ell;          // new-block rows (== 256)
  int kchunk;       // K elements per CTA (multiple of 32)
  int brow;         // first ring row of the new block
  int arow[GRAM_TC_MAX_MTILES];  // first ring row of each 128-row window tile
};

bool gram_tc_supported(int ell, int64_t n);
// 2D fp64 TMA map (cols innermost), box (box_cols, box_rows), SWIZZLE_128B
bool tma_map_f64_sw128(CUtensorMap* m, const double* base, int64_t rows, int64_t cols,
                       int box_cols, int box_rows);
size_t gram_tc_smem_bytes();
int gram_tc_kchunk(int64_t n, int mtiles);
cudaError_t launch_gram_tf32x3(const float* ring_hi, const float* ring_lo, int64_t ring_rows,
                               int64_t n, const GramTcParams& P, int mtiles, int kchunks,
                               cudaStream_t s);
void launch_split_tf32(const float* x, float* hi, float* lo, int64_t count, cudaStream_t s);

}  // namespace slim
