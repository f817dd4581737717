// siddon.h -- device parallel-beam projector (siddon.cu)
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace slim {

struct SiddonSpec {
  int dims;               // 2 or 3
  int64_t grid;           // image / volume side
  int64_t rows_per_view;  // rays (2D) or side^2 (3D)
  int64_t side;           // 3D detector side
  double spacing;         // detector spacing
  const double* views;    // device: 9 doubles per view (d, axis / e1, -- / e2)
  const int* ray_of_row;  // device: within-view ray index of each row, or null
  int64_t m;              // rows
};

// nnz per row -> rowptr (m + 1, int64, device)
cudaError_t siddon_count(const SiddonSpec& S, int64_t* rowptr, cudaStream_t s);
// columns and lengths (fp64 or fp32) of every row; err |= 1 on a count
// mismatch, 2 on a row that is not strictly ordered
cudaError_t siddon_fill(const SiddonSpec& S, const int64_t* rowptr, int* col, void* val, bool f64,
                        int* err, cudaStream_t s);
// y = A x over all m rows (problem setup: clean data)
cudaError_t csr_spmv(const int64_t* rowptr, const int* col, const void* val, bool f64,
                     const double* x, double* y, int64_t m, cudaStream_t s);

}  // namespace slim
