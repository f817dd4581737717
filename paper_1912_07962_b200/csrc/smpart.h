// smpart.h -- green-context SM partition (smpart.cu)
#pragma once
#include <cuda_runtime.h>

#include <string>

namespace slim {

struct SmPartition {
  void* gx = nullptr;  // CUgreenCtx of the x-chain partition
  void* gr = nullptr;  // CUgreenCtx of the rest
  int x_sms = 0, rest_sms = 0;
  cudaStream_t sx = nullptr, sg = nullptr, sf = nullptr, su = nullptr;
};

// x-chain stream on xsms SMs; Gram, factorization and upload streams on the rest
bool sm_partition_create(int device, int xsms, int prio_hi, int prio_lo, SmPartition* out,
                         std::string& err);
void sm_partition_destroy(SmPartition* p);

}  // namespace slim
