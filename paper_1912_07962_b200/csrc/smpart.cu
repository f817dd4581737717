// smpart.cu -- spatial SM partition for the slimLS pipeline (green contexts).
//
// The x-chain (residual -> triangular solves -> M^T w -> x update) is a
// latency chain of small launches; the batched factorization fills every SM
// with long tile tasks.  Sharing SMs, each x-chain launch waits for
// factorization CTAs to drain (and the 16-CTA solve cluster for a whole
// GPC's worth), and the factorization loses SMs to the x-chain bursts.  With
// SLIM_XSMS = n > 0 the x-chain stream lives in a green context of n SMs and
// the Gram / factorization / upload streams in one of the remaining SMs, so
// the two pipelines stop interfering.  The driver entry points are resolved
// at run time (no link-time libcuda dependency).
#include <cuda.h>
#include <cuda_runtime.h>

#include <string>

#include "smpart.h"

namespace slim {

template <typename F>
static F sym(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}

bool sm_partition_create(int device, int xsms, int prio_hi, int prio_lo, SmPartition* out,
                         std::string& err) {
  auto pDeviceGet = sym<decltype(&cuDeviceGet)>("cuDeviceGet");
  auto pGetRes = sym<decltype(&cuDeviceGetDevResource)>("cuDeviceGetDevResource");
  auto pSplit = sym<decltype(&cuDevSmResourceSplitByCount)>("cuDevSmResourceSplitByCount");
  auto pDesc = sym<decltype(&cuDevResourceGenerateDesc)>("cuDevResourceGenerateDesc");
  auto pCreate = sym<decltype(&cuGreenCtxCreate)>("cuGreenCtxCreate");
  auto pStream = sym<decltype(&cuGreenCtxStreamCreate)>("cuGreenCtxStreamCreate");
  if (!pDeviceGet || !pGetRes || !pSplit || !pDesc || !pCreate || !pStream) {
    err = "green-context driver entry points unavailable";
    return false;
  }
  CUdevice dev;
  CUdevResource all, grp[1], rest;
  unsigned n = 1;
  CUdevResourceDesc dx, dr;
  CUgreenCtx gx = nullptr, gr = nullptr;
  CUstream s[4] = {nullptr, nullptr, nullptr, nullptr};
  auto fail = [&](const char* what) {
    err = std::string("SM partition: ") + what + " failed";
    return false;
  };
  if (pDeviceGet(&dev, device) != CUDA_SUCCESS) return fail("cuDeviceGet");
  if (pGetRes(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return fail("cuDeviceGetDevResource");
  if (pSplit(grp, &n, &all, &rest, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE, (unsigned)xsms) !=
          CUDA_SUCCESS ||
      n != 1)
    return fail("cuDevSmResourceSplitByCount");
  if (pDesc(&dx, grp, 1) != CUDA_SUCCESS || pDesc(&dr, &rest, 1) != CUDA_SUCCESS)
    return fail("cuDevResourceGenerateDesc");
  if (pCreate(&gx, dx, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
      pCreate(&gr, dr, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
    return fail("cuGreenCtxCreate");
  if (pStream(&s[0], gx, CU_STREAM_NON_BLOCKING, prio_hi) != CUDA_SUCCESS ||
      pStream(&s[1], gr, CU_STREAM_NON_BLOCKING, prio_hi) != CUDA_SUCCESS ||
      pStream(&s[2], gr, CU_STREAM_NON_BLOCKING, prio_lo) != CUDA_SUCCESS ||
      pStream(&s[3], gr, CU_STREAM_NON_BLOCKING, prio_hi) != CUDA_SUCCESS)
    return fail("cuGreenCtxStreamCreate");
  out->gx = gx;
  out->gr = gr;
  out->x_sms = (int)grp[0].sm.smCount;
  out->rest_sms = (int)rest.sm.smCount;
  out->sx = (cudaStream_t)s[0];
  out->sg = (cudaStream_t)s[1];
  out->sf = (cudaStream_t)s[2];
  out->su = (cudaStream_t)s[3];
  return true;
}

void sm_partition_destroy(SmPartition* p) {
  if (!p->gx && !p->gr) return;
  auto pDestroy = sym<decltype(&cuGreenCtxDestroy)>("cuGreenCtxDestroy");
  for (cudaStream_t s : {p->sx, p->sg, p->sf, p->su})
    if (s) cudaStreamDestroy(s);
  if (pDestroy) {
    if (p->gx) pDestroy((CUgreenCtx)p->gx);
    if (p->gr) pDestroy((CUgreenCtx)p->gr);
  }
  *p = SmPartition{};
}

}  // namespace slim
