// fused_common.cuh — device helpers shared by the fused kernels (fused.cu, sweep.cu).
#pragma once
#include "adct_host.h"

namespace adct {

template <int CLIP>
__device__ __forceinline__ float clipv(float v, float lo, float hi) {
  if (CLIP == ADCT_CLIP_NONE) return v;
  v = fminf(fmaxf(v, lo), hi);
  if (CLIP == ADCT_CLIP_ROUND) v = rintf(v);
  return v;
}

template <typename SrcT>
__device__ __forceinline__ void load_rows(const SrcT* __restrict__ base, const KGeom& g, const FastDiv& dbw,
                                          uint32_t q, typename Src<SrcT>::Row (&r)[8]) {
  const uint32_t by = fdiv(q, dbw);
  const uint32_t bx = q - by * g.bw;
  const SrcT* p = base + (int64_t)by * 8 * g.row_stride + (int64_t)bx * 8;
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = Src<SrcT>::load(p + (int64_t)i * g.row_stride);
}


}  // namespace adct
