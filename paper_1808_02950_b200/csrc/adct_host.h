// adct_host.h — host-side internals shared by the library's translation units.
#pragma once
#include <atomic>
#include <cstdint>

#include "adct.h"
#include "adct_internal.cuh"

struct adct_matrix {
  adct::DevMat dev;       // what kernels receive (by value, kernel parameter space)
  int32_t t[64];          // integer matrix (is_int)
  double chat[64];        // C_hat = S T (or the real matrix)
  double g[64];           // synthesis: A = G B' G^T
  double s[8];            // row scaling
  int64_t n[8];           // n_k = ||t_k||^2 (integer matrices)
  int32_t is_int;
  int32_t row_orth;
  int32_t specialized;    // 1 = the paper's T1 (compile-time network available)
  int64_t max_u8, max_i16;
};

namespace adct {

extern std::atomic<int64_t> g_launches;

inline void count_launch(int64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

inline adct_status check_geom(const adct_geom& g) {
  if (g.n_images < 0 || g.height <= 0 || g.width <= 0) return ADCT_E_INVALID_ARGUMENT;
  if ((g.height % 8) || (g.width % 8)) return ADCT_E_INVALID_ARGUMENT;
  if (g.row_stride < g.width || (g.row_stride % 8)) return ADCT_E_ALIGNMENT;
  if (g.n_images > 1 && g.image_stride < (int64_t)g.height * g.row_stride) return ADCT_E_INVALID_ARGUMENT;
  if (g.image_stride % 8) return ADCT_E_ALIGNMENT;
  const int64_t nb = g.n_images * (int64_t)(g.height / 8) * (g.width / 8);
  if (nb >= ((int64_t)1 << 31)) return ADCT_E_INVALID_ARGUMENT;  // per-call block index is 32-bit
  return ADCT_OK;
}

inline bool aligned(const void* p, uintptr_t a) { return ((uintptr_t)p % a) == 0; }

inline adct_status launch_status() {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ADCT_OK : ADCT_E_CUDA;
}

// geometry passed to kernels
struct KGeom {
  int64_t image_stride, row_stride;
  uint32_t bw, bh, nbi;  // blocks per row, block rows, blocks per image
  uint32_t n_images;
};

inline KGeom make_kgeom(const adct_geom& g) {
  KGeom k;
  k.image_stride = g.image_stride;
  k.row_stride = g.row_stride;
  k.bw = (uint32_t)(g.width / 8);
  k.bh = (uint32_t)(g.height / 8);
  k.nbi = k.bw * k.bh;
  k.n_images = (uint32_t)g.n_images;
  return k;
}

// number of CTAs per image of the two-level deterministic reductions
constexpr int kRedNT = 128;   // threads per CTA
constexpr int kFusedBPT = 8;    // blocks per thread, generic fused kernels
constexpr int kFusedBPTU8 = 9;  // blocks per thread, hot u8 kernel (3-deep prefetch ring)
inline int64_t fused_chunks(const adct_geom& g, int bpt = kFusedBPT) {
  const int64_t nbi = (int64_t)(g.height / 8) * (g.width / 8);
  const int64_t per = (int64_t)kRedNT * bpt;
  return (nbi + per - 1) / per;
}
constexpr int kSseRows = 8;  // image rows per CTA in psnr_reduce
inline int64_t sse_chunks(const adct_geom& g) { return (g.height + kSseRows - 1) / kSseRows; }

}  // namespace adct
