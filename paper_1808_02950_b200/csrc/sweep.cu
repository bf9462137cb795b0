// sweep.cu — forward -> retention -> inverse -> squared error for a whole list of r in one
// read of every block (§6.1: the r = 1..64 curves of configs 1-2).
#include "adct_host.h"
#include "fused_common.cuh"

namespace adct {
namespace {

constexpr int NT = 32;  // one warp per CTA: small images still spread over every SM

// ---- any list of r: incremental inverse of the dropped coefficients ----------------------
// Coefficients are added in decreasing zig-zag rank z = 63..1; after adding rank z the
// register block e = H (W o Y o [rank >= z]) H^T is x - x_hat for r = z.  Each step is a
// rank-one update e += (w y)_z h_k h_l^T (the inverse applied to one coefficient).
template <typename SrcT, class MP>
__global__ void __launch_bounds__(NT) fused_sweep_kernel(const SrcT* __restrict__ src, KGeom g, DevMat dm,
                                                         FastDiv dbw, int32_t chunks, int32_t bpt, uint64_t rmask,
                                                         int32_t rmin, int clip, double* __restrict__ partial) {
  __shared__ float zacc[64][NT];
  const MP m(dm);
#pragma unroll
  for (int z = 0; z < 64; ++z) zacc[z][threadIdx.x] = 0.0f;
  const SrcT* base = src + (int64_t)blockIdx.y * g.image_stride;
  const uint32_t q0 = blockIdx.x * (NT * bpt) + threadIdx.x;
#pragma unroll 1
  for (int mb = 0; mb < bpt; ++mb) {
    const uint32_t q = q0 + mb * NT;
    if (q >= g.nbi) break;
    typename Src<SrcT>::Row rows[8];
    load_rows(base, g, dbw, q, rows);
    float x[8][8], y[8][8], e[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i) Src<SrcT>::to_f(rows[i], x[i]);
    fwd2d(m, x, y);
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) e[i][j] = 0.0f;
#pragma unroll
    for (int zr = 63; zr >= 1; --zr) {
      if (zr < rmin) break;
      const int pos = zz_order_at(zr);
      const int k = pos >> 3, l = pos & 7;
      const float c = y[k][l] * m.wy(k, l);
      float a[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fmac<MP>(m.h(i, k), c, -0.0f);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) e[i][j] = fmac<MP>(m.h(j, l), a[i], e[i][j]);
      if ((rmask >> zr) & 1ull) {
        float s[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        if (clip == ADCT_CLIP_NONE) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) s[j & 3] = fmaf(e[i][j], e[i][j], s[j & 3]);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float v = fminf(fmaxf(x[i][j] - e[i][j], Src<SrcT>::lo), Src<SrcT>::hi);
              if (clip == ADCT_CLIP_ROUND) v = rintf(v);
              const float d = x[i][j] - v;
              s[j & 3] = fmaf(d, d, s[j & 3]);
            }
        }
        zacc[zr - 1][threadIdx.x] += (s[0] + s[1]) + (s[2] + s[3]);
      }
    }
  }
  __syncwarp();
  // r = z+1 slots 0..62 (slot 63, r = 64, stays 0: nothing dropped); fixed shuffle order
  double* out = partial + ((int64_t)blockIdx.y * chunks + blockIdx.x) * 64;
  for (int z = 0; z < 64; ++z) {
    double v = (z == 63 || !((rmask >> (z + 1)) & 1ull)) ? 0.0 : (double)zacc[z][threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) out[z] = v;
  }
}

}  // namespace

// blocks per thread of the sweep kernel: depends on the image size only, so that the partial
// layout (and the summation order) is the same however the images are batched or sharded
int32_t sweep_bpt(const adct_geom& g) {
  const int64_t nbi = (int64_t)(g.height / 8) * (g.width / 8);
  return nbi <= 65536 ? 1 : 8;
}
int64_t sweep_chunks(const adct_geom& g) {
  const int64_t nbi = (int64_t)(g.height / 8) * (g.width / 8);
  const int64_t per = (int64_t)NT * sweep_bpt(g);
  return (nbi + per - 1) / per;
}

void launch_sweep_any(bool u8, bool specialized, int clip, cudaStream_t st, const void* src, const adct_geom& g,
                      const KGeom& kg, const DevMat& dm, const FastDiv& dbw, uint64_t rmask, int32_t rmin,
                      double* partial) {
  const int32_t chunks = (int32_t)sweep_chunks(g), bpt = sweep_bpt(g);
  const dim3 grid((unsigned)chunks, (unsigned)g.n_images);
#define ADCT_SWEEP_C(T, MP) \
  fused_sweep_kernel<T, MP><<<grid, NT, 0, st>>>((const T*)src, kg, dm, dbw, chunks, bpt, rmask, rmin, clip, partial);
  if (u8) {
    if (specialized) { ADCT_SWEEP_C(uint8_t, T1Mat) } else { ADCT_SWEEP_C(uint8_t, RtMat) }
  } else {
    if (specialized) { ADCT_SWEEP_C(int16_t, T1Mat) } else { ADCT_SWEEP_C(int16_t, RtMat) }
  }
#undef ADCT_SWEEP_C
}

}  // namespace adct
