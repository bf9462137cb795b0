// sweep.cu — forward -> retention -> inverse -> squared error for a whole list of r in one
// read of every block (§6.1: the r = 1..64 curves of configs 1-2).
#include "adct_host.h"
#include "fused_common.cuh"

// ADCT_SWEEP_PACKED: the rank-one updates and the squared error of CLIP_NONE on column pairs
// (FFMA2: two pixels per issue slot, each element the same fma sequence as the scalar code)
#ifndef ADCT_SWEEP_PACKED
#define ADCT_SWEEP_PACKED 1
#endif

namespace adct {
namespace {

constexpr int NT = 32;  // one warp per CTA: small images still spread over every SM

// ---- any list of r: incremental inverse of the dropped coefficients ----------------------
// Coefficients are added in decreasing zig-zag rank z = 63..1; after adding rank z the
// register block e = H (W o Y o [rank >= z]) H^T is x - x_hat for r = z.  Each step is a
// rank-one update e += (w y)_z h_k h_l^T (the inverse applied to one coefficient).
// zig-zag position of rank z (reading A5), for the rolled loop below
__constant__ int8_t c_zz[64];

// The rank loop is rolled (runtime coefficient position): an unrolled 63-step body is
// ~10^4 instructions and thrashed the instruction cache (ncu: 72% "no instruction" stalls).
// The matrix comes from kernel parameters for every matrix, T1 included: products by 0 and +-1
// are exact in fp32, so the sums are the same as with the compile-time network.
template <typename SrcT>
__global__ void __launch_bounds__(NT) fused_sweep_kernel(const SrcT* __restrict__ src, KGeom g, DevMat dm,
                                                         FastDiv dbw, int32_t chunks, int32_t bpt, uint64_t rmask,
                                                         int32_t rmin, int clip, double* __restrict__ partial) {
  __shared__ float zacc[64][NT];
  __shared__ float ys[64][NT];
  const RtMat m(dm);
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
    float x[8][8], e[8][8];
    {
      float y[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i) Src<SrcT>::to_f(rows[i], x[i]);
      fwd2d(m, x, y);
#pragma unroll
      for (int p = 0; p < 64; ++p) ys[p][threadIdx.x] = y[p >> 3][p & 7] * dm.wy[p];
    }
#if ADCT_SWEEP_PACKED
    if (clip == ADCT_CLIP_NONE) {
      float2 e2[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) e2[i][c] = make_float2(0.0f, 0.0f);
#pragma unroll 1
      for (int zr = 63; zr >= rmin && zr >= 1; --zr) {
        const int pos = c_zz[zr];
        const int k = pos >> 3, l = pos & 7;
        const float cz = ys[pos][threadIdx.x];
        float a[8];
        float2 hl2[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(dm.h[i * 8 + k], cz, -0.0f);
#pragma unroll
        for (int c = 0; c < 4; ++c) hl2[c] = make_float2(dm.h[(2 * c) * 8 + l], dm.h[(2 * c + 1) * 8 + l]);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int c = 0; c < 4; ++c) e2[i][c] = __ffma2_rn(hl2[c], make_float2(a[i], a[i]), e2[i][c]);
        if ((rmask >> zr) & 1ull) {
          float2 sa = make_float2(0.0f, 0.0f), sb = make_float2(0.0f, 0.0f);  // (s0, s1), (s2, s3)
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              if (c & 1) sb = __ffma2_rn(e2[i][c], e2[i][c], sb);
              else sa = __ffma2_rn(e2[i][c], e2[i][c], sa);
            }
          zacc[zr - 1][threadIdx.x] += (sa.x + sa.y) + (sb.x + sb.y);
        }
      }
      continue;
    }
#endif
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) e[i][j] = 0.0f;
#pragma unroll 1
    for (int zr = 63; zr >= rmin && zr >= 1; --zr) {
      const int pos = c_zz[zr];
      const int k = pos >> 3, l = pos & 7;
      const float c = ys[pos][threadIdx.x];
      float a[8], hl[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        a[i] = fmaf(dm.h[i * 8 + k], c, -0.0f);
        hl[i] = dm.h[i * 8 + l];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) e[i][j] = fmaf(hl[j], a[i], e[i][j]);
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

bool launch_sweep_any(bool u8, bool specialized, int clip, cudaStream_t st, const void* src, const adct_geom& g,
                      const KGeom& kg, const DevMat& dm, const FastDiv& dbw, uint64_t rmask, int32_t rmin,
                      double* partial) {
  const int32_t chunks = (int32_t)sweep_chunks(g), bpt = sweep_bpt(g);
  const dim3 grid((unsigned)chunks, (unsigned)g.n_images);
  (void)specialized;
  // c_zz is __constant__ memory of the current device: uploaded once per device
  static std::mutex mu;
  static int8_t state[kMaxDevices] = {};
  if (!once_per_device(mu, state, [] {
        int8_t zz[64];
        for (int z = 0; z < 64; ++z) zz[z] = (int8_t)kZZ.order[z];
        return cudaMemcpyToSymbol(c_zz, zz, sizeof(zz)) == cudaSuccess;
      }))
    return false;
  if (u8)
    fused_sweep_kernel<uint8_t><<<grid, NT, 0, st>>>((const uint8_t*)src, kg, dm, dbw, chunks, bpt, rmask, rmin, clip,
                                                     partial);
  else
    fused_sweep_kernel<int16_t><<<grid, NT, 0, st>>>((const int16_t*)src, kg, dm, dbw, chunks, bpt, rmask, rmin, clip,
                                                     partial);
  return true;
}

}  // namespace adct
