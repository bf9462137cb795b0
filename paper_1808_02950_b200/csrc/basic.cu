// basic.cu — the four calls of the method as separate kernels (§6.1):
//   approx_dct8x8_fwd   B = C_hat A C_hat^T
//   zonal_retain        first r in zig-zag order
//   approx_dct8x8_inv   A = C_hat^T B' C_hat          P:L2237-2242 (C_hat^{-1}: reading A4)
//   psnr_reduce         MSE / PSNR per image
// plus the config-3 forward+quantiser.  One thread owns one 8x8 block; grid-stride loops
// sized in multiples of the SM count.
#include <cmath>
#include <mutex>

#include "adct_host.h"
#include "tma.cuh"

namespace adct {
namespace {

int g_num_sms = 0;
int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

unsigned grid_for(int64_t work, int nt, int per_sm) {
  const int64_t need = (work + nt - 1) / nt;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  return (unsigned)(need < cap ? (need > 0 ? need : 1) : cap);
}

template <typename SrcT>
__device__ __forceinline__ void load_block(const SrcT* __restrict__ src, const KGeom& g, uint32_t b,
                                           const FastDiv& dnbi, const FastDiv& dbw, float (&x)[8][8]) {
  const uint32_t img = fdiv(b, dnbi);
  const uint32_t q = b - img * g.nbi;
  const uint32_t by = fdiv(q, dbw);
  const uint32_t bx = q - by * g.bw;
  const SrcT* p = src + (int64_t)img * g.image_stride + (int64_t)by * 8 * g.row_stride + (int64_t)bx * 8;
#pragma unroll
  for (int i = 0; i < 8; ++i) Src<SrcT>::to_f(Src<SrcT>::load(p + (int64_t)i * g.row_stride), x[i]);
}

// ---- forward -----------------------------------------------------------------------------
template <typename SrcT, typename OutT, class MP>
__global__ void __launch_bounds__(256) fwd_kernel(const SrcT* __restrict__ src, KGeom g, DevMat dm,
                                                  FastDiv dnbi, FastDiv dbw, uint32_t nblocks,
                                                  OutT* __restrict__ coef) {
  const MP m(dm);
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nblocks; b += gridDim.x * blockDim.x) {
    float x[8][8], y[8][8];
    load_block(src, g, b, dnbi, dbw, x);
    fwd2d(m, x, y);
    OutT* o = coef + (int64_t)b * 64;
    if constexpr (sizeof(OutT) == 4 && !std::is_same<OutT, float>::value) {  // int32: exact Y
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int l = 0; l < 8; l += 4) {
          int4 v = make_int4(__float2int_rn(y[k][l]), __float2int_rn(y[k][l + 1]), __float2int_rn(y[k][l + 2]),
                             __float2int_rn(y[k][l + 3]));
          *reinterpret_cast<int4*>(o + k * 8 + l) = v;
        }
    } else if constexpr (std::is_same<OutT, float>::value) {  // B = sb o Y
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int l = 0; l < 8; l += 4) {
          float4 v = make_float4(y[k][l] * dm.sb[k * 8 + l], y[k][l + 1] * dm.sb[k * 8 + l + 1],
                                 y[k][l + 2] * dm.sb[k * 8 + l + 2], y[k][l + 3] * dm.sb[k * 8 + l + 3]);
          *reinterpret_cast<float4*>(o + k * 8 + l) = v;
        }
    } else {  // int16: exact Y (range checked on the host)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        uint4 v;
        v.x = (uint32_t)(uint16_t)__float2int_rn(y[k][0]) | ((uint32_t)(uint16_t)__float2int_rn(y[k][1]) << 16);
        v.y = (uint32_t)(uint16_t)__float2int_rn(y[k][2]) | ((uint32_t)(uint16_t)__float2int_rn(y[k][3]) << 16);
        v.z = (uint32_t)(uint16_t)__float2int_rn(y[k][4]) | ((uint32_t)(uint16_t)__float2int_rn(y[k][5]) << 16);
        v.w = (uint32_t)(uint16_t)__float2int_rn(y[k][6]) | ((uint32_t)(uint16_t)__float2int_rn(y[k][7]) << 16);
        *reinterpret_cast<uint4*>(o + k * 8) = v;
      }
    }
  }
}

// ---- zonal retention ------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) retain_kernel(T* __restrict__ coef, int64_t n_vec, uint64_t keep) {
  constexpr int E = 16 / sizeof(T);  // elements per 16-byte vector
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n_vec; v += (int64_t)gridDim.x * blockDim.x) {
    uint4 d = reinterpret_cast<uint4*>(coef)[v];
    T* e = reinterpret_cast<T*>(&d);
    const int pos0 = (int)((v * E) & 63);
#pragma unroll
    for (int i = 0; i < E; ++i)
      if (!((keep >> (pos0 + i)) & 1ull)) e[i] = T(0);
    reinterpret_cast<uint4*>(coef)[v] = d;
  }
}

// ---- inverse ---------------------------------------------------------------------------------
template <typename OutT>
__device__ __forceinline__ void store_row(OutT* p, const float* x, int clip, float lo, float hi);

template <>
__device__ __forceinline__ void store_row<float>(float* p, const float* x, int clip, float lo, float hi) {
  float v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    v[j] = x[j];
    if (clip != ADCT_CLIP_NONE) v[j] = fminf(fmaxf(v[j], lo), hi);
    if (clip == ADCT_CLIP_ROUND) v[j] = rintf(v[j]);
  }
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}
template <>
__device__ __forceinline__ void store_row<uint8_t>(uint8_t* p, const float* x, int, float, float) {
  uint32_t b[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) b[j] = (uint32_t)rintf(fminf(fmaxf(x[j], 0.0f), 255.0f));
  uint2 v;
  v.x = b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24);
  v.y = b[4] | (b[5] << 8) | (b[6] << 16) | (b[7] << 24);
  *reinterpret_cast<uint2*>(p) = v;
}
template <>
__device__ __forceinline__ void store_row<int16_t>(int16_t* p, const float* x, int, float, float) {
  uint32_t b[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) b[j] = (uint32_t)(uint16_t)(int16_t)rintf(fminf(fmaxf(x[j], -32768.0f), 32767.0f));
  uint4 v;
  v.x = b[0] | (b[1] << 16);
  v.y = b[2] | (b[3] << 16);
  v.z = b[4] | (b[5] << 16);
  v.w = b[6] | (b[7] << 16);
  *reinterpret_cast<uint4*>(p) = v;
}

template <typename CoefT, typename OutT, class MP>
__global__ void __launch_bounds__(256) inv_kernel(const CoefT* __restrict__ coef, KGeom g, DevMat dm,
                                                  FastDiv dnbi, FastDiv dbw, uint32_t nblocks, int clip,
                                                  float lo, float hi, OutT* __restrict__ recon) {
  const MP m(dm);
  constexpr bool kIntIn = !std::is_same<CoefT, float>::value;
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nblocks; b += gridDim.x * blockDim.x) {
    float z[8][8], x[8][8];
    const CoefT* c = coef + (int64_t)b * 64;
    if constexpr (sizeof(CoefT) == 4) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int l = 0; l < 8; l += 4) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(c + k * 8 + l));
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float f = kIntIn ? (float)(int32_t)w[q] : __uint_as_float(w[q]);
            z[k][l + q] = f * (kIntIn ? dm.wy[k * 8 + l + q] : dm.wb[k * 8 + l + q]);
          }
        }
    } else {  // int16
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(c + k * 8));
        float f[8];
        i16row_to_f(v, f);
#pragma unroll
        for (int l = 0; l < 8; ++l) z[k][l] = f[l] * dm.wy[k * 8 + l];
      }
    }
    inv2d<MP, ~0ull>(m, z, x);
    const uint32_t img = fdiv(b, dnbi);
    const uint32_t q = b - img * g.nbi;
    const uint32_t by = fdiv(q, dbw);
    const uint32_t bx = q - by * g.bw;
    OutT* p = recon + (int64_t)img * g.image_stride + (int64_t)by * 8 * g.row_stride + (int64_t)bx * 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) store_row<OutT>(p + (int64_t)i * g.row_stride, x[i], clip, lo, hi);
  }
}

// ---- fused round trip: forward -> zonal retention -> inverse -> reconstruction --------------------
// The composition approx_dct8x8_fwd -> zonal_retain -> approx_dct8x8_inv in one pass (config 5:
// forward + inverse of int16 residual blocks): each block is read once and its reconstruction
// written once; the coefficients never leave registers.  wk[k*8+l] = the inverse weight of the
// coefficient times its zig-zag keep bit (0 for dropped coefficients).
struct Wk {
  float w[64];
};

template <typename SrcT, class MP>
__global__ void __launch_bounds__(256) roundtrip_kernel(const SrcT* __restrict__ src, KGeom g, DevMat dm, Wk wk,
                                                        FastDiv dnbi, FastDiv dbw, uint32_t nblocks, int out_t,
                                                        int clip, float lo, float hi, void* __restrict__ recon) {
  const MP m(dm);
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nblocks; b += gridDim.x * blockDim.x) {
    float x[8][8], y[8][8];
    load_block(src, g, b, dnbi, dbw, x);
    fwd2d(m, x, y);
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int l = 0; l < 8; ++l) y[k][l] *= wk.w[k * 8 + l];
    inv2d<MP, ~0ull>(m, y, x);
    const uint32_t img = fdiv(b, dnbi);
    const uint32_t q = b - img * g.nbi;
    const uint32_t by = fdiv(q, dbw);
    const uint32_t bx = q - by * g.bw;
    const int64_t off = (int64_t)img * g.image_stride + (int64_t)by * 8 * g.row_stride + (int64_t)bx * 8;
    if (out_t == ADCT_F32) {
#pragma unroll
      for (int i = 0; i < 8; ++i) store_row<float>((float*)recon + off + (int64_t)i * g.row_stride, x[i], clip, lo, hi);
    } else if (out_t == ADCT_I16) {
#pragma unroll
      for (int i = 0; i < 8; ++i) store_row<int16_t>((int16_t*)recon + off + (int64_t)i * g.row_stride, x[i], clip, lo, hi);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) store_row<uint8_t>((uint8_t*)recon + off + (int64_t)i * g.row_stride, x[i], clip, lo, hi);
    }
  }
}

// ---- per-image squared error (deterministic two-level reduction) ------------------------------
template <typename T>
__device__ __forceinline__ float sample_at(const T* p) { return (float)*p; }

template <typename OrigT, typename RecT>
__global__ void __launch_bounds__(kRedNT) sse_kernel(const OrigT* __restrict__ orig, const RecT* __restrict__ rec,
                                                     KGeom g, int32_t height, int32_t width, int clip, float lo,
                                                     float hi, int32_t chunks, double* __restrict__ partial) {
  __shared__ double red[kRedNT / 32];
  const uint32_t img = blockIdx.y;
  const int32_t r0 = blockIdx.x * kSseRows;
  double acc = 0.0;
  for (int32_t r = r0; r < r0 + kSseRows && r < height; ++r) {
    const int64_t rowoff = (int64_t)img * g.image_stride + (int64_t)r * g.row_stride;
    for (int32_t c = threadIdx.x; c < width; c += kRedNT) {
      const float xo = (float)orig[rowoff + c];
      float xr = (float)rec[rowoff + c];
      if (clip != ADCT_CLIP_NONE) xr = fminf(fmaxf(xr, lo), hi);
      if (clip == ADCT_CLIP_ROUND) xr = rintf(xr);
      const double d = (double)xo - (double)xr;
      acc = fma(d, d, acc);
    }
  }
  const double tot = block_sum<kRedNT>(acc, red);
  if (threadIdx.x == 0) partial[(int64_t)img * chunks + blockIdx.x] = tot;
}

// one CTA per (image, output): thread t adds chunks t, t + 256, ... in order, then a fixed
// shared-memory tree combines the 256 sums — deterministic, independent of the grid that
// produced the partials.
constexpr int kFinNT = 256;
__global__ void __launch_bounds__(kFinNT) finalize_kernel(const double* __restrict__ partial, int32_t chunks,
                                                          int64_t n_images, int32_t slots, SlotMap slot_of,
                                                          int32_t n_out, double npix, double peak,
                                                          double* __restrict__ sse, double* __restrict__ psnr,
                                                          double scale) {
  __shared__ double red[kFinNT];
  const int64_t img = blockIdx.x;
  const int32_t o = blockIdx.y;
  const int32_t s = slot_of.s[o];
  double acc = 0.0;
  if (s >= 0)
    for (int32_t c = threadIdx.x; c < chunks; c += kFinNT) acc += partial[((int64_t)img * chunks + c) * slots + s];
  red[threadIdx.x] = acc;
  __syncthreads();
#pragma unroll
  for (int w = kFinNT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double tot = red[0] * scale;
    const int64_t t = img * n_out + o;
    sse[t] = tot;
    if (psnr) psnr[t] = tot == 0.0 ? INFINITY : 10.0 * log10(peak * peak / (tot / npix));
  }
}

// ---- SSIM (reading A18: 8x8 uniform windows, K1 = 0.01, K2 = 0.03, L = peak) -------------------
// One CTA per 32x32 tile of window positions: the 39x39 samples of both images are staged in
// shared memory, horizontal 8-sums of x, y, x^2, y^2, xy are formed per row, then vertical
// 8-sums per position, all in fp64; per-CTA sums of the window SSIMs are reduced in a fixed
// order and finalize_kernel averages an image's tiles in index order.
constexpr int kSsimT = 32, kSsimIn = kSsimT + 7, kSsimNT = 256, kSsimSeg = 4;  // positions per running-sum segment

// the window SSIMs of one 32x32 tile of positions from the 39x39 samples in sx, sy
__device__ __forceinline__ double ssim_tile_compute(const float* sx, const float* sy, double* hs, int32_t y0,
                                                    int32_t x0, int32_t height, int32_t width, double c1, double c2) {
  // horizontal 8-sums as running sums along row segments of 8 positions
  for (int it = threadIdx.x; it < kSsimIn * (kSsimT / kSsimSeg); it += kSsimNT) {
    const int r = it / (kSsimT / kSsimSeg), c0 = (it % (kSsimT / kSsimSeg)) * kSsimSeg;
    const float* px = sx + r * 40;
    const float* py = sy + r * 40;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double a = px[c0 + k], b = py[c0 + k];
      s0 += a;
      s1 += b;
      s2 = fma(a, a, s2);
      s3 = fma(b, b, s3);
      s4 = fma(a, b, s4);
    }
#pragma unroll
    for (int c = c0; c < c0 + kSsimSeg; ++c) {
      if (c > c0) {  // slide the window by one: add sample c+7, drop sample c-1
        const double a = px[c + 7], b = py[c + 7], a0 = px[c - 1], b0 = py[c - 1];
        s0 += a - a0;
        s1 += b - b0;
        s2 += fma(a, a, -a0 * a0);
        s3 += fma(b, b, -b0 * b0);
        s4 += fma(a, b, -a0 * b0);
      }
      const int i = r * kSsimT + c;
      hs[0 * kSsimIn * kSsimT + i] = s0;
      hs[1 * kSsimIn * kSsimT + i] = s1;
      hs[2 * kSsimIn * kSsimT + i] = s2;
      hs[3 * kSsimIn * kSsimT + i] = s3;
      hs[4 * kSsimIn * kSsimT + i] = s4;
    }
  }
  __syncthreads();
  // vertical 8-sums as running sums down column segments of 8 positions, then the window SSIM
  double acc = 0.0;
  for (int it = threadIdx.x; it < kSsimT * (kSsimT / kSsimSeg); it += kSsimNT) {
    const int c = it % kSsimT, r0 = (it / kSsimT) * kSsimSeg;
    double v[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) t += hs[q * kSsimIn * kSsimT + (r0 + k) * kSsimT + c];
      v[q] = t;
    }
#pragma unroll
    for (int r = r0; r < r0 + kSsimSeg; ++r) {
      if (r > r0) {
#pragma unroll
        for (int q = 0; q < 5; ++q)
          v[q] += hs[q * kSsimIn * kSsimT + (r + 7) * kSsimT + c] - hs[q * kSsimIn * kSsimT + (r - 1) * kSsimT + c];
      }
      if (y0 + r + 8 > height || x0 + c + 8 > width) continue;
      const double mx = v[0] * (1.0 / 64.0), my = v[1] * (1.0 / 64.0);
      const double vx = v[2] * (1.0 / 64.0) - mx * mx, vy = v[3] * (1.0 / 64.0) - my * my;
      const double cxy = v[4] * (1.0 / 64.0) - mx * my;
      acc += ((2.0 * mx * my + c1) * (2.0 * cxy + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2));
    }
  }
  return acc;
}

template <typename OrigT, typename RecT>
__global__ void __launch_bounds__(kSsimNT) ssim_kernel(const OrigT* __restrict__ orig, const RecT* __restrict__ rec,
                                                       KGeom g, int32_t height, int32_t width, int32_t ntx,
                                                       int32_t tiles, int clip, float lo, float hi, double c1,
                                                       double c2, double* __restrict__ partial) {
  extern __shared__ double ssm[];
  float* sx = reinterpret_cast<float*>(ssm);                 // [39][40]
  float* sy = sx + kSsimIn * 40;                             // [39][40]
  double* hs = ssm + (kSsimIn * 40 * 2 + 1) / 2;             // [5][39][32]
  __shared__ double red[kSsimNT / 32];
  const uint32_t img = blockIdx.y;
  const int32_t tx = (int32_t)blockIdx.x % ntx, ty = (int32_t)blockIdx.x / ntx;
  const int32_t x0 = tx * kSsimT, y0 = ty * kSsimT;
  const int64_t ibase = (int64_t)img * g.image_stride;
  for (int i = threadIdx.x; i < kSsimIn * kSsimIn; i += kSsimNT) {
    const int r = i / kSsimIn, c = i % kSsimIn;
    const int yy = y0 + r, xx = x0 + c;
    float a = 0.0f, b = 0.0f;
    if (yy < height && xx < width) {
      const int64_t off = ibase + (int64_t)yy * g.row_stride + xx;
      a = (float)orig[off];
      b = (float)rec[off];
      if (clip != ADCT_CLIP_NONE) b = fminf(fmaxf(b, lo), hi);
      if (clip == ADCT_CLIP_ROUND) b = rintf(b);
    }
    sx[r * 40 + c] = a;
    sy[r * 40 + c] = b;
  }
  __syncthreads();
  const double acc = ssim_tile_compute(sx, sy, hs, y0, x0, height, width, c1, c2);
  const double tot = block_sum<kSsimNT>(acc, red);
  if (threadIdx.x == 0) partial[(int64_t)img * tiles + blockIdx.x] = tot;
}

// Persistent variant for u8 originals and fp32 reconstructions: each CTA walks its tiles with a
// 2-slot TMA ring (the 48x39 u8 and 40x39 fp32 boxes of the next tile land while the current one
// is computed), so the global-load latency that bounds ssim_kernel is hidden.
constexpr int kSsimBoxO = 48, kSsimBoxR = 40;  // box widths: 16-byte multiples >= 39
constexpr uint32_t kSsimStageO = kSsimIn * kSsimBoxO, kSsimStageR = kSsimIn * kSsimBoxR * 4;
constexpr uint32_t kSsimStage = ((kSsimStageO + 127) / 128 * 128 + kSsimStageR + 127) / 128 * 128;  // TMA
// destinations are 128-byte aligned

__global__ void __launch_bounds__(kSsimNT) ssim_tma_kernel(const __grid_constant__ CUtensorMap to,
                                                           const __grid_constant__ CUtensorMap tr, int32_t height,
                                                           int32_t width, int32_t ntx, int32_t tiles,
                                                           int64_t n_tiles, int clip, float lo, float hi, double c1,
                                                           double c2, double* __restrict__ partial) {
  extern __shared__ __align__(128) uint8_t sraw[];
  uint8_t* base = reinterpret_cast<uint8_t*>(((uintptr_t)sraw + 127) & ~(uintptr_t)127);
  uint8_t* stage = base;                                        // 2 x kSsimStage
  float* sx = reinterpret_cast<float*>(base + 2 * kSsimStage);  // [39][40]
  float* sy = sx + kSsimIn * 40;
  double* hs = reinterpret_cast<double*>(sy + kSsimIn * 40);   // [5][39][32]
  uint64_t* full = reinterpret_cast<uint64_t*>(hs + 5 * kSsimIn * kSsimT);
  __shared__ double red[kSsimNT / 32];
  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t t, int slot) {
    const int32_t img = (int32_t)(t / tiles), tl = (int32_t)(t % tiles);
    const int32_t x0 = (tl % ntx) * kSsimT, y0 = (tl / ntx) * kSsimT;
    uint8_t* st = stage + slot * kSsimStage;
    mbar_arrive_expect_tx(&full[slot], kSsimStageO + kSsimStageR);
    tma_load_3d(smem_u32(st), &to, x0, y0, img, smem_u32(&full[slot]));
    tma_load_3d(smem_u32(st + (kSsimStageO + 127) / 128 * 128), &tr, x0, y0, img, smem_u32(&full[slot]));
  };
  if (threadIdx.x == 0 && (int64_t)blockIdx.x < n_tiles) issue(blockIdx.x, 0);
  uint32_t k = 0;
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
    const int slot = (int)(k & 1u);
    mbar_wait(&full[slot], (k >> 1) & 1u);
    const uint8_t* so = stage + slot * kSsimStage;
    const float* sr = reinterpret_cast<const float*>(so + (kSsimStageO + 127) / 128 * 128);
    for (int i = threadIdx.x; i < kSsimIn * kSsimIn; i += kSsimNT) {
      const int r = i / kSsimIn, c = i % kSsimIn;
      float b = sr[r * kSsimBoxR + c];
      if (clip != ADCT_CLIP_NONE) b = fminf(fmaxf(b, lo), hi);
      if (clip == ADCT_CLIP_ROUND) b = rintf(b);
      sx[r * 40 + c] = (float)so[r * kSsimBoxO + c];
      sy[r * 40 + c] = b;
    }
    __syncthreads();  // the slot is consumed: prefetch the CTA's next tile into the other slot
    if (threadIdx.x == 0 && t + gridDim.x < n_tiles) {
      fence_proxy_async();
      issue(t + gridDim.x, slot ^ 1);
    }
    const int32_t img = (int32_t)(t / tiles), tl = (int32_t)(t % tiles);
    const double acc =
        ssim_tile_compute(sx, sy, hs, (tl / ntx) * kSsimT, (tl % ntx) * kSsimT, height, width, c1, c2);
    const double tot = block_sum<kSsimNT>(acc, red);  // also orders this tile's reads before the next
    if (threadIdx.x == 0) partial[(int64_t)img * tiles + tl] = tot;
  }
}

constexpr size_t kSsimTmaSmem = 128 + 2 * (size_t)kSsimStage + (size_t)kSsimIn * 40 * 4 * 2 +
                                (size_t)5 * kSsimIn * kSsimT * 8 + 16;

constexpr size_t kSsimSmem = (size_t)(kSsimIn * 40 * 2 + 1) / 2 * 8 + (size_t)5 * kSsimIn * kSsimT * 8;

}  // namespace

int64_t ssim_tiles(const adct_geom& g) {
  if (g.height < 8 || g.width < 8) return 0;
  return (int64_t)((g.width - 7 + kSsimT - 1) / kSsimT) * ((g.height - 7 + kSsimT - 1) / kSsimT);
}

void launch_finalize_scaled(const double* partial, int32_t chunks, int64_t n_images, double scale, double* out,
                            cudaStream_t st) {
  if (n_images == 0) return;
  SlotMap sm{};
  finalize_kernel<<<dim3((unsigned)n_images, 1u), kFinNT, 0, st>>>(partial, chunks, n_images, 1, sm, 1, 1.0, 1.0, out,
                                                                   nullptr, scale);
  count_launch();
}

// exported to fused.cu
void launch_finalize(const double* partial, int32_t chunks, int64_t n_images, int32_t slots, const SlotMap& slot_of,
                     int32_t n_out, double npix, double peak, double* sse, double* psnr, cudaStream_t st) {
  if (n_images * n_out == 0) return;
  finalize_kernel<<<dim3((unsigned)n_images, (unsigned)n_out), kFinNT, 0, st>>>(partial, chunks, n_images, slots,
                                                                                slot_of, n_out, npix, peak, sse, psnr,
                                                                                1.0);
  count_launch();
}

}  // namespace adct

namespace adct {
bool roundtrip_blockmajor(const adct_matrix* m, const void* src, const adct_geom& g, const float* wk_in, void* recon,
                          adct_dtype recon_t, adct_clip clip, float lo, float hi, cudaStream_t st, adct_status* status);
}
using namespace adct;

namespace {

template <typename SrcT, typename OutT>
adct_status launch_fwd(const adct_matrix* m, const void* src, const adct_geom& g, void* coef, cudaStream_t st) {
  const KGeom kg = make_kgeom(g);
  const uint32_t nb = (uint32_t)(g.n_images * kg.nbi);
  if (nb == 0) return ADCT_OK;
  const FastDiv dnbi = make_fastdiv(kg.nbi), dbw = make_fastdiv(kg.bw);
  const unsigned grid = grid_for(nb, 256, 8);
  if (m->specialized)
    fwd_kernel<SrcT, OutT, T1Mat><<<grid, 256, 0, st>>>((const SrcT*)src, kg, m->dev, dnbi, dbw, nb, (OutT*)coef);
  else
    fwd_kernel<SrcT, OutT, RtMat><<<grid, 256, 0, st>>>((const SrcT*)src, kg, m->dev, dnbi, dbw, nb, (OutT*)coef);
  count_launch();
  return launch_status();
}

template <typename CoefT, typename OutT>
adct_status launch_inv(const adct_matrix* m, const void* coef, const adct_geom& g, void* recon, adct_clip clip,
                       float lo, float hi, cudaStream_t st) {
  const KGeom kg = make_kgeom(g);
  const uint32_t nb = (uint32_t)(g.n_images * kg.nbi);
  if (nb == 0) return ADCT_OK;
  const FastDiv dnbi = make_fastdiv(kg.nbi), dbw = make_fastdiv(kg.bw);
  const unsigned grid = grid_for(nb, 256, 8);
  if (m->specialized)
    inv_kernel<CoefT, OutT, T1Mat><<<grid, 256, 0, st>>>((const CoefT*)coef, kg, m->dev, dnbi, dbw, nb, (int)clip,
                                                         lo, hi, (OutT*)recon);
  else
    inv_kernel<CoefT, OutT, RtMat><<<grid, 256, 0, st>>>((const CoefT*)coef, kg, m->dev, dnbi, dbw, nb, (int)clip,
                                                         lo, hi, (OutT*)recon);
  count_launch();
  return launch_status();
}

template <typename OrigT, typename RecT>
void launch_sse(const void* orig, const void* rec, const adct_geom& g, int clip, float lo, float hi, double* partial,
                int32_t chunks, cudaStream_t st) {
  dim3 grid((unsigned)chunks, (unsigned)g.n_images);
  sse_kernel<OrigT, RecT><<<grid, kRedNT, 0, st>>>((const OrigT*)orig, (const RecT*)rec, make_kgeom(g), g.height,
                                                   g.width, clip, lo, hi, chunks, partial);
  count_launch();
}

}  // namespace

extern "C" {

adct_status approx_dct8x8_fwd(const adct_matrix* m, const void* src, adct_dtype src_t, adct_geom g, void* coef,
                              adct_dtype coef_t, void* stream) {
  if (!m || !src || !coef) return ADCT_E_INVALID_ARGUMENT;
  if (adct_status s = check_geom(g)) return s;
  if (src_t != ADCT_U8 && src_t != ADCT_I16) return ADCT_E_INVALID_ARGUMENT;
  if (coef_t != ADCT_I32 && coef_t != ADCT_I16 && coef_t != ADCT_F32) return ADCT_E_INVALID_ARGUMENT;
  if (!aligned(src, src_t == ADCT_U8 ? 8 : 16) || !aligned(coef, 16)) return ADCT_E_ALIGNMENT;
  if (coef_t != ADCT_F32) {
    if (!m->is_int) return ADCT_E_OVERFLOW;
    const int64_t bound = src_t == ADCT_U8 ? m->max_u8 : m->max_i16;
    if (coef_t == ADCT_I16 && bound > 32767) return ADCT_E_OVERFLOW;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (src_t == ADCT_U8) {
    if (coef_t == ADCT_I32) return launch_fwd<uint8_t, int32_t>(m, src, g, coef, st);
    if (coef_t == ADCT_I16) return launch_fwd<uint8_t, int16_t>(m, src, g, coef, st);
    return launch_fwd<uint8_t, float>(m, src, g, coef, st);
  }
  if (coef_t == ADCT_I32) return launch_fwd<int16_t, int32_t>(m, src, g, coef, st);
  if (coef_t == ADCT_I16) return launch_fwd<int16_t, int16_t>(m, src, g, coef, st);
  return launch_fwd<int16_t, float>(m, src, g, coef, st);
}

adct_status zonal_retain(void* coef, adct_dtype coef_t, int64_t n_blocks, int32_t r, void* stream) {
  if (!coef || n_blocks < 0) return ADCT_E_INVALID_ARGUMENT;
  if (r < 1 || r > 64) return ADCT_E_INVALID_ARGUMENT;
  if (coef_t != ADCT_I32 && coef_t != ADCT_I16 && coef_t != ADCT_F32) return ADCT_E_INVALID_ARGUMENT;
  if (!aligned(coef, 16)) return ADCT_E_ALIGNMENT;
  if (n_blocks == 0) return ADCT_OK;
  const uint64_t keep = keep_mask(r);
  cudaStream_t st = (cudaStream_t)stream;
  const int esz = coef_t == ADCT_I16 ? 2 : 4;
  const int64_t n_vec = n_blocks * 64 * esz / 16;
  const unsigned grid = grid_for(n_vec, 256, 16);
  if (esz == 2)
    retain_kernel<int16_t><<<grid, 256, 0, st>>>((int16_t*)coef, n_vec, keep);
  else
    retain_kernel<int32_t><<<grid, 256, 0, st>>>((int32_t*)coef, n_vec, keep);
  count_launch();
  return launch_status();
}

adct_status approx_dct8x8_inv(const adct_matrix* m, const void* coef, adct_dtype coef_t, adct_geom g, void* recon,
                              adct_dtype recon_t, adct_clip clip, void* stream) {
  if (!m || !coef || !recon) return ADCT_E_INVALID_ARGUMENT;
  if (adct_status s = check_geom(g)) return s;
  if (coef_t != ADCT_I32 && coef_t != ADCT_I16 && coef_t != ADCT_F32) return ADCT_E_INVALID_ARGUMENT;
  if (coef_t != ADCT_F32 && !m->is_int) return ADCT_E_INVALID_ARGUMENT;
  if (clip != ADCT_CLIP_NONE && clip != ADCT_CLIP && clip != ADCT_CLIP_ROUND) return ADCT_E_INVALID_ARGUMENT;
  if (recon_t == ADCT_U8 || recon_t == ADCT_I16) {
    if (clip != ADCT_CLIP_ROUND) return ADCT_E_INVALID_ARGUMENT;
  } else if (recon_t != ADCT_F32) {
    return ADCT_E_INVALID_ARGUMENT;
  }
  const int rb = recon_t == ADCT_U8 ? 8 : 16;
  if (!aligned(coef, 16) || !aligned(recon, rb)) return ADCT_E_ALIGNMENT;
  // F32 reconstructions clip to the range of 8-bit images (the paper's setting)
  const float lo = recon_t == ADCT_I16 ? -32768.0f : 0.0f, hi = recon_t == ADCT_I16 ? 32767.0f : 255.0f;
  cudaStream_t st = (cudaStream_t)stream;
#define ADCT_INV_DISPATCH(CT)                                                                  \
  if (recon_t == ADCT_F32) return launch_inv<CT, float>(m, coef, g, recon, clip, lo, hi, st);  \
  if (recon_t == ADCT_U8) return launch_inv<CT, uint8_t>(m, coef, g, recon, clip, lo, hi, st); \
  return launch_inv<CT, int16_t>(m, coef, g, recon, clip, lo, hi, st);
  if (coef_t == ADCT_I32) { ADCT_INV_DISPATCH(int32_t) }
  if (coef_t == ADCT_I16) { ADCT_INV_DISPATCH(int16_t) }
  ADCT_INV_DISPATCH(float)
#undef ADCT_INV_DISPATCH
}

adct_status approx_dct8x8_roundtrip(const adct_matrix* m, const void* src, adct_dtype src_t, adct_geom g, int32_t r,
                                    void* recon, adct_dtype recon_t, adct_clip clip, void* stream) {
  if (!m || !src || !recon) return ADCT_E_INVALID_ARGUMENT;
  if (adct_status s = check_geom(g)) return s;
  if (src_t != ADCT_U8 && src_t != ADCT_I16) return ADCT_E_INVALID_ARGUMENT;
  if (r < 1 || r > 64) return ADCT_E_INVALID_ARGUMENT;
  if (clip != ADCT_CLIP_NONE && clip != ADCT_CLIP && clip != ADCT_CLIP_ROUND) return ADCT_E_INVALID_ARGUMENT;
  if (recon_t == ADCT_U8 || recon_t == ADCT_I16) {
    if (clip != ADCT_CLIP_ROUND) return ADCT_E_INVALID_ARGUMENT;
  } else if (recon_t != ADCT_F32) {
    return ADCT_E_INVALID_ARGUMENT;
  }
  if (!aligned(src, src_t == ADCT_U8 ? 8 : 16) || !aligned(recon, recon_t == ADCT_U8 ? 8 : 16)) return ADCT_E_ALIGNMENT;
  const KGeom kg = make_kgeom(g);
  const uint32_t nb = (uint32_t)(g.n_images * kg.nbi);
  if (nb == 0) return ADCT_OK;
  Wk wk;
  const uint64_t keep = keep_mask(r);
  for (int p = 0; p < 64; ++p) wk.w[p] = ((keep >> p) & 1ull) ? (m->is_int ? m->dev.wy[p] : m->dev.wb[p]) : 0.0f;
  const float lo = src_t == ADCT_U8 ? 0.0f : -32768.0f, hi = src_t == ADCT_U8 ? 255.0f : 32767.0f;
  cudaStream_t st = (cudaStream_t)stream;
  if (src_t == ADCT_I16) {  // block-major int16 stacks (config 5): TMA-streamed kernel
    adct_status bs = ADCT_OK;
    if (roundtrip_blockmajor(m, src, g, wk.w, recon, recon_t, clip, lo, hi, st, &bs)) return bs;
  }
  const FastDiv dnbi = make_fastdiv(kg.nbi), dbw = make_fastdiv(kg.bw);
  const unsigned grid = grid_for(nb, 256, 8);
#define ADCT_RT(T, MP)                                                                                       \
  roundtrip_kernel<T, MP><<<grid, 256, 0, st>>>((const T*)src, kg, m->dev, wk, dnbi, dbw, nb, (int)recon_t, \
                                                (int)clip, lo, hi, recon)
  if (src_t == ADCT_U8) {
    if (m->specialized) ADCT_RT(uint8_t, T1Mat); else ADCT_RT(uint8_t, RtMat);
  } else {
    if (m->specialized) ADCT_RT(int16_t, T1Mat); else ADCT_RT(int16_t, RtMat);
  }
#undef ADCT_RT
  count_launch();
  return launch_status();
}

adct_status ssim_reduce(const void* orig, adct_dtype orig_t, const void* recon, adct_dtype recon_t, adct_geom g,
                        double peak, adct_clip clip, double* ssim, void* workspace, size_t workspace_bytes,
                        void* stream) {
  if (!orig || !recon || !ssim) return ADCT_E_INVALID_ARGUMENT;
  if (adct_status s = check_geom(g)) return s;
  if (orig_t != ADCT_U8 && orig_t != ADCT_I16) return ADCT_E_INVALID_ARGUMENT;
  if (recon_t != ADCT_U8 && recon_t != ADCT_I16 && recon_t != ADCT_F32) return ADCT_E_INVALID_ARGUMENT;
  if (clip != ADCT_CLIP_NONE && clip != ADCT_CLIP && clip != ADCT_CLIP_ROUND) return ADCT_E_INVALID_ARGUMENT;
  if (!(peak > 0.0)) return ADCT_E_INVALID_ARGUMENT;
  if (!workspace || workspace_bytes < adct_workspace_bytes(g, 1)) return ADCT_E_WORKSPACE;
  if (g.n_images == 0) return ADCT_OK;
  if (g.n_images > 65535) return ADCT_E_INVALID_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  const KGeom kg = make_kgeom(g);
  const int32_t ntx = (g.width - 7 + kSsimT - 1) / kSsimT;
  const int32_t tiles = (int32_t)ssim_tiles(g);
  const float lo = 0.0f, hi = (float)peak;  // clip range of the reconstruction: [0, peak]
  const double c1 = (0.01 * peak) * (0.01 * peak), c2 = (0.03 * peak) * (0.03 * peak);
  double* partial = (double*)workspace;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(ssim_kernel<uint8_t, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSsimSmem);
    cudaFuncSetAttribute(ssim_kernel<uint8_t, uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSsimSmem);
    cudaFuncSetAttribute(ssim_kernel<uint8_t, int16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSsimSmem);
    cudaFuncSetAttribute(ssim_kernel<int16_t, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSsimSmem);
    cudaFuncSetAttribute(ssim_kernel<int16_t, uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSsimSmem);
    cudaFuncSetAttribute(ssim_kernel<int16_t, int16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSsimSmem);
  });
  if (orig_t == ADCT_U8 && recon_t == ADCT_F32 && g.row_stride % 16 == 0 &&
      (g.n_images == 1 || g.image_stride % 16 == 0) && aligned(orig, 16) && aligned(recon, 16)) {
    auto enc = tmap_encoder();
    CUtensorMap to, tr;
    const cuuint64_t dims[3] = {(cuuint64_t)g.width, (cuuint64_t)g.height, (cuuint64_t)g.n_images};
    const int64_t istr = g.n_images > 1 ? g.image_stride : (int64_t)g.height * g.row_stride;
    const cuuint64_t so[2] = {(cuuint64_t)g.row_stride, (cuuint64_t)istr};
    const cuuint64_t sr[2] = {(cuuint64_t)g.row_stride * 4, (cuuint64_t)istr * 4};
    const cuuint32_t bo[3] = {(cuuint32_t)kSsimBoxO, (cuuint32_t)kSsimIn, 1}, br[3] = {(cuuint32_t)kSsimBoxR, (cuuint32_t)kSsimIn, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    if (enc &&
        enc(&to, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(orig), dims, so, bo, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
            CUDA_SUCCESS &&
        enc(&tr, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(recon), dims, sr, br, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
      static std::once_flag once_tma;
      std::call_once(once_tma, [] {
        cudaFuncSetAttribute(ssim_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSsimTmaSmem);
      });
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int64_t n_tiles = (int64_t)tiles * g.n_images;
      const int64_t cap = (int64_t)sms * 2;
      ssim_tma_kernel<<<(unsigned)(n_tiles < cap ? n_tiles : cap), kSsimNT, kSsimTmaSmem, st>>>(
          to, tr, g.height, g.width, ntx, tiles, n_tiles, (int)clip, lo, hi, c1, c2, partial);
      count_launch();
      if (adct_status e = launch_status()) return e;
      const double nwin = (double)(g.height - 7) * (double)(g.width - 7);
      launch_finalize_scaled(partial, tiles, g.n_images, 1.0 / nwin, ssim, st);
      return launch_status();
    }
  }
  const dim3 grid((unsigned)tiles, (unsigned)g.n_images);
#define ADCT_SSIM(OT, RT)                                                                                      \
  ssim_kernel<OT, RT><<<grid, kSsimNT, kSsimSmem, st>>>((const OT*)orig, (const RT*)recon, kg, g.height, g.width, \
                                                        ntx, tiles, (int)clip, lo, hi, c1, c2, partial)
  if (orig_t == ADCT_U8) {
    if (recon_t == ADCT_F32) ADCT_SSIM(uint8_t, float); else if (recon_t == ADCT_U8) ADCT_SSIM(uint8_t, uint8_t);
    else ADCT_SSIM(uint8_t, int16_t);
  } else {
    if (recon_t == ADCT_F32) ADCT_SSIM(int16_t, float); else if (recon_t == ADCT_U8) ADCT_SSIM(int16_t, uint8_t);
    else ADCT_SSIM(int16_t, int16_t);
  }
#undef ADCT_SSIM
  count_launch();
  if (adct_status e = launch_status()) return e;
  const double nwin = (double)(g.height - 7) * (double)(g.width - 7);
  launch_finalize_scaled(partial, tiles, g.n_images, 1.0 / nwin, ssim, st);
  return launch_status();
}

adct_status psnr_reduce(const void* orig, adct_dtype orig_t, const void* recon, adct_dtype recon_t, adct_geom g,
                        double peak, adct_clip clip, double* sse, double* psnr, void* workspace,
                        size_t workspace_bytes, void* stream) {
  if (!orig || !recon || !sse) return ADCT_E_INVALID_ARGUMENT;
  if (adct_status s = check_geom(g)) return s;
  if (orig_t != ADCT_U8 && orig_t != ADCT_I16) return ADCT_E_INVALID_ARGUMENT;
  if (recon_t != ADCT_U8 && recon_t != ADCT_I16 && recon_t != ADCT_F32) return ADCT_E_INVALID_ARGUMENT;
  if (!(peak > 0.0)) return ADCT_E_INVALID_ARGUMENT;
  if (!workspace || workspace_bytes < adct_workspace_bytes(g, 1)) return ADCT_E_WORKSPACE;
  if (g.n_images == 0) return ADCT_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int32_t chunks = (int32_t)sse_chunks(g);
  double* partial = (double*)workspace;
  const float lo = orig_t == ADCT_U8 ? 0.0f : -32768.0f, hi = orig_t == ADCT_U8 ? 255.0f : 32767.0f;
  const int c = (int)clip;
  if (orig_t == ADCT_U8) {
    if (recon_t == ADCT_F32) launch_sse<uint8_t, float>(orig, recon, g, c, lo, hi, partial, chunks, st);
    else if (recon_t == ADCT_U8) launch_sse<uint8_t, uint8_t>(orig, recon, g, c, lo, hi, partial, chunks, st);
    else launch_sse<uint8_t, int16_t>(orig, recon, g, c, lo, hi, partial, chunks, st);
  } else {
    if (recon_t == ADCT_F32) launch_sse<int16_t, float>(orig, recon, g, c, lo, hi, partial, chunks, st);
    else if (recon_t == ADCT_U8) launch_sse<int16_t, uint8_t>(orig, recon, g, c, lo, hi, partial, chunks, st);
    else launch_sse<int16_t, int16_t>(orig, recon, g, c, lo, hi, partial, chunks, st);
  }
  SlotMap sm{};
  launch_finalize(partial, chunks, g.n_images, 1, sm, 1, (double)g.height * g.width, peak, sse, psnr, st);
  return launch_status();
}

}  // extern "C"
