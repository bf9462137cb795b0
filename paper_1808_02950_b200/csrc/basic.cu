// basic.cu — the four calls of the method as separate kernels (§6.1):
//   approx_dct8x8_fwd   B = C_hat A C_hat^T
//   zonal_retain        first r in zig-zag order
//   approx_dct8x8_inv   A = C_hat^T B' C_hat          P:L2237-2242 (C_hat^{-1}: reading A4)
//   psnr_reduce         MSE / PSNR per image
// plus the config-3 forward+quantiser.  One thread owns one 8x8 block; grid-stride loops
// sized in multiples of the SM count.
#include <cmath>
#include <mutex>
#include <type_traits>

#include "adct_host.h"
#include "packed.cuh"

// ADCT_RT_PACKED: the round trips of roundtrip_kernel and ssim_fused_kernel on column pairs with
// packed fp32 (packed.cuh); 0 = the scalar networks (A/B)
#ifndef ADCT_RT_PACKED
#define ADCT_RT_PACKED 1
#endif
// the fused SSIM kernel keeps the scalar round trip: packed, it needs 136 registers instead of
// 128 and ran 6.59 -> 7.06 ms per 128 4K frames (occupancy); the reconstruction is the same
#ifndef ADCT_SF_PACKED
#define ADCT_SF_PACKED 0
#endif

namespace adct {

int device_sms() {
  static std::mutex mu;
  static int cache[kMaxDevices] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 148;
  std::lock_guard<std::mutex> lk(mu);
  if (cache[dev] <= 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

namespace {

int num_sms() { return device_sms(); }

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
    float x[8][8];
    load_block(src, g, b, dnbi, dbw, x);
#if ADCT_RT_PACKED
    {
      float2 x2[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) x2[i][c] = pk(x[i][2 * c], x[i][2 * c + 1]);
      roundtrip2d_p(m, x2, wk.w);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          x[i][2 * c] = x2[i][c].x;
          x[i][2 * c + 1] = x2[i][c].y;
        }
    }
#else
    {
      float y[8][8];
      fwd2d(m, x, y);
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int l = 0; l < 8; ++l) y[k][l] *= wk.w[k * 8 + l];
      inv2d<MP, ~0ull>(m, y, x);
    }
#endif
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
  pdl_launch_dependents();
  pdl_wait();  // the kernel that wrote the partials has completed
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
// One warp per (image, band of kSsTY window rows, strip of 25 window columns): lane l owns input
// column x0 + l and walks down the band's kSsTY + 7 input rows with vertical running 8-sums of
// x, y, x^2, y^2, xy held in registers (the previous 8 rows stay in a register ring, so each
// row is loaded once); the 8-wide horizontal window sums are three shuffle-add steps across
// lanes l..l+7, so lanes 0..24 each own one window per row.  No shared memory, no barriers;
// rows are prefetched one 8-row group ahead.  Sums of a u8 original are exact in fp32 (integers
// < 2^24); the rest is fp64.  The window SSIM is evaluated on sums scaled by 64^2:
//   SSIM = (2P + 4096 C1)(128 S_xy - 2P + 4096 C2) / ((Q + 4096 C1)(64 (S_xx + S_yy) - Q + 4096 C2)),
//   P = S_x S_y, Q = S_x^2 + S_y^2,
// the definition's mu = S/64, sigma^2 = S_xx/64 - mu^2, sigma_xy = S_xy/64 - mu_x mu_y
// multiplied through.  Each warp's windows are summed in a fixed shuffle tree and
// finalize_kernel adds an image's warps in index order.
constexpr int kSsOut = 25, kSsTY = 64, kSsNT = 32;  // one warp per CTA: the control flow is
// provably warp-uniform (blockIdx only), so the shuffles need no re-convergence code

// Sums of x and x^2: fp32 for a u8 original (integers < 2^24: exact), fp64 for int16.
template <typename OrigT>
using SsAcc = std::conditional_t<sizeof(OrigT) == 1, float, double>;

template <typename T>
__device__ __forceinline__ T win8(T v) {  // lane l: v_l + ... + v_{l+7} in a fixed order
  v += __shfl_down_sync(0xffffffffu, v, 1);
  v += __shfl_down_sync(0xffffffffu, v, 2);
  v += __shfl_down_sync(0xffffffffu, v, 4);
  return v;
}

// n / d for d > 0 (the SSIM denominator is >= 4096^2 C1 C2): MUFU reciprocal seed and two
// Newton steps, then one product -- within 2 ulp, no slow-path branch of the IEEE division
__device__ __forceinline__ double ss_div(double n, double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  return n * r;
}

template <typename OrigT, typename RecT>
struct SsGroup {  // one lane's raw samples of 8 consecutive rows (converted when used, so the
  OrigT a[8];     // loads of the prefetched group have a whole group of work to land)
  RecT b[8];
};

template <typename Acc>
struct SsState {
  Acc A, AA;          // vertical 8-sums of x, x^2 (the lane's column)
  double B, BB, AB;   // ... of y, y^2, xy
  double acc;         // the lane's window SSIMs
};

template <typename OrigT, typename RecT>
__device__ __forceinline__ void ss_load(SsGroup<OrigT, RecT>& gr, const OrigT* po, const RecT* pr, int64_t rs, int r0,
                                        int nin, bool col_ok) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const bool ok = col_ok && r0 + k < nin;
    gr.a[k] = ok ? __ldg(po + k * rs) : (OrigT)0;
    gr.b[k] = ok ? __ldg(pr + k * rs) : (RecT)0;
  }
}

// rows 8 gi .. 8 gi + 7: add row r, drop row r - 8 (the previous group's slot), and for r >= 7
// evaluate the windows whose top row is r - 7.  Padding rows / columns are 0 before and after
// the clip (they only reach windows that are not counted).
template <int CLIP, typename Acc, typename OrigT, typename RecT>
__device__ __forceinline__ void ss_group(SsState<Acc>& s, const SsGroup<OrigT, RecT>& cur,
                                         const SsGroup<OrigT, RecT>& prev, int gi, int nout, bool win_ok, float lo,
                                         float hi, double c1s, double c2s) {
  auto y_of = [&](RecT v) {
    float b = (float)v;
    if constexpr (CLIP != ADCT_CLIP_NONE) b = fminf(fmaxf(b, lo), hi);
    if constexpr (CLIP == ADCT_CLIP_ROUND && std::is_same_v<RecT, float>) b = rintf(b);
    return (double)b;
  };
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const Acc an = (Acc)cur.a[k], ao = (Acc)prev.a[k];
    const double bn = y_of(cur.b[k]), bo = y_of(prev.b[k]);
    s.A += an - ao;
    s.AA += an * an - ao * ao;
    s.B += bn - bo;
    s.BB = fma(bn, bn, s.BB);
    s.BB = fma(-bo, bo, s.BB);
    s.AB = fma((double)an, bn, s.AB);
    s.AB = fma(-(double)ao, bo, s.AB);
    // every lane shuffles (converged); only windows inside the band and the image count
    const double sa = (double)win8(s.A), saa = (double)win8(s.AA);
    const double sb = win8(s.B), sbb = win8(s.BB), sab = win8(s.AB);
    const int orow = gi * 8 + k - 7;
    if (win_ok && orow >= 0 && orow < nout) {
      const double p = sa * sb, qq = fma(sa, sa, sb * sb);
      const double num = fma(2.0, p, c1s) * (fma(128.0, sab, c2s) - 2.0 * p);
      const double den = (qq + c1s) * (fma(64.0, saa + sbb, c2s) - qq);
      s.acc += ss_div(num, den);
    }
  }
}

template <typename OrigT, typename RecT, int CLIP>
__global__ void __launch_bounds__(kSsNT) ssim_strip_kernel(const OrigT* __restrict__ orig,
                                                           const RecT* __restrict__ rec, KGeom g, int32_t height,
                                                           int32_t width, int32_t nstrips, int32_t units,
                                                           int64_t total_units, float lo, float hi,
                                                           double c1s, double c2s, double* __restrict__ partial) {
  using Acc = SsAcc<OrigT>;
  const int lane = threadIdx.x;
  const int64_t u = blockIdx.x;
  const int32_t img = (int32_t)(u / units), q = (int32_t)(u % units);
  const int32_t band = q / nstrips, strip = q - band * nstrips;
  const int32_t x = strip * kSsOut + lane, y0 = band * kSsTY;
  const int32_t nout = min(kSsTY, height - 7 - y0);  // window rows of this band
  const int32_t nin = nout + 7;                      // input rows it reads
  const bool col_ok = x < width;
  const bool win_ok = lane < kSsOut && x <= width - 8;
  const int64_t rs = g.row_stride;
  const int64_t base = (int64_t)img * g.image_stride + (int64_t)y0 * rs + (col_ok ? x : 0);
  const OrigT* po = orig + base;
  const RecT* pr = rec + base;
  // three 8-row buffers in rotation (current, previous, prefetched next): no register copies
  SsGroup<OrigT, RecT> g0, g1, g2;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    g2.a[k] = 0;
    g2.b[k] = 0;
  }
  ss_load(g0, po, pr, rs, 0, nin, col_ok);
  SsState<Acc> s{0, 0, 0.0, 0.0, 0.0, 0.0};
  const int ngroups = (nin + 7) / 8;
  for (int gi = 0; gi < ngroups; gi += 3) {
    ss_load(g1, po + 8 * (gi + 1) * rs, pr + 8 * (gi + 1) * rs, rs, 8 * (gi + 1), nin, col_ok);
    ss_group<CLIP>(s, g0, g2, gi, nout, win_ok, lo, hi, c1s, c2s);
    if (gi + 1 >= ngroups) break;
    ss_load(g2, po + 8 * (gi + 2) * rs, pr + 8 * (gi + 2) * rs, rs, 8 * (gi + 2), nin, col_ok);
    ss_group<CLIP>(s, g1, g0, gi + 1, nout, win_ok, lo, hi, c1s, c2s);
    if (gi + 2 >= ngroups) break;
    ss_load(g0, po + 8 * (gi + 3) * rs, pr + 8 * (gi + 3) * rs, rs, 8 * (gi + 3), nin, col_ok);
    ss_group<CLIP>(s, g2, g1, gi + 2, nout, win_ok, lo, hi, c1s, c2s);
  }
  double acc = s.acc;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) partial[(int64_t)img * units + q] = acc;
}

// ---- fused round trip + SSIM (next row f1 "in the fused epilogue"): no reconstruction in HBM --
// One warp per (image, strip of 24 window columns = 32 pixel columns = 4 block columns, block
// aligned); the warp walks the whole image height in chunks of 8 block rows.  Per chunk, lane l
// reconstructs block (row 8c + l/4, column 3s + l%4) exactly as roundtrip_kernel does (fwd2d,
// weights wk, inv2d) and writes it (fp32 reconstruction, u8 original) into the warp's shared
// 72-row window (rows 0..7 carry the previous chunk's last 8 rows); then lane l takes pixel
// column 24s + l through those 64 rows with ss_group -- the strip kernel's vertical running sums,
// shuffle window sums and SSIM formula (lanes 0..23 own windows).  The running sums continue
// across chunks: they add and subtract exactly representable fp64 values (u8 sums in fp32), so
// they never drift.  HBM traffic: the u8 original once, + 1/3 re-read of the neighbour strips'
// shared block column (mostly from L2); nothing is written but one fp64 partial per warp.
constexpr int kSfOut = 24, kSfWarps = 3, kSfPitch = 36, kSfRows = 72;  // 38 KB static smem

#ifndef ADCT_SF_MINB
#define ADCT_SF_MINB 1
#endif
template <class MP, int CLIP>
__global__ void __launch_bounds__(32 * kSfWarps, ADCT_SF_MINB) ssim_fused_kernel(const uint8_t* __restrict__ src, KGeom g,
                                                                   int32_t height, int32_t width, DevMat dm, Wk wk,
                                                                   int32_t nstrips, int64_t total_units, float lo,
                                                                   float hi, double c1s, double c2s,
                                                                   double* __restrict__ partial) {
  __shared__ __align__(16) float sy[kSfWarps][kSfRows][kSfPitch];
  __shared__ __align__(16) uint8_t sx[kSfWarps][kSfRows][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t u = (int64_t)blockIdx.x * kSfWarps + w;
  if (u >= total_units) return;  // warp-uniform; the warps never synchronise with each other
  const int32_t img = (int32_t)(u / nstrips), strip = (int32_t)(u - (int64_t)img * nstrips);
  const int32_t nbh = height / 8, nbw = width / 8;
  const int32_t bx = 3 * strip + (lane & 3), brl = lane >> 2;  // this lane's block (column, row in chunk)
  const int32_t xcol = 24 * strip + lane;                      // this lane's pixel column (SSIM phase)
  const bool win_ok = lane < kSfOut && xcol <= width - 8;
  const MP m(dm);
  const uint8_t* base = src + (int64_t)img * g.image_stride + (int64_t)bx * 8;
  float(*Y)[kSfPitch] = sy[w];
  uint8_t(*X)[32] = sx[w];
#pragma unroll
  for (int i = 0; i < 8; ++i) {  // the rows above the image: zero
    Y[i][lane] = 0.0f;
    X[i][lane] = 0;
  }
  // this lane's block of chunk 0, raw
  uint2 raw[8];
  auto load_raw = [&](int32_t c) {
    const int32_t by = 8 * c + brl;
    const bool ok = by < nbh && bx < nbw;
    const uint8_t* p = base + (int64_t)by * 8 * g.row_stride;
#pragma unroll
    for (int i = 0; i < 8; ++i) raw[i] = ok ? Src<uint8_t>::load(p + (int64_t)i * g.row_stride) : make_uint2(0u, 0u);
  };
  load_raw(0);
  SsState<float> st{0.0f, 0.0f, 0.0, 0.0, 0.0, 0.0};
  const int32_t nchunks = (height + 63) / 64;
  for (int32_t c = 0; c < nchunks; ++c) {
    {  // round trip of the lane's block (the composition approx_dct8x8_roundtrip, F32, no clip)
      float x[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i) Src<uint8_t>::to_f(raw[i], x[i]);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        *reinterpret_cast<uint2*>(&X[8 + 8 * brl + i][8 * (lane & 3)]) = raw[i];
#if ADCT_SF_PACKED
      {
        float2 x2[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int c = 0; c < 4; ++c) x2[i][c] = pk(x[i][2 * c], x[i][2 * c + 1]);
        roundtrip2d_p(m, x2, wk.w);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            x[i][2 * c] = x2[i][c].x;
            x[i][2 * c + 1] = x2[i][c].y;
          }
      }
#else
      {
        float y[8][8];
        fwd2d(m, x, y);
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
          for (int l = 0; l < 8; ++l) y[k][l] *= wk.w[k * 8 + l];
        inv2d<MP, ~0ull>(m, y, x);
      }
#endif
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float* d = &Y[8 + 8 * brl + i][8 * (lane & 3)];
        *reinterpret_cast<float4*>(d) = make_float4(x[i][0], x[i][1], x[i][2], x[i][3]);
        *reinterpret_cast<float4*>(d + 4) = make_float4(x[i][4], x[i][5], x[i][6], x[i][7]);
      }
    }
    if (c + 1 < nchunks) load_raw(c + 1);  // the next chunk's block lands during the SSIM phase
    __syncwarp();
    // SSIM phase: groups of 8 rows gi = 8c + q (global rows 64c + 8q ..), dropping the group 8 rows up
#pragma unroll 1
    for (int q = 0; q < 8; ++q) {
      SsGroup<uint8_t, float> cur, prev;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        cur.a[k] = X[8 + 8 * q + k][lane];
        cur.b[k] = Y[8 + 8 * q + k][lane];
        prev.a[k] = X[8 * q + k][lane];
        prev.b[k] = Y[8 * q + k][lane];
      }
      ss_group<CLIP>(st, cur, prev, 8 * c + q, height - 7, win_ok, lo, hi, c1s, c2s);
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 8; ++i) {  // carry the chunk's last 8 rows
      Y[i][lane] = Y[64 + i][lane];
      X[i][lane] = X[64 + i][lane];
    }
    __syncwarp();
  }
  double acc = st.acc;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) partial[u] = acc;
}

}  // namespace

int64_t ssim_tiles(const adct_geom& g) {  // warps (strip x band units) per image
  if (g.height < 8 || g.width < 8) return 0;
  return (int64_t)((g.width - 7 + kSsOut - 1) / kSsOut) * ((g.height - 7 + kSsTY - 1) / kSsTY);
}

int64_t ssim_fused_strips(const adct_geom& g) {  // warps of ssim_fused_kernel per image
  if (g.height < 8 || g.width < 8) return 0;
  return (int64_t)((g.width - 7 + kSfOut - 1) / kSfOut);
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
  launch_pdl(finalize_kernel, dim3((unsigned)n_images, (unsigned)n_out), dim3(kFinNT), 0, st, partial, chunks, n_images,
             slots, slot_of, n_out, npix, peak, sse, psnr, 1.0);
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
  const int32_t nstrips = (g.width - 7 + kSsOut - 1) / kSsOut;
  const int32_t units = (int32_t)ssim_tiles(g);
  const int64_t total = (int64_t)units * g.n_images;
  const float lo = 0.0f, hi = (float)peak;  // clip range of the reconstruction: [0, peak]
  const double c1 = (0.01 * peak) * (0.01 * peak), c2 = (0.03 * peak) * (0.03 * peak);
  double* partial = (double*)workspace;
  const unsigned grid = (unsigned)total;
#define ADCT_SSIM_C(OT, RT, C)                                                                     \
  ssim_strip_kernel<OT, RT, C><<<grid, kSsNT, 0, st>>>((const OT*)orig, (const RT*)recon, kg, g.height, g.width, \
                                                       nstrips, units, total, lo, hi, 4096.0 * c1, 4096.0 * c2,  \
                                                       partial)
#define ADCT_SSIM(OT, RT)                                                  \
  do {                                                                     \
    if (clip == ADCT_CLIP_NONE) ADCT_SSIM_C(OT, RT, ADCT_CLIP_NONE);       \
    else if (clip == ADCT_CLIP) ADCT_SSIM_C(OT, RT, ADCT_CLIP);            \
    else ADCT_SSIM_C(OT, RT, ADCT_CLIP_ROUND);                             \
  } while (0)
  if (orig_t == ADCT_U8) {
    if (recon_t == ADCT_F32) ADCT_SSIM(uint8_t, float); else if (recon_t == ADCT_U8) ADCT_SSIM(uint8_t, uint8_t);
    else ADCT_SSIM(uint8_t, int16_t);
  } else {
    if (recon_t == ADCT_F32) ADCT_SSIM(int16_t, float); else if (recon_t == ADCT_U8) ADCT_SSIM(int16_t, uint8_t);
    else ADCT_SSIM(int16_t, int16_t);
  }
#undef ADCT_SSIM
#undef ADCT_SSIM_C
  count_launch();
  if (adct_status e = launch_status()) return e;
  const double nwin = (double)(g.height - 7) * (double)(g.width - 7);
  launch_finalize_scaled(partial, units, g.n_images, 1.0 / nwin, ssim, st);
  return launch_status();
}

adct_status approx_dct8x8_ssim(const adct_matrix* m, const uint8_t* src, adct_geom g, int32_t r, adct_clip clip,
                               double* ssim, void* workspace, size_t workspace_bytes, void* stream) {
  if (!m || !src || !ssim) return ADCT_E_INVALID_ARGUMENT;
  if (adct_status s = check_geom(g)) return s;
  if (r < 1 || r > 64) return ADCT_E_INVALID_ARGUMENT;
  if (clip != ADCT_CLIP_NONE && clip != ADCT_CLIP && clip != ADCT_CLIP_ROUND) return ADCT_E_INVALID_ARGUMENT;
  if (!aligned(src, 8)) return ADCT_E_ALIGNMENT;
  if (!workspace || workspace_bytes < adct_workspace_bytes(g, 1) || !aligned(workspace, 8)) return ADCT_E_WORKSPACE;
  if (g.n_images == 0) return ADCT_OK;
  const KGeom kg = make_kgeom(g);
  Wk wk;
  const uint64_t keep = keep_mask(r);
  for (int p = 0; p < 64; ++p) wk.w[p] = ((keep >> p) & 1ull) ? (m->is_int ? m->dev.wy[p] : m->dev.wb[p]) : 0.0f;
  const int32_t nstrips = (int32_t)ssim_fused_strips(g);
  const int64_t total = (int64_t)nstrips * g.n_images;
  const double peak = 255.0, c1 = (0.01 * peak) * (0.01 * peak), c2 = (0.03 * peak) * (0.03 * peak);
  const unsigned grid = (unsigned)((total + kSfWarps - 1) / kSfWarps);
  double* partial = (double*)workspace;
  cudaStream_t st = (cudaStream_t)stream;
#define ADCT_SF(MP, C)                                                                                        \
  ssim_fused_kernel<MP, C><<<grid, 32 * kSfWarps, 0, st>>>(src, kg, g.height, g.width, m->dev, wk, nstrips, total, \
                                                           0.0f, (float)peak, 4096.0 * c1, 4096.0 * c2, partial)
#define ADCT_SF_M(MP)                                         \
  do {                                                        \
    if (clip == ADCT_CLIP_NONE) ADCT_SF(MP, ADCT_CLIP_NONE);  \
    else if (clip == ADCT_CLIP) ADCT_SF(MP, ADCT_CLIP);       \
    else ADCT_SF(MP, ADCT_CLIP_ROUND);                        \
  } while (0)
  if (m->specialized) ADCT_SF_M(T1Mat); else ADCT_SF_M(RtMat);
#undef ADCT_SF_M
#undef ADCT_SF
  count_launch();
  if (adct_status e = launch_status()) return e;
  const double nwin = (double)(g.height - 7) * (double)(g.width - 7);
  launch_finalize_scaled(partial, nstrips, g.n_images, 1.0 / nwin, ssim, st);
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
