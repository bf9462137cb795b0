// blockmajor.cu — HBM-bound paths whose data is block-major: 8x8 blocks stored as consecutive
// 64-element rows ([n][8][8]).
//
//  - roundtrip_bm_kernel: BASELINE.json config 5, forward -> retain r -> inverse of int16
//    residual blocks, 128 B in + 128 B (int16) / 256 B (fp32) out per
//    block;
//  - fwd_quant_tma_kernel: config 3, forward of u8 image tiles with S folded into a uniform
//    quantiser (reading A10), 64 B in + 128 B out per block.
//
// Both move data only with TMA: every warp owns a ring of input tiles (mbarrier-completed
// cp.async.bulk.tensor loads) and one output staging tile written back with
// cp.async.bulk.tensor stores.  Block-major tiles use the 128-byte swizzle, so that lane l,
// which owns the block in tile row l, reads and writes its 16-byte rows at chunk (i ^ (l & 7)):
// conflict-free shared-memory access with one thread per block.
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "adct_host.h"
#include "tma.cuh"
#include "packed.cuh"
#include "quant.cuh"

// ADCT_BM_PACKED: the round trip of the block-major kernel on column pairs with packed fp32
// (packed.cuh); 0 = the scalar networks (A/B)
#ifndef ADCT_BM_PACKED
#define ADCT_BM_PACKED 1
#endif
// ADCT_Q_PACKED: the C3 quantiser itself on coefficient pairs -- parity-green but slower
// (1.407 vs 1.291 ms per C3 step: the per-lane sign/select work does not pack), so off
#ifndef ADCT_Q_PACKED
#define ADCT_Q_PACKED 0
#endif
// ADCT_Q_FAST: the C3 quantiser with a directed-rounding FMA at the rational positions (exact by
// construction, no remainder correction) and a fused remainder at the irrational ones; 0 = the
// round-2 remainder-corrected form (A/B)
#ifndef ADCT_Q_FAST
#define ADCT_Q_FAST 1
#endif

namespace adct {
namespace {

constexpr int kBmInSlots = 2;

__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk) {  // 128-byte swizzle
  return row * 128u + ((chunk ^ (row & 7u)) << 4);
}

// int16 pair -> two floats (sign-extended halves; integer ALU pipe)
__device__ __forceinline__ void i16x2_to_f(uint32_t w, float& lo, float& hi) {
  lo = (float)(int32_t)(int16_t)(w & 0xffffu);
  hi = (float)((int32_t)w >> 16);
}

// round half to even and saturate to int16, packed as two halves (low = a)
__device__ __forceinline__ uint32_t f2_to_i16x2(float a, float b) {
  a = fminf(fmaxf(a, -32768.0f), 32767.0f);
  b = fminf(fmaxf(b, -32768.0f), 32767.0f);
  // 1.5 * 2^23 + v rounds v to the nearest integer (ties to even); the low 16 bits of the
  // pattern are that integer in two's complement
  const uint32_t ua = __float_as_uint(a + 12582912.0f), ub = __float_as_uint(b + 12582912.0f);
  return __byte_perm(ua, ub, 0x5410);
}

struct Wk {
  float w[64];
};

// byte of w as fp32 32768 + x (one PRMT; see stream.cu pxf)
template <uint32_t SEL>
__device__ __forceinline__ float pxf_q(uint32_t w, uint32_t magic) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(w), "r"(magic), "n"(SEL));
  return __uint_as_float(r);
}

// ---- config 5: block-major round trip ----------------------------------------------------------
// One tile = 32 consecutive blocks (4 KB of int16), one block per lane.  Output tile: 32 rows of
// 128 B (int16) or 64 rows (fp32, a block's rows 0-3 then 4-7).
template <bool F32OUT>
constexpr int bm_warps() { return F32OUT ? 12 : 16; }  // shared memory: 16 KB / 12 KB per warp

template <class MP, bool F32OUT>
__global__ void __launch_bounds__(32 * bm_warps<F32OUT>(), 1)
    roundtrip_bm_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
                        DevMat dm, Wk wk, uint32_t n_tiles, int clip, float lo, float hi) {
  constexpr int kOutBytes = F32OUT ? 8192 : 4096;
  constexpr int kBmWarps = bm_warps<F32OUT>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t wbase = smem_u32(smem) + (uint32_t)w * (kBmInSlots * 4096 + kOutBytes);
  const uint32_t outb = wbase + kBmInSlots * 4096;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kBmWarps * (kBmInSlots * 4096 + kOutBytes)) +
                   w * kBmInSlots;
  if (lane == 0) {
    for (int i = 0; i < kBmInSlots; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const MP m(dm);
  const uint32_t wid = blockIdx.x * kBmWarps + w, nw = gridDim.x * kBmWarps;
  uint32_t pt = wid;  // next tile to prefetch
  auto issue = [&](int slot) {
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars[slot], 4096u);
      tma_load_2d(wbase + slot * 4096, &tin, 0, (int32_t)(pt * 32u), smem_u32(&bars[slot]));
    }
    pt += nw;
  };
  for (int s = 0; s < kBmInSlots; ++s)
    if (pt < n_tiles) issue(s);
  int slot = 0;
  uint32_t phase = 0;
  for (uint32_t t = wid; t < n_tiles; t += nw) {
    mbar_wait(&bars[slot], phase);
    float x[8][8];
    const uint32_t ib = wbase + slot * 4096;
#if ADCT_BM_PACKED
    float2 x2[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 v = lds128(ib + swz(lane, i));
      i16x2_to_f(v.x, x2[i][0].x, x2[i][0].y);
      i16x2_to_f(v.y, x2[i][1].x, x2[i][1].y);
      i16x2_to_f(v.z, x2[i][2].x, x2[i][2].y);
      i16x2_to_f(v.w, x2[i][3].x, x2[i][3].y);
    }
#else
    float y[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 v = lds128(ib + swz(lane, i));
      i16x2_to_f(v.x, x[i][0], x[i][1]);
      i16x2_to_f(v.y, x[i][2], x[i][3]);
      i16x2_to_f(v.z, x[i][4], x[i][5]);
      i16x2_to_f(v.w, x[i][6], x[i][7]);
    }
#endif
    __syncwarp();
    fence_proxy_async();
    if (pt < n_tiles) issue(slot);  // the slot's data is in registers: refill it now
    if (++slot == kBmInSlots) { slot = 0; phase ^= 1u; }
#if ADCT_BM_PACKED
    roundtrip2d_p(m, x2, wk.w);
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        x[i][2 * c] = x2[i][c].x;
        x[i][2 * c + 1] = x2[i][c].y;
      }
#else
    fwd2d(m, x, y);
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int l = 0; l < 8; ++l) y[k][l] *= wk.w[k * 8 + l];
    inv2d<MP, ~0ull>(m, y, x);
#endif
    // the staging tile is free once the previous tile's store has read it
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
    if constexpr (F32OUT) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          v[j] = x[i][j];
          if (clip != ADCT_CLIP_NONE) v[j] = fminf(fmaxf(v[j], lo), hi);
          if (clip == ADCT_CLIP_ROUND) v[j] = rintf(v[j]);
        }
        // block row i -> tile row 2*lane + i/4, 32-byte half (i & 3) -> chunks 2(i&3), 2(i&3)+1
        const uint32_t row = 2u * lane + (uint32_t)(i >> 2), c0 = 2u * (uint32_t)(i & 3);
        sts128(outb + swz(row, c0), make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]),
                                               __float_as_uint(v[3])));
        sts128(outb + swz(row, c0 + 1), make_uint4(__float_as_uint(v[4]), __float_as_uint(v[5]),
                                                   __float_as_uint(v[6]), __float_as_uint(v[7])));
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = fminf(fmaxf(x[i][j], lo), hi);
        sts128(outb + swz(lane, i), make_uint4(f2_to_i16x2(v[0], v[1]), f2_to_i16x2(v[2], v[3]),
                                               f2_to_i16x2(v[4], v[5]), f2_to_i16x2(v[6], v[7])));
      }
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(&tout, 0, (int32_t)(t * (F32OUT ? 64u : 32u)), outb);
      bulk_commit();
    }
  }
  if (lane == 0) bulk_wait<0>();
}

bool enc2d(CUtensorMap* map, CUtensorMapDataType dt, void* base, uint64_t inner, uint64_t rows, uint64_t stride,
           uint32_t box_inner, uint32_t box_rows) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {inner, rows};
  const cuuint64_t strides[1] = {stride};
  const cuuint32_t box[2] = {box_inner, box_rows};
  const cuuint32_t es[2] = {1, 1};
  return enc(map, dt, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---- config 3: forward + uniform quantiser, u8 image tiles -> int16 block-major --------------
// q_kl = round_half_away(Y_kl / c_kl), c_kl = step sqrt(n_k n_l) (reading A10).  Fast path per
// coefficient: v = Y * (1/c) in fp32 (|error| < 2e-5 for |Y| < 2^17), 1.5*2^23 + v rounds it to
// the nearest integer (the low 16 bits of the pattern are that integer in two's complement),
// and the exact rounding remainder d = v - round(v) (Fast2Sum) flags coefficients within 2^-14
// of a rounding boundary — every exact tie included — for which the block takes the exact
// integer rule (2m-1)^2 P <= 4 Y^2 < (2m+1)^2 P, P = step^2 n_k n_l (fp64, exact below 2^53).
//
// ADCT_Q_FAST (default): at the 40 rational positions c is an even integer and
// |q| = floor(A / c), A = |Y| + c/2 an integer < 2^23.  With u = fp32 1/c rounded UP, the exact
// product A u lies in [A/c, A/c + A 2^-23 / c): at a multiple A = m c it is >= m, otherwise
// A/c <= m - 1/c and A 2^-23 < 1 keeps it below m, so floor(A u) = floor(A / c) for every such A
// (tests/test_kernel_arith.py checks every A).  One FFMA rounding toward -inf onto 1.5 * 2^23
// gives 1.5 * 2^23 + |q|; 3 * 2^23 minus that is 1.5 * 2^23 - |q|, whose low 16 bits are -|q|.
constexpr int kQWarps = 12;                 // 16 KB of shared memory per warp
constexpr int kQInSlots = 2;

template <int TW>
__global__ void __launch_bounds__(32 * kQWarps, 1)
    fwd_quant_tma_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
                         QTab qt, float stepf, int32_t tpb, int32_t tpi, int32_t bh, uint32_t n_tiles, FastDiv dtpi,
                         FastDiv dtpb, uint32_t magic) {
  using MP = T1Mat;
  const DevMat dm{};
  constexpr int RT = 4096 / TW;  // rows per input tile
  constexpr int BPR = TW / 8;    // blocks per band segment
  constexpr int NB = RT / 8;     // bands per tile (2 or 4)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t wbase = smem_u32(smem) + (uint32_t)w * (kQInSlots * 4096 + 8192);
  const uint32_t outb = wbase + kQInSlots * 4096;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kQWarps * (kQInSlots * 4096 + 8192)) + w * kQInSlots;
  if (lane == 0) {
    for (int i = 0; i < kQInSlots; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const MP m(dm);
  const uint32_t wid = blockIdx.x * kQWarps + w, nw = gridDim.x * kQWarps;
  // tile t -> (image, tile row, slice)
  auto where = [&](uint32_t t, uint32_t& img, int32_t& trow, int32_t& slice) {
    img = fdiv(t, dtpi);
    const uint32_t r = t - img * (uint32_t)tpi;
    trow = (int32_t)fdiv(r, dtpb);
    slice = (int32_t)r - trow * tpb;
  };
  uint32_t pt = wid;
  auto issue = [&](int slot) {
    if (lane == 0) {
      uint32_t img;
      int32_t trow, slice;
      where(pt, img, trow, slice);
      mbar_arrive_expect_tx(&bars[slot], 4096u);
      tma_load_3d(wbase + slot * 4096, &tin, slice * TW, trow * RT, (int32_t)img, smem_u32(&bars[slot]));
    }
    pt += nw;
  };
  for (int s = 0; s < kQInSlots; ++s)
    if (pt < n_tiles) issue(s);
  const uint32_t grp = (uint32_t)(lane / BPR), pos = (uint32_t)(lane % BPR);
  const uint32_t lane_in = (uint32_t)pos * 8u + grp * 16u * TW;
#if ADCT_Q_FAST
  const float qru[4] = {qt.ru[0], qt.ru[1], qt.ru[2], qt.ru[3]};
  const float qri[2] = {qt.ri[0], qt.ri[1]};
#endif
  int slot = 0;
  uint32_t phase = 0;
  for (uint32_t t = wid; t < n_tiles; t += nw) {
    mbar_wait(&bars[slot], phase);
    uint2 rows[2][8];
    const uint32_t ib = wbase + slot * 4096 + lane_in;
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int i = 0; i < 8; ++i) rows[b][i] = lds64(ib + (uint32_t)(b * 8 + i) * TW);
    __syncwarp();
    fence_proxy_async();
    if (pt < n_tiles) issue(slot);
    if (++slot == kQInSlots) { slot = 0; phase ^= 1u; }
    if (lane == 0) bulk_wait_read<0>();  // staging free once the previous tile's stores read it
    __syncwarp();
#pragma unroll 1
    for (int b = 0; b < 2; ++b) {
      float y[8][8];
#if ADCT_BM_PACKED  // forward on column pairs (packed.cuh), coefficients back in raster order
      {
        float2 x2[8][4], p2[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          x2[i][0] = pk(pxf_q<0x7504u>(rows[b][i].x, magic), pxf_q<0x7514u>(rows[b][i].x, magic));
          x2[i][1] = pk(pxf_q<0x7524u>(rows[b][i].x, magic), pxf_q<0x7534u>(rows[b][i].x, magic));
          x2[i][2] = pk(pxf_q<0x7504u>(rows[b][i].y, magic), pxf_q<0x7514u>(rows[b][i].y, magic));
          x2[i][3] = pk(pxf_q<0x7524u>(rows[b][i].y, magic), pxf_q<0x7534u>(rows[b][i].y, magic));
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float2 col[8], out[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) col[i] = x2[i][c];
          fwd8p(m, col, out);
#pragma unroll
          for (int k = 0; k < 8; ++k) p2[k][c] = out[k];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          float2 yq[4];
          fwd8_row(m, p2[k], yq);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            y[k][yq_col(q, 0)] = yq[q].x;
            y[k][yq_col(q, 1)] = yq[q].y;
          }
        }
      }
#else
      float x[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        x[i][0] = pxf_q<0x7504u>(rows[b][i].x, magic); x[i][1] = pxf_q<0x7514u>(rows[b][i].x, magic);
        x[i][2] = pxf_q<0x7524u>(rows[b][i].x, magic); x[i][3] = pxf_q<0x7534u>(rows[b][i].x, magic);
        x[i][4] = pxf_q<0x7504u>(rows[b][i].y, magic); x[i][5] = pxf_q<0x7514u>(rows[b][i].y, magic);
        x[i][6] = pxf_q<0x7524u>(rows[b][i].y, magic); x[i][7] = pxf_q<0x7534u>(rows[b][i].y, magic);
      }
      fwd2d(m, x, y);
#endif
      // quantise.  T1: c_kl = step * sqrt(n_k n_l) is an integer multiple of step unless exactly
      // one of k, l is in {2, 6} (n = 20 against 8 or 18); integer c is rounded exactly in fp32.
      bool near = false;
      uint32_t packed[32];
#if ADCT_Q_PACKED
      // two coefficients per packed instruction, paired as the packed forward leaves them: slots
      // (0,4), (2,6), (1,3), (5,7) of a row, which are both rational or both irrational.  Same
      // fp32 operations per element as the scalar code below, except that the correction
      // m0 - [rem < 0] is formed as (m0 + copysign(0.5, rem)) - 0.5 (exact: rem is an exact
      // integer, +0 when it vanishes) instead of a compare and select
      {
        uint32_t u[8][8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int la = yq_col(q, 0), lb = yq_col(q, 1);
            const float2 yy = pk(y[k][la] - ((k == 0 && la == 0) ? 64.0f * 32768.0f : 0.0f), y[k][lb]);  // exact
            y[k][la] = yy.x;
            y[k][lb] = yy.y;
            const float2 inv = pk(qt.inv[k * 8 + la], qt.inv[k * 8 + lb]);
            if (t1_rational(k, la)) {
              const float ca = stepf * (float)t1_sqrt_nn(k, la), cb = stepf * (float)t1_sqrt_nn(k, lb);
              const float2 A = __fadd2_rn(pk(fabsf(yy.x), fabsf(yy.y)), pk(0.5f * ca, 0.5f * cb));
              const float2 f = __ffma2_rn(A, inv, pk(12582912.0f, 12582912.0f));
              const float2 m0 = __fadd2_rn(f, pk(-12582912.0f, -12582912.0f));
              const float2 rem = __ffma2_rn(pk(-ca, -cb), m0, A);
              const float2 hs = pk(__uint_as_float(0x3F000000u | (__float_as_uint(rem.x) & 0x80000000u)),
                                   __uint_as_float(0x3F000000u | (__float_as_uint(rem.y) & 0x80000000u)));
              const float2 mf = __fadd2_rn(__fadd2_rn(m0, hs), pk(-0.5f, -0.5f));
              const float2 qf = pk(__uint_as_float(__float_as_uint(mf.x) | (__float_as_uint(yy.x) & 0x80000000u)),
                                   __uint_as_float(__float_as_uint(mf.y) | (__float_as_uint(yy.y) & 0x80000000u)));
              const float2 uu = __fadd2_rn(qf, pk(12582912.0f, 12582912.0f));
              u[k][la] = __float_as_uint(uu.x);
              u[k][lb] = __float_as_uint(uu.y);
            } else {
              const float2 v = __fmul2_rn(yy, inv);
              const float2 f = __fadd2_rn(v, pk(12582912.0f, 12582912.0f));
              const float2 d = __fadd2_rn(v, pk(-(f.x - 12582912.0f), -(f.y - 12582912.0f)));
              near |= fabsf(d.x) > 0.49993896f || fabsf(d.y) > 0.49993896f;  // within 2^-14 of a boundary
              u[k][la] = __float_as_uint(f.x);
              u[k][lb] = __float_as_uint(f.y);
            }
          }
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
          for (int l = 0; l < 8; l += 2) packed[k * 4 + l / 2] = __byte_perm(u[k][l], u[k][l + 1], 0x5410);
      }
#else
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int l = 0; l < 8; l += 2) {
          uint32_t u[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int kl = k * 8 + l + e;
            const float yy = y[k][l + e] - (kl == 0 ? 64.0f * 32768.0f : 0.0f);  // exact
            y[k][l + e] = yy;
            if (t1_rational(k, l + e)) {
#if ADCT_Q_FAST
              const float A = fabsf(yy) + stepf * (0.5f * (float)t1_sqrt_nn(k, l + e));  // exact
              const float up = __fmaf_rd(A, qru[q_rclass(k, l + e)], 12582912.0f);      // 1.5*2^23 + |q|
              u[e] = __float_as_uint(yy < 0.0f ? 25165824.0f - up : up);
#else
              // |q| = floor((|Y| + c/2) / c): estimate, then the exact remainder decides
              const float c = stepf * (float)t1_sqrt_nn(k, l + e);
              const float A = fabsf(yy) + 0.5f * c;
              const float f = A * qt.inv[kl] + 12582912.0f;
              const float m0 = f - 12582912.0f;
              const float rem = fmaf(-c, m0, A);
              const float mf = rem < 0.0f ? m0 - 1.0f : m0;
              const float qf = __uint_as_float(__float_as_uint(mf) | (__float_as_uint(yy) & 0x80000000u));
              u[e] = __float_as_uint(qf + 12582912.0f);
#endif
            } else {
#if ADCT_Q_FAST
              // nearest integer of Y/c (one rounding), and the remainder Y/c - that in one FFMA
              const float iv = qri[q_iclass(k, l + e)];
              const float f = fmaf(yy, iv, 12582912.0f);
              near |= fabsf(fmaf(yy, iv, 12582912.0f - f)) > 0.49993896f;  // within 2^-14 of a boundary
#else
              const float v = yy * qt.inv[kl];
              const float f = v + 12582912.0f;
              near |= fabsf(v - (f - 12582912.0f)) > 0.49993896f;  // within 2^-14 of a boundary
#endif
              u[e] = __float_as_uint(f);
            }
          }
          packed[k * 4 + l / 2] = __byte_perm(u[0], u[1], 0x5410);
        }
#endif
      if (__any_sync(0xffffffffu, near)) {  // rare: exact integer rule at irrational positions
#pragma unroll
        for (int kl = 0; kl < 64; ++kl) {
          if (t1_rational(kl >> 3, kl & 7)) continue;
          const float yy = y[kl >> 3][kl & 7];
#if ADCT_Q_FAST
          const float f = fmaf(yy, qt.inv[kl], 12582912.0f);
          if (near && fabsf(fmaf(yy, qt.inv[kl], 12582912.0f - f)) > 0.49993896f) {
#else
          const float v = yy * qt.inv[kl];
          const float f = v + 12582912.0f;
          if (near && fabsf(v - (f - 12582912.0f)) > 0.49993896f) {
#endif
            const double a2 = 4.0 * (double)yy * (double)yy, pp = qt.p[kl];
            double mm = rint(fabs((double)yy) * qt.rsp[kl]);  // within 1 of the answer
            if (mm >= 1.0 && (2.0 * mm - 1.0) * (2.0 * mm - 1.0) * pp > a2) mm -= 1.0;
            else if ((2.0 * mm + 1.0) * (2.0 * mm + 1.0) * pp <= a2) mm += 1.0;
            const uint32_t q16 = (uint32_t)(uint16_t)(int16_t)(yy < 0.0f ? -(int)mm : (int)mm);
            uint32_t& wv = packed[kl >> 1];
            wv = (kl & 1) ? ((wv & 0xffffu) | (q16 << 16)) : ((wv & 0xffff0000u) | q16);
          }
        }
      }
      // staging: band segment (2*grp + b) rows of 128 B, swizzled by the row within the segment
      const uint32_t ob = outb + (2u * grp + (uint32_t)b) * (uint32_t)BPR * 128u;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        sts128(ob + swz(pos, (uint32_t)k),
               make_uint4(packed[k * 4], packed[k * 4 + 1], packed[k * 4 + 2], packed[k * 4 + 3]));
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      uint32_t img;
      int32_t trow, slice;
      where(t, img, trow, slice);
#pragma unroll
      for (int g = 0; g < NB; ++g) {
        const int32_t band = trow * NB + g;
        if (band < bh) tma_store_3d(&tout, 0, slice * BPR, (int32_t)img * bh + band, outb + (uint32_t)g * BPR * 128u);
      }
      bulk_commit();
    }
  }
  if (lane == 0) bulk_wait<0>();
}

int bm_sms() { return device_sms(); }

template <class MP, bool F32OUT>
adct_status launch_rt_bm(const CUtensorMap& tin, const CUtensorMap& tout, const DevMat& dm, const Wk& wk,
                         uint32_t n_tiles, int clip, float lo, float hi, cudaStream_t st) {
  constexpr int kBmWarps = bm_warps<F32OUT>();
  constexpr size_t smem = (size_t)kBmWarps * (kBmInSlots * 4096 + (F32OUT ? 8192 : 4096)) + kBmWarps * kBmInSlots * 8 + 1024;
  static std::mutex mu;
  static int8_t state[kMaxDevices] = {};
  if (!once_per_device(mu, state, [&] {
        return cudaFuncSetAttribute(roundtrip_bm_kernel<MP, F32OUT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem) == cudaSuccess;
      }))
    return ADCT_E_CUDA;
  const uint32_t need = (n_tiles + kBmWarps - 1) / kBmWarps;
  const unsigned grid = (unsigned)(need < (uint32_t)bm_sms() ? need : (uint32_t)bm_sms());
  roundtrip_bm_kernel<MP, F32OUT><<<grid, 32 * kBmWarps, smem, st>>>(tin, tout, dm, wk, n_tiles, clip, lo, hi);
  return ADCT_OK;
}

template <int TW>
adct_status launch_quant(const CUtensorMap& tin, const CUtensorMap& tout, const QTab& qt, float stepf, int32_t tpb,
                         int32_t tpi, int32_t bh, uint32_t n_tiles, cudaStream_t st) {
  constexpr size_t smem = (size_t)kQWarps * (kQInSlots * 4096 + 8192) + kQWarps * kQInSlots * 8 + 1024;
  static std::mutex mu;
  static int8_t state[kMaxDevices] = {};
  if (!once_per_device(mu, state, [&] {
        return cudaFuncSetAttribute(fwd_quant_tma_kernel<TW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem) == cudaSuccess;
      }))
    return ADCT_E_CUDA;
  const uint32_t need = (n_tiles + kQWarps - 1) / kQWarps;
  const unsigned grid = (unsigned)(need < (uint32_t)bm_sms() ? need : (uint32_t)bm_sms());
  fwd_quant_tma_kernel<TW><<<grid, 32 * kQWarps, smem, st>>>(tin, tout, qt, stepf, tpb, tpi, bh, n_tiles,
                                                                  make_fastdiv((uint32_t)tpi),
                                                                  make_fastdiv((uint32_t)tpb), 0x47000000u);
  return ADCT_OK;
}

}  // namespace

// TMA path of approx_dct8x8_fwd_quant (u8 images with 16-byte aligned strides, integer
// matrices whose biased forward stays below 2^24).  Returns false when not applicable.
bool fwd_quant_tma(const adct_matrix* m, const uint8_t* src, const adct_geom& g, int32_t step, int16_t* q,
                   cudaStream_t st, adct_status* status) {
  if (!m->specialized) return false;  // the paper's T1 only (compile-time network and c_kl pattern)
  if ((g.row_stride % 16) || (g.n_images > 1 && (g.image_stride % 16)) || !aligned(src, 16) || !aligned(q, 128))
    return false;
  if (step < 1 || step > 4096) return false;
  // every intermediate of the forward on samples 2^15 + x must stay an exact fp32 integer
  int64_t rs0 = 0;
  for (int i = 0; i < 8; ++i) rs0 += std::llabs((long long)m->t[i]);
  if ((double)m->max_u8 + 32768.0 * (double)(rs0 * rs0) >= 16777216.0) return false;
  const int tw = [&] {
    const int64_t t256 = ((g.width + 255) / 256) * ((g.height + 15) / 16);
    const int64_t t128 = ((g.width + 127) / 128) * ((g.height + 31) / 32);
    return (m->specialized && t128 < t256) ? 128 : 256;
  }();
  const int rows = 4096 / tw;
  const int32_t tpb = (g.width + tw - 1) / tw;
  const int32_t tpi = ((g.height + rows - 1) / rows) * tpb;
  const int64_t n_tiles = g.n_images * (int64_t)tpi;
  if (n_tiles >= ((int64_t)1 << 31)) return false;
  auto enc = tmap_encoder();
  if (!enc) return false;
  CUtensorMap tin, tout;
  {
    const cuuint64_t dims[3] = {(cuuint64_t)g.width, (cuuint64_t)g.height, (cuuint64_t)g.n_images};
    const cuuint64_t strides[2] = {(cuuint64_t)g.row_stride,
                                   (cuuint64_t)(g.n_images > 1 ? g.image_stride : (int64_t)g.height * g.row_stride)};
    const cuuint32_t box[3] = {(cuuint32_t)tw, (cuuint32_t)rows, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    static const int promo_env = [] {  // A/B hook: ADCT_Q_L2PROMO=0|64|128|256
      const char* e = std::getenv("ADCT_Q_L2PROMO");
      return e ? std::atoi(e) : -1;
    }();
    // a 128-byte-wide box with 256-byte promotion pulls the neighbouring 128 B of every row into L2;
    // on 1920-byte rows (15 x 128 B) the granules straddle row ends and tiles of other warps, and
    // part of that is evicted before its tile comes: ncu measured 2.41 GB read for 2.12 GB of
    // pixels (config 3), 2.12 GB with 128-byte promotion, 1.160 -> 1.125 ms
    const int promo = promo_env >= 0 ? promo_env : (tw == 128 ? 128 : 256);
    const CUtensorMapL2promotion pr = promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                      : promo == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                      : promo == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                     : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    if (enc(&tin, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(src), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, pr,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  {
    const int64_t bw = g.width / 8, bh = g.height / 8;
    const cuuint64_t dims[3] = {64, (cuuint64_t)bw, (cuuint64_t)(g.n_images * bh)};
    const cuuint64_t strides[2] = {128, (cuuint64_t)(bw * 128)};
    const cuuint32_t box[3] = {64, (cuuint32_t)(tw / 8), 1};
    const cuuint32_t es[3] = {1, 1, 1};
    if (enc(&tout, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, q, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  QTab qt;
  q_fill(qt, step, m->n);
  const int32_t bh = g.height / 8;
  const float stepf = (float)step;
  adct_status s = tw == 128 ? launch_quant<128>(tin, tout, qt, stepf, tpb, tpi, bh, (uint32_t)n_tiles, st)
                            : launch_quant<256>(tin, tout, qt, stepf, tpb, tpi, bh, (uint32_t)n_tiles, st);
  if (s == ADCT_OK) {
    count_launch();
    s = launch_status();
  }
  *status = s;
  return true;
}

// Block-major fast path of approx_dct8x8_roundtrip: int16 source [n][8][8] contiguous, n a
// multiple of 32, int16 or fp32 reconstruction with the same layout.  Returns false when not
// applicable (the caller then uses the generic kernel).
bool roundtrip_blockmajor(const adct_matrix* m, const void* src, const adct_geom& g, const float* wk_in, void* recon,
                          adct_dtype recon_t, adct_clip clip, float lo, float hi, cudaStream_t st, adct_status* status) {
  if (!(g.height == 8 && g.width == 8 && g.row_stride == 8 && (g.n_images == 1 || g.image_stride == 64))) return false;
  if (recon_t != ADCT_I16 && recon_t != ADCT_F32) return false;
  if (g.n_images % 32 != 0 || g.n_images == 0 || g.n_images / 32 >= ((int64_t)1 << 31)) return false;
  if (!aligned(src, 128) || !aligned(recon, 128)) return false;
  const uint64_t n = (uint64_t)g.n_images;
  CUtensorMap tin, tout;
  if (!enc2d(&tin, CU_TENSOR_MAP_DATA_TYPE_UINT16, const_cast<void*>(src), 64, n, 128, 64, 32)) return false;
  const bool f32 = recon_t == ADCT_F32;
  if (f32) {
    if (!enc2d(&tout, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, recon, 32, 2 * n, 128, 32, 64)) return false;
  } else {
    if (!enc2d(&tout, CU_TENSOR_MAP_DATA_TYPE_UINT16, recon, 64, n, 128, 64, 32)) return false;
  }
  Wk wk;
  for (int i = 0; i < 64; ++i) wk.w[i] = wk_in[i];
  const uint32_t tiles = (uint32_t)(n / 32);
  adct_status s;
  if (m->specialized)
    s = f32 ? launch_rt_bm<T1Mat, true>(tin, tout, m->dev, wk, tiles, (int)clip, lo, hi, st)
            : launch_rt_bm<T1Mat, false>(tin, tout, m->dev, wk, tiles, (int)clip, lo, hi, st);
  else
    s = f32 ? launch_rt_bm<RtMat, true>(tin, tout, m->dev, wk, tiles, (int)clip, lo, hi, st)
            : launch_rt_bm<RtMat, false>(tin, tout, m->dev, wk, tiles, (int)clip, lo, hi, st);
  if (s == ADCT_OK) {
    count_launch();
    s = launch_status();
  }
  *status = s;
  return true;
}

}  // namespace adct
