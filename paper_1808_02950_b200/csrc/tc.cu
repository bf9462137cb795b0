// tc.cu — the tensor-core hot kernel of BASELINE.json config 4: forward -> zonal retention ->
// inverse -> squared error per image (§6.1) for uint8 planes, every 8x8
// block read from HBM exactly once, the forward's dense contraction on tcgen05 (kind::i8).
//
// Operand A is the raw pixel tile exactly as TMA lands it.  A 5-D tensor map over the u8 plane
// with dims {128 bytes, 8 rows, bands, 128-byte chunks, images} and strides {row, 8 rows, 128 B,
// image} (non-monotonic, accepted by the driver; probes/i8_probe.cu) places a box
// {128, 8, BH, CW, 1} (CW chunks x BH bands, CW * BH = 16) in shared memory as
// [chunk][band][row][128 B]: the canonical K-major no-swizzle layout of A = [pair p][k] with
// row p = two horizontally adjacent blocks (16 bytes of each of their 8 rows, k = 16 i + c),
// 8-pair groups 1024 B apart (SBO) and pixel rows 128 B apart (LBO).  So M = 128 pairs = 256
// blocks per tile, K = 128 u8 samples per pair, and no thread touches the pixels.
//
// Operand B (shared memory, s8) is the constant block-diagonal [2 NB x 128] matrix that gives,
// per block, exactly (Eq. 1):
//   Y_kl = sum_ij T_ki T_lj x_ij     for the coefficients the inverse needs (retained; for
//                                    r > 32 the dropped ones, reading A17)
//   s_i[j] = x_ij + x_(7-i)j,  t_i[j] = x_ij - x_(7-i)j   (i < 4, the first column butterfly)
// |b| <= 4, products and sums are exact in the s32 TMEM accumulators.  D column n of lane p:
// block 2p + n / NB, output n % NB.  4 MMAs of K = 32 per 256 blocks.
//
// The epilogue thread that owns lane p converts its two blocks' outputs to fp32 (exact) and
// runs the same fp32 arithmetic as the SIMT kernel (stream.cu, block_sse_u8s): weights
// 2/(n_k n_l), the horizontal inverse Q = (W o Y') T of the retained rows, and the vertical
// inverse fused with the error, (x_i - x^_i)^2 + (x_7-i - x^_7-i)^2 = ((s_i - 2E_i)^2 +
// (t_i - 2O_i)^2)/2; for r > 32 the inverse of the dropped coefficients is x - x^ itself.
//
// Warp roles of the persistent CTA (one per SM): kTcEpi epilogue warps per TMEM
// lane quarter (tiles round-robin), kTcIssuers MMA-issuer warps (one per SM sub-partition, tiles
// round-robin: a tcgen05.mma waits for its sub-partition's issue slots, which the FP32 epilogue
// saturates, so one issuer alone would pace the kernel; probes/tc_contend.cu), one TMA producer.  Rings: kTcSlots
// pixel tiles in shared memory (refilled when the tile's MMA has completed), kTcDStages D stages
// in TMEM (released by the epilogue warps once their tcgen05.ld completed).  Deterministic fp64
// partials per (chunk, tile index in the chunk mod kTcEpi, lane quarter).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "adct_host.h"
#include "quant.cuh"
#include "tc05.cuh"
#include "tma.cuh"

namespace adct {

void launch_finalize(const double* partial, int32_t chunks, int64_t n_images, int32_t slots, const SlotMap& slot_of,
                     int32_t n_out, double npix, double peak, double* sse, double* psnr, cudaStream_t st);
int sms_s();

namespace {

__host__ __device__ constexpr int popc64t(uint64_t v) {
  int c = 0;
  for (int i = 0; i < 64; ++i) c += (int)((v >> i) & 1u);
  return c;
}
__host__ __device__ constexpr uint32_t row_mask_t(uint64_t nz) {
  uint32_t r = 0;
  for (int k = 0; k < 8; ++k)
    if ((nz >> (8 * k)) & 0xffull) r |= 1u << k;
  return r;
}

// compile-time shape of the MMA outputs for retention r
template <int R>
struct TcShape {
  static constexpr uint64_t KEEP = keep_mask(R);
  static constexpr bool RESID = popc64t(KEEP) > 32;
  static constexpr uint64_t NZ = RESID ? ~KEEP : KEEP;  // coefficients the inverse uses
  static constexpr int NNZ = popc64t(NZ);
  static constexpr int NY = (NNZ + 15) / 16 * 16;       // coefficient columns (x16 loads)
  static constexpr int NB = NY + (RESID ? 0 : 64);      // per block: + s_i[j] at NY + 8j + i, t_i[j] at +4
  static constexpr int N = 2 * NB;                      // MMA N: the pair's two blocks
  static constexpr uint32_t ROWS = row_mask_t(NZ);
  static_assert(NNZ >= 1 && NNZ <= 32, "1..32 coefficient columns");
  static_assert(N <= 256 && N % 16 == 0, "MMA N");
};

// T1 in constant memory for the B construction, where the row index is a runtime value (the
// constexpr table of T1Mat would be copied to local memory there)
__constant__ float c_t1f[64] = {1, 1, 1,  1,  1,  1,  1,  1,  2, 2,  1,  0,  0,  -1, -2, -2,
                                2, 1, -1, -2, -2, -1, 1,  2,  1, 0,  -2, -2, 2,  2,  0,  -1,
                                1, -1, -1, 1, 1,  -1, -1, 1,  2, -2, 0,  1,  -1, 0,  2,  -2,
                                1, -2, 2, -1, -1, 2,  -2, 1,  0, -1, 2,  -2, 2,  -2, 1,  0};
template <class MP>
__device__ __forceinline__ float frt(const MP& m, int k, int i) {
  if constexpr (MP::kConst) return c_t1f[k * 8 + i];
  else return m.f(k, i);
}

// index of coefficient p = k*8+l among the set bits of NZ (its D column)
template <uint64_t NZ>
__host__ __device__ constexpr int nz_index(int p) {
  return popc64t(NZ & ((p == 0) ? 0ull : (~0ull >> (64 - p))));
}

#ifndef ADCT_TC_FFMA2
#define ADCT_TC_FFMA2 0
#endif
// s32 accumulator -> fp32.  ADCT_TC_FBIAS: every accumulator starts at 12582912.0f = 1.5 * 2^23
// (one kind::f16 MMA of two constant tiles, 16 x 1024 x 768, written as f32 bits); the kind::i8
// MMAs then add the integer result to that bit pattern, so D = 0x4B400000 + v is the fp32 number
// 12582912 + v exactly (|v| < 2^22) and the conversion is one subtraction -- packed (FADD2) for
// two values, where I2FP converts one per issue slot.  The epilogue is issue-bound.
#ifndef ADCT_TC_FBIAS
#define ADCT_TC_FBIAS 0  // the f16 bias MMA measured 10 % slower
#endif
constexpr float kTcMagic = 12582912.0f;
#if ADCT_TC_FBIAS
__device__ __forceinline__ float i2f(uint32_t v) { return __uint_as_float(v) - kTcMagic; }  // exact
#else
__device__ __forceinline__ float i2f(uint32_t v) { return __int2float_rn((int32_t)v); }  // exact, |v| < 2^24
#endif

// ---- packed fp32 (FFMA2 / FADD2, sm_100): two columns of a block per instruction -------------
// The epilogue is issue-bound; a packed instruction does two FMAs for one issue slot (its pipe
// occupancy is that of two), so pairing the vertical pass over column pairs cuts issued
// instructions (the A/B in DESIGN.md §5.2).  Same roundings as the scalar code, per element.
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
// c*x + acc for a compile-time coefficient c in {0, +-1, +-2, ...}
template <class M>
__device__ __forceinline__ float2 fmac2(float c, float2 x, float2 acc) {
  if (M::kConst) {
    if (c == 0.0f) return acc;
    if (c == 1.0f) return __fadd2_rn(acc, x);
    if (c == -1.0f) return __fadd2_rn(acc, f2(-x.x, -x.y));
  }
  return __ffma2_rn(f2(c, c), x, acc);
}
template <class M, uint32_t MASK, class C>
__device__ __forceinline__ float2 lsum2(C c, const float2* x) {
  int sd = -1;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (sd < 0 && ((MASK >> i) & 1u) && M::kConst && (c(i) == 1.0f || c(i) == -1.0f)) sd = i;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (sd < 0 && ((MASK >> i) & 1u) && (!M::kConst || c(i) != 0.0f)) sd = i;
  if (sd < 0) return f2(0.0f, 0.0f);
  float2 acc = (M::kConst && c(sd) == 1.0f) ? x[sd]
               : ((M::kConst && c(sd) == -1.0f) ? f2(-x[sd].x, -x[sd].y) : __fmul2_rn(f2(c(sd), c(sd)), x[sd]));
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (i != sd && ((MASK >> i) & 1u)) acc = fmac2<M>(c(i), x[i], acc);
  return acc;
}
template <class M, uint32_t MASK, class C>
__device__ __forceinline__ float2 lsub2(float2 acc, C c, const float2* x) {
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if ((MASK >> i) & 1u) acc = fmac2<M>(-c(i), x[i], acc);
  return acc;
}
// the even half e_i of x = H y (inv8_e) for a column pair
template <class M, uint32_t NZ>
__device__ __forceinline__ void inv8_e2(const M& m, const float2* y, float2* e) {
  constexpr uint32_t EV = NZ & 0x55u;
  constexpr int nev = ((EV & 1u) ? 1 : 0) + ((EV & 4u) ? 1 : 0) + ((EV & 16u) ? 1 : 0) + ((EV & 64u) ? 1 : 0);
  if constexpr (nev <= 2) {
#pragma unroll
    for (int i = 0; i < 4; ++i) e[i] = lsum2<M, EV>([&](int k) { return m.h(i, k); }, y);
  } else {
    float2 ee[2], eo[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      ee[i] = lsum2<M, NZ & 0x11u>([&](int k) { return m.h(i, k); }, y);
      eo[i] = lsum2<M, NZ & 0x44u>([&](int k) { return m.h(i, k); }, y);
    }
    e[0] = __fadd2_rn(ee[0], eo[0]);
    e[3] = __fadd2_rn(ee[0], f2(-eo[0].x, -eo[0].y));
    e[1] = __fadd2_rn(ee[1], eo[1]);
    e[2] = __fadd2_rn(ee[1], f2(-eo[1].x, -eo[1].y));
  }
}
// sum over l in MASK of z_l * (c(0, l), c(1, l)) for scalar z (two outputs per instruction)
template <class M, uint32_t MASK, class C>
__device__ __forceinline__ float2 psum2(C c, const float* z) {
  float2 acc = f2(0.0f, 0.0f);
  bool first = true;
#pragma unroll
  for (int l = 0; l < 8; ++l) {
    if (!((MASK >> l) & 1u)) continue;
    const float a = c(0, l), b = c(1, l);
    if (M::kConst && a == 0.0f && b == 0.0f) continue;
    const float2 zz = f2(z[l], z[l]);
    if (first) {
      acc = (M::kConst && a == 1.0f && b == 1.0f) ? zz : __fmul2_rn(f2(a, b), zz);
      first = false;
    } else {
      acc = (M::kConst && a == 1.0f && b == 1.0f) ? __fadd2_rn(acc, zz) : __ffma2_rn(f2(a, b), zz, acc);
    }
  }
  return acc;
}
// x = H z (one row of the horizontal inverse) as the column pairs (x0,x1), (x2,x3), (x4,x5),
// (x6,x7): e_i over the even inputs, o_i over the odd ones, x_i = e_i + o_i, x_(7-i) = e_i - o_i
template <class M, uint32_t NZ>
__device__ __forceinline__ void inv8_pairs(const M& m, const float* z, float2* x) {
  const float2 e01 = psum2<M, NZ & 0x55u>([&](int i, int l) { return m.h(i, l); }, z);
  const float2 e23 = psum2<M, NZ & 0x55u>([&](int i, int l) { return m.h(2 + i, l); }, z);
  const float2 o01 = psum2<M, NZ & 0xaau>([&](int i, int l) { return m.h(i, l); }, z);
  const float2 o23 = psum2<M, NZ & 0xaau>([&](int i, int l) { return m.h(2 + i, l); }, z);
  x[0] = __fadd2_rn(e01, o01);
  x[1] = __fadd2_rn(e23, o23);
  const float2 d23 = __fadd2_rn(e23, f2(-o23.x, -o23.y)), d01 = __fadd2_rn(e01, f2(-o01.x, -o01.y));
  x[2] = f2(d23.y, d23.x);  // (x4, x5) = (e3 - o3, e2 - o2)
  x[3] = f2(d01.y, d01.x);  // (x6, x7) = (e1 - o1, e0 - o0)
}
#ifndef ADCT_TC_PACKED
#define ADCT_TC_PACKED 1  // 1: packed vertical pass; 2: the horizontal pass too (measured 1.5 % slower)
#endif
// two adjacent accumulators (a pair of s_i / t_i values, laid out as neighbours by tcB) as fp32
__device__ __forceinline__ float2 i2f2(uint32_t a, uint32_t b) {
#if ADCT_TC_FBIAS
  return __fadd2_rn(f2(__uint_as_float(a), __uint_as_float(b)), f2(-kTcMagic, -kTcMagic));
#else
  return f2(i2f(a), i2f(b));
#endif
}
// D column of s_i[j] (t = 0) / t_i[j] (t = 1) among the 64 butterfly columns: columns j = 2jp,
// 2jp + 1 of the same (s/t, i) are neighbours, so a packed conversion reads an aligned pair
#ifndef ADCT_TC_STPAIR
#define ADCT_TC_STPAIR 1
#endif
__host__ __device__ constexpr int st_col(int j, int i, int t) {
  return ADCT_TC_STPAIR ? 16 * (j >> 1) + 8 * t + 2 * i + (j & 1) : 8 * j + 4 * t + i;
}

// ---- one block from its D row (s32 in registers): fp32 inverse and squared error ------------
// yr: the NY coefficient columns; st: s_i[j] at 8j + i, t_i[j] at 8j + 4 + i (unused for r > 32)
template <class MP, int R, int CLIP = 0>
__device__ __forceinline__ float tc_block_sse(const MP& m, const uint32_t* yr, const uint32_t* st) {
  using S = TcShape<R>;
  // CLIP (the reconstruction clipped to [0, 255] before the error, reading A6): the
  // weights carry an extra 1/510, so q, e, o below are 2 x^ / 510 and one saturating add clips
  constexpr float kWs = CLIP ? (1.0f / 510.0f) : 1.0f;
  static_assert(!CLIP || !S::RESID, "the clipped error needs x^ itself: kept form only");
  constexpr uint64_t NZ = S::NZ;
  constexpr uint32_t ROWS = S::ROWS;
  // horizontal inverse of the weighted coefficients, Q = (W o Y') T, rows in ROWS
  float q[8][8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (!((ROWS >> k) & 1u)) continue;
    float z[8];
#pragma unroll
    for (int l = 0; l < 8; ++l)
      z[l] = ((NZ >> (k * 8 + l)) & 1ull) ? i2f(yr[nz_index<NZ>(k * 8 + l)]) * (m.wy2(k, l) * kWs) : 0.0f;
#define ADCT_TC_ROWINV(K)                                              \
  if (k == K) {                                                        \
    constexpr uint32_t rm = (uint32_t)((NZ >> (8 * K)) & 0xffull);     \
    if constexpr (rm != 0) inv8<MP, rm>(m, z, q[K]);                   \
  }
    ADCT_TC_ROWINV(0) ADCT_TC_ROWINV(1) ADCT_TC_ROWINV(2) ADCT_TC_ROWINV(3)
    ADCT_TC_ROWINV(4) ADCT_TC_ROWINV(5) ADCT_TC_ROWINV(6) ADCT_TC_ROWINV(7)
#undef ADCT_TC_ROWINV
  }
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#if ADCT_TC_FFMA2
  float2 acc2[4] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
#endif
#if ADCT_TC_PACKED
  if constexpr (!S::RESID) {
#if ADCT_TC_PACKED >= 2
    // the horizontal inverse again, straight into column pairs (q above is then dead code)
    float2 q2[8][4];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (!((ROWS >> k) & 1u)) continue;
      float z[8];
#pragma unroll
      for (int l = 0; l < 8; ++l)
        z[l] = ((NZ >> (k * 8 + l)) & 1ull) ? i2f(yr[nz_index<NZ>(k * 8 + l)]) * m.wy2(k, l) : 0.0f;
#define ADCT_TC_ROWINV2(K)                                             \
  if (k == K) {                                                        \
    constexpr uint32_t rm = (uint32_t)((NZ >> (8 * K)) & 0xffull);     \
    if constexpr (rm != 0) inv8_pairs<MP, rm>(m, z, q2[K]);            \
  }
      ADCT_TC_ROWINV2(0) ADCT_TC_ROWINV2(1) ADCT_TC_ROWINV2(2) ADCT_TC_ROWINV2(3)
      ADCT_TC_ROWINV2(4) ADCT_TC_ROWINV2(5) ADCT_TC_ROWINV2(6) ADCT_TC_ROWINV2(7)
#undef ADCT_TC_ROWINV2
    }
#endif
    // vertical inverse fused with the error, two columns (j, j + 1) per packed instruction
    float2 a2[4] = {f2(0.0f, 0.0f), f2(0.0f, 0.0f), f2(0.0f, 0.0f), f2(0.0f, 0.0f)};
#pragma unroll
    for (int jp = 0; jp < 4; ++jp) {
      const int j0 = 2 * jp, j1 = 2 * jp + 1;
      float2 col[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
#if ADCT_TC_PACKED >= 2
        col[k] = ((ROWS >> k) & 1u) ? q2[k][jp] : f2(0.0f, 0.0f);
#else
        col[k] = ((ROWS >> k) & 1u) ? f2(q[k][j0], q[k][j1]) : f2(0.0f, 0.0f);
#endif
      float2 e[4];
      inv8_e2<MP, ROWS>(m, col, e);
      if constexpr (CLIP != 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 sv = i2f2(st[st_col(j0, i, 0)], st[st_col(j1, i, 0)]);
          const float2 tv = i2f2(st[st_col(j0, i, 1)], st[st_col(j1, i, 1)]);
          const float2 o = lsum2<MP, ROWS & 0xaau>([&](int k) { return m.h(i, k); }, col);
          // clip(2 x^_i, 0, 510) / 510 and the same for x^_(7-i): one FADD.SAT each
          const float2 ca = f2(__saturatef(e[i].x + o.x), __saturatef(e[i].y + o.y));
          const float2 cb = f2(__saturatef(e[i].x - o.x), __saturatef(e[i].y - o.y));
          // 2 (x_i - clip x^_i) = (s_i + t_i) - 510 ca, 2 (x_(7-i) - clip x^_(7-i)) = (s_i - t_i) - 510 cb
          const float2 da = __ffma2_rn(ca, f2(-510.0f, -510.0f), __fadd2_rn(sv, tv));
          const float2 db = __ffma2_rn(cb, f2(-510.0f, -510.0f), __fadd2_rn(sv, f2(-tv.x, -tv.y)));
          a2[i] = __ffma2_rn(da, da, a2[i]);
          a2[i] = __ffma2_rn(db, db, a2[i]);
        }
        continue;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 sv = i2f2(st[st_col(j0, i, 0)], st[st_col(j1, i, 0)]);
        const float2 tv = i2f2(st[st_col(j0, i, 1)], st[st_col(j1, i, 1)]);
        const float2 dp = __fadd2_rn(sv, f2(-e[i].x, -e[i].y));
        const float2 dm = lsub2<MP, ROWS & 0xaau>(tv, [&](int k) { return m.h(i, k); }, col);
        a2[i] = __ffma2_rn(dp, dp, a2[i]);
        a2[i] = __ffma2_rn(dm, dm, a2[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = a2[i].x + a2[i].y;
    return (CLIP ? 0.25f : 0.5f) * ((acc[0] + acc[1]) + (acc[2] + acc[3]));
  }
#endif
  static_assert(!CLIP || ADCT_TC_PACKED == 1, "the clipped epilogue is written for the packed vertical pass");
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float col[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) col[k] = ((ROWS >> k) & 1u) ? q[k][j] : 0.0f;
    if constexpr (S::RESID) {  // x - x^ = inverse of the dropped coefficients
      float e[4], o[4];
      inv8_eo<MP, ROWS>(m, col, e, o);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[i] = fmaf(e[i], e[i], acc[i]);
        acc[i] = fmaf(o[i], o[i], acc[i]);
      }
    } else {
      float e[4];
      inv8_e<MP, ROWS>(m, col, e);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float dp = i2f(st[st_col(j, i, 0)]) - e[i];
        const float dm = lsub<MP, 8, ROWS & 0xaau>(i2f(st[st_col(j, i, 1)]), [&](int k) { return m.h(i, k); }, col);
#if ADCT_TC_FFMA2  // A/B: the two squares as one packed FFMA2 (half the issued instructions, same datapath)
        acc2[i] = __ffma2_rn(make_float2(dp, dm), make_float2(dp, dm), acc2[i]);
#else
        acc[i] = fmaf(dp, dp, acc[i]);
        acc[i] = fmaf(dm, dm, acc[i]);
#endif
      }
    }
  }
#if ADCT_TC_FFMA2
  if constexpr (!S::RESID) {
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = acc2[i].x + acc2[i].y;
  }
#endif
  return 0.5f * ((acc[0] + acc[1]) + (acc[2] + acc[3]));
}

// ---- the CTA's tiles: chunks cg = blockIdx.x, +gridDim.x, ...; a chunk is kTcChunkTiles
// consecutive tiles of one image (fewer at the image's end), taken in order ------------------
struct TcArgs {
  int32_t tpr, tpi, cpi;  // tiles per tile row, per image; chunks per image
  int32_t ct;             // tiles per chunk (tc_chunk_tiles)
  uint32_t n_chunks;
  FastDiv dcpi, dtpr;
  int32_t dmain, dlast, dc0;  // donor tiles (CW = 15): main tiles per image; the leftover tile's band, first chunk
};

__device__ __forceinline__ int32_t chunk_tiles(const TcArgs& a, uint32_t cg, uint32_t& img, int32_t& tt0) {
  img = fdiv(cg, a.dcpi);
  tt0 = (int32_t)(cg - img * (uint32_t)a.cpi) * a.ct;
  return min(a.ct, a.tpi - tt0);
}

struct TcPf {  // the TMA producer's walk: coordinates of the next tile to load
  uint32_t cg, img;
  int32_t j, n, trow, tcol;
  int32_t dband, dchunk;  // donor tiles: the donor chunk-band of tile trow
};
__device__ __forceinline__ void pf_enter(const TcArgs& a, TcPf& f) {
  if (f.cg >= a.n_chunks) return;
  int32_t tt0;
  f.n = chunk_tiles(a, f.cg, f.img, tt0);
  f.j = 0;
  f.trow = (int32_t)fdiv((uint32_t)tt0, a.dtpr);
  f.tcol = tt0 - f.trow * a.tpr;
  f.dband = a.dmain + tt0 / 15;  // (donor tiles only; once per chunk)
  f.dchunk = tt0 % 15;
}
__device__ __forceinline__ void pf_next(const TcArgs& a, TcPf& f) {
  if (++f.j < f.n) {
    if (++f.tcol == a.tpr) {
      f.tcol = 0;
      ++f.trow;
    }
    if (++f.dchunk == 15) {
      f.dchunk = 0;
      ++f.dband;
    }
  } else {
    f.cg += gridDim.x;
    pf_enter(a, f);
  }
}

__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2,
                                            int32_t c3, int32_t c4, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], "
      "[%7];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
      : "memory");
}

// CW = 15 is the donor tiling of 15-chunk rows (1920-byte planes, config 4's chroma): main tile
// b < dmain is band b's 15 chunk-bands (one box of the main map) plus one chunk-band of a donor
// band (a 1-chunk box of the donor map into the tile's 16th KB); donors are the last
// ceil(bands / 16) bands, taken in order, and what is left of them (at most 15 chunk-bands, all
// in the last band) is one more tile, its 16th KB a fully out-of-bounds box (zero fill).  So a
// 1920 x 1080 plane is 127 tiles instead of 135 with a 1/16 zero fill each.
template <class MP, int R, int CW, int CLIP = 0>
__global__ void __launch_bounds__(kTcThreads, 1)
    fused_u8_tc_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap tmap_d, TcArgs a,
                       DevMat dm, double* __restrict__ partial) {
  using S = TcShape<R>;
  constexpr int N = S::N, NB = S::NB;
  constexpr bool DON = CW == 15;
  constexpr int BH = DON ? 1 : 16 / CW;  // bands per tile
  // kind::i8: D s32 (2 << 4), A u8 (0 << 7), B s8 (1 << 10), both K-major, N >> 3, M >> 4
  // each tile is two MMA sets of N = NB (half h: block 2p + h of every pair), each into its own
  // TMEM half-stage, so an epilogue warp releases block 2p's columns before it computes
  constexpr uint32_t kIdesc = (2u << 4) | (1u << 10) | ((uint32_t)(NB >> 3) << 17) | (8u << 24);
  constexpr uint32_t kTmemCols = 512;
  static_assert(2 * kTcDStages * NB <= (int)kTmemCols, "TMEM columns");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  pdl_launch_dependents();  // the next launch may start its prologue as our CTAs retire
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = w & 3;  // TMEM lane quarter of this warp (hardware: warp w accesses lanes 32 (w % 4) ..)
  uint8_t* sB = smem + (size_t)kTcSlots * kTcTileBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kTcBBytes);  // [kTcSlots]  TMA tile landed
  uint64_t* sfree = full + kTcSlots;                              // [kTcSlots]  MMA done reading the tile
  uint64_t* dfull = sfree + kTcSlots;                             // [2D] MMA done writing a half-stage
  uint64_t* dfree = dfull + 2 * kTcDStages;                       // [2D] half-stage read by 4 epilogue warps
  uint32_t* holder = reinterpret_cast<uint32_t*>(dfree + 2 * kTcDStages);
#if ADCT_TC_FBIAS
  // the two constant f16 operands of the bias MMA: A' = 1024 (128 rows x 16), B' = 768 (96 x 16)
  uint32_t* cbias = reinterpret_cast<uint32_t*>(
      smem + (((size_t)kTcSlots * kTcTileBytes + kTcBBytes + (size_t)kTcBars * 8 + 16 + 127) & ~(size_t)127));
  for (int i = threadIdx.x; i < (kTcBiasA + kTcBiasB) / 4; i += kTcThreads)
    cbias[i] = i < kTcBiasA / 4 ? 0x64006400u : 0x62006200u;
#endif
  const MP m(dm);

  // B in the canonical K-major no-swizzle layout: core matrix (n/8, k/16) at (n/8)*1024 + (k/16)*128;
  // one thread per (output n, pixel row i) writes that 16-byte row (both blocks of the pair; the
  // other block's 8 bytes are 0).  Part of every launch's ramp, so no local-memory arrays.
  for (int idx = threadIdx.x; idx < N * 8; idx += kTcThreads) {
    const int n = idx >> 3, i = idx & 7;
    const int blk = n / NB, o = n % NB;
    int pk = -1, pl = -1, sj = -1, sr = -1;
    if (o < S::NNZ) {
      int cnt = -1;
#pragma unroll 1
      for (int p = 0; p < 64; ++p)
        if (((S::NZ >> p) & 1ull) && ++cnt == o) {
          pk = p >> 3;
          pl = p & 7;
          break;
        }
    } else if (o >= S::NY) {  // inverse of st_col: column j of s_r (sr < 4) / t_(sr-4)
      const int id = o - S::NY;
      sj = ADCT_TC_STPAIR ? 2 * (id >> 4) + (id & 1) : id >> 3;
      sr = ADCT_TC_STPAIR ? 4 * ((id >> 3) & 1) + ((id >> 1) & 3) : id & 7;
    }
    const float fki = pk >= 0 ? frt(m, pk, i) : 0.0f;
    uint32_t lo = 0u, hi = 0u;  // bytes j = 0..3 and 4..7 of this block's 8
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int v = 0;
      if (pk >= 0) v = (int)lrintf(fki * frt(m, pl, j));
      else if (sj == j) v = sr < 4 ? ((i == sr || i == 7 - sr) ? 1 : 0) : (i == sr - 4 ? 1 : (i == 11 - sr ? -1 : 0));
      const uint32_t b = (uint32_t)(uint8_t)(int8_t)v;
      if (j < 4) lo |= b << (8 * j);
      else hi |= b << (8 * (j - 4));
    }
    *reinterpret_cast<uint4*>(sB + (n >> 3) * 1024 + i * 128 + (n & 7) * 16) =
        blk ? make_uint4(0u, 0u, lo, hi) : make_uint4(lo, hi, 0u, 0u);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kTcSlots; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&sfree[i], 1);
    }
    for (int i = 0; i < 2 * kTcDStages; ++i) {
      mbar_init(&dfull[i], 1);
      mbar_init(&dfree[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (w == 0) tmem_alloc<kTmemCols>(smem_u32(holder));  // warp 0 allocates and frees
  fence_proxy_async();  // B written through the generic proxy, read by the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *holder;
  pdl_wait();  // the previous kernel of the stream has completed: inputs ready, partials free
  const uint32_t full0 = smem_u32(full), ring0 = smem_u32(smem), sB_u = smem_u32(sB);

  if (w == kTcEpiWarps + kTcIssuers) {
    // ======== TMA producer: one 16 KB tile per slot, refilled when its MMA has completed ========
    TcPf pf;
    pf.cg = blockIdx.x;
    pf_enter(a, pf);
    uint32_t slot = 0, sph = 0, t = 0;
#pragma unroll 1
    for (; pf.cg < a.n_chunks; ++t) {
      if (t >= (uint32_t)kTcSlots) mbar_wait_sleep(&sfree[slot], sph ^ 1u);  // MMA of tile t - kTcSlots done
      if (elect_one()) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full0 + slot * 8),
                     "r"((uint32_t)kTcTileBytes)
                     : "memory");
        if constexpr (DON) {
          const bool main = pf.trow < a.dmain;
          tma_load_5d(ring0 + slot * kTcTileBytes, &tmap, 0, 0, main ? pf.trow : a.dlast, main ? 0 : a.dc0,
                      (int32_t)pf.img, full0 + slot * 8);
          tma_load_5d(ring0 + slot * kTcTileBytes + 15 * 1024, &tmap_d, 0, 0, main ? pf.dband : 0,
                      main ? pf.dchunk : 15, (int32_t)pf.img, full0 + slot * 8);
        } else {
          tma_load_5d(ring0 + slot * kTcTileBytes, &tmap, 0, 0, pf.trow * BH, pf.tcol * CW, (int32_t)pf.img,
                      full0 + slot * 8);
        }
      }
      __syncwarp();
      pf_next(a, pf);
      if (++slot == kTcSlots) {
        slot = 0;
        sph ^= 1u;
      }
    }
  } else if (w >= kTcEpiWarps) {
    // ======== MMA issuers: warp kTcEpiWarps + i issues the 4 MMAs of the tiles t = i (mod kTcIssuers) ========
    const uint32_t iss = (uint32_t)(w - kTcEpiWarps);
    // descriptors of slot 0 / k-step 0: the others differ only in the start address (bits 0-13)
    const uint64_t adesc0 = smem_desc_kmajor(ring0, 128, 1024), bdesc0 = smem_desc_kmajor(sB_u, 128, 1024);
#if ADCT_TC_FBIAS
    // uniform constant tiles: any layout reads the same values (LBO 128, SBO 256 stay inside)
    const uint64_t adescc = smem_desc_kmajor(smem_u32(cbias), 128, 256);
    const uint64_t bdescc = smem_desc_kmajor(smem_u32(cbias) + kTcBiasA, 128, 256);
    constexpr uint32_t kIdescF16 = idesc_f16_f32<128, NB>();
#endif
    uint32_t t = 0;
#pragma unroll 1
    for (uint32_t cg = blockIdx.x; cg < a.n_chunks; cg += gridDim.x) {
      uint32_t img;
      int32_t tt0;
      const int32_t n = chunk_tiles(a, cg, img, tt0);
      const int32_t j0 = (int32_t)((iss + kTcIssuers - t % kTcIssuers) % kTcIssuers);
#pragma unroll 1
      for (int32_t j = j0; j < n; j += kTcIssuers) {
        const uint32_t tt = t + (uint32_t)j;
        const uint32_t slot = tt % kTcSlots, ds = tt % kTcDStages, dpar = ((tt / kTcDStages) & 1u) ^ 1u;
        mbar_wait_sleep(&full[slot], (tt / kTcSlots) & 1u);  // pixels landed
        const uint64_t ad = adesc0 + (uint64_t)(slot * (kTcTileBytes >> 4));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t hs = 2 * ds + (uint32_t)h;
          if (tt >= (uint32_t)kTcDStages) mbar_wait_sleep(&dfree[hs], dpar);  // tile tt - D's half h read
          tc_fence_after();
          if (elect_one()) {
#if ADCT_TC_ABL >= 3  // ablation build: no MMA, the ring only (pure TMA stream rate)
            mbar_arrive(&dfull[hs]);
            if (h == 1) mbar_arrive(&sfree[slot]);
#else
            const uint32_t td = tbase + (uint32_t)NB * hs;
#if ADCT_TC_FBIAS
            mma_f16_ss(td, adescc, bdescc, kIdescF16, 0u);  // D := 16 x 1024 x 768 = 1.5 * 2^23 (f32 bits)
#endif
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_i8_ss(td, ad + (uint64_t)(kk * 16), bdesc0 + (uint64_t)(h * (NB / 8) * 64 + kk * 16), kIdesc,
                        (ADCT_TC_FBIAS || kk > 0) ? 1u : 0u);
            mma_commit(smem_u32(&dfull[hs]));                // half h of tile tt written
            if (h == 1) mma_commit(smem_u32(&sfree[slot]));  // the slot may be refilled
#endif
          }
          __syncwarp();
        }
      }
      t += (uint32_t)n;
    }
  } else {
    // ======== epilogue warps: quarter q, index e; tiles t = e, e + kTcEpi, ... of the CTA ========
    const int e = w >> 2;
    const uint32_t lane_q = (uint32_t)(32 * q) << 16;
    uint32_t t = 0;
#pragma unroll 1
    for (uint32_t cg = blockIdx.x; cg < a.n_chunks; cg += gridDim.x) {
      uint32_t img;
      int32_t tt0;
      const int32_t n = chunk_tiles(a, cg, img, tt0);
      // this warp takes the chunk's tiles j = sl, sl + kTcEpi, ... (sl fixed by where the chunk
      // starts in the CTA's sequence); partial slot sl depends on the geometry only
      const int32_t sl = (int32_t)(((uint32_t)e + kTcEpi - t % kTcEpi) % kTcEpi);
      float acc = 0.0f;
#pragma unroll 1
      for (int32_t j = sl; j < n; j += kTcEpi) {
        const uint32_t tt = t + (uint32_t)j;
        const uint32_t d = tt % kTcDStages, dpar = (tt / kTcDStages) & 1u;
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // block 2p + h from half-stage 2d + h
          const uint32_t hs = 2 * d + (uint32_t)h;
          mbar_wait_sleep(&dfull[hs], dpar);
          tc_fence_after();
          const uint32_t tD = tbase + lane_q + (uint32_t)(NB * hs);
          uint32_t yr[S::NY], st[64];
#if ADCT_TC_ABL >= 2  // ablation build: no TMEM load and no epilogue arithmetic
          __syncwarp();
          if (lane == 0) mbar_arrive(&dfree[hs]);
          acc += (float)tD;
          continue;
#endif
          if constexpr (S::NY == 16) tmem_ld16(tD, yr);
          else tmem_ld32(tD, yr);
          if constexpr (!S::RESID) {
            tmem_ld32(tD + S::NY, *reinterpret_cast<uint32_t(*)[32]>(&st[0]));
            tmem_ld32(tD + S::NY + 32, *reinterpret_cast<uint32_t(*)[32]>(&st[32]));
          }
          tmem_wait_ld(yr);
          if constexpr (!S::RESID) tmem_wait_ld(st);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&dfree[hs]);  // the MMA of tile tt + D may overwrite the half-stage
#if ADCT_TC_ABL >= 1  // ablation build: TMEM load, no epilogue arithmetic
          acc += i2f(yr[0]) + i2f(st[0]);
          continue;
#endif
          acc += tc_block_sse<MP, R, CLIP>(m, yr, st);
        }
      }
      float v = acc;  // fixed shuffle order: the partial depends on the geometry only
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) partial[((int64_t)cg * kTcEpi + sl) * 4 + q] = (double)v;
      t += (uint32_t)n;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<kTmemCols>(tbase);
}

// ---- config 3 on the tensor core: forward + uniform quantiser, u8 planes -> int16 block-major --
// The same pipeline as fused_u8_tc_kernel (TMA tile = the kind::i8 MMA's A operand, 3 MMA issuers,
// 12 epilogue warps) with B = all 64 coefficients of both blocks of a pair (N = 64 per half, every
// Y_kl exact in s32) and an epilogue that quantises (quant.cuh) and writes the block's 128 bytes
// through a swizzled staging row and one TMA store per (warp, half tile).  Tiles are 1 chunk x 16
// bands, so TMEM lane p = 8 (band - band0) + pair: the 32 lanes of an epilogue warp are 4 bands x 8
// pairs, and with the output viewed as {64 codes, 2 halves, W/16 pairs, H/8 bands, images} their
// blocks 2 pair + h are one box {64, 1, 8, 4, 1} whose rows are the warp's lanes in order.
constexpr int kTqSlots = 9;
static_assert(kTqSlots % kTcWays == 0, "slot s only ever holds tiles of issuer s % kTcWays");
constexpr int kTqNB = 64;
constexpr int kTqStageBytes = 4096;  // 32 blocks x 128 B per epilogue warp
constexpr int kTqBBytes = 2 * kTqNB * 128;
constexpr int kTqBars = 2 * kTqSlots + 4 * kTcDStages;
constexpr size_t kTqSmem = (size_t)kTqSlots * kTcTileBytes + (size_t)kTcEpiWarps * kTqStageBytes + kTqBBytes +
                           (size_t)kTqBars * 8 + 16 + 1024;
static_assert(kTqSmem <= 227 * 1024, "quantiser tensor-core kernel exceeds shared memory");

__global__ void __launch_bounds__(kTcThreads, 1)
    fwd_quant_tc_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap tout, TcArgs a,
                        QTab qt, float stepf, int32_t bh) {
  constexpr int NB = kTqNB;
  constexpr uint32_t kIdesc = (2u << 4) | (1u << 10) | ((uint32_t)(NB >> 3) << 17) | (8u << 24);
  constexpr uint32_t kTmemCols = 512;
  static_assert(2 * kTcDStages * NB <= (int)kTmemCols, "TMEM columns");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = w & 3;
  uint8_t* stage = smem + (size_t)kTqSlots * kTcTileBytes;
  uint8_t* sB = stage + (size_t)kTcEpiWarps * kTqStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kTqBBytes);
  uint64_t* sfree = full + kTqSlots;
  uint64_t* dfull = sfree + kTqSlots;
  uint64_t* dfree = dfull + 2 * kTcDStages;
  uint32_t* holder = reinterpret_cast<uint32_t*>(dfree + 2 * kTcDStages);
  // B: row n = 64 blk + 8 k + l holds T_ki T_lj at byte 16 i + 8 blk + j (|b| <= 4)
  for (int idx = threadIdx.x; idx < 2 * NB * 8; idx += kTcThreads) {
    const int n = idx >> 3, i = idx & 7;
    const int blk = n / NB, o = n % NB;
    const float fki = c_t1f[(o >> 3) * 8 + i];
    uint32_t lo = 0u, hi = 0u;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t b = (uint32_t)(uint8_t)(int8_t)(int)lrintf(fki * c_t1f[(o & 7) * 8 + j]);
      if (j < 4) lo |= b << (8 * j);
      else hi |= b << (8 * (j - 4));
    }
    *reinterpret_cast<uint4*>(sB + (n >> 3) * 1024 + i * 128 + (n & 7) * 16) =
        blk ? make_uint4(0u, 0u, lo, hi) : make_uint4(lo, hi, 0u, 0u);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kTqSlots; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&sfree[i], 1);
    }
    for (int i = 0; i < 2 * kTcDStages; ++i) {
      mbar_init(&dfull[i], 1);
      mbar_init(&dfree[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (w == 0) tmem_alloc<kTmemCols>(smem_u32(holder));
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *holder;
  const uint32_t full0 = smem_u32(full), ring0 = smem_u32(smem), sB_u = smem_u32(sB);

  if (w == kTcEpiWarps + kTcIssuers) {
    // ======== TMA producer ========
    TcPf pf;
    pf.cg = blockIdx.x;
    pf_enter(a, pf);
    uint32_t slot = 0, sph = 0, t = 0;
#pragma unroll 1
    for (; pf.cg < a.n_chunks; ++t) {
      if (t >= (uint32_t)kTqSlots) mbar_wait_sleep(&sfree[slot], sph ^ 1u);
      if (elect_one()) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full0 + slot * 8),
                     "r"((uint32_t)kTcTileBytes)
                     : "memory");
        tma_load_5d(ring0 + slot * kTcTileBytes, &tmap, 0, 0, pf.trow * 16, pf.tcol, (int32_t)pf.img,
                    full0 + slot * 8);
      }
      __syncwarp();
      pf_next(a, pf);
      if (++slot == kTqSlots) {
        slot = 0;
        sph ^= 1u;
      }
    }
  } else if (w >= kTcEpiWarps) {
    // ======== MMA issuers ========
    const uint32_t iss = (uint32_t)(w - kTcEpiWarps);
    const uint64_t adesc0 = smem_desc_kmajor(ring0, 128, 1024), bdesc0 = smem_desc_kmajor(sB_u, 128, 1024);
    uint32_t t = 0;
#pragma unroll 1
    for (uint32_t cg = blockIdx.x; cg < a.n_chunks; cg += gridDim.x) {
      uint32_t img;
      int32_t tt0;
      const int32_t n = chunk_tiles(a, cg, img, tt0);
      const int32_t j0 = (int32_t)((iss + kTcIssuers - t % kTcIssuers) % kTcIssuers);
#pragma unroll 1
      for (int32_t j = j0; j < n; j += kTcIssuers) {
        const uint32_t tt = t + (uint32_t)j;
        const uint32_t slot = tt % kTqSlots, ds = tt % kTcDStages, dpar = ((tt / kTcDStages) & 1u) ^ 1u;
        mbar_wait_sleep(&full[slot], (tt / kTqSlots) & 1u);
        const uint64_t ad = adesc0 + (uint64_t)(slot * (kTcTileBytes >> 4));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t hs = 2 * ds + (uint32_t)h;
          if (tt >= (uint32_t)kTcDStages) mbar_wait_sleep(&dfree[hs], dpar);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t td = tbase + (uint32_t)NB * hs;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_i8_ss(td, ad + (uint64_t)(kk * 16), bdesc0 + (uint64_t)(h * (NB / 8) * 64 + kk * 16), kIdesc,
                        kk > 0 ? 1u : 0u);
            mma_commit(smem_u32(&dfull[hs]));
            if (h == 1) mma_commit(smem_u32(&sfree[slot]));
          }
          __syncwarp();
        }
      }
      t += (uint32_t)n;
    }
  } else {
    // ======== epilogue warps ========
    const int e = w >> 2;
    const uint32_t lane_q = (uint32_t)(32 * q) << 16;
    const uint32_t stg = smem_u32(stage) + (uint32_t)w * kTqStageBytes;
    const float qru[4] = {qt.ru[0], qt.ru[1], qt.ru[2], qt.ru[3]};
    const float qri[2] = {qt.ri[0], qt.ri[1]};
    uint32_t t = 0;
#pragma unroll 1
    for (uint32_t cg = blockIdx.x; cg < a.n_chunks; cg += gridDim.x) {
      uint32_t img;
      int32_t tt0;
      const int32_t n = chunk_tiles(a, cg, img, tt0);
      const int32_t sl = (int32_t)(((uint32_t)e + kTcEpi - t % kTcEpi) % kTcEpi);
#pragma unroll 1
      for (int32_t j = sl; j < n; j += kTcEpi) {
        const uint32_t tt = t + (uint32_t)j;
        const uint32_t d = tt % kTcDStages, dpar = (tt / kTcDStages) & 1u;
        const int32_t trow = (int32_t)fdiv((uint32_t)(tt0 + j), a.dtpr);
        const int32_t tcol = tt0 + j - trow * a.tpr;
        const int32_t band0 = trow * 16 + 4 * q;  // this warp's 4 bands
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          const uint32_t hs = 2 * d + (uint32_t)h;
          mbar_wait_sleep(&dfull[hs], dpar);
          tc_fence_after();
          const uint32_t tD = tbase + lane_q + (uint32_t)(NB * hs);
          uint32_t yr[64];
          tmem_ld32(tD, *reinterpret_cast<uint32_t(*)[32]>(&yr[0]));
          tmem_ld32(tD + 32, *reinterpret_cast<uint32_t(*)[32]>(&yr[32]));
          tmem_wait_ld(yr);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&dfree[hs]);
          if (band0 >= bh) continue;  // below the image: zero fill, nothing to write (warp-uniform)
          float y[64];
#pragma unroll
          for (int c = 0; c < 64; ++c) y[c] = __int2float_rn((int32_t)yr[c]);  // exact, |Y| <= 18360
          uint32_t packed[32];
          q_block_t1(y, qru, qri, stepf, qt, packed);
          if (lane == 0) bulk_wait_read<0>();  // the staging rows are free once the previous store read them
          __syncwarp();
#pragma unroll
          for (int k = 0; k < 8; ++k)
            sts128(stg + (uint32_t)lane * 128u + (((uint32_t)k ^ ((uint32_t)lane & 7u)) << 4),
                   make_uint4(packed[4 * k], packed[4 * k + 1], packed[4 * k + 2], packed[4 * k + 3]));
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tma_store_5d(&tout, 0, h, tcol * 8, band0, (int32_t)img, stg);
            bulk_commit();
          }
        }
      }
      t += (uint32_t)n;
    }
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<kTmemCols>(tbase);
}

template <class MP, int R, int CW, int CLIP = 0>
bool launch_tc_rc(const CUtensorMap& map, const CUtensorMap& map_d, const TcArgs& a, const DevMat& dm, double* partial,
                  cudaStream_t st) {
  // the shared-memory opt-in is a per-device function attribute: set it once per device
  static std::mutex mu;
  static int8_t state[kMaxDevices] = {};
  if (!once_per_device(mu, state, [] {
        return cudaFuncSetAttribute(fused_u8_tc_kernel<MP, R, CW, CLIP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)kTcSmem) == cudaSuccess;
      }))
    return false;
  const int64_t grid = (int64_t)a.n_chunks < sms_s() ? (int64_t)a.n_chunks : sms_s();
  if (launch_pdl(fused_u8_tc_kernel<MP, R, CW, CLIP>, dim3((unsigned)grid), dim3(kTcThreads), kTcSmem, st, map, map_d, a,
                 dm, partial) != cudaSuccess)
    return false;
  return true;
}

template <class MP, int R, int CLIP = 0>
bool launch_tc_r(int cw, const CUtensorMap& map, const CUtensorMap& map_d, const TcArgs& a, const DevMat& dm,
                 double* partial, cudaStream_t st) {
  switch (cw) {
    case 2: return launch_tc_rc<MP, R, 2, CLIP>(map, map_d, a, dm, partial, st);
    case 1: return launch_tc_rc<MP, R, 1, CLIP>(map, map_d, a, dm, partial, st);
    case 16: return launch_tc_rc<MP, R, 16, CLIP>(map, map_d, a, dm, partial, st);
    case 15: return launch_tc_rc<MP, R, 15, CLIP>(map, map_d, a, dm, partial, st);
    default: return false;
  }
}

// compiled (matrix, r) pairs: T1 at config 4's r = 10, the Lena figures' r = 3, 14
// and the other transpose-symmetric zig-zag prefixes that fit the accumulator budget (r <= 16 kept
// coefficients, or r > 32 with at most 32 dropped: reading A5 lists the symmetric prefixes):
// 1, 6, 15 and 36; runtime integer matrices at r = 10.  Any other r takes the SIMT kernels.
constexpr bool tc_r_compiled(int r) { return r == 1 || r == 3 || r == 6 || r == 10 || r == 14 || r == 15 || r == 36; }
template <class MP>
bool launch_tc(int r, int cw, const CUtensorMap& map, const CUtensorMap& map_d, const TcArgs& a, const DevMat& dm,
               double* partial, cudaStream_t st, int clip) {
  if (clip) {  // ADCT_CLIP (the SPEC's metric policy): T1 at config 4's r
    if constexpr (MP::kConst) return r == 10 && launch_tc_r<MP, 10, 1>(cw, map, map_d, a, dm, partial, st);
    else return false;
  }
  if constexpr (!MP::kConst) {
    return r == 10 && launch_tc_r<MP, 10>(cw, map, map_d, a, dm, partial, st);
  } else {
    switch (r) {
      case 1: return launch_tc_r<MP, 1>(cw, map, map_d, a, dm, partial, st);
      case 3: return launch_tc_r<MP, 3>(cw, map, map_d, a, dm, partial, st);
      case 6: return launch_tc_r<MP, 6>(cw, map, map_d, a, dm, partial, st);
      case 10: return launch_tc_r<MP, 10>(cw, map, map_d, a, dm, partial, st);
      case 14: return launch_tc_r<MP, 14>(cw, map, map_d, a, dm, partial, st);
      case 15: return launch_tc_r<MP, 15>(cw, map, map_d, a, dm, partial, st);
      case 36: return launch_tc_r<MP, 36>(cw, map, map_d, a, dm, partial, st);
      default: return false;
    }
  }
}

// 5-D map {128 B, 8 rows, bands, chunks, images}, strides {row, 8 rows, 128 B, image}; box of
// bh bands x cw chunks
bool make_tc_tmap(CUtensorMap* map, const uint8_t* src, const adct_geom& g, int bh, int cw, bool promo128 = false) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  const int64_t istride = g.n_images > 1 ? g.image_stride : (int64_t)g.height * g.row_stride;
  const cuuint64_t dims[5] = {128, 8, (cuuint64_t)(g.height / 8), (cuuint64_t)(g.width / 128),
                              (cuuint64_t)g.n_images};
  const cuuint64_t strides[4] = {(cuuint64_t)g.row_stride, (cuuint64_t)(8 * g.row_stride), 128, (cuuint64_t)istride};
  const cuuint32_t box[5] = {128, 8, (cuuint32_t)bh, (cuuint32_t)cw, 1};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, const_cast<uint8_t*>(src), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             // one-chunk boxes: 256-byte promotion would pull the neighbouring chunk too (blockmajor.cu)
             promo128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// tile shape of the tensor-core kernel: CW 128-byte chunks x 16/CW bands, the CW in {2, 16, 1}
// with the fewest tiles (zero-filled parts of edge tiles cost MMA rows, never HBM bytes), or the
// donor tiling (CW = 15) of 15-chunk rows
TcPlan tc_plan(const adct_geom& g) {
  TcPlan p{};
  if (g.width <= 0 || g.height <= 0 || (g.width % 128) != 0) return p;  // whole 128-byte chunks only
  const int64_t nch = g.width / 128, nbd = g.height / 8;
  int64_t best = -1;
  static const int force_cw = [] {  // A/B hook: ADCT_TC_CW=1|2|16|15 forces the tile shape
    const char* e = std::getenv("ADCT_TC_CW");
    return e ? std::atoi(e) : 0;
  }();
  for (int cw : {2, 16, 1, 15}) {
    if (force_cw && cw != force_cw) continue;
    int64_t tiles;
    if (cw == 15) {
      static const bool no_donor = std::getenv("ADCT_TC_NODONOR") != nullptr;  // A/B hook
      if (nch != 15 || no_donor) continue;
      const int64_t d = (nbd + 15) / 16;  // donor bands
      tiles = (nbd - d) + ((16 * d - nbd) > 0 ? 1 : 0);
    } else {
      const int64_t bh = 16 / cw;
      tiles = ((nch + cw - 1) / cw) * ((nbd + bh - 1) / bh);
    }
    if (best < 0 || tiles < best) {
      best = tiles;
      p.cw = cw;
    }
  }
  if (p.cw == 0) return p;
  if (p.cw == 15) {
    const int64_t d = (nbd + 15) / 16;
    p.dmain = (int32_t)(nbd - d);
    p.dlast = (int32_t)(nbd - 1);
    p.dc0 = (int32_t)(p.dmain - 15 * (d - 1));
    p.tpr = 1;
    p.tpi = (int32_t)best;
  } else {
    p.tpr = (int32_t)((nch + p.cw - 1) / p.cw);
    p.tpi = (int32_t)(p.tpr * ((nbd + 16 / p.cw - 1) / (16 / p.cw)));
  }
  p.ct = tc_chunk_tiles(p.tpi);
  p.cpi = (p.tpi + p.ct - 1) / p.ct;
  p.n_chunks = g.n_images * (int64_t)p.cpi;
  p.ok = (g.row_stride % 16) == 0 && (g.n_images <= 1 || (g.image_stride % 16) == 0) &&
         g.image_stride < ((int64_t)1 << 40) && 8 * g.row_stride < ((int64_t)1 << 40) &&
         p.n_chunks < ((int64_t)1 << 31);
  return p;
}

// The tensor-core streaming path for (u8 source, integer matrix, no clip, one r); false when
// the geometry or r is not covered (the caller then uses the SIMT streaming kernel).
// split > 0: the images are two planes of one geometry stacked in memory (see fused_u8_tc_planes);
// images [0, split) finalize into sse/psnr, the rest into sse2/psnr2
bool fused_u8_tc(const adct_matrix* m, const uint8_t* src, const adct_geom& g, int32_t r, double* sse, double* psnr,
                 double* partial, cudaStream_t st, adct_status* status, int64_t split, double* sse2, double* psnr2,
                 int clip) {
  const TcPlan p = tc_plan(g);
  if (!p.ok || g.n_images == 0 || !aligned(src, 16) || !m->is_int) return false;
  CUtensorMap map, map_d;
  if (p.cw == 15) {
    if (!make_tc_tmap(&map, src, g, 1, 15) || !make_tc_tmap(&map_d, src, g, 1, 1)) return false;
  } else {
    if (!make_tc_tmap(&map, src, g, 16 / p.cw, p.cw)) return false;
    map_d = map;
  }
  TcArgs a;
  a.tpr = p.tpr;
  a.tpi = p.tpi;
  a.cpi = p.cpi;
  a.ct = p.ct;
  a.n_chunks = (uint32_t)p.n_chunks;
  a.dcpi = make_fastdiv((uint32_t)p.cpi);
  a.dtpr = make_fastdiv((uint32_t)p.tpr);
  a.dmain = p.dmain;
  a.dlast = p.dlast;
  a.dc0 = p.dc0;
  const bool ok = m->specialized ? launch_tc<T1Mat>(r, p.cw, map, map_d, a, m->dev, partial, st, clip)
                                 : launch_tc<RtMat>(r, p.cw, map, map_d, a, m->dev, partial, st, clip);
  if (!ok) return false;
  count_launch();
  if ((*status = launch_status()) != ADCT_OK) return true;
  SlotMap sm{};
  sm.s[0] = 0;
  const int32_t ppi = p.cpi * kTcPartials;  // partials per image
  if (split > 0) {
    launch_finalize(partial, ppi, split, 1, sm, 1, (double)g.height * g.width, 255.0, sse, psnr, st);
    launch_finalize(partial + split * ppi, ppi, g.n_images - split, 1, sm, 1, (double)g.height * g.width, 255.0,
                    sse2, psnr2, st);
  } else {
    launch_finalize(partial, ppi, g.n_images, 1, sm, 1, (double)g.height * g.width, 255.0, sse, psnr, st);
  }
  *status = launch_status();
  return true;
}

// Several planes (the Y, U, V planes of config 4) on the tensor-core path: all of them or none
// (false, nothing launched), one launch per plane on the stream -- except that two consecutive
// planes of the same geometry that lie back to back in memory (plane i + 1 starts where plane i's
// last image ends, as the U and V stacks of bench.py do) run as ONE launch over both image ranges:
// one ramp and one tail instead of two, per-image sums bit-identical (chunks follow the geometry).  A single launch over the
// concatenated chunk lists of the planes (runtime tile shape, plane table) was built and measured:
// it removed two ramps and tails but its epilogue compiled to a different schedule that ran the
// luma plane 3-10 % slower and under the power cap (1.49-1.50 ms vs 1.46 ms per C4 step, same box;
// DESIGN.md §5.2), so the planes run one after the other.
bool fused_u8_tc_planes(const adct_matrix* m, int n, const uint8_t* const* src, const adct_geom* g, int32_t r,
                        double* const* sse, double* const* psnr, double* const* partial, cudaStream_t st,
                        adct_status* status) {
  if (n < 1 || n > kTcMaxPlanes || !m->is_int) return false;
  const bool r_ok = m->specialized ? tc_r_compiled(r) : r == 10;
  if (!r_ok) return false;
  for (int i = 0; i < n; ++i) {
    const TcPlan p = tc_plan(g[i]);
    if (!p.ok || g[i].n_images == 0 || !aligned(src[i], 16)) return false;
  }
  static const bool no_merge = std::getenv("ADCT_TC_NOMERGE") != nullptr;  // A/B hook
  for (int i = 0; i < n; ++i) {
    const int64_t is0 = g[i].n_images > 1 ? g[i].image_stride : (int64_t)g[i].height * g[i].row_stride;
    bool merge = !no_merge && i + 1 < n;
    if (merge) {
      const adct_geom& h = g[i + 1];
      const int64_t is1 = h.n_images > 1 ? h.image_stride : (int64_t)h.height * h.row_stride;
      adct_geom gm = g[i];
      gm.n_images = g[i].n_images + h.n_images;
      gm.image_stride = is0;
      const TcPlan pm = tc_plan(gm);
      const int64_t need = g[i].n_images * (int64_t)pm.cpi * kTcPartials;  // plane i's partials, merged plan
      merge = h.width == g[i].width && h.height == g[i].height && h.row_stride == g[i].row_stride && is1 == is0 &&
              src[i + 1] == src[i] + g[i].n_images * is0 && pm.ok && partial[i + 1] >= partial[i] + need;
      if (merge) {
        if (!fused_u8_tc(m, src[i], gm, r, sse[i], psnr ? psnr[i] : nullptr, partial[i], st, status, g[i].n_images,
                         sse[i + 1], psnr ? psnr[i + 1] : nullptr)) {
          *status = ADCT_E_CUDA;
          return true;
        }
        if (*status != ADCT_OK) return true;
        ++i;
        continue;
      }
    }
    if (!fused_u8_tc(m, src[i], g[i], r, sse[i], psnr ? psnr[i] : nullptr, partial[i], st, status)) {
      *status = ADCT_E_CUDA;  // a plane that passed the checks failed to launch
      return true;
    }
    if (*status != ADCT_OK) return true;
  }
  return true;
}

// Tensor-core path of approx_dct8x8_fwd_quant (the paper's T1, u8 planes of whole 128-byte chunks,
// 16-byte aligned strides); false when it does not cover the call (the SIMT TMA kernel then runs).
bool fwd_quant_tc(const adct_matrix* m, const uint8_t* src, const adct_geom& g, int32_t step, int16_t* q,
                  cudaStream_t st, adct_status* status) {
  // Opt-in (ADCT_Q_TC=1): parity-green and 34 % fewer issued instructions than the SIMT TMA kernel
  // (549 M vs 837 M warp-instructions on config 3), but no faster -- 1.146 vs 1.116 ms: both run at
  // the same 5.7 TB/s of DRAM traffic, the ceiling of config 3's 1 : 2 read : write mix (read-only
  // streams at 7.29 TB/s, 1 : 1 copies at 6.2 TB/s), so the SIMT kernel stays the default
  static const bool off = [] {
    const char* e = std::getenv("ADCT_Q_TC");
    return !(e && std::atoi(e) == 1);
  }();
  if (off || !m->specialized || g.n_images <= 0 || (g.width % 128) != 0 || (g.height % 8) != 0) return false;
  if ((g.row_stride % 16) || (g.n_images > 1 && (g.image_stride % 16)) || !aligned(src, 16) || !aligned(q, 128))
    return false;
  if (step < 1 || step > 4096) return false;
  const int64_t nch = g.width / 128, nbd = g.height / 8;
  const int64_t istride = g.n_images > 1 ? g.image_stride : (int64_t)g.height * g.row_stride;
  TcArgs a{};
  a.tpr = (int32_t)nch;
  a.tpi = (int32_t)(nch * ((nbd + 15) / 16));
  a.ct = tc_chunk_tiles(a.tpi);
  a.cpi = (a.tpi + a.ct - 1) / a.ct;
  const int64_t n_chunks = g.n_images * (int64_t)a.cpi;
  if (n_chunks >= ((int64_t)1 << 31) || istride >= ((int64_t)1 << 40) || 8 * (int64_t)g.row_stride >= ((int64_t)1 << 40))
    return false;
  a.n_chunks = (uint32_t)n_chunks;
  a.dcpi = make_fastdiv((uint32_t)a.cpi);
  a.dtpr = make_fastdiv((uint32_t)a.tpr);
  CUtensorMap map, mout;
  if (!make_tc_tmap(&map, src, g, 16, 1, true)) return false;
  {
    auto enc = tmap_encoder();
    if (!enc) return false;
    const uint64_t bw = (uint64_t)g.width / 8;
    const cuuint64_t dims[5] = {64, 2, bw / 2, (cuuint64_t)nbd, (cuuint64_t)g.n_images};
    const cuuint64_t strides[4] = {128, 256, bw * 128, (cuuint64_t)nbd * bw * 128};
    const cuuint32_t box[5] = {64, 1, 8, 4, 1};
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    if (enc(&mout, CU_TENSOR_MAP_DATA_TYPE_UINT16, 5, q, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  QTab qt;
  q_fill(qt, step, m->n);
  static std::mutex mu;
  static int8_t state[kMaxDevices] = {};
  if (!once_per_device(mu, state, [] {
        return cudaFuncSetAttribute(fwd_quant_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)kTqSmem) == cudaSuccess;
      }))
    return false;
  const int64_t grid = n_chunks < sms_s() ? n_chunks : sms_s();
  fwd_quant_tc_kernel<<<(unsigned)grid, kTcThreads, kTqSmem, st>>>(map, mout, a, qt, (float)step, (int32_t)nbd);
  count_launch();
  *status = launch_status();
  return true;
}

}  // namespace adct
