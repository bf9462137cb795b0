// jam.cu — next row f2: 16- and 32-point transforms of §6.2, the
// Jridi-Alfalou-Meher scaling of the paper's T1, through the round trip
// forward -> zonal retention (N x N zig-zag, reading A20) -> inverse -> reconstruction.
//
// The N-point network is the JAM recursion itself (reading A19): u_i = x_i + x_{N-1-i},
// v_i = x_i - x_{N-1-i}; rows 2k / 2k+1 of T(N) are row k of T(N/2) on u / v; the base is the
// compile-time T1 network (24 adds + 6 shifts).  Its transpose (the inverse) runs the halves
// first and the butterfly last.  All intermediates are integers < 2^24 for |x| <= 7281, so the
// forward is exact in fp32 there; beyond (int16 sources) it rounds (tested over the whole int16
// range: 1e-5 per block, int16 round trip at r = N^2 still the identity).
//
// One CTA of 256 threads owns 256/N blocks per iteration.  Pass 1: thread (block b, row i) loads row i,
// applies T(N) (row transform) and stores it to shared memory.  Pass 2: thread (b, column k)
// applies T(N) down the column, the weights W_kl = keep_kl / (d_k d_l), d = diag(T T^T)
// (P:L2742-2770), and T(N)^T back up the column.  Pass 3: thread (b, i) applies T(N)^T to its row
// and writes the reconstruction.  A row pitch of an odd number of 16-byte units (N + 4) keeps
// the 128-bit row passes and the scalar column pass conflict-free.
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "adct_host.h"
#include "packed.cuh"

// ADCT_JAM_PACKED: the N-point networks on consecutive element pairs with packed fp32 (FFMA2 /
// FADD2; packed.cuh), coefficients in the permuted "slot" order the packed recursion produces
// (the weight table is permuted to match on the host); 0 = the scalar networks (A/B)
#ifndef ADCT_JAM_PACKED
#define ADCT_JAM_PACKED 0  // packed: parity-green but no faster (4.56 vs 4.52 ms T(16)): the kernel is not FP-issue-bound
#endif

namespace adct {
namespace {

constexpr int kJamNT = 256;
// Resident CTAs per SM the register budget is cut for (B200 sweep, int16 r = N^2: T(16) 5 -> 48
// registers, T(32) 3 -> 80, both spill-free; tighter budgets spill and run up to 1.6x slower)
#ifndef ADCT_JAM_MINB16
#define ADCT_JAM_MINB16 5
#endif
#ifndef ADCT_JAM_MINB32
#define ADCT_JAM_MINB32 3
#endif

// y = T(N) x
template <int N>
struct Jam {
  __device__ __forceinline__ static void fwd(const float* x, float* y) {
    float u[N / 2], v[N / 2], yu[N / 2], yv[N / 2];
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      u[i] = x[i] + x[N - 1 - i];
      v[i] = x[i] - x[N - 1 - i];
    }
    Jam<N / 2>::fwd(u, yu);
    Jam<N / 2>::fwd(v, yv);
#pragma unroll
    for (int k = 0; k < N / 2; ++k) {
      y[2 * k] = yu[k];
      y[2 * k + 1] = yv[k];
    }
  }
  // x = T(N)^T y
  __device__ __forceinline__ static void inv(const float* y, float* x) {
    float ye[N / 2], yo[N / 2], a[N / 2], b[N / 2];
#pragma unroll
    for (int k = 0; k < N / 2; ++k) {
      ye[k] = y[2 * k];
      yo[k] = y[2 * k + 1];
    }
    Jam<N / 2>::inv(ye, a);
    Jam<N / 2>::inv(yo, b);
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      x[i] = a[i] + b[i];
      x[N - 1 - i] = a[i] - b[i];
    }
  }
};

__device__ DevMat g_jam_unused;  // T1Mat ignores its DevMat: the network is compile-time

template <>
struct Jam<8> {
  __device__ __forceinline__ static void fwd(const float* x, float* y) { fwd8(T1Mat(g_jam_unused), x, y); }
  __device__ __forceinline__ static void inv(const float* y, float* x) {
    inv8<T1Mat, 0xffu>(T1Mat(g_jam_unused), y, x);
  }
};

// Packed JAM recursion.  In: N/2 consecutive pairs (x0,x1), (x2,x3), ...  Out: N/2 pairs in the
// slot layout L_N -- L_8 is packed.cuh's yq layout (y0,y4), (y2,y6), (y1,y3), (y5,y7); L_N puts
// the even outputs (T(N/2) of u, in L_(N/2)) in the first N/4 pairs and the odd ones (T(N/2) of
// v) in the rest.  The inverse reads L_N and writes consecutive pairs.  The butterflies pair
// element i with N-1-i, i.e. pair c with the swapped pair N/2-1-c.
template <int N>
struct JamP {
  __device__ __forceinline__ static void fwd(const float2* x, float2* y) {
    float2 u[N / 4], v[N / 4];
#pragma unroll
    for (int c = 0; c < N / 4; ++c) {
      u[c] = padd(x[c], pswap(x[N / 2 - 1 - c]));
      v[c] = psub(x[c], pswap(x[N / 2 - 1 - c]));
    }
    JamP<N / 2>::fwd(u, y);
    JamP<N / 2>::fwd(v, y + N / 4);
  }
  __device__ __forceinline__ static void inv(const float2* y, float2* x) {
    float2 a[N / 4], b[N / 4];
    JamP<N / 2>::inv(y, a);
    JamP<N / 2>::inv(y + N / 4, b);
#pragma unroll
    for (int c = 0; c < N / 4; ++c) {
      x[c] = padd(a[c], b[c]);
      x[N / 2 - 1 - c] = pswap(psub(a[c], b[c]));
    }
  }
};
template <>
struct JamP<8> {
  __device__ __forceinline__ static void fwd(const float2* x, float2* y) { fwd8_row(T1Mat(g_jam_unused), x, y); }
  __device__ __forceinline__ static void inv(const float2* y, float2* x) { inv8_row(T1Mat(g_jam_unused), y, x); }
};
// scalar interface: x natural order -> y in slot order (float 2c + h of pair c), and back
template <int N>
struct JamPk {
  __device__ __forceinline__ static void fwd(const float* x, float* y) {
    float2 x2[N / 2], y2[N / 2];
#pragma unroll
    for (int c = 0; c < N / 2; ++c) x2[c] = pk(x[2 * c], x[2 * c + 1]);
    JamP<N>::fwd(x2, y2);
#pragma unroll
    for (int c = 0; c < N / 2; ++c) {
      y[2 * c] = y2[c].x;
      y[2 * c + 1] = y2[c].y;
    }
  }
  __device__ __forceinline__ static void inv(const float* y, float* x) {
    float2 y2[N / 2], x2[N / 2];
#pragma unroll
    for (int c = 0; c < N / 2; ++c) y2[c] = pk(y[2 * c], y[2 * c + 1]);
    JamP<N>::inv(y2, x2);
#pragma unroll
    for (int c = 0; c < N / 2; ++c) {
      x[2 * c] = x2[c].x;
      x[2 * c + 1] = x2[c].y;
    }
  }
};
#if ADCT_JAM_PACKED
template <int N>
using JamNet = JamPk<N>;
#else
template <int N>
using JamNet = Jam<N>;
#endif
// host: slot of output frequency k in L_N (inverse of the layout above)
inline int jam_slot(int n, int k) {
  if (n == 8) {
    constexpr int s8[8] = {0, 4, 2, 5, 1, 6, 3, 7};  // y0->0, y4->1, y2->2, y6->3, y1->4, y3->5, y5->6, y7->7
    return s8[k];
  }
  return (k % 2 == 0) ? jam_slot(n / 2, k / 2) : n / 2 + jam_slot(n / 2, k / 2);
}

template <int N>
struct JamW {
  float w[N * N];  // keep_kl / (d_k d_l)
};

// One row of N samples, raw (16-byte vector loads; rows are 16-byte aligned), then as fp32.
// Conversions avoid the quarter-rate XU pipe (I2F/F2I): a u8 sample is placed in the mantissa of
// 2^23 by one PRMT and the 2^23 removed by an FADD; an int16 sample is sign-extended (PRMT / SHF)
// and converted by I2FP on the ALU pipe; results are rounded with the 1.5*2^23 trick.
template <int N, typename SrcT>
struct RawRow {
  static constexpr int NV = N * (int)sizeof(SrcT) / 16;
  uint4 v[NV];
  __device__ __forceinline__ void load(const SrcT* p) {
#pragma unroll
    for (int c = 0; c < NV; ++c) v[c] = __ldg(reinterpret_cast<const uint4*>(p) + c);
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int c = 0; c < NV; ++c) v[c] = make_uint4(0u, 0u, 0u, 0u);
  }
};
template <int N>
__device__ __forceinline__ void to_float(const RawRow<N, uint8_t>& r, float* x) {
#pragma unroll
  for (int c = 0; c < N / 16; ++c) {
    const uint32_t w[4] = {r.v[c].x, r.v[c].y, r.v[c].z, r.v[c].w};
#pragma unroll
    for (int q = 0; q < 16; ++q)
      x[c * 16 + q] = __uint_as_float(__byte_perm(w[q >> 2], 0x4B000000u, 0x7440u | (uint32_t)(q & 3))) - 8388608.0f;
  }
}
template <int N>
__device__ __forceinline__ void to_float(const RawRow<N, int16_t>& r, float* x) {
#pragma unroll
  for (int c = 0; c < N / 8; ++c) {
    const uint32_t w[4] = {r.v[c].x, r.v[c].y, r.v[c].z, r.v[c].w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      // low half sign-extended by PRMT's sign-replicate mode (selector nibble bit 3).  Written in
      // PTX: __byte_perm uses only the low 3 bits of each nibble (it would COPY byte 1, which
      // equals its sign fill only for |x| <= 255 -- found by the full int16-range test)
      uint32_t lo;
      asm("prmt.b32 %0, %1, 0, 0x9910;" : "=r"(lo) : "r"(w[q]));
      x[c * 8 + 2 * q] = (float)(int32_t)lo;
      x[c * 8 + 2 * q + 1] = (float)((int32_t)w[q] >> 16);
    }
  }
}

// low 16 (or 8) bits of 1.5*2^23 + v: v rounded half to even, two's complement
__device__ __forceinline__ uint32_t rbits(float v) { return __float_as_uint(v + 12582912.0f); }

// v rounded half to even as an int32 (|v| < 2^22: the reconstruction is an orthogonal projection
// of the block, so |v| <= ||x||_2 <= 32768 * N)
__device__ __forceinline__ int32_t rint_s32(float v) { return (int32_t)(rbits(v) - 0x4B400000u); }
// (sat_s16(hi) << 16) | sat_s16(lo): one I2IP for two samples
__device__ __forceinline__ uint32_t pack_sat_s16(int32_t hi, int32_t lo) {
  uint32_t d;
  asm("cvt.pack.sat.s16.s32 %0, %1, %2;" : "=r"(d) : "r"(hi), "r"(lo));
  return d;
}

// SAT16: x is unclipped and the int16 range is the clip range (int16 source)
template <int N, bool SAT16>
__device__ __forceinline__ void store_row_any(void* recon, int64_t off, int out_t, const float* x) {
  if (out_t == ADCT_F32) {
    float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(recon) + off);
#pragma unroll
    for (int c = 0; c < N / 4; ++c) o[c] = make_float4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
  } else if (out_t == ADCT_I16 && SAT16) {  // rounded here, saturated by the pack (CLIP_ROUND)
    uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<int16_t*>(recon) + off);
#pragma unroll
    for (int c = 0; c < N / 8; ++c) {
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = pack_sat_s16(rint_s32(x[8 * c + 2 * q + 1]), rint_s32(x[8 * c + 2 * q]));
      o[c] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  } else if (out_t == ADCT_I16) {  // x already rounded and saturated (CLIP_ROUND)
    uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<int16_t*>(recon) + off);
#pragma unroll
    for (int c = 0; c < N / 8; ++c) {
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = __byte_perm(rbits(x[8 * c + 2 * q]), rbits(x[8 * c + 2 * q + 1]), 0x5410u);
      o[c] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  } else {
    uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(recon) + off);
#pragma unroll
    for (int c = 0; c < N / 16; ++c) {
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t lo = __byte_perm(rbits(x[16 * c + 4 * q]), rbits(x[16 * c + 4 * q + 1]), 0x0040u);
        const uint32_t hi = __byte_perm(rbits(x[16 * c + 4 * q + 2]), rbits(x[16 * c + 4 * q + 3]), 0x0040u);
        w[q] = __byte_perm(lo, hi, 0x5410u);
      }
      o[c] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

template <int N>
__device__ __forceinline__ int64_t jam_row_offset(uint32_t b, int i, const KGeom& g, FastDiv dnbi, FastDiv dbw) {
  const uint32_t img = fdiv(b, dnbi);
  const uint32_t q = b - img * g.nbi;
  const uint32_t by = fdiv(q, dbw);
  const uint32_t bx = q - by * g.bw;
  return (int64_t)img * g.image_stride + ((int64_t)by * N + i) * g.row_stride + (int64_t)bx * N;
}

// Persistent (grid = SMs x resident CTAs).  The next iteration's row is loaded into registers
// right after pass 1 consumes the current one, so its HBM latency overlaps passes 2-3.  A warp
// owns whole blocks (N = 32: one, N = 16: two), so every shared-memory exchange stays inside the
// warp: two __syncwarp per iteration, no CTA barrier (pass 3 and the next pass 1 touch only the
// thread's own row).
template <int N, typename SrcT>
__global__ void __launch_bounds__(kJamNT, N == 16 ? ADCT_JAM_MINB16 : ADCT_JAM_MINB32) jam_roundtrip_kernel(const SrcT* __restrict__ src, KGeom g, JamW<N> wt,
                                                               uint32_t nblocks, FastDiv dnbi, FastDiv dbw,
                                                               int out_t, int clip, float lo, float hi,
                                                               void* __restrict__ recon) {
  constexpr int BPC = kJamNT / N;  // blocks per CTA
  constexpr bool kSat16 = sizeof(SrcT) == 2;
  static_assert(32 % N == 0 || N % 32 == 0, "a warp must own whole blocks");
  static_assert(N <= 32, "one block per warp at most");
  // row pitch N + 4 floats = an odd number of 16-byte units: 128-bit row accesses (8 lanes per
  // phase, rows i..i+7) and scalar column accesses (consecutive columns) are both conflict-free
  constexpr int P = N + 4;
  __shared__ __align__(16) float sm[BPC * N * P];
  __shared__ __align__(16) float sw[N * P];  // weights transposed, sw[l][k]: column l reads its k's as float4
  for (int t = threadIdx.x; t < N * N; t += kJamNT) sw[(t % N) * P + t / N] = wt.w[t];
  const int bl = threadIdx.x / N, i = threadIdx.x % N;  // thread = (block, row i) = (block, column i)
  const uint32_t stride = gridDim.x * BPC;
  float* row = sm + (bl * N + i) * P;
  uint32_t b = blockIdx.x * BPC + bl;
  bool valid = b < nblocks;
  int64_t off = valid ? jam_row_offset<N>(b, i, g, dnbi, dbw) : 0;
  RawRow<N, SrcT> raw;
  if (valid) raw.load(src + off);
  else raw.zero();
  __syncthreads();
  for (uint32_t b0 = blockIdx.x * BPC; b0 < nblocks; b0 += stride) {
    {  // pass 1: row i of block bl, forward
      float x[N], y[N];
      to_float<N>(raw, x);
      JamNet<N>::fwd(x, y);
#pragma unroll
      for (int j = 0; j < N; j += 4) *reinterpret_cast<float4*>(row + j) = make_float4(y[j], y[j + 1], y[j + 2], y[j + 3]);
    }
    const uint32_t bn = b + stride;  // prefetch the next iteration's row
    const bool vn = bn < nblocks;
    const int64_t offn = vn ? jam_row_offset<N>(bn, i, g, dnbi, dbw) : 0;
    if (vn) raw.load(src + offn);
    else raw.zero();
    __syncwarp();
    {  // pass 2: column i (frequency l = i) of block bl: forward, weights, inverse
      float c[N], y[N];
#pragma unroll
      for (int k = 0; k < N; ++k) c[k] = sm[(bl * N + k) * P + i];
      JamNet<N>::fwd(c, y);
#pragma unroll
      for (int k = 0; k < N; k += 4) {
        const float4 w4 = *reinterpret_cast<const float4*>(sw + i * P + k);
        y[k] *= w4.x;
        y[k + 1] *= w4.y;
        y[k + 2] *= w4.z;
        y[k + 3] *= w4.w;
      }
      JamNet<N>::inv(y, c);
#pragma unroll
      for (int k = 0; k < N; ++k) sm[(bl * N + k) * P + i] = c[k];
    }
    __syncwarp();
    {  // pass 3: row i, inverse, store
      float z[N], x[N];
#pragma unroll
      for (int j = 0; j < N; j += 4) {
        const float4 r4 = *reinterpret_cast<const float4*>(row + j);
        z[j] = r4.x;
        z[j + 1] = r4.y;
        z[j + 2] = r4.z;
        z[j + 3] = r4.w;
      }
      JamNet<N>::inv(z, x);
      if (valid && kSat16 && out_t == ADCT_I16) {  // int16 -> int16: the saturating pack is the clip
        store_row_any<N, true>(recon, off, out_t, x);
      } else if (valid) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
          float v = x[j];
          if (clip != ADCT_CLIP_NONE) v = fminf(fmaxf(v, lo), hi);
          if (clip == ADCT_CLIP_ROUND && out_t == ADCT_F32) v = rintf(v);  // integer stores round themselves
          x[j] = v;
        }
        store_row_any<N, false>(recon, off, out_t, x);
      }
    }
    b = bn;
    valid = vn;
    off = offn;
  }
}


// ---- version 2: two rows / two columns per thread on packed fp32 ------------------------------
// The networks run on float2 values whose halves are two INDEPENDENT vectors (two rows of a block
// in passes 1 and 3, two adjacent columns in pass 2), so the recursion is the scalar one with
// FADD2 / FFMA2 -- no lane swaps -- and every exchange through shared memory is a 128-bit access:
// half the issued FP32 instructions and a third of the shared-memory instructions per sample of
// the one-row-per-thread kernel above (which was bound by issue slots and the MIO queue).
template <int N>
struct Jam2 {
  __device__ __forceinline__ static void fwd(const float2* x, float2* y) {
    float2 u[N / 2], v[N / 2], yu[N / 2], yv[N / 2];
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      u[i] = padd(x[i], x[N - 1 - i]);
      v[i] = psub(x[i], x[N - 1 - i]);
    }
    Jam2<N / 2>::fwd(u, yu);
    Jam2<N / 2>::fwd(v, yv);
#pragma unroll
    for (int k = 0; k < N / 2; ++k) {
      y[2 * k] = yu[k];
      y[2 * k + 1] = yv[k];
    }
  }
  __device__ __forceinline__ static void inv(const float2* y, float2* x) {
    float2 ye[N / 2], yo[N / 2], a[N / 2], b[N / 2];
#pragma unroll
    for (int k = 0; k < N / 2; ++k) {
      ye[k] = y[2 * k];
      yo[k] = y[2 * k + 1];
    }
    Jam2<N / 2>::inv(ye, a);
    Jam2<N / 2>::inv(yo, b);
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      x[i] = padd(a[i], b[i]);
      x[N - 1 - i] = psub(a[i], b[i]);
    }
  }
};
template <>
struct Jam2<8> {
  __device__ __forceinline__ static void fwd(const float2* x, float2* y) { fwd8p(T1Mat(g_jam_unused), x, y); }
  __device__ __forceinline__ static void inv(const float2* y, float2* x) { inv8p(T1Mat(g_jam_unused), y, x); }
};

constexpr int kJam2NT = 128;  // threads per CTA: 256 rows = 256 / N blocks per iteration
#ifndef ADCT_JAM2_MINB16
#define ADCT_JAM2_MINB16 5
#endif
#ifndef ADCT_JAM2_MINB32
#define ADCT_JAM2_MINB32 4
#endif
#ifndef ADCT_JAM2_PF
#define ADCT_JAM2_PF 1  // L2 prefetch of the next iteration's rows
#endif
template <int N>
constexpr size_t jam2_smem() {  // row-pair tile + weights
  return (size_t)(kJam2NT * (2 * N + 4) + (N / 2) * (2 * N + 4)) * sizeof(float);
}

// two horizontally adjacent samples (columns 2cp, 2cp + 1 of one row) as one load
template <typename SrcT>
__device__ __forceinline__ float2 ld_pair(const SrcT* p);
template <>
__device__ __forceinline__ float2 ld_pair<int16_t>(const int16_t* p) {
  const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(p));
  uint32_t lo;
  asm("prmt.b32 %0, %1, 0, 0x9910;" : "=r"(lo) : "r"(w));  // sign-extended low half
  return pk((float)(int32_t)lo, (float)((int32_t)w >> 16));
}
template <>
__device__ __forceinline__ float2 ld_pair<uint8_t>(const uint8_t* p) {
  const uint32_t w = __ldg(reinterpret_cast<const uint16_t*>(p));
  return psub(pk(__uint_as_float(__byte_perm(w, 0x4B000000u, 0x7440u)),
                 __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7441u))),
              pk(8388608.0f, 8388608.0f));
}

// Thread t of a CTA has two roles over the CTA's 256-row group (256 / N blocks).  COLUMN role
// (passes 1 and 3): columns 2cp, 2cp + 1 of block t / (N/2) -- one 32-bit (int16) or 16-bit (u8)
// global access per row holds exactly the pair a packed instruction works on, and the lanes of a
// warp instruction cover whole 64-byte row segments (two 128-byte wavefronts per 32-point row
// where the row-per-thread kernel needs sixteen: its LSU data stage, not issue or HBM, was the
// limiter -- ncu l1tex__data_pipe_lsu_wavefronts 97 %).  ROW role (pass 2): rows 2t, 2t + 1 of the
// group.  A warp's 32 column pairs and its 64 rows are the same 64 / N blocks, so only __syncwarp
// separates the passes.  Shared memory holds the group as [row pair][column][2] (pitch 2N + 4
// floats = an odd number of 16-byte units): every exchange is a conflict-free 128-bit access.
// The 2-D transform is separable, so columns-then-rows gives the same T X T^T (exact integers
// forward) and the inverse runs rows-then-columns.
template <int N, typename SrcT>
__global__ void __launch_bounds__(kJam2NT, N == 16 ? ADCT_JAM2_MINB16 : ADCT_JAM2_MINB32)
    jam2_roundtrip_kernel(const SrcT* __restrict__ src, KGeom g, JamW<N> wt, uint32_t nblocks, FastDiv dnbi,
                          FastDiv dbw, int out_t, int clip, float lo, float hi, void* __restrict__ recon) {
  constexpr int BPC = 2 * kJam2NT / N;  // blocks per CTA iteration
  constexpr bool kSat16 = sizeof(SrcT) == 2;
  constexpr int PP = 2 * N + 4;
  extern __shared__ __align__(16) float jsm[];
  float* sm = jsm;
  float* sw = jsm + kJam2NT * PP;  // sw[rp][l][h] = w[2rp + h][l]
  for (int t = threadIdx.x; t < N * N; t += kJam2NT) {
    const int k = t / N, l = t % N;
    sw[(k >> 1) * PP + 2 * l + (k & 1)] = wt.w[t];
  }
  const int t = threadIdx.x;
  const int bl = t / (N / 2), cp = t % (N / 2);  // column role
  const uint32_t stride = gridDim.x * BPC;
  float* rowp = sm + t * PP;                            // row role: rows 2t, 2t + 1 of the group
  float* colp = sm + (bl * (N / 2)) * PP + 4 * cp;      // column role: + rp * PP
  const float* wp = sw + (t % (N / 2)) * PP;            // row role: weights of rows 2t % N, + 1
  uint32_t b = blockIdx.x * BPC + bl;
  bool valid = b < nblocks;
  int64_t off = valid ? jam_row_offset<N>(b, 0, g, dnbi, dbw) + 2 * cp : 0;
  __syncthreads();
  for (uint32_t b0 = blockIdx.x * BPC; b0 < nblocks; b0 += stride) {
    {  // pass 1: columns 2cp, 2cp + 1 forward
      float2 x2[N], y2[N];
      if (valid) {
#pragma unroll
        for (int i = 0; i < N; ++i) x2[i] = ld_pair<SrcT>(src + off + (int64_t)i * g.row_stride);
      } else {
#pragma unroll
        for (int i = 0; i < N; ++i) x2[i] = pk(0.0f, 0.0f);
      }
      Jam2<N>::fwd(x2, y2);
#pragma unroll
      for (int rp = 0; rp < N / 2; ++rp)
        *reinterpret_cast<float4*>(colp + rp * PP) =
            make_float4(y2[2 * rp].x, y2[2 * rp + 1].x, y2[2 * rp].y, y2[2 * rp + 1].y);
    }
    const uint32_t bn = b + stride;  // the next iteration's block: rows 2cp, 2cp + 1 into L2
    const bool vn = bn < nblocks;
    const int64_t offn = vn ? jam_row_offset<N>(bn, 0, g, dnbi, dbw) + 2 * cp : 0;
#if ADCT_JAM2_PF
    if (vn) {
      const SrcT* pn = src + offn - 2 * cp + (int64_t)(2 * cp) * g.row_stride;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pn));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pn + g.row_stride));
    }
#endif
    __syncwarp();
    {  // pass 2: rows 2t, 2t + 1: forward, weights, inverse
      float2 z2[N], y2[N];
#pragma unroll
      for (int j = 0; j < N; j += 2) {
        const float4 r4 = *reinterpret_cast<const float4*>(rowp + 2 * j);
        z2[j] = pk(r4.x, r4.y);
        z2[j + 1] = pk(r4.z, r4.w);
      }
      Jam2<N>::fwd(z2, y2);
#pragma unroll
      for (int l = 0; l < N; l += 2) {
        const float4 w4 = *reinterpret_cast<const float4*>(wp + 2 * l);
        y2[l] = __fmul2_rn(y2[l], pk(w4.x, w4.y));
        y2[l + 1] = __fmul2_rn(y2[l + 1], pk(w4.z, w4.w));
      }
      Jam2<N>::inv(y2, z2);
#pragma unroll
      for (int j = 0; j < N; j += 2)
        *reinterpret_cast<float4*>(rowp + 2 * j) = make_float4(z2[j].x, z2[j].y, z2[j + 1].x, z2[j + 1].y);
    }
    __syncwarp();
    {  // pass 3: columns 2cp, 2cp + 1 inverse, store
      float2 c2[N], x2[N];
#pragma unroll
      for (int rp = 0; rp < N / 2; ++rp) {
        const float4 v = *reinterpret_cast<const float4*>(colp + rp * PP);
        c2[2 * rp] = pk(v.x, v.z);
        c2[2 * rp + 1] = pk(v.y, v.w);
      }
      Jam2<N>::inv(c2, x2);
      if (valid && kSat16 && out_t == ADCT_I16) {  // int16 -> int16: the saturating pack is the clip
        uint32_t* o = reinterpret_cast<uint32_t*>(reinterpret_cast<int16_t*>(recon) + off);
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const float2 r = padd(x2[i], pk(12582912.0f, 12582912.0f));  // half to even (rint_s32)
          o[(int64_t)i * (g.row_stride / 2)] = pack_sat_s16((int32_t)(__float_as_uint(r.y) - 0x4B400000u),
                                                            (int32_t)(__float_as_uint(r.x) - 0x4B400000u));
        }
      } else if (valid) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
          float va = x2[i].x, vb = x2[i].y;
          if (clip != ADCT_CLIP_NONE) {
            va = fminf(fmaxf(va, lo), hi);
            vb = fminf(fmaxf(vb, lo), hi);
          }
          const int64_t o = off + (int64_t)i * g.row_stride;
          if (out_t == ADCT_F32) {
            if (clip == ADCT_CLIP_ROUND) {
              va = rintf(va);
              vb = rintf(vb);
            }
            *reinterpret_cast<float2*>(reinterpret_cast<float*>(recon) + o) = make_float2(va, vb);
          } else if (out_t == ADCT_I16) {  // already clipped to the source's range (CLIP_ROUND)
            *reinterpret_cast<uint32_t*>(reinterpret_cast<int16_t*>(recon) + o) =
                __byte_perm(rbits(va), rbits(vb), 0x5410u);
          } else {
            *reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(recon) + o) =
                (uint16_t)__byte_perm(rbits(va), rbits(vb), 0x0040u);
          }
        }
      }
    }
    b = bn;
    valid = vn;
    off = offn;
  }
}

// n x n zig-zag walk (reading A20): anti-diagonals d = k + l in order, even ones bottom-left
// to top-right
template <int N>
void zigzag_keep(int r, bool* keep) {
  int z = 0;
  for (int d = 0; d < 2 * N - 1; ++d) {
    int ks[2 * N];
    int c = 0;
    for (int k = 0; k < N; ++k)
      if (d - k >= 0 && d - k < N) ks[c++] = k;
    for (int t = 0; t < c; ++t) {
      const int k = (d % 2 == 0) ? ks[c - 1 - t] : ks[t];
      keep[k * N + (d - k)] = z < r;
      ++z;
    }
  }
}

template <int N, typename SrcT>
adct_status launch_jam(const void* src, const adct_geom& g, int32_t r, void* recon, adct_dtype recon_t,
                       adct_clip clip, float lo, float hi, cudaStream_t st) {
  // d = diag(T(N) T(N)^T): D(16) = 4 (I2 x diag(4,9,10,9) x I2), D(32) = 2 D(16) x I2
  double d8[8] = {8, 18, 20, 18, 8, 18, 20, 18};
  double d[N];
  for (int k = 0; k < N; ++k) d[k] = d8[k / (N / 8)] * (double)(N / 8);
  bool keep[N * N];
  zigzag_keep<N>(r, keep);
  JamW<N> wt;
  for (int k = 0; k < N; ++k)
    for (int l = 0; l < N; ++l) {
      // the kernel sees coefficient (k, l) at (slot(k), slot(l)) when the networks are packed
      const int sk = ADCT_JAM_PACKED ? jam_slot(N, k) : k, sl = ADCT_JAM_PACKED ? jam_slot(N, l) : l;
      wt.w[sk * N + sl] = keep[k * N + l] ? (float)(1.0 / (d[k] * d[l])) : 0.0f;
    }
  KGeom kg;
  kg.image_stride = g.image_stride;
  kg.row_stride = g.row_stride;
  kg.bw = (uint32_t)(g.width / N);
  kg.bh = (uint32_t)(g.height / N);
  kg.nbi = kg.bw * kg.bh;
  kg.n_images = (uint32_t)g.n_images;
  const uint32_t nb = (uint32_t)(g.n_images * kg.nbi);
  if (nb == 0) return ADCT_OK;
  int dev = 0, sms = 148, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // the column-pair / row-pair packed kernel (jam2_roundtrip_kernel) is parity-green and issues 39 %
  // fewer instructions, but runs level with the one-row-per-thread kernel at N = 32 (5.01 vs 4.95 ms)
  // and slower at N = 16 (4.77 vs 4.52 ms): both sit on the FP32 datapath (23 adds per sample =
  // 98 % of the HBM time at full FMA-pipe rate) with too few warps to fill it (f2).
  // ADCT_JAM_V2=1 selects it (tests/test_gpu_parity.py runs the JAM parity suite on it)
  static const bool v1 = std::getenv("ADCT_JAM_V2") == nullptr || ADCT_JAM_PACKED;
  if (!v1 && dev >= 0 && dev < kMaxDevices) {
    constexpr int BPC2 = 2 * kJam2NT / N;
    constexpr size_t smem = jam2_smem<N>();
    static std::mutex mu;
    static int8_t state[kMaxDevices] = {};
    static int occ2[kMaxDevices] = {};
    if (!once_per_device(mu, state, [&] {
          if (cudaFuncSetAttribute(jam2_roundtrip_kernel<N, SrcT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem) != cudaSuccess)
            return false;
          int o = 0;
          if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, jam2_roundtrip_kernel<N, SrcT>, kJam2NT, smem) !=
                  cudaSuccess || o < 1)
            o = 1;
          occ2[dev] = o;
          return true;
        }))
      return ADCT_E_CUDA;
    const int64_t need2 = ((int64_t)nb + BPC2 - 1) / BPC2, cap2 = (int64_t)sms * occ2[dev];
    const unsigned grid2 = (unsigned)(need2 < cap2 ? need2 : cap2);
    jam2_roundtrip_kernel<N, SrcT><<<grid2, kJam2NT, smem, st>>>((const SrcT*)src, kg, wt, nb, make_fastdiv(kg.nbi),
                                                                 make_fastdiv(kg.bw), (int)recon_t, (int)clip, lo, hi,
                                                                 recon);
    count_launch();
    return launch_status();
  }
  constexpr int BPC = kJamNT / N;
  // one wave of resident CTAs: a grid beyond it would leave a second, partly occupied wave
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, jam_roundtrip_kernel<N, SrcT>, kJamNT, 0) != cudaSuccess ||
      occ < 1)
    occ = 1;
  const int64_t need = ((int64_t)nb + BPC - 1) / BPC, cap = (int64_t)sms * occ;
  const unsigned grid = (unsigned)(need < cap ? need : cap);
  jam_roundtrip_kernel<N, SrcT><<<grid, kJamNT, 0, st>>>((const SrcT*)src, kg, wt, nb, make_fastdiv(kg.nbi),
                                                         make_fastdiv(kg.bw), (int)recon_t, (int)clip, lo, hi, recon);
  count_launch();
  return launch_status();
}

}  // namespace
}  // namespace adct

using namespace adct;

extern "C" adct_status approx_dct_jam_roundtrip(int32_t n, const void* src, adct_dtype src_t, adct_geom g, int32_t r,
                                               void* recon, adct_dtype recon_t, adct_clip clip, void* stream) {
  if (!src || !recon) return ADCT_E_INVALID_ARGUMENT;
  if (n != 16 && n != 32) return ADCT_E_INVALID_ARGUMENT;
  if (g.n_images < 0 || g.height <= 0 || g.width <= 0 || g.height % n || g.width % n) return ADCT_E_INVALID_ARGUMENT;
  if (g.row_stride < g.width || (g.n_images > 1 && g.image_stride < (int64_t)g.height * g.row_stride))
    return ADCT_E_INVALID_ARGUMENT;
  if (g.n_images * (int64_t)(g.height / n) * (g.width / n) >= ((int64_t)1 << 31)) return ADCT_E_INVALID_ARGUMENT;
  if (src_t != ADCT_U8 && src_t != ADCT_I16) return ADCT_E_INVALID_ARGUMENT;
  if (r < 1 || r > n * n) return ADCT_E_INVALID_ARGUMENT;
  if (clip != ADCT_CLIP_NONE && clip != ADCT_CLIP && clip != ADCT_CLIP_ROUND) return ADCT_E_INVALID_ARGUMENT;
  if (recon_t == ADCT_U8 || recon_t == ADCT_I16) {
    if (clip != ADCT_CLIP_ROUND) return ADCT_E_INVALID_ARGUMENT;
  } else if (recon_t != ADCT_F32) {
    return ADCT_E_INVALID_ARGUMENT;
  }
  const int esz = src_t == ADCT_U8 ? 1 : 2, osz = recon_t == ADCT_F32 ? 4 : (recon_t == ADCT_I16 ? 2 : 1);
  // 16-byte vector rows: aligned bases and strides (in both element sizes)
  if ((uintptr_t)src % 16 || (uintptr_t)recon % 16 || (g.row_stride * esz) % 16 || (g.row_stride * osz) % 16 ||
      (g.n_images > 1 && ((g.image_stride * esz) % 16 || (g.image_stride * osz) % 16)))
    return ADCT_E_ALIGNMENT;
  const float lo = src_t == ADCT_U8 ? 0.0f : -32768.0f, hi = src_t == ADCT_U8 ? 255.0f : 32767.0f;
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 16)
    return src_t == ADCT_U8 ? launch_jam<16, uint8_t>(src, g, r, recon, recon_t, clip, lo, hi, st)
                            : launch_jam<16, int16_t>(src, g, r, recon, recon_t, clip, lo, hi, st);
  return src_t == ADCT_U8 ? launch_jam<32, uint8_t>(src, g, r, recon, recon_t, clip, lo, hi, st)
                          : launch_jam<32, int16_t>(src, g, r, recon, recon_t, clip, lo, hi, st);
}
