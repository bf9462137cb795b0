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
#include <mutex>

#include "adct_host.h"
#include "tma.cuh"

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
    float x[8][8], y[8][8];
    const uint32_t ib = wbase + slot * 4096;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 v = lds128(ib + swz(lane, i));
      i16x2_to_f(v.x, x[i][0], x[i][1]);
      i16x2_to_f(v.y, x[i][2], x[i][3]);
      i16x2_to_f(v.z, x[i][4], x[i][5]);
      i16x2_to_f(v.w, x[i][6], x[i][7]);
    }
    __syncwarp();
    fence_proxy_async();
    if (pt < n_tiles) issue(slot);  // the slot's data is in registers: refill it now
    if (++slot == kBmInSlots) { slot = 0; phase ^= 1u; }
    fwd2d(m, x, y);
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int l = 0; l < 8; ++l) y[k][l] *= wk.w[k * 8 + l];
    inv2d<MP, ~0ull>(m, y, x);
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

int g_bm_sms = 0;
int bm_sms() {
  if (!g_bm_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_bm_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_bm_sms <= 0) g_bm_sms = 148;
  }
  return g_bm_sms;
}

template <class MP, bool F32OUT>
adct_status launch_rt_bm(const CUtensorMap& tin, const CUtensorMap& tout, const DevMat& dm, const Wk& wk,
                         uint32_t n_tiles, int clip, float lo, float hi, cudaStream_t st) {
  constexpr int kBmWarps = bm_warps<F32OUT>();
  constexpr size_t smem = (size_t)kBmWarps * (kBmInSlots * 4096 + (F32OUT ? 8192 : 4096)) + kBmWarps * kBmInSlots * 8 + 1024;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [&] {
    err = cudaFuncSetAttribute(roundtrip_bm_kernel<MP, F32OUT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (err != cudaSuccess) return ADCT_E_CUDA;
  const uint32_t need = (n_tiles + kBmWarps - 1) / kBmWarps;
  const unsigned grid = (unsigned)(need < (uint32_t)bm_sms() ? need : (uint32_t)bm_sms());
  roundtrip_bm_kernel<MP, F32OUT><<<grid, 32 * kBmWarps, smem, st>>>(tin, tout, dm, wk, n_tiles, clip, lo, hi);
  return ADCT_OK;
}

}  // namespace

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
