// stream.cu — the hot kernel of BASELINE.json config 4: forward -> zonal retention -> inverse
// -> squared error per image (§6.1) for uint8 planes, every 8x8 block
// read from HBM exactly once through per-warp TMA tile rings in shared memory
// (fused_u8_wtile_kernel; design, measurements and the issue-bound analysis: DESIGN.md §5.2).
//
// The block computation (block_sse_u8s) is the exact-integer fp32 forward Y = T X T^T (all
// intermediates are integers < 2^24), weights W = 2/(n_k n_l) folded into the retained
// coefficients, the inverse x_hat = T^T (W o Y') T of the retained coefficients, and the
// squared error.  The inverse's last (vertical) butterfly x_hat_i = E_i + O_i,
// x_hat_{7-i} = E_i - O_i is fused with the error through the forward's first butterfly
// s_i = x_i + x_{7-i}, t_i = x_i - x_{7-i}:
//   (x_i - x_hat_i)^2 + (x_{7-i} - x_hat_{7-i})^2 = ((s_i - 2E_i)^2 + (t_i - 2O_i)^2) / 2.
// For r > 32 the inverse of the dropped coefficients is formed instead (x - x_hat directly,
// exactly 0 at r = 64; reading A17).  Samples enter fp32 by PRMT (pxf) or I2F.U8 (ubyte).
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstring>
#include <mutex>

#include "adct_host.h"
#include "tma.cuh"

namespace adct {

void launch_finalize(const double* partial, int32_t chunks, int64_t n_images, int32_t slots, const SlotMap& slot_of,
                     int32_t n_out, double npix, double peak, double* sse, double* psnr, cudaStream_t st);

bool make_u8_tmap(CUtensorMap* map, const uint8_t* src, const adct_geom& g, int tw, int rows) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)g.width, (cuuint64_t)g.height, (cuuint64_t)g.n_images};
  const cuuint64_t strides[2] = {(cuuint64_t)g.row_stride,
                                 (cuuint64_t)(g.n_images > 1 ? g.image_stride : (int64_t)g.height * g.row_stride)};
  const cuuint32_t box[3] = {(cuuint32_t)tw, (cuuint32_t)rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(src), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             // 128-byte boxes: 256-byte promotion over-fetches 14 % on 1920-byte rows (see blockmajor.cu)
             tw == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int sms_s() {
  return device_sms();
}

namespace {

__host__ __device__ constexpr int popc64s(uint64_t v) {
  int c = 0;
  for (int i = 0; i < 64; ++i) c += (int)((v >> i) & 1u);
  return c;
}
__host__ __device__ constexpr uint32_t row_mask_s(uint64_t nz) {
  uint32_t r = 0;
  for (int k = 0; k < 8; ++k)
    if ((nz >> (8 * k)) & 0xffull) r |= 1u << k;
  return r;
}

// Byte B of w as fp32 M + x with M = 2^15: one PRMT builds the bit pattern 0x4700xx00 from the
// constant 0x47000000 (held in a register).  PRMT issues on the ALU pipe at half rate, next to
// the FP32 work; I2F.U8 (byte-select convert) would run on the quarter-rate XU pipe
// (profiles/r01_probe_pipes.txt) and throttle the kernel.  Every row of T but the first sums
// to zero, so the bias only enters Y_00 (removed exactly in the weighting) and the sums
// s_i = x_i + x_{7-i} kept for the error (removed exactly, integers < 2^24).
template <uint32_t SEL>
__device__ __forceinline__ float pxf(uint32_t w, uint32_t magic) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(w), "r"(magic), "n"(SEL));
  return __uint_as_float(r);
}

// byte B of w as fp32 through I2F.U8 with a byte selector (no bias; quarter-rate XU pipe, used
// for a few columns only so that the XU pipe works next to the FMA and ALU pipes)
template <int B>
__device__ __forceinline__ float ubyte(uint32_t w) {
  float f;
  if constexpr (B == 0) asm("cvt.rn.f32.u8 %0, %1;" : "=f"(f) : "r"(w));
  else asm("{.reg .b32 t; shr.b32 t, %1, %2; cvt.rn.f32.u8 %0, t;}" : "=f"(f) : "r"(w), "n"(8 * B));
  return f;
}

#ifndef ADCT_XU_COLS
#define ADCT_XU_COLS 3
#endif
constexpr int kXuCols = ADCT_XU_COLS;  // columns of each block converted on the XU pipe

// ---- one 8x8 block: SSE of fwd -> retain R -> inv, u8 samples, no clip -------------------------
template <class MP, int R>
__device__ __forceinline__ float block_sse_u8s(const MP& m, const uint2 (&rows)[8], uint32_t magic) {
  constexpr uint64_t KEEP = keep_mask(R);
  constexpr bool RESID = popc64s(KEEP) > 32;
  constexpr uint64_t NZ = RESID ? ~KEEP : KEEP;
  constexpr uint32_t ROWS = row_mask_s(NZ);
  if constexpr (NZ == 0) {
    return 0.0f;  // r = 64: nothing dropped, x_hat = x
  } else {
    // vertical pass of the forward, P = T X (columns j), keeping s, t for the error
    float sv[4][8], tv[4][8], p[8][8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float xc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t w = j < 4 ? rows[i].x : rows[i].y;
        if (j < kXuCols) {
          switch (j & 3) {
            case 0: xc[i] = ubyte<0>(w); break;
            case 1: xc[i] = ubyte<1>(w); break;
            case 2: xc[i] = ubyte<2>(w); break;
            default: xc[i] = ubyte<3>(w); break;
          }
        } else {
          switch (j & 3) {
            case 0: xc[i] = pxf<0x7504u>(w, magic); break;
            case 1: xc[i] = pxf<0x7514u>(w, magic); break;
            case 2: xc[i] = pxf<0x7524u>(w, magic); break;
            default: xc[i] = pxf<0x7534u>(w, magic); break;
          }
        }
      }
      // s carries the bias 2M for PRMT-converted columns: removed exactly (integers < 2^24),
      // and the forward runs on the unbiased sums, so no coefficient carries a bias
      float t[4], col[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float sb = xc[i] + xc[7 - i];
        sv[i][j] = (j < kXuCols) ? sb : sb - 2.0f * kSampleBias;
        t[i] = xc[i] - xc[7 - i];
        tv[i][j] = t[i];
      }
      float su[4] = {sv[0][j], sv[1][j], sv[2][j], sv[3][j]};
      fwd8_st(m, su, t, col);
#pragma unroll
      for (int k = 0; k < 8; ++k) p[k][j] = col[k];
    }
    // horizontal pass Y = P T^T on the rows that hold retained (or dropped) coefficients,
    // weighting, and the horizontal pass of the inverse Q = (W o Y') T
    float q[8][8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (!((ROWS >> k) & 1u)) continue;
      float y[8], z[8];
      fwd8(m, p[k], y);
#pragma unroll
      for (int l = 0; l < 8; ++l)
        z[l] = ((NZ >> (k * 8 + l)) & 1ull) ? y[l] * m.wy2(k, l) : 0.0f;
#define ADCT_ROWINV_S(K)                                                        \
  if (k == K) {                                                                 \
    constexpr uint32_t rm = (uint32_t)((NZ >> (8 * K)) & 0xffull);              \
    if constexpr (rm != 0) inv8<MP, rm>(m, z, q[K]);                            \
  }
      ADCT_ROWINV_S(0) ADCT_ROWINV_S(1) ADCT_ROWINV_S(2) ADCT_ROWINV_S(3)
      ADCT_ROWINV_S(4) ADCT_ROWINV_S(5) ADCT_ROWINV_S(6) ADCT_ROWINV_S(7)
#undef ADCT_ROWINV_S
    }
    // vertical pass of the inverse up to its last butterfly, fused with the error:
    // dp_i = s_i - 2E_i, dm_i = t_i - 2O_i (the factor 2 is in the weights)
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float col[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) col[k] = ((ROWS >> k) & 1u) ? q[k][j] : 0.0f;
      if constexpr (RESID) {
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
          const float dp = sv[i][j] - e[i];
          const float dm = lsub<MP, 8, ROWS & 0xaau>(tv[i][j], [&](int k) { return m.h(i, k); }, col);
          acc[i] = fmaf(dp, dp, acc[i]);
          acc[i] = fmaf(dm, dm, acc[i]);
        }
      }
    }
    return 0.5f * ((acc[0] + acc[1]) + (acc[2] + acc[3]));
  }
}

// ---- warp-tile kernel ----------------------------------------------------------------------------
struct WtArgs {
  int32_t tpb, tpi, cpi;  // tiles per band pair / per image, chunks per image
  int32_t adv_pair, adv_slice;  // kWtWarps tiles = adv_pair tile rows + adv_slice tiles (adv_slice < tpb)
  uint32_t n_chunks;
  FastDiv dcpi, dtpb;
};

// The warp's walk over its tiles: chunks cg = blockIdx.x, +gridDim.x, ...; inside chunk cg the
// warp takes tiles w, w + 16, ... (< n).  Positions advance incrementally (no divisions per tile).
struct WtIt {
  uint32_t cg;
  int32_t j, n;
  uint32_t img;
  int32_t pair, slice;  // tile row (16 image rows) and column (256 bytes)
};

__device__ __forceinline__ void wt_enter(const WtArgs& a, int w, WtIt& it) {
  while (it.cg < a.n_chunks) {  // first chunk at or after it.cg in which this warp has a tile
    it.img = fdiv(it.cg, a.dcpi);
    const int32_t c = (int32_t)(it.cg - it.img * (uint32_t)a.cpi);
    it.n = min(kWtChunkTiles, a.tpi - c * kWtChunkTiles);
    if (w < it.n) {
      const uint32_t tt = (uint32_t)(c * kWtChunkTiles + w);
      it.pair = (int32_t)fdiv(tt, a.dtpb);
      it.slice = (int32_t)tt - it.pair * a.tpb;
      it.j = 0;
      return;
    }
    it.cg += gridDim.x;
  }
}

// advance to the next tile; returns true when the chunk changed
__device__ __forceinline__ bool wt_next(const WtArgs& a, int w, WtIt& it) {
  ++it.j;
  if (w + kWtWarps * it.j < it.n) {
    it.slice += a.adv_slice;  // both < tpb: at most one carry
    it.pair += a.adv_pair;
    if (it.slice >= a.tpb) {
      it.slice -= a.tpb;
      ++it.pair;
    }
    return false;
  }
  it.cg += gridDim.x;
  wt_enter(a, w, it);
  return true;
}

// The consumer's view of the same walk: only the chunk and the tiles left in it (the tile
// coordinates are needed by the prefetch walk alone).
struct WcIt {
  uint32_t cg;
  int32_t left;  // tiles of chunk cg this warp has still to consume
};

__device__ __forceinline__ void wc_enter(const WtArgs& a, int w, WcIt& it) {
  while (it.cg < a.n_chunks) {
    const uint32_t img = fdiv(it.cg, a.dcpi);
    const int32_t c = (int32_t)(it.cg - img * (uint32_t)a.cpi);
    const int32_t n = min(kWtChunkTiles, a.tpi - c * kWtChunkTiles);
    if (w < n) {
      it.left = (n - 1 - w) / kWtWarps + 1;  // tiles w, w + kWtWarps, ... < n
      return;
    }
    it.cg += gridDim.x;
  }
}

__device__ __forceinline__ bool wc_next(const WtArgs& a, int w, WcIt& it) {
  if (--it.left > 0) return false;
  it.cg += gridDim.x;
  wc_enter(a, w, it);
  return true;
}

#ifndef ADCT_WT_UNROLL
#define ADCT_WT_UNROLL 2
#endif
constexpr int kWtUnroll = ADCT_WT_UNROLL;  // unrolling of the per-lane block loop (code size vs ILP)

template <class MP, int R, int TW>
__global__ void __launch_bounds__(kWtThreads, 1)
    fused_u8_wtile_kernel(const __grid_constant__ CUtensorMap tmap, WtArgs a, DevMat dm, double* __restrict__ partial,
                          uint32_t magic) {
  constexpr int RT = kWtTileBytes / TW;  // rows per tile
  constexpr int BPR = TW / 8;            // blocks per band in a tile = lanes per band group
  static_assert(RT == 8 * kWtBPL * (32 / BPR), "tile shape");
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 127) & ~(uintptr_t)127);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wring = smem + (size_t)w * kWtSlots * kWtTileBytes;
  uint64_t* wfull = reinterpret_cast<uint64_t*>(smem + (size_t)kWtWarps * kWtSlots * kWtTileBytes) + w * kWtSlots;
  if (lane == 0) {
    for (int i = 0; i < kWtSlots; ++i) mbar_init(&wfull[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const MP m(dm);
  const uint32_t ring0 = smem_u32(wring), full0 = smem_u32(wfull);

  // prefetch walk: the same tile sequence the warp consumes, kWtSlots tiles ahead (lane 0)
  WtIt pf;
  pf.cg = blockIdx.x;
  wt_enter(a, w, pf);
  auto issue = [&](int slot) {
    if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full0 + slot * 8),
                   "r"((uint32_t)kWtTileBytes)
                   : "memory");
      tma_load_3d(ring0 + slot * kWtTileBytes, &tmap, pf.slice * TW, pf.pair * RT, (int32_t)pf.img,
                  full0 + slot * 8);
    }
    wt_next(a, w, pf);
  };
#pragma unroll 1
  for (int s = 0; s < kWtSlots; ++s)
    if (pf.cg < a.n_chunks) issue(s);

  // lane -> block column (lane % BPR) and its kWtBPL consecutive bands from kWtBPL*(lane / BPR)
  const uint32_t lane_u32 = ring0 + (uint32_t)(lane % BPR) * 8u + (uint32_t)(lane / BPR) * (8u * kWtBPL) * TW;
  int slot = 0;
  uint32_t phase = 0;
  WcIt it;
  it.cg = blockIdx.x;
  wc_enter(a, w, it);
  float acc = 0.0f;
  // chunks in which this warp has no tile keep a zero partial
  if (lane == 0)
    for (uint32_t cz = blockIdx.x; cz < min(it.cg, a.n_chunks); cz += gridDim.x) partial[(int64_t)cz * kWtWarps + w] = 0.0;
  while (it.cg < a.n_chunks) {
    mbar_wait(&wfull[slot], phase);
    const uint32_t p = lane_u32 + (uint32_t)slot * kWtTileBytes;
#pragma unroll kWtUnroll
    for (int b = 0; b < kWtBPL; ++b) {  // the lane's blocks (consecutive bands of the tile)
      uint2 rows[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) rows[i] = lds64(p + (uint32_t)(b * 8 + i) * TW);
      acc += block_sse_u8s<MP, R>(m, rows, magic);
    }
    __syncwarp();
    // the slot was read through the generic proxy; order that before the async-proxy refill
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (pf.cg < a.n_chunks) issue(slot);
    if (++slot == kWtSlots) { slot = 0; phase ^= 1u; }
    const uint32_t cg = it.cg;
    if (wc_next(a, w, it)) {  // chunk done: per-(chunk, warp) partial in a fixed shuffle order
      double v = (double)acc;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) {
        partial[(int64_t)cg * kWtWarps + w] = v;
        for (uint32_t cz = cg + gridDim.x; cz < min(it.cg, a.n_chunks); cz += gridDim.x)
          partial[(int64_t)cz * kWtWarps + w] = 0.0;
      }
      acc = 0.0f;
    }
  }
}

template <class MP, int R, int TW>
bool launch_wtile_rt(const CUtensorMap& map, const WtArgs& a, const DevMat& dm, double* partial, cudaStream_t st) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  // the shared-memory opt-in is a per-device function attribute: set it once per device
  static std::mutex mu;
  static bool done[64] = {};
  {
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 0 || dev >= 64) return false;
    if (!done[dev]) {
      if (cudaFuncSetAttribute(fused_u8_wtile_kernel<MP, R, TW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)kWtSmem) != cudaSuccess)
        return false;
      done[dev] = true;
    }
  }
  const int64_t grid = (int64_t)a.n_chunks < sms_s() ? (int64_t)a.n_chunks : sms_s();
  fused_u8_wtile_kernel<MP, R, TW><<<(unsigned)grid, kWtThreads, kWtSmem, st>>>(map, a, dm, partial, 0x47000000u);
  return true;
}

// the 128-byte tile shape is compiled for the paper's T1 only; other matrices use 256-byte tiles
template <class MP, int R>
bool launch_wtile_r(int tw, const CUtensorMap& map, const WtArgs& a, const DevMat& dm, double* partial,
                    cudaStream_t st) {
  if constexpr (MP::kConst && R == 10) {
    if (tw == 128) return launch_wtile_rt<MP, R, 128>(map, a, dm, partial, st);
  }
  return tw == 256 && launch_wtile_rt<MP, R, 256>(map, a, dm, partial, st);
}

// compiled (matrix, r) pairs: the paper's T1 at config 4's r = 10 and the r of the paper's
// Lena figures (3, 14), runtime matrices at r = 10; other pairs take the generic
// fused kernels (each instantiation of this kernel costs minutes of front-end compile time)
template <class MP>
bool launch_wtile(int r, int tw, const CUtensorMap& map, const WtArgs& a, const DevMat& dm, double* partial,
                  cudaStream_t st) {
  if constexpr (!MP::kConst) {
    return r == 10 && launch_wtile_r<MP, 10>(tw, map, a, dm, partial, st);
  } else {
    switch (r) {
#define ADCT_WT_CASE(R) \
  case R:               \
    return launch_wtile_r<MP, R>(tw, map, a, dm, partial, st);
      ADCT_WT_CASE(3) ADCT_WT_CASE(10) ADCT_WT_CASE(14)
#undef ADCT_WT_CASE
      default:
        return false;
    }
  }
}

}  // namespace

// The streaming path for (u8 source, integer matrix, no clip, one r); returns false when the
// geometry or r is not covered (the caller then uses the generic fused kernels).
// On success the per-image SSE is in sse[n_images] (finalize launched on st).

// ADCT_HOT=simt selects this file's SIMT streaming kernel instead of the tensor-core one (tc.cu;
// A/B runs and the SIMT parity tests)
static const bool g_hot_simt = [] {
  const char* e = std::getenv("ADCT_HOT");
  return e && std::strcmp(e, "simt") == 0;
}();

bool tc_hot_enabled() { return !g_hot_simt; }

bool fused_u8_stream(const adct_matrix* m, const uint8_t* src, const adct_geom& g, int32_t r, double* sse, double* psnr,
                     double* partial, cudaStream_t st, adct_status* status) {
  if (!g_hot_simt && fused_u8_tc(m, src, g, r, sse, psnr, partial, st, status)) return true;
  {
    WtPlan p = wt_plan(g);
    if (!p.ok || g.n_images == 0 || !aligned(src, 16)) return false;
    if (!m->specialized && p.tw != 256) {  // runtime matrices: 256-byte tiles only
      p.tw = 256;
      p.rows = kWtTileBytes / 256;
      p.tpb = (g.width + 255) / 256;
      p.tpi = ((g.height + p.rows - 1) / p.rows) * p.tpb;
      p.cpi = (p.tpi + kWtChunkTiles - 1) / kWtChunkTiles;
      p.n_chunks = g.n_images * (int64_t)p.cpi;
    }
    CUtensorMap map;
    if (!make_u8_tmap(&map, src, g, p.tw, p.rows)) return false;
    WtArgs a;
    a.tpb = p.tpb;
    a.tpi = p.tpi;
    a.cpi = p.cpi;
    a.n_chunks = (uint32_t)p.n_chunks;
    a.dcpi = make_fastdiv((uint32_t)p.cpi);
    a.dtpb = make_fastdiv((uint32_t)p.tpb);
    a.adv_pair = kWtWarps / p.tpb;
    a.adv_slice = kWtWarps % p.tpb;
    const bool ok = m->specialized ? launch_wtile<T1Mat>(r, p.tw, map, a, m->dev, partial, st)
                                   : launch_wtile<RtMat>(r, p.tw, map, a, m->dev, partial, st);
    if (!ok) return false;
    count_launch();
    if ((*status = launch_status()) != ADCT_OK) return true;
    SlotMap sm{};
    sm.s[0] = 0;
    launch_finalize(partial, p.cpi * kWtWarps, g.n_images, 1, sm, 1, (double)g.height * g.width, 255.0, sse,
                    psnr, st);
    *status = launch_status();
    return true;
  }
  return false;
}

}  // namespace adct
