// tc.cu — the tensor-core hot kernel of BASELINE.json config 4: forward -> zonal retention ->
// inverse -> squared error per image (§6.1) for uint8 planes, every 8x8
// block read from HBM exactly once (TMA tile rings), the linear part of the forward on tcgen05.
//
// Per block x (64 samples, k = 8i + j) the tensor core computes, exactly, the outputs
//   Y_kl = sum_ij T_ki T_lj x_ij     for the retained (k,l)          (Eq. 1)
//   s_i[j] = x_ij + x_(7-i)j,  t_i[j] = x_ij - x_(7-i)j   (i < 4)     (first column butterfly)
// as D = A B^T with A = the block as f16 (one row of the M = 128 tile per block; a u8 sample x
// is the f16 SUBNORMAL x * 2^-24, built by one PRMT per two samples) and B = the constant
// [outputs x 64] matrix of those coefficients (integers |b| <= 4, exact in f16).  Products and
// partial sums are integers times 2^-24 below 2^24 * 2^-24, so the fp32 accumulators hold the
// exact integer results scaled by 2^-24 (probes/tc_probe.cu).  The thread that owns the block
// then runs the same fp32 arithmetic as the SIMT kernel (stream.cu, block_sse_u8s): weights
// 2/(n_k n_l), the horizontal inverse Q = (W o Y') T of the retained rows, and the vertical
// inverse fused with the error, (x_i - x^_i)^2 + (x_7-i - x^_7-i)^2 = ((s_i - 2E_i)^2 +
// (t_i - 2O_i)^2)/2.  Every fp32 value carries the exact factor 2^-24 (no subnormal occurs), so
// the per-block SSE is 2^-48 times that of the SIMT kernel bit for bit; the fp64 partial
// removes the factor exactly.  For r > 32 the inverse of the dropped coefficients is formed
// (exactly 0 at r = 64; reading A17) and s, t are not needed.
//
// Roles inside a persistent CTA (one per SM): kTcGroups groups of 4 warps; warp q of a group
// reads TMEM lanes 32q..32q+31.  Per group and tile: one lane issues the TMA load of the 8 KB
// tile (kTcSlots-deep ring), every thread converts its block and tcgen05.st's it into the
// group's A columns, a named barrier joins the 4 warps, one lane issues 4 MMAs (K = 64) and
// commits to the group's mbarrier, and every thread tcgen05.ld's its block's outputs.  Groups
// never wait for each other, so the SM's issue slots stay busy while one group waits for its
// MMA.  DESIGN.md §5.2.
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "adct_host.h"
#include "tc05.cuh"
#include "tma.cuh"

namespace adct {

void launch_finalize(const double* partial, int32_t chunks, int64_t n_images, int32_t slots, const SlotMap& slot_of,
                     int32_t n_out, double npix, double peak, double* sse, double* psnr, cudaStream_t st);
bool make_u8_tmap(CUtensorMap* map, const uint8_t* src, const adct_geom& g, int tw, int rows);
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
  static constexpr int N = NY + (RESID ? 0 : 64);       // + s_i[j], t_i[j]: column NY + 8j + i (+4 for t)
  static constexpr uint32_t ROWS = row_mask_t(NZ);
  static_assert(NNZ <= 32, "at most 32 coefficient columns");
  static_assert(N <= 96, "TMEM budget: kTcGroups x (N + 32) <= 512 columns");
};

// index of coefficient p = k*8+l among the set bits of NZ (its D column)
template <uint64_t NZ>
__host__ __device__ constexpr int nz_index(int p) {
  return popc64t(NZ & ((p == 0) ? 0ull : (~0ull >> (64 - p))));
}

// ---- one block from its D row (in registers): the fp32 inverse and squared error ------------
// yr: the NY coefficient columns; st: s_i[j] at 8j + i, t_i[j] at 8j + 4 + i.  Returns 2^-48 x SSE.
template <class MP, int R>
__device__ __forceinline__ float tc_block_sse(const MP& m, const uint32_t* yr, const uint32_t* st) {
  using S = TcShape<R>;
  constexpr uint64_t NZ = S::NZ;
  constexpr uint32_t ROWS = S::ROWS;
  if constexpr (S::NNZ == 0) {
    return 0.0f;  // r = 64
  } else {
    // horizontal inverse of the weighted retained coefficients, Q = (W o Y') T, rows in ROWS
    float q[8][8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (!((ROWS >> k) & 1u)) continue;
      float z[8];
#pragma unroll
      for (int l = 0; l < 8; ++l)
        z[l] = ((NZ >> (k * 8 + l)) & 1ull) ? __uint_as_float(yr[nz_index<NZ>(k * 8 + l)]) * m.wy2(k, l) : 0.0f;
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
          const float dp = __uint_as_float(st[8 * j + i]) - e[i];
          const float dm =
              lsub<MP, 8, ROWS & 0xaau>(__uint_as_float(st[8 * j + 4 + i]), [&](int k) { return m.h(i, k); }, col);
          acc[i] = fmaf(dp, dp, acc[i]);
          acc[i] = fmaf(dm, dm, acc[i]);
        }
      }
    }
    return 0.5f * ((acc[0] + acc[1]) + (acc[2] + acc[3]));
  }
}

// ---- the CTA's tiles: chunks cg = blockIdx.x, +gridDim.x, ...; a chunk is kTcChunkTiles
// consecutive tiles of one image (fewer at the image's end), taken in order ------------------
struct TcArgs {
  int32_t tpb, tpi, cpi;
  uint32_t n_chunks;
  FastDiv dcpi, dtpb;
};

__device__ __forceinline__ int32_t chunk_tiles(const TcArgs& a, uint32_t cg, uint32_t& img, int32_t& tt0) {
  img = fdiv(cg, a.dcpi);
  tt0 = (int32_t)(cg - img * (uint32_t)a.cpi) * kTcChunkTiles;
  return min(kTcChunkTiles, a.tpi - tt0);
}

struct TcPf {  // the TMA issuer's walk: coordinates of the next tile to load
  uint32_t cg, img;
  int32_t j, n, pair, slice;
};
__device__ __forceinline__ void pf_enter(const TcArgs& a, TcPf& f) {
  if (f.cg >= a.n_chunks) return;
  int32_t tt0;
  f.n = chunk_tiles(a, f.cg, f.img, tt0);
  f.j = 0;
  f.pair = (int32_t)fdiv((uint32_t)tt0, a.dtpb);
  f.slice = tt0 - f.pair * a.tpb;
}
__device__ __forceinline__ void pf_next(const TcArgs& a, TcPf& f) {
  if (++f.j < f.n) {
    if (++f.slice == a.tpb) {
      f.slice = 0;
      ++f.pair;
    }
  } else {
    f.cg += gridDim.x;
    pf_enter(a, f);
  }
}

// B[n][k] of the MMA (row n = output, k = 8i + j), integers |b| <= 4
template <class MP, int R>
__device__ __forceinline__ float tc_bval(const MP& m, int n, int k) {
  using S = TcShape<R>;
  const int i = k >> 3, j = k & 7;
  if (n < S::NNZ) {
    int p = 0, c = -1;
    for (; p < 64; ++p)
      if ((S::NZ >> p) & 1ull)
        if (++c == n) break;
    return m.f(p >> 3, i) * m.f(p & 7, j);
  }
  if (n < S::NY) return 0.0f;
  const int jj = (n - S::NY) >> 3, r = (n - S::NY) & 7;
  if (j != jj) return 0.0f;
  if (r < 4) return (i == r || i == 7 - r) ? 1.0f : 0.0f;       // s_r[j]
  return i == r - 4 ? 1.0f : (i == 11 - r ? -1.0f : 0.0f);      // t_(r-4)[j]
}

template <class MP, int R, int TW>
__global__ void __launch_bounds__(kTcThreads, 1)
    fused_u8_tc_kernel(const __grid_constant__ CUtensorMap tmap, TcArgs a, DevMat dm, double* __restrict__ partial,
                       long long* __restrict__ trace) {
  // trace (debug builds with ADCT_TC_TRACE): clock64 stamps of CTA 0's first kTrTiles tiles
  constexpr int kTrTiles = 64;
#ifdef ADCT_TC_TRACE
#define TR(slot, tile) \
  { if (trace && blockIdx.x == 0 && (tile) < kTrTiles && lane == 0) trace[(tile) * 16 + (slot)] = clock64(); }
#else
#define TR(slot, tile) {}
#endif
  using S = TcShape<R>;
  constexpr int N = S::N;
  constexpr int RT = kTcTileBytes / TW;  // rows per tile
  constexpr int BPR = TW / 8;            // blocks per band in a tile
  constexpr uint32_t kIdesc = idesc_f16_f32<128, N>();
  constexpr uint32_t kTmemCols = 512;
  constexpr uint32_t kACol0 = (uint32_t)(kTcDStages * N);  // A stages after the D stages
  static_assert(kTcDStages * N + kTcAStages * 32 <= (int)kTmemCols, "TMEM columns");
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 127) & ~(uintptr_t)127);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = w & 3;  // TMEM lane quarter of this warp (hardware: warp w accesses lanes 32 (w % 4) ..)
  uint8_t* sB = smem + (size_t)kTcSlots * kTcTileBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kTcBBytes);  // [kTcSlots]  TMA tile landed
  uint64_t* afull = full + kTcSlots;                              // [2]  A stage written (4 warps)
  uint64_t* dfull = afull + kTcAStages;                           // [D]  MMA of the tile done (commit)
  uint64_t* dfree = dfull + kTcDStages;                           // [D]  D read by the 4 epilogue warps
  uint64_t* sfree = dfree + kTcDStages;                           // [kTcSlots]  slot read by the 4 converters
  uint32_t* holder = reinterpret_cast<uint32_t*>(sfree + kTcSlots);
  const MP m(dm);

  // B in the canonical K-major no-swizzle layout: core matrix (n/8, k/8) at (n/8)*1024 + (k/8)*128
  for (int idx = threadIdx.x; idx < N * 64; idx += kTcThreads) {
    const int n = idx >> 6, k = idx & 63;
    const __half h = __float2half_rn(tc_bval<MP, R>(m, n, k));
    *reinterpret_cast<__half*>(sB + (n >> 3) * 1024 + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2) = h;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kTcSlots; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&sfree[i], 4);
    }
    for (int i = 0; i < kTcAStages; ++i) {
      mbar_init(&afull[i], 4);
    }
    for (int i = 0; i < kTcDStages; ++i) {
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
  const uint32_t lane_q = (uint32_t)(32 * q) << 16;
  const uint32_t full0 = smem_u32(full), ring0 = smem_u32(smem), sB_u = smem_u32(sB);

  if (w == kTcConv0 + 5) {
    // ======== TMA producer: a slot is refilled once every quarter has converted its tile ========
    TcPf pf;
    pf.cg = blockIdx.x;
    pf_enter(a, pf);
    uint32_t slot = 0, sph = 0, t = 0;
#pragma unroll 1
    for (; pf.cg < a.n_chunks; ++t) {
      if (t >= (uint32_t)kTcSlots) mbar_wait(&sfree[slot], sph ^ 1u);  // tile t - kTcSlots read by all 4 quarters
      if (elect_one()) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full0 + slot * 8),
                     "r"((uint32_t)kTcTileBytes)
                     : "memory");
        tma_load_3d(ring0 + slot * kTcTileBytes, &tmap, pf.slice * TW, pf.pair * RT, (int32_t)pf.img,
                    full0 + slot * 8);
      }
      __syncwarp();
      pf_next(a, pf);
      if (++slot == kTcSlots) {
        slot = 0;
        sph ^= 1u;
      }
    }
  } else if (w == kTcConv0 + 4) {
    // ======== MMA issuer: one elected lane issues every tile's MMA ========
    uint32_t ds = 0, dph = 0, as = 0, aph = 0, t = 0;
#pragma unroll 1
    for (uint32_t cg = blockIdx.x; cg < a.n_chunks; cg += gridDim.x) {
      uint32_t img;
      int32_t tt0;
      const int32_t n = chunk_tiles(a, cg, img, tt0);
#pragma unroll 1
      for (int32_t j = 0; j < n; ++j, ++t) {
        TR(4, t)
        mbar_wait(&afull[as], aph);                                      // all 4 quarters of A written
        TR(5, t)
        if (t >= (uint32_t)kTcDStages) mbar_wait(&dfree[ds], dph ^ 1u);  // tile t - D read by the epilogue
        tc_fence_after();
        if (elect_one()) {
          const uint32_t tDs = tbase + (uint32_t)(N * ds), tAs = tbase + kACol0 + 32 * as;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_f16_ts(tDs, tAs + 8 * kk, smem_desc_kmajor(sB_u + kk * 256, 128, 1024), kIdesc, kk > 0 ? 1u : 0u);
          mma_commit(smem_u32(&dfull[ds]));  // D of tile t written (A of tile t free again)
        }
        __syncwarp();
        TR(6, t)
        if (++ds == kTcDStages) {
          ds = 0;
          dph ^= 1u;
        }
        if (++as == (uint32_t)kTcAStages) {
          as = 0;
          aph ^= 1u;
        }
      }
    }
  } else if (w >= kTcConv0) {
    // ======== converters (warps kTcConv0 .. +3, one per TMEM lane quarter) ========
    // the thread's block in a tile: band (q or 2q + lane/16) and column, rows at stride TW
    const int band = (BPR == 32) ? q : 2 * q + (lane >> 4);
    const uint32_t my_off = (uint32_t)(band * 8 * TW + (lane % BPR) * 8);
    uint32_t slot = 0, phase = 0, as = 0, aph = 0, t = 0;
#pragma unroll 1
    for (uint32_t cg = blockIdx.x; cg < a.n_chunks; cg += gridDim.x) {
      uint32_t img;
      int32_t tt0;
      const int32_t n = chunk_tiles(a, cg, img, tt0);
#pragma unroll 1
      for (int32_t j = 0; j < n; ++j, ++t) {
        if (q == 1) TR(0, t)
        if (t >= (uint32_t)kTcAStages) {  // the MMA of tile t - A (the last reader of A[as]) has completed
          const uint32_t tp = t - kTcAStages;
          mbar_wait(&dfull[tp % kTcDStages], (tp / kTcDStages) & 1u);
        }
        if (q == 1) TR(1, t)
        mbar_wait(&full[slot], phase);
        if (q == 1) TR(2, t)
        const uint32_t p = ring0 + slot * kTcTileBytes + my_off;
        const uint32_t tA = tbase + lane_q + kACol0 + 32 * as;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t av[16];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint2 r = lds64(p + (uint32_t)((4 * h + i) * TW));
            // f16x2 subnormals {x_2c, x_2c+1} * 2^-24: bytes [x, 0, x', 0]
            asm("prmt.b32 %0, %1, 0, 0x4140;" : "=r"(av[4 * i + 0]) : "r"(r.x));
            asm("prmt.b32 %0, %1, 0, 0x4342;" : "=r"(av[4 * i + 1]) : "r"(r.x));
            asm("prmt.b32 %0, %1, 0, 0x4140;" : "=r"(av[4 * i + 2]) : "r"(r.y));
            asm("prmt.b32 %0, %1, 0, 0x4342;" : "=r"(av[4 * i + 3]) : "r"(r.y));
          }
#ifndef ADCT_TC_ABL_NOSTTM
          tmem_st16(tA + 16 * h, av);
#else
          if (av[0] == 0x12345u && av[15] == 7u) tmem_st16(tA + 16 * h, av);
#endif
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&sfree[slot]);  // the producer may refill the slot
          mbar_arrive(&afull[as]);    // the issuer may run the MMA
        }
        if (q == 1) TR(3, t)
        if (++slot == kTcSlots) {
          slot = 0;
          phase ^= 1u;
        }
        if (++as == (uint32_t)kTcAStages) {
          as = 0;
          aph ^= 1u;
        }
      }
    }
  } else {
    // ======== epilogue warps: quarter q, index e; tiles t = e, e + kTcEpi, ... of the CTA ========
    const int e = w >> 2;
    uint32_t yr[S::NY], st[64];
    (void)st;
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
        const uint32_t d = tt % kTcDStages;
        if (q == 0) TR(8, tt)
        mbar_wait(&dfull[d], (tt / kTcDStages) & 1u);
        if (q == 0) TR(9, tt)
        tc_fence_after();
        const uint32_t tD = tbase + lane_q + (uint32_t)(N * d);
#ifdef ADCT_TC_ABL_NOLDTM
        if (tt == 0xffffffffu)
#endif
        if constexpr (S::NY == 16) tmem_ld16(tD, yr);
        else tmem_ld32(tD, yr);
#ifdef ADCT_TC_ABL_NOLDTM
        if (tt == 0xffffffffu)
#endif
        if constexpr (!S::RESID) {
          tmem_ld32(tD + S::NY, *reinterpret_cast<uint32_t(*)[32]>(&st[0]));
          tmem_ld32(tD + S::NY + 32, *reinterpret_cast<uint32_t(*)[32]>(&st[32]));
        }
        tmem_wait_ld(yr);
        if constexpr (!S::RESID) tmem_wait_ld(st);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dfree[d]);  // the MMA of tile tt + D may overwrite the stage
        if (q == 0) TR(10, tt)
#ifndef ADCT_TC_ABL_NOEPI
        acc += tc_block_sse<MP, R>(m, yr, st);
#else
        acc += __uint_as_float(yr[0]);
#endif
        if (q == 0) TR(11, tt)
      }
      double v = (double)acc;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) partial[((int64_t)cg * kTcEpi + sl) * 4 + q] = v * 0x1p48;  // remove 2^-48
      t += (uint32_t)n;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<kTmemCols>(tbase);
#undef TR
}

template <class MP, int R, int TW>
bool launch_tc_rt(const CUtensorMap& map, const TcArgs& a, const DevMat& dm, double* partial, cudaStream_t st) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  // the shared-memory opt-in is a per-device function attribute: set it once per device
  static std::mutex mu;
  static bool done[64] = {};
  {
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 0 || dev >= 64) return false;
    if (!done[dev]) {
      if (cudaFuncSetAttribute(fused_u8_tc_kernel<MP, R, TW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)kTcSmem) != cudaSuccess)
        return false;
      done[dev] = true;
    }
  }
  const int64_t grid = (int64_t)a.n_chunks < sms_s() ? (int64_t)a.n_chunks : sms_s();
  long long* trace = nullptr;
#ifdef ADCT_TC_TRACE
  static long long* tbuf = nullptr;
  if (!tbuf && cudaMalloc(&tbuf, 64 * 16 * sizeof(long long)) != cudaSuccess) tbuf = nullptr;
  if (tbuf) cudaMemsetAsync(tbuf, 0, 64 * 16 * sizeof(long long), st);
  trace = tbuf;
#endif
  fused_u8_tc_kernel<MP, R, TW><<<(unsigned)grid, kTcThreads, kTcSmem, st>>>(map, a, dm, partial, trace);
#ifdef ADCT_TC_TRACE
  if (tbuf) {
    long long h[64 * 16];
    cudaMemcpyAsync(h, tbuf, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (FILE* f = std::fopen("gpurun_out/tc_trace.txt", "w")) {
      for (int i = 0; i < 64; ++i) {
        for (int k = 0; k < 16; ++k) std::fprintf(f, "%lld ", h[i * 16 + k] ? h[i * 16 + k] - h[0] : -1);
        std::fprintf(f, "\n");
      }
      std::fclose(f);
    }
  }
#endif
  return true;
}

template <class MP, int R>
bool launch_tc_r(int tw, const CUtensorMap& map, const TcArgs& a, const DevMat& dm, double* partial,
                 cudaStream_t st) {
  if (tw == 128) return launch_tc_rt<MP, R, 128>(map, a, dm, partial, st);
  return tw == 256 && launch_tc_rt<MP, R, 256>(map, a, dm, partial, st);
}

// compiled (matrix, r) pairs: T1 at config 4's r = 10 and the Lena figures' r = 3, 14
// (P:L2380-2444); runtime integer matrices at r = 10
template <class MP>
bool launch_tc(int r, int tw, const CUtensorMap& map, const TcArgs& a, const DevMat& dm, double* partial,
               cudaStream_t st) {
  if constexpr (!MP::kConst) {
    return r == 10 && launch_tc_r<MP, 10>(tw, map, a, dm, partial, st);
  } else {
    switch (r) {
      case 3: return launch_tc_r<MP, 3>(tw, map, a, dm, partial, st);
      case 10: return launch_tc_r<MP, 10>(tw, map, a, dm, partial, st);
      case 14: return launch_tc_r<MP, 14>(tw, map, a, dm, partial, st);
      default: return false;
    }
  }
}

}  // namespace

// The tensor-core streaming path for (u8 source, integer matrix, no clip, one r); false when
// the geometry or r is not covered (the caller then tries the SIMT streaming kernel).
bool fused_u8_tc(const adct_matrix* m, const uint8_t* src, const adct_geom& g, int32_t r, double* sse,
                 double* partial, cudaStream_t st, adct_status* status) {
  const WtPlan p = tc_plan(g);
  if (!p.ok || g.n_images == 0 || !aligned(src, 16) || !m->is_int) return false;
  CUtensorMap map;
  if (!make_u8_tmap(&map, src, g, p.tw, p.rows)) return false;
  TcArgs a;
  a.tpb = p.tpb;
  a.tpi = p.tpi;
  a.cpi = p.cpi;
  a.n_chunks = (uint32_t)p.n_chunks;
  a.dcpi = make_fastdiv((uint32_t)p.cpi);
  a.dtpb = make_fastdiv((uint32_t)p.tpb);
  const bool ok = m->specialized ? launch_tc<T1Mat>(r, p.tw, map, a, m->dev, partial, st)
                                 : launch_tc<RtMat>(r, p.tw, map, a, m->dev, partial, st);
  if (!ok) return false;
  count_launch();
  if ((*status = launch_status()) != ADCT_OK) return true;
  SlotMap sm{};
  sm.s[0] = 0;
  launch_finalize(partial, p.cpi * kTcPartials, g.n_images, 1, sm, 1, (double)g.height * g.width, 255.0, sse, nullptr,
                  st);
  *status = launch_status();
  return true;
}

}  // namespace adct
