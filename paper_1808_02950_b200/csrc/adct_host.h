// adct_host.h — host-side internals shared by the library's translation units.
#pragma once
#include <atomic>
#include <cstdint>

#include "adct.h"
#include "adct_internal.cuh"

struct adct_matrix {
  adct::DevMat dev;       // what kernels receive (by value, kernel parameter space)
  int32_t t[64];          // integer matrix (is_int)
  double chat[64];        // C_hat = S T (or the real matrix)
  double g[64];           // synthesis: A = G B' G^T
  double s[8];            // row scaling
  int64_t n[8];           // n_k = ||t_k||^2 (integer matrices)
  int32_t is_int;
  int32_t row_orth;
  int32_t specialized;    // 1 = the paper's T1 (compile-time network available)
  int64_t max_u8, max_i16;
};

namespace adct {

extern std::atomic<int64_t> g_launches;

inline void count_launch(int64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

inline adct_status check_geom(const adct_geom& g) {
  if (g.n_images < 0 || g.height <= 0 || g.width <= 0) return ADCT_E_INVALID_ARGUMENT;
  if ((g.height % 8) || (g.width % 8)) return ADCT_E_INVALID_ARGUMENT;
  if (g.row_stride < g.width || (g.row_stride % 8)) return ADCT_E_ALIGNMENT;
  if (g.n_images > 1 && g.image_stride < (int64_t)g.height * g.row_stride) return ADCT_E_INVALID_ARGUMENT;
  if (g.image_stride % 8) return ADCT_E_ALIGNMENT;
  const int64_t nb = g.n_images * (int64_t)(g.height / 8) * (g.width / 8);
  if (nb >= ((int64_t)1 << 31)) return ADCT_E_INVALID_ARGUMENT;  // per-call block index is 32-bit
  return ADCT_OK;
}

inline bool aligned(const void* p, uintptr_t a) { return ((uintptr_t)p % a) == 0; }

inline adct_status launch_status() {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ADCT_OK : ADCT_E_CUDA;
}

// geometry passed to kernels
struct KGeom {
  int64_t image_stride, row_stride;
  uint32_t bw, bh, nbi;  // blocks per row, block rows, blocks per image
  uint32_t n_images;
};

inline KGeom make_kgeom(const adct_geom& g) {
  KGeom k;
  k.image_stride = g.image_stride;
  k.row_stride = g.row_stride;
  k.bw = (uint32_t)(g.width / 8);
  k.bh = (uint32_t)(g.height / 8);
  k.nbi = k.bw * k.bh;
  k.n_images = (uint32_t)g.n_images;
  return k;
}

// number of CTAs per image of the two-level deterministic reductions
constexpr int kRedNT = 128;   // threads per CTA
constexpr int kFusedBPT = 8;    // blocks per thread, generic fused kernels
inline int64_t fused_chunks(const adct_geom& g, int bpt = kFusedBPT) {
  const int64_t nbi = (int64_t)(g.height / 8) * (g.width / 8);
  const int64_t per = (int64_t)kRedNT * bpt;
  return (nbi + per - 1) / per;
}
constexpr int kSseRows = 8;  // image rows per CTA in psnr_reduce
inline int64_t sse_chunks(const adct_geom& g) { return (g.height + kSseRows - 1) / kSseRows; }

// ---- warp-tile streaming kernel (the default hot kernel) ---------------------------------------
// Every warp owns a private ring of kWtSlots tiles.  A tile is 16 image rows x 256 bytes (two
// bands of 32 horizontally adjacent 8x8 blocks: 2 blocks per lane), fetched by ONE TMA tensor
// copy (cp.async.bulk.tensor.3d over a {W, H, n_images} uint8 tensor map, box {256, 16, 1};
// out-of-range parts are zero-filled, and an all-zero block has exactly zero error) that
// completes on the warp's own mbarrier.  No producer warp and no cross-warp barrier: each warp
// refills the slot it just consumed.  A chunk is kWtChunkTiles consecutive tiles of one image;
// per-(chunk, warp) fp64 partials keep the per-image sums independent of the grid.
#ifndef ADCT_WT_WARPS
#define ADCT_WT_WARPS 16
#endif
constexpr int kWtWarps = ADCT_WT_WARPS;
constexpr int kWtThreads = 32 * kWtWarps;
#ifndef ADCT_WT_BPL
#define ADCT_WT_BPL 2
#endif
constexpr int kWtBPL = ADCT_WT_BPL;                 // blocks per lane per tile
constexpr int kWtTileBytes = 2048 * kWtBPL;         // 32 * kWtBPL blocks of 64 bytes
#ifndef ADCT_WT_SLOTS
#define ADCT_WT_SLOTS 3
#endif
constexpr int kWtSlots = ADCT_WT_SLOTS;             // ring depth (16 x 3 x 4 KB = 192 KB of shared memory)
static_assert((size_t)kWtWarps * kWtSlots * kWtTileBytes <= 200 * 1024, "warp-tile rings exceed shared memory");
#ifndef ADCT_WT_CHUNK
#define ADCT_WT_CHUNK 16
#endif
constexpr int kWtChunkTiles = kWtWarps * ADCT_WT_CHUNK;  // tiles per warp per chunk x 16 warps
constexpr size_t kWtSmem = (size_t)kWtWarps * kWtSlots * kWtTileBytes + (size_t)kWtWarps * kWtSlots * 8 + 128;

// tile shape: tw bytes wide (256 = 32 blocks per band, or 128 = 16 blocks) x 4096/tw rows
// (2 or 4 bands); the shape that wastes the fewest zero-filled blocks is chosen per geometry
struct WtPlan {
  int32_t tw, rows;  // tile width (bytes) and height (rows)
  int32_t tpb;       // tiles per tile row (ceil(W / tw))
  int32_t tpi;       // tiles per image
  int32_t cpi;       // chunks per image
  int64_t n_chunks;
  bool ok;
};
inline WtPlan tile_plan(const adct_geom& g, int tile_bytes, int chunk_tiles) {
  WtPlan p{};
  const int64_t W = g.width, H = g.height;
  if (W <= 0 || H <= 0) return p;
  int64_t best = -1;
  for (int tw : {256, 128}) {
    const int64_t rows = tile_bytes / tw;
    const int64_t tiles = ((W + tw - 1) / tw) * ((H + rows - 1) / rows);
    if (best < 0 || tiles < best) {  // equal tile counts -> equal waste; keep the wider tile
      best = tiles;
      p.tw = tw;
      p.rows = (int32_t)rows;
    }
  }
  p.tpb = (int32_t)((W + p.tw - 1) / p.tw);
  p.tpi = (int32_t)(((H + p.rows - 1) / p.rows) * p.tpb);
  p.cpi = (p.tpi + chunk_tiles - 1) / chunk_tiles;
  p.n_chunks = g.n_images * (int64_t)p.cpi;
  // tensor-map constraints: 16-byte aligned strides (< 2^40), dimensions < 2^32
  p.ok = (g.row_stride % 16) == 0 && (g.image_stride % 16) == 0 && g.image_stride < ((int64_t)1 << 40) &&
         p.n_chunks < ((int64_t)1 << 31);
  return p;
}

inline WtPlan wt_plan(const adct_geom& g) { return tile_plan(g, kWtTileBytes, kWtChunkTiles); }

// ---- tensor-core streaming kernel (fused_u8_tc_kernel, tc.cu; the default hot kernel) ----------
// One persistent CTA per SM, warp-specialized.  A tile is 128 blocks (8 KB of u8 pixels, one TMA
// box of 256 B x 32 rows or 128 B x 64 rows) = one M = 128 MMA.  Warps 0-3 (one per TMEM lane
// quarter) convert the tile's blocks to f16 (exact subnormals x * 2^-24) into one of kTcAStages A
// stages in TMEM; lane 0 of warp 0 also issues the kind::f16 MMA against the constant matrix B
// in shared memory (retained Y = T X T^T and the column butterflies s, t of X, exact in fp32)
// into one of kTcDStages D stages, and the TMA loads of the kTcSlots-deep tile ring.  Warps
// 4.. are epilogue warps, kTcEpi per lane quarter, taking the CTA's tiles round-robin: each
// reads its 32 blocks' D rows, releases the stage, and runs the fp32 inverse and squared error.
// Per-(chunk, slot, quarter) fp64 partials, slot = tile index in the chunk mod kTcEpi.
#ifndef ADCT_TC_EPI
#define ADCT_TC_EPI 3
#endif
constexpr int kTcEpi = ADCT_TC_EPI;                 // epilogue warps per lane quarter
constexpr int kTcWarps = 4 * kTcEpi + 4 + 2;      // epilogue, converters, MMA issuer, TMA producer
constexpr int kTcConv0 = 4 * kTcEpi;              // first converter warp (a multiple of 4)
constexpr int kTcThreads = 32 * kTcWarps;
constexpr int kTcTileBytes = 8192;
#ifndef ADCT_TC_SLOTS
#define ADCT_TC_SLOTS 12
#endif
constexpr int kTcSlots = ADCT_TC_SLOTS;  // TMA ring depth (tiles)
#ifndef ADCT_TC_ASTAGES
#define ADCT_TC_ASTAGES 2
#endif
constexpr int kTcAStages = ADCT_TC_ASTAGES;

#ifndef ADCT_TC_DSTAGES
#define ADCT_TC_DSTAGES 5
#endif
constexpr int kTcDStages = ADCT_TC_DSTAGES;
#ifndef ADCT_TC_CHUNK
#define ADCT_TC_CHUNK 16
#endif
constexpr int kTcChunkTiles = ADCT_TC_CHUNK;      // tiles per chunk
constexpr int kTcPartials = 4 * kTcEpi;           // partials per chunk
constexpr int kTcBBytes = 96 * 64 * 2;            // B: N <= 96 outputs x K = 64 f16
constexpr int kTcBars = 2 * kTcSlots + kTcAStages + 2 * kTcDStages;
static_assert(kTcAStages < kTcDStages, "converters wait on the D barrier of tile t - kTcAStages");
constexpr size_t kTcSmem = (size_t)kTcSlots * kTcTileBytes + kTcBBytes + (size_t)kTcBars * 8 + 16 + 128;
static_assert(kTcSmem <= 227 * 1024, "tensor-core kernel exceeds shared memory");
inline WtPlan tc_plan(const adct_geom& g) { return tile_plan(g, kTcTileBytes, kTcChunkTiles); }

inline int64_t stream_partials_per_image(const adct_geom& g) {
  int64_t best = 0;
  for (int tw : {256, 128}) {  // either tensor-core tile shape may be used
    const int64_t rows = kTcTileBytes / tw;
    const int64_t tpi = ((g.width + tw - 1) / tw) * ((g.height + rows - 1) / rows);
    const int64_t c = (tpi + kTcChunkTiles - 1) / kTcChunkTiles * kTcPartials;
    if (c > best) best = c;
  }
  for (int tw : {256, 128}) {  // either warp-tile shape may be used (runtime matrices: 256 only)
    const int64_t rows = kWtTileBytes / tw;
    const int64_t tpi = ((g.width + tw - 1) / tw) * ((g.height + rows - 1) / rows);
    const int64_t c = (tpi + kWtChunkTiles - 1) / kWtChunkTiles * kWtWarps;
    if (c > best) best = c;
  }
  return best;
}

}  // namespace adct
