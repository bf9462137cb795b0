// adct_host.h — host-side internals shared by the library's translation units.
#pragma once
#include <atomic>
#include <cstdint>
#include <mutex>
#include <utility>

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

// Function attributes, __constant__ data, streams and SM counts are per device: everything the
// library sets up lazily is keyed by the current device (cudaGetDevice), so a process that
// calls it on cuda:1 after cuda:0 gets its own setup there.
constexpr int kMaxDevices = 64;
int device_sms();  // SM count of the current device (basic.cu), 148 on B200
// Run f() (returning bool) once per device; the result is remembered, so a failed setup keeps
// failing.  false also when the current device cannot be determined.
template <class F>
inline bool once_per_device(std::mutex& mu, int8_t (&state)[kMaxDevices], F&& f) {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return false;
  std::lock_guard<std::mutex> lk(mu);
  if (state[dev] == 0) state[dev] = f() ? 1 : -1;
  return state[dev] == 1;
}

// Programmatic dependent launch (ADCT_PDL): the persistent stream kernels and their finalize are
// launched with programmatic stream serialization, call griddepcontrol.launch_dependents at
// entry and griddepcontrol.wait before their first global memory access, so a launch's
// prologue (barrier init, TMEM allocation, the B operand) overlaps the previous kernel's tail
// while every kernel still completes after the one before it.
#ifndef ADCT_PDL
#define ADCT_PDL 1
#endif
__device__ __forceinline__ void pdl_launch_dependents() {
#if ADCT_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_wait() {
#if ADCT_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
template <typename... K, typename... A>
inline cudaError_t launch_pdl(void (*kernel)(K...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = ADCT_PDL ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);
}

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
// One persistent CTA per SM, warp-specialized: kTcEpi epilogue warps per TMEM lane quarter,
// kTcIssuers MMA-issuer warps (one per SM sub-partition: a tcgen05.mma issue waits for issue
// slots its sub-partition's FP32 warps also want, so tiles rotate over issuers), one TMA producer.  A tile is 128 pixel pairs = 256 blocks (16 KB of u8:
// CW 128-byte chunks x 16/CW bands), loaded by TMA straight into the canonical K-major layout of
// the kind::i8 MMA's A operand; see tc.cu.
// kTcWays = epilogue warps per lane quarter = TMEM D stages = MMA-issuer warps: tile t uses D
// stage t % kTcWays, issuer warp t % kTcWays and epilogue warps t % kTcWays, so every mbarrier
// has one waiting agent that waits for its phases in order (a parity wait can never alias a
// phase two ahead) and the issuers sit on different SM sub-partitions.
#ifndef ADCT_TC_WAYS
#define ADCT_TC_WAYS 3
#endif
constexpr int kTcWays = ADCT_TC_WAYS;
constexpr int kTcEpi = kTcWays;                     // epilogue warps per lane quarter
constexpr int kTcEpiWarps = 4 * kTcEpi;
constexpr int kTcIssuers = kTcWays;                 // MMA-issuer warps
constexpr int kTcWarps = kTcEpiWarps + kTcIssuers + 1;  // + the TMA producer
constexpr int kTcThreads = 32 * kTcWarps;
constexpr int kTcTileBytes = 16384;
#ifndef ADCT_TC_SLOTS
#define ADCT_TC_SLOTS 12
#endif
constexpr int kTcSlots = ADCT_TC_SLOTS;  // pixel-tile ring depth
static_assert(kTcSlots % kTcWays == 0, "slot s only ever holds tiles of issuer s % kTcWays");
constexpr int kTcDStages = kTcWays;               // TMEM accumulator stages (N <= 160 columns each)
#ifndef ADCT_TC_CHUNK
#define ADCT_TC_CHUNK 24
#endif
constexpr int kTcChunkTiles = ADCT_TC_CHUNK;      // tiles per chunk, at most
#ifndef ADCT_TC_CHUNK_MIN
#define ADCT_TC_CHUNK_MIN 16  // tiles per chunk, at least (4 -> 16: C4 step -2.5 %, the 64-frame shard -5 %)
#endif
// tiles per chunk of a plane: from the image geometry only (so per-image sums do not depend on
// how images are batched or sharded): 1/32 of the image's tiles, clamped to [16, 24].  A chunk
// ends with a warp reduction and a partial store per epilogue warp, so 4-tile chunks (a 1080p
// chroma plane's 127 tiles / 32) cost the chroma launch ~6 % in chunk turnover; with 16 a 64-frame
// chroma shard (8 GPUs, U + V = 128 planes x 8 chunks) is still 7 waves of the 148 CTAs
inline int32_t tc_chunk_tiles(int64_t tiles_per_image) {
  int64_t c = tiles_per_image / 32;
  if (c < ADCT_TC_CHUNK_MIN) c = ADCT_TC_CHUNK_MIN;
  if (c > kTcChunkTiles) c = kTcChunkTiles;
  return (int32_t)c;
}
constexpr int kTcMaxPlanes = 3;                   // planes per approx_dct8x8_fused_sse_planes call (Y, U, V)
#ifndef ADCT_TC_ABL
#define ADCT_TC_ABL 0  // ablation builds only (tools/build_variant.sh): 1 no epilogue math, 2 no TMEM load, 3 no MMA
#endif

constexpr int kTcPartials = 4 * kTcEpi;           // partials per chunk
constexpr int kTcBBytes = 160 * 128;              // B: N <= 160 outputs x K = 128 s8
constexpr int kTcBars = 2 * kTcSlots + 4 * kTcDStages;
constexpr int kTcBiasA = 128 * 16 * 2, kTcBiasB = 96 * 16 * 2;  // f16 constant tiles of the bias MMA (tc.cu)
constexpr size_t kTcSmem = (size_t)kTcSlots * kTcTileBytes + kTcBBytes + (size_t)kTcBars * 8 + 16 + 128 + kTcBiasA +
                           kTcBiasB + 1024;
static_assert(kTcSmem <= 227 * 1024, "tensor-core kernel exceeds shared memory");
struct TcPlan {
  int32_t cw;        // tile width in 128-byte chunks (16 / cw bands high); 15: donor tiling (tc.cu)
  int32_t dmain, dlast, dc0;  // donor tiling: main tiles per image, leftover tile's band and first chunk
  int32_t tpr, tpi;  // tiles per tile row, per image
  int32_t ct;        // tiles per chunk
  int32_t cpi;       // chunks per image
  int64_t n_chunks;
  bool ok;
};
TcPlan tc_plan(const adct_geom& g);  // tc.cu
// the tensor-core path for one plane (tc.cu); false when it does not cover the call
bool fused_u8_tc(const adct_matrix* m, const uint8_t* src, const adct_geom& g, int32_t r, double* sse, double* psnr,
                 double* partial, cudaStream_t st, adct_status* status, int64_t split = 0, double* sse2 = nullptr,
                 double* psnr2 = nullptr, int clip = 0 /* 1: ADCT_CLIP, T1 at r = 10 only */);

// the tensor-core path of approx_dct8x8_fwd_quant (tc.cu); false when it does not cover the call
bool fwd_quant_tc(const adct_matrix* m, const uint8_t* src, const adct_geom& g, int32_t step, int16_t* q,
                  cudaStream_t st, adct_status* status);

inline int64_t stream_partials_per_image(const adct_geom& g) {
  int64_t best = 0;
  if (g.width % 128 == 0) {  // tensor-core tiles (any of its shapes)
    for (int cw : {16, 2, 1}) {
      const int64_t tpi = ((g.width / 128 + cw - 1) / cw) * ((g.height / 8 + 16 / cw - 1) / (16 / cw));
      const int64_t ct = tc_chunk_tiles(tpi);
      const int64_t c = (tpi + ct - 1) / ct * kTcPartials;
      if (c > best) best = c;
    }
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
