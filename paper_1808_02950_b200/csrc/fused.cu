// fused.cu — the performance paths: forward -> zonal retention -> inverse -> squared error
// per image with every block read once (§6.1), the host-buffer
// pipeline around it, and the config-3 forward + quantiser.
//
// Deterministic reductions: CTA (chunk c of image i) owns blocks [c*NT*BPT, (c+1)*NT*BPT)
// of image i in raster order; each thread's fp64 sum is reduced in a fixed shuffle/smem
// order into partial[i][c][slot]; a finalize kernel adds the chunks of an image in order.
// Results therefore do not depend on scheduling, and sharding images over GPUs gives the
// same per-image sums bit for bit.
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "adct_host.h"
#include "fused_common.cuh"
#include "packed.cuh"

namespace adct {

void launch_finalize(const double* partial, int32_t chunks, int64_t n_images, int32_t slots, const SlotMap& slot_of,
                     int32_t n_out, double npix, double peak, double* sse, double* psnr, cudaStream_t st);
bool launch_sweep_any(bool u8, bool specialized, int clip, cudaStream_t st, const void* src, const adct_geom& g,
                      const KGeom& kg, const DevMat& dm, const FastDiv& dbw, uint64_t rmask, int32_t rmin,
                      double* partial);
int64_t sweep_chunks(const adct_geom& g);
bool fwd_quant_tma(const adct_matrix* m, const uint8_t* src, const adct_geom& g, int32_t step, int16_t* q,
                   cudaStream_t st, adct_status* status);
bool fused_u8_stream(const adct_matrix* m, const uint8_t* src, const adct_geom& g, int32_t r, double* sse, double* psnr,
                     double* partial, cudaStream_t st, adct_status* status);
bool fused_u8_tc_planes(const adct_matrix* m, int n, const uint8_t* const* src, const adct_geom* g, int32_t r,
                        double* const* sse, double* const* psnr, double* const* partial, cudaStream_t st,
                        adct_status* status);
bool tc_hot_enabled();

namespace {

// ADCT_DISABLE_STREAM=1 selects the generic fused kernels instead of the TMA-streamed ones (tests)
const bool g_disable_stream = [] {
  const char* e = std::getenv("ADCT_DISABLE_STREAM");
  return e && e[0] == '1';
}();

constexpr int NT = kRedNT;
constexpr int BPT = kFusedBPT;

__host__ __device__ constexpr int popc64(uint64_t v) {
  int c = 0;
  for (int i = 0; i < 64; ++i) c += (int)((v >> i) & 1u);
  return c;
}

// ---- single r, compile-time retention pattern ------------------------------------------
// r <= 32: reconstruct from the kept coefficients, e = x - x_hat.
// r >  32: inverse of the dropped coefficients, e = H (W o Y o drop) H^T = x - x_hat
//          (exactly 0 at r = 64, reading A17).
template <typename SrcT, class MP, int R, int CLIP>
__device__ __forceinline__ float block_sse(const MP& m, const typename Src<SrcT>::Row (&rows)[8]) {
  constexpr uint64_t KEEP = keep_mask(R);
  constexpr bool RESID = popc64(KEEP) > 32;
  constexpr uint64_t NZ = RESID ? ~KEEP : KEEP;
  float x[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) Src<SrcT>::to_f(rows[i], x[i]);
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  if constexpr (NZ == 0) {
    return 0.0f;  // r = 64: nothing dropped, x_hat = x
  } else {
    float y[8][8];
    fwd2d(m, x, y);
    float z[8][8], xh[8][8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int l = 0; l < 8; ++l) z[k][l] = ((NZ >> (k * 8 + l)) & 1ull) ? y[k][l] * m.wy(k, l) : 0.0f;
    inv2d<MP, NZ>(m, z, xh);
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float d;
        if constexpr (RESID) d = (CLIP == ADCT_CLIP_NONE) ? xh[i][j] : x[i][j] - clipv<CLIP>(x[i][j] - xh[i][j], Src<SrcT>::lo, Src<SrcT>::hi);
        else d = x[i][j] - clipv<CLIP>(xh[i][j], Src<SrcT>::lo, Src<SrcT>::hi);
        acc[j & 3] = fmaf(d, d, acc[j & 3]);
      }
  }
  return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

template <typename SrcT, class MP, int R, int CLIP>
__global__ void __launch_bounds__(NT) fused_single_kernel(const SrcT* __restrict__ src, KGeom g, DevMat dm,
                                                          FastDiv dbw, int32_t chunks,
                                                          double* __restrict__ partial) {
  __shared__ double red[NT / 32];
  const MP m(dm);
  const SrcT* base = src + (int64_t)blockIdx.y * g.image_stride;
  const uint32_t q0 = blockIdx.x * (NT * BPT) + threadIdx.x;
  using Row = typename Src<SrcT>::Row;
  Row a[8], b[8];
  double acc = 0.0;
  if (q0 < g.nbi) load_rows(base, g, dbw, q0, a);
#pragma unroll 1
  for (int mb = 0; mb < BPT; mb += 2) {
    const uint32_t qa = q0 + mb * NT, qb = qa + NT, qc = qb + NT;
    if (qb < g.nbi) load_rows(base, g, dbw, qb, b);
    if (qa < g.nbi) acc += (double)block_sse<SrcT, MP, R, CLIP>(m, a);
    if (mb + 2 < BPT && qc < g.nbi) load_rows(base, g, dbw, qc, a);
    if (qb < g.nbi) acc += (double)block_sse<SrcT, MP, R, CLIP>(m, b);
  }
  const double tot = block_sum<NT>(acc, red);
  if (threadIdx.x == 0) partial[(int64_t)blockIdx.y * chunks + blockIdx.x] = tot;
}

// ---- single r, runtime retention pattern (any matrix, any r) ------------------------------------
// The retentions that have no compiled kernel used to take the r-list sweep (63 - r rank-one
// updates per block: 128 4K frames at r = 21 in 3.7 ms).  One pass instead: the packed round trip
// of packed.cuh with the weight table w = (inverse weight) x (zig-zag keep bit) as a kernel
// parameter -- kept form for r <= 32 (e = x - x_hat), dropped form for r > 32 (the round trip of the
// dropped coefficients is x - x_hat itself: exactly 0 at r = 64, reading A17).
#ifndef ADCT_RT_RECONVERT
#define ADCT_RT_RECONVERT 1
#endif
#ifndef ADCT_RT_MINB
#define ADCT_RT_MINB 3  // 168 registers, 12 warps per SM: 0.72-0.89 ms vs 0.84-0.97 (2) and 0.70-0.94 (4, spills) on 128 4K frames
#endif
struct WkS {
  float w[64];
};
template <typename SrcT, class MP, int CLIP>
__device__ __forceinline__ float block_sse_rt(const MP& m, const typename Src<SrcT>::Row (&rows)[8], const float* w,
                                              bool resid) {
  float x[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) Src<SrcT>::to_f(rows[i], x[i]);
  float2 x2[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) x2[i][c] = pk(x[i][2 * c], x[i][2 * c + 1]);
  roundtrip2d_p(m, x2, w);
  float2 acc[2] = {pk(0.0f, 0.0f), pk(0.0f, 0.0f)};
#pragma unroll
  for (int i = 0; i < 8; ++i) {
#if ADCT_RT_RECONVERT  // the samples again from the raw row instead of 64 registers held across the round trip
    asm volatile("" : "+r"(*reinterpret_cast<uint32_t*>(const_cast<typename Src<SrcT>::Row*>(&rows[i]))));
    Src<SrcT>::to_f(rows[i], x[i]);
#endif
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float2 xo = pk(x[i][2 * c], x[i][2 * c + 1]), v = x2[i][c];
      float2 d;
      if (CLIP == ADCT_CLIP_NONE) {
        d = resid ? v : psub(xo, v);
      } else {
        const float2 xh = resid ? psub(xo, v) : v;
        d = pk(xo.x - clipv<CLIP>(xh.x, Src<SrcT>::lo, Src<SrcT>::hi),
               xo.y - clipv<CLIP>(xh.y, Src<SrcT>::lo, Src<SrcT>::hi));
      }
      acc[c & 1] = __ffma2_rn(d, d, acc[c & 1]);
    }
  }
  return (acc[0].x + acc[0].y) + (acc[1].x + acc[1].y);
}

template <typename SrcT, class MP, int CLIP>
__global__ void __launch_bounds__(NT, ADCT_RT_MINB) fused_single_rt_kernel(const SrcT* __restrict__ src, KGeom g, DevMat dm, WkS wk,
                                                             int resid, FastDiv dbw, int32_t chunks,
                                                             double* __restrict__ partial) {
  __shared__ double red[NT / 32];
  const MP m(dm);
  const SrcT* base = src + (int64_t)blockIdx.y * g.image_stride;
  const uint32_t q0 = blockIdx.x * (NT * BPT) + threadIdx.x;
  using Row = typename Src<SrcT>::Row;
  Row a[8], b[8];
  double acc = 0.0;
  if (q0 < g.nbi) load_rows(base, g, dbw, q0, a);
#pragma unroll 1
  for (int mb = 0; mb < BPT; mb += 2) {
    const uint32_t qa = q0 + mb * NT, qb = qa + NT, qc = qb + NT;
    if (qb < g.nbi) load_rows(base, g, dbw, qb, b);
    if (qa < g.nbi) acc += (double)block_sse_rt<SrcT, MP, CLIP>(m, a, wk.w, resid != 0);
    if (mb + 2 < BPT && qc < g.nbi) load_rows(base, g, dbw, qc, a);
    if (qb < g.nbi) acc += (double)block_sse_rt<SrcT, MP, CLIP>(m, b, wk.w, resid != 0);
  }
  const double tot = block_sum<NT>(acc, red);
  if (threadIdx.x == 0) partial[(int64_t)blockIdx.y * chunks + blockIdx.x] = tot;
}

// ---- config 3: forward with S folded into a uniform quantiser ------------------------------
// q = sign(Y) floor(|Y| / (step sqrt(n_k n_l)) + 1/2) (reading A10).  fp32 estimate; when the
// estimate is within 1e-4 of a rounding boundary the exact integer rule
// (2m-1)^2 step^2 n_k n_l <= 4 Y^2 < (2m+1)^2 step^2 n_k n_l decides (in fp64, exact below 2^53).
template <class MP>
__global__ void __launch_bounds__(256) fwd_quant_kernel(const uint8_t* __restrict__ src, KGeom g, DevMat dm,
                                                        FastDiv dnbi, FastDiv dbw, uint32_t nblocks,
                                                        int16_t* __restrict__ out) {
  const MP m(dm);
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nblocks; b += gridDim.x * blockDim.x) {
    const uint32_t img = fdiv(b, dnbi);
    const uint32_t q = b - img * g.nbi;
    const uint32_t by = fdiv(q, dbw);
    const uint32_t bx = q - by * g.bw;
    const uint8_t* p = src + (int64_t)img * g.image_stride + (int64_t)by * 8 * g.row_stride + (int64_t)bx * 8;
    float x[8][8], y[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i) u8row_to_f(ldg_u8row(p + (int64_t)i * g.row_stride), x[i]);
    fwd2d(m, x, y);
    int16_t* o = out + (int64_t)b * 64;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t w[4];
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        const float a = fabsf(y[k][l]);
        const float t = fmaf(a, dm.q_inv[k * 8 + l], 0.5f);
        float mq = floorf(t);
        const float fr = t - mq;
        if (fr < 1e-4f || fr > 1.0f - 1e-4f) {  // near a boundary: exact decision
          const double a2 = 4.0 * (double)a * (double)a;
          const double pp = dm.q_p[k * 8 + l];
          double mm = (double)mq;
          if (mm >= 1.0 && (2.0 * mm - 1.0) * (2.0 * mm - 1.0) * pp > a2) mm -= 1.0;
          else if ((2.0 * mm + 1.0) * (2.0 * mm + 1.0) * pp <= a2) mm += 1.0;
          mq = (float)mm;
        }
        const int v = y[k][l] < 0.0f ? -(int)mq : (int)mq;
        const uint32_t u = (uint32_t)(uint16_t)(int16_t)v;
        if (l & 1) w[l >> 1] |= u << 16; else w[l >> 1] = u;
      }
      *reinterpret_cast<uint4*>(o + k * 8) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

int sms() { return device_sms(); }

// single-r kernels compiled in: (matrix, r) pairs of the benchmark configurations
template <typename SrcT, class MP, int CLIP>
bool launch_single(int r, dim3 grid, cudaStream_t st, const SrcT* src, const KGeom& kg, const DevMat& dm,
                   const FastDiv& dbw, int32_t chunks, double* partial) {
  switch (r) {
    case 10:
      fused_single_kernel<SrcT, MP, 10, CLIP><<<grid, NT, 0, st>>>(src, kg, dm, dbw, chunks, partial);
      return true;
    case 64:
      fused_single_kernel<SrcT, MP, 64, CLIP><<<grid, NT, 0, st>>>(src, kg, dm, dbw, chunks, partial);
      return true;
    default:
      return false;
  }
}


template <typename SrcT, class MP>
adct_status fused_dispatch(const adct_matrix* m, const void* src, const adct_geom& g, const int32_t* r_list,
                           int32_t n_r, adct_clip clip, double* sse, double* psnr, double* partial, cudaStream_t st) {
  const KGeom kg = make_kgeom(g);
  const FastDiv dbw = make_fastdiv(kg.bw);
  int32_t chunks = (int32_t)fused_chunks(g);
  const SrcT* s = (const SrcT*)src;
  SlotMap sm{};
  bool single = false;
  if (n_r == 1) {
    if constexpr (std::is_same<SrcT, uint8_t>::value) {
      if (clip == ADCT_CLIP_NONE && m->is_int && !g_disable_stream) {
        adct_status stt = ADCT_OK;
        if (fused_u8_stream(m, (const uint8_t*)src, g, r_list[0], sse, psnr, partial, st, &stt)) return stt;
      }
    }
    if constexpr (std::is_same<SrcT, uint8_t>::value) {
      // the SPEC's metric policy (clip to [0, 255], no rounding) on the tensor-core kernel: T1, r = 10
      if (clip == ADCT_CLIP && m->is_int && m->specialized && !g_disable_stream && tc_hot_enabled()) {
        adct_status stt = ADCT_OK;
        if (fused_u8_tc(m, (const uint8_t*)src, g, r_list[0], sse, psnr, partial, st, &stt, 0, nullptr, nullptr, 1))
          return stt;
      }
    }
    dim3 grid((unsigned)chunks, (unsigned)g.n_images);
    if (!single && clip == ADCT_CLIP_NONE)
      single = launch_single<SrcT, MP, ADCT_CLIP_NONE>(r_list[0], grid, st, s, kg, m->dev, dbw, chunks, partial);
    else if (!single && clip == ADCT_CLIP)
      single = launch_single<SrcT, MP, ADCT_CLIP>(r_list[0], grid, st, s, kg, m->dev, dbw, chunks, partial);
    static const bool no_rt = std::getenv("ADCT_NO_SINGLE_RT") != nullptr;  // A/B hook: the r-list sweep instead
    if (!single && !no_rt) {  // any other r: one pass with a runtime weight table
      const uint64_t keep = keep_mask(r_list[0]);
      const bool resid = popc64(keep) > 32;
      const uint64_t nz = resid ? ~keep : keep;
      WkS wk;
      for (int p = 0; p < 64; ++p) wk.w[p] = ((nz >> p) & 1ull) ? m->dev.wy[p] : 0.0f;
      if (clip == ADCT_CLIP_NONE)
        fused_single_rt_kernel<SrcT, MP, ADCT_CLIP_NONE><<<grid, NT, 0, st>>>(s, kg, m->dev, wk, (int)resid, dbw,
                                                                              chunks, partial);
      else if (clip == ADCT_CLIP)
        fused_single_rt_kernel<SrcT, MP, ADCT_CLIP><<<grid, NT, 0, st>>>(s, kg, m->dev, wk, (int)resid, dbw, chunks,
                                                                         partial);
      else
        fused_single_rt_kernel<SrcT, MP, ADCT_CLIP_ROUND><<<grid, NT, 0, st>>>(s, kg, m->dev, wk, (int)resid, dbw,
                                                                               chunks, partial);
      single = true;
    }
  }
  dim3 grid((unsigned)chunks, (unsigned)g.n_images);
  int32_t slots = 1;
  if (!single) {
    uint64_t rmask = 0;
    int32_t rmin = 64;
    for (int i = 0; i < n_r; ++i) {
      if (r_list[i] < 64) rmask |= 1ull << r_list[i];  // r = 64 is slot 63, always 0
      if (r_list[i] < rmin) rmin = r_list[i];
      sm.s[i] = r_list[i] - 1;
    }
    if (!launch_sweep_any(std::is_same<SrcT, uint8_t>::value, MP::kConst, (int)clip, st, s, g, kg, m->dev, dbw,
                          rmask, rmin, partial))
      return ADCT_E_CUDA;
    chunks = (int32_t)sweep_chunks(g);
    slots = 64;
  }
  count_launch();
  if (adct_status e = launch_status()) return e;
  launch_finalize(partial, chunks, g.n_images, slots, sm, n_r, (double)g.height * g.width, 255.0, sse, psnr, st);
  return launch_status();
}

adct_status fused_check(const adct_matrix* m, const void* src, adct_dtype src_t, const adct_geom& g,
                        const int32_t* r_list, int32_t n_r, adct_clip clip) {
  if (!m || !src || !r_list) return ADCT_E_INVALID_ARGUMENT;
  if (adct_status s = check_geom(g)) return s;
  if (src_t != ADCT_U8 && src_t != ADCT_I16) return ADCT_E_INVALID_ARGUMENT;
  if (n_r < 1 || n_r > 64) return ADCT_E_INVALID_ARGUMENT;
  for (int i = 0; i < n_r; ++i)
    if (r_list[i] < 1 || r_list[i] > 64) return ADCT_E_INVALID_ARGUMENT;
  if (clip != ADCT_CLIP_NONE && clip != ADCT_CLIP && clip != ADCT_CLIP_ROUND) return ADCT_E_INVALID_ARGUMENT;
  if (!aligned(src, src_t == ADCT_U8 ? 8 : 16)) return ADCT_E_ALIGNMENT;
  return ADCT_OK;
}

adct_status fused_run(const adct_matrix* m, const void* src, adct_dtype src_t, const adct_geom& g,
                      const int32_t* r_list, int32_t n_r, adct_clip clip, double* sse, double* psnr, double* partial,
                      cudaStream_t st) {
  if (g.n_images == 0) return ADCT_OK;
  if (src_t == ADCT_U8) {
    if (m->specialized) return fused_dispatch<uint8_t, T1Mat>(m, src, g, r_list, n_r, clip, sse, psnr, partial, st);
    return fused_dispatch<uint8_t, RtMat>(m, src, g, r_list, n_r, clip, sse, psnr, partial, st);
  }
  if (m->specialized) return fused_dispatch<int16_t, T1Mat>(m, src, g, r_list, n_r, clip, sse, psnr, partial, st);
  return fused_dispatch<int16_t, RtMat>(m, src, g, r_list, n_r, clip, sse, psnr, partial, st);
}

// copy stream of the host-buffer pipeline (one per device, created on first use there)
cudaStream_t copy_stream() {
  static std::mutex mu;
  static cudaStream_t s[kMaxDevices] = {};
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!s[dev] && cudaStreamCreateWithFlags(&s[dev], cudaStreamNonBlocking) != cudaSuccess) s[dev] = nullptr;
  return s[dev];
}

}  // namespace
}  // namespace adct

using namespace adct;

extern "C" {

adct_status approx_dct8x8_fused_sse(const adct_matrix* m, const void* src, adct_dtype src_t, adct_geom g,
                                    const int32_t* r_list, int32_t n_r, adct_clip clip, double* sse, double* psnr,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  if (adct_status s = fused_check(m, src, src_t, g, r_list, n_r, clip)) return s;
  if (!sse) return ADCT_E_INVALID_ARGUMENT;
  if (!workspace || workspace_bytes < adct_workspace_bytes(g, n_r) || !aligned(workspace, 8)) return ADCT_E_WORKSPACE;
  return fused_run(m, src, src_t, g, r_list, n_r, clip, sse, psnr, (double*)workspace, (cudaStream_t)stream);
}

namespace {
// Layout of the host-buffer pipeline's device workspace: two staging buffers of chunk_images
// dense planes (the host stack is dense: image_stride = H * row_stride, whatever g says for a
// single image), two partial buffers, then the SSE and PSNR tables [n_images][n_r].
struct HostWs {
  size_t stage, part, out;
};
HostWs host_ws(const adct_geom& g, int32_t n_r, int64_t chunk_images, adct_dtype src_t) {
  if (chunk_images < 1) chunk_images = 1;
  adct_geom gc = g;
  gc.n_images = chunk_images;
  gc.image_stride = (int64_t)g.height * g.row_stride;
  const size_t esz = src_t == ADCT_I16 ? 2 : 1;
  HostWs w;
  w.stage = ((size_t)chunk_images * (size_t)gc.image_stride * esz + 255) / 256 * 256;
  w.part = (adct_workspace_bytes(gc, n_r) + 255) / 256 * 256;
  w.out = ((size_t)(g.n_images > 0 ? g.n_images : 0) * (size_t)(n_r > 0 ? n_r : 1) * sizeof(double) + 255) / 256 * 256;
  return w;
}
}  // namespace

size_t adct_host_workspace_bytes(adct_geom g, int32_t n_r, int64_t chunk_images, adct_dtype src_t) {
  if (g.height <= 0 || g.row_stride <= 0) return 0;
  const HostWs w = host_ws(g, n_r, chunk_images, src_t);
  return 2 * w.stage + 2 * w.part + 2 * w.out;
}

adct_status approx_dct8x8_fused_sse_host(const adct_matrix* m, const void* src_host, adct_dtype src_t, adct_geom g,
                                         const int32_t* r_list, int32_t n_r, adct_clip clip, double* sse_host,
                                         double* psnr_host, int64_t chunk_images, void* workspace,
                                         size_t workspace_bytes, void* stream) {
  if (adct_status s = fused_check(m, src_host, src_t, g, r_list, n_r, clip)) return s;
  if (!sse_host || chunk_images < 1) return ADCT_E_INVALID_ARGUMENT;
  if (g.n_images > 1 && g.image_stride != (int64_t)g.height * g.row_stride) return ADCT_E_INVALID_ARGUMENT;
  if (!workspace || workspace_bytes < adct_host_workspace_bytes(g, n_r, chunk_images, src_t)) return ADCT_E_WORKSPACE;
  if (g.n_images == 0) return ADCT_OK;
  g.image_stride = (int64_t)g.height * g.row_stride;  // dense host stack (a lone image's stride is unused)
  cudaStream_t cs = (cudaStream_t)stream;
  cudaStream_t xs = copy_stream();
  if (!xs) return ADCT_E_CUDA;
  const HostWs w = host_ws(g, n_r, chunk_images, src_t);
  const size_t esz = src_t == ADCT_I16 ? 2 : 1;
  char* ws = (char*)workspace;
  char* stg[2] = {ws, ws + w.stage};
  double* prt[2] = {(double*)(ws + 2 * w.stage), (double*)(ws + 2 * w.stage + w.part)};
  double* dsse = (double*)(ws + 2 * w.stage + 2 * w.part);
  double* dpsnr = psnr_host ? (double*)(ws + 2 * w.stage + 2 * w.part + w.out) : nullptr;
  cudaEvent_t copied[2], freed[2];
  for (int i = 0; i < 2; ++i) {
    if (cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming) != cudaSuccess) return ADCT_E_CUDA;
    if (cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming) != cudaSuccess) return ADCT_E_CUDA;
  }
  adct_status st = ADCT_OK;
  // the copy stream must not overwrite a staging buffer before earlier compute finished
  cudaEventRecord(freed[0], cs);
  cudaEventRecord(freed[1], cs);
  int64_t c = 0;
  for (int64_t i0 = 0; i0 < g.n_images && st == ADCT_OK; i0 += chunk_images, ++c) {
    const int b = (int)(c & 1);
    const int64_t n = (g.n_images - i0) < chunk_images ? (g.n_images - i0) : chunk_images;
    const size_t bytes = (size_t)(n * g.image_stride) * esz;
    cudaStreamWaitEvent(xs, freed[b], 0);
    if (cudaMemcpyAsync(stg[b], (const char*)src_host + (size_t)i0 * g.image_stride * esz, bytes,
                        cudaMemcpyHostToDevice, xs) != cudaSuccess) { st = ADCT_E_CUDA; break; }
    cudaEventRecord(copied[b], xs);
    cudaStreamWaitEvent(cs, copied[b], 0);
    adct_geom gi = g;
    gi.n_images = n;
    st = fused_run(m, stg[b], src_t, gi, r_list, n_r, clip, dsse + i0 * n_r, dpsnr ? dpsnr + i0 * n_r : nullptr,
                   prt[b], cs);
    cudaEventRecord(freed[b], cs);
  }
  const size_t tab = (size_t)g.n_images * n_r * sizeof(double);
  if (st == ADCT_OK && cudaMemcpyAsync(sse_host, dsse, tab, cudaMemcpyDeviceToHost, cs) != cudaSuccess)
    st = ADCT_E_CUDA;
  if (st == ADCT_OK && dpsnr && cudaMemcpyAsync(psnr_host, dpsnr, tab, cudaMemcpyDeviceToHost, cs) != cudaSuccess)
    st = ADCT_E_CUDA;
  if (cudaStreamSynchronize(cs) != cudaSuccess) st = ADCT_E_CUDA;
  for (int i = 0; i < 2; ++i) {
    cudaEventDestroy(copied[i]);
    cudaEventDestroy(freed[i]);
  }
  return st;
}

size_t adct_planes_workspace_bytes(int32_t n_planes, const adct_geom* g) {
  if (n_planes < 1 || n_planes > ADCT_MAX_PLANES || !g) return 0;
  size_t tot = 0;
  for (int i = 0; i < n_planes; ++i) tot += (adct_workspace_bytes(g[i], 1) + 255) / 256 * 256;
  return tot;
}

adct_status approx_dct8x8_fused_sse_planes(const adct_matrix* m, int32_t n_planes, const void* const* src,
                                           adct_dtype src_t, const adct_geom* g, int32_t r, adct_clip clip,
                                           double* const* sse, double* const* psnr, void* workspace,
                                           size_t workspace_bytes, void* stream) {
  if (!m || !src || !g || !sse || n_planes < 1 || n_planes > ADCT_MAX_PLANES) return ADCT_E_INVALID_ARGUMENT;
  for (int i = 0; i < n_planes; ++i) {
    if (g[i].n_images == 0) {  // an empty plane: geometry checked, its buffers may be NULL
      if (adct_status s = check_geom(g[i])) return s;
      continue;
    }
    if (adct_status s = fused_check(m, src[i], src_t, g[i], &r, 1, clip)) return s;
    if (!sse[i]) return ADCT_E_INVALID_ARGUMENT;
  }
  if (!workspace || workspace_bytes < adct_planes_workspace_bytes(n_planes, g) || !aligned(workspace, 8))
    return ADCT_E_WORKSPACE;
  double* part[ADCT_MAX_PLANES];
  size_t off = 0;
  for (int i = 0; i < n_planes; ++i) {
    part[i] = (double*)((char*)workspace + off);
    off += (adct_workspace_bytes(g[i], 1) + 255) / 256 * 256;
  }
  cudaStream_t st = (cudaStream_t)stream;
  // the tensor-core kernel for every non-empty plane when all of them qualify
  if (src_t == ADCT_U8 && clip == ADCT_CLIP_NONE && m->is_int && !g_disable_stream && tc_hot_enabled() &&
      n_planes <= kTcMaxPlanes) {
    const uint8_t* s8[kTcMaxPlanes];
    adct_geom gg[kTcMaxPlanes];
    double *ss[kTcMaxPlanes], *pp[kTcMaxPlanes], *pt[kTcMaxPlanes];
    int n = 0;
    for (int i = 0; i < n_planes; ++i) {
      if (g[i].n_images == 0) continue;
      s8[n] = (const uint8_t*)src[i];
      gg[n] = g[i];
      ss[n] = sse[i];
      pp[n] = psnr ? psnr[i] : nullptr;
      pt[n] = part[i];
      ++n;
    }
    if (n == 0) return ADCT_OK;
    adct_status stt = ADCT_OK;
    if (fused_u8_tc_planes(m, n, s8, gg, r, ss, pp, pt, st, &stt)) return stt;
  }
  for (int i = 0; i < n_planes; ++i)  // the per-plane composition
    if (g[i].n_images > 0)
      if (adct_status s = fused_run(m, src[i], src_t, g[i], &r, 1, clip, sse[i], psnr ? psnr[i] : nullptr, part[i], st))
      return s;
  return ADCT_OK;
}

adct_status approx_dct8x8_fwd_quant(const adct_matrix* m, const uint8_t* src, adct_geom g, int32_t step, int16_t* q,
                                    void* stream) {
  if (!m || !src || !q) return ADCT_E_INVALID_ARGUMENT;
  if (adct_status s = check_geom(g)) return s;
  if (!m->is_int || step < 1) return ADCT_E_INVALID_ARGUMENT;
  if (!aligned(src, 8) || !aligned(q, 16)) return ADCT_E_ALIGNMENT;
  const KGeom kg = make_kgeom(g);
  const uint32_t nb = (uint32_t)(g.n_images * kg.nbi);
  if (nb == 0) return ADCT_OK;
  if (!g_disable_stream) {  // TMA-streamed kernel (u8 tiles in, swizzled int16 tiles out)
    adct_status qs = ADCT_OK;
    if (fwd_quant_tc(m, src, g, step, q, (cudaStream_t)stream, &qs)) return qs;  // tensor-core forward
    if (fwd_quant_tma(m, src, g, step, q, (cudaStream_t)stream, &qs)) return qs;
  }
  DevMat dm = m->dev;
  for (int k = 0; k < 8; ++k)
    for (int l = 0; l < 8; ++l) {
      const double p = (double)step * step * (double)m->n[k] * (double)m->n[l];
      dm.q_p[k * 8 + l] = p;
      dm.q_inv[k * 8 + l] = (float)(1.0 / std::sqrt(p));
      const double c = std::sqrt(p);
      dm.q_c[k * 8 + l] = (std::floor(c) == c) ? (int32_t)c : 0;
    }
  const FastDiv dnbi = make_fastdiv(kg.nbi), dbw = make_fastdiv(kg.bw);
  const int64_t need = ((int64_t)nb + 255) / 256;
  const int64_t cap = (int64_t)sms() * 8;
  const unsigned grid = (unsigned)(need < cap ? need : cap);
  cudaStream_t st = (cudaStream_t)stream;
  if (m->specialized)
    fwd_quant_kernel<T1Mat><<<grid, 256, 0, st>>>(src, kg, dm, dnbi, dbw, nb, q);
  else
    fwd_quant_kernel<RtMat><<<grid, 256, 0, st>>>(src, kg, dm, dnbi, dbw, nb, q);
  count_launch();
  return launch_status();
}

}  // extern "C"
static_assert(ADCT_MAX_PLANES == adct::kTcMaxPlanes, "plane count of the C-ABI and the kernel");
