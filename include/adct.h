/*
 * adct.h — C-ABI of the B200 hot path of arXiv 1808.02950 (Oliveira, Cintra, Bayer,
 * da Silveira, Madanayake, Leite: "Low-complexity 8-point DCT approximation based on
 * angle similarity for image and video coding").
 *
 * The library implements §6.1 "Still Image Compression" on
 * batches of images: every 8x8 sub-block A is transformed to B = C_hat A C_hat^T
 * with C_hat = S T (Eq. 1), the first r coefficients in
 * zig-zag order are retained, the block is inverted with
 * A = C_hat^T B' C_hat and the reconstruction is scored by MSE/PSNR
 * (P:L2258-2265).  The matrix is a parameter (a descriptor), so the paper's T1
 * (P:L1116-1130), the exact DCT C and the comparison approximations of
 * Table 2 all run through the same calls.
 *
 * Conventions (apply to every call):
 *  - Device buffers are owned by the caller (e.g. torch tensors' data_ptr()).  No call
 *    allocates device memory; scratch comes from a caller workspace sized by
 *    adct_workspace_bytes().  Matrix descriptors are owned by the library
 *    (create/destroy) and are immutable and thread-safe once created.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All
 *    device calls are asynchronous on that stream.
 *  - Argument, shape and alignment errors are returned synchronously before any launch;
 *    a launch failure returns ADCT_E_CUDA; execution faults surface at the caller's
 *    synchronisation.  No exception crosses the ABI.
 *  - Images are planes of samples, row-major: sample (img, y, x) lives at element
 *    img*image_stride + y*row_stride + x.  height and width must be multiples of 8
 *    (every workload of the paper and BASELINE.json is); edge padding is the caller's.
 *  - Coefficients are block-major: block (img, by, bx) occupies 64 consecutive elements
 *    at ((img*H/8 + by)*W/8 + bx)*64, raster index k*8+l inside the block, k = vertical
 *    frequency (row of B), l = horizontal frequency.
 *  - Zig-zag order is the JPEG order (reading A5 in DESIGN.md): raster indices
 *    0,1,8,16,9,2,3,10,17,24,...
 */
#ifndef ADCT_H
#define ADCT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ADCT_OK = 0,
  ADCT_E_INVALID_ARGUMENT = 1,  /* null pointer, r outside 1..64, H/W not multiples of 8, bad dtype */
  ADCT_E_UNSUPPORTED_MATRIX = 2, /* matrix lacks the even/odd symmetry T J = diag((-1)^k) T */
  ADCT_E_SINGULAR = 3,          /* T T^T (or C_hat) is singular */
  ADCT_E_OVERFLOW = 4,          /* requested coefficient dtype cannot hold the worst-case |Y|,
                                   or an integer output was requested from a real matrix */
  ADCT_E_ALIGNMENT = 5,         /* a buffer/stride violates the vector-load alignment stated below */
  ADCT_E_CUDA = 6,              /* a CUDA launch or runtime call failed */
  ADCT_E_WORKSPACE = 7          /* workspace missing or smaller than adct_workspace_bytes() */
} adct_status;

typedef enum { ADCT_U8 = 0, ADCT_I16 = 1, ADCT_I32 = 2, ADCT_F32 = 3 } adct_dtype;

/* Reconstruction policy before the error is measured (reading A6 in DESIGN.md).
 * NONE: real-valued reconstruction, no clip (the default; the path stays linear).
 * CLIP: clip to the sample range ([0,255] for u8 sources, [-32768,32767] for int16),
 *       no rounding.
 * ROUND: clip, then round half to even (integer reconstruction). */
typedef enum { ADCT_CLIP_NONE = 0, ADCT_CLIP = 1, ADCT_CLIP_ROUND = 2 } adct_clip;

typedef struct adct_matrix adct_matrix; /* opaque */

typedef struct {
  int64_t n_images;     /* number of planes (images / frames) */
  int32_t height;       /* H, multiple of 8 */
  int32_t width;        /* W, multiple of 8 */
  int64_t image_stride; /* elements between consecutive planes (>= H*row_stride) */
  int64_t row_stride;   /* elements between consecutive rows (>= W, multiple of 8) */
} adct_geom;

/* --- matrix descriptors -------------------------------------------------------------- */

/* Integer low-complexity matrix T (row-major t[k*8+i]).  S = diag(1/||t_k||) (Eq. 2,
 * P:L363-367, exact for row-orthogonal T; reading A2 for SDCT / BAS-2008b).  Matrices with
 * fractional entries are passed pre-multiplied (LO as 2*T_LO, reading A11): S absorbs it.
 * The inverse uses C_hat^T when T T^T is diagonal, C_hat^{-1} otherwise
 * (reading A4).  Errors: INVALID_ARGUMENT (null), UNSUPPORTED_MATRIX (no even/odd
 * symmetry or a zero row), SINGULAR, OVERFLOW (|Y| could exceed 2^24 for int16 input). */
adct_status adct_matrix_create_int(const int32_t t[64], adct_matrix** out);

/* Real matrix C_hat (row-major, fp64), e.g. the orthonormal exact DCT (reading A1).
 * Used as is for the forward; inverse by C_hat^T if orthonormal to 1e-9, else C_hat^{-1}. */
adct_status adct_matrix_create_real(const double c[64], adct_matrix** out);

/* Query a descriptor.  Any output pointer may be NULL.
 * s[8]: row scaling; g[64]: synthesis matrix G with A = G B' G^T (row-major);
 * row_orthogonal: 1 if the inverse is the transpose; is_integer: 1 for create_int;
 * max_abs_y_u8 / max_abs_y_i16: exact worst-case |Y_kl| over u8 / int16 blocks (integer
 * matrices; 0 for real ones).  `specialized` = 1 when a compile-time network for this
 * exact matrix is built into the library (currently the paper's T1). */
adct_status adct_matrix_info(const adct_matrix* m, double s[8], double g[64], int32_t* row_orthogonal,
                             int32_t* is_integer, int64_t* max_abs_y_u8, int64_t* max_abs_y_i16,
                             int32_t* specialized);

void adct_matrix_destroy(adct_matrix* m);

/* C_hat = S T (integer matrices) or the real matrix itself, row-major fp64 (host). */
adct_status adct_matrix_chat(const adct_matrix* m, double chat[64]);

/* The zig-zag order the device path uses: order[z] = raster index (k*8+l) of the z-th
 * coefficient.  Host-only. */
adct_status adct_zigzag_order(int32_t order[64]);

/* --- the four calls of the method ------------------------------------------------------ */

/* Forward 2-D transform of every 8x8 block.
 * src: device, samples of dtype src_t (ADCT_U8 or ADCT_I16), geometry g.
 * coef: device, block-major, n_images*H*W elements of coef_t:
 *   ADCT_I32 / ADCT_I16: Y = T X T^T exactly (integer matrices only; I16 requires the
 *                        worst-case |Y| to fit, else ADCT_E_OVERFLOW)
 *   ADCT_F32:           B = S Y S = C_hat X C_hat^T (any matrix)
 * Alignment: src 8-byte aligned (u8) / 16-byte (int16), row_stride and image_stride
 * multiples of 8; coef 16-byte aligned. */
adct_status approx_dct8x8_fwd(const adct_matrix* m, const void* src, adct_dtype src_t, adct_geom g, void* coef,
                              adct_dtype coef_t, void* stream);

/* Zonal retention in place: zero every coefficient whose zig-zag position
 * is >= r, for n_blocks consecutive blocks.  r in 1..64, else
 * ADCT_E_INVALID_ARGUMENT.  coef_t: ADCT_I32, ADCT_I16 or ADCT_F32; 16-byte aligned. */
adct_status zonal_retain(void* coef, adct_dtype coef_t, int64_t n_blocks, int32_t r, void* stream);

/* Inverse 2-D transform of block-major coefficients into an image.
 * coef_t ADCT_I32/ADCT_I16: unscaled Y' (integer matrices only), the call applies S both
 * sides; ADCT_F32: B'.  recon: device image with geometry g, dtype recon_t:
 *   ADCT_F32 (clip policy applied as given), ADCT_U8 (requires ADCT_CLIP_ROUND: round half
 *   even, clip [0,255]), ADCT_I16 (requires ADCT_CLIP_ROUND: round half even, saturate). */
adct_status approx_dct8x8_inv(const adct_matrix* m, const void* coef, adct_dtype coef_t, adct_geom g, void* recon,
                              adct_dtype recon_t, adct_clip clip, void* stream);

/* Per-image squared error and PSNR (reading A7):
 * sse[i] = sum (orig - clip(recon))^2 over image i, psnr[i] = 10 log10(peak^2 / (sse/(H W))),
 * +inf when sse == 0.  orig: ADCT_U8/ADCT_I16, recon: ADCT_F32/ADCT_U8/ADCT_I16, both
 * with geometry g.  sse / psnr: device fp64 [n_images] (psnr may be NULL).  The sum is
 * deterministic (fixed two-level order).  workspace: device, >= adct_workspace_bytes(g, 1). */
adct_status psnr_reduce(const void* orig, adct_dtype orig_t, const void* recon, adct_dtype recon_t, adct_geom g,
                        double peak, adct_clip clip, double* sse, double* psnr, void* workspace,
                        size_t workspace_bytes, void* stream);

/* 16- and 32-point transforms of §6.2: the Jridi-Alfalou-Meher scaling of
 * T1 (Eq. 7; printed T(16), T(32) at P:L2669-2739, D(N) = diag(T T^T) at P:L2742-2770), as
 * the round trip forward -> retention of the first r coefficients of the N x N zig-zag walk
 * (reading A20) -> inverse C_hat^T B' C_hat, one pass, written as a reconstruction.
 * n: 16 or 32.  src: device U8/I16 images with geometry g, H and W multiples of n, 16-byte
 * aligned base and strides; recon: same geometry, dtype/clip policy as approx_dct8x8_roundtrip.
 * r in 1..n^2.  Every intermediate of the fp32 forward is an exact integer for |samples| <=
 * 7281; beyond that (int16 sources) the forward rounds like any fp32 transform: tested over the
 * whole int16 range to the north star's 1e-5 per-block bound, and the int16 round trip at
 * r = n^2 stays the identity there (tests/test_gpu_parity.py::test_jam_full_int16_range). */
adct_status approx_dct_jam_roundtrip(int32_t n, const void* src, adct_dtype src_t, adct_geom g, int32_t r,
                                     void* recon, adct_dtype recon_t, adct_clip clip, void* stream);

/* The greedy angle search of §3 (Eq. 5-6; Fig. 2) that produces T1
 * and T2 (§4.1), one permutation sequence per CTA.  For each sequence the free
 * rows are placed in the given order; row k is the vector of D = P^8 with the largest
 * s(d) = <c_k, d> / (|d| |c_k|) (fp64, reading A21: smallest angle) among the non-zero
 * vectors orthogonal to every placed row (A23), ties to the earliest vector of the
 * lexicographic enumeration with the entries in ascending order (A22).
 * c: HOST fp64 [64], rows of the matrix to approximate (the orthonormal DCT, reading A1).
 * entries: HOST int32 [n_entries] (1..8 distinct values in [-127, 127]; sorted internally).
 * fixed / fixed_mask: HOST rows pre-assigned before the search (bit k of the mask: row k taken
 * from fixed[8k..8k+7]; §4.1 fixes rows 0 and 4).  orders: DEVICE int32
 * [n_orders][8 - popcount(fixed_mask)], the free row indices in placement order.
 * out: DEVICE int32 [n_orders][64] (zero for infeasible sequences); status: DEVICE int32
 * [n_orders], 0 = ok, 1 = no orthogonal candidate left at some step (A24), 2 = invalid
 * sequence (an index outside 0..7, a fixed row, or a repeated row).
 * ties: DEVICE int32 [n_orders][4] or NULL -- the exact ties met (several orthogonal candidates
 * with the same fp64 score; the earliest was taken, A22; the paper's §3.4 examples have such
 * ties): {steps with a tie, row of the first tie (-1 if none), number of tied
 * candidates at the first tie, largest number of tied candidates at any step}; the steps counted
 * are those actually searched (up to an infeasible step, none for an invalid sequence).
 * The search space may be any entry set P, e.g. the extended sets of P:L1206-1235
 * ({0,+-1,+-4}, {0,+-1,+-8}, {0,+-1,+-2,+-4}, ...; |D| = |P|^8).
 * workspace >= adct_greedy_workspace_bytes(n_entries) (the packed space and the scores). */
size_t adct_greedy_workspace_bytes(int32_t n_entries);
adct_status adct_greedy_search(const double c[64], const int32_t* entries, int32_t n_entries, const int32_t fixed[64],
                               uint32_t fixed_mask, const int32_t* orders, int32_t n_orders, int32_t* out,
                               int32_t* status, int32_t* ties, void* workspace, size_t workspace_bytes, void* stream);

/* Matrix figures of merit of §4.2 for every (matrix, rho) pair: Table 4's
 * total error energy eps = pi ||C - C_hat||_F^2, MSE = tr((C - C_hat) R_x (C - C_hat)^T)/8,
 * unified coding gain C*_g (B_i from the rows of C_hat^{-1}, reading A3) and transform
 * efficiency eta, with (R_x)_ij = rho^|i-j| — the Fig. 1 curves are C*_g
 * against rho.  c: HOST fp64 [64] exact DCT (reading A1); chat, ginv: DEVICE fp64 [n][64]
 * (C_hat = S T and its inverse, row-major); rho: DEVICE fp64 [m]; out: DEVICE fp64
 * [n][m][4] = (eps, MSE, C*_g in dB, eta in %). */
adct_status adct_merit_batch(const double c[64], const double* chat, const double* ginv, int32_t n,
                             const double* rho, int32_t m, double* out, void* stream);

/* Structural similarity per image (citing Wang et al. 2004; the paper prints no
 * parameters — reading A18 in DESIGN.md, after SPEC S:L605): mean over every 8x8 window fully
 * inside the image (stride 1, uniform weights) of
 *   (2 mu_x mu_y + C1)(2 sigma_xy + C2) / ((mu_x^2 + mu_y^2 + C1)(sigma_x^2 + sigma_y^2 + C2)),
 * C1 = (0.01 peak)^2, C2 = (0.03 peak)^2, population (1/64) statistics.  orig: ADCT_U8 or
 * ADCT_I16; recon: ADCT_F32/ADCT_U8/ADCT_I16 with the same geometry; the clip policy (reading
 * A6) is applied to recon with the range [0, peak].  ssim: device fp64 [n_images].  H, W >= 8,
 * n_images <= 65535; workspace >= adct_workspace_bytes(g, 1).  Deterministic (fixed-order
 * reductions). */
adct_status ssim_reduce(const void* orig, adct_dtype orig_t, const void* recon, adct_dtype recon_t, adct_geom g,
                        double peak, adct_clip clip, double* ssim, void* workspace, size_t workspace_bytes,
                        void* stream);

/* --- fused performance paths (must equal the composition of the calls above) ----------- */

/* Forward -> retain r -> inverse -> SSIM per image, reading each block once and never writing
 * the reconstruction (SSIM as the paper's second figure of merit, P:L2258-2283,
 * P:L2345-2361; reading A18): exactly ssim_reduce(src, ADCT_U8, recon, ADCT_F32, g, 255, clip,
 * ssim, ...) of recon = approx_dct8x8_roundtrip(m, src, ADCT_U8, g, r, ADCT_F32, ADCT_CLIP_NONE).
 * src: device u8 images (8-byte aligned rows), H, W >= 8 multiples of 8; any matrix; r in 1..64;
 * clip: the policy ssim_reduce applies to the reconstruction ([0, 255]).  ssim: device fp64
 * [n_images].  workspace >= adct_workspace_bytes(g, 1).  Deterministic. */
adct_status approx_dct8x8_ssim(const adct_matrix* m, const uint8_t* src, adct_geom g, int32_t r, adct_clip clip,
                               double* ssim, void* workspace, size_t workspace_bytes, void* stream);

/* Forward -> zonal retention (first r in zig-zag order) -> inverse, written as a
 * reconstruction, with each block read once and its coefficients kept in registers: the
 * composition approx_dct8x8_fwd -> zonal_retain -> approx_dct8x8_inv (
 * BASELINE.json config 5 runs it at r = 64 on int16 residual blocks).  src: device, U8 or
 * I16 samples with geometry g (8-byte / 16-byte aligned rows); recon: device, same geometry,
 * dtype recon_t with the clip policy of approx_dct8x8_inv, except that the clip range is the
 * source's sample range ([0,255] for U8, [-32768,32767] for I16).  r in 1..64 else
 * ADCT_E_INVALID_ARGUMENT.  Any matrix (integer or real).  In place is allowed: recon may be
 * src itself (same pointer, geometry and dtype; BASELINE config 5 runs 2^30 blocks = 137 GB in
 * place) -- every block is read completely before its reconstruction is written, by the thread
 * or warp that owns it; any other overlap of src and recon is undefined. */
adct_status approx_dct8x8_roundtrip(const adct_matrix* m, const void* src, adct_dtype src_t, adct_geom g, int32_t r,
                                    void* recon, adct_dtype recon_t, adct_clip clip, void* stream);

/* Forward -> retain r -> inverse -> clip -> per-image SSE and PSNR for every r in r_list,
 * reading each block once (PSNR per image and per plane, P:L2258-2265, P:L2868;
 * reading A7).  r_list: HOST array of n_r values in 1..64 (n_r <= 64).
 * sse: device fp64 [n_images][n_r] (required).  psnr: device fp64 [n_images][n_r] or NULL:
 * psnr = 10 log10(255^2 / (sse / (H W))), +inf where sse == 0 (r = 64), computed in fp64 by the
 * library's finalize kernel from the same sum.  workspace >= adct_workspace_bytes(g, n_r).
 * Kernels (results do not depend on which one runs beyond fp32 rounding order): a single r on u8
 * planes of whole 128-byte chunks takes the tensor-core kernel for the paper's T1 at
 * r in {1, 3, 6, 10, 14, 15, 36} without clip and at r = 10 with ADCT_CLIP, and for any other
 * integer matrix at r = 10 without clip; any other single r takes a one-pass generic kernel;
 * an r list takes the sweep kernel. */
adct_status approx_dct8x8_fused_sse(const adct_matrix* m, const void* src, adct_dtype src_t, adct_geom g,
                                    const int32_t* r_list, int32_t n_r, adct_clip clip, double* sse, double* psnr,
                                    void* workspace, size_t workspace_bytes, void* stream);

/* The same on HOST buffers: src is a host (preferably pinned) dense image stack with geometry
 * g (image_stride == H*row_stride when n_images > 1, else ADCT_E_INVALID_ARGUMENT; a lone
 * image's image_stride is ignored), sse_host a host fp64 [n_images][n_r], psnr_host the same
 * or NULL.  The library stages chunks of images through the caller's device workspace
 * (>= adct_host_workspace_bytes(g, n_r, chunk_images, src_t)), overlapping host->device copies
 * with compute on two streams, and synchronises before returning.  chunk_images = images per
 * chunk (>= 1). */
size_t adct_host_workspace_bytes(adct_geom g, int32_t n_r, int64_t chunk_images, adct_dtype src_t);
adct_status approx_dct8x8_fused_sse_host(const adct_matrix* m, const void* src_host, adct_dtype src_t, adct_geom g,
                                         const int32_t* r_list, int32_t n_r, adct_clip clip, double* sse_host,
                                         double* psnr_host, int64_t chunk_images, void* workspace,
                                         size_t workspace_bytes, void* stream);

/* Several planes in ONE call -- the Y, U and V planes of a 4:2:0 stack (BASELINE config 4,
 * per-plane PSNR as in P:L2868): for each plane i exactly approx_dct8x8_fused_sse(m, src[i],
 * src_t, g[i], &r, 1, clip, sse[i], psnr[i], ...), one r.  n_planes in 1..ADCT_MAX_PLANES; the
 * planes may differ in geometry (not in n_images semantics: each plane's sse[i] / psnr[i] is a
 * device fp64 [g[i].n_images]).  psnr may be NULL, or hold NULL entries.  The planes run one
 * after the other on the stream (u8 planes without clip whose widths are multiples of 128 on the
 * tensor-core kernel, all of them or none).  workspace >= adct_planes_workspace_bytes(n_planes, g)
 * (the planes' partials side by side). */
#define ADCT_MAX_PLANES 3
size_t adct_planes_workspace_bytes(int32_t n_planes, const adct_geom* g);
adct_status approx_dct8x8_fused_sse_planes(const adct_matrix* m, int32_t n_planes, const void* const* src,
                                           adct_dtype src_t, const adct_geom* g, int32_t r, adct_clip clip,
                                           double* const* sse, double* const* psnr, void* workspace,
                                           size_t workspace_bytes, void* stream);

/* Forward transform with S folded into a uniform quantiser (BASELINE.json config 3):
 * q_kl = round_half_away(Y_kl / (step * sqrt(n_k n_l)))  (reading A10), int16 block-major.
 * Integer matrices only; src u8. */
adct_status approx_dct8x8_fwd_quant(const adct_matrix* m, const uint8_t* src, adct_geom g, int32_t step,
                                    int16_t* q, void* stream);

/* Workspace for psnr_reduce (n_r = 1) and approx_dct8x8_fused_sse. */
size_t adct_workspace_bytes(adct_geom g, int32_t n_r);

const char* adct_status_str(adct_status s);

/* Number of kernels this library has launched since load (for launch accounting). */
int64_t adct_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* ADCT_H */
