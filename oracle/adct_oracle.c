/*
 * adct_oracle.c — plain, slow, by-definition CPU oracle for the hot path of
 * arXiv 1808.02950 (§6.1 "Still Image Compression").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_1808_02950_b200/), and the
 * CUDA path never calls it.
 *
 * Every step is written as the paper defines it, in int64 (integer transform) or
 * fp64 (scaling, inverse, error), with no fast algorithm, butterfly, blocking or
 * Parseval shortcut:
 *   forward    B = C_hat A C_hat^T, C_hat = S T               P:L2205-2217, Eq.(1)
 *              integer part Y = T X T^T as two 8x8 products   (S applied afterwards)
 *   scaling    S = diag(1/||t_k||)                             Eq.(2); reading A2
 *   retention  keep the first r of 64 in zig-zag order        P:L2219-2233; reading A5
 *   inverse    A = C_hat^T B' C_hat  (orthogonal C_hat)
 *              A = C_hat^-1 B' C_hat^-T (non-orthogonal)       reading A4
 *   error      SSE, MSE = SSE/(H W), PSNR = 10 log10(255^2/MSE) P:L2258-2265; reading A7
 *   quantiser  q = round_half_away(Y / (step sqrt(n_k n_l)))   BASELINE C3; reading A10
 *
 * Layout conventions (shared with the C-ABI only by documentation):
 *   images  row-major planes [img][H][W], u8 or int16 samples
 *   blocks  block-major [img][by][bx][8][8], raster index k*8+l inside a block,
 *           k = vertical frequency (row of B), l = horizontal frequency.
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC -o oracle/liboracle.so oracle/adct_oracle.c -lm
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { OR_CLIP_NONE = 0, OR_CLIP = 1, OR_CLIP_ROUND = 2 };

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Timing only (bench.py cpu_baseline): the OpenMP thread count of later calls.  The results do
 * not depend on it (per-block work, per-image sums in block order). */
void oracle_set_num_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n > 0 ? n : 1);
#else
  (void)n;
#endif
}

/* ---- zig-zag order (reading A5: JPEG order) ---------------------------
 * Built from the anti-diagonal rule: coefficients are visited by increasing k+l; on an
 * odd anti-diagonal k increases, on an even one k decreases.  order[z] = k*8+l. */
void oracle_zigzag_order(int32_t order[64]) {
  int z = 0;
  for (int d = 0; d <= 14; ++d) {
    if (d % 2 == 1) {
      for (int k = 0; k <= 7; ++k) {
        int l = d - k;
        if (l >= 0 && l <= 7) order[z++] = k * 8 + l;
      }
    } else {
      for (int k = 7; k >= 0; --k) {
        int l = d - k;
        if (l >= 0 && l <= 7) order[z++] = k * 8 + l;
      }
    }
  }
}

/* n_k = sum_i T_ki^2 (exact) and s_k = 1/sqrt(n_k): Eq.(2) for row-orthogonal T. */
void oracle_row_scaling(const int32_t t[64], int64_t n[8], double s[8]) {
  for (int k = 0; k < 8; ++k) {
    int64_t acc = 0;
    for (int i = 0; i < 8; ++i) acc += (int64_t)t[k * 8 + i] * t[k * 8 + i];
    n[k] = acc;
    s[k] = 1.0 / sqrt((double)acc);
  }
}

/* C_hat = S T (Eq. 1). */
void oracle_chat_from_int(const int32_t t[64], double chat[64]) {
  int64_t n[8];
  double s[8];
  oracle_row_scaling(t, n, s);
  for (int k = 0; k < 8; ++k)
    for (int i = 0; i < 8; ++i) chat[k * 8 + i] = s[k] * (double)t[k * 8 + i];
}

/* Synthesis matrix G used by the inverse A = G B' G^T.
 * Orthonormal rows (C_hat C_hat^T = I within 1e-12): G = C_hat^T.
 * Otherwise G = C_hat^{-1} by Gauss-Jordan elimination with partial pivoting (A4).
 * Returns 1 if orthonormal, 0 if inverted, -1 if singular. */
int oracle_synthesis_matrix(const double chat[64], double g[64]) {
  double maxdev = 0.0;
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b) {
      double dot = 0.0;
      for (int i = 0; i < 8; ++i) dot += chat[a * 8 + i] * chat[b * 8 + i];
      double dev = fabs(dot - (a == b ? 1.0 : 0.0));
      if (dev > maxdev) maxdev = dev;
    }
  if (maxdev <= 1e-12) {
    for (int i = 0; i < 8; ++i)
      for (int k = 0; k < 8; ++k) g[i * 8 + k] = chat[k * 8 + i];
    return 1;
  }
  double m[8][16];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 16; ++j) m[i][j] = j < 8 ? chat[i * 8 + j] : (j - 8 == i ? 1.0 : 0.0);
  for (int c = 0; c < 8; ++c) {
    int p = c;
    for (int i = c + 1; i < 8; ++i)
      if (fabs(m[i][c]) > fabs(m[p][c])) p = i;
    if (fabs(m[p][c]) < 1e-12) return -1;
    if (p != c)
      for (int j = 0; j < 16; ++j) {
        double tmp = m[c][j];
        m[c][j] = m[p][j];
        m[p][j] = tmp;
      }
    double piv = m[c][c];
    for (int j = 0; j < 16; ++j) m[c][j] /= piv;
    for (int i = 0; i < 8; ++i)
      if (i != c) {
        double f = m[i][c];
        for (int j = 0; j < 16; ++j) m[i][j] -= f * m[c][j];
      }
  }
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) g[i * 8 + j] = m[i][8 + j];
  return 0;
}

static double sample(const void* src, int bits, int64_t idx) {
  return bits == 8 ? (double)((const uint8_t*)src)[idx] : (double)((const int16_t*)src)[idx];
}
static int64_t isample(const void* src, int bits, int64_t idx) {
  return bits == 8 ? (int64_t)((const uint8_t*)src)[idx] : (int64_t)((const int16_t*)src)[idx];
}

/* Integer forward Y = T X T^T of every 8x8 block (P:L2205-2217 without S):
 * P = T X, then Y = P T^T, int64 accumulation.  y is block-major. */
int oracle_forward_int(const int32_t t[64], const void* src, int bits, int64_t n_img, int32_t h, int32_t w,
                       int64_t* y) {
  if ((h % 8) || (w % 8) || (bits != 8 && bits != 16)) return -1;
  const int64_t bh = h / 8, bw = w / 8, nb = n_img * bh * bw;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t img = b / (bh * bw), by = (b / bw) % bh, bx = b % bw;
    int64_t x[8][8], p[8][8];
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) x[i][j] = isample(src, bits, img * h * w + (by * 8 + i) * w + bx * 8 + j);
    for (int k = 0; k < 8; ++k)
      for (int j = 0; j < 8; ++j) {
        int64_t acc = 0;
        for (int i = 0; i < 8; ++i) acc += (int64_t)t[k * 8 + i] * x[i][j];
        p[k][j] = acc;
      }
    for (int k = 0; k < 8; ++k)
      for (int l = 0; l < 8; ++l) {
        int64_t acc = 0;
        for (int j = 0; j < 8; ++j) acc += p[k][j] * (int64_t)t[l * 8 + j];
        y[b * 64 + k * 8 + l] = acc;
      }
  }
  return 0;
}

/* Real forward B = C X C^T in fp64 (e.g. the exact DCT). */
int oracle_forward_real(const double c[64], const void* src, int bits, int64_t n_img, int32_t h, int32_t w,
                        double* out) {
  if ((h % 8) || (w % 8) || (bits != 8 && bits != 16)) return -1;
  const int64_t bh = h / 8, bw = w / 8, nb = n_img * bh * bw;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t img = b / (bh * bw), by = (b / bw) % bh, bx = b % bw;
    double x[8][8], p[8][8];
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) x[i][j] = sample(src, bits, img * h * w + (by * 8 + i) * w + bx * 8 + j);
    for (int k = 0; k < 8; ++k)
      for (int j = 0; j < 8; ++j) {
        double acc = 0.0;
        for (int i = 0; i < 8; ++i) acc += c[k * 8 + i] * x[i][j];
        p[k][j] = acc;
      }
    for (int k = 0; k < 8; ++k)
      for (int l = 0; l < 8; ++l) {
        double acc = 0.0;
        for (int j = 0; j < 8; ++j) acc += p[k][j] * c[l * 8 + j];
        out[b * 64 + k * 8 + l] = acc;
      }
  }
  return 0;
}

/* B_kl = s_k s_l Y_kl  (B = S Y S, S diagonal). */
void oracle_scale(const int64_t* y, const double s[8], int64_t n_blocks, double* out) {
  for (int64_t b = 0; b < n_blocks; ++b)
    for (int k = 0; k < 8; ++k)
      for (int l = 0; l < 8; ++l) out[b * 64 + k * 8 + l] = s[k] * s[l] * (double)y[b * 64 + k * 8 + l];
}

/* keep[k*8+l] = 1 iff the zig-zag position of (k,l) is < r. */
static void keep_mask(int r, int keep[64]) {
  int32_t order[64];
  oracle_zigzag_order(order);
  for (int z = 0; z < 64; ++z) keep[order[z]] = z < r;
}

int oracle_retain_i64(int64_t* y, int64_t n_blocks, int32_t r) {
  if (r < 1 || r > 64) return -1;
  int keep[64];
  keep_mask(r, keep);
  for (int64_t b = 0; b < n_blocks; ++b)
    for (int i = 0; i < 64; ++i)
      if (!keep[i]) y[b * 64 + i] = 0;
  return 0;
}

int oracle_retain_f64(double* y, int64_t n_blocks, int32_t r) {
  if (r < 1 || r > 64) return -1;
  int keep[64];
  keep_mask(r, keep);
  for (int64_t b = 0; b < n_blocks; ++b)
    for (int i = 0; i < 64; ++i)
      if (!keep[i]) y[b * 64 + i] = 0.0;
  return 0;
}

/* A = G B' G^T per block (G = C_hat^T or C_hat^{-1}), fp64. */
void oracle_inverse(const double g[64], const double* bp, int64_t n_blocks, double* a) {
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < n_blocks; ++b) {
    double p[8][8];
    for (int i = 0; i < 8; ++i)
      for (int l = 0; l < 8; ++l) {
        double acc = 0.0;
        for (int k = 0; k < 8; ++k) acc += g[i * 8 + k] * bp[b * 64 + k * 8 + l];
        p[i][l] = acc;
      }
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) {
        double acc = 0.0;
        for (int l = 0; l < 8; ++l) acc += p[i][l] * g[j * 8 + l];
        a[b * 64 + i * 8 + j] = acc;
      }
  }
}

/* Reconstruction value after the clip policy (reading A6). lo/hi = sample range. */
static double apply_clip(double v, int clip, double lo, double hi) {
  if (clip == OR_CLIP_NONE) return v;
  if (v < lo) v = lo;
  if (v > hi) v = hi;
  if (clip == OR_CLIP_ROUND) v = nearbyint(v); /* round half to even (default FP mode) */
  return v;
}

/* SSE per image between the original samples and a block-major reconstruction. */
int oracle_sse(const void* orig, int bits, const double* recon, int64_t n_img, int32_t h, int32_t w, int clip,
               double* sse) {
  if ((h % 8) || (w % 8)) return -1;
  const double lo = bits == 8 ? 0.0 : -32768.0, hi = bits == 8 ? 255.0 : 32767.0;
  const int64_t bh = h / 8, bw = w / 8;
  for (int64_t img = 0; img < n_img; ++img) {
    double acc = 0.0;
    for (int64_t by = 0; by < bh; ++by)
      for (int64_t bx = 0; bx < bw; ++bx) {
        const int64_t b = (img * bh + by) * bw + bx;
        for (int i = 0; i < 8; ++i)
          for (int j = 0; j < 8; ++j) {
            double x = sample(orig, bits, img * h * w + (by * 8 + i) * w + bx * 8 + j);
            double d = x - apply_clip(recon[b * 64 + i * 8 + j], clip, lo, hi);
            acc += d * d;
          }
      }
    sse[img] = acc;
  }
  return 0;
}

/* PSNR = 10 log10(peak^2 / MSE), MSE = SSE / n_pixels; +inf when SSE = 0. */
double oracle_psnr(double sse, int64_t n_pixels, double peak) {
  if (sse == 0.0) return INFINITY;
  return 10.0 * log10(peak * peak / (sse / (double)n_pixels));
}

/* C3 quantiser (reading A10): q = sign(Y) * |q|,
 * |q| = max{ m >= 0 : m = 0 or (2m-1)^2 step^2 n_k n_l <= 4 Y^2 },
 * i.e. round-half-away-from-zero of Y / (step sqrt(n_k n_l)) decided in integers. */
void oracle_quantize(const int64_t* y, const int64_t n[8], int32_t step, int64_t n_blocks, int16_t* q) {
  for (int64_t b = 0; b < n_blocks; ++b)
    for (int k = 0; k < 8; ++k)
      for (int l = 0; l < 8; ++l) {
        const int64_t v = y[b * 64 + k * 8 + l];
        const int64_t av = v < 0 ? -v : v;
        const int64_t p = n[k] * n[l] * (int64_t)step * step;
        int64_t m = 0;
        while ((2 * m + 1) * (2 * m + 1) * p <= 4 * av * av) ++m;
        q[b * 64 + k * 8 + l] = (int16_t)(v < 0 ? -m : m);
      }
}

/* The whole experiment of §6.1 for a list of r values, one block at a time:
 * forward -> (scale) -> retain r -> inverse -> clip -> squared error, summed per image.
 * t != NULL: integer path (Y = T X T^T in int64, B = S Y S, G from C_hat = S T);
 * t == NULL: real path with c (fp64 C_hat).  sse is [n_img][n_r].
 * Deterministic: each image's sum runs over its blocks in raster order. */
int oracle_codec_sse(const int32_t* t, const double* c, const void* src, int bits, int64_t n_img, int32_t h,
                     int32_t w, const int32_t* r_list, int32_t n_r, int clip, double* sse) {
  if ((h % 8) || (w % 8) || (bits != 8 && bits != 16) || n_r < 1) return -1;
  for (int i = 0; i < n_r; ++i)
    if (r_list[i] < 1 || r_list[i] > 64) return -1;
  double chat[64], g[64], s[8];
  int64_t n[8];
  if (t) {
    oracle_row_scaling(t, n, s);
    oracle_chat_from_int(t, chat);
  } else {
    memcpy(chat, c, sizeof(chat));
  }
  if (oracle_synthesis_matrix(chat, g) < 0) return -2;
  const double lo = bits == 8 ? 0.0 : -32768.0, hi = bits == 8 ? 255.0 : 32767.0;
  const int64_t bh = h / 8, bw = w / 8, nb = n_img * bh * bw;
  /* per-block partial errors, then per-image sums in block order (thread-count independent) */
  double* part = (double*)malloc(sizeof(double) * (size_t)(nb * n_r));
  if (!part) return -3;
  int32_t order[64];
  oracle_zigzag_order(order);
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t img = b / (bh * bw), by = (b / bw) % bh, bx = b % bw;
    double x[64], bcoef[64];
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) x[i * 8 + j] = sample(src, bits, img * h * w + (by * 8 + i) * w + bx * 8 + j);
    if (t) {
      int64_t p[64], xi[64];
      for (int i = 0; i < 64; ++i) xi[i] = (int64_t)x[i];
      for (int k = 0; k < 8; ++k)
        for (int j = 0; j < 8; ++j) {
          int64_t acc = 0;
          for (int i = 0; i < 8; ++i) acc += (int64_t)t[k * 8 + i] * xi[i * 8 + j];
          p[k * 8 + j] = acc;
        }
      for (int k = 0; k < 8; ++k)
        for (int l = 0; l < 8; ++l) {
          int64_t acc = 0;
          for (int j = 0; j < 8; ++j) acc += p[k * 8 + j] * (int64_t)t[l * 8 + j];
          bcoef[k * 8 + l] = s[k] * s[l] * (double)acc;
        }
    } else {
      double p[64];
      for (int k = 0; k < 8; ++k)
        for (int j = 0; j < 8; ++j) {
          double acc = 0.0;
          for (int i = 0; i < 8; ++i) acc += chat[k * 8 + i] * x[i * 8 + j];
          p[k * 8 + j] = acc;
        }
      for (int k = 0; k < 8; ++k)
        for (int l = 0; l < 8; ++l) {
          double acc = 0.0;
          for (int j = 0; j < 8; ++j) acc += p[k * 8 + j] * chat[l * 8 + j];
          bcoef[k * 8 + l] = acc;
        }
    }
    for (int ri = 0; ri < n_r; ++ri) {
      double bp[64], q[64];
      for (int i = 0; i < 64; ++i) bp[i] = 0.0;
      for (int z = 0; z < r_list[ri]; ++z) bp[order[z]] = bcoef[order[z]];
      for (int i = 0; i < 8; ++i)
        for (int l = 0; l < 8; ++l) {
          double acc = 0.0;
          for (int k = 0; k < 8; ++k) acc += g[i * 8 + k] * bp[k * 8 + l];
          q[i * 8 + l] = acc;
        }
      double e = 0.0;
      for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) {
          double acc = 0.0;
          for (int l = 0; l < 8; ++l) acc += q[i * 8 + l] * g[j * 8 + l];
          double d = x[i * 8 + j] - apply_clip(acc, clip, lo, hi);
          e += d * d;
        }
      part[b * n_r + ri] = e;
    }
  }
  for (int64_t img = 0; img < n_img; ++img)
    for (int ri = 0; ri < n_r; ++ri) {
      double acc = 0.0;
      for (int64_t b = img * bh * bw; b < (img + 1) * bh * bw; ++b) acc += part[b * n_r + ri];
      sse[img * n_r + ri] = acc;
    }
  free(part);
  return 0;
}
