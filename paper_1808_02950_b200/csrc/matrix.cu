// matrix.cu — matrix descriptors of the C-ABI (host only).
//
// A descriptor validates a matrix once and precomputes what the kernels need:
//   integer T:  S = diag(1/||t_k||) (Eq. 2; reading A2), C_hat = S T (Eq. 1),
//               orthogonal rows -> inverse by C_hat^T: H = T^T, W = 1/(n_k n_l);
//               otherwise C_hat^{-1} (reading A4): H = T^{-1}, W = 1 (S cancels).
//   real C_hat: F = C_hat, inverse by C_hat^T (orthonormal) or C_hat^{-1}.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>

#include "adct_host.h"

namespace adct {
std::atomic<int64_t> g_launches{0};

int64_t sweep_chunks(const adct_geom& g);
int64_t ssim_tiles(const adct_geom& g);
int64_t ssim_fused_strips(const adct_geom& g);


namespace {

// the paper's T1 — selects the compile-time network
const int32_t kT1[64] = {1, 1, 1, 1, 1, 1, 1, 1,  2, 2, 1, 0, 0, -1, -2, -2, 2, 1, -1, -2, -2, -1, 1, 2,
                         1, 0, -2, -2, 2, 2, 0, -1, 1, -1, -1, 1, 1, -1, -1, 1, 2, -2, 0, 1, -1, 0, 2, -2,
                         1, -2, 2, -1, -1, 2, -2, 1, 0, -1, 2, -2, 2, -2, 1, 0};

// Gauss-Jordan inverse with partial pivoting; false if singular
bool invert8(const double* a, double* inv) {
  double m[8][16];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 16; ++j) m[i][j] = j < 8 ? a[i * 8 + j] : (j - 8 == i ? 1.0 : 0.0);
  for (int c = 0; c < 8; ++c) {
    int p = c;
    for (int i = c + 1; i < 8; ++i)
      if (std::fabs(m[i][c]) > std::fabs(m[p][c])) p = i;
    if (std::fabs(m[p][c]) < 1e-12) return false;
    if (p != c)
      for (int j = 0; j < 16; ++j) std::swap(m[c][j], m[p][j]);
    const double piv = m[c][c];
    for (int j = 0; j < 16; ++j) m[c][j] /= piv;
    for (int i = 0; i < 8; ++i)
      if (i != c) {
        const double f = m[i][c];
        if (f != 0.0)
          for (int j = 0; j < 16; ++j) m[i][j] -= f * m[c][j];
      }
  }
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) inv[i * 8 + j] = m[i][8 + j];
  return true;
}

// even/odd symmetry F J = diag((-1)^k) F and the second-level symmetry of the even rows
// (rows 0,4 symmetric, rows 2,6 antisymmetric on the first half) that fwd8 relies on
bool forward_symmetric(const double* f, double tol) {
  for (int k = 0; k < 8; ++k)
    for (int i = 0; i < 8; ++i) {
      const double sg = (k % 2) ? -1.0 : 1.0;
      if (std::fabs(f[k * 8 + 7 - i] - sg * f[k * 8 + i]) > tol) return false;
    }
  for (int k = 0; k < 8; k += 2)
    for (int i = 0; i < 4; ++i) {
      const double sg = (k == 0 || k == 4) ? 1.0 : -1.0;
      if (std::fabs(f[k * 8 + 3 - i] - sg * f[k * 8 + i]) > tol) return false;
    }
  return true;
}

// the same structure for a synthesis matrix H (x = H y): H[7-i][k] = (-1)^k H[i][k] and
// H[3-i][k] = +H[i][k] (k = 0,4), -H[i][k] (k = 2,6) — what inv8 relies on
bool synthesis_symmetric(const double* h, double tol) {
  double ht[64];
  for (int i = 0; i < 8; ++i)
    for (int k = 0; k < 8; ++k) ht[k * 8 + i] = h[i * 8 + k];
  return forward_symmetric(ht, tol);
}

void fill_common(adct_matrix* m, const double* f, const double* h, const double* wy, const double* wb,
                 const double* sb) {
  for (int i = 0; i < 64; ++i) {
    m->dev.f[i] = (float)f[i];
    m->dev.h[i] = (float)h[i];
    m->dev.wy[i] = (float)wy[i];
    m->dev.wb[i] = (float)wb[i];
    m->dev.sb[i] = (float)sb[i];
    m->dev.wy2[i] = (float)(2.0 * wy[i]);
    m->dev.q_inv[i] = 0.0f;
    m->dev.q_c[i] = 0;
    m->dev.q_p[i] = 0.0;
  }
  // offset of Y when every sample is stored as kSampleBias + x (fused u8 path)
  for (int k = 0; k < 8; ++k)
    for (int l = 0; l < 8; ++l) {
      double rk = 0, rl = 0;
      for (int i = 0; i < 8; ++i) {
        rk += f[k * 8 + i];
        rl += f[l * 8 + i];
      }
      m->dev.ybias[k * 8 + l] = (float)((double)kSampleBias * rk * rl);
    }
  m->dev.is_int = m->is_int;
}

}  // namespace
}  // namespace adct

using namespace adct;

extern "C" {

adct_status adct_matrix_create_int(const int32_t t[64], adct_matrix** out) {
  if (!t || !out) return ADCT_E_INVALID_ARGUMENT;
  *out = nullptr;
  adct_matrix* m = new (std::nothrow) adct_matrix();
  if (!m) return ADCT_E_INVALID_ARGUMENT;
  std::memcpy(m->t, t, sizeof(m->t));
  m->is_int = 1;
  double f[64];
  for (int i = 0; i < 64; ++i) f[i] = (double)t[i];
  for (int k = 0; k < 8; ++k) {
    int64_t acc = 0;
    for (int i = 0; i < 8; ++i) acc += (int64_t)t[k * 8 + i] * t[k * 8 + i];
    if (acc == 0) { delete m; return ADCT_E_SINGULAR; }
    m->n[k] = acc;
    m->s[k] = 1.0 / std::sqrt((double)acc);
  }
  if (!forward_symmetric(f, 0.0)) { delete m; return ADCT_E_UNSUPPORTED_MATRIX; }
  // exact worst-case |Y_kl| (u8: samples in [0,255]; int16: [-32768, 32767])
  m->max_u8 = 0;
  m->max_i16 = 0;
  for (int k = 0; k < 8; ++k)
    for (int l = 0; l < 8; ++l) {
      int64_t pos = 0, neg = 0;
      for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) {
          const int64_t w = (int64_t)t[k * 8 + i] * t[l * 8 + j];
          if (w > 0) pos += w; else neg -= w;
        }
      const int64_t u8 = 255 * (pos > neg ? pos : neg);
      const int64_t i16 = 32768 * (pos + neg);
      if (u8 > m->max_u8) m->max_u8 = u8;
      if (i16 > m->max_i16) m->max_i16 = i16;
    }
  if (m->max_i16 >= ((int64_t)1 << 24)) { delete m; return ADCT_E_OVERFLOW; }  // fp32 exactness
  bool orth = true;
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b)
      if (a != b) {
        int64_t dot = 0;
        for (int i = 0; i < 8; ++i) dot += (int64_t)t[a * 8 + i] * t[b * 8 + i];
        if (dot != 0) orth = false;
      }
  m->row_orth = orth ? 1 : 0;
  for (int k = 0; k < 8; ++k)
    for (int i = 0; i < 8; ++i) m->chat[k * 8 + i] = m->s[k] * f[k * 8 + i];
  double h[64], wy[64], wb[64], sb[64];
  for (int k = 0; k < 8; ++k)
    for (int l = 0; l < 8; ++l) sb[k * 8 + l] = m->s[k] * m->s[l];
  if (orth) {
    for (int i = 0; i < 8; ++i)
      for (int k = 0; k < 8; ++k) {
        h[i * 8 + k] = f[k * 8 + i];                    // H = T^T
        m->g[i * 8 + k] = m->chat[k * 8 + i];           // G = C_hat^T
      }
    for (int k = 0; k < 8; ++k)
      for (int l = 0; l < 8; ++l) {
        wy[k * 8 + l] = 1.0 / ((double)m->n[k] * (double)m->n[l]);
        wb[k * 8 + l] = m->s[k] * m->s[l];
      }
  } else {
    double tinv[64];
    if (!invert8(f, tinv)) { delete m; return ADCT_E_SINGULAR; }
    for (int i = 0; i < 64; ++i) h[i] = tinv[i];       // H = T^{-1}
    for (int i = 0; i < 8; ++i)
      for (int k = 0; k < 8; ++k) m->g[i * 8 + k] = tinv[i * 8 + k] / m->s[k];  // C_hat^{-1} = T^{-1} S^{-1}
    for (int k = 0; k < 8; ++k)
      for (int l = 0; l < 8; ++l) {
        wy[k * 8 + l] = 1.0;
        wb[k * 8 + l] = 1.0 / (m->s[k] * m->s[l]);
      }
    if (!synthesis_symmetric(h, 1e-9)) { delete m; return ADCT_E_UNSUPPORTED_MATRIX; }
  }
  m->specialized = std::memcmp(t, kT1, sizeof(kT1)) == 0 ? 1 : 0;
  fill_common(m, f, h, wy, wb, sb);
  *out = m;
  return ADCT_OK;
}

adct_status adct_matrix_create_real(const double c[64], adct_matrix** out) {
  if (!c || !out) return ADCT_E_INVALID_ARGUMENT;
  *out = nullptr;
  for (int i = 0; i < 64; ++i)
    if (!std::isfinite(c[i])) return ADCT_E_INVALID_ARGUMENT;
  if (!forward_symmetric(c, 1e-9)) return ADCT_E_UNSUPPORTED_MATRIX;
  adct_matrix* m = new (std::nothrow) adct_matrix();
  if (!m) return ADCT_E_INVALID_ARGUMENT;
  m->is_int = 0;
  m->specialized = 0;
  m->max_u8 = m->max_i16 = 0;
  std::memcpy(m->chat, c, sizeof(m->chat));
  for (int k = 0; k < 8; ++k) {
    double acc = 0;
    for (int i = 0; i < 8; ++i) acc += c[k * 8 + i] * c[k * 8 + i];
    if (acc == 0.0) { delete m; return ADCT_E_SINGULAR; }
    m->s[k] = 1.0;
    m->n[k] = 0;
  }
  double dev = 0.0;
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b) {
      double dot = 0;
      for (int i = 0; i < 8; ++i) dot += c[a * 8 + i] * c[b * 8 + i];
      dev = std::fmax(dev, std::fabs(dot - (a == b ? 1.0 : 0.0)));
    }
  m->row_orth = dev <= 1e-9 ? 1 : 0;
  double h[64], ones[64];
  if (m->row_orth) {
    for (int i = 0; i < 8; ++i)
      for (int k = 0; k < 8; ++k) h[i * 8 + k] = c[k * 8 + i];
  } else if (!invert8(c, h)) {
    delete m;
    return ADCT_E_SINGULAR;
  }
  if (!synthesis_symmetric(h, 1e-9)) { delete m; return ADCT_E_UNSUPPORTED_MATRIX; }
  std::memcpy(m->g, h, sizeof(h));
  for (int i = 0; i < 64; ++i) ones[i] = 1.0;
  fill_common(m, c, h, ones, ones, ones);
  *out = m;
  return ADCT_OK;
}

adct_status adct_matrix_info(const adct_matrix* m, double s[8], double g[64], int32_t* row_orthogonal,
                             int32_t* is_integer, int64_t* max_abs_y_u8, int64_t* max_abs_y_i16,
                             int32_t* specialized) {
  if (!m) return ADCT_E_INVALID_ARGUMENT;
  if (s) std::memcpy(s, m->s, sizeof(m->s));
  if (g) std::memcpy(g, m->g, sizeof(m->g));
  if (row_orthogonal) *row_orthogonal = m->row_orth;
  if (is_integer) *is_integer = m->is_int;
  if (max_abs_y_u8) *max_abs_y_u8 = m->max_u8;
  if (max_abs_y_i16) *max_abs_y_i16 = m->max_i16;
  if (specialized) *specialized = m->specialized;
  return ADCT_OK;
}

void adct_matrix_destroy(adct_matrix* m) { delete m; }

adct_status adct_zigzag_order(int32_t order[64]) {
  if (!order) return ADCT_E_INVALID_ARGUMENT;
  for (int z = 0; z < 64; ++z) order[z] = kZZ.order[z];
  return ADCT_OK;
}

const char* adct_status_str(adct_status s) {
  switch (s) {
    case ADCT_OK: return "ok";
    case ADCT_E_INVALID_ARGUMENT: return "invalid argument";
    case ADCT_E_UNSUPPORTED_MATRIX: return "unsupported matrix (no even/odd symmetry)";
    case ADCT_E_SINGULAR: return "singular matrix";
    case ADCT_E_OVERFLOW: return "coefficient type cannot hold the worst-case value";
    case ADCT_E_ALIGNMENT: return "misaligned buffer or stride";
    case ADCT_E_CUDA: return "CUDA error";
    case ADCT_E_WORKSPACE: return "workspace missing or too small";
  }
  return "unknown status";
}

int64_t adct_launch_count(void) { return g_launches.load(); }

adct_status adct_matrix_chat(const adct_matrix* m, double chat[64]) {
  if (!m || !chat) return ADCT_E_INVALID_ARGUMENT;
  for (int i = 0; i < 64; ++i) chat[i] = m->chat[i];
  return ADCT_OK;
}

size_t adct_workspace_bytes(adct_geom g, int32_t n_r) {
  (void)n_r;  // per-image partials hold all 64 r slots of the sweep kernel
  const int64_t a = (fused_chunks(g) > sweep_chunks(g) ? fused_chunks(g) : sweep_chunks(g)) * 64;
  const int64_t b = sse_chunks(g);
  int64_t c = stream_partials_per_image(g) > ssim_tiles(g) ? stream_partials_per_image(g) : ssim_tiles(g);
  if (ssim_fused_strips(g) > c) c = ssim_fused_strips(g);
  int64_t per = a > b ? a : b;
  if (c > per) per = c;
  return (size_t)(g.n_images > 0 ? g.n_images : 0) * (size_t)per * sizeof(double) + 256;
}

}  // extern "C"
