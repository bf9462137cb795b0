// merit.cu — next row f4: the matrix figures of merit of §4.2 for a
// batch of (matrix, rho) pairs — Table 4's columns and the Fig. 1 curves of the coding gain
// against the interpixel correlation rho.  One thread per pair, fp64:
//   eps(C_hat)  = pi ||C - C_hat||_F^2                                  (§4.2.1)
//   MSE(C_hat)  = tr((C - C_hat) R_x (C - C_hat)^T) / 8                   (§4.2.2)
//   C*_g        = 10 log10 prod_i (A_i B_i)^(-1/8), A_i = su((c_i c_i^T) o R_x),
//                 B_i = ||g_i||^2, g_i the i-th row of C_hat^{-1} (reading A3) (§4.2.3)
//   eta         = sum_i |r_ii| / sum_ij |r_ij| * 100, R_y = C_hat R_x C_hat^T (§4.2.4)
// with the Markov-1 covariance (R_x)_ij = rho^|i-j|.
#include <cmath>

#include "adct_host.h"

namespace adct {
namespace {

struct CExact {
  double c[64];
};

__global__ void merit_kernel(const double* __restrict__ chat, const double* __restrict__ ginv, int32_t n,
                             const double* __restrict__ rho, int32_t m, CExact ce, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * m) return;
  const int32_t a = (int32_t)(t / m), b = (int32_t)(t % m);
  const double* ch = chat + (int64_t)a * 64;
  const double* gi = ginv + (int64_t)a * 64;
  const double r = rho[b];
  double R[8][8];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) R[i][j] = pow(r, (double)abs(i - j));
  double eps = 0.0, tr = 0.0;
  double d[8][8];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      d[i][j] = ce.c[i * 8 + j] - ch[i * 8 + j];
      eps += d[i][j] * d[i][j];
    }
  for (int i = 0; i < 8; ++i)  // tr(D R D^T) = sum_i d_i R d_i^T
    for (int j = 0; j < 8; ++j) {
      double s = 0.0;
      for (int k = 0; k < 8; ++k) s += R[j][k] * d[i][k];
      tr += d[i][j] * s;
    }
  double logprod = 0.0;
  for (int i = 0; i < 8; ++i) {
    double A = 0.0, B = 0.0;
    for (int j = 0; j < 8; ++j) {
      for (int k = 0; k < 8; ++k) A += ch[i * 8 + j] * ch[i * 8 + k] * R[j][k];
      B += gi[i * 8 + j] * gi[i * 8 + j];
    }
    logprod += -log10(A * B) / 8.0;
  }
  double diag = 0.0, all = 0.0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      double s = 0.0;  // (C_hat R C_hat^T)_ij
      for (int k = 0; k < 8; ++k) {
        double u = 0.0;
        for (int l = 0; l < 8; ++l) u += R[k][l] * ch[j * 8 + l];
        s += ch[i * 8 + k] * u;
      }
      all += fabs(s);
      if (i == j) diag += fabs(s);
    }
  double* o = out + t * 4;
  o[0] = M_PI * eps;
  o[1] = tr / 8.0;
  o[2] = 10.0 * logprod;
  o[3] = diag / all * 100.0;
}

}  // namespace
}  // namespace adct

using namespace adct;

extern "C" adct_status adct_merit_batch(const double c[64], const double* chat, const double* ginv, int32_t n,
                                        const double* rho, int32_t m, double* out, void* stream) {
  if (!c || !chat || !ginv || !rho || !out || n < 0 || m < 0) return ADCT_E_INVALID_ARGUMENT;
  const int64_t pairs = (int64_t)n * m;
  if (pairs == 0) return ADCT_OK;
  if (pairs >= ((int64_t)1 << 31)) return ADCT_E_INVALID_ARGUMENT;
  CExact ce;
  for (int i = 0; i < 64; ++i) ce.c[i] = c[i];
  merit_kernel<<<(unsigned)((pairs + 127) / 128), 128, 0, (cudaStream_t)stream>>>(chat, ginv, n, rho, m, ce, out);
  count_launch();
  return launch_status();
}
