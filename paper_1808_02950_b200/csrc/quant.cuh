// quant.cuh — the uniform quantiser of BASELINE.json config 3 for the paper's T1 (S1):
// q_kl = round_half_away(Y_kl / c_kl), c_kl = step sqrt(n_k n_l) (reading A10), shared by the SIMT
// kernel (blockmajor.cu) and the tensor-core kernel (tc.cu).
//
// At the 40 positions where sqrt(n_k n_l) is an integer (8, 12, 18, 20), c is an even integer and
// |q| = floor(A / c), A = |Y| + c/2 an integer < 2^23.  With u = fp32 1/c rounded UP, the exact
// product A u lies in [A/c, A/c + A 2^-23 / c): at a multiple A = m c it is >= m, otherwise
// A/c <= m - 1/c and A 2^-23 < 1 keeps it below m, so floor(A u) = floor(A / c) for every such A
// (tests/test_kernel_arith.py checks every A).  One FFMA rounding toward -inf onto 1.5 * 2^23
// gives 1.5 * 2^23 + |q|; 3 * 2^23 minus that is 1.5 * 2^23 - |q|, whose low 16 bits are -|q|.
// At the 24 irrational positions (n_k n_l = 160, 360) ties are impossible; Y/c is rounded to
// nearest by one FFMA onto 1.5 * 2^23, and a coefficient within 2^-14 of a rounding boundary
// sends the warp to the exact integer rule (2m-1)^2 P <= 4 Y^2 < (2m+1)^2 P, P = step^2 n_k n_l
// (fp64, exact below 2^53).
#pragma once
#include <cmath>
#include <cstdint>

namespace adct {

struct QTab {
  float inv[64];    // fp32(1 / c_kl)
  float invu[64];   // fp32(1 / c_kl) rounded up (rational positions; ADCT_Q_FAST)
  double p[64];     // P_kl = step^2 n_k n_l
  double rsp[64];   // 1 / sqrt(P_kl) (fp64; the exact rule's estimate, corrected by the integer tests)
  float ru[4];      // invu by sqrt(n_k n_l) = 8, 12, 18, 20 (ADCT_Q_FAST: 6 registers, not 64 loads)
  float ri[2];      // inv at the irrational positions, n_k n_l = 160, 360
};
__host__ __device__ constexpr int q_rclass(int k, int l) {  // index of sqrt(n_k n_l) in {8, 12, 18, 20}
  return ((k & 3) == 2) ? 3 : (((k & 1) + (l & 1)) == 0 ? 0 : (((k & 1) + (l & 1)) == 1 ? 1 : 2));
}
__host__ __device__ constexpr int q_iclass(int k, int l) {  // 0: n_k n_l = 160, 1: 360
  return ((k & 1) | (l & 1));
}
__host__ __device__ constexpr bool t1_rational(int k, int l) {
  return ((k & 3) == 2) == ((l & 3) == 2);
}
__host__ __device__ constexpr int t1_sqrt_nn(int k, int l) {  // sqrt(n_k n_l) where it is an integer
  return ((k & 3) == 2) ? 20 : ((k & 3) == 0 ? ((l & 3) == 0 ? 8 : 12) : ((l & 3) == 0 ? 12 : 18));
}

// host: the tables for (step, n = diag(T T^T))
inline void q_fill(QTab& qt, int32_t step, const int64_t* n) {
  for (int k = 0; k < 8; ++k)
    for (int l = 0; l < 8; ++l) {
      const double p = (double)step * step * (double)n[k] * (double)n[l];
      qt.p[k * 8 + l] = p;
      qt.rsp[k * 8 + l] = 1.0 / std::sqrt(p);
      qt.inv[k * 8 + l] = (float)(1.0 / std::sqrt(p));
      qt.invu[k * 8 + l] = 0.0f;
      if (t1_rational(k, l)) {  // c = step sqrt(n_k n_l), an integer: fp32 1/c rounded up
        const double c = (double)step * t1_sqrt_nn(k, l);
        float u = (float)(1.0 / c);
        if ((double)u * c < 1.0) u = std::nextafter(u, 1.0f);  // exact product: 24 + 17 bits
        qt.invu[k * 8 + l] = u;
      }
    }
  for (int j = 0; j < 4; ++j) {  // the same values by class
    constexpr int kk[4] = {0, 0, 1, 2}, ll[4] = {0, 1, 1, 2};
    qt.ru[j] = qt.invu[kk[j] * 8 + ll[j]];
  }
  qt.ri[0] = qt.inv[2 * 8 + 0];  // n = 20 x 8
  qt.ri[1] = qt.inv[2 * 8 + 1];  // n = 20 x 18
}

#ifdef __CUDACC__
// One block: y[k * 8 + l] = Y_kl as fp32 (exact integers) -> 32 words of two int16 codes (raster
// order, low half first).  Warp-collective (the rare exact path is taken by the whole warp).
__device__ __forceinline__ void q_block_t1(const float (&y)[64], const float (&qru)[4], const float (&qri)[2],
                                           float stepf, const QTab& qt, uint32_t (&packed)[32]) {
  bool near = false;
#pragma unroll
  for (int k = 0; k < 8; ++k)
#pragma unroll
    for (int l = 0; l < 8; l += 2) {
      uint32_t u[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float yy = y[k * 8 + l + e];
        if (t1_rational(k, l + e)) {
          const float A = fabsf(yy) + stepf * (0.5f * (float)t1_sqrt_nn(k, l + e));  // exact
          const float up = __fmaf_rd(A, qru[q_rclass(k, l + e)], 12582912.0f);      // 1.5*2^23 + |q|
          u[e] = __float_as_uint(yy < 0.0f ? 25165824.0f - up : up);
        } else {
          const float iv = qri[q_iclass(k, l + e)];
          const float f = fmaf(yy, iv, 12582912.0f);
          near |= fabsf(fmaf(yy, iv, 12582912.0f - f)) > 0.49993896f;  // within 2^-14 of a boundary
          u[e] = __float_as_uint(f);
        }
      }
      packed[k * 4 + l / 2] = __byte_perm(u[0], u[1], 0x5410);
    }
  if (__any_sync(0xffffffffu, near)) {  // rare: exact integer rule at irrational positions
#pragma unroll
    for (int kl = 0; kl < 64; ++kl) {
      if (t1_rational(kl >> 3, kl & 7)) continue;
      const float yy = y[kl];
      const float f = fmaf(yy, qt.inv[kl], 12582912.0f);
      if (near && fabsf(fmaf(yy, qt.inv[kl], 12582912.0f - f)) > 0.49993896f) {
        const double a2 = 4.0 * (double)yy * (double)yy, pp = qt.p[kl];
        double mm = rint(fabs((double)yy) * qt.rsp[kl]);  // within 1 of the answer
        if (mm >= 1.0 && (2.0 * mm - 1.0) * (2.0 * mm - 1.0) * pp > a2) mm -= 1.0;
        else if ((2.0 * mm + 1.0) * (2.0 * mm + 1.0) * pp <= a2) mm += 1.0;
        const uint32_t q16 = (uint32_t)(uint16_t)(int16_t)(yy < 0.0f ? -(int)mm : (int)mm);
        uint32_t& wv = packed[kl >> 1];
        wv = (kl & 1) ? ((wv & 0xffffu) | (q16 << 16)) : ((wv & 0xffff0000u) | q16);
      }
    }
  }
}
#endif

}  // namespace adct
