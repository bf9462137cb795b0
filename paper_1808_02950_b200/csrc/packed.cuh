// packed.cuh — the 8x8 forward / inverse networks of adct_internal.cuh on COLUMN PAIRS with the
// packed fp32 instructions of sm_100 (FFMA2 / FADD2 / FMUL2: two lanes' FP32 work per issue slot).
//
// A block is held as x2[i][c] = (x[i][2c], x[i][2c+1]).  Vertical passes (along i) run the scalar
// networks on float2 with the coefficient broadcast to both lanes.  Horizontal passes (along j)
// compute two OUTPUTS per instruction with the input broadcast from one half of a pair (SASS
// operand `R.F32`) and a coefficient pair; their results come out in the pair layout
//   yq[0] = (y0, y4), yq[1] = (y2, y6), yq[2] = (y1, y3), yq[3] = (y5, y7)
// which the horizontal inverse reads back.  Every output is the same sum of the same products as
// the scalar network computes, term by term in the same order, so the roundings are unchanged
// wherever the scalar code uses the same association (the parity tests hold either path to the
// oracle).  Matrices: the even/odd symmetry the scalar networks assume (T J = diag((-1)^k) T).
#pragma once

#include "adct_internal.cuh"

namespace adct {

__device__ __forceinline__ float2 pk(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 padd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 psub(float2 a, float2 b) { return __fadd2_rn(a, pk(-b.x, -b.y)); }
__device__ __forceinline__ float2 pswap(float2 a) { return pk(a.y, a.x); }

// c x + acc with c the same in both lanes (compile-time 0 / +-1 fold for constant matrices)
template <class M>
__device__ __forceinline__ float2 pfmac(float c, float2 x, float2 acc) {
  if (M::kConst) {
    if (c == 0.0f) return acc;
    if (c == 1.0f) return padd(acc, x);
    if (c == -1.0f) return psub(acc, x);
  }
  return __ffma2_rn(pk(c, c), x, acc);
}
// (ca, cb) s + acc for a scalar s broadcast to both lanes
template <class M>
__device__ __forceinline__ float2 pfmac2(float ca, float cb, float s, float2 acc) {
  if (M::kConst && ca == cb) return pfmac<M>(ca, pk(s, s), acc);
  return __ffma2_rn(pk(ca, cb), pk(s, s), acc);
}
// sum over i in MASK of c(i) x[i] (vector x, broadcast coefficients)
template <class M, int N, uint32_t MASK, class C>
__device__ __forceinline__ float2 plsum(C c, const float2* x) {
  float2 acc = pk(0.0f, 0.0f);
  bool first = true;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    if (!((MASK >> i) & 1u)) continue;
    const float ci = c(i);
    if (M::kConst && ci == 0.0f) continue;
    if (first) {
      acc = (M::kConst && ci == 1.0f) ? x[i] : ((M::kConst && ci == -1.0f) ? pk(-x[i].x, -x[i].y) : __fmul2_rn(pk(ci, ci), x[i]));
      first = false;
    } else {
      acc = pfmac<M>(ci, x[i], acc);
    }
  }
  return acc;
}
// sum over l in MASK of (ca(l), cb(l)) s[l] (scalar inputs broadcast, coefficient pairs)
template <class M, uint32_t MASK, class CA, class CB>
__device__ __forceinline__ float2 plsum2(CA ca, CB cb, const float* s) {
  float2 acc = pk(0.0f, 0.0f);
  bool first = true;
#pragma unroll
  for (int l = 0; l < 8; ++l) {
    if (!((MASK >> l) & 1u)) continue;
    const float a = ca(l), b = cb(l);
    if (M::kConst && a == 0.0f && b == 0.0f) continue;
    if (first) {
      acc = (M::kConst && a == 1.0f && b == 1.0f) ? pk(s[l], s[l]) : __fmul2_rn(pk(a, b), pk(s[l], s[l]));
      first = false;
    } else {
      acc = pfmac2<M>(a, b, s[l], acc);
    }
  }
  return acc;
}

// ---- vertical passes (column pairs) ----------------------------------------------------------
// y = F x, the structure of fwd8 / fwd8_st
template <class M>
__device__ __forceinline__ void fwd8p(const M& m, const float2* x, float2* y) {
  float2 s[4], t[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    s[i] = padd(x[i], x[7 - i]);
    t[i] = psub(x[i], x[7 - i]);
  }
  const float2 av[2] = {padd(s[0], s[3]), padd(s[1], s[2])};
  const float2 bv[2] = {psub(s[0], s[3]), psub(s[1], s[2])};
  y[0] = plsum<M, 2, 0x3u>([&](int i) { return m.f(0, i); }, av);
  y[4] = plsum<M, 2, 0x3u>([&](int i) { return m.f(4, i); }, av);
  y[2] = plsum<M, 2, 0x3u>([&](int i) { return m.f(2, i); }, bv);
  y[6] = plsum<M, 2, 0x3u>([&](int i) { return m.f(6, i); }, bv);
  y[1] = plsum<M, 4, 0xfu>([&](int i) { return m.f(1, i); }, t);
  y[3] = plsum<M, 4, 0xfu>([&](int i) { return m.f(3, i); }, t);
  y[5] = plsum<M, 4, 0xfu>([&](int i) { return m.f(5, i); }, t);
  y[7] = plsum<M, 4, 0xfu>([&](int i) { return m.f(7, i); }, t);
}
// x = H y (all inputs present), the structure of inv8 / inv8_e with the ee/eo butterfly
template <class M>
__device__ __forceinline__ void inv8p(const M& m, const float2* y, float2* x) {
  float2 ee[2], eo[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    ee[i] = plsum<M, 8, 0x11u>([&](int k) { return m.h(i, k); }, y);
    eo[i] = plsum<M, 8, 0x44u>([&](int k) { return m.h(i, k); }, y);
  }
  const float2 e[4] = {padd(ee[0], eo[0]), padd(ee[1], eo[1]), psub(ee[1], eo[1]), psub(ee[0], eo[0])};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 o = plsum<M, 8, 0xaau>([&](int k) { return m.h(i, k); }, y);
    x[i] = padd(e[i], o);
    x[7 - i] = psub(e[i], o);
  }
}

// ---- horizontal passes (one row: 4 column pairs <-> the yq pair layout) ----------------------
template <class M>
__device__ __forceinline__ void fwd8_row(const M& m, const float2* p, float2* yq) {
  // (s0, s1) = (v0 + v7, v1 + v6), (s2, s3) = (v2 + v5, v3 + v4); t likewise with minus
  const float2 s01 = padd(p[0], pswap(p[3])), s23 = padd(p[1], pswap(p[2]));
  const float2 t01 = psub(p[0], pswap(p[3])), t23 = psub(p[1], pswap(p[2]));
  const float2 a = padd(s01, pswap(s23));  // (s0 + s3, s1 + s2)
  const float2 b = psub(s01, pswap(s23));  // (s0 - s3, s1 - s2)
  const float av[2] = {a.x, a.y}, bv[2] = {b.x, b.y}, tv[4] = {t01.x, t01.y, t23.x, t23.y};
  yq[0] = plsum2<M, 0x3u>([&](int i) { return m.f(0, i); }, [&](int i) { return m.f(4, i); }, av);
  yq[1] = plsum2<M, 0x3u>([&](int i) { return m.f(2, i); }, [&](int i) { return m.f(6, i); }, bv);
  yq[2] = plsum2<M, 0xfu>([&](int i) { return m.f(1, i); }, [&](int i) { return m.f(3, i); }, tv);
  yq[3] = plsum2<M, 0xfu>([&](int i) { return m.f(5, i); }, [&](int i) { return m.f(7, i); }, tv);
}
template <class M>
__device__ __forceinline__ void inv8_row(const M& m, const float2* yq, float2* q) {
  float z[8];
  z[0] = yq[0].x; z[4] = yq[0].y; z[2] = yq[1].x; z[6] = yq[1].y;
  z[1] = yq[2].x; z[3] = yq[2].y; z[5] = yq[3].x; z[7] = yq[3].y;
  // (ee0, ee1) over z0, z4; (eo0, eo1) over z2, z6; e01 = ee + eo, (e3, e2) = ee - eo
  const float2 ee = plsum2<M, 0x11u>([&](int l) { return m.h(0, l); }, [&](int l) { return m.h(1, l); }, z);
  const float2 eo = plsum2<M, 0x44u>([&](int l) { return m.h(0, l); }, [&](int l) { return m.h(1, l); }, z);
  const float2 e01 = padd(ee, eo), e32 = psub(ee, eo);
  const float2 o01 = plsum2<M, 0xaau>([&](int l) { return m.h(0, l); }, [&](int l) { return m.h(1, l); }, z);
  const float2 o23 = plsum2<M, 0xaau>([&](int l) { return m.h(2, l); }, [&](int l) { return m.h(3, l); }, z);
  const float2 e23 = pswap(e32);
  q[0] = padd(e01, o01);         // (x0, x1)
  q[1] = padd(e23, o23);         // (x2, x3)
  q[2] = pswap(psub(e23, o23));  // (x4, x5) = (e3 - o3, e2 - o2)
  q[3] = pswap(psub(e01, o01));  // (x6, x7) = (e1 - o1, e0 - o0)
}

// yq pair slot q holds raster columns (yq_col(q, 0), yq_col(q, 1)) of a row
__host__ __device__ constexpr int yq_col(int q, int h) {
  return q == 0 ? (h ? 4 : 0) : q == 1 ? (h ? 6 : 2) : q == 2 ? (h ? 3 : 1) : (h ? 7 : 5);
}

// forward -> weights (raster w[k*8+l], 0 drops the coefficient; read at compile-time offsets) ->
// inverse, in place: x2[i][c] (column pairs) becomes the reconstruction
template <class M>
__device__ __forceinline__ void roundtrip2d_p(const M& m, float2 (&x2)[8][4], const float* w) {
  float2 p2[8][4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {  // vertical forward, two columns at a time
    float2 col[8], out[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) col[i] = x2[i][c];
    fwd8p(m, col, out);
#pragma unroll
    for (int k = 0; k < 8; ++k) p2[k][c] = out[k];
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {  // horizontal forward, weights, horizontal inverse per row
    float2 yq[4];
    fwd8_row(m, p2[k], yq);
#pragma unroll
    for (int q = 0; q < 4; ++q) yq[q] = __fmul2_rn(yq[q], pk(w[k * 8 + yq_col(q, 0)], w[k * 8 + yq_col(q, 1)]));
    inv8_row(m, yq, p2[k]);
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {  // vertical inverse
    float2 col[8], out[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) col[k] = p2[k][c];
    inv8p(m, col, out);
#pragma unroll
    for (int i = 0; i < 8; ++i) x2[i][c] = out[i];
  }
}

}  // namespace adct
