// greedy.cu — next row f3: the greedy angle search of §3 (Eq. 5-6; Fig. 2
// "abmApprox") that produces T1 and T2 (§4.1), as a GPU workload.
//
// For every permutation sequence (one CTA each) the rows are placed greedily: row p(k) is the
// vector of D = P^8 with the largest cosine to row p(k) of C (reading A21: the smallest angle)
// among the non-zero vectors orthogonal to every row already placed (A23), ties to the
// earliest vector of the lexicographic enumeration (A22); an order that runs out of
// candidates is reported infeasible (A24).
//
//  - digits_kernel: the |P|^8 vectors as packed int8 (8 bytes each, L2-resident);
//  - score_kernel:  s_k(d) = <c_k, d> / (|d| |c_k|) for every row k and vector d, in fp64 with
//                   explicit round-to-nearest operations in the oracle's order (no contraction),
//                   so both sides take every argmax decision on identical values;
//  - search_kernel: per step, each thread scans a strided share of D, tests orthogonality with
//                   the placed rows by DP4A on the packed digits, and keeps the best
//                   (score, -index) and how many candidates share that score; the CTA
//                   reduction of that total order is deterministic, and the tie counts of
//                   equal scores add up, so exact ties (A22) are reported per sequence.
#include <cmath>
#include <utility>

#include "adct_host.h"

namespace adct {
namespace {

constexpr int kGrNT = 512;

__global__ void digits_kernel(int8_t* __restrict__ digits, int32_t n_entries, uint32_t n_vec, int4 e0, int4 e1) {
  const int32_t ent[8] = {e0.x, e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_vec; i += gridDim.x * blockDim.x) {
    uint32_t v = i;
    int8_t d[8];
#pragma unroll
    for (int j = 7; j >= 0; --j) {  // first coordinate most significant
      d[j] = (int8_t)ent[v % (uint32_t)n_entries];
      v /= (uint32_t)n_entries;
    }
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      lo |= (uint32_t)(uint8_t)d[j] << (8 * j);
      hi |= (uint32_t)(uint8_t)d[4 + j] << (8 * j);
    }
    reinterpret_cast<uint2*>(digits)[i] = make_uint2(lo, hi);
  }
}

struct CRows {
  double c[64];
};

__global__ void score_kernel(const int8_t* __restrict__ digits, uint32_t n_vec, CRows cr, double* __restrict__ score) {
  __shared__ double nc[8];
  if (threadIdx.x < 8) {
    double s = 0.0;
    for (int j = 0; j < 8; ++j) s = __dadd_rn(s, __dmul_rn(cr.c[threadIdx.x * 8 + j], cr.c[threadIdx.x * 8 + j]));
    nc[threadIdx.x] = sqrt(s);
  }
  __syncthreads();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_vec; i += gridDim.x * blockDim.x) {
    const uint2 w = reinterpret_cast<const uint2*>(digits)[i];
    double d[8];
    int32_t n2 = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int32_t v = (int32_t)(int8_t)((j < 4 ? w.x : w.y) >> (8 * (j & 3)));
      d[j] = (double)v;
      n2 += v * v;
    }
    const double nd = sqrt((double)n2);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double dot = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) dot = __dadd_rn(dot, __dmul_rn(cr.c[k * 8 + j], d[j]));
      score[(size_t)k * n_vec + i] = n2 == 0 ? -INFINITY : __ddiv_rn(dot, __dmul_rn(nd, nc[k]));
    }
  }
}

struct Fixed {
  int32_t t[64];
};

__device__ __forceinline__ bool rows_placed_before(const int32_t*, int k, uint32_t, const int32_t* orders, int order,
                                                   int32_t n_free, int step) {
  for (int q = 0; q < step; ++q)
    if (orders[(size_t)order * n_free + q] == k) return true;
  return false;
}

__global__ void __launch_bounds__(kGrNT) search_kernel(const int8_t* __restrict__ digits, const double* __restrict__ score,
                                                      uint32_t n_vec, Fixed fx, uint32_t fixed_mask,
                                                      const int32_t* __restrict__ orders, int32_t n_free,
                                                      int32_t* __restrict__ out, int32_t* __restrict__ status,
                                                      int32_t* __restrict__ ties) {
  __shared__ uint2 placed[8];
  __shared__ double best_s[kGrNT / 32];
  __shared__ uint32_t best_i[kGrNT / 32];
  __shared__ uint32_t best_n[kGrNT / 32];
  __shared__ int32_t tie[4];  // steps with a tie, first tied row, its tie size, largest tie size
  __shared__ int32_t rows[64];
  __shared__ int n_placed;
  const int order = blockIdx.x;
  if (threadIdx.x == 0) {
    int np = 0;
    for (int k = 0; k < 8; ++k) {
      uint32_t lo = 0, hi = 0;
      for (int j = 0; j < 8; ++j) {
        const int32_t v = (fixed_mask >> k) & 1u ? fx.t[k * 8 + j] : 0;
        rows[k * 8 + j] = v;
        if (j < 4) lo |= (uint32_t)(uint8_t)(int8_t)v << (8 * j);
        else hi |= (uint32_t)(uint8_t)(int8_t)v << (8 * (j - 4));
      }
      if ((fixed_mask >> k) & 1u) placed[np++] = make_uint2(lo, hi);
    }
    n_placed = np;
    tie[0] = 0;
    tie[1] = -1;
    tie[2] = 0;
    tie[3] = 0;
  }
  __syncthreads();
  int32_t st = 0;
  for (int step = 0; step < n_free; ++step) {
    const int k = orders[(size_t)order * n_free + step];
    if (k < 0 || k > 7 || ((fixed_mask >> k) & 1u) || rows_placed_before(rows, k, fixed_mask, orders, order, n_free, step)) {
      st = 2;  // not a row index, a fixed row, or a row already placed: invalid sequence
      break;
    }
    const int np = n_placed;
    uint2 pr[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) pr[p] = p < np ? placed[p] : make_uint2(0u, 0u);
    double bs = -INFINITY;
    uint32_t bi = 0xffffffffu, bn = 0;  // best score, its first index, candidates at that score
    const double* sk = score + (size_t)k * n_vec;
    for (uint32_t i = threadIdx.x; i < n_vec; i += kGrNT) {
      const uint2 w = reinterpret_cast<const uint2*>(digits)[i];
      if ((w.x | w.y) == 0u) continue;  // the zero vector has no angle
      bool orth = true;
#pragma unroll
      for (int p = 0; p < 8; ++p)
        if (p < np) orth &= (__dp4a((int)w.x, (int)pr[p].x, __dp4a((int)w.y, (int)pr[p].y, 0)) == 0);
      if (!orth) continue;
      const double s = sk[i];
      if (s >= bs) {  // one compare on the common path (s < bs); ties are rare
        if (s > bs) {   // strided scan visits i in increasing order: the first maximum is kept
          bs = s;
          bi = i;
          bn = 1;
        } else {
          ++bn;
        }
      }
    }
    // CTA argmax of (score, -index): a total order, so the reduction order does not matter
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double os = __shfl_xor_sync(0xffffffffu, bs, o);
      const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      const uint32_t on = __shfl_xor_sync(0xffffffffu, bn, o);
      if (os > bs) {
        bs = os;
        bi = oi;
        bn = on;
      } else if (os == bs) {
        bi = oi < bi ? oi : bi;
        bn += on;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      best_s[threadIdx.x >> 5] = bs;
      best_i[threadIdx.x >> 5] = bi;
      best_n[threadIdx.x >> 5] = bn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = best_s[0];
      uint32_t idx = best_i[0], cnt = best_n[0];
      for (int q = 1; q < kGrNT / 32; ++q)
        if (best_s[q] > s) {
          s = best_s[q];
          idx = best_i[q];
          cnt = best_n[q];
        } else if (best_s[q] == s) {
          idx = best_i[q] < idx ? best_i[q] : idx;
          cnt += best_n[q];
        }
      if (idx != 0xffffffffu && cnt > 1) {  // an exact tie: the earliest vector was taken (A22)
        if (tie[0] == 0) {
          tie[1] = k;
          tie[2] = (int32_t)cnt;
        }
        ++tie[0];
        tie[3] = (int32_t)cnt > tie[3] ? (int32_t)cnt : tie[3];
      }
      if (idx == 0xffffffffu) {
        n_placed = -1;  // infeasible
      } else {
        const uint2 w = reinterpret_cast<const uint2*>(digits)[idx];
        placed[n_placed] = w;
        n_placed = n_placed + 1;
        for (int j = 0; j < 8; ++j) rows[k * 8 + j] = (int32_t)(int8_t)((j < 4 ? w.x : w.y) >> (8 * (j & 3)));
      }
    }
    __syncthreads();
    if (n_placed < 0) {
      st = 1;
      break;
    }
  }
  for (int t = threadIdx.x; t < 64; t += kGrNT) out[(size_t)order * 64 + t] = st ? 0 : rows[t];
  // status: 0 ok, 1 infeasible (no orthogonal candidate left), 2 invalid sequence
  if (threadIdx.x == 0) status[order] = st;
  if (ties && threadIdx.x < 4) ties[(size_t)order * 4 + threadIdx.x] = tie[threadIdx.x];
}

uint32_t ipow8(int32_t n) {
  uint32_t v = 1;
  for (int i = 0; i < 8; ++i) v *= (uint32_t)n;
  return v;
}

}  // namespace
}  // namespace adct

using namespace adct;

extern "C" {

size_t adct_greedy_workspace_bytes(int32_t n_entries) {
  if (n_entries < 1 || n_entries > 8) return 0;
  const size_t n = ipow8(n_entries);
  return n * 8 + 8 * n * sizeof(double) + 256;
}

adct_status adct_greedy_search(const double c[64], const int32_t* entries, int32_t n_entries, const int32_t fixed[64],
                               uint32_t fixed_mask, const int32_t* orders, int32_t n_orders, int32_t* out,
                               int32_t* status, int32_t* ties, void* workspace, size_t workspace_bytes,
                               void* stream) {
  if (!c || !entries || !orders || !out || !status || (fixed_mask && !fixed)) return ADCT_E_INVALID_ARGUMENT;
  if (n_entries < 1 || n_entries > 8 || n_orders < 0 || fixed_mask > 0xffu) return ADCT_E_INVALID_ARGUMENT;
  int32_t ent[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < n_entries; ++i) {
    if (entries[i] < -127 || entries[i] > 127) return ADCT_E_INVALID_ARGUMENT;
    ent[i] = entries[i];
  }
  for (int i = 1; i < n_entries; ++i)  // reading A22: ascending entry order, no duplicates
    for (int j = i; j > 0 && ent[j] < ent[j - 1]; --j) std::swap(ent[j], ent[j - 1]);
  for (int i = 1; i < n_entries; ++i)
    if (ent[i] == ent[i - 1]) return ADCT_E_INVALID_ARGUMENT;
  if (fixed_mask)
    for (int t = 0; t < 64; ++t)
      if (((fixed_mask >> (t / 8)) & 1u) && (fixed[t] < -127 || fixed[t] > 127)) return ADCT_E_INVALID_ARGUMENT;
  if (!workspace || workspace_bytes < adct_greedy_workspace_bytes(n_entries)) return ADCT_E_WORKSPACE;
  if (n_orders == 0) return ADCT_OK;
  const int32_t n_free = 8 - __builtin_popcount(fixed_mask);
  const uint32_t n_vec = ipow8(n_entries);
  cudaStream_t st = (cudaStream_t)stream;
  int8_t* digits = (int8_t*)workspace;
  double* score = (double*)((char*)workspace + (((size_t)n_vec * 8 + 255) / 256) * 256);
  const unsigned g1 = (unsigned)((n_vec + 255) / 256 < 4096 ? (n_vec + 255) / 256 : 4096);
  digits_kernel<<<g1, 256, 0, st>>>(digits, n_entries, n_vec, make_int4(ent[0], ent[1], ent[2], ent[3]),
                                    make_int4(ent[4], ent[5], ent[6], ent[7]));
  CRows cr;
  for (int t = 0; t < 64; ++t) cr.c[t] = c[t];
  score_kernel<<<g1, 256, 0, st>>>(digits, n_vec, cr, score);
  Fixed fx;
  for (int t = 0; t < 64; ++t) fx.t[t] = fixed_mask ? fixed[t] : 0;
  search_kernel<<<(unsigned)n_orders, kGrNT, 0, st>>>(digits, score, n_vec, fx, fixed_mask, orders, n_free, out, status,
                                                     ties);
  count_launch(3);
  return launch_status();
}

}  // extern "C"
