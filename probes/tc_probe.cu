// tc_probe.cu — standalone check of the tcgen05 building blocks the tensor-core hot kernel uses
// (not part of the library):
//   * u8 samples enter f16 as SUBNORMALS: PRMT puts byte x into the low mantissa bits of an
//     f16 with exponent 0, i.e. the value x * 2^-24 exactly (no bias, one PRMT per two samples);
//   * A (128 rows x K=64 f16) written by each thread into its own TMEM lane with tcgen05.st
//     (TS form) or into shared memory in the canonical K-major no-swizzle layout (SS form);
//   * B (N=80 x K=64 f16, small integers) in shared memory, K-major, no swizzle;
//   * D = A B^T in fp32 TMEM accumulators, read back with tcgen05.ld.
// Every product is an integer times 2^-24 and every partial sum an integer below 2^24 (times
// 2^-24), so D must equal the exact integer product scaled by 2^-24.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probes/tc_probe probes/tc_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);  \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

constexpr int M = 128, N = 80, K = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm_100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

// kind::f16 instruction descriptor: D f32, A/B f16, both K-major, N>>3 at bit 17, M>>4 at bit 24
constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);

template <bool TS>
__global__ void probe(const uint8_t* __restrict__ x, const uint16_t* __restrict__ b, float* __restrict__ out,
                      int sub) {
  __shared__ __align__(1024) uint8_t sA[M * K * 2];
  __shared__ __align__(1024) uint8_t sB[N * K * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, w = t >> 5;
  // B: core matrix (n/8, k/8) at (n/8)*1024 + (k/8)*128, row n%8 at 16 B, element k%8 at 2 B
  for (int i = t; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    *(uint16_t*)(sB + (n / 8) * 1024 + (k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2) = b[i];
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  const uint32_t lane_base = (uint32_t)(32 * (w & 3)) << 16;
  const uint32_t a_col = 80, d_col = 0;  // A in columns 80..111, D in 0..79
  // this thread's row m = t: 64 samples -> 32 f16x2 words
  uint32_t a[32];
  const uint32_t* xr = reinterpret_cast<const uint32_t*>(x + t * K);
  for (int q = 0; q < 16; ++q) {
    const uint32_t v = xr[q];
    if (sub) {  // subnormal: x * 2^-24
      asm("prmt.b32 %0, %1, 0, 0x4140;" : "=r"(a[2 * q]) : "r"(v));
      asm("prmt.b32 %0, %1, 0, 0x4342;" : "=r"(a[2 * q + 1]) : "r"(v));
    } else {  // normal with bias: 1024 + x
      asm("prmt.b32 %0, %1, %2, 0x4140;" : "=r"(a[2 * q]) : "r"(v), "r"(0x64646464u));
      asm("prmt.b32 %0, %1, %2, 0x4342;" : "=r"(a[2 * q + 1]) : "r"(v), "r"(0x64646464u));
    }
  }
  if (TS) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tm + lane_base + a_col),
        "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]), "r"(a[8]),
        "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(a[12]), "r"(a[13]), "r"(a[14]), "r"(a[15]), "r"(a[16]),
        "r"(a[17]), "r"(a[18]), "r"(a[19]), "r"(a[20]), "r"(a[21]), "r"(a[22]), "r"(a[23]), "r"(a[24]),
        "r"(a[25]), "r"(a[26]), "r"(a[27]), "r"(a[28]), "r"(a[29]), "r"(a[30]), "r"(a[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  } else {
    // A: core matrix (m/8, k/8) at (m/8)*1024 + (k/8)*128, row m%8 at 16 B
    for (int c = 0; c < 8; ++c) {
      uint4 v = make_uint4(a[4 * c], a[4 * c + 1], a[4 * c + 2], a[4 * c + 3]);
      *(uint4*)(sA + (t / 8) * 1024 + c * 128 + (t % 8) * 16) = v;
    }
    asm volatile("fence.proxy.async.shared::cta;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (t == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int kk = 0; kk < K / 16; ++kk) {
      const uint64_t bd = sdesc(smem_u32(sB) + kk * 256, 128, 1024);
      const uint32_t acc = kk > 0;
      if (TS) {
        asm volatile(
            "{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(tm + d_col),
            "r"(tm + a_col + kk * 8), "l"(bd), "r"(kIdesc), "r"(acc));
      } else {
        const uint64_t ad = sdesc(smem_u32(sA) + kk * 256, 128, 1024);
        asm volatile(
            "{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(tm + d_col),
            "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
  }
  asm volatile(
      "{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(tm + lane_base + d_col + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 16; ++i) out[t * N + c0 + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

static uint16_t f16_of_int(int v) {  // small integers |v| <= 2048, exact
  if (v == 0) return 0;
  uint16_t s = v < 0 ? 0x8000 : 0;
  int a = v < 0 ? -v : v;
  int e = 0;
  while ((a >> e) > 1) ++e;
  const int mant = (a << (10 - e)) & 0x3ff;
  return s | (uint16_t)((e + 15) << 10) | (uint16_t)mant;
}

int main() {
  std::vector<uint8_t> hx(M * K);
  std::vector<int> hbi(N * K);
  std::vector<uint16_t> hb(N * K);
  srand(7);
  for (int i = 0; i < M * K; ++i) hx[i] = (i < 2 * K) ? 255 : (uint8_t)(rand() & 0xff);
  for (int i = 0; i < N * K; ++i) {
    const int v = (rand() % 9) - 4;  // {-4..4}: the entries of T1 (x) T1
    hbi[i] = v;
    hb[i] = f16_of_int(v);
  }
  uint8_t* dx;
  uint16_t* db;
  float* dout;
  CK(cudaMalloc(&dx, M * K));
  CK(cudaMalloc(&db, N * K * 2));
  CK(cudaMalloc(&dout, M * N * 4));
  CK(cudaMemcpy(dx, hx.data(), M * K, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, hb.data(), N * K * 2, cudaMemcpyHostToDevice));
  std::vector<float> out(M * N);
  int fails_total = 0;
  for (int mode = 0; mode < 4; ++mode) {
    const bool ts = mode < 2;
    const int sub = (mode & 1) == 0;
    CK(cudaMemset(dout, 0xff, M * N * 4));
    if (ts) probe<true><<<1, 128>>>(dx, db, dout, sub);
    else probe<false><<<1, 128>>>(dx, db, dout, sub);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out.data(), dout, M * N * 4, cudaMemcpyDeviceToHost));
    int fails = 0;
    double maxerr = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        long long s = 0;
        for (int k = 0; k < K; ++k) s += (long long)((sub ? 0 : 1024) + hx[m * K + k]) * hbi[n * K + k];
        const double ref = sub ? (double)s * 0x1p-24 : (double)s;
        const double e = fabs((double)out[m * N + n] - ref);
        if (e > maxerr) maxerr = e;
        if (e != 0.0) {
          if (fails < 5) printf("  mode %d m=%d n=%d got %.10g want %.10g\n", mode, m, n, out[m * N + n], ref);
          ++fails;
        }
      }
    printf("mode %s %s: %d mismatches of %d, max abs err %.3g\n", ts ? "TS(A in TMEM)" : "SS(A in smem)",
           sub ? "subnormal-u8" : "biased-1024", fails, M * N, maxerr);
    fails_total += fails;
  }
  printf("tc_probe %s\n", fails_total == 0 ? "PASS" : "FAIL");
  return fails_total != 0;
}
