// tc_lat.cu — latency of a tcgen05.mma batch (issue -> commit -> mbarrier wait), standalone probe.
// One CTA of 128 threads; thread 0 issues NK MMAs (M = 128, N, K = 16, kind::f16) with A in TMEM
// (TS) or shared memory (SS), commits to an mbarrier and waits; clock64 around each batch.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probes/tc_lat probes/tc_lat.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46);
}

template <int N, bool TS, int NK>
__global__ void lat(long long* out, int reps) {
  __shared__ __align__(1024) uint8_t sA[128 * 64 * 2];
  __shared__ __align__(1024) uint8_t sB[160 * 64 * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x;
  for (int i = t; i < (int)sizeof(sA) / 4; i += blockDim.x) ((uint32_t*)sA)[i] = 0x00010001u;
  for (int i = t; i < (int)sizeof(sB) / 4; i += blockDim.x) ((uint32_t*)sB)[i] = 0x3c003c00u;
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  if (t == 0) {
    uint32_t ph = 0;
    long long tot = 0, mn = 1ll << 60;
    for (int r = 0; r < reps; ++r) {
      const long long c0 = clock64();
#pragma unroll
      for (int kk = 0; kk < NK; ++kk) {
        const uint64_t bd = sdesc(smem_u32(sB) + (kk & 3) * 256, 128, 1024);
        if (TS) {
          asm volatile(
              "{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(tm),
              "r"(tm + 400 + 8 * (kk & 3)), "l"(bd), "r"(idesc), "r"(kk));
        } else {
          const uint64_t ad = sdesc(smem_u32(sA) + (kk & 3) * 256, 128, 1024);
          asm volatile(
              "{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(tm),
              "l"(ad), "l"(bd), "r"(idesc), "r"(kk));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&bar)));
      asm volatile(
          "{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(smem_u32(&bar)),
          "r"(ph));
      ph ^= 1;
      const long long c1 = clock64();
      if (r > 0) {
        tot += c1 - c0;
        if (c1 - c0 < mn) mn = c1 - c0;
      }
    }
    out[0] = tot / (reps - 1);
    out[1] = mn;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, bool TS, int NK>
void run(long long* d) {
  lat<N, TS, NK><<<1, 128>>>(d, 50);
  cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%s N=%3d NK=%d: mean %lld cycles, min %lld cycles per batch (%s)\n", TS ? "TS" : "SS", N, NK, h[0], h[1],
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  run<16, true, 1>(d);
  run<16, true, 4>(d);
  run<80, true, 1>(d);
  run<80, true, 4>(d);
  run<80, true, 8>(d);
  run<80, false, 4>(d);
  run<64, true, 4>(d);
  run<128, true, 4>(d);
  run<144, true, 4>(d);
  run<144, false, 4>(d);
  return 0;
}
