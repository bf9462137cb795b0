// tc_contend.cu — does TMEM load/store traffic from other warps slow a tcgen05.mma batch down?
// One CTA of 512 threads.  Warp 0 lane 0 times batches of 4 MMAs (M = 128, N = 80, K = 16,
// kind::f16, A in TMEM) + commit + wait; warps 1..15 meanwhile run a loop of tcgen05.ld x32
// (mode 1), tcgen05.st x16 (mode 2), both (mode 3) or nothing (mode 0) on other TMEM columns.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probes/tc_contend probes/tc_contend.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46);
}

__global__ void contend(long long* out, int mode, int reps, int iw, int nn, int smsp_mask) {
  __shared__ __align__(1024) uint8_t sB[160 * 64 * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  for (int i = t; i < (int)sizeof(sB) / 4; i += blockDim.x) ((uint32_t*)sB)[i] = 0x3c003c00u;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(nn >> 3) << 17) | (8u << 24);  // M = 128
  if (w == iw) {
    if (lane == 0) {
      uint32_t ph = 0;
      long long tot = 0, tiss = 0;
      for (int r = 0; r < reps; ++r) {
        const long long c0 = clock64();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bd = sdesc(smem_u32(sB) + kk * 256, 128, 1024);
          asm volatile(
              "{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(tm),
              "r"(tm + 480 + 8 * kk), "l"(bd), "r"(idesc), "r"(kk));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&bar)));
        const long long ci = clock64();
        if (r > 4) tiss += ci - c0;
        asm volatile(
            "{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(
                smem_u32(&bar)),
            "r"(ph));
        ph ^= 1;
        if (r > 4) tot += clock64() - c0;
      }
      out[0] = tot / (reps - 5);
      out[3] = tiss / (reps - 5);
      stop = 1;
    }
    __syncwarp();
  } else {
    const uint32_t lq = (uint32_t)(32 * (w & 3)) << 16;
    const uint32_t col = 96 + 96 * ((w >> 2) % 4);  // 96..383: not the MMA's columns
    long long n = 0;
    const long long c0 = clock64();
    const bool active = (smsp_mask >> (w & 3)) & 1;
    while (!stop && active) {
      if (mode & 1) {
        uint32_t r[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
              "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
              "=r"(r[30]), "=r"(r[31])
            : "r"(tm + lq + col));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t x = 0;
        for (int i = 0; i < 32; ++i) x ^= r[i];
        if (x == 0x12345678u) out[2] = x;
      }
      if (mode & 2) {
        uint32_t v = (uint32_t)n;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                tm + lq + col + 32),
            "r"(v));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      if (mode & 4) {  // FP32 work only, no TMEM traffic
        float a0 = (float)n, a1 = a0 + 1.f, a2 = a0 + 2.f, a3 = a0 + 3.f;
#pragma unroll 16
        for (int i = 0; i < 256; ++i) {
          a0 = fmaf(a0, 1.0001f, 0.5f); a1 = fmaf(a1, 0.9999f, 0.25f);
          a2 = fmaf(a2, 1.0002f, 0.125f); a3 = fmaf(a3, 0.9998f, 0.0625f);
        }
        if (a0 + a1 + a2 + a3 == 1.2345f) out[2] = 1;
      }
      if (mode & 8) {  // integer ALU work only
        uint32_t a0 = (uint32_t)n, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
#pragma unroll 16
        for (int i = 0; i < 256; ++i) {
          a0 = (a0 ^ 0x9e37u) + a1; a1 = (a1 ^ 0x79b9u) + a2; a2 = (a2 ^ 0x7f4au) + a3; a3 = (a3 ^ 0x7c15u) + a0;
        }
        if ((a0 ^ a1 ^ a2 ^ a3) == 0x12345u) out[2] = 1;
      }
      if (mode & 16) {  // int -> float conversions only
        float a0 = 0.f, a1 = 0.f;
        uint32_t v = (uint32_t)n;
#pragma unroll 16
        for (int i = 0; i < 256; ++i) {
          a0 += __int2float_rn((int)(v + i)); a1 += __int2float_rn((int)(v ^ i));
        }
        if (a0 + a1 == 1.2345f) out[2] = 1;
      }
      ++n;
      if (mode == 0) break;
    }
    if (t == (iw == 0 ? 32 : 0)) out[1] = (clock64() - c0) / (n ? n : 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 32);
  const int modes[2] = {0, 4};
  const char* names[2] = {"idle", "ffma"};
  const int iw = 15;  // SMSP 3
  for (int nn : {16, 80, 160})
  for (int msk : {0xf, 0x7, 0x8})
  for (int mi = 0; mi < 2; ++mi) {
    const int mode = modes[mi];
    if (mode == 0 && msk != 0xf) continue;
    printf("N=%3d ffma on SMSPs mask %x  ", nn, msk);
    contend<<<1, 512>>>(d, mode, 200, iw, nn, msk);
    cudaDeviceSynchronize();
    long long h[4];
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("background %-10s: MMA batch (4 x N=80) %lld cycles (issue %lld); background loop %lld cycles/iter (%s)\n",
           names[mi], h[0], h[3], h[1], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
