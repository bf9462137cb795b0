// i8_probe.cu — standalone check of the kind::i8 tensor-core path (not part of the library):
//   * a 4-D TMA tensor map over a u8 image with NON-monotonic strides {W, 128, H*W} for the
//     dims {128 bytes, rows, 128-byte column chunks, images}: a box {128, 8, 16, 1} lands in
//     shared memory as [chunk][row][128 B], which IS the canonical K-major no-swizzle layout of
//     A = [pair of blocks p][k = 16 i + c] (u8), with LBO = 128 (k chunks = pixel rows i) and
//     SBO = 1024 (8-pair groups = 128-byte chunks); row p of A = both blocks of pair p;
//   * B = [N = 160][K = 128] s8 in shared memory (K-major), D = A B^T exact in s32 TMEM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probes/i8_probe probes/i8_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int W = 2048, H = 16, NIMG = 2, NOUT = 160, KB = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46);
}

// idesc kind::i8: D s32 (2 << 4), A u8 (0 << 7), B s8 (1 << 10), K-major, N >> 3 << 17, M >> 4 << 24
constexpr uint32_t kIdesc = (2u << 4) | (1u << 10) | ((uint32_t)(NOUT >> 3) << 17) | (8u << 24);

__global__ void probe(const __grid_constant__ CUtensorMap map, const int8_t* __restrict__ b, int32_t* __restrict__ out,
                      int band, int img) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;               // 16 KB
  uint8_t* sB = sm + 16384;       // 160 x 128 = 20 KB
  __shared__ __align__(8) uint64_t bar, mbar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, w = t >> 5;
  for (int i = t; i < NOUT * KB; i += blockDim.x) {
    const int n = i / KB, k = i % KB;
    sB[(n / 8) * 1024 + (k / 16) * 128 + (n % 8) * 16 + (k % 16)] = (uint8_t)b[i];
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (t == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(16384));
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(smem_u32(sA)),
        "l"(&map), "r"(0), "r"(band * 8), "r"(0), "r"(img), "r"(smem_u32(&bar))
        : "memory");
    asm volatile("{.reg .pred p; W1: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W1;}" ::"r"(
        smem_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int kk = 0; kk < KB / 32; ++kk) {
      const uint64_t ad = sdesc(smem_u32(sA) + kk * 256, 128, 1024);
      const uint64_t bd = sdesc(smem_u32(sB) + kk * 256, 128, 1024);
      asm volatile(
          "{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}" ::"r"(tm),
          "l"(ad), "l"(bd), "r"(kIdesc), "r"(kk));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&mbar)));
  }
  asm volatile("{.reg .pred p; W2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W2;}" ::"r"(
      smem_u32(&mbar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t lq = (uint32_t)(32 * w) << 16;
  for (int c0 = 0; c0 < NOUT; c0 += 16) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(tm + lq + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 16; ++i) out[t * NOUT + c0 + i] = (int32_t)r[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

int main() {
  std::vector<uint8_t> img((size_t)NIMG * H * W);
  std::vector<int8_t> b(NOUT * KB);
  srand(11);
  for (auto& v : img) v = (uint8_t)(rand() & 0xff);
  for (int i = 0; i < 64; ++i) img[i] = 255;
  for (auto& v : b) v = (int8_t)((rand() % 9) - 4);
  uint8_t* dimg;
  int8_t* db;
  int32_t* dout;
  cudaMalloc(&dimg, img.size());
  cudaMalloc(&db, b.size());
  cudaMalloc(&dout, 128 * NOUT * 4);
  cudaMemcpy(dimg, img.data(), img.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap map;
  const cuuint64_t dims[4] = {128, H, W / 128, NIMG};
  const cuuint64_t strides[3] = {W, 128, (cuuint64_t)H * W};
  const cuuint32_t box[4] = {128, 8, 16, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, dimg, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("cuTensorMapEncodeTiled (non-monotonic strides): %d\n", (int)cr);
  if (cr != CUDA_SUCCESS) return 1;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 20480);
  int fails = 0;
  std::vector<int32_t> out(128 * NOUT);
  for (int im = 0; im < NIMG; ++im)
    for (int band = 0; band < H / 8; ++band) {
      probe<<<1, 128, 16384 + 20480>>>(map, db, dout, band, im);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("kernel error %s\n", cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
      for (int p = 0; p < 128; ++p)
        for (int n = 0; n < NOUT; ++n) {
          long long s = 0;
          for (int k = 0; k < KB; ++k) {
            const int i = k / 16, c = k % 16;
            s += (long long)img[(size_t)im * H * W + (size_t)(band * 8 + i) * W + 16 * p + c] * b[n * KB + k];
          }
          if (s != out[p * NOUT + n]) {
            if (fails < 5) printf("  img %d band %d pair %d n %d: got %d want %lld\n", im, band, p, n, out[p * NOUT + n], s);
            ++fails;
          }
        }
    }
  printf("i8_probe %s (%d mismatches)\n", fails ? "FAIL" : "PASS", fails);
  return fails != 0;
}
