// Box probe: issue throughput of the SASS instructions the
// 8x8 transform path can be built from, and streaming HBM bandwidth.
// Not part of the product; decides FP32-pair vs packed-int16 arithmetic.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probes/pipes probes/pipes.cu
#include <cstdlib>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 2048;

template <int OP>
__global__ void __launch_bounds__(1024) pipe_kernel(const uint32_t* in, uint32_t* out, long long* cyc) {
  uint32_t a0 = in[threadIdx.x & 63], a1 = in[(threadIdx.x + 1) & 63];
  uint32_t r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = in[(threadIdx.x + 7 * i) & 63];
  float2 f2[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) f2[i] = make_float2(__uint_as_float(r[i]) , __uint_as_float(r[(i + 3) & 7]));
  float2 fa = make_float2(__uint_as_float(a0), __uint_as_float(a1));
  float d[8][4], g[8][4];
  uint32_t di[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int u = 0; u < 4; ++u) { d[i][u] = 0.f; g[i][u] = __uint_as_float(r[(i + u) & 7]); di[i][u] = r[u]; }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 16
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(a0), "r"(a1));  // FFMA 3-reg
      if (OP == 1) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, %1;" : "+r"(r[i]) : "r"(a0));   // FFMA imm
      if (OP == 2) asm volatile("add.f32 %0, %0, %1;" : "+r"(r[i]) : "r"(a0));                 // FADD
      if (OP == 3) f2[i] = __ffma2_rn(f2[i], fa, fa);                                          // FFMA2
      if (OP == 4) f2[i] = __fadd2_rn(f2[i], fa);                                              // FADD2
      if (OP == 5) asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(r[i]) : "r"(a0), "r"(a1)); // IADD3
      if (OP == 6) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[i]) : "r"(a0), "r"(a1)); // LOP3
      if (OP == 7) asm volatile("prmt.b32 %0, %0, %1, 0x5140;" : "+r"(r[i]) : "r"(a0));            // PRMT
      if (OP == 8) asm volatile("{.reg .u32 t; shl.b32 t, %0, 1; add.u32 %0, t, %1;}" : "+r"(r[i]) : "r"(a0)); // LEA
      if (OP == 9) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(a0), "r"(a1));    // IMAD
      if (OP == 10) asm volatile("cvt.rn.f32.u32 %0, %0;" : "+r"(r[i]));                          // I2FP
      if (OP == 11) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(a0), "r"(a1)); // HFMA2
      if (OP == 12) {  // FFMA2 + IADD3 interleaved (dual-pipe)
        f2[i] = __ffma2_rn(f2[i], fa, fa);
        asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(r[i]) : "r"(a0), "r"(a1));
      }
      if (OP == 13) {  // FFMA + IADD3 interleaved
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(a0), "r"(a1));
        asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(r[(i + 4) & 7]) : "r"(a0), "r"(a1));
      }
      if (OP == 14) asm volatile("cvt.rn.f32.s32 %0, %0;" : "+r"(r[i]));                         // I2F s32
      if (OP == 15) asm volatile("mul.f32 %0, %0, %1;" : "+r"(r[i]) : "r"(a0));                  // FMUL
      if (OP == 16) f2[i] = __fmul2_rn(f2[i], fa);                                              // FMUL2
      if (OP == 17) asm volatile("fma.rn.f32 %0, %1, %1, %0;" : "+r"(r[i]) : "r"(a0));           // FFMA acc (2 distinct regs)
      if (OP == 18) asm volatile("sub.f32 %0, %1, %0;" : "+r"(r[i]) : "r"(a0));                  // FADD variant
      if (OP == 19) asm volatile("{.reg .b32 t; shr.b32 t, %0, 8; cvt.rn.f32.u8 %0, t;}" : "+r"(r[i]));  // I2F.U8 .B1
      if (OP == 20) {  // I2F.U8 .B1 + FFMA interleaved
        asm volatile("{.reg .b32 t; shr.b32 t, %0, 8; cvt.rn.f32.u8 %0, t;}" : "+r"(r[i]));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(r[(i + 4) & 7]) : "r"(a0), "r"(a1));
      }
      if (OP == 21) asm volatile("{.reg .b32 t; shr.b32 t, %0, 16; cvt.rn.f32.s16 %0, t;}" : "+r"(r[i]));  // I2F.S16 .H1
      if (OP == 22) {  // PRMT + FFMA interleaved
        asm volatile("prmt.b32 %0, %0, %1, 0x5140;" : "+r"(r[i]) : "r"(a0));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(r[(i + 4) & 7]) : "r"(a0), "r"(a1));
      }
      if (OP == 23) {  // FFMA + FADD + I2F.U8 (2:1 FMA-pipe : conversion)
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(r[(i + 4) & 7]) : "r"(a0), "r"(a1));
        asm volatile("add.f32 %0, %0, %1;" : "+r"(r[(i + 2) & 7]) : "r"(a0));
        asm volatile("{.reg .b32 t; shr.b32 t, %0, 8; cvt.rn.f32.u8 %0, t;}" : "+r"(r[i]));
      }
      if (OP == 24) asm volatile("cvt.rn.f32.u8 %0, %0;" : "+r"(r[i]));  // I2F.U8 .B0
      if (OP == 25 || OP == 26)  // HMMA m16n8k16 f16 -> f32 (legacy mma.sync)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3])
                     : "r"(r[i]), "r"(r[(i + 1) & 7]), "r"(a0), "r"(a1), "r"(r[(i + 2) & 7]), "r"(a0));
      if (OP == 27 || OP == 28)  // IMMA m16n8k32 u8 x s8 -> s32
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(di[i][0]), "+r"(di[i][1]), "+r"(di[i][2]), "+r"(di[i][3])
                     : "r"(r[i]), "r"(r[(i + 1) & 7]), "r"(a0), "r"(a1), "r"(r[(i + 2) & 7]), "r"(a0));
      if (OP == 26 || OP == 28) {  // + 4 independent FFMA per MMA
#pragma unroll
        for (int u = 0; u < 4; ++u)
          asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(g[i][u]) : "r"(a0), "r"(a1));
      }
    }
  }
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    acc ^= r[i] ^ __float_as_uint(f2[i].x) ^ __float_as_uint(f2[i].y);
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= __float_as_uint(d[i][u]) ^ __float_as_uint(g[i][u]) ^ di[i][u];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void read_u4(const uint4* __restrict__ p, size_t n, uint32_t* out) {
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride * 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = (i + u * stride < n) ? __ldg(p + i + u * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// thread-owns-an-8x8-u8-block read pattern: 8 x 8-byte rows, warp = 32 adjacent blocks
__global__ void read_blocks_u8(const uint8_t* __restrict__ img, int W, int H, int nimg, uint32_t* out) {
  int bw = W / 8, bh = H / 8;
  long long nb = (long long)bw * bh * nimg;
  uint32_t acc = 0;
  for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (long long)gridDim.x * blockDim.x) {
    long long im = b / ((long long)bw * bh);
    int rem = (int)(b - im * bw * bh);
    int by = rem / bw, bx = rem - by * bw;
    const uint8_t* base = img + im * (long long)W * H + (long long)by * 8 * W + bx * 8;
    uint2 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __ldg(reinterpret_cast<const uint2*>(base + (long long)i * W));
#pragma unroll
    for (int i = 0; i < 8; ++i) acc ^= v[i].x + v[i].y;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

static const char* names[] = {"FFMA(3reg)", "FFMA(imm)", "FADD", "FFMA2", "FADD2", "IADD3", "LOP3", "PRMT", "LEA",
                              "IMAD", "I2FP.U32", "HFMA2", "FFMA2+IADD3", "FFMA+IADD3", "I2F.S32", "FMUL", "FMUL2",
                              "FFMA(acc a*a+d)", "FADD(sub)", "I2F.U8.B1", "I2F.U8.B1+FFMA", "I2F.S16.H1",
                              "PRMT+FFMA", "FFMA+FADD+I2F.U8", "I2F.U8.B0", "HMMA.16816.F32",
                              "HMMA+4FFMA", "IMMA.16832.S32", "IMMA+4FFMA"};

template <int OP>
int run_one(const uint32_t* din, uint32_t* dout, long long* dcyc, int nsm) {
  pipe_kernel<OP><<<nsm, 1024>>>(din, dout, dcyc);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  pipe_kernel<OP><<<nsm, 1024>>>(din, dout, dcyc);
  CK(cudaDeviceSynchronize());
  long long h[1024];
  CK(cudaMemcpy(h, dcyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));
  double mean = 0;
  for (int i = 0; i < nsm; ++i) mean += (double)h[i];
  mean /= nsm;
  int per = (OP == 12 || OP == 13 || OP == 20 || OP == 22) ? 16 : (OP == 23 ? 24 : (OP == 26 || OP == 28) ? 40 : 8);
  double warp_inst = 32.0 * ITERS * per;  // warp-instructions per SM (32 warps)
  printf("%-18s %7.3f warp-inst/clk/SM  (%5.3f per SMSP)\n", names[OP], warp_inst / mean, warp_inst / mean / 4);
  return 0;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s sm_%d%d SMs=%d L2=%d MB smem/SM=%zu KB regs/SM=%d mem=%.1f GB clock=%d kHz memclk=%d kHz bus=%d\n",
         p.name, p.major, p.minor, p.multiProcessorCount, p.l2CacheSize >> 20, p.sharedMemPerMultiprocessor >> 10,
         p.regsPerMultiprocessor, p.totalGlobalMem / 1e9, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  int nsm = p.multiProcessorCount;
  uint32_t hin[64];
  for (int i = 0; i < 64; ++i) hin[i] = 0x3F800000u + i;
  uint32_t *din, *dout;
  long long* dcyc;
  CK(cudaMalloc(&din, 256));
  CK(cudaMalloc(&dout, (size_t)nsm * 1024 * 4));
  CK(cudaMalloc(&dcyc, 1024 * 8));
  CK(cudaMemcpy(din, hin, 256, cudaMemcpyHostToDevice));
  run_one<0>(din, dout, dcyc, nsm);  run_one<1>(din, dout, dcyc, nsm);  run_one<2>(din, dout, dcyc, nsm);
  run_one<3>(din, dout, dcyc, nsm);  run_one<4>(din, dout, dcyc, nsm);  run_one<5>(din, dout, dcyc, nsm);
  run_one<6>(din, dout, dcyc, nsm);  run_one<7>(din, dout, dcyc, nsm);  run_one<8>(din, dout, dcyc, nsm);
  run_one<9>(din, dout, dcyc, nsm);  run_one<10>(din, dout, dcyc, nsm); run_one<11>(din, dout, dcyc, nsm);
  run_one<12>(din, dout, dcyc, nsm); run_one<13>(din, dout, dcyc, nsm); run_one<14>(din, dout, dcyc, nsm);
  run_one<15>(din, dout, dcyc, nsm); run_one<16>(din, dout, dcyc, nsm); run_one<17>(din, dout, dcyc, nsm);
  run_one<18>(din, dout, dcyc, nsm); run_one<19>(din, dout, dcyc, nsm); run_one<20>(din, dout, dcyc, nsm);
  run_one<21>(din, dout, dcyc, nsm); run_one<22>(din, dout, dcyc, nsm); run_one<23>(din, dout, dcyc, nsm);
  run_one<24>(din, dout, dcyc, nsm);
  run_one<25>(din, dout, dcyc, nsm); run_one<26>(din, dout, dcyc, nsm); run_one<27>(din, dout, dcyc, nsm);
  run_one<28>(din, dout, dcyc, nsm);
  if (getenv("PIPES_ONLY")) return 0;

  // streaming read bandwidth
  size_t bytes = (size_t)8 << 30;
  uint8_t* buf;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 1, bytes));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int g = 1; g <= 16; g *= 2) {
    int grid = nsm * g;
    read_u4<<<grid, 512>>>((const uint4*)buf, bytes / 16, dout);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      read_u4<<<grid, 512>>>((const uint4*)buf, bytes / 16, dout);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("read LDG.128 grid=%d x512: %.1f GB/s\n", grid, bytes / best / 1e6);
  }
  // 8x8 u8 block pattern, 4K frames: W=3840 H=2160, nimg = 8GB/8.3MB
  int W = 3840, H = 2160;
  int nimg = (int)(bytes / ((size_t)W * H));
  for (int tpb = 128; tpb <= 512; tpb *= 2) {
    for (int g = 4; g <= 16; g *= 2) {
      int grid = nsm * g;
      read_blocks_u8<<<grid, tpb>>>(buf, W, H, nimg, dout);
      CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        read_blocks_u8<<<grid, tpb>>>(buf, W, H, nimg, dout);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      double b = (double)W * H * nimg;
      printf("read 8x8-u8 blocks (LDG.64 x8) grid=%d x%d: %.1f GB/s  %.1f Gblk/s\n", grid, tpb, b / best / 1e6,
             b / 64 / best / 1e6);
    }
  }
  // copy bandwidth reference (read+write)
  {
    size_t half = bytes / 2;
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      CK(cudaMemcpyAsync(buf + half, buf, half, cudaMemcpyDeviceToDevice));
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("cudaMemcpy D2D %zu MB: %.1f GB/s (read+write)\n", half >> 20, 2.0 * half / best / 1e6);
  }
  printf("OK\n");
  return 0;
}
