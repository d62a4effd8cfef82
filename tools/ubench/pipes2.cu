// Pipe-throughput microbenchmark, part 2: packed fp32x2 with independent
// chains, and MUFU + FMA-pipe co-issue (does the poly GELU overlap MUFU?).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t r; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r;
}

template <int OP>
__global__ void k(uint32_t* out, int iters, long long* cyc) {
  uint64_t p[8];
  float f[8];
  uint32_t h[8];
  for (int i = 0; i < 8; i++) {
    p[i] = 0x3f0000003f000000ull + threadIdx.x + i;
    f[i] = 0.01f * (threadIdx.x + i);
    h[i] = 0x3f003f00u + threadIdx.x * 7 + i;
  }
  const uint64_t c2 = 0x3f7000003f700000ull;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (OP == 0) p[i] = ffma2(p[i], c2, p[i]);                        // FFMA2, 8 chains
      if (OP == 1) p[i] = fmul2(p[i], c2);                              // FMUL2
      if (OP == 2) {                                                    // 1 MUFU + 4 FFMA per element
        asm volatile("tanh.approx.f32 %0, %0;" : "+f"(f[i]));
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(f[(i + 4) & 7]));
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(f[(i + 5) & 7]));
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(f[(i + 6) & 7]));
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(f[(i + 7) & 7]));
      }
      if (OP == 3) {                                                    // 1 MUFU + 8 FFMA
        asm volatile("tanh.approx.f32 %0, %0;" : "+f"(f[i]));
#pragma unroll
        for (int j = 1; j < 8; j++) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(f[(i + j) & 7]));
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(f[(i + 3) & 7]));
      }
      if (OP == 4) {                                                    // 1 packed MUFU + 2 HFMA2
        asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(h[i]));
        asm volatile("fma.rn.bf16x2 %0, %0, %0, %0;" : "+r"(h[(i + 3) & 7]));
        asm volatile("fma.rn.bf16x2 %0, %0, %0, %0;" : "+r"(h[(i + 5) & 7]));
      }
      if (OP == 5) asm volatile("mul.rn.bf16x2 %0, %0, %0;" : "+r"(h[i]));  // HMUL2
      if (OP == 6) asm volatile("prmt.b32 %0, %0, %1, 0x7632;" : "+r"(h[i]) : "r"(h[(i + 1) & 7]));  // PRMT
      if (OP == 7) asm volatile("min.f32 %0, %0, %1;" : "+f"(f[i]) : "f"(f[(i + 3) & 7]));  // FMNMX reg
    }
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t acc = 0;
  for (int i = 0; i < 8; i++) acc ^= (uint32_t)p[i] ^ (uint32_t)(p[i] >> 32) ^ __float_as_uint(f[i]) ^ h[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int threads, double ops_per_inner) {
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 2048;
  k<OP><<<148, threads>>>(out, iters, cyc);
  k<OP><<<148, threads>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long hc[148]; cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
  double c = 0; for (int i = 0; i < 148; i++) c += hc[i]; c /= 148;
  printf("%-34s threads %4d  %.2f units/clk/SM\n", name, threads, (double)threads * iters * 8 * ops_per_inner / c);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int t : {512, 1024}) {
    run<0>("ffma2 (elements)", t, 2); run<1>("fmul2 (elements)", t, 2);
    run<2>("tanh.f32 + 4 ffma (tanh/clk)", t, 1); run<3>("tanh.f32 + 8 ffma (tanh/clk)", t, 1);
    run<4>("tanh.bf16x2 + 2 hfma2 (pairs/clk)", t, 1); run<5>("hmul2.bf16 (instr)", t, 1);
    run<6>("prmt (instr)", t, 1); run<7>("fmnmx reg (instr)", t, 1);
  }
  return 0;
}
