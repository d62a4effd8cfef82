// Pipe-throughput microbenchmark (sm_100a): lane-ops per clock per SM for the
// activation building blocks of the chain epilogue.  Each thread runs 8
// independent dependency chains; per-SM cycles from clock64 in warp 0.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(uint32_t* out, int iters, long long* cyc) {
  uint32_t v[8];
  for (int i = 0; i < 8; i++) v[i] = 0x3f003f00u + threadIdx.x * 7 + i;
  float f[8];
  for (int i = 0; i < 8; i++) f[i] = 0.1f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (OP == 0) asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(v[i]));
      if (OP == 1) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(f[i]));
      if (OP == 2) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
      if (OP == 3) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(f[i]));
      if (OP == 4) asm volatile("fma.rn.bf16x2 %0, %0, %0, %0;" : "+r"(v[i]));
      if (OP == 5) asm volatile("max.f32 %0, %0, 0f3F000000;" : "+f"(f[i]));
      if (OP == 6) asm volatile("tanh.approx.f16x2 %0, %0;" : "+r"(v[i]));
      if (OP == 7) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(v[i]) : "f"(f[i]), "f"(__uint_as_float(v[i])));
      if (OP == 8) asm volatile("fma.rn.f32 %0, %0, 0f3F000000, 0f3E000000;" : "+f"(f[i]));
      if (OP == 9) asm volatile("{.reg .b64 a; mov.b64 a, {%0,%1}; fma.rn.f32x2 a, a, a, a; mov.b64 {%0,%1}, a;}" : "+f"(f[i]), "+f"(f[(i+1)&7]));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t acc = 0;
  for (int i = 0; i < 8; i++) acc ^= v[i] ^ __float_as_uint(f[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int threads) {
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  k<OP><<<148, threads>>>(out, iters, cyc);
  k<OP><<<148, threads>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0; for (int i = 0; i < 148; i++) c += h[i]; c /= 148;
  double ops = (double)threads * iters * 8 * ((OP == 0 || OP == 4 || OP == 6 || OP == 9) ? 2 : 1);
  printf("%-22s threads %4d  %.2f lane-ops/clk/SM (elements)  %.2f instr/clk/SM\n", name, threads, ops / c,
         (double)threads * iters * 8 / c);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int t : {256, 512, 1024}) {
    run<0>("tanh.bf16x2", t); run<6>("tanh.f16x2", t); run<1>("tanh.f32", t); run<2>("ex2.f32", t);
    run<3>("ffma 3reg", t); run<8>("ffma imm", t); run<4>("hfma2.bf16", t); run<5>("fmax imm", t);
    run<7>("cvt.bf16x2.f32", t); run<9>("ffma2 f32x2", t);
  }
  return 0;
}
