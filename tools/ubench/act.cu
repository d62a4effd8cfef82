// Throughput of the chain epilogue's activation sequence in isolation:
// per element pair FMUL2, FFMA2, FMUL2, 2x MUFU.TANH, FFMA2, F2FP (act8 of
// kernels_tc.cu), 16 independent pairs per thread, swept over warps per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2308_14258_b200/csrc/tc_common.cuh"

using namespace mfp::tcx;
using mfp::tanh_approx;

template <int FAKE>
__device__ __forceinline__ f2 act(f2 x) {
  float u0, u1;
  f2_split(fmul2(x, ffma2(fmul2(x, x), f2_make(0.0356774f, 0.0356774f), f2_make(0.79788f, 0.79788f))), u0, u1);
  if (FAKE == 1) return ffma2(x, f2_make(fminf(fmaxf(u0, -1.f), 1.f), fminf(fmaxf(u1, -1.f), 1.f)), x);
  if (FAKE == 2) return ffma2(x, f2_make(u0, u1), x);
  return ffma2(x, f2_make(tanh_approx(u0), tanh_approx(u1)), x);
}

// FMA-pipe polynomial GELU (tools/fit_gelu_poly.py, n = 7, a = 3.9)
__device__ __forceinline__ f2 act_poly(f2 x) {
  float x0, x1;
  f2_split(x, x0, x1);
  const float A = 3.9f;
  const f2 xc = f2_make(fminf(fmaxf(x0, -A), A), fminf(fmaxf(x1, -A), A));
  const f2 t = fmul2(xc, xc);
  f2 P = ffma2(t, f2_make(4.559065658e-08f, 4.559065658e-08f), f2_make(-3.193779321e-06f, -3.193779321e-06f));
  P = ffma2(P, t, f2_make(9.576256707e-05f, 9.576256707e-05f));
  P = ffma2(P, t, f2_make(-1.625960576e-03f, -1.625960576e-03f));
  P = ffma2(P, t, f2_make(1.753236353e-02f, 1.753236353e-02f));
  P = ffma2(P, t, f2_make(-1.291151345e-01f, -1.291151345e-01f));
  P = ffma2(P, t, f2_make(7.957426310e-01f, 7.957426310e-01f));
  return ffma2(x, fmul2(xc, P), x);
}

template <int FAKE>
__global__ void k(uint32_t* out, int iters, long long* cyc) {
  float v[32];
  for (int i = 0; i < 32; i++) v[i] = 0.001f * (threadIdx.x + i);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int e = 0; e < 16; e++) {
      float h0, h1;
      const f2 xx = f2_make(v[2 * e], v[2 * e + 1]);
      const bool poly = (FAKE == 3 && (e & 3) == 3) || (FAKE == 4 && (e & 1)) || FAKE == 5 || (FAKE == 6 && (e % 3) == 2);
      f2_split(poly ? act_poly(xx) : act<FAKE>(xx), h0, h1);
      uint32_t w;
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w) : "f"(h1), "f"(h0));
      acc += w;
      v[2 * e] = __uint_as_float(w << 16) * 0.5f;
      v[2 * e + 1] = __uint_as_float(w & 0xffff0000u) * 0.5f;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int FAKE>
void run(const char* name, int threads) {
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 256;
  k<FAKE><<<148, threads>>>(out, iters, cyc);
  k<FAKE><<<148, threads>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0; for (int i = 0; i < 148; i++) c += h[i]; c /= 148;
  printf("%-10s warps/SM %2d  %.2f pairs/clk/SM\n", name, threads / 32, (double)threads * iters * 16 / c);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int t : {512, 576, 1024}) {
    run<0>("mufu", t); run<3>("poly 1/4", t); run<6>("poly 1/3", t); run<4>("poly 1/2", t); run<5>("poly all", t);
  }
  return 0;
}
