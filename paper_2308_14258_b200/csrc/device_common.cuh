// device_common.cuh — small device helpers shared by the libmfp kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "mfp_internal.h"

namespace mfp {

#define MFP_CUDA_OK(x) ((x) == cudaSuccess)

// Exact GELU x * Phi(x) ([hendrycks2016gelu]).
__device__ __forceinline__ float gelu_erf(float x) {
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
}

// tanh approximation of GELU (bf16 path only, mfp_sdnet_desc.gelu = 1).
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float u = k0 * x * fmaf(k1, x * x, 1.0f);
  float hx = 0.5f * x;
  return fmaf(hx, tanh_approx(u), hx);
}

// Lattice accessors.  Anchor packed as a | b << 16 where
// (a, b) are local vertical/horizontal line indices of the subdomain's left /
// bottom edge (lx = 16 a, ly = 16 b).
__device__ __forceinline__ void unpack_anchor(uint32_t p, int& a, int& b) {
  a = (int)(p & 0xffffu);
  b = (int)(p >> 16);
}

// Perimeter value i (0..127) in G1 order: bottom L->R, right B->T, top R->L, left T->B.
__device__ __forceinline__ int64_t perim_cell(int a, int b, int i, int strideH, int strideV,
                                              int64_t offV) {
  const int lx = kH * a, ly = kH * b;
  const int e = i >> 5, t = i & 31;
  switch (e) {
    case 0: return (int64_t)b * strideH + lx + t;
    case 1: return offV + (int64_t)(a + 2) * strideV + ly + t;
    case 2: return (int64_t)(b + 2) * strideH + lx + kM - t;
    default: return offV + (int64_t)a * strideV + ly + kM - t;
  }
}

// Centre-line cell of query p (G3).  Returns the primary cell; *dup = second
// copy for the centre point (p == 15, crossing of both lines) or -1.
__device__ __forceinline__ int64_t centre_cell(int a, int b, int p, int strideH, int strideV,
                                               int64_t offV, int64_t* dup) {
  const int lx = kH * a, ly = kH * b;
  if (p < kM - 1) {
    const int k = p + 1;
    *dup = (k == kH) ? (int64_t)(b + 1) * strideH + lx + kH : -1;
    return offV + (int64_t)(a + 1) * strideV + ly + k;
  }
  const int j = p - (kM - 1);
  const int k = j + 1 + (j >= kH - 1 ? 1 : 0);
  *dup = -1;
  return (int64_t)(b + 1) * strideH + lx + k;
}

// Local normalised query coordinates (x/m, y/m): centre lines (G3, q = 61) or
// the interior grid (q = 961, i fastest).
__device__ __forceinline__ void query_xy(int q, int p, float* x, float* y) {
  if (q == kQC) {
    if (p < kM - 1) { *x = 0.5f; *y = (float)(p + 1) / kM; }
    else {
      const int j = p - (kM - 1);
      const int k = j + 1 + (j >= kH - 1 ? 1 : 0);
      *x = (float)k / kM; *y = 0.5f;
    }
  } else {
    *x = (float)(p % (kM - 1) + 1) / kM;
    *y = (float)(p / (kM - 1) + 1) / kM;
  }
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Write one chain output (row = s * q + p) to its sink.
__device__ __forceinline__ void sink_store(const Sink& sk, int64_t s, int p, float y) {
  if (sk.mode == 0) {
    int a, b;
    unpack_anchor(__ldg(sk.anchors + s), a, b);
    int64_t dup;
    int64_t c = centre_cell(a, b, p, sk.strideH, sk.strideV, sk.offV, &dup);
    sk.lat[c] = y;
    if (dup >= 0) sk.lat[dup] = y;
  } else if (sk.mode == 1) {
    uint32_t pk = __ldg(sk.anchors + s);
    int bx = (int)(pk & 0xffffu), by = (int)(pk >> 16);
    int i = p % (kM - 1) + 1, j = p / (kM - 1) + 1;
    sk.field[(int64_t)(by + j) * sk.ld + bx + i] = y;
  } else {
    sk.out[s * sk.q + p] = y;
  }
}

}  // namespace mfp
