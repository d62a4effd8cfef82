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

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Fast GELU (mfp_sdnet_desc.gelu = 1; reading GELU): the tanh form
// 0.5 x (1 + tanh(c0 x + c1 x^3)), c0 = sqrt(2/pi), c1 = 0.044715 c0, of the
// exact GELU x Phi(x).  Max |error of 2 GELU| against erf: 9.5e-4 near
// |x| = 2, but O(x^5) near 0 where most pre-activations sit.  Refitted
// coefficients (tools/fit_gelu_poly.py) were tried: a minimax (c0, c1) halves
// the max error yet doubled the measured fp16 field error (it is worse for
// small |x|); a 3-coefficient clamped form is accurate everywhere but costs 11%
// of the chain's throughput — DESIGN.md §7.
constexpr float kGF0 = 0.7978845608028654f, kGF1 = 0.7978845608028654f * 0.044715f;

// Accurate form (mfp_sdnet_desc.gelu = 2; the accuracy mode MFP_FP16X):
// 2 GELU(x) ~= x + x tanh(x (a0 + t (a1 + t a2))), t = min(x^2, 16), minimax fit
// of x erf(x / sqrt 2) (tools/fit_gelu_poly.py --three): |error of 2 GELU| <=
// 5.04e-5 everywhere (the classic form: 9.5e-4), for two more instructions per
// element.
constexpr float kGA0 = 0.79750786895f, kGA1 = 0.037005660849f, kGA2 = -3.5151936221e-4f;
__device__ __forceinline__ float gelu2_acc(float x) {
  const float t = fminf(x * x, 16.0f);
  const float u = x * fmaf(t, fmaf(t, kGA2, kGA1), kGA0);
  return fmaf(x, tanh_approx(u), x);
}

// 2 GELU(x) (scalar).
__device__ __forceinline__ float gelu2_fast(float x) {
  const float u = x * fmaf(kGF1, x * x, kGF0);
  return fmaf(x, tanh_approx(u), x);
}
__device__ __forceinline__ float gelu_fast(float x) { return 0.5f * gelu2_fast(x); }

// Lattice accessors.  Anchor packed as a | b << 16 where
// (a, b) are local vertical/horizontal line indices of the subdomain's left /
// bottom edge (lx = 16 a, ly = 16 b).
__device__ __forceinline__ void unpack_anchor(uint32_t p, int& a, int& b) {
  a = (int)(p & 0xffffu);
  b = (int)((p >> 16) & 0x7fffu);   // bit 31: "writes a cell some peer holds as halo" (put mode)
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

// ---- boundary embedding helpers (reading G7) -----------------------
// Window [i0-2, i0+5] of a circular length-128 signal held 4-per-lane (lane l
// owns positions 4l..4l+3): two values from each neighbouring lane.
__device__ __forceinline__ void circ_window(const float (&v)[4], int lane, float (&w)[8]) {
  const int left = (lane + 31) & 31, right = (lane + 1) & 31;
  w[0] = __shfl_sync(0xffffffffu, v[2], left);
  w[1] = __shfl_sync(0xffffffffu, v[3], left);
  w[2] = v[0]; w[3] = v[1]; w[4] = v[2]; w[5] = v[3];
  w[6] = __shfl_sync(0xffffffffu, v[0], right);
  w[7] = __shfl_sync(0xffffffffu, v[1], right);
}

template <int GELU>
__device__ __forceinline__ float emb_act(float x) {
  if constexpr (GELU == 1) return gelu_fast(x);
  else if constexpr (GELU == 2) return 0.5f * gelu2_acc(x);
  else return gelu_erf(x);
}

// conv1 (1 -> 8, k = 5, circular) + GELU, conv2 (8 -> 1) + GELU on the 4
// positions this lane owns; cw = {c1w[40], c1b[8], c2w[40], c2b[1]} (smem).
template <int GELU>
__device__ __forceinline__ void conv_stack(const float (&g4)[4], int lane, const float* cw, float (&e)[4]) {
  float win[8];
  circ_window(g4, lane, win);
  float acc2[4] = {cw[88], cw[88], cw[88], cw[88]};
#pragma unroll
  for (int o = 0; o < kC1; o++) {
    float c1v[4];
#pragma unroll
    for (int p = 0; p < 4; p++) {
      float v = cw[40 + o];
#pragma unroll
      for (int t = 0; t < kK; t++) v = fmaf(cw[o * kK + t], win[p + t], v);
      c1v[p] = emb_act<GELU>(v);
    }
    float w2[8];
    circ_window(c1v, lane, w2);
#pragma unroll
    for (int p = 0; p < 4; p++)
#pragma unroll
      for (int t = 0; t < kK; t++) acc2[p] = fmaf(cw[48 + o * kK + t], w2[p + t], acc2[p]);
  }
#pragma unroll
  for (int p = 0; p < 4; p++) e[p] = emb_act<GELU>(acc2[p]);
}

// Gather the 4 perimeter values (G1 order) lane `lane` owns: positions 4l..4l+3
// of edge l/8 — one float4 for the two forward edges, 4 scalars for the
// reversed ones (top R->L, left T->B).
__device__ __forceinline__ float4 gather4(const float* lat, const LatticeGeom& L, uint32_t packed, int lane) {
  int a, b;
  unpack_anchor(packed, a, b);
  const int lx = kH * a, ly = kH * b, edge = lane >> 3, t0 = 4 * (lane & 7);
  if (edge == 0) return *reinterpret_cast<const float4*>(lat + (int64_t)b * L.strideH + lx + t0);
  if (edge == 1) return *reinterpret_cast<const float4*>(lat + L.offV + (int64_t)(a + 2) * L.strideV + ly + t0);
  const float* r = edge == 2 ? lat + (int64_t)(b + 2) * L.strideH + lx + kM - t0
                             : lat + L.offV + (int64_t)a * L.strideV + ly + kM - t0;
  return make_float4(r[0], r[-1], r[-2], r[-3]);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// NEXT-2 put transport: an owned cell some peer holds as a halo cell is also
// stored into that peer's put buffer (peer memory over NVLink, or this device
// under MFP_ALL_RANKS) of parity (put epoch + 1) & 1; a cell sits in at most 3
// peers' halos (a corner).  Only subdomains whose anchor carries bit 31 look
// their cells up, so the common path costs one predicated branch.
__device__ __forceinline__ void put_halo(const Sink& sk, int64_t c, float y) {
  const int32_t pm = __ldg(sk.putmap + c);
  if (pm < 0) return;
  const int par = (int)((*sk.put_epoch + 1ull) & 1ull);
  for (int k = 0; k < (pm & 3); k++) {
    const int32_t d = __ldg(sk.putdst + (pm >> 2) + k);
    sk.putbufs[2 * (d >> 24) + par][d & 0xffffff] = y;
  }
}

// Write one chain output (row = s * q + p) to its sink.
__device__ __forceinline__ void sink_store(const Sink& sk, int64_t s, int p, float y) {
  if (sk.mode == 0) {
    int a, b;
    const uint32_t pk = __ldg(sk.anchors + s);
    unpack_anchor(pk, a, b);
    int64_t dup;
    int64_t c = centre_cell(a, b, p, sk.strideH, sk.strideV, sk.offV, &dup);
    sk.lat[c] = y;
    if (dup >= 0) sk.lat[dup] = y;
    if (sk.putmap && (pk >> 31)) {   // only subdomains whose centre lines feed a peer's halo
      put_halo(sk, c, y);
      if (dup >= 0) put_halo(sk, dup, y);
    }
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
