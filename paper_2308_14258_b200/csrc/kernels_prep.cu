// kernels_prep.cu — one-time device-side preparation in mfp_init (a0):
// weight layout transforms, the query tables Q = X W2^T of the split layer
// (Eq. 5), the bf16 SW128 K-major images of the hidden weights for the
// tcgen05 chain, and the exact harmonic-extension matrices of the discrete
// Laplace subsolver (N9), evaluated from the closed-form discrete sine
// expansion of the 5-point Dirichlet problem on the (m+1)^2 patch.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "device_common.cuh"

namespace mfp {

// Byte offset of element (row r, k) in a 128 x 128 bf16 K-major tile stored as
// two SW128 atoms-columns (k < 64, k >= 64) of 16 KB each: 128 B rows, the
// 16-byte chunk index XOR-ed with (r mod 8) — the layout tcgen05 smem
// descriptors with layout type SWIZZLE_128B expect.
__host__ __device__ __forceinline__ uint32_t sw128_offset(int r, int k) {
  const int kb = k >> 6, kk = k & 63;
  const int chunk = kk >> 3, within = kk & 7;
  return (uint32_t)(kb * 16384 + r * 128 + ((chunk ^ (r & 7)) << 4) + within * 2);
}

// 16-bit operand value of a weight (B operands are scaled by 1/2, exact,
// because the tensor-core epilogue feeds h' = 2 GELU(x) into the next layer)
__device__ __forceinline__ void put16(uint8_t* p, float v, int f16) {
  if (f16) *reinterpret_cast<__half*>(p) = __float2half_rn(v);
  else *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(v);
}
// b = b_hi + b_lo in the operand type (the bias step's two K columns)
__device__ __forceinline__ void put_bias(uint8_t* p, float b, int f16) {
  if (f16) {
    const __half hi = __float2half_rn(b), lo = __float2half_rn(b - __half2float(hi));
    *reinterpret_cast<__half*>(p) = hi;
    *reinterpret_cast<__half*>(p + 2) = lo;
  } else {
    const __nv_bfloat16 hi = __float2bfloat16_rn(b), lo = __float2bfloat16_rn(b - __bfloat162float(hi));
    *reinterpret_cast<__nv_bfloat16*>(p) = hi;
    *reinterpret_cast<__nv_bfloat16*>(p + 2) = lo;
  }
}

__global__ void k_prep(PrepArgs a) {
  const int d = a.d;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  // W1T[k][c] = W1[c][k]; and the bf16 split images W1 = W1_hi + W1_lo (row c,
  // K k) of the tensor-core embed
  for (int64_t i = tid; i < (int64_t)kNB * d; i += nth) {
    int k = (int)(i / d), c = (int)(i % d);
    const float w = a.P[a.oW1 + (int64_t)c * kNB + k];
    a.W1T[i] = w;
    {
      // [half c / 128][hi | lo][128 rows x 128 K] (d = 256 holds two halves)
      const __nv_bfloat16 hi = __float2bfloat16_rn(w);
      const __nv_bfloat16 lo = __float2bfloat16_rn(w - __bfloat162float(hi));
      uint8_t* img = reinterpret_cast<uint8_t*>(a.W1img) + (size_t)(c >> 7) * 2 * (kD * kNB * 2);
      *reinterpret_cast<__nv_bfloat16*>(img + sw128_offset(c & 127, k)) = hi;
      *reinterpret_cast<__nv_bfloat16*>(img + kD * kNB * 2 + sw128_offset(c & 127, k)) = lo;
    }
  }
  // hidden layers
  for (int64_t i = tid; i < (int64_t)a.n_hidden * d * d; i += nth) {
    int l = (int)(i / ((int64_t)d * d));
    int rem = (int)(i % ((int64_t)d * d));
    int k = rem / d, n = rem % d;
    const float* Wl = a.P + a.oWh0 + (int64_t)l * (d * d + d);
    const float w = Wl[(int64_t)n * d + k];
    a.WhT[i] = w;                                    // [l][k][n]
    if (d == kD) {
      // CTA-pair image: half n/64 holds rows n%64 as a 64-row SW128 K-major
      // block (two 8 KB K-halves) followed by its 2 KB bias block
      uint8_t* img2 = reinterpret_cast<uint8_t*>(a.Wsw2 + (int64_t)l * kWImg) + (n >> 6) * (kWImg);
      const int rr = n & 63;
      const uint32_t off2 = (uint32_t)((k >> 6) * 8192 + rr * 128 + ((((k & 63) >> 3) ^ (rr & 7)) << 4) + (k & 7) * 2);
      put16(img2 + off2, 0.5f * w, a.f16);
    } else {
      // d = 256: CTA n/128 holds rows n%128 as four 16 KB SW128 K-chunks of 64
      uint8_t* img = reinterpret_cast<uint8_t*>(a.Wsw2 + (int64_t)l * kW2Layer + (int64_t)(n >> 7) * kW2Cta);
      const int rr = n & 127;
      const uint32_t off = (uint32_t)((k >> 6) * 16384 + rr * 128 + ((((k & 63) >> 3) ^ (rr & 7)) << 4) + (k & 7) * 2);
      put16(img + off, 0.5f * w, a.f16);
    }
  }
  for (int64_t i = tid; i < (int64_t)a.n_hidden * d; i += nth) {
    int l = (int)(i / d), c = (int)(i % d);
    const float b = a.P[a.oWh0 + (int64_t)l * (d * d + d) + (int64_t)d * d + c];
    a.bh[i] = b;
    // bias block of the tensor-core image: row n = c, K columns 0/1 = b_hi, b_lo
    // (SWIZZLE_NONE K-major: 8-row x 16-byte core matrices, LBO 128 B, SBO 256 B);
    // the A operand carries a constant 1 in those two columns, so the MMA adds
    // b_hi + b_lo (accurate to ~2^-17 relative) to the fp32 accumulator.
    if (d == kD) {
      const int rr = c & 63;
      uint8_t* blk2 = reinterpret_cast<uint8_t*>(a.Wsw2 + (int64_t)l * kWImg) + (c >> 6) * kWImg + 16384;
      put_bias(blk2 + (rr >> 3) * 256 + (rr & 7) * 16, b, a.f16);
    } else {
      const int rr = c & 127;
      uint8_t* blk = reinterpret_cast<uint8_t*>(a.Wsw2 + (int64_t)l * kW2Layer + (int64_t)(c >> 7) * kW2Cta) + 65536;
      put_bias(blk + (rr >> 3) * 256 + (rr & 7) * 16, b, a.f16);
    }
  }
  // Q = X W2^T (b1 is folded into z): centre (64 padded) and interior (961)
  for (int64_t i = tid; i < (int64_t)64 * d; i += nth) {
    int p = (int)(i / d), c = (int)(i % d);
    float v = 0.f;
    if (p < kQC) {
      float x, y;
      query_xy(kQC, p, &x, &y);
      v = fmaf(a.P[a.oW2 + 2 * c], x, a.P[a.oW2 + 2 * c + 1] * y);
    }
    a.QTc[(int64_t)c * 64 + p] = v;
  }
  for (int64_t i = tid; i < (int64_t)kQF * d; i += nth) {
    int p = (int)(i / d), c = (int)(i % d);
    float x, y;
    query_xy(kQF, p, &x, &y);
    float v = fmaf(a.P[a.oW2 + 2 * c], x, a.P[a.oW2 + 2 * c + 1] * y);
    a.QTf[(int64_t)c * kQF + p] = v;
  }
}

void launch_prep(const PrepArgs& a, cudaStream_t s) { k_prep<<<num_sms() * 2, 256, 0, s>>>(a); }

// Harmonic-extension matrix H^T [k][q] for the 5-point Dirichlet problem on the
// (m+1)^2 patch: separation of variables with the DST-I basis,
//   u(i,j) = sum_k (2/m) f^_k sin(pi k i/m) sinh(l_k (m-j)) / sinh(l_k m),
// cosh(l_k) = 2 - cos(pi k/m), for data on the bottom side; the other three
// sides by symmetry.  fp64 evaluation, stored fp32.  Corners never enter the
// 5-point stencil: their columns are 0.
__global__ void k_harmonic(int q, int ld, float* __restrict__ HT) {
  const int total = kNB * q;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int kb = t / q, p = t % q;
    int qi, qj;  // query grid point (i, j) in the patch
    if (q == kQC) {
      if (p < kM - 1) { qi = kH; qj = p + 1; }
      else { int j = p - (kM - 1); qi = j + 1 + (j >= kH - 1 ? 1 : 0); qj = kH; }
    } else { qi = p % (kM - 1) + 1; qj = p / (kM - 1) + 1; }
    const int side = kb >> 5, pos = kb & 31;
    // s_b: position of the boundary point along its side (0 or m = corner);
    // along: the query's coordinate along that side; dist: the query's
    // distance from that side.  Factor sinh(l (m - dist)) / sinh(l m).
    int s_b, along, dist;
    switch (side) {
      case 0: s_b = pos;      along = qi; dist = qj;      break;  // bottom, point (pos, 0)
      case 1: s_b = pos;      along = qj; dist = kM - qi; break;  // right,  point (m, pos)
      case 2: s_b = kM - pos; along = qi; dist = kM - qj; break;  // top,    point (m - pos, m)
      default: s_b = kM - pos; along = qj; dist = qi;     break;  // left,   point (0, m - pos)
    }
    double v = 0.0;
    if (s_b > 0 && s_b < kM) {
      for (int k = 1; k < kM; k++) {
        const double th = M_PI * k / kM;
        const double lk = acosh(2.0 - cos(th));
        v += (2.0 / kM) * sin(th * s_b) * sin(th * along) * sinh(lk * (kM - dist)) / sinh(lk * kM);
      }
    }
    HT[(int64_t)kb * ld + p] = (float)v;
  }
}

void launch_harmonic(int q, float* HT, cudaStream_t s) {
  k_harmonic<<<num_sms(), 256, 0, s>>>(q, q == kQC ? 64 : q, HT);
}

}  // namespace mfp
