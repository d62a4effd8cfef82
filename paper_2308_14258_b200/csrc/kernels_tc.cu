// kernels_tc.cu — bf16 SDNet MLP chain on the 5th-generation tensor cores (N4).
//
// The hidden GEMM chain h <- GELU(h W_l^T + b_l) is the path's one
// dense contraction: rows = (subdomain, query) pairs packed densely
// (row = s*q + p), K = N = d = 128.  Design:
//   * persistent CTAs (one per SM), 128-row tiles (UMMA M = 128, N = 128,
//     K = 16 x 8 per layer), fp32 accumulators in TMEM;
//   * the n_hidden weight matrices stay resident in shared memory for the
//     whole kernel as bf16 SWIZZLE_128B K-major images (B operand);
//   * two epilogue warpgroups ping-pong on two tiles (TMEM slots 0/1, smem A
//     buffers 0/1): while the tensor core runs layer l of one tile, the other
//     warpgroup's epilogue (tcgen05.ld -> +bias -> GELU -> bf16 -> st.shared
//     into the swizzled A operand of layer l+1) runs on the other;
//   * one elected thread issues tcgen05.mma and tcgen05.commit -> mbarrier;
//   * the layer-1 input is Eq. 5's broadcasted sum GELU(z[s] + Q[p]) built
//     directly into the A buffer (Q = X W2^T resident in smem for the 61
//     centre-line queries); the last epilogue does the head dot y = wo.h + bo
//     and the scatter onto the lattice (fused N5).
#include <cuda_bf16.h>

#include "device_common.cuh"

namespace mfp {
namespace tc {

constexpr int kRows = 128;
constexpr int kThreads = 384;          // warp 0: MMA issue, warp 1: TMEM alloc, warps 4-11: epilogue
constexpr int kTile = kRows * kD * 2;  // 32 KB bf16 operand image
constexpr int kQStride = 132;          // padded fp32 row of the smem Q table (bank spread)
constexpr int kTmemCols = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Shared-memory matrix descriptor, K-major, SWIZZLE_128B: start address >> 4,
// LBO = 1 (unused for swizzled K-major), SBO = 1024 B (8 rows x 128 B),
// version 1 (sm_100), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor, kind::f16: D fp32 (bits 4-5 = 1), A/B bf16 (bits
// 7-9, 10-12 = 1), both K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28.
// A/B format 1 = bf16, 0 = fp16.
template <int F16>
constexpr uint32_t idesc() {
  return (1u << 4) | ((F16 ? 0u : 1u) << 7) | ((F16 ? 0u : 1u) << 10) | ((uint32_t)(kD >> 3) << 17) |
         ((uint32_t)(kRows >> 4) << 24);
}

template <int F16>
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc<F16>()), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Round two fp32 values to the operand type (lo -> bits 0-15).
template <int F16>
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  uint32_t r;
  if constexpr (F16) asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  else asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

// Byte offset of (row, k) in a 128 x 128 bf16 SW128 K-major image (two 16 KB
// K-halves; 16-byte chunk index XOR row mod 8).  Same formula as kernels_prep.
__device__ __forceinline__ uint32_t sw128_off(int r, int k) {
  const int kb = k >> 6, chunk = (k & 63) >> 3;
  return (uint32_t)(kb * 16384 + r * 128 + ((chunk ^ (r & 7)) << 4));
}

template <int GELU>
__device__ __forceinline__ float act(float x) {
  if constexpr (GELU == 1) return gelu_tanh(x);
  else return gelu_erf(x);
}

template <int GELU, int F16>
__global__ void __launch_bounds__(kThreads, 1)
k_chain_tc(const float* __restrict__ z, int64_t total_rows, int q, const float* __restrict__ Qg,
           DevNet net, Sink sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int nh = net.n_hidden;
  uint8_t* sW = base;
  uint8_t* sA = base + nh * kTile;
  float* sQ = (float*)(sA + 2 * kTile);
  float* sBh = sQ + 64 * kQStride;
  float* sWo = sBh + kMaxHidden * kD;
  uint64_t* bars = (uint64_t*)(sWo + kD);  // a_full[2], d_full[2]
  uint32_t* tmem_slot = (uint32_t*)(bars + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- prologue: resident weights / tables
  {
    const uint4* src = reinterpret_cast<const uint4*>(net.Wh_sw);
    uint4* dst = reinterpret_cast<uint4*>(sW);
    for (int i = threadIdx.x; i < nh * kTile / 16; i += kThreads) dst[i] = __ldg(src + i);
    if (q == kQC)
      for (int i = threadIdx.x; i < 64 * kD; i += kThreads) sQ[(i >> 7) * kQStride + (i & 127)] = __ldg(net.Qc + i);
    for (int i = threadIdx.x; i < nh * kD; i += kThreads) sBh[i] = __ldg(net.bh + i);
    for (int i = threadIdx.x; i < kD; i += kThreads) sWo[i] = __ldg(net.wo + i);
  }
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 128);
    mbar_init(&bars[1], 128);
    mbar_init(&bars[2], 1);
    mbar_init(&bars[3], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_proxy_async();  // generic-proxy writes of W visible to the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const float bo = __ldg(net.bo);

  const int64_t ntiles = (total_rows + kRows - 1) / kRows;
  const int64_t nloc = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  if (warp == 0) {
    // ---- MMA issuer: round-robin over (tile pair, layer, slot)
    if (lane == 0) {
      uint32_t pa[2] = {0u, 0u};
      for (int64_t j0 = 0; j0 < nloc; j0 += 2) {
        for (int l = 0; l < nh; l++) {
          for (int s = 0; s < 2; s++) {
            if (j0 + s >= nloc) continue;
            mbar_wait(&bars[s], pa[s]);
            pa[s] ^= 1u;
            tc_fence_after();
            const uint32_t a0 = smem_u32(sA + s * kTile), b0 = smem_u32(sW + l * kTile);
#pragma unroll
            for (int k = 0; k < kD / 16; k++) {
              const uint32_t off = (uint32_t)((k >> 2) * 16384 + (k & 3) * 32);
              mma_f16<F16>(tmem + (uint32_t)(s * kD), sw128_desc(a0 + off), sw128_desc(b0 + off), k > 0 ? 1u : 0u);
            }
            mma_commit(&bars[2 + s]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ---- epilogue warpgroups: slot wg = 0 / 1, thread <-> tile row <-> TMEM lane
    const int wg = (warp - 4) >> 2;
    const int quad = (warp - 4) & 3;
    const int row = quad * 32 + lane;
    uint8_t* A = sA + wg * kTile;
    const uint32_t a_base = smem_u32(A);
    const uint32_t t_row = tmem + (uint32_t)(wg * kD) + ((uint32_t)(quad * 32) << 16);
    uint32_t pd = 0u;
    for (int64_t j = wg; j < nloc; j += 2) {
      const int64_t tile = blockIdx.x + j * (int64_t)gridDim.x;
      const int64_t grow = tile * kRows + row;
      const bool valid = grow < total_rows;
      const int64_t gr = valid ? grow : total_rows - 1;
      const int64_t sidx = gr / q;
      const int p = (int)(gr - sidx * q);
      // layer-1 input (Eq. 5): GELU(z[s] + Q[p]) -> bf16 A operand
      {
        const float4* zr = reinterpret_cast<const float4*>(z + sidx * kD);
        const float4* qr = reinterpret_cast<const float4*>(q == kQC ? sQ + p * kQStride : Qg + (int64_t)p * kD);
#pragma unroll 2
        for (int cc = 0; cc < kD / 8; cc++) {
          const float4 z0 = __ldg(zr + 2 * cc), z1 = __ldg(zr + 2 * cc + 1);
          const float4 q0 = qr[2 * cc], q1 = qr[2 * cc + 1];
          const uint32_t w0 = pack2<F16>(act<GELU>(z0.x + q0.x), act<GELU>(z0.y + q0.y));
          const uint32_t w1 = pack2<F16>(act<GELU>(z0.z + q0.z), act<GELU>(z0.w + q0.w));
          const uint32_t w2 = pack2<F16>(act<GELU>(z1.x + q1.x), act<GELU>(z1.y + q1.y));
          const uint32_t w3 = pack2<F16>(act<GELU>(z1.z + q1.z), act<GELU>(z1.w + q1.w));
          st_shared_v4(a_base + sw128_off(row, cc * 8), w0, w1, w2, w3);
        }
      }
      fence_proxy_async();
      mbar_arrive(&bars[wg]);
      float y = 0.f;
      for (int l = 0; l < nh; l++) {
        mbar_wait(&bars[2 + wg], pd);
        pd ^= 1u;
        tc_fence_after();
        const float* bl = sBh + l * kD;
        const bool last = (l == nh - 1);
#pragma unroll 1
        for (int ch = 0; ch < kD / 32; ch++) {
          uint32_t r[32];
          tmem_ld32(t_row + (uint32_t)(ch * 32), r);
          tmem_wait_ld();
          if (!last) {
#pragma unroll
            for (int c8 = 0; c8 < 4; c8++) {
              const int c = ch * 32 + c8 * 8;
              uint32_t w[4];
#pragma unroll
              for (int e = 0; e < 4; e++) {
                const float v0 = act<GELU>(__uint_as_float(r[c8 * 8 + 2 * e]) + bl[c + 2 * e]);
                const float v1 = act<GELU>(__uint_as_float(r[c8 * 8 + 2 * e + 1]) + bl[c + 2 * e + 1]);
                w[e] = pack2<F16>(v0, v1);
              }
              st_shared_v4(a_base + sw128_off(row, c), w[0], w[1], w[2], w[3]);
            }
          } else {
#pragma unroll
            for (int e = 0; e < 32; e++)
              y = fmaf(sWo[ch * 32 + e], act<GELU>(__uint_as_float(r[e]) + bl[ch * 32 + e]), y);
          }
        }
        tc_fence_before();
        if (!last) {
          fence_proxy_async();
          mbar_arrive(&bars[wg]);
        }
      }
      if (valid) sink_store(sink, sidx, p, y + bo);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

size_t smem_bytes(int n_hidden) {
  return 1024 + (size_t)n_hidden * kTile + 2 * kTile + (size_t)64 * kQStride * 4 + (size_t)kMaxHidden * kD * 4 +
         (size_t)kD * 4 + 64;
}

}  // namespace tc

bool chain_tc_available() { return true; }

void launch_chain_tc(const float* z, int64_t B, int q, const DevNet& net, const Sink& sink, int num_sms,
                     cudaStream_t s) {
  if (B <= 0) return;
  const size_t sm = tc::smem_bytes(net.n_hidden);
  static bool attr = false;
  if (!attr) {
    const int mx = (int)tc::smem_bytes(kMaxHidden);
    cudaFuncSetAttribute(tc::k_chain_tc<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(tc::k_chain_tc<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(tc::k_chain_tc<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(tc::k_chain_tc<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    attr = true;
  }
  const int64_t rows = B * q;
  const int64_t tiles = (rows + tc::kRows - 1) / tc::kRows;
  const int grid = (int)(tiles < num_sms ? tiles : num_sms);
  const float* Qg = q == kQC ? net.Qc : net.Qf;
  if (net.f16) {
    if (net.gelu_tanh) tc::k_chain_tc<1, 1><<<grid, tc::kThreads, sm, s>>>(z, rows, q, Qg, net, sink);
    else tc::k_chain_tc<0, 1><<<grid, tc::kThreads, sm, s>>>(z, rows, q, Qg, net, sink);
  } else {
    if (net.gelu_tanh) tc::k_chain_tc<1, 0><<<grid, tc::kThreads, sm, s>>>(z, rows, q, Qg, net, sink);
    else tc::k_chain_tc<0, 0><<<grid, tc::kThreads, sm, s>>>(z, rows, q, Qg, net, sink);
  }
}

}  // namespace mfp
