// kernels_embed_tc.cu — boundary gather + embedding (N2 + N3) for the
// tensor-core paths (precision bf16 / fp16).
//
// PAPER.md P:239 (1-D convolutions over g give the boundary embedding) and
// Eq. 5 P:270 (z = g W1^T is computed once per boundary and broadcast over
// the queries).  Per round a CTA embeds up to 128 subdomains:
//   * a producer warp stages every subdomain's four perimeter edges (a1) into
//     shared memory with TMA bulk copies (cp.async.bulk, one 128/144-byte edge
//     segment per lane, completion counted in bytes on the consuming warp's
//     mbarrier); it issues a warp's next round as soon as that warp has pulled
//     the current one into registers, so the gathers overlap the conv stack,
//     the MMAs and the z stores.  The W1 images arrive the same way before the
//     PDL wait (weights do not depend on the previous kernel);
//   * 16 warps x 8 subdomains: the 128 perimeter values (G1 order; lane l owns
//     positions 4l..4l+3) from the staging slots, conv1 1->8 / conv2 8->1
//     (k = 5, circular) + GELU in registers with warp-shuffle windows;
//   * the embedding e (fp32) is split e = e_hi + e_lo into two bf16 SWIZZLE_128B
//     A operands; W1 = W1_hi + W1_lo is resident as two bf16 B operands; one
//     elected thread issues the three products hi.hi + hi.lo + lo.hi
//     (tcgen05.mma, M = N = 128, 24 x K16) into a TMEM accumulator, so
//     z = W1 e keeps ~fp32 accuracy (error ~2^-16 of the terms) at tensor-core
//     speed;
//   * 16 warps drain TMEM (tcgen05.ld, 32 columns each) and store z + b1.
// The fp32 path keeps the SIMT embed (kernels_sdnet.cu).
#include <cuda_bf16.h>

#include "tc_common.cuh"

namespace mfp {
namespace emb {

using namespace tcx;

constexpr int kRowsE = 128;              // subdomains per round (UMMA M)
constexpr int kThreadsE = 512;           // 16 warps
constexpr int kImg = kRowsE * kNB * 2;   // 32 KB bf16 image

// W1 buffer (hi + lo images of 128 output rows) + A hi / lo + staging + vectors + barriers
constexpr size_t smem_bytes(int D) { return 4 * (size_t)kImg + (size_t)kRowsE * 576 + 4 * (96 + D) + 8 * 19 + 16; }

// The conv stack (G7: conv1d 1->8 -> GELU -> conv1d 8->1 -> GELU, k = 5,
// circular) of N subdomains, interleaved for ILP.  Lane l owns perimeter
// positions 4l..4l+3; the circular windows come from the neighbour lanes by
// shuffles.  Channels are packed in PAIRS (2c, 2c+1) into fp32x2 values, so
// every FFMA2 takes its weight pair as ONE 64-bit constant-bank operand
// (DevNet::convw, pair order) and its input as a scalar broadcast operand:
// no register moves to build operand pairs.  conv2 accumulates the even and
// odd channels in the two halves of a pair, added at the end.
template <int GELU>
__device__ __forceinline__ f2 ch_act2(f2 x) {   // conv1 outputs: 2 GELU (GELU 1 / 2; conv2 weights hold w / 2) or GELU (0)
  if constexpr (GELU == 1) {
    float u0, u1;
    f2_split(fmul2(x, ffma2(fmul2(x, x), f2_make(kGF1, kGF1), f2_make(kGF0, kGF0))), u0, u1);
    return ffma2(x, f2_make(tanh_approx(u0), tanh_approx(u1)), x);
  } else {
    float a, b;
    f2_split(x, a, b);
    if constexpr (GELU == 2) return f2_make(gelu2_acc(a), gelu2_acc(b));
    else return f2_make(gelu_erf(a), gelu_erf(b));
  }
}
template <int GELU>
__device__ __forceinline__ f2 emb_act2(f2 x) {   // the embedding itself: GELU (proper scale)
  if constexpr (GELU == 2) {
    float a, b;
    f2_split(x, a, b);
    return f2_make(0.5f * gelu2_acc(a), 0.5f * gelu2_acc(b));
  } else if constexpr (GELU == 1) {
    float u0, u1;
    f2_split(fmul2(x, ffma2(fmul2(x, x), f2_make(kGF1, kGF1), f2_make(kGF0, kGF0))), u0, u1);
    const f2 hx = fmul2(x, f2_make(0.5f, 0.5f));
    return ffma2(hx, f2_make(tanh_approx(u0), tanh_approx(u1)), hx);   // x/2 (1 + tanh u)
  } else {
    float a, b;
    f2_split(x, a, b);
    return f2_make(gelu_erf(a), gelu_erf(b));
  }
}
__device__ __forceinline__ f2 cpair(const DevNet& net, int i) {   // 64-bit constant-bank operand
  return f2{*reinterpret_cast<const uint64_t*>(net.convw + i)};
}
__device__ __forceinline__ f2 bcast(float x) { return f2_make(x, x); }   // FFMA2 scalar (.F32) operand
__device__ __forceinline__ f2 shfl2(f2 v, int src) { return f2{__shfl_sync(0xffffffffu, v.v, src)}; }

template <int GELU, int N>
__device__ __forceinline__ void conv_stack(const float (&g)[N][4], int lane, const DevNet& net, float (&e)[N][4]) {
  const int left = (lane + 31) & 31, right = (lane + 1) & 31;
  float win[N][8];
#pragma unroll
  for (int n = 0; n < N; n++) {
    win[n][0] = __shfl_sync(0xffffffffu, g[n][2], left);
    win[n][1] = __shfl_sync(0xffffffffu, g[n][3], left);
#pragma unroll
    for (int p = 0; p < 4; p++) win[n][2 + p] = g[n][p];
    win[n][6] = __shfl_sync(0xffffffffu, g[n][0], right);
    win[n][7] = __shfl_sync(0xffffffffu, g[n][1], right);
  }
  f2 acc[N][4];   // conv2: (even channels, odd channels) per position
#pragma unroll
  for (int n = 0; n < N; n++)
#pragma unroll
    for (int p = 0; p < 4; p++) acc[n][p] = f2_make(net.convw[88], 0.0f);
#pragma unroll
  for (int cp = 0; cp < kC1 / 2; cp++) {
    const f2 bias = cpair(net, 40 + 2 * cp);
    f2 aw[N][8];
#pragma unroll
    for (int n = 0; n < N; n++)
#pragma unroll
      for (int p = 0; p < 4; p++) {
        f2 v = ffma2(bcast(win[n][p]), cpair(net, 2 * (cp * kK)), bias);
#pragma unroll
        for (int t = 1; t < kK; t++) v = ffma2(bcast(win[n][p + t]), cpair(net, 2 * (cp * kK + t)), v);
        aw[n][2 + p] = ch_act2<GELU>(v);
      }
#pragma unroll
    for (int n = 0; n < N; n++) {
      aw[n][0] = shfl2(aw[n][4], left);
      aw[n][1] = shfl2(aw[n][5], left);
      aw[n][6] = shfl2(aw[n][2], right);
      aw[n][7] = shfl2(aw[n][3], right);
    }
#pragma unroll
    for (int n = 0; n < N; n++)
#pragma unroll
      for (int p = 0; p < 4; p++)
#pragma unroll
        for (int t = 0; t < kK; t++) acc[n][p] = ffma2(cpair(net, 48 + 2 * (cp * kK + t)), aw[n][p + t], acc[n][p]);
  }
#pragma unroll
  for (int n = 0; n < N; n++) {
    float s[4];
#pragma unroll
    for (int p = 0; p < 4; p++) {
      float lo, hi;
      f2_split(acc[n][p], lo, hi);
      s[p] = lo + hi;
    }
    f2_split(emb_act2<GELU>(f2_make(s[0], s[1])), e[n][0], e[n][1]);
    f2_split(emb_act2<GELU>(f2_make(s[2], s[3])), e[n][2], e[n][3]);
  }
}

// Staged perimeter of one subdomain (TMA bulk copies of the four edge
// segments): bottom [lx, lx+32) at 0, right [ly, ly+32) at 144, top
// [lx, lx+36) at 288 and left [ly, ly+36) at 432 (floats; the reversed edges
// need points lx+1..lx+32, and a bulk copy's source must be 16-byte aligned, so
// their window starts at the 64-byte aligned corner).  A gb batch row (512 B)
// is staged contiguously at 0.
constexpr int kSlotB = 576;
constexpr uint32_t kEdgeB = 4 * kM, kEdgeRB = 4 * (kM + 4);

// D = 256: z has two 128-column halves; the W1 buffer holds one half's hi / lo
// images at a time (the three images would not fit beside the staging), so the
// MMA issuer runs half A, waits for those MMAs, reloads the buffer with half B
// by TMA and runs it; the order alternates per round so the half loaded last is
// reused by the next round's first MMAs.
template <int GELU, int D>
__global__ void __launch_bounds__(kThreadsE, 1)
k_embed_tc(const float* __restrict__ lat, LatticeGeom L, const uint32_t* __restrict__ anchors,
           const float* __restrict__ gb, int64_t B, int rows, DevNet net, float* __restrict__ z) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sWhi = smem_raw;
  uint8_t* sWlo = sWhi + kImg;
  uint8_t* sAhi = sWlo + kImg;
  uint8_t* sAlo = sAhi + kImg;
  uint8_t* sStage = sAlo + kImg;                         // [128][kSlotB]
  float* sB1 = reinterpret_cast<float*>(sStage + kRowsE * kSlotB) + 96;   // (96 floats spare)
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB1 + D);   // [0] MMA done, [1] W1 landed, [2] W1 free
  uint64_t* full = bar + 3;                                // [3..18] warp's perimeters landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(full + 16);
  constexpr int NH = D / 128;                              // W1 halves
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < D; i += kThreadsE) sB1[i] = __ldg(net.b1 + i);
  if ((smem_u32(smem_raw) & 1023u) != 0u) __trap();
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    for (int w = 0; w < 16; w++) mbar_init(&full[w], 1);   // lane 0's arrive.expect_tx + the copies' bytes
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(D)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // W1 = W1_hi + W1_lo images (weights: no dependence on the previous grid)
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar[1], 2u * kImg);
    for (int i = 0; i < 4; i++)
      bulk_g2s(smem_u32(sWhi) + i * (kImg / 2), reinterpret_cast<const uint8_t*>(net.W1img) + i * (kImg / 2),
               kImg / 2, &bar[1]);
  }
  pdl_launch_dependents();
  pdl_wait();      // the lattice (previous phase's scatter) and z's readers complete from here on
  // `rows` (a multiple of 16, <= 128) subdomains per round: the batch spread
  // over every SM (C5: 112 rows on 146 CTAs), small batches (a rank's share on
  // 8 GPUs) with fewer subdomains per warp, so the serial conv work per warp
  // shrinks with the batch; rows >= `rows` of the 128-row MMA are don't-care
  // (rows are independent in the MMA, never stored)
  const int pw = rows >> 4;   // subdomains per warp (1..8)
  const int64_t step = (int64_t)gridDim.x * rows;

  // ---- a1: TMA bulk copies of this warp's pw perimeters (four edge segments
  // each, one copy per lane) into its staging slots, completing on full[warp];
  // a warp issues round r + 1 as soon as it has pulled round r into registers,
  // so the gathers overlap the conv stack, the MMAs and the z stores
  auto stage = [&](int64_t base) {
    if (lane == 0) mbar_arrive_expect_tx(&full[warp], (uint32_t)pw * (gb ? 4u * kNB : 2u * (kEdgeB + kEdgeRB)));
    __syncwarp();
    const int j = lane >> 2, e = lane & 3;
    if (j < pw) {
      int64_t s = base + warp * pw + j;
      if (s > B - 1) s = B - 1;
      const uint32_t slot = smem_u32(sStage) + (uint32_t)((warp * pw + j) * kSlotB);
      if (gb) {
        if (e == 0) bulk_g2s(slot, gb + s * kNB, 4u * kNB, &full[warp]);
      } else {
        int a, b;
        unpack_anchor(__ldg(anchors + s), a, b);
        const int lx = kH * a, ly = kH * b;
        const float* src = e == 0 ? lat + (int64_t)b * L.strideH + lx
                         : e == 1 ? lat + L.offV + (int64_t)(a + 2) * L.strideV + ly
                         : e == 2 ? lat + (int64_t)(b + 2) * L.strideH + lx
                                  : lat + L.offV + (int64_t)a * L.strideV + ly;
        bulk_g2s(slot + (uint32_t)e * 144u, src, e < 2 ? kEdgeB : kEdgeRB, &full[warp]);
      }
    }
  };
  {
    const int i0 = 4 * lane;
    const uint32_t a_hi = smem_u32(sAhi), a_lo = smem_u32(sAlo);
    const int edge = lane >> 3, t0 = 4 * (lane & 7);
    // byte offset of this lane's first value inside a staging slot
    const uint32_t st_lane = smem_u32(sStage) + 4u * (uint32_t)(gb ? i0 : edge < 2 ? 36 * edge + t0 : 36 * edge + kM - t0);
    uint32_t phase = 0u, pf = 0u;
    uint32_t wph = 0u, fph = 0u;   // (thread 0) W1-landed / W1-free barrier parities
    bool w1_pending = true;        // the prologue load not waited for yet
    int round = 0;
    if ((int64_t)blockIdx.x * rows < B) stage((int64_t)blockIdx.x * rows);
    for (int64_t base = (int64_t)blockIdx.x * rows; base < B; base += step) {
      // ---- this warp's pw perimeters from the staging slots (G1 order; lane l
      // owns positions 4l..4l+3)
      mbar_wait(&full[warp], pf);
      pf ^= 1u;
      // smem reads right before use (2 subdomains live at a time), 32-bit
      // shared addresses: lane offset within a slot fixed per lane
      auto perim4 = [&](int j) -> float4 {
        const uint32_t sl = st_lane + (uint32_t)((warp * pw + j) * kSlotB);
        float4 v;
        if (gb || edge < 2) {
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(sl));
        } else {
          asm volatile("ld.shared.f32 %0, [%4];\n\tld.shared.f32 %1, [%4+-4];\n\tld.shared.f32 %2, [%4+-8];\n\tld.shared.f32 %3, [%4+-12];"
                       : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(sl));
        }
        return v;
      };
      // e = e_hi + e_lo, both bf16 (round to nearest), into the two A operands
      auto store_row = [&](int row, const float (&e)[4]) {
        uint32_t h01, h23, l01, l23;
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h01) : "f"(e[1]), "f"(e[0]));
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h23) : "f"(e[3]), "f"(e[2]));
        const float r0 = e[0] - __uint_as_float(h01 << 16), r1 = e[1] - __uint_as_float(h01 & 0xffff0000u);
        const float r2 = e[2] - __uint_as_float(h23 << 16), r3 = e[3] - __uint_as_float(h23 & 0xffff0000u);
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(l01) : "f"(r1), "f"(r0));
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(l23) : "f"(r3), "f"(r2));
        const uint32_t off = sw128_off(row, i0) + (uint32_t)((i0 & 7) * 2);
        asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(a_hi + off), "r"(h01), "r"(h23) : "memory");
        asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(a_lo + off), "r"(l01), "r"(l23) : "memory");
      };
      // two subdomains interleaved per step (ILP), an odd last one alone
#pragma unroll 1
      for (int jp = 0; jp < pw; jp += 2) {
        if (jp + 1 < pw) {
          const float4 ga = perim4(jp), gb4 = perim4(jp + 1);
          const float g[2][4] = {{ga.x, ga.y, ga.z, ga.w}, {gb4.x, gb4.y, gb4.z, gb4.w}};
          float e[2][4];
          conv_stack<GELU, 2>(g, lane, net, e);
          store_row(warp * pw + jp, e[0]);
          store_row(warp * pw + jp + 1, e[1]);
        } else {
          const float4 ga = perim4(jp);
          const float g[1][4] = {{ga.x, ga.y, ga.z, ga.w}};
          float e[1][4];
          conv_stack<GELU, 1>(g, lane, net, e);
          store_row(warp * pw + jp, e[0]);
        }
      }
      // next round's perimeters: the slots' generic-proxy reads (long since
      // consumed) are ordered before the async-proxy (TMA) writes into them
      fence_proxy_async();
      __syncwarp();
      if (base + step < B) stage(base + step);
      __syncthreads();
      // ---- z = e W1^T on the tensor core: hi.hi + hi.lo + lo.hi (per W1 half)
      if (threadIdx.x == 0) {
        const uint32_t w_hi = smem_u32(sWhi), w_lo = smem_u32(sWlo);
        for (int hh = 0; hh < NH; hh++) {
          const int h = (NH == 2 && (round & 1)) ? 1 - hh : hh;
          if (hh > 0) {
            // the buffer is overwritten with half h once the MMAs reading it are done
            mma_commit(&bar[2]);
            mbar_wait(&bar[2], fph);
            fph ^= 1u;
            mbar_arrive_expect_tx(&bar[1], 2u * kImg);
            for (int i = 0; i < 4; i++)
              bulk_g2s(smem_u32(sWhi) + i * (kImg / 2),
                       reinterpret_cast<const uint8_t*>(net.W1img) + (size_t)h * 2 * kImg + i * (kImg / 2), kImg / 2,
                       &bar[1]);
            w1_pending = true;
          }
          if (w1_pending) {
            mbar_wait(&bar[1], wph);
            wph ^= 1u;
            w1_pending = false;
          }
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(128 * h);
#pragma unroll
          for (int k = 0; k < kNB / 16; k++) {
            const uint32_t off = (uint32_t)((k >> 2) * 16384 + (k & 3) * 32);
            mma_f16<0>(d, sw128_desc(a_hi + off), sw128_desc(w_hi + off), k > 0 ? 1u : 0u);
            mma_f16<0>(d, sw128_desc(a_hi + off), sw128_desc(w_lo + off), 1u);
            mma_f16<0>(d, sw128_desc(a_lo + off), sw128_desc(w_hi + off), 1u);
          }
        }
        mma_commit(&bar[0]);
      }
      round++;
      mbar_wait(&bar[0], phase);
      phase ^= 1u;
      tc_fence_after();
      // ---- drain: warp w reads lanes 32 (w % 4).., columns 32 NH (w / 4)..
      {
        const int quad = warp & 3, cb = warp >> 2;
        const int64_t s = base + quad * 32 + lane;
#pragma unroll
        for (int hc = 0; hc < NH; hc++) {
          const int col = (cb * NH + hc) * 32;
          uint32_t r[32];
          tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)col, r);
          tmem_wait_ld();
          if (quad * 32 + lane < rows && s < B) {
            float4* dst = reinterpret_cast<float4*>(z + s * D + col);
            const float* bb = sB1 + col;
#pragma unroll
            for (int v = 0; v < 8; v++)
              dst[v] = make_float4(__uint_as_float(r[4 * v]) + bb[4 * v], __uint_as_float(r[4 * v + 1]) + bb[4 * v + 1],
                                   __uint_as_float(r[4 * v + 2]) + bb[4 * v + 2], __uint_as_float(r[4 * v + 3]) + bb[4 * v + 3]);
          }
        }
      }
      tc_fence_before();
      __syncthreads();   // A operands and the accumulator are reused next round
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(D) : "memory");
  }
}

}  // namespace emb

bool embed_tc_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MFP_EMBED_SIMT");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

void embed_tc_kernel_attributes() {
  const int a = (int)emb::smem_bytes(kD), b = (int)emb::smem_bytes(kD2);
  cudaFuncSetAttribute(emb::k_embed_tc<0, kD>, cudaFuncAttributeMaxDynamicSharedMemorySize, a);
  cudaFuncSetAttribute(emb::k_embed_tc<1, kD>, cudaFuncAttributeMaxDynamicSharedMemorySize, a);
  cudaFuncSetAttribute(emb::k_embed_tc<2, kD>, cudaFuncAttributeMaxDynamicSharedMemorySize, a);
  cudaFuncSetAttribute(emb::k_embed_tc<0, kD2>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(emb::k_embed_tc<1, kD2>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(emb::k_embed_tc<2, kD2>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
}

void launch_embed_tc(const float* lat, const LatticeGeom& L, const uint32_t* anchors, const float* gb,
                     int64_t B, const DevNet& net, float* z, cudaStream_t s) {
  if (B <= 0) return;
  // rows per CTA round: the smallest multiple of 16 that covers B over the SMs
  const int sms = num_sms();
  int64_t per = (B + sms - 1) / sms;
  int rows = (int)((per + 15) / 16) * 16;
  if (rows > emb::kRowsE) rows = emb::kRowsE;
  if (rows < 16) rows = 16;
  int64_t blocks = (B + rows - 1) / rows;
  if (blocks > sms) blocks = sms;
  const size_t sm = emb::smem_bytes(net.d);
#define MFP_EMB(G, D) launch_pdl(emb::k_embed_tc<G, D>, (int)blocks, emb::kThreadsE, sm, s, lat, L, anchors, gb, B, rows, net, z)
  if (net.d == kD2) {
    if (net.gelu_tanh == 2) MFP_EMB(2, kD2); else if (net.gelu_tanh == 1) MFP_EMB(1, kD2); else MFP_EMB(0, kD2);
  } else {
    if (net.gelu_tanh == 2) MFP_EMB(2, kD); else if (net.gelu_tanh == 1) MFP_EMB(1, kD); else MFP_EMB(0, kD);
  }
#undef MFP_EMB
}

}  // namespace mfp
