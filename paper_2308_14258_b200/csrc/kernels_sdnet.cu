// kernels_sdnet.cu — SDNet boundary gather + embedding (N2 + N3) and the fp32
// SIMT MLP chain (N4-fp32) with the scatter fused into its epilogue (N5).
//
// PAPER.md: P:239 (1-D convolutions over g give the boundary embedding)
// (Eq. 5: U = phi(g W1^T (+) X W2^T), a broadcasted sum), P:241 (stack of
// linear layers each followed by GELU), P:43 (predictions written onto the
// centre lines, which are other subdomains' boundaries).  Architecture sizes:
// reading G7 (conv 1->8->1, k=5, circular padding, GELU after every conv layer,
// d=128, 3 hidden layers).
#include "device_common.cuh"

namespace mfp {

// ------------------------------------------------------------ N2+N3: embed
// A block embeds 64 subdomains per round.  Phase A (per warp, 8 subdomains):
// gather the 128 perimeter values (G1 order), conv1 (1 -> 8, k = 5, circular)
// + GELU and conv2 (8 -> 1) + GELU with each lane owning 4 consecutive
// positions; the circular neighbours come from the adjacent lanes by warp
// shuffles (no per-warp smem), e written k-major into smem.
// Phase B (whole block): z = e W1^T + b1 as a register-tiled 64 x 128 x 128
// SIMT GEMM — W1^T (64 KB, smem-resident) is read once per 64 subdomains.
// ~99 KB of smem per block: two blocks per SM.
// z is the boundary half of the split layer (Eq. 5); the query half
// Q = X W2^T is a per-query constant table built at init.
constexpr int kEmbWarps = 8;
constexpr int kEmbSub = 64;                  // subdomains per block round
constexpr int kEmbPerWarp = kEmbSub / kEmbWarps;
constexpr int kEs = kEmbSub + 4;             // padded row of e^T (bank spread)
template <int D>
constexpr int emb_smem() { return (kNB * D + kNB * kEs + 96 + D) * 4; }

// D = 128: ~99 KB, two blocks per SM; D = 256 (the wide variant, also the
// embed of the d = 256 tensor-core path): ~164 KB, one block per SM.
template <int GELU, int D>
__global__ void __launch_bounds__(kEmbWarps * 32, D == kD ? 2 : 1)
k_gather_embed(const float* __restrict__ lat, LatticeGeom L, const uint32_t* __restrict__ anchors,
               const float* __restrict__ gb, int64_t B, DevNet net, float* __restrict__ z) {
  extern __shared__ float smem[];
  float* sW1T = smem;                        // [128 k][D]
  float* sE = sW1T + kNB * D;                // e^T [128 k][68]
  float* sCw = sE + kNB * kEs;               // c1w[40] c1b[8] c2w[40] c2b[1]
  float* sB1 = sCw + 96;                     // b1 (the raw parameter block is not 16 B aligned)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    const float4* src = reinterpret_cast<const float4*>(net.W1T);
    float4* dst = reinterpret_cast<float4*>(sW1T);
    for (int i = threadIdx.x; i < kNB * D / 4; i += blockDim.x) dst[i] = __ldg(src + i);
    for (int i = threadIdx.x; i < D; i += blockDim.x) sB1[i] = __ldg(net.b1 + i);
    if (threadIdx.x < 40) sCw[threadIdx.x] = __ldg(net.conv1_w + threadIdx.x);
    if (threadIdx.x < 8) sCw[40 + threadIdx.x] = __ldg(net.conv1_b + threadIdx.x);
    if (threadIdx.x < 40) sCw[48 + threadIdx.x] = __ldg(net.conv2_w + threadIdx.x);
    if (threadIdx.x == 0) sCw[88] = __ldg(net.conv2_b);
  }
  __syncthreads();
  const int i0 = 4 * lane;                   // this lane's 4 consecutive perimeter positions
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  for (int64_t base = (int64_t)blockIdx.x * kEmbSub; base < B; base += (int64_t)gridDim.x * kEmbSub) {
    // ---- phase A: gather + conv stack, 8 subdomains per warp.  All 8
    // perimeter gathers are issued up front (one exposed L2 latency per round).
    float4 gpre[kEmbPerWarp];
#pragma unroll
    for (int j = 0; j < kEmbPerWarp; j++) {
      int64_t s = base + warp * kEmbPerWarp + j;
      if (s > B - 1) s = B - 1;
      gpre[j] = gb ? __ldg(reinterpret_cast<const float4*>(gb + s * kNB + i0)) : gather4(lat, L, __ldg(anchors + s), lane);
    }
#pragma unroll
    for (int j = 0; j < kEmbPerWarp; j++) {
      const int col = warp * kEmbPerWarp + j;
      const float gv4[4] = {gpre[j].x, gpre[j].y, gpre[j].z, gpre[j].w};
      float e[4];
      conv_stack<GELU>(gv4, lane, sCw, e);
#pragma unroll
      for (int p = 0; p < 4; p++) sE[(i0 + p) * kEs + col] = e[p];
    }
    __syncthreads();
    // ---- phase B: z[64 x D] = e[64 x 128] W1^T, thread = 4 subdomains x D/16
    // outputs (columns 4 tx + 64 j)
    {
      constexpr int NJ = D / 64;
      float acc[4][4 * NJ];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int jj = 0; jj < 4 * NJ; jj++) acc[i][jj] = 0.f;
#pragma unroll 4
      for (int k = 0; k < kNB; k++) {
        const float4 a = *reinterpret_cast<const float4*>(sE + k * kEs + ty * 4);
        const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int j = 0; j < NJ; j++) {
          const float4 w = *reinterpret_cast<const float4*>(sW1T + k * D + 64 * j + tx * 4);
          const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int i = 0; i < 4; i++)
#pragma unroll
            for (int jj = 0; jj < 4; jj++) acc[i][4 * j + jj] = fmaf(av[i], wv[jj], acc[i][4 * j + jj]);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const int64_t s = base + ty * 4 + i;
        if (s >= B) continue;
        float* zr = z + s * D;
#pragma unroll
        for (int j = 0; j < NJ; j++) {
          const float4 bb = *reinterpret_cast<const float4*>(sB1 + 64 * j + tx * 4);
          *reinterpret_cast<float4*>(zr + 64 * j + tx * 4) =
              make_float4(acc[i][4 * j] + bb.x, acc[i][4 * j + 1] + bb.y, acc[i][4 * j + 2] + bb.z, acc[i][4 * j + 3] + bb.w);
        }
      }
    }
    __syncthreads();
  }
}

void launch_gather_embed(const float* lat, const LatticeGeom& L, const uint32_t* anchors,
                         const float* gb, int64_t B, const DevNet& net, float* z, cudaStream_t s) {
  if (B <= 0) return;
  int64_t blocks = (B + kEmbSub - 1) / kEmbSub;
  const int per_sm = net.d == kD ? 2 : 1;   // resident blocks per SM
  if (blocks > per_sm * num_sms()) blocks = per_sm * num_sms();
#define MFP_EMB(G, D) k_gather_embed<G, D><<<(int)blocks, kEmbWarps * 32, emb_smem<D>(), s>>>(lat, L, anchors, gb, B, net, z)
  if (net.d == kD) {
    if (net.gelu_tanh == 2) MFP_EMB(2, kD); else if (net.gelu_tanh) MFP_EMB(1, kD); else MFP_EMB(0, kD);
  } else {
    if (net.gelu_tanh == 2) MFP_EMB(2, kD2); else if (net.gelu_tanh) MFP_EMB(1, kD2); else MFP_EMB(0, kD2);
  }
#undef MFP_EMB
}

// ------------------------------------------------------ N4-fp32: SIMT chain
// Rows are (subdomain, query) pairs packed densely: row = s*q + p.  A block
// owns a 64-row tile; activations live in H^T [D][68].  D = 128: the hidden
// weights (W^T, fp32, 3 x 64 KB) stay resident in shared memory for the whole
// persistent loop.  D = 256 (3 x 256 KB does not fit): each layer streams W^T
// through shared memory in K-chunks of 32 rows (32 KB).  Exact-erf GELU, fp32
// FMA: the parity twin of the tcgen05 path.
constexpr int kSimtRows = 64;
constexpr int kHTs = 68;  // padded row stride of H^T (bank spread)
constexpr int kWChunk = 32;   // D = 256: K rows of W^T per staged chunk

template <int D>
constexpr size_t simt_smem(int n_hidden) {
  return (D == kD ? (size_t)n_hidden * D * D * 4 : (size_t)kWChunk * D * 4) + (size_t)D * kHTs * 4;
}

template <int D>
__global__ void __launch_bounds__(256, 1)
k_chain_fp32(const float* __restrict__ z, int64_t total_rows, int q, int qpad,
             const float* __restrict__ QT, DevNet net, Sink sink) {
  constexpr bool kResident = (D == kD);
  constexpr int NJ = D / 64;                 // 4-column groups per thread
  extern __shared__ float smem[];
  const int nh = net.n_hidden;
  float* sW = smem;                          // resident [nh][k][n] or one [kWChunk][n] chunk
  float* sHT = smem + (kResident ? nh * D * D : kWChunk * D);   // [c][row] stride 68
  if (kResident) {
    const float4* src = reinterpret_cast<const float4*>(net.WhT);
    float4* dst = reinterpret_cast<float4*>(sW);
    for (int i = threadIdx.x; i < nh * D * D / 4; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t ntiles = (total_rows + kSimtRows - 1) / kSimtRows;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * kSimtRows;
    // layer 1 (Eq. 5): h = GELU(z[s] + Q[p]), broadcast sum of the two halves
    {
      const int r = tid & 63, c0 = tid >> 6;
      int64_t row = row0 + r;
      if (row >= total_rows) row = total_rows - 1;
      const int64_t s = row / q;
      const int p = (int)(row - s * q);
      for (int c = c0; c < D; c += 4) {
        const float v = __ldg(z + s * D + c) + __ldg(QT + (int64_t)c * qpad + p);
        sHT[c * kHTs + r] = gelu_erf(v);
      }
    }
    __syncthreads();
    for (int l = 0; l < nh; l++) {
      float acc[4][4 * NJ];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4 * NJ; j++) acc[i][j] = 0.f;
      for (int kc = 0; kc < D; kc += (kResident ? D : kWChunk)) {
        const float* W;
        if (kResident) {
          W = sW + l * D * D;
        } else {
          const float4* src = reinterpret_cast<const float4*>(net.WhT + ((int64_t)l * D + kc) * D);
          float4* dst = reinterpret_cast<float4*>(sW);
          for (int i = threadIdx.x; i < kWChunk * D / 4; i += blockDim.x) dst[i] = __ldg(src + i);
          __syncthreads();
          W = sW - kc * D;   // row k of W^T at W + k * D for k in [kc, kc + kWChunk)
        }
        const int kend = kResident ? D : kc + kWChunk;
#pragma unroll 4
        for (int k = kc; k < kend; k++) {
          const float4 a = *reinterpret_cast<const float4*>(sHT + k * kHTs + ty * 4);
          const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
          for (int j = 0; j < NJ; j++) {
            const float4 w = *reinterpret_cast<const float4*>(W + k * D + 64 * j + tx * 4);
            const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
              for (int jj = 0; jj < 4; jj++) acc[i][4 * j + jj] = fmaf(av[i], wv[jj], acc[i][4 * j + jj]);
          }
        }
        if (!kResident) __syncthreads();   // the chunk is overwritten next
      }
      __syncthreads();
      const float* bl = net.bh + l * D;
#pragma unroll
      for (int j = 0; j < 4 * NJ; j++) {
        const int c = 64 * (j >> 2) + tx * 4 + (j & 3);
        const float bb = __ldg(bl + c);
        float4 v;
        v.x = gelu_erf(acc[0][j] + bb);
        v.y = gelu_erf(acc[1][j] + bb);
        v.z = gelu_erf(acc[2][j] + bb);
        v.w = gelu_erf(acc[3][j] + bb);
        *reinterpret_cast<float4*>(sHT + c * kHTs + ty * 4) = v;
      }
      __syncthreads();
    }
    // head y = wo . h + bo, then the fused scatter (N5)
    if (tid < kSimtRows) {
      const int64_t row = row0 + tid;
      float y = 0.f;
#pragma unroll 8
      for (int c = 0; c < D; c++) y = fmaf(__ldg(net.wo + c), sHT[c * kHTs + tid], y);
      y += __ldg(net.bo);
      if (row < total_rows) {
        const int64_t s = row / q;
        sink_store(sink, s, (int)(row - s * q), y);
      }
    }
    __syncthreads();
  }
}

void launch_chain_fp32(const float* z, int64_t B, int q, const DevNet& net, const Sink& sink,
                       cudaStream_t s) {
  if (B <= 0) return;
  const int64_t rows = B * q;
  int64_t tiles = (rows + kSimtRows - 1) / kSimtRows;
  int blocks = (int)(tiles < num_sms() ? tiles : num_sms());
  const float* QT = q == kQC ? net.QTc : net.QTf;
  const int qpad = q == kQC ? 64 : kQF;
  if (net.d == kD)
    k_chain_fp32<kD><<<blocks, 256, simt_smem<kD>(net.n_hidden), s>>>(z, rows, q, qpad, QT, net, sink);
  else
    k_chain_fp32<kD2><<<blocks, 256, simt_smem<kD2>(net.n_hidden), s>>>(z, rows, q, qpad, QT, net, sink);
}

// Opt-in shared-memory sizes, set once from mfp_init (never inside a graph capture).
void sdnet_kernel_attributes() {
  cudaFuncSetAttribute(k_gather_embed<0, kD>, cudaFuncAttributeMaxDynamicSharedMemorySize, emb_smem<kD>());
  cudaFuncSetAttribute(k_gather_embed<1, kD>, cudaFuncAttributeMaxDynamicSharedMemorySize, emb_smem<kD>());
  cudaFuncSetAttribute(k_gather_embed<0, kD2>, cudaFuncAttributeMaxDynamicSharedMemorySize, emb_smem<kD2>());
  cudaFuncSetAttribute(k_gather_embed<1, kD2>, cudaFuncAttributeMaxDynamicSharedMemorySize, emb_smem<kD2>());
  cudaFuncSetAttribute(k_gather_embed<2, kD>, cudaFuncAttributeMaxDynamicSharedMemorySize, emb_smem<kD>());
  cudaFuncSetAttribute(k_gather_embed<2, kD2>, cudaFuncAttributeMaxDynamicSharedMemorySize, emb_smem<kD2>());
  cudaFuncSetAttribute(k_chain_fp32<kD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)simt_smem<kD>(kMaxHidden));
  cudaFuncSetAttribute(k_chain_fp32<kD2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)simt_smem<kD2>(kMaxHidden));
}

}  // namespace mfp
