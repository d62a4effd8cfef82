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
// One warp per subdomain.  Shared memory: W1^T (64 KB) + conv weights +
// per-warp scratch.  z = W1 e + b1 is the boundary half of the split layer; the
// query half Q = X W2^T is a per-query constant table built at init.
constexpr int kEmbWarps = 8;
constexpr int kEmbSmem = (kNB * kD + 96 + kEmbWarps * (kNB + kC1 * kNB + kNB)) * 4;

__global__ void __launch_bounds__(kEmbWarps * 32, 2)
k_gather_embed(const float* __restrict__ lat, LatticeGeom L, const uint32_t* __restrict__ anchors,
               const float* __restrict__ gb, int64_t B, DevNet net, float* __restrict__ z) {
  extern __shared__ float smem[];
  float* sW1T = smem;                        // [128][128]
  float* sCw = sW1T + kNB * kD;              // c1w[40] c1b[8] c2w[40] c2b[1]
  float* sWarp = sCw + 96;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    const float4* src = reinterpret_cast<const float4*>(net.W1T);
    float4* dst = reinterpret_cast<float4*>(sW1T);
    for (int i = threadIdx.x; i < kNB * kD / 4; i += blockDim.x) dst[i] = __ldg(src + i);
    if (threadIdx.x < 40) sCw[threadIdx.x] = __ldg(net.conv1_w + threadIdx.x);
    if (threadIdx.x < 8) sCw[40 + threadIdx.x] = __ldg(net.conv1_b + threadIdx.x);
    if (threadIdx.x < 40) sCw[48 + threadIdx.x] = __ldg(net.conv2_w + threadIdx.x);
    if (threadIdx.x == 0) sCw[88] = __ldg(net.conv2_b);
  }
  __syncthreads();
  float* g = sWarp + warp * (kNB + kC1 * kNB + kNB);
  float* c1 = g + kNB;
  float* e = c1 + kC1 * kNB;
  const int64_t nwarps = (int64_t)gridDim.x * kEmbWarps;
  for (int64_t s = (int64_t)blockIdx.x * kEmbWarps + warp; s < B; s += nwarps) {
    // gather ĝ in G1 order: 4 edges x 32 contiguous values (coalesced)
    if (gb) {
#pragma unroll
      for (int e4 = 0; e4 < 4; e4++) g[e4 * 32 + lane] = __ldg(gb + s * kNB + e4 * 32 + lane);
    } else {
      int a, b;
      unpack_anchor(__ldg(anchors + s), a, b);
#pragma unroll
      for (int e4 = 0; e4 < 4; e4++)
        g[e4 * 32 + lane] = lat[perim_cell(a, b, e4 * 32 + lane, L.strideH, L.strideV, L.offV)];
    }
    __syncwarp();
    // conv1: 1 -> 8 channels, k = 5, circular padding 2, GELU
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int i = lane + 32 * u;
      float gv[kK];
#pragma unroll
      for (int t = 0; t < kK; t++) gv[t] = g[(i + t - 2) & (kNB - 1)];
#pragma unroll
      for (int o = 0; o < kC1; o++) {
        float acc = sCw[40 + o];
#pragma unroll
        for (int t = 0; t < kK; t++) acc = fmaf(sCw[o * kK + t], gv[t], acc);
        c1[o * kNB + i] = gelu_erf(acc);
      }
    }
    __syncwarp();
    // conv2: 8 -> 1 channel, GELU -> e (ch_last * 4m = 128)
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int i = lane + 32 * u;
      float acc = sCw[88];
#pragma unroll
      for (int o = 0; o < kC1; o++)
#pragma unroll
        for (int t = 0; t < kK; t++) acc = fmaf(sCw[48 + o * kK + t], c1[o * kNB + ((i + t - 2) & (kNB - 1))], acc);
      e[i] = gelu_erf(acc);
    }
    __syncwarp();
    // z = W1 e + b1
    float acc[4];
#pragma unroll
    for (int u = 0; u < 4; u++) acc[u] = 0.f;
#pragma unroll 4
    for (int k = 0; k < kNB; k++) {
      const float ek = e[k];
#pragma unroll
      for (int u = 0; u < 4; u++) acc[u] = fmaf(sW1T[k * kD + lane + 32 * u], ek, acc[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; u++) z[s * kD + lane + 32 * u] = acc[u] + __ldg(net.b1 + lane + 32 * u);
    __syncwarp();
  }
}

void launch_gather_embed(const float* lat, const LatticeGeom& L, const uint32_t* anchors,
                         const float* gb, int64_t B, const DevNet& net, float* z, cudaStream_t s) {
  if (B <= 0) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gather_embed, cudaFuncAttributeMaxDynamicSharedMemorySize, kEmbSmem);
    attr = true;
  }
  int64_t blocks = (B + kEmbWarps - 1) / kEmbWarps;
  if (blocks > 148 * 2) blocks = 148 * 2;
  k_gather_embed<<<(int)blocks, kEmbWarps * 32, kEmbSmem, s>>>(lat, L, anchors, gb, B, net, z);
}

// ------------------------------------------------------ N4-fp32: SIMT chain
// Rows are (subdomain, query) pairs packed densely: row = s*q + p.  A block
// owns a 64-row tile; the hidden weights (W^T, fp32) stay resident in shared
// memory for the whole persistent loop; activations live in H^T [128][68].
// Exact-erf GELU, fp32 FMA: the parity twin of the tcgen05 path.
constexpr int kSimtRows = 64;
constexpr int kHTs = 68;  // padded row stride of H^T (bank spread)

static size_t simt_smem(int n_hidden) {
  return (size_t)n_hidden * kD * kD * 4 + (size_t)kD * kHTs * 4;
}

__global__ void __launch_bounds__(256, 1)
k_chain_fp32(const float* __restrict__ z, int64_t total_rows, int q, int qpad,
             const float* __restrict__ QT, DevNet net, Sink sink) {
  extern __shared__ float smem[];
  const int nh = net.n_hidden;
  float* sW = smem;                          // [nh][k][n]
  float* sHT = smem + nh * kD * kD;          // [c][row] stride 68
  {
    const float4* src = reinterpret_cast<const float4*>(net.WhT);
    float4* dst = reinterpret_cast<float4*>(sW);
    for (int i = threadIdx.x; i < nh * kD * kD / 4; i += blockDim.x) dst[i] = __ldg(src + i);
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
      for (int c = c0; c < kD; c += 4) {
        const float v = __ldg(z + s * kD + c) + __ldg(QT + (int64_t)c * qpad + p);
        sHT[c * kHTs + r] = gelu_erf(v);
      }
    }
    __syncthreads();
    for (int l = 0; l < nh; l++) {
      const float* W = sW + l * kD * kD;
      float acc[4][8];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) acc[i][j] = 0.f;
#pragma unroll 4
      for (int k = 0; k < kD; k++) {
        const float4 a = *reinterpret_cast<const float4*>(sHT + k * kHTs + ty * 4);
        const float4 w0 = *reinterpret_cast<const float4*>(W + k * kD + tx * 4);
        const float4 w1 = *reinterpret_cast<const float4*>(W + k * kD + 64 + tx * 4);
        const float av[4] = {a.x, a.y, a.z, a.w};
        const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
          for (int j = 0; j < 8; j++) acc[i][j] = fmaf(av[i], wv[j], acc[i][j]);
      }
      __syncthreads();
      const float* bl = net.bh + l * kD;
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const int c = (j < 4) ? tx * 4 + j : 64 + tx * 4 + (j - 4);
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
      for (int c = 0; c < kD; c++) y = fmaf(__ldg(net.wo + c), sHT[c * kHTs + tid], y);
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
  const size_t sm = simt_smem(net.n_hidden);
  static size_t attr = 0;
  if (attr < sm) {
    cudaFuncSetAttribute(k_chain_fp32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = sm;
  }
  const int64_t rows = B * q;
  int64_t tiles = (rows + kSimtRows - 1) / kSimtRows;
  int blocks = (int)(tiles < 148 ? tiles : 148);
  const float* QT = q == kQC ? net.QTc : net.QTf;
  const int qpad = q == kQC ? 64 : kQF;
  k_chain_fp32<<<blocks, 256, sm, s>>>(z, rows, q, qpad, QT, net, sink);
}

}  // namespace mfp
