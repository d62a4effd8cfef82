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
constexpr int kEmbSmem = (kNB * kD + kNB * kEs + 96 + kD) * 4;

template <int GELU>
__global__ void __launch_bounds__(kEmbWarps * 32, 2)
k_gather_embed(const float* __restrict__ lat, LatticeGeom L, const uint32_t* __restrict__ anchors,
               const float* __restrict__ gb, int64_t B, DevNet net, float* __restrict__ z) {
  extern __shared__ float smem[];
  float* sW1T = smem;                        // [128 k][128 d]
  float* sE = sW1T + kNB * kD;               // e^T [128 k][68]
  float* sCw = sE + kNB * kEs;               // c1w[40] c1b[8] c2w[40] c2b[1]
  float* sB1 = sCw + 96;                     // b1 (the raw parameter block is not 16 B aligned)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    const float4* src = reinterpret_cast<const float4*>(net.W1T);
    float4* dst = reinterpret_cast<float4*>(sW1T);
    for (int i = threadIdx.x; i < kNB * kD / 4; i += blockDim.x) dst[i] = __ldg(src + i);
    if (threadIdx.x < kD) sB1[threadIdx.x] = __ldg(net.b1 + threadIdx.x);
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
    // ---- phase B: z[64 x 128] = e[64 x 128] W1^T, thread = 4 subdomains x 8 outputs
    {
      float acc[4][8];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int jj = 0; jj < 8; jj++) acc[i][jj] = 0.f;
#pragma unroll 4
      for (int k = 0; k < kNB; k++) {
        const float4 a = *reinterpret_cast<const float4*>(sE + k * kEs + ty * 4);
        const float4 w0 = *reinterpret_cast<const float4*>(sW1T + k * kD + tx * 4);
        const float4 w1 = *reinterpret_cast<const float4*>(sW1T + k * kD + 64 + tx * 4);
        const float av[4] = {a.x, a.y, a.z, a.w};
        const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
          for (int jj = 0; jj < 8; jj++) acc[i][jj] = fmaf(av[i], wv[jj], acc[i][jj]);
      }
      const float4 b0 = *reinterpret_cast<const float4*>(sB1 + tx * 4);
      const float4 b1 = *reinterpret_cast<const float4*>(sB1 + 64 + tx * 4);
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const int64_t s = base + ty * 4 + i;
        if (s >= B) continue;
        float* zr = z + s * kD;
        *reinterpret_cast<float4*>(zr + tx * 4) =
            make_float4(acc[i][0] + b0.x, acc[i][1] + b0.y, acc[i][2] + b0.z, acc[i][3] + b0.w);
        *reinterpret_cast<float4*>(zr + 64 + tx * 4) =
            make_float4(acc[i][4] + b1.x, acc[i][5] + b1.y, acc[i][6] + b1.z, acc[i][7] + b1.w);
      }
    }
    __syncthreads();
  }
}

void launch_gather_embed(const float* lat, const LatticeGeom& L, const uint32_t* anchors,
                         const float* gb, int64_t B, const DevNet& net, float* z, cudaStream_t s) {
  if (B <= 0) return;
  int64_t blocks = (B + kEmbSub - 1) / kEmbSub;
  if (blocks > 2 * num_sms()) blocks = 2 * num_sms();   // two resident blocks per SM
  if (net.gelu_tanh)
    k_gather_embed<1><<<(int)blocks, kEmbWarps * 32, kEmbSmem, s>>>(lat, L, anchors, gb, B, net, z);
  else
    k_gather_embed<0><<<(int)blocks, kEmbWarps * 32, kEmbSmem, s>>>(lat, L, anchors, gb, B, net, z);
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
  const int64_t rows = B * q;
  int64_t tiles = (rows + kSimtRows - 1) / kSimtRows;
  int blocks = (int)(tiles < num_sms() ? tiles : num_sms());
  const float* QT = q == kQC ? net.QTc : net.QTf;
  const int qpad = q == kQC ? 64 : kQF;
  k_chain_fp32<<<blocks, 256, sm, s>>>(z, rows, q, qpad, QT, net, sink);
}

// Opt-in shared-memory sizes, set once from mfp_init (never inside a graph capture).
void sdnet_kernel_attributes() {
  cudaFuncSetAttribute(k_gather_embed<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kEmbSmem);
  cudaFuncSetAttribute(k_gather_embed<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kEmbSmem);
  cudaFuncSetAttribute(k_chain_fp32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)simt_smem(kMaxHidden));
}

}  // namespace mfp
