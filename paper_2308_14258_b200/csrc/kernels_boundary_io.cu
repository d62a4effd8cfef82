// kernels_boundary_io.cu — the paper's "Boundaries IO" as standalone
// kernels: the phase gather (a1, N2), the centre-line scatter with the per-block
// update norm (a6, N5), and the convergence reduction of the block maxima (a8).
//
// In the solve these steps are fused into their neighbours (the gather into the
// embed, the scatter into the chain epilogue).  The standalone
// forms are the unfused pipeline gather -> mfp_sdnet_batch -> scatter of one
// phase ("predict ... for all subdomains of one batch ... update the
// boundaries"), and the HBM-roofline evidence of north_star: both are pure data
// movement, so they are measured against the copy bandwidth on lattices larger
// than L2 (bench.py "boundary_io").
//
// Layout: every perimeter edge of a subdomain is one contiguous
// 32-float segment of the line lattice (bottom / right forward, top / left
// reversed); every centre line one contiguous 31-float segment.
#include "device_common.cuh"

namespace mfp {

constexpr int kIoWarps = 8;   // 256 threads
constexpr int kIoUnroll = 4;  // subdomains per warp per round: 4 x 512 B of loads in flight

// ------------------------------------------------------------ a1: phase gather
// gb[s][0..127] = perimeter of subdomain s in G1 order.  One warp per subdomain:
// lane l moves perimeter entries 4l..4l+3 (edge l/8) — one 16-byte load for the
// forward edges, four scalar loads (one coalesced 128 B span per warp) for the
// reversed ones — and one coalesced 16-byte store, so a warp writes 512
// contiguous bytes per subdomain.  Each warp keeps kIoUnroll subdomains' loads
// in flight before storing (memory-level parallelism for HBM latency).
__global__ void __launch_bounds__(kIoWarps * 32)
k_gather_phase(const float* __restrict__ lat, LatticeGeom L, const uint32_t* __restrict__ anchors, int64_t B,
               float* __restrict__ gb) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)blockIdx.x * kIoWarps + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * kIoWarps;
  for (int64_t s0 = w0 * kIoUnroll; s0 < B; s0 += nw * kIoUnroll) {
    float4 v[kIoUnroll];
#pragma unroll
    for (int u = 0; u < kIoUnroll; u++)
      if (s0 + u < B) v[u] = gather4(lat, L, __ldg(anchors + s0 + u), lane);
#pragma unroll
    for (int u = 0; u < kIoUnroll; u++)
      if (s0 + u < B) __stcs(reinterpret_cast<float4*>(gb + (s0 + u) * kNB) + lane, v[u]);
  }
}

// ---------------------------------------------- a6: scatter + per-block update norm
// For each subdomain s: the 61 predictions pred[s][p] (G3 order) overwrite the
// centre-line cells (the centre point in both line arrays), and the block
// accumulates max |new - old| over the cells it overwrites (warp shuffles, then
// one shared-memory step).  blockmax[blockIdx.x] = that maximum (fp32 bits) and
// bit 31 of blockflag set on a non-finite prediction.  Cells of one phase are
// written by exactly one subdomain, so the result is order independent.
__global__ void __launch_bounds__(kIoWarps * 32, 5)
k_scatter_phase(float* __restrict__ lat, LatticeGeom L, const uint32_t* __restrict__ anchors, int64_t B,
                const float* __restrict__ pred, unsigned int* __restrict__ blockmax) {
  __shared__ float red[kIoWarps];
  __shared__ int bad_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) bad_s = 0;
  __syncthreads();
  const int64_t nw = (int64_t)gridDim.x * kIoWarps;
  float m = 0.f;
  bool bad = false;
  const bool two = lane + 32 < kQC;
  // kIoUnroll subdomains per warp per round: every load of the round (predictions
  // and old values) is issued before the first store, so a warp keeps
  // 4 x ~0.5 KB in flight instead of one dependent load/store pair at a time.
  // Cell indices are 32-bit (a rank's lattice holds < 2^31 cells; checked at
  // launch), which keeps the kernel at <= 48 registers: 5 resident blocks per SM.
  for (int64_t s0 = ((int64_t)blockIdx.x * kIoWarps + warp) * kIoUnroll; s0 < B; s0 += nw * kIoUnroll) {
    int32_t c0[kIoUnroll], c1[kIoUnroll], cd[kIoUnroll];   // cd: the centre's second copy or -1
    float y0[kIoUnroll], y1[kIoUnroll], o0[kIoUnroll], o1[kIoUnroll];
#pragma unroll
    for (int u = 0; u < kIoUnroll; u++) {
      const int64_t s = s0 + u < B ? s0 + u : B - 1;   // tail: clamp (stores are skipped)
      int a, b;
      unpack_anchor(__ldg(anchors + s), a, b);
      int64_t d0c, d1;
      c0[u] = (int32_t)centre_cell(a, b, lane, L.strideH, L.strideV, L.offV, &d0c);
      cd[u] = (int32_t)d0c;
      c1[u] = two ? (int32_t)centre_cell(a, b, lane + 32, L.strideH, L.strideV, L.offV, &d1) : c0[u];
      y0[u] = __ldcs(pred + s * kQC + lane);
      y1[u] = two ? __ldcs(pred + s * kQC + lane + 32) : y0[u];
    }
#pragma unroll
    for (int u = 0; u < kIoUnroll; u++) {
      o0[u] = __ldcg(lat + c0[u]);
      o1[u] = two ? __ldcg(lat + c1[u]) : o0[u];
    }
#pragma unroll
    for (int u = 0; u < kIoUnroll; u++) {
      if (s0 + u >= B) continue;
      const float d0 = fabsf(y0[u] - o0[u]), d1 = two ? fabsf(y1[u] - o1[u]) : 0.f;
      if (!(d0 <= 3.0e38f) || !(d1 <= 3.0e38f)) bad = true;   // NaN or Inf
      else m = fmaxf(m, fmaxf(d0, d1));
    }
#pragma unroll
    for (int u = 0; u < kIoUnroll; u++) {
      if (s0 + u >= B) continue;
      lat[c0[u]] = y0[u];
      if (cd[u] >= 0) lat[cd[u]] = y0[u];
      if (two) lat[c1[u]] = y1[u];
    }
  }
  m = warp_max(m);
  if (lane == 0) red[warp] = m;
  if (__any_sync(0xffffffffu, bad) && lane == 0) bad_s = 1;
  __syncthreads();
  if (warp == 0) {
    float v = lane < kIoWarps ? red[lane] : 0.f;
    v = warp_max(v);
    if (lane == 0) blockmax[blockIdx.x] = __float_as_uint(v) | (bad_s ? 0x80000000u : 0u);
  }
}

// ------------------------------------------------------ a8: convergence reduction
// One block reduces the n block maxima: out[0] = max (fp32 bits; non-negative
// floats order like unsigned ints), out[1] = 1 if any block saw a non-finite value.
__global__ void __launch_bounds__(1024) k_reduce_max(const unsigned int* __restrict__ blockmax, int n,
                                                     unsigned int* __restrict__ out) {
  __shared__ unsigned int red[32];
  __shared__ unsigned int anybad;
  if (threadIdx.x == 0) anybad = 0u;
  __syncthreads();
  unsigned int m = 0u, bad = 0u;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned int v = blockmax[i];
    bad |= v >> 31;
    m = max(m, v & 0x7fffffffu);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (__any_sync(0xffffffffu, bad != 0u) && (threadIdx.x & 31) == 0) atomicOr(&anybad, 1u);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned int v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) {
      out[0] = v;
      out[1] = anybad;
    }
  }
}

// Grid: a multiple of the SM count (8 warps per block, up to 8 blocks per SM).
static int io_blocks(int64_t units, int per_block) {
  int64_t b = (units + per_block - 1) / per_block;
  const int64_t cap = (int64_t)(num_sms() < kMaxSMs ? num_sms() : kMaxSMs) * 8;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

int scatter_grid(int64_t B) { return io_blocks(B, kIoWarps * kIoUnroll); }

void launch_gather_phase(const float* lat, const LatticeGeom& L, const uint32_t* anchors, int64_t B, float* gb,
                         cudaStream_t s) {
  if (B <= 0) return;
  k_gather_phase<<<io_blocks(B, kIoWarps * kIoUnroll), kIoWarps * 32, 0, s>>>(lat, L, anchors, B, gb);
}

void launch_scatter_phase(float* lat, const LatticeGeom& L, const uint32_t* anchors, int64_t B, const float* pred,
                          unsigned int* blockmax, unsigned int* out, cudaStream_t s) {
  const int nb = scatter_grid(B);
  if (L.cells >= ((int64_t)1 << 31)) __builtin_trap();   // 32-bit cell indices (never at 16385^2: 3.4e7 cells)
  if (B > 0) k_scatter_phase<<<nb, kIoWarps * 32, 0, s>>>(lat, L, anchors, B, pred, blockmax);
  else cudaMemsetAsync(blockmax, 0, sizeof(unsigned int) * nb, s);
  k_reduce_max<<<1, 1024, 0, s>>>(blockmax, nb, out);
}

}  // namespace mfp
