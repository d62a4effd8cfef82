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
// bit 31 set on a non-finite prediction.  Cells of one phase are written by
// exactly one subdomain, so the result is order independent.
//
// a8 reduction fused: the last block to finish (an atomic ticket, re-armed by
// that block) reduces the block maxima into out[0] (max, fp32 bits: non-negative
// floats order like unsigned ints) and out[1] (1 if any prediction was
// non-finite) — no second kernel and no launch gap.
//
// Measured on B200 (bench.py boundary_io, 262,144 subdomains, L2 flushed;
// tools/gpu/round2/r3m.sh, r3n.sh): the grid is ONE wave of resident blocks
// (the round-1 grid of 8 blocks per SM ran 1.6 waves at 5 resident), and the
// most warps per SM win over more subdomains per warp: kScU = 2 subdomains per
// warp per round at 8 blocks (64 warps) per SM 0.67 of HBM, 4 at 5 blocks 0.59,
// 8 at 2 blocks 0.56, an anchor prefetch across rounds no better (0.54-0.66),
// one thread per cell 0.42; + the fused reduction 0.71 (round 1: 0.53).  Cache
// hints (session 3, tools/gpu/round2/r4r.sh): any store hint on the lattice
// (st.cs / st.cg / st.wt) halves it (0.35); ld.cs for the old values 0.67, ld.cv
// 0.71 — plain stores and ld.cg stay.
constexpr int kScU = 2;      // subdomains per warp per round
constexpr int kScMinB = 8;   // resident blocks per SM (<= 32 registers)

__global__ void __launch_bounds__(kIoWarps * 32, kScMinB)
k_scatter_phase(float* __restrict__ lat, LatticeGeom L, const uint32_t* __restrict__ anchors, int64_t B,
                const float* __restrict__ pred, unsigned int* __restrict__ blockmax, unsigned int* __restrict__ ticket,
                unsigned int* __restrict__ out) {
  __shared__ float red[kIoWarps];
  __shared__ int bad_s;
  __shared__ unsigned int last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) bad_s = 0;
  __syncthreads();
  const int64_t nw = (int64_t)gridDim.x * kIoWarps;
  float m = 0.f;
  bool bad = false;
  const bool two = lane + 32 < kQC;
  // every load of a round (predictions and old values) is issued before its
  // first store; cell indices are 32-bit (a rank's lattice holds < 2^31 cells;
  // checked at launch)
  for (int64_t s0 = ((int64_t)blockIdx.x * kIoWarps + warp) * kScU; s0 < B; s0 += nw * kScU) {
    int32_t c0[kScU], c1[kScU], cd[kScU];   // cd: the centre's second copy or -1
    float y0[kScU], y1[kScU], o0[kScU], o1[kScU];
#pragma unroll
    for (int u = 0; u < kScU; u++) {
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
    for (int u = 0; u < kScU; u++) {
      o0[u] = __ldcg(lat + c0[u]);
      o1[u] = two ? __ldcg(lat + c1[u]) : o0[u];
    }
#pragma unroll
    for (int u = 0; u < kScU; u++) {
      if (s0 + u >= B) continue;
      const float d0 = fabsf(y0[u] - o0[u]), d1 = two ? fabsf(y1[u] - o1[u]) : 0.f;
      if (!(d0 <= 3.0e38f) || !(d1 <= 3.0e38f)) bad = true;   // NaN or Inf
      else m = fmaxf(m, fmaxf(d0, d1));
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
    if (lane == 0) {
      blockmax[blockIdx.x] = __float_as_uint(v) | (bad_s ? 0x80000000u : 0u);
      __threadfence();
      last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!last) return;
  // the last block: every other block's maximum is visible (fence before ticket)
  __threadfence();
  unsigned int mu = 0u, nb = 0u;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
    const unsigned int v = __ldcg(blockmax + i);
    nb |= v >> 31;
    mu = max(mu, v & 0x7fffffffu);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mu = max(mu, __shfl_xor_sync(0xffffffffu, mu, o));
    nb |= __shfl_xor_sync(0xffffffffu, nb, o);
  }
  __shared__ unsigned int rm[kIoWarps], rb[kIoWarps];
  if (lane == 0) {
    rm[warp] = mu;
    rb[warp] = nb;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kIoWarps; w++) {
      mu = max(mu, rm[w]);
      nb |= rb[w];
    }
    out[0] = mu;
    out[1] = nb;
    *ticket = 0u;   // re-armed for the next launch (stream order)
  }
}

// Grids: a multiple of the SM count.  The gather: 8 warps per block, up to 8
// blocks per SM.  The scatter: exactly one wave of resident blocks.
static int io_blocks(int64_t units, int per_block) {
  int64_t b = (units + per_block - 1) / per_block;
  const int64_t cap = (int64_t)(num_sms() < kMaxSMs ? num_sms() : kMaxSMs) * 8;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

int scatter_grid(int64_t B) {
  static int occ = 0;
  if (occ == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_scatter_phase, kIoWarps * 32, 0);
    occ = occ < 1 ? 1 : occ > 8 ? 8 : occ;
  }
  int64_t b = (B + kIoWarps * kScU - 1) / (kIoWarps * kScU);
  const int64_t cap = (int64_t)(num_sms() < kMaxSMs ? num_sms() : kMaxSMs) * occ;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

void launch_gather_phase(const float* lat, const LatticeGeom& L, const uint32_t* anchors, int64_t B, float* gb,
                         cudaStream_t s) {
  if (B <= 0) return;
  k_gather_phase<<<io_blocks(B, kIoWarps * kIoUnroll), kIoWarps * 32, 0, s>>>(lat, L, anchors, B, gb);
}

void launch_scatter_phase(float* lat, const LatticeGeom& L, const uint32_t* anchors, int64_t B, const float* pred,
                          unsigned int* blockmax, unsigned int* out, cudaStream_t s) {
  if (L.cells >= ((int64_t)1 << 31)) __builtin_trap();   // 32-bit cell indices (never at 16385^2: 3.4e7 cells)
  if (B <= 0) {
    cudaMemsetAsync(out, 0, 2 * sizeof(unsigned int), s);
    return;
  }
  k_scatter_phase<<<scatter_grid(B), kIoWarps * 32, 0, s>>>(lat, L, anchors, B, pred, blockmax,
                                                             blockmax + kMaxSMs * 8, out);
}

}  // namespace mfp
