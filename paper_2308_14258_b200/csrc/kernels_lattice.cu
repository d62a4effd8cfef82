// kernels_lattice.cu — line-lattice kernels of libmfp: init (a0), exact
// discrete-Laplace subsolver phase (N9), convergence reduction (N6, a8), halo
// pack/unpack (N7, a7), final-phase line copy (a9).  HBM-bound or latency-bound
// work: coalesced line segments, grids sized in multiples of the SM count.
#include "device_common.cuh"
#include "tc_common.cuh"   // f2 packed fp32x2 helpers

namespace mfp {

using tcx::f2;
using tcx::f2_make;
using tcx::f2_split;
using tcx::ffma2;

// ---------------------------------------------------------------- a0: init
// g (2(nx+ny), reading G6) onto the boundary lines of the local lattice; the
// interior lines were zeroed by cudaMemsetAsync (initial guess 0).
__global__ void k_init_boundary(float* __restrict__ lat, LatticeGeom L, int nx, int ny,
                                const float* __restrict__ g) {
  const int n = 2 * (nx + ny);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    int x, y;
    if (k < nx) { x = k; y = 0; }
    else if (k < nx + ny) { x = nx; y = k - nx; }
    else if (k < 2 * nx + ny) { x = nx - (k - nx - ny); y = ny; }
    else { x = 0; y = ny - (k - 2 * nx - ny); }
    if (x < L.RX0 || x > L.RX1 || y < L.RY0 || y > L.RY1) continue;
    const float v = __ldg(g + k);
    if (y % kH == 0) lat[(int64_t)((y - L.RY0) / kH) * L.strideH + (x - L.RX0)] = v;
    if (x % kH == 0) lat[L.offV + (int64_t)((x - L.RX0) / kH) * L.strideV + (y - L.RY0)] = v;
  }
}

void launch_init_lattice(float* lat, const LatticeGeom& L, int nx, int ny, const float* g,
                         cudaStream_t s) {
  cudaMemsetAsync(lat, 0, sizeof(float) * L.cells, s);
  int n = 2 * (nx + ny);
  int blocks = (n + 255) / 256;
  if (blocks > num_sms() * 4) blocks = num_sms() * 4;
  k_init_boundary<<<blocks, 256, 0, s>>>(lat, L, nx, ny, g);
}

// ---------------------------------------------------- N9: exact subsolver phase
// y = H_c g for every subdomain of one class, written onto its centre lines
// (P:43).  Reads and writes of one class are disjoint, so gather and
// scatter fuse into one kernel without a grid barrier.  Register-blocked: a warp
// takes 8 subdomains at a time (their perimeters staged in smem by 16-byte
// gathers), lane l owns outputs p = l and l + 32, and every H_c^T element it
// loads from smem feeds 8 FMAs (one per subdomain) — 0.25 shared loads per FMA
// instead of 1, packed: one FFMA2 updates a lane's two outputs.  Persistent blocks
// (one per SM, 16 warps) load H_c^T (32 KB) once.  Each output keeps the plain k-ascending
// FMA chain (FFMA2 rounds per lane like FFMA), so results are unchanged.
constexpr int kExactWarps = 16;
#ifndef MFP_EXACT_UNROLL
#define MFP_EXACT_UNROLL 8
#endif
constexpr int kExactUnroll = MFP_EXACT_UNROLL;   // k-loop unroll of exact_group (A/B builds)
constexpr int kExactSub = 8;   // subdomains per warp per round

// One warp's group of kExactSub consecutive subdomains [s0, s0 + 8) of a
// phase: gather (16-byte loads; CG = L2-coherent loads for the persistent
// kernel, whose lattice is written by other SMs within the launch), y = H_c g
// with every H_c^T element feeding 8 FFMA2s, scatter onto the centre lines.
template <bool CG, int SUB = kExactSub>
__device__ __forceinline__ void exact_group(float* __restrict__ lat, const LatticeGeom& L,
                                            const uint32_t* __restrict__ anchors, int64_t s0, int64_t B,
                                            const float2* sH, float* g, int lane) {
  uint32_t pk[SUB];
  float4 gv[SUB];
#pragma unroll
  for (int j = 0; j < SUB; j++) pk[j] = __ldg(anchors + (s0 + j < B ? s0 + j : B - 1));
#pragma unroll
  for (int j = 0; j < SUB; j++) {   // 8 gathers in flight
    if constexpr (CG) {
      int a, b;
      unpack_anchor(pk[j], a, b);
      const int lx = kH * a, ly = kH * b, edge = lane >> 3, t0 = 4 * (lane & 7);
      if (edge == 0) gv[j] = __ldcg(reinterpret_cast<const float4*>(lat + (int64_t)b * L.strideH + lx + t0));
      else if (edge == 1) gv[j] = __ldcg(reinterpret_cast<const float4*>(lat + L.offV + (int64_t)(a + 2) * L.strideV + ly + t0));
      else {
        const float* r = edge == 2 ? lat + (int64_t)(b + 2) * L.strideH + lx + kM - t0
                                   : lat + L.offV + (int64_t)a * L.strideV + ly + kM - t0;
        gv[j] = make_float4(__ldcg(r), __ldcg(r - 1), __ldcg(r - 2), __ldcg(r - 3));
      }
    } else {
      gv[j] = gather4(lat, L, pk[j], lane);
    }
  }
#pragma unroll
  for (int j = 0; j < SUB; j++) reinterpret_cast<float4*>(g + j * kNB)[lane] = gv[j];
  __syncwarp();
  f2 y[SUB];
#pragma unroll
  for (int j = 0; j < SUB; j++) y[j] = f2_make(0.f, 0.f);
#pragma unroll (kExactUnroll)
  for (int k = 0; k < kNB; k += 4) {
    f2 h[4];
#pragma unroll
    for (int t = 0; t < 4; t++) {
      const float2 hv = sH[(k + t) * 32 + lane];
      h[t] = f2_make(hv.x, hv.y);
    }
#pragma unroll
    for (int j = 0; j < SUB; j++) {
      const float4 gk = *reinterpret_cast<const float4*>(g + j * kNB + k);
      y[j] = ffma2(h[0], f2_make(gk.x, gk.x), y[j]);
      y[j] = ffma2(h[1], f2_make(gk.y, gk.y), y[j]);
      y[j] = ffma2(h[2], f2_make(gk.z, gk.z), y[j]);
      y[j] = ffma2(h[3], f2_make(gk.w, gk.w), y[j]);
    }
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < SUB; j++) {
    if (s0 + j >= B) continue;
    float y0, y1;
    f2_split(y[j], y0, y1);
    int a, b;
    unpack_anchor(pk[j], a, b);
    int64_t dup;
    const int64_t c0 = centre_cell(a, b, lane, L.strideH, L.strideV, L.offV, &dup);
    lat[c0] = y0;
    if (dup >= 0) lat[dup] = y0;
    if (lane + 32 < kQC) lat[centre_cell(a, b, lane + 32, L.strideH, L.strideV, L.offV, &dup)] = y1;
  }
}

__device__ __forceinline__ void load_hct(float2* sH, const float* __restrict__ HcT) {
  for (int i = threadIdx.x; i < kNB * 32; i += blockDim.x) {
    const int k = i >> 5, l = i & 31;
    sH[i] = make_float2(__ldg(HcT + k * 64 + l), __ldg(HcT + k * 64 + 32 + l));
  }
}

template <int SUB>
__global__ void __launch_bounds__(kExactWarps * 32)
k_exact_phase(float* __restrict__ lat, LatticeGeom L, const uint32_t* __restrict__ anchors,
              int64_t B, const float* __restrict__ HcT) {
  extern __shared__ __align__(16) float ex_smem[];
  // H_c^T interleaved per lane: sH[k][lane] = (H^T[k][lane], H^T[k][lane + 32]), so one
  // 8-byte load gives a lane both of its outputs' coefficients and one packed FFMA2
  // updates both outputs (p = lane, lane + 32) of a subdomain
  float2* sH = reinterpret_cast<float2*>(ex_smem);
  float* sg = ex_smem + kNB * 64;                        // [warp][sub][k]
  load_hct(sH, HcT);   // a constant of the context: loaded before the PDL wait, under the predecessor's tail
  __syncthreads();
  tcx::pdl_launch_dependents();
  tcx::pdl_wait();     // the lattice (previous phases) complete from here on
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* g = sg + warp * SUB * kNB;
  const int64_t step = (int64_t)gridDim.x * kExactWarps * SUB;
  for (int64_t s0 = ((int64_t)blockIdx.x * kExactWarps + warp) * SUB; s0 < B; s0 += step)
    exact_group<false, SUB>(lat, L, anchors, s0, B, sH, g, lane);
}

// ---- NEXT-2: the fully persistent exact-subsolver iteration (SURVEY §8(f)
// "a fully persistent 4-phase kernel; dataflow flags replace grid barriers").
// ONE launch runs K whole iterations: work item = (iteration, phase, group of 8
// subdomains); warp w takes groups w, w + W, ... of every phase in stage order
// (stage = 4 * iteration + phase).  A group may run stage (k, p) once every group of the
// other phases that writes one of its perimeter cells (RAW) or reads one of the
// cells it writes (WAR) has finished its latest stage before (k, p), and the
// group itself has finished (k - 1, p): per-group completion stamps done[g] =
// absolute stage + 1 (release after the group's stores; the waiting lanes poll
// with acquire loads, one dependency per lane), so the four phase barriers of
// an iteration become local waits and the phases of neighbouring iterations
// overlap wherever the dependencies allow.  Same FMA order per output as
// k_exact_phase: the field is bit-identical.  Deadlock freedom: every warp takes
// its items in increasing stage order and every dependency points to an
// earlier stage; the grid is at most one block per SM (co-resident) and the
// launch is plainly stream-ordered.  A bounded spin (2^28 polls) traps instead
// of hanging on a broken plan.
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(kExactWarps * 32)
k_exact_iter(ExactIterArgs A) {
  extern __shared__ __align__(16) float ex_smem[];
  float2* sH = reinterpret_cast<float2*>(ex_smem);
  float* sg = ex_smem + kNB * 64;
  load_hct(sH, A.HcT);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* g = sg + warp * kExactSub * kNB;
  // absolute iteration of this launch (device counter: graph replays advance it)
  const int64_t iter0 = (int64_t)*(volatile const unsigned long long*)A.iter_ctr;
  const int64_t W = (int64_t)gridDim.x * kExactWarps;
  const int64_t wid = (int64_t)blockIdx.x * kExactWarps + warp;
  // warp w takes groups w, w + W, ... of EVERY phase, in stage order: the i-th
  // group of each phase covers about the same rows of the domain (anchors are
  // row-major in every phase), so a group's dependencies are mostly its own
  // warp's previous group or a neighbouring warp's, progressing in lock step
  for (int64_t kk = 0; kk < A.K; kk++) {
    const int64_t k = iter0 + kk;
    for (int p = 0; p < 4; p++) {
      for (int64_t gl = wid; gl < A.g0[p + 1] - A.g0[p]; gl += W) {
        const int64_t gid = A.g0[p] + gl;
        const unsigned long long stage = (unsigned long long)(4 * k + p);
        // ---- wait for the dependencies' latest stage before (k, p)
        const int d0 = __ldg(A.dep_off + gid), d1 = __ldg(A.dep_off + gid + 1);
        for (int d = d0 + lane; d < d1; d += 32) {
          const int h = __ldg(A.dep_ids + d);
          int q = 0;
          while (h >= A.g0[q + 1]) q++;
          // latest run of h before (k, p): (k, q) if q < p, else (k - 1, q); stamps are stage + 1
          const long long need = (q < p ? 4 * k + q : 4 * (k - 1) + q) + 1;
          if (need > 0) {
            unsigned int spins = 0;
            while ((long long)ld_acquire_gpu(A.done + h) < need) {
              __nanosleep(32);
              if (++spins > (1u << 28)) __trap();
            }
          }
        }
        __syncwarp();
        exact_group<true>(A.lat, A.L, A.anchors[p], gl * kExactSub, A.B[p], sH, g, lane);
        __syncwarp();
        __threadfence();   // this warp's scatter before the stamp
        if (lane == 0)
          asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(A.done + gid), "l"(stage + 1) : "memory");
      }
    }
  }
  // the last block to finish advances the iteration counter for the next launch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(A.ticket, 1u) == gridDim.x - 1) {
      *A.ticket = 0u;
      *A.iter_ctr = (unsigned long long)(iter0 + A.K);
    }
  }
}

void launch_exact_iter(const ExactIterArgs& a, cudaStream_t s) {
  if (a.K <= 0 || a.g0[4] <= 0) return;
  int64_t blocks = (a.g0[4] + kExactWarps - 1) / kExactWarps;
  if (blocks > num_sms()) blocks = num_sms();   // one co-resident block per SM
  const size_t smem = sizeof(float) * ((size_t)kNB * 64 + (size_t)kExactWarps * kExactSub * kNB);
  k_exact_iter<<<(int)blocks, kExactWarps * 32, smem, s>>>(a);
}

// Subdomains per warp: 8 (every H_c^T smem load feeds 8 FFMA2) while the phase
// still gives (about) a block of 16 warps per SM; smaller phases — a rank's
// share at 4-8 GPUs — use 4 / 2 / 1 per warp so the grid still spreads over the
// SMs (at 8 subdomains per warp a 2,048-subdomain phase ran on 16 SMs).
// MFP_EXACT_SUB=1|2|4|8 forces one (A/B).
static int exact_sub(int64_t B) {
  static int forced = -1;
  if (forced < 0) {
    const char* e = getenv("MFP_EXACT_SUB");
    const int v = e ? atoi(e) : 0;
    forced = (v == 1 || v == 2 || v == 4 || v == 7 || v == 8) ? v : 0;
  }
  if (forced) return forced;
  const int64_t sms = num_sms();
  int sub = 8;
  while (sub > 1 && (B + kExactWarps * sub - 1) / (kExactWarps * sub) < (3 * sms) / 4) sub >>= 1;
  // a full-size phase that leaves SMs idle at 8 per warp (C5: 127 blocks on 148 SMs)
  // but fits one wave at 7 (146 blocks) takes 7: 1/8 less serial work per warp
  if (sub == 8 && (B + kExactWarps * 8 - 1) / (kExactWarps * 8) < sms &&
      (B + kExactWarps * 7 - 1) / (kExactWarps * 7) <= sms)
    sub = 7;
  return sub;
}

static size_t exact_smem(int sub) { return sizeof(float) * ((size_t)kNB * 64 + (size_t)kExactWarps * sub * kNB); }

void launch_exact_phase(float* lat, const LatticeGeom& L, const uint32_t* anchors, int64_t B,
                        const float* HcT, cudaStream_t s) {
  if (B <= 0) return;
  const int sub = exact_sub(B);
  const int per_block = kExactWarps * sub;
  int64_t blocks = (B + per_block - 1) / per_block;
  const int per_sm = sub >= 7 ? 1 : 2;   // 88-96 KB of smem at 7-8 per warp, <= 64 KB below
  if (blocks > per_sm * num_sms()) blocks = per_sm * num_sms();
  // PDL (the next phase's H_c^T load under this one's tail) only for full-size phases
  // (one block per SM): with the small per-rank batches' 2 blocks per SM the early
  // dependents co-reside and slow the phase down (23 -> 42 us per iteration at the
  // 8-GPU share, tools/gpu/round2/r4k.sh)
#define MFP_EX(S)                                                                                     \
  do {                                                                                                \
    if (per_sm == 1) launch_pdl(k_exact_phase<S>, (int)blocks, kExactWarps * 32, exact_smem(S), s, lat, L, anchors, B, HcT); \
    else k_exact_phase<S><<<(int)blocks, kExactWarps * 32, exact_smem(S), s>>>(lat, L, anchors, B, HcT);     \
  } while (0)
  switch (sub) {
    case 1: MFP_EX(1); break;
    case 2: MFP_EX(2); break;
    case 4: MFP_EX(4); break;
    case 7: MFP_EX(7); break;
    default: MFP_EX(8); break;
  }
#undef MFP_EX
}

void exact_kernel_attributes() {
  cudaFuncSetAttribute(k_exact_phase<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)exact_smem(8));
  cudaFuncSetAttribute(k_exact_phase<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)exact_smem(7));
  cudaFuncSetAttribute(k_exact_phase<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)exact_smem(4));
  cudaFuncSetAttribute(k_exact_phase<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)exact_smem(2));
  cudaFuncSetAttribute(k_exact_phase<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)exact_smem(1));
  cudaFuncSetAttribute(k_exact_iter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(sizeof(float) * ((size_t)kNB * 64 + (size_t)kExactWarps * kExactSub * kNB)));
}

// Exact subsolver, general query set (final phase / batch API): a block takes
// up to 8 subdomains so every H^T element read from L2 is reused 8 times.
constexpr int kExactGroup = 8;

__global__ void __launch_bounds__(256)
k_exact_general(const float* __restrict__ lat, LatticeGeom L, const uint32_t* __restrict__ lat_anchors,
                const float* __restrict__ gb, int64_t B, int q, const float* __restrict__ HT,
                Sink sink) {
  __shared__ float sg[kExactGroup][kNB];
  for (int64_t s0 = (int64_t)blockIdx.x * kExactGroup; s0 < B; s0 += (int64_t)gridDim.x * kExactGroup) {
    const int ns = (int)min((int64_t)kExactGroup, B - s0);
    for (int i = threadIdx.x; i < kExactGroup * kNB; i += blockDim.x) {
      int j = i / kNB, k = i % kNB;
      float v = 0.f;
      if (j < ns) {
        if (gb) v = __ldg(gb + (s0 + j) * kNB + k);
        else {
          int a, b;
          unpack_anchor(__ldg(lat_anchors + s0 + j), a, b);
          v = lat[perim_cell(a, b, k, L.strideH, L.strideV, L.offV)];
        }
      }
      sg[j][k] = v;
    }
    __syncthreads();
    const int ld = (q == kQC) ? 64 : q;  // H_c^T is stored [128][64]
    for (int p = threadIdx.x; p < q; p += blockDim.x) {
      float acc[kExactGroup];
#pragma unroll
      for (int j = 0; j < kExactGroup; j++) acc[j] = 0.f;
      for (int k = 0; k < kNB; k++) {
        const float h = __ldg(HT + (int64_t)k * ld + p);
#pragma unroll
        for (int j = 0; j < kExactGroup; j++) acc[j] = fmaf(h, sg[j][k], acc[j]);
      }
      for (int j = 0; j < ns; j++) sink_store(sink, s0 + j, p, acc[j]);
    }
    __syncthreads();
  }
}

void launch_exact_general(const float* lat, const LatticeGeom& L, const uint32_t* lat_anchors,
                          const float* gb, int64_t B, int q, const float* HT, const Sink& sink,
                          cudaStream_t s) {
  if (B <= 0) return;
  int64_t blocks = (B + kExactGroup - 1) / kExactGroup;
  if (blocks > num_sms() * 8) blocks = num_sms() * 8;
  k_exact_general<<<(int)blocks, 256, 0, s>>>(lat, L, lat_anchors, gb, B, q, HT, sink);
}

// ------------------------------------------------------ N6: convergence delta
// delta = max |U_k - U_{k-1}| over the owned interior line cells (reading G5),
// one block per contiguous line segment, warp-shuffle max, one atomicMax on the
// fp32 bit pattern (non-negative floats order like unsigned ints).
__global__ void __launch_bounds__(256)
k_delta(const float* __restrict__ lat, const float* __restrict__ snap,
        const int64_t* __restrict__ segs, int nseg, unsigned int* out) {
  __shared__ float red[8];
  float m = 0.f;
  bool bad = false;
  for (int sgi = blockIdx.x; sgi < nseg; sgi += gridDim.x) {
    const int64_t sd = __ldg(segs + sgi);
    const int64_t off = sd >> 20;
    const int len = (int)(sd & 0xfffff);
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
      const float d = fabsf(lat[off + i] - snap[off + i]);
      if (!(d <= 3.0e38f)) bad = true;   // NaN or Inf
      else m = fmaxf(m, d);
    }
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(out + 1, 1u);
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_max(v);
    if (threadIdx.x == 0) atomicMax(out, __float_as_uint(v));
  }
}

void launch_delta(const float* lat, const float* snap, const int64_t* segs, int nseg,
                  unsigned int* out, cudaStream_t s) {
  // out is zeroed by the caller once per check (max accumulates over local ranks)
  if (nseg <= 0) return;
  int blocks = nseg < num_sms() * 4 ? nseg : num_sms() * 4;
  k_delta<<<blocks, 256, 0, s>>>(lat, snap, segs, nseg, out);
}

// ------------------------------------------------ a8: on-device stopping rule
// The body of the solve's WHILE graph (api.cu run_loop) ends with this kernel:
// after a block of c iterations and its delta, decide on the device whether
// another block runs (iterate until delta <= eps or t iterations),
// so a converging solve needs no host round trip per block.
// st = {iterations done, t, tol bits, blocks run}; delta = {max bits, non-finite}.
__global__ void k_loop_ctl(cudaGraphConditionalHandle h, const unsigned int* __restrict__ delta,
                           unsigned int* __restrict__ st, int ce) {
  const unsigned int it = st[0] + (unsigned int)ce;
  st[0] = it;
  st[3] += 1u;
  const float d = __uint_as_float(delta[0]);
  const float tol = __uint_as_float(st[2]);
  const bool stop = delta[1] != 0u || d <= tol || it + (unsigned int)ce > st[1];
  cudaGraphSetConditional(h, stop ? 0u : 1u);
}

void launch_loop_ctl(cudaGraphConditionalHandle h, const unsigned int* delta, unsigned int* st, int ce,
                     cudaStream_t s) {
  k_loop_ctl<<<1, 1, 0, s>>>(h, delta, st, ce);
}

// --------------------------------------------------------- N7: halo pack/unpack
__global__ void k_pack(const float* __restrict__ lat, const int32_t* __restrict__ idx, int64_t n,
                       float* __restrict__ buf) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = lat[__ldg(idx + i)];
}
__global__ void k_unpack(float* __restrict__ lat, const int32_t* __restrict__ idx, int64_t n,
                         const float* __restrict__ buf) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    lat[__ldg(idx + i)] = buf[i];
}

static int grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > num_sms() * 4) b = num_sms() * 4;
  return b < 1 ? 1 : (int)b;
}

void launch_pack(const float* lat, const int32_t* idx, int64_t n, float* buf, cudaStream_t s) {
  if (n > 0) k_pack<<<grid_for(n), 256, 0, s>>>(lat, idx, n, buf);
}
void launch_unpack(float* lat, const int32_t* idx, int64_t n, const float* buf, cudaStream_t s) {
  if (n > 0) k_unpack<<<grid_for(n), 256, 0, s>>>(lat, idx, n, buf);
}

// ---------------------------------------------------------- a9: final lines
// Atomic-subdomain boundary lines (x or y a multiple of m) of the owned block
// take the lattice values (DESIGN.md §2 reading F1); interior points are
// written by the final-phase predictions.
// Only the line points are visited (≈ 1/16 of the block): the rows y ≡ 0 (mod m)
// x-fastest from the horizontal lines, then the columns x ≡ 0 (mod m)
// y-fastest from the vertical lines (crossings written twice, same value).  The
// block origin (X0, Y0) is a multiple of m.
__global__ void k_final_lines(const float* __restrict__ lat, LatticeGeom L, int X0, int Y0, int bw,
                              int bh, float* __restrict__ field, int ld) {
  const int nr = (bh + kM - 1) / kM, nc = (bw + kM - 1) / kM;
  const int64_t na = (int64_t)nr * bw, n = na + (int64_t)nc * bh;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    int i, j;
    float v;
    if (t < na) {
      j = kM * (int)(t / bw);
      i = (int)(t % bw);
      v = lat[(int64_t)((Y0 + j - L.RY0) / kH) * L.strideH + (X0 + i - L.RX0)];
    } else {
      const int64_t u = t - na;
      i = kM * (int)(u / bh);
      j = (int)(u % bh);
      v = lat[L.offV + (int64_t)((X0 + i - L.RX0) / kH) * L.strideV + (Y0 + j - L.RY0)];
    }
    field[(int64_t)j * ld + i] = v;
  }
}

void launch_final_lines(const float* lat, const LatticeGeom& L, int X0, int Y0, int bw, int bh,
                        float* field, int ld, cudaStream_t s) {
  k_final_lines<<<num_sms() * 4, 256, 0, s>>>(lat, L, X0, Y0, bw, bh, field, ld);
}

}  // namespace mfp
