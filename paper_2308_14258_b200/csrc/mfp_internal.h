// mfp_internal.h — internal types of libmfp (plan, rank state, kernel entry points).
// Not part of the ABI; include/mfp.h is.  See DESIGN.md §5 for the HBM layout.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/mfp.h"

namespace mfp {

constexpr int kM = 32;             // subdomain intervals per side (reading G1)
constexpr int kH = kM / 2;         // lattice spacing m/2
constexpr int kNB = 4 * kM;        // perimeter length 4m = 128 (G1)
constexpr int kQC = 2 * kM - 3;    // centre-line queries 61 (G3)
constexpr int kQF = (kM - 1) * (kM - 1);  // interior queries 961
constexpr int kD = 128;            // SDNet width, canonical (G7)
constexpr int kD2 = 256;           // the wide variant (d = 128 | 256)
constexpr int kC1 = 8;             // conv channels 1 -> 8 -> 1, k = 5 (G7)
constexpr int kK = 5;
constexpr int kMaxHidden = 3;
// 16-bit tensor-core image of one hidden layer: the 128 x 128 weight block
// (SWIZZLE_128B K-major, 32 KB) followed by a 128 x 16 bias block (SWIZZLE_NONE
// K-major, 4 KB) whose columns 0/1 hold the bias split b = b_hi + b_lo.
constexpr int kWImgW = kD * kD;             // elements
constexpr int kWImgB = kD * 16;
constexpr int kWImg = kWImgW + kWImgB;      // 18432 elements = 36 KB
// d = 256: per hidden layer and CTA of the pair, this CTA's 128 output rows
// (B operand rows 128 r .. 128 r + 127 of the N = 256 pair MMA) as four K-chunks
// of 64 (128 rows x 128 B SWIZZLE_128B, 16 KB each, streamed by TMA) followed by
// its 128 x 16 bias block (4 KB, resident).
constexpr int kW2Chunk = 128 * 64;            // elements (16 KB)
constexpr int kW2Cta = 4 * kW2Chunk + 128 * 16;   // 34816 elements = 68 KB
constexpr int kW2Layer = 2 * kW2Cta;
// 16-bit hidden-weight image elements for width d
inline size_t wimg_elems(int d, int n_hidden) {
  return (size_t)n_hidden * (d == kD2 ? (size_t)kW2Layer : (size_t)kWImg);
}

// Local lattice of one rank: horizontal lines y = RY0 + 16 i
// (x-contiguous, RX0..RX1) then vertical lines x = RX0 + 16 j (y-contiguous,
// RY0..RY1); row strides padded to 32 floats (128 B).  Crossing points exist in
// both arrays and are always written to both.
struct LatticeGeom {
  int RX0, RX1, RY0, RY1;
  int nH, nV, lenH, lenV, strideH, strideV;
  int64_t offV, cells;  // cells incl. padding
};

struct PeerPlan {
  int rank;
  std::vector<int32_t> send_idx, recv_idx;        // flat local lattice cells
  std::vector<int32_t> send_kind, send_x, send_y;  // canonical global keys (plan API)
  std::vector<int32_t> recv_kind, recv_x, recv_y;
};

struct RankPlan {
  int rank, ry, rx;
  int X0, X1, Y0, Y1;           // owned block (half-open; last col/row closed at nx/ny)
  int bw, bh;                   // owned block extent in points
  LatticeGeom lat;
  std::vector<uint32_t> phase_anchor[4];  // packed (a | b << 16), local line indices
  // phase_anchor[0] is ordered interior-first: its first n0_interior subdomains
  // neither read nor write a halo (received) cell, so they may run while the
  // previous iteration's exchange is still in flight on the side stream.
  int64_t n0_interior = 0;
  std::vector<int32_t> phase_ax[4], phase_ay[4];   // global (plan API)
  std::vector<uint32_t> final_anchor;     // packed block-local (bx | by << 16) + lattice (a|b<<16)
  std::vector<uint32_t> final_lat_anchor;
  std::vector<int32_t> final_ax, final_ay;
  std::vector<PeerPlan> peers;  // row-major neighbour order
  std::vector<int64_t> delta_seg;  // (offset << 20) | len — owned interior line cells
};

struct GlobalPlan {
  mfp_config cfg;
  int R;
  std::vector<RankPlan> ranks;
};

// SM count of the current device (cudaDevAttrMultiProcessorCount, cached per
// device): every grid is sized from it, never from a literal.  kMaxSMs bounds
// the per-SM scratch carved from the workspace before a device is known.
int num_sms();
constexpr int kMaxSMs = 256;

// Validates cfg and builds the plan for one rank (or every rank when rank < 0).
mfp_status build_plan(const mfp_config* cfg, int rank, GlobalPlan* out, std::string* err);
mfp_status validate_config(const mfp_config* cfg, std::string* err);

// ---- device-side parameter blocks ----------------------------------------
struct DevNet {
  // fp32 tables (SIMT path + embed)
  // conv stack weights by value, channel-PAIR order (api.cu, kernels_embed_tc.cu
  // conv_stack): kernel parameters live in the constant bank, so the tensor-core
  // embed's FFMA2s take each weight pair as one 64-bit constant operand (no
  // shared-memory loads, no registers); 8-byte aligned as the first member
  alignas(8) float convw[89];
  // W2[:,0] then W2[:,1] by value, stride d (the tensor-core chains' split layers
  // take each column pair as one 64-bit constant-bank operand of FFMA2)
  alignas(8) float w2c[2 * 256];
  const float* conv1_w;  // [8][5]
  const float* conv1_b;  // [8]
  const float* conv2_w;  // [8][5]
  const float* conv2_b;  // [1]
  const float* W1T;      // [128 k][128 d]   (W1 transposed)
  const float* b1;       // [d]
  const float* W2;       // [d][2] (query half of the split layer, Eq. 5)
  const float* QTc;      // [d][64]  centre queries Q = X W2^T (b1 folded into z)
  const float* QTf;      // [d][961] interior queries
  const float* WhT;      // [n_hidden][k][n] fp32 (transposed for SIMT)
  const float* bh;       // [n_hidden][d]
  const float* wo;       // [d]
  const float* bo;       // [1]
  int d;                 // SDNet width: kD (128) or kD2 (256)
  int n_hidden;
  int gelu_tanh;
  int f16;               // tensor-core operands fp16 (1) or bf16 (0)
  int split;             // MFP_FP16X: activations split h_hi + h_lo (two MMAs per K step)
  // bf16 tables (tcgen05 path): weights pre-swizzled into the SW128 K-major image
  const uint16_t* Wh_sw2; // d = 128: [n_hidden][2][18 KB half] (CTA-pair chain: rows 64h..64h+63)
                          // d = 256: [n_hidden][2 CTAs][4 chunks x 16 KB + 4 KB bias] (kW2Cta)
  const uint16_t* W1img;  // [d/128][2][128*128] bf16 SW128 images of W1 = W1_hi + W1_lo (tensor-core embed)
  // exact subsolver
  const float* HcT;      // [128 k][64]  (61 used)
  const float* HfT;      // [128 k][961]
};

// Where chain outputs go.
struct Sink {
  int mode;  // 0: lattice centre lines, 1: field block (final phase), 2: dense out
  int q;
  float* lat;
  int64_t offV;
  int strideH, strideV;
  const uint32_t* anchors;    // mode 0: lattice (a|b<<16); mode 1: block-local (bx|by<<16)
  float* field;
  int ld;
  float* out;
  // mode 0, NEXT-2 put transport (nullptr otherwise): owned cells in a peer's
  // halo are also stored straight into that peer's put buffer of parity
  // (*put_epoch + 1) & 1.  putmap[cell] = -1 or (first << 2 | count) into
  // putdst; putdst = peer index << 24 | slot; putbufs[2 * peer + parity].
  const int32_t* putmap;
  const int32_t* putdst;
  float* const* putbufs;
  const unsigned long long* put_epoch;
};

// Launch with programmatic stream serialization (PDL, see tc_common.cuh) so the
// kernel's prologue overlaps its predecessor's tail; MFP_NO_PDL=1 launches
// plainly (A/B).  The kernel must call griddepcontrol.wait before touching
// anything its predecessors write.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// ---- kernel launchers (kernels_*.cu) --------------------------------------
void launch_init_lattice(float* lat, const LatticeGeom& L, int nx, int ny, const float* g,
                         cudaStream_t s);
// gather + embed: z[s][d] from lattice anchors (gb == nullptr) or from gb rows.
void launch_gather_embed(const float* lat, const LatticeGeom& L, const uint32_t* anchors,
                         const float* gb, int64_t B, const DevNet& net, float* z,
                         cudaStream_t s);
// exact subsolver phase (gather + H_c + scatter) for lattice anchors
void exact_kernel_attributes();
void launch_exact_phase(float* lat, const LatticeGeom& L, const uint32_t* anchors, int64_t B,
                        const float* HcT, cudaStream_t s);
// exact subsolver for the final phase / batches: gb rows or lattice anchors -> sink
void launch_exact_general(const float* lat, const LatticeGeom& L, const uint32_t* lat_anchors,
                          const float* gb, int64_t B, int q, const float* HT, const Sink& sink,
                          cudaStream_t s);
// NEXT-2: the persistent exact-subsolver iteration (kernels_lattice.cu
// k_exact_iter): K iterations per launch, per-group dataflow stamps instead of
// phase barriers (single-rank contexts).
struct ExactIterArgs {
  float* lat;
  LatticeGeom L;
  const uint32_t* anchors[4];
  int64_t B[4];
  int64_t g0[5];                 // first group id of each phase (groups phase-major), g0[4] = groups
  const int32_t* dep_off;        // [groups + 1]
  const int32_t* dep_ids;        // dependency group ids (the group itself included)
  unsigned long long* done;      // [groups] absolute stage + 1 of the last completed run
  unsigned long long* iter_ctr;  // absolute iteration of the next launch (advanced on device)
  unsigned int* ticket;          // last-block ticket
  const float* HcT;
  int K;                         // iterations per launch
};
void launch_exact_iter(const ExactIterArgs& a, cudaStream_t s);
void launch_chain_fp32(const float* z, int64_t B, int q, const DevNet& net, const Sink& sink,
                       cudaStream_t s);
bool chain_tc_available();
void launch_chain_tc(const float* z, int64_t B, int q, const DevNet& net, const Sink& sink,
                     int num_sms, cudaStream_t s);
// standalone boundary IO (kernels_boundary_io.cu): a1 gather, a6 scatter + update norm + a8 reduction (one kernel)
int scatter_grid(int64_t B);
void launch_gather_phase(const float* lat, const LatticeGeom& L, const uint32_t* anchors, int64_t B, float* gb,
                         cudaStream_t s);
void launch_scatter_phase(float* lat, const LatticeGeom& L, const uint32_t* anchors, int64_t B, const float* pred,
                          unsigned int* blockmax /* kMaxSMs * 8 maxima + the ticket */, unsigned int* out /* [2] */,
                          cudaStream_t s);
void launch_loop_ctl(cudaGraphConditionalHandle h, const unsigned int* delta, unsigned int* st, int ce,
                     cudaStream_t s);
void launch_delta(const float* lat, const float* snap, const int64_t* segs, int nseg,
                  unsigned int* out /* [0]=max bits, [1]=nonfinite flag */, cudaStream_t s);
void launch_pack(const float* lat, const int32_t* idx, int64_t n, float* buf, cudaStream_t s);
void launch_unpack(float* lat, const int32_t* idx, int64_t n, const float* buf, cudaStream_t s);
// NEXT-2 peer-memory halo transport (kernels_p2p.cu).  A rank's P2P region
// (one cudaMalloc, IPC-exportable): u64 flags at 0 — packed epoch at
// kP2PPacked, consumed epoch of consumer rank r at kP2PConsumed + r, put-done
// epoch of sender rank r at kP2PPutDone + r — then the u64 epochs at
// kP2PEpochOff (pull epoch, put epoch of this sender, put-unpack epoch of this
// receiver), u32 block counters at kP2PCounterOff, then sendbuf[0], sendbuf[1]
// (pull mode, nsend floats each) and putbuf[0], putbuf[1] (put mode: written by
// the SENDERS' chain epilogues, nrecv floats each) from kP2PHeader.
constexpr int kP2PMaxRanks = 256;
constexpr int kP2PPacked = 0;
constexpr int kP2PConsumed = 8;
constexpr int kP2PPutDone = kP2PConsumed + kP2PMaxRanks;
constexpr size_t kP2PEpochOff = (size_t)(kP2PPutDone + kP2PMaxRanks) * 8;
constexpr size_t kP2PCounterOff = kP2PEpochOff + 64;
constexpr size_t kP2PHeader = 8192;
inline size_t p2p_parity_bytes(int64_t n) { return ((size_t)(n > 0 ? n : 1) * 4 + 255) / 256 * 256; }
inline size_t p2p_region_bytes(int64_t nsend, int64_t nrecv) {
  return kP2PHeader + 2 * p2p_parity_bytes(nsend) + 2 * p2p_parity_bytes(nrecv);
}
struct P2PSelf {
  int rank;
  unsigned long long* flags;  // own region
  unsigned long long* epoch;  // [0] pull epoch, [1] put epoch (sender), [2] put-unpack epoch (receiver)
  unsigned int* counter;      // [3]: pack, pull, put-unpack last-block tickets
  float* sendbuf[2];
  float* putbuf[2];           // own put-receive buffers
};
struct P2PPeer {               // device table, one entry per stencil peer, recv_off ascending
  int rank;
  unsigned long long* flags;  // the peer's region (peer memory)
  const float* sendbuf[2];    // the peer's send buffers
  int64_t send_off;           // this rank's segment inside the peer's send buffer
  int64_t recv_off;           // the segment's start in this rank's recv list
};
void launch_pack_p2p(const float* lat, const int32_t* idx, int64_t n, const P2PSelf& self, int npeers,
                     const P2PPeer* peers, cudaStream_t s);
void launch_pull_p2p(float* lat, const int32_t* idx, int64_t n, const P2PSelf& self, int npeers,
                     const P2PPeer* peers, cudaStream_t s);
// put mode: publish (sender, end of iteration) and unpack (receiver, side stream)
void launch_put_publish(const P2PSelf& self, int npeers, const P2PPeer* peers, cudaStream_t s);
void launch_put_unpack(float* lat, const int32_t* idx, const int32_t* slot, int64_t n, const P2PSelf& self,
                       int npeers, const P2PPeer* peers, cudaStream_t s);
void launch_final_lines(const float* lat, const LatticeGeom& L, int X0, int Y0, int bw, int bh,
                        float* field, int ld, cudaStream_t s);
// one-time preparation (kernels_prep.cu)
struct PrepArgs {
  const float* P;          // raw params, MFCK order
  int n_hidden;
  int d;                   // 128 or 256
  int f16;                 // tensor-core operand images in fp16 (1) or bf16 (0)
  int64_t oW1, oW2, oWh0;  // offsets; Wh_l at oWh0 + l*(d*d + d), bh_l right after
  float* W1T; float* WhT; float* bh;
  float* QTc; float* QTf;
  uint16_t* Wsw2;          // [n_hidden][kWImg] CTA-pair half images
  uint16_t* W1img;         // [d/128][2][128*128] W1 hi / lo bf16 images
};
bool embed_tc_enabled();
void launch_embed_tc(const float* lat, const LatticeGeom& L, const uint32_t* anchors, const float* gb,
                     int64_t B, const DevNet& net, float* z, cudaStream_t s);
void embed_tc_kernel_attributes();
void launch_prep(const PrepArgs& a, cudaStream_t s);
void sdnet_kernel_attributes();
void tc_kernel_attributes();
void launch_harmonic(int q, float* HT, cudaStream_t s);

}  // namespace mfp
