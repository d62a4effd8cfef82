// api.cu — the C ABI of include/mfp.h: validation, workspace carving, device
// preparation, the Algorithm-2 driver and its two transports:
//   * NCCL (one process per GPU; grouped ncclSend/ncclRecv to the <= 8 stencil
//     neighbours once per iteration; ncclAllReduce(MAX) for the
//     convergence test; point-to-point gather of the owned blocks), and
//   * local (MFP_ALL_RANKS: every rank of the processor grid on one device,
//     exchange by device-to-device copies of the same packed buffers).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include <time.h>

#include <nvtx3/nvToolsExt.h>

#include "mfp_internal.h"


using namespace mfp;

namespace {

struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base((char*)b) {}
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~(size_t)255;
    T* p = base ? (T*)(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
};

struct RankState {
  RankPlan plan;
  float* lat = nullptr;
  float* snap = nullptr;
  float* z = nullptr;
  int64_t zcap = 0;
  uint32_t* anchors[4] = {nullptr, nullptr, nullptr, nullptr};
  uint32_t* final_anchor = nullptr;
  uint32_t* final_lat_anchor = nullptr;
  int64_t* segs = nullptr;
  int nseg = 0;
  int32_t* send_idx = nullptr;
  int32_t* recv_idx = nullptr;
  float* sendbuf = nullptr;
  float* recvbuf = nullptr;
  std::vector<int64_t> send_off, recv_off;
  int64_t nsend = 0, nrecv = 0;
  float* block = nullptr;  // owned block field (NCCL transport with R > 1)
  char* p2p = nullptr;         // NEXT-2 peer-memory region (own cudaMalloc, IPC-exportable)
  P2PPeer* p2p_tab = nullptr;  // device table of the stencil peers' regions
  int p2p_np = 0;
  // put mode (mfp_p2p_set_mode): sender tables and the receiver's unpack list
  int32_t* putmap = nullptr;   // [lattice cells]: -1 or first << 2 | count into putdst
  int32_t* putdst = nullptr;   // peer index << 24 | slot in the peer's putbuf
  float** putbufs = nullptr;   // [2 * npeers]: peer i's putbuf[parity]
  int32_t* pu_idx = nullptr;   // receiver: halo cells refreshed by puts (∂Ω cells excluded)
  int32_t* pu_slot = nullptr;  //           and their slots in the own putbuf
  int64_t npu = 0;
};

}  // namespace

struct mfp_ctx {
  mfp_config cfg;
  mfp_sdnet_desc net;
  int rank = 0;          // this process's rank, or MFP_ALL_RANKS
  int R = 1;
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;         // halo exchange (overlaps interior phase 0)
  cudaEvent_t ev_packed = nullptr, ev_unpacked = nullptr;
  float* pipe_host = nullptr;          // mfp_solve, one rank: D2H of the field overlapped with the final phase
  cudaEvent_t ev_band[4] = {nullptr, nullptr, nullptr, nullptr};
  bool pending = false;                // an exchange is in flight on `side`
  bool use_graphs = false;             // replay blocks of c iterations as CUDA graphs
  int exchange_every = 1;              // halo exchange after every s-th iteration (NEXT-4)
  bool p2p = false;                    // halo transport: peer-memory kernels (NEXT-2) instead of NCCL / copies
  bool p2p_put = false;                // ... with puts from the chain epilogue instead of pack + pull
  std::vector<void*> p2p_opened;       // IPC-mapped peer regions (multi-process)
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};  // [0] plain block, [1] block ending in a check
  cudaGraphExec_t gloop = nullptr;     // WHILE graph: blocks of c iterations + on-device stopping rule
  bool exact_persist = false;          // exact subsolver, one rank: persistent dataflow iteration kernel
  ExactIterArgs xargs{};               // its tables (device, owned by the context)
  int gloop_launches = 0;              // kernels per loop-body block
  unsigned int* loopst = nullptr;      // device {iterations, t, tol bits, blocks}
  unsigned int* hloop = nullptr;       // pinned host mirror
  int glaunches[2] = {0, 0};
  std::vector<RankState> ranks;
  DevNet dn{};
  float* params = nullptr;
  float* full = nullptr;     // (ny+1)(nx+1) device field (rank 0 / ALL)
  float* gstage = nullptr;   // 2(nx+ny)
  float* gather = nullptr;   // rank 0, NCCL: other ranks' blocks
  unsigned int* delta = nullptr;  // [2]
  unsigned int* hdelta = nullptr;  // pinned
  unsigned int* iomax = nullptr;   // scatter block maxima (a6 standalone)
  unsigned int* ioout = nullptr;   // [2] reduced update norm + non-finite flag
  int num_sms = 0;   // set from the device in mfp_init
  int launches = 0;
  bool poisoned = false;
  std::string err;
  // profiling
  bool profiling = false;
  std::vector<cudaEvent_t> evpool;
  size_t evnext = 0;
  struct Span { cudaEvent_t a, b; int kind; int64_t units; };
  std::vector<Span> spans;
};

namespace {

}  // namespace

int mfp::num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v > 0 ? v : 148;
  }
  return cache[dev];
}

bool mfp::pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MFP_NO_PDL");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

namespace {

// NVTX ranges (header-only NVTX 3: no-ops unless a tool such as ncu --nvtx or
// nsys attaches) around the host-side steps of a solve, so a profile of any
// caller shows init / blocks of c iterations / convergence loop / final phase /
// halo exchange / batch calls by name.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

const int kKindGather = 0, kKindChain = 1, kKindExact = 2, kKindHalo = 3, kKindDelta = 4;

mfp_status fail(mfp_ctx* c, mfp_status st, const std::string& msg) {
  if (c) {
    c->err = msg;
    if (st == MFP_ERR_CUDA || st == MFP_ERR_NCCL) c->poisoned = true;
  }
  return st;
}

#define CK(call)                                                                           \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(c, MFP_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));    \
  } while (0)
#define NK(call)                                                                           \
  do {                                                                                     \
    ncclResult_t r_ = (call);                                                              \
    if (r_ != ncclSuccess) {                                                               \
      if (c && c->comm) ncclCommAbort(c->comm), c->comm = nullptr;                         \
      return fail(c, MFP_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_));    \
    }                                                                                      \
  } while (0)

// Host wait on `stream` that also watches the NCCL communicator: a peer that
// died or errored never completes its side of a collective, which would leave
// this rank blocked in cudaStreamSynchronize forever.  Polls the stream and
// ncclCommGetAsyncError; on an async error or after MFP_NCCL_TIMEOUT_S seconds
// (default 600) the communicator is aborted and the context poisoned
// (NCCL errors are sticky; SPEC's watchdog analog).
double nccl_timeout_s() {
  static double v = -1.0;
  if (v < 0.0) {
    const char* e = getenv("MFP_NCCL_TIMEOUT_S");
    v = (e && atof(e) > 0.0) ? atof(e) : 600.0;
  }
  return v;
}

mfp_status wait_stream(mfp_ctx* c, cudaStream_t st) {
  if (!c->comm) {
    CK(cudaStreamSynchronize(st));
    return MFP_OK;
  }
  struct timespec t0, now;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (unsigned spin = 0;; spin++) {
    const cudaError_t q = cudaStreamQuery(st);
    if (q == cudaSuccess) return MFP_OK;
    if (q != cudaErrorNotReady) return fail(c, MFP_ERR_CUDA, std::string("stream: ") + cudaGetErrorString(q));
    ncclResult_t ar = ncclSuccess;
    ncclCommGetAsyncError(c->comm, &ar);
    clock_gettime(CLOCK_MONOTONIC, &now);
    const double el = (double)(now.tv_sec - t0.tv_sec) + 1e-9 * (double)(now.tv_nsec - t0.tv_nsec);
    if (ar != ncclSuccess && ar != ncclInProgress) {
      ncclCommAbort(c->comm);
      c->comm = nullptr;
      return fail(c, MFP_ERR_NCCL, std::string("NCCL async error: ") + ncclGetErrorString(ar));
    }
    if (el > nccl_timeout_s()) {
      ncclCommAbort(c->comm);
      c->comm = nullptr;
      return fail(c, MFP_ERR_NCCL, "NCCL watchdog: collective did not complete within MFP_NCCL_TIMEOUT_S");
    }
    if (spin > 64) {   // short spin first (sub-ms checks), then back off
      struct timespec ts = {0, 50000};
      nanosleep(&ts, nullptr);
    }
  }
}

// Collective agreement over the communicator (no-op without one): every rank
// contributes {digest, ~digest, flag}; after an allreduce-MAX, a rank sees
// max(d) == d and max(~d) == ~d only if every rank holds the same digest, and
// max(flag) != 0 if any rank raised its flag.  Returns MFP_OK / INVALID
// (digests differ) / `flag_status` (some rank flagged) on EVERY rank alike.
mfp_status agree(mfp_ctx* c, uint64_t digest, uint64_t flag, mfp_status flag_status, const char* what) {
  if (!c->comm) return flag ? fail(c, flag_status, what) : MFP_OK;
  uint64_t h[3] = {digest, ~digest, flag ? 1ull : 0ull};
  uint64_t* d = nullptr;
  CK(cudaMalloc((void**)&d, sizeof(h)));
  struct Free { uint64_t* p; ~Free() { cudaFree(p); } } fr{d};
  CK(cudaMemcpyAsync(d, h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
  NK(ncclAllReduce(d, d, 3, ncclUint64, ncclMax, c->comm, c->stream));
  uint64_t r[3];
  CK(cudaMemcpyAsync(r, d, sizeof(r), cudaMemcpyDeviceToHost, c->stream));
  if (mfp_status st = wait_stream(c, c->stream)) return st;
  if (r[2]) return fail(c, flag_status, std::string(what) + " (on at least one rank)");
  if (r[0] != digest || r[1] != ~digest)
    return fail(c, MFP_ERR_INVALID, "configuration / weights differ across ranks (collective digest mismatch)");
  return MFP_OK;
}

uint64_t fnv1a(uint64_t h, const void* p, size_t n) {
  const unsigned char* b = (const unsigned char*)p;
  for (size_t i = 0; i < n; i++) { h ^= b[i]; h *= 1099511628211ull; }
  return h;
}

mfp_status check_net(const mfp_sdnet_desc* n, std::string* err) {
  if (!n) { *err = "net is NULL"; return MFP_ERR_INVALID; }
  if (n->n_conv != 2 || n->conv_k[0] != kK || n->conv_k[1] != kK || n->conv_ch[0] != 1 ||
      n->conv_ch[1] != kC1 || n->conv_ch[2] != 1) {
    *err = "round-1 SDNet: conv 1->8->1, k=5 (reading G7)";
    return MFP_ERR_INVALID;
  }
  if (n->d != kD && n->d != kD2) { *err = "SDNet width d must be 128 or 256 (SURVEY §8(b))"; return MFP_ERR_INVALID; }
  if (n->n_hidden < 1 || n->n_hidden > kMaxHidden) { *err = "n_hidden must be 1..3"; return MFP_ERR_INVALID; }
  if (n->gelu < 0 || n->gelu > 2) { *err = "gelu must be 0, 1 or 2"; return MFP_ERR_INVALID; }
  return MFP_OK;
}

size_t param_count_of(const mfp_sdnet_desc* n) {
  size_t p = 0;
  for (int l = 0; l < n->n_conv; l++) {
    p += (size_t)n->conv_ch[l + 1] * n->conv_ch[l] * n->conv_k[l];
    p += (size_t)n->conv_ch[l + 1];
  }
  p += (size_t)n->d * n->conv_ch[n->n_conv] * kNB + (size_t)n->d * 2 + n->d;
  p += (size_t)n->n_hidden * ((size_t)n->d * n->d + n->d);
  p += (size_t)n->d + 1;
  return p;
}

// Carve (or size, when base == nullptr) the workspace.
void carve(mfp_ctx* c, void* base, size_t* total) {
  Carver cv(base);
  const int nh = c->net.n_hidden;
  DevNet& dn = c->dn;
  c->params = cv.take<float>(param_count_of(&c->net));
  const float* P = c->params;
  // parameter views (MFCK order)
  dn.conv1_w = P; dn.conv1_b = P + 40; dn.conv2_w = P + 48; dn.conv2_b = P + 88;
  const int d = c->net.d;
  const int64_t oW1 = 89, oW2 = oW1 + (int64_t)d * kNB, ob1 = oW2 + 2 * d, oWh0 = ob1 + d;
  const int64_t owo = oWh0 + (int64_t)nh * ((int64_t)d * d + d);
  dn.b1 = P ? P + ob1 : nullptr;
  dn.W2 = P ? P + oW2 : nullptr;
  dn.wo = P ? P + owo : nullptr;
  dn.bo = P ? P + owo + d : nullptr;
  dn.d = d;
  dn.n_hidden = nh;
  dn.gelu_tanh = c->net.gelu;
  dn.f16 = (c->cfg.precision == MFP_FP16 || c->cfg.precision == MFP_FP16X) ? 1 : 0;
  dn.split = c->cfg.precision == MFP_FP16X ? 1 : 0;
  dn.W1T = cv.take<float>((size_t)kNB * d);
  dn.WhT = cv.take<float>((size_t)nh * d * d);
  dn.bh = cv.take<float>((size_t)nh * d);
  dn.QTc = cv.take<float>((size_t)d * 64);
  dn.QTf = cv.take<float>((size_t)d * kQF);
  dn.Wh_sw2 = cv.take<uint16_t>(wimg_elems(d, nh));
  dn.W1img = cv.take<uint16_t>((size_t)2 * d * kNB);   // [d / 128 halves][hi | lo][128 x 128]
  dn.HcT = cv.take<float>((size_t)kNB * 64);
  dn.HfT = cv.take<float>((size_t)kNB * kQF);
  c->gstage = cv.take<float>((size_t)2 * (c->cfg.nx + c->cfg.ny));
  c->delta = cv.take<unsigned int>(4);
  c->loopst = cv.take<unsigned int>(4);
  c->iomax = cv.take<unsigned int>(kMaxSMs * 8 + 32);   // >= scatter_grid(B) for any B, + the ticket
  c->ioout = cv.take<unsigned int>(2);
  const bool need_full = (c->rank == MFP_ALL_RANKS || c->rank == 0);
  c->full = need_full ? cv.take<float>((size_t)(c->cfg.nx + 1) * (c->cfg.ny + 1)) : nullptr;
  if (c->rank == 0 && c->R > 1) c->gather = cv.take<float>((size_t)(c->cfg.nx + 1) * (c->cfg.ny + 1));
  for (auto& rs : c->ranks) {
    const RankPlan& p = rs.plan;
    rs.lat = cv.take<float>(p.lat.cells);
    rs.snap = cv.take<float>(p.lat.cells);
    int64_t zc = 1;
    for (int k = 0; k < 4; k++) zc = std::max<int64_t>(zc, p.phase_anchor[k].size());
    zc = std::max<int64_t>(zc, p.final_anchor.size());
    zc = std::max<int64_t>(zc, 4096);  // staging for mfp_sdnet_batch chunks
    rs.zcap = zc;
    rs.z = cv.take<float>((size_t)zc * d);
    for (int k = 0; k < 4; k++) rs.anchors[k] = cv.take<uint32_t>(std::max<size_t>(1, p.phase_anchor[k].size()));
    rs.final_anchor = cv.take<uint32_t>(std::max<size_t>(1, p.final_anchor.size()));
    rs.final_lat_anchor = cv.take<uint32_t>(std::max<size_t>(1, p.final_lat_anchor.size()));
    rs.nseg = (int)p.delta_seg.size();
    rs.segs = cv.take<int64_t>(std::max<size_t>(1, p.delta_seg.size()));
    rs.nsend = rs.nrecv = 0;
    rs.send_off.clear(); rs.recv_off.clear();
    for (auto& pp : p.peers) {
      rs.send_off.push_back(rs.nsend); rs.nsend += pp.send_idx.size();
      rs.recv_off.push_back(rs.nrecv); rs.nrecv += pp.recv_idx.size();
    }
    rs.send_idx = cv.take<int32_t>(std::max<int64_t>(1, rs.nsend));
    rs.recv_idx = cv.take<int32_t>(std::max<int64_t>(1, rs.nrecv));
    rs.sendbuf = cv.take<float>(std::max<int64_t>(1, rs.nsend));
    rs.recvbuf = cv.take<float>(std::max<int64_t>(1, rs.nrecv));
    rs.block = (c->rank != MFP_ALL_RANKS && c->R > 1) ? cv.take<float>((size_t)p.bw * p.bh) : nullptr;
  }
  *total = cv.off + 256;
}

Sink lattice_sink(RankState& rs, int kphase) {
  Sink s{};
  s.mode = 0; s.q = kQC; s.lat = rs.lat; s.offV = rs.plan.lat.offV;
  s.strideH = rs.plan.lat.strideH; s.strideV = rs.plan.lat.strideV;
  s.anchors = rs.anchors[kphase];
  if (rs.putmap) {   // NEXT-2 put transport
    s.putmap = rs.putmap;
    s.putdst = rs.putdst;
    s.putbufs = rs.putbufs;
    s.put_epoch = (const unsigned long long*)(rs.p2p + kP2PEpochOff) + 1;
  }
  return s;
}

cudaEvent_t ev(mfp_ctx* c) {
  if (c->evnext >= c->evpool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->evpool.push_back(e);
  }
  return c->evpool[c->evnext++];
}

struct SpanGuard {
  mfp_ctx* c; int kind; int64_t units; cudaEvent_t a = nullptr;
  SpanGuard(mfp_ctx* c_, int k, int64_t u) : c(c_), kind(k), units(u) {
    if (c->profiling) { a = ev(c); cudaEventRecord(a, c->stream); }
  }
  ~SpanGuard() {
    if (c->profiling) {
      cudaEvent_t b = ev(c);
      cudaEventRecord(b, c->stream);
      c->spans.push_back({a, b, kind, units});
    }
  }
};

// N2 + N3: gather + embedding z = W1 e + b1; the tensor-core precisions use the
// tcgen05 split-bf16 embed (kernels_embed_tc.cu), fp32 the SIMT one.
void embed(mfp_ctx* c, const float* lat, const LatticeGeom& L, const uint32_t* anchors, const float* gb,
           int64_t B, float* z) {
  if (c->cfg.precision != MFP_FP32 && embed_tc_enabled())
    launch_embed_tc(lat, L, anchors, gb, B, c->dn, z, c->stream);
  else launch_gather_embed(lat, L, anchors, gb, B, c->dn, z, c->stream);
}

void chain(mfp_ctx* c, const float* z, int64_t B, int q, const Sink& sk) {
  SpanGuard g(c, kKindChain, B * q);
  if (c->cfg.precision != MFP_FP32) launch_chain_tc(z, B, q, c->dn, sk, c->num_sms, c->stream);
  else launch_chain_fp32(z, B, q, c->dn, sk, c->stream);
  c->launches++;
}

// One phase (or the anchor sub-range [b0, b1) of it) of one rank.
void run_phase(mfp_ctx* c, RankState& rs, int ph, int64_t b0 = 0, int64_t b1 = -1) {
  if (b1 < 0) b1 = (int64_t)rs.plan.phase_anchor[ph].size();
  const int64_t B = b1 - b0;
  if (B <= 0) return;
  const uint32_t* anchors = rs.anchors[ph] + b0;
  if (c->cfg.subsolver == MFP_EXACT_LAPLACE) {
    SpanGuard g(c, kKindExact, B);
    launch_exact_phase(rs.lat, rs.plan.lat, anchors, B, c->dn.HcT, c->stream);
    c->launches++;
  } else {
    {
      SpanGuard g(c, kKindGather, B);
      embed(c, rs.lat, rs.plan.lat, anchors, nullptr, B, rs.z);
      c->launches++;
    }
    Sink sk = lattice_sink(rs, ph);
    sk.anchors = anchors;
    chain(c, rs.z, B, kQC, sk);
  }
}

// communicate_new_boundaries, once per iteration, split in two
// halves so the exchange overlaps the next iteration's interior phase-0
// subdomains (north_star): exchange_begin packs on the main stream (a snapshot
// of the owned cells), then the transport — grouped ncclSend/ncclRecv, or
// device copies for MFP_ALL_RANKS — and the unpack run on the side stream;
// exchange_wait makes the main stream wait for the unpack.
P2PSelf p2p_self(const RankState& rs) {
  P2PSelf s{};
  s.rank = rs.plan.rank;
  s.flags = (unsigned long long*)rs.p2p;
  s.epoch = (unsigned long long*)(rs.p2p + kP2PEpochOff);
  s.counter = (unsigned int*)(rs.p2p + kP2PCounterOff);
  s.sendbuf[0] = (float*)(rs.p2p + kP2PHeader);
  s.sendbuf[1] = (float*)(rs.p2p + kP2PHeader + p2p_parity_bytes(rs.nsend));
  s.putbuf[0] = (float*)(rs.p2p + kP2PHeader + 2 * p2p_parity_bytes(rs.nsend));
  s.putbuf[1] = (float*)(rs.p2p + kP2PHeader + 2 * p2p_parity_bytes(rs.nsend) + p2p_parity_bytes(rs.nrecv));
  return s;
}

// NEXT-2 transport (kernels_p2p.cu): pack + publish on the main stream, then
// the fused pull + unpack on the side stream; no NCCL call, no host wait.
mfp_status exchange_begin_p2p(mfp_ctx* c) {
  if (c->p2p_put) {
    // put mode: the epilogues already stored the halo values into the peers'
    // put buffers; publish them, then unpack the own put buffer on the side stream
    for (auto& rs : c->ranks) {
      launch_put_publish(p2p_self(rs), rs.p2p_np, rs.p2p_tab, c->stream);
      c->launches++;
    }
    CK(cudaEventRecord(c->ev_packed, c->stream));
    CK(cudaStreamWaitEvent(c->side, c->ev_packed, 0));
    cudaEvent_t h0 = nullptr;
    if (c->profiling) {
      h0 = ev(c);
      cudaEventRecord(h0, c->side);
    }
    for (auto& rs : c->ranks) {
      launch_put_unpack(rs.lat, rs.pu_idx, rs.pu_slot, rs.npu, p2p_self(rs), rs.p2p_np, rs.p2p_tab, c->side);
      c->launches++;
    }
    CK(cudaEventRecord(c->ev_unpacked, c->side));
    if (c->profiling) {
      cudaEvent_t h1 = ev(c);
      cudaEventRecord(h1, c->side);
      c->spans.push_back({h0, h1, kKindHalo, 0});
    }
    c->pending = true;
    return MFP_OK;
  }
  for (auto& rs : c->ranks) {
    launch_pack_p2p(rs.lat, rs.send_idx, rs.nsend, p2p_self(rs), rs.p2p_np, rs.p2p_tab, c->stream);
    c->launches++;
  }
  CK(cudaEventRecord(c->ev_packed, c->stream));
  CK(cudaStreamWaitEvent(c->side, c->ev_packed, 0));
  cudaEvent_t h0 = nullptr;
  if (c->profiling) {
    h0 = ev(c);
    cudaEventRecord(h0, c->side);
  }
  for (auto& rs : c->ranks) {
    launch_pull_p2p(rs.lat, rs.recv_idx, rs.nrecv, p2p_self(rs), rs.p2p_np, rs.p2p_tab, c->side);
    c->launches++;
  }
  CK(cudaEventRecord(c->ev_unpacked, c->side));
  if (c->profiling) {
    cudaEvent_t h1 = ev(c);
    cudaEventRecord(h1, c->side);
    c->spans.push_back({h0, h1, kKindHalo, 0});
  }
  c->pending = true;
  return MFP_OK;
}

mfp_status exchange_begin(mfp_ctx* c) {
  if (c->R == 1) return MFP_OK;
  Nvtx nv("mfp: halo exchange (a7)");
  if (c->p2p) return exchange_begin_p2p(c);
  for (auto& rs : c->ranks) {
    launch_pack(rs.lat, rs.send_idx, rs.nsend, rs.sendbuf, c->stream);
    c->launches++;
  }
  CK(cudaEventRecord(c->ev_packed, c->stream));
  CK(cudaStreamWaitEvent(c->side, c->ev_packed, 0));
  cudaEvent_t h0 = nullptr;
  if (c->profiling) {  // transport + unpack span, timed on the side stream
    h0 = ev(c);
    cudaEventRecord(h0, c->side);
  }
  if (c->rank == MFP_ALL_RANKS) {
    for (auto& dst : c->ranks)
      for (size_t i = 0; i < dst.plan.peers.size(); i++) {
        const RankState& src = c->ranks[dst.plan.peers[i].rank];
        size_t j = 0;  // dst's index in src's peer list
        while (j < src.plan.peers.size() && src.plan.peers[j].rank != dst.plan.rank) j++;
        const int64_t n = (int64_t)dst.plan.peers[i].recv_idx.size();
        if (n == 0) continue;
        CK(cudaMemcpyAsync(dst.recvbuf + dst.recv_off[i], src.sendbuf + src.send_off[j],
                           n * sizeof(float), cudaMemcpyDeviceToDevice, c->side));
      }
  } else {
    RankState& rs = c->ranks[0];
    NK(ncclGroupStart());
    for (size_t i = 0; i < rs.plan.peers.size(); i++) {
      const auto& pp = rs.plan.peers[i];
      if (!pp.send_idx.empty())
        NK(ncclSend(rs.sendbuf + rs.send_off[i], pp.send_idx.size(), ncclFloat32, pp.rank, c->comm, c->side));
      if (!pp.recv_idx.empty())
        NK(ncclRecv(rs.recvbuf + rs.recv_off[i], pp.recv_idx.size(), ncclFloat32, pp.rank, c->comm, c->side));
    }
    NK(ncclGroupEnd());
  }
  for (auto& rs : c->ranks) {
    launch_unpack(rs.lat, rs.recv_idx, rs.nrecv, rs.recvbuf, c->side);
    c->launches++;
  }
  CK(cudaEventRecord(c->ev_unpacked, c->side));
  if (c->profiling) {
    cudaEvent_t h1 = ev(c);
    cudaEventRecord(h1, c->side);
    c->spans.push_back({h0, h1, kKindHalo, 0});
  }
  c->pending = true;
  return MFP_OK;
}

mfp_status exchange_wait(mfp_ctx* c) {
  if (!c->pending) return MFP_OK;
  CK(cudaStreamWaitEvent(c->stream, c->ev_unpacked, 0));
  c->pending = false;
  return MFP_OK;
}

// One iteration: phase 0 (interior subdomains first while a pending exchange
// is in flight, then the halo-touching ones), phases 1-3, then the exchange.
mfp_status iterate(mfp_ctx* c, bool exchange = true) {
  mfp_status st;
  if (c->exact_persist) {   // one launch: the 4 phases with dataflow stamps (single rank, no exchange)
    SpanGuard g(c, kKindExact, c->xargs.B[0] + c->xargs.B[1] + c->xargs.B[2] + c->xargs.B[3]);
    ExactIterArgs a = c->xargs;
    a.K = 1;
    launch_exact_iter(a, c->stream);
    c->launches++;
    return MFP_OK;
  }
  if (c->pending) {
    for (auto& rs : c->ranks) run_phase(c, rs, 0, 0, rs.plan.n0_interior);
    if ((st = exchange_wait(c))) return st;
    for (auto& rs : c->ranks) run_phase(c, rs, 0, rs.plan.n0_interior, -1);
  } else {
    for (auto& rs : c->ranks) run_phase(c, rs, 0);
  }
  for (int ph = 1; ph < 4; ph++)
    for (auto& rs : c->ranks) run_phase(c, rs, ph);
  return exchange ? exchange_begin(c) : MFP_OK;
}

// delta_k (reading G5) -> host, max over ranks; returns nonfinite flag
// Enqueue the delta reduction (no host sync: capturable into a graph).
mfp_status enqueue_delta(mfp_ctx* c, bool to_host = true) {
  CK(cudaMemsetAsync(c->delta, 0, 2 * sizeof(unsigned int), c->stream));
  {
    SpanGuard g(c, kKindDelta, 0);
    for (auto& rs : c->ranks) {
      launch_delta(rs.lat, rs.snap, rs.segs, rs.nseg, c->delta, c->stream);
      c->launches++;
    }
  }
  if (c->comm) NK(ncclAllReduce(c->delta, c->delta, 2, ncclUint32, ncclMax, c->comm, c->stream));
  if (to_host) CK(cudaMemcpyAsync(c->hdelta, c->delta, 2 * sizeof(unsigned int), cudaMemcpyDeviceToHost, c->stream));
  return MFP_OK;
}

// Host side of the check: wait for the pinned copy and decode it.
mfp_status read_delta(mfp_ctx* c, float* delta, bool* nonfinite) {
  if (mfp_status st = wait_stream(c, c->stream)) return st;
  uint32_t bits = c->hdelta[0];
  float d;
  memcpy(&d, &bits, 4);
  *delta = d;
  *nonfinite = c->hdelta[1] != 0;
  return MFP_OK;
}

mfp_status reduce_delta(mfp_ctx* c, float* delta, bool* nonfinite) {
  mfp_status st = enqueue_delta(c);
  if (st) return st;
  return read_delta(c, delta, nonfinite);
}

// Capture (once) and replay a block of c iterations as a CUDA graph.  kind 1
// ends with the snapshot-delta-allreduce of a check iteration (the pinned D2H
// copy of delta is a graph node; the host reads it after the launch).
mfp_status run_block(mfp_ctx* c, int kind) {
  Nvtx nv(kind ? "mfp: block of c iterations + delta (graph)" : "mfp: block of c iterations (graph)");
  const int ce = c->cfg.check_every;
  if (!c->gexec[kind]) {
    const int l0 = c->launches;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    mfp_status st = MFP_OK;
    for (int i = 0; i < ce && st == MFP_OK; i++) {
      if (kind == 1 && i == ce - 1)
        for (auto& rs : c->ranks)
          cudaMemcpyAsync(rs.snap, rs.lat, rs.plan.lat.cells * sizeof(float), cudaMemcpyDeviceToDevice, c->stream);
      st = iterate(c, (i + 1) % c->exchange_every == 0);
    }
    if (st == MFP_OK) st = exchange_wait(c);
    if (st == MFP_OK && kind == 1) st = enqueue_delta(c);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    if (st != MFP_OK) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    if (e != cudaSuccess) return fail(c, MFP_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    const cudaError_t ei = cudaGraphInstantiate(&c->gexec[kind], g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) return fail(c, MFP_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei));
    c->glaunches[kind] = c->launches - l0;
    c->launches = l0;
  }
  CK(cudaGraphLaunch(c->gexec[kind], c->stream));
  c->launches += c->glaunches[kind];
  return MFP_OK;
}

// On-device convergence loop: ONE graph launch runs blocks of
// c iterations until delta <= tol, a non-finite prediction, or no whole block
// fits into t — a CUDA graph WHILE node whose body is the check block (c
// iterations, snapshot, delta) followed by k_loop_ctl, which sets the node's
// condition on the device.  The host reads the loop state once at the end.
// Used for single-process contexts (R == 1 or MFP_ALL_RANKS); with an NCCL
// communicator the host checks every c iterations (NCCL kernels inside a
// conditional body are not validated on a one-GPU box).  MFP_NO_DEVICE_LOOP=1
// disables it (A/B).
bool device_loop_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MFP_NO_DEVICE_LOOP");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

mfp_status run_loop(mfp_ctx* c, int it, int t, float tol) {
  Nvtx nv("mfp: on-device convergence loop (WHILE graph)");
  const int ce = c->cfg.check_every;
  if (!c->gloop) {
    cudaGraph_t g = nullptr;
    CK(cudaGraphCreate(&g, 0));
    struct G { cudaGraph_t g; ~G() { if (g) cudaGraphDestroy(g); } } guard{g};
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1u, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, g, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    const int l0 = c->launches;
    CK(cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    mfp_status st = MFP_OK;
    for (int i = 0; i < ce && st == MFP_OK; i++) {
      if (i == ce - 1)
        for (auto& rs : c->ranks)
          cudaMemcpyAsync(rs.snap, rs.lat, rs.plan.lat.cells * sizeof(float), cudaMemcpyDeviceToDevice, c->stream);
      st = iterate(c, (i + 1) % c->exchange_every == 0);
    }
    if (st == MFP_OK) st = exchange_wait(c);
    if (st == MFP_OK) st = enqueue_delta(c, false);
    if (st == MFP_OK) {
      launch_loop_ctl(h, c->delta, c->loopst, ce, c->stream);
      c->launches++;
    }
    cudaGraph_t out = nullptr;
    const cudaError_t e = cudaStreamEndCapture(c->stream, &out);
    if (st != MFP_OK) return st;
    if (e != cudaSuccess) return fail(c, MFP_ERR_CUDA, std::string("loop capture: ") + cudaGetErrorString(e));
    const cudaError_t ei = cudaGraphInstantiate(&c->gloop, g, 0);
    if (ei != cudaSuccess) return fail(c, MFP_ERR_CUDA, std::string("loop instantiate: ") + cudaGetErrorString(ei));
    c->gloop_launches = c->launches - l0;
    c->launches = l0;
  }
  float tolv = tol;
  c->hloop[0] = (unsigned int)it;
  c->hloop[1] = (unsigned int)t;
  memcpy(&c->hloop[2], &tolv, 4);
  c->hloop[3] = 0u;
  CK(cudaMemcpyAsync(c->loopst, c->hloop, 4 * sizeof(unsigned int), cudaMemcpyHostToDevice, c->stream));
  CK(cudaGraphLaunch(c->gloop, c->stream));
  CK(cudaMemcpyAsync(c->hloop + 4, c->loopst, 4 * sizeof(unsigned int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(c->hdelta, c->delta, 2 * sizeof(unsigned int), cudaMemcpyDeviceToHost, c->stream));
  return MFP_OK;
}

// Final phase into the device field u (row-major, ld = nx+1).
// Single-rank SDNet final phase for mfp_solve with a HOST field: the atomic
// subdomains run in 4 row bands, and each band's rows are copied to the host on
// the side stream as soon as its chain kernel finishes, so the 67 MB D2H of C5
// overlaps the remaining bands instead of following the whole phase.  Same
// kernels, same per-row arithmetic as the one-shot path (bit-identical field).
mfp_status final_phase_banded(mfp_ctx* c, float* u) {
  RankState& rs = c->ranks[0];
  const RankPlan& p = rs.plan;
  const int W = c->cfg.nx + 1;
  launch_final_lines(rs.lat, p.lat, 0, 0, p.bw, p.bh, u, W, c->stream);
  c->launches++;
  const int Kx = c->cfg.nx / kM, Ky = c->cfg.ny / kM;
  const int nb = Ky < 4 ? Ky : 4;
  const int per = (Ky + nb - 1) / nb;
  for (int k = 0; k < nb; k++) {
    const int r0 = k * per, r1 = std::min(Ky, (k + 1) * per);
    if (r0 >= r1) break;
    const int64_t s0 = (int64_t)r0 * Kx, nbk = (int64_t)(r1 - r0) * Kx;
    embed(c, rs.lat, p.lat, rs.final_lat_anchor + s0, nullptr, nbk, rs.z);
    c->launches++;
    Sink sk{};
    sk.mode = 1; sk.q = kQF; sk.anchors = rs.final_anchor + s0; sk.field = u; sk.ld = W;
    chain(c, rs.z, nbk, kQF, sk);
    if (!c->ev_band[k]) CK(cudaEventCreateWithFlags(&c->ev_band[k], cudaEventDisableTiming));
    CK(cudaEventRecord(c->ev_band[k], c->stream));
    CK(cudaStreamWaitEvent(c->side, c->ev_band[k], 0));
    const int y0 = r0 * kM, y1 = (r1 == Ky) ? c->cfg.ny : r1 * kM - 1;   // line rows y = 32 r belong to the band above
    CK(cudaMemcpyAsync(c->pipe_host + (int64_t)y0 * W, u + (int64_t)y0 * W, (size_t)(y1 - y0 + 1) * W * sizeof(float),
                       cudaMemcpyDeviceToHost, c->side));
  }
  return MFP_OK;
}

mfp_status final_phase(mfp_ctx* c, float* u) {
  Nvtx nv("mfp: final phase (a9)");
  if (c->pipe_host && c->R == 1 && c->cfg.subsolver == MFP_SDNET) return final_phase_banded(c, u);
  const int W = c->cfg.nx + 1;
  for (auto& rs : c->ranks) {
    const RankPlan& p = rs.plan;
    float* field;
    int ld;
    if (rs.block) { field = rs.block; ld = p.bw; }
    else { field = u + (int64_t)p.Y0 * W + p.X0; ld = W; }
    launch_final_lines(rs.lat, p.lat, p.X0, p.Y0, p.bw, p.bh, field, ld, c->stream);
    c->launches++;
    const int64_t B = (int64_t)p.final_anchor.size();
    if (B == 0) continue;
    Sink sk{};
    sk.mode = 1; sk.q = kQF; sk.anchors = rs.final_anchor; sk.field = field; sk.ld = ld;
    if (c->cfg.subsolver == MFP_EXACT_LAPLACE) {
      launch_exact_general(rs.lat, p.lat, rs.final_lat_anchor, nullptr, B, kQF, c->dn.HfT, sk, c->stream);
      c->launches++;
    } else {
      for (int64_t s0 = 0; s0 < B; s0 += rs.zcap) {
        const int64_t nb = std::min(rs.zcap, B - s0);
        embed(c, rs.lat, p.lat, rs.final_lat_anchor + s0, nullptr, nb, rs.z);
        Sink sk2 = sk;
        sk2.anchors = rs.final_anchor + s0;
        c->launches++;
        chain(c, rs.z, nb, kQF, sk2);
      }
    }
  }
  if (c->rank != MFP_ALL_RANKS && c->R > 1) {
    // gather of the owned blocks to rank 0 (the paper's all_gather)
    RankState& rs = c->ranks[0];
    if (c->rank == 0) {
      GlobalPlan gp;
      std::string err;
      build_plan(&c->cfg, MFP_ALL_RANKS, &gp, &err);
      std::vector<int64_t> off(c->R, 0);
      int64_t o = 0;
      for (int r = 1; r < c->R; r++) { off[r] = o; o += (int64_t)gp.ranks[r].bw * gp.ranks[r].bh; }
      NK(ncclGroupStart());
      for (int r = 1; r < c->R; r++)
        NK(ncclRecv(c->gather + off[r], (size_t)gp.ranks[r].bw * gp.ranks[r].bh, ncclFloat32, r, c->comm, c->stream));
      NK(ncclGroupEnd());
      CK(cudaMemcpy2DAsync(u + (int64_t)rs.plan.Y0 * W + rs.plan.X0, W * sizeof(float), rs.block,
                           rs.plan.bw * sizeof(float), rs.plan.bw * sizeof(float), rs.plan.bh,
                           cudaMemcpyDeviceToDevice, c->stream));
      for (int r = 1; r < c->R; r++) {
        const RankPlan& q = gp.ranks[r];
        CK(cudaMemcpy2DAsync(u + (int64_t)q.Y0 * W + q.X0, W * sizeof(float), c->gather + off[r],
                             q.bw * sizeof(float), q.bw * sizeof(float), q.bh, cudaMemcpyDeviceToDevice,
                             c->stream));
      }
    } else {
      NK(ncclSend(rs.block, (size_t)rs.plan.bw * rs.plan.bh, ncclFloat32, 0, c->comm, c->stream));
    }
  }
  return MFP_OK;
}

mfp_status solve_impl(mfp_ctx* c, const float* g_dev, int32_t t, float tol, float* u_dev, bool do_final,
                      mfp_report* rep) {
  Nvtx nv("mfp_solve");
  if (c->poisoned) return MFP_ERR_STATE;
  if (t < 1 || !(tol >= 0.f)) return fail(c, MFP_ERR_INVALID, "max_iters >= 1 and tol >= 0 required");
  struct Events {   // destroyed on every return path
    cudaEvent_t e[3] = {nullptr, nullptr, nullptr};
    ~Events() {
      for (auto x : e)
        if (x) cudaEventDestroy(x);
    }
  } ev3;
  CK(cudaEventCreate(&ev3.e[0])); CK(cudaEventCreate(&ev3.e[1])); CK(cudaEventCreate(&ev3.e[2]));
  cudaEvent_t e0 = ev3.e[0], e1 = ev3.e[1], e2 = ev3.e[2];
  c->launches = 0;
  CK(cudaEventRecord(e0, c->stream));
  if (g_dev) {
    for (auto& rs : c->ranks) {
      launch_init_lattice(rs.lat, rs.plan.lat, c->cfg.nx, c->cfg.ny, g_dev, c->stream);
      c->launches += 1;
    }
  }
  const int ce = c->cfg.check_every;
  int it = 0;  // iterations completed
  bool converged = false;
  float delta = -1.f;
  while (it < t) {
    // A whole block of c iterations (starting on a block boundary, no exchange
    // in flight) replays one captured CUDA graph: c x (4 phases + exchange),
    // plus the snapshot / delta / allreduce of the check iteration.
    if (c->use_graphs && !c->comm && tol > 0.f && device_loop_enabled() && it % ce == 0 && t - it >= ce &&
        !c->pending) {
      mfp_status st = run_loop(c, it, t, tol);
      if (st) return st;
      bool bad = false;
      if ((st = read_delta(c, &delta, &bad))) return st;   // waits for the loop
      it = (int)c->hloop[4];
      c->launches += (int)c->hloop[7] * c->gloop_launches;
      if (bad) return fail(c, MFP_ERR_NONFINITE, "non-finite prediction (S:345)");
      if (delta <= tol) { converged = true; break; }
      continue;   // fewer than c iterations left: the per-iteration path below
    }
    if (c->use_graphs && it % ce == 0 && t - it >= ce && !c->pending) {
      // every block ends in a check (delta every c iterations, reading G5),
      // also in parity mode (tol == 0), where only the stop is disabled
      const int end = it + ce;
      const bool check = true;
      mfp_status st = run_block(c, check ? 1 : 0);
      if (st) return st;
      it = end;
      if (check) {
        bool bad = false;
        if ((st = read_delta(c, &delta, &bad))) return st;
        if (bad) return fail(c, MFP_ERR_NONFINITE, "non-finite prediction (S:345)");
        if (tol > 0.f && delta <= tol) { converged = true; break; }
      }
      continue;
    }
    it++;
    const bool check = (it % ce == 0) || it == t;
    // snapshot for delta (only owned cells are compared; halo cells being
    // unpacked concurrently on the side stream are never read back)
    if (check)
      for (auto& rs : c->ranks)
        CK(cudaMemcpyAsync(rs.snap, rs.lat, rs.plan.lat.cells * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
    mfp_status st = iterate(c, it % c->exchange_every == 0 || it == t);
    if (st) return st;
    if (check) {
      // complete the exchange first: NCCL ops on one communicator must not be
      // reordered across streams (allreduce on `stream`, send/recv on `side`)
      if ((st = exchange_wait(c))) return st;
      bool bad = false;
      st = reduce_delta(c, &delta, &bad);
      if (st) return st;
      if (bad) return fail(c, MFP_ERR_NONFINITE, "non-finite prediction (S:345)");
      if (tol > 0.f && it % ce == 0 && delta <= tol) { converged = true; break; }
    }
  }
  {
    mfp_status st = exchange_wait(c);
    if (st) return st;
  }
  CK(cudaEventRecord(e1, c->stream));
  if (do_final) {
    mfp_status st = final_phase(c, u_dev);
    if (st) return st;
  }
  CK(cudaEventRecord(e2, c->stream));
  if (mfp_status st = wait_stream(c, c->stream)) return st;
  CK(cudaGetLastError());
  if (rep) {
    memset(rep, 0, sizeof(*rep));
    rep->iterations = it;
    rep->converged = converged ? 1 : 0;
    rep->last_delta = delta;
    const double Kx = c->cfg.nx / kM, Ky = c->cfg.ny / kM;
    rep->predictions = (2 * Kx - 1) * (2 * Ky - 1) * it;
    double comp = 0;
    for (auto& rs : c->ranks)
      for (int k = 0; k < 4; k++) comp += rs.plan.phase_anchor[k].size();
    rep->predictions_computed = comp * it;
    float ms;
    cudaEventElapsedTime(&ms, e0, e2); rep->ms_total = ms;
    cudaEventElapsedTime(&ms, e1, e2); rep->ms_final = ms;
    int64_t bytes = 0;
    int msgs = 0;
    for (auto& rs : c->ranks) {
      bytes += rs.nsend * 4;
      int m = 0;
      for (auto& pp : rs.plan.peers) m += !pp.send_idx.empty();
      msgs = std::max(msgs, m);
    }
    // exchanges issued: after every s-th iteration and after the last one
    // (s | c, so a convergence stop also lands on an exchange): ceil(it / s)
    const int64_t s_ex = c->exchange_every;
    rep->halo_bytes_sent = bytes * ((it + s_ex - 1) / s_ex);
    rep->halo_msgs_per_iter = msgs;
    rep->gpu_launches = c->launches;
  }
  if (tol > 0.f && !converged) return MFP_NOT_CONVERGED;
  return MFP_OK;
}

}  // namespace

namespace {
// Dependency plan of the persistent exact-subsolver iteration (k_exact_iter):
// groups of 8 consecutive subdomains per phase (the warp granularity of the
// exact phase kernel); a group depends on every group of another phase that
// writes one of its perimeter cells (RAW) and, symmetrically, on every group
// that reads one of the cells it writes (WAR) or writes one of them too (WAW),
// and on itself.
mfp_status build_exact_persist(mfp_ctx* c) {
  RankState& rs = c->ranks[0];
  const RankPlan& p = rs.plan;
  const LatticeGeom& L = p.lat;
  ExactIterArgs& A = c->xargs;
  A.g0[0] = 0;
  for (int ph = 0; ph < 4; ph++) {
    A.B[ph] = (int64_t)p.phase_anchor[ph].size();
    A.g0[ph + 1] = A.g0[ph] + (A.B[ph] + 7) / 8;
  }
  const int64_t ng = A.g0[4];
  if (ng == 0) return MFP_OK;
  auto sub_of = [&](int ph, int64_t i, int& lx, int& ly, int& a, int& b) {
    const uint32_t pk = p.phase_anchor[ph][(size_t)i];
    a = (int)(pk & 0xffffu); b = (int)(pk >> 16); lx = kH * a; ly = kH * b;
  };
  std::vector<std::vector<int32_t>> wr(4, std::vector<int32_t>((size_t)L.cells, -1));
  for (int ph = 0; ph < 4; ph++)
    for (int64_t i = 0; i < A.B[ph]; i++) {
      int lx, ly, a, b;
      sub_of(ph, i, lx, ly, a, b);
      const int32_t gid = (int32_t)(A.g0[ph] + i / 8);
      for (int k = 1; k < kM; k++) {
        wr[ph][(size_t)(L.offV + (int64_t)(a + 1) * L.strideV + ly + k)] = gid;
        wr[ph][(size_t)((int64_t)(b + 1) * L.strideH + lx + k)] = gid;
      }
    }
  std::vector<std::vector<int32_t>> dep((size_t)ng);
  for (int ph = 0; ph < 4; ph++)
    for (int64_t i = 0; i < A.B[ph]; i++) {
      int lx, ly, a, b;
      sub_of(ph, i, lx, ly, a, b);
      const int32_t gid = (int32_t)(A.g0[ph] + i / 8);
      // WAW: a cell written in two phases keeps the later phase's value
      for (int k = 1; k < kM; k++) {
        const int64_t wc[2] = {L.offV + (int64_t)(a + 1) * L.strideV + ly + k, (int64_t)(b + 1) * L.strideH + lx + k};
        for (int64_t cell : wc)
          for (int q = 0; q < 4; q++) {
            if (q == ph) continue;
            const int32_t w = wr[q][(size_t)cell];
            if (w >= 0) { dep[(size_t)gid].push_back(w); dep[(size_t)w].push_back(gid); }
          }
      }
      for (int t = 0; t <= kM; t++) {
        const int64_t cells[4] = {(int64_t)b * L.strideH + lx + t, L.offV + (int64_t)(a + 2) * L.strideV + ly + t,
                                  (int64_t)(b + 2) * L.strideH + lx + t, L.offV + (int64_t)a * L.strideV + ly + t};
        for (int64_t cell : cells)
          for (int q = 0; q < 4; q++) {
            if (q == ph) continue;
            const int32_t w = wr[q][(size_t)cell];
            if (w >= 0) { dep[(size_t)gid].push_back(w); dep[(size_t)w].push_back(gid); }
          }
      }
    }
  std::vector<int32_t> off(1, 0), ids;
  for (int64_t g = 0; g < ng; g++) {
    auto& d = dep[(size_t)g];
    d.push_back((int32_t)g);
    std::sort(d.begin(), d.end());
    d.erase(std::unique(d.begin(), d.end()), d.end());
    ids.insert(ids.end(), d.begin(), d.end());
    off.push_back((int32_t)ids.size());
  }
  CK(cudaMalloc((void**)&A.dep_off, off.size() * 4));
  CK(cudaMalloc((void**)&A.dep_ids, std::max<size_t>(1, ids.size()) * 4));
  CK(cudaMalloc((void**)&A.done, (size_t)ng * 8 + 64));
  CK(cudaMemcpy((void*)A.dep_off, off.data(), off.size() * 4, cudaMemcpyHostToDevice));
  if (!ids.empty()) CK(cudaMemcpy((void*)A.dep_ids, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(A.done, 0, (size_t)ng * 8 + 64));
  A.iter_ctr = A.done + ng;
  A.ticket = (unsigned int*)(A.done + ng + 1);
  A.lat = rs.lat;
  A.L = L;
  for (int ph = 0; ph < 4; ph++) A.anchors[ph] = rs.anchors[ph];
  A.HcT = c->dn.HcT;
  A.K = 1;
  c->exact_persist = true;
  return MFP_OK;
}

// Before a rank frees its IPC-exported region (mfp_destroy), every stencil peer
// must have finished its last pull from it: peer r stores consumed[r] = e into
// THIS rank's region after reading exchange e (kernels_p2p.cu).  Poll those
// flags until they reach this rank's epoch (bounded: 30 s, then give up).
void p2p_quiesce(mfp_ctx* c) {
  RankState& rs = c->ranks[0];
  if (!rs.p2p) return;
  unsigned long long epoch = 0;   // the exchanges this rank published (pull epoch, or put epoch)
  if (cudaMemcpy(&epoch, rs.p2p + kP2PEpochOff + (c->p2p_put ? 8 : 0), 8, cudaMemcpyDeviceToHost) != cudaSuccess)
    return;
  std::vector<unsigned long long> flags(kP2PConsumed + kP2PMaxRanks);
  for (int spin = 0; spin < 300000; spin++) {
    if (cudaMemcpy(flags.data(), rs.p2p, flags.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return;
    bool done = true;
    for (const auto& pp : rs.plan.peers)
      if (flags[kP2PConsumed + pp.rank] < epoch) done = false;
    if (done) return;
    struct timespec ts = {0, 100000};
    nanosleep(&ts, nullptr);
  }
}

}  // namespace

// ============================================================== C ABI
extern "C" {

mfp_status mfp_param_count(const mfp_sdnet_desc* net, int32_t m, size_t* n) {
  std::string err;
  if (!n || m != kM) return MFP_ERR_INVALID;
  mfp_status st = check_net(net, &err);
  if (st) return st;
  *n = param_count_of(net);
  return MFP_OK;
}

mfp_status mfp_workspace_size(const mfp_config* cfg, const mfp_sdnet_desc* net, int rank, size_t* bytes) {
  if (!bytes) return MFP_ERR_INVALID;
  std::string err;
  mfp_ctx tmp;
  mfp_status st = check_net(net, &err);
  if (st) return st;
  GlobalPlan gp;
  st = build_plan(cfg, rank, &gp, &err);
  if (st) return st;
  tmp.cfg = *cfg; tmp.net = *net; tmp.rank = rank; tmp.R = gp.R;
  tmp.ranks.resize(gp.ranks.size());
  for (size_t i = 0; i < gp.ranks.size(); i++) tmp.ranks[i].plan = std::move(gp.ranks[i]);
  carve(&tmp, nullptr, bytes);
  return MFP_OK;
}

const char* mfp_last_error(const mfp_ctx* c) { return c ? c->err.c_str() : "ctx is NULL"; }

mfp_status mfp_init(const mfp_config* cfg, const mfp_sdnet_desc* net, const float* params,
                    size_t n_params, int rank, void* nccl_comm, void* workspace, size_t ws_bytes,
                    void* stream, mfp_ctx** out) {
  if (!out) return MFP_ERR_INVALID;
  *out = nullptr;
  mfp_ctx* c = new mfp_ctx();
  *out = c;
  std::string err;
  mfp_status st = check_net(net, &err);
  if (st) return fail(c, st, err);
  GlobalPlan gp;
  st = build_plan(cfg, rank, &gp, &err);
  if (st) return fail(c, st, err);
  c->cfg = *cfg; c->net = *net; c->rank = rank; c->R = gp.R;
  if (gp.R > 1 && rank != MFP_ALL_RANKS && !nccl_comm)
    return fail(c, MFP_ERR_INVALID, "nccl_comm required for a multi-rank grid");
  // (R == 1 may take a 1-rank communicator: the collective code paths — digest
  // agreement, delta allreduce inside the graphs, the NCCL watchdog — then run
  // on one GPU, which is how they are tested without a second device)
  if (rank == MFP_ALL_RANKS && nccl_comm)
    return fail(c, MFP_ERR_INVALID, "nccl_comm must be NULL for MFP_ALL_RANKS");
  c->comm = (ncclComm_t)nccl_comm;
  c->stream = (cudaStream_t)stream;
  if (cfg->subsolver == MFP_SDNET) {
    if (!params) return fail(c, MFP_ERR_INVALID, "params required for the SDNet subsolver");
    if (n_params != param_count_of(net)) return fail(c, MFP_ERR_INVALID, "n_params mismatch (S:387 order)");
    // (identical weights on every rank are enforced by the collective digest
    // below, so a non-finite parameter is seen by every rank alike)
    for (size_t i = 0; i < n_params; i++)
      if (!std::isfinite(params[i])) return fail(c, MFP_ERR_NONFINITE, "non-finite parameter");
  }
  if (cfg->precision != MFP_FP32 && cfg->subsolver == MFP_SDNET && !chain_tc_available())
    return fail(c, MFP_ERR_INVALID, "tcgen05 chain not built into this library");
  if (cfg->precision == MFP_FP16X && cfg->subsolver == MFP_SDNET && net->d != kD)
    return fail(c, MFP_ERR_INVALID, "MFP_FP16X (split activations) supports d = 128");
  // collective validation: every rank of the communicator must
  // hold the same config, SDNet shape and weights; a rank whose local checks
  // failed makes every rank fail instead of leaving its peers blocked in the
  // first collective
  if (c->comm) {
    int nr = 0;
    NK(ncclCommCount(c->comm, &nr));
    if (nr != c->R) return fail(c, MFP_ERR_INVALID, "communicator size != grid_rows * grid_cols");
    uint64_t dg = 1469598103934665603ull;
    dg = fnv1a(dg, cfg, sizeof(*cfg));
    dg = fnv1a(dg, net, sizeof(*net));
    dg = fnv1a(dg, &n_params, sizeof(n_params));
    if (params) dg = fnv1a(dg, params, n_params * sizeof(float));
    if (mfp_status st2 = agree(c, dg, 0, MFP_OK, "")) return st2;
  }
  int dev = 0;
  cudaDeviceProp prop;
  CK(cudaGetDevice(&dev));
  CK(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10) return fail(c, MFP_ERR_CUDA, "libmfp requires an sm_100 (B200) device");
  c->num_sms = prop.multiProcessorCount;
  c->ranks.resize(gp.ranks.size());
  for (size_t i = 0; i < gp.ranks.size(); i++) c->ranks[i].plan = std::move(gp.ranks[i]);
  size_t need = 0;
  carve(c, nullptr, &need);
  if (!workspace || ws_bytes < need || ((uintptr_t)workspace & 255))
    return fail(c, MFP_ERR_WORKSPACE, "workspace too small or not 256-byte aligned");
  carve(c, workspace, &need);
  CK(cudaMallocHost(&c->hdelta, 4 * sizeof(unsigned int)));
  CK(cudaMallocHost(&c->hloop, 8 * sizeof(unsigned int)));
  CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  // graphs need a capturable (non-legacy) stream; MFP_NO_GRAPHS=1 disables them
  c->use_graphs = c->stream != nullptr && !(getenv("MFP_NO_GRAPHS") && getenv("MFP_NO_GRAPHS")[0] == '1');
  sdnet_kernel_attributes();
  exact_kernel_attributes();
  tc_kernel_attributes();
  embed_tc_kernel_attributes();
  CK(cudaEventCreateWithFlags(&c->ev_packed, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_unpacked, cudaEventDisableTiming));
  cudaStream_t s = c->stream;
  // scatter block maxima, the last-block ticket and the reduced norm start at 0
  CK(cudaMemsetAsync(c->iomax, 0, (kMaxSMs * 8 + 32) * sizeof(unsigned int), s));
  CK(cudaMemsetAsync(c->ioout, 0, 2 * sizeof(unsigned int), s));
  // upload plan tables
  for (auto& rs : c->ranks) {
    const RankPlan& p = rs.plan;
    for (int k = 0; k < 4; k++)
      if (!p.phase_anchor[k].empty())
        CK(cudaMemcpyAsync(rs.anchors[k], p.phase_anchor[k].data(), p.phase_anchor[k].size() * 4, cudaMemcpyHostToDevice, s));
    if (!p.final_anchor.empty()) {
      CK(cudaMemcpyAsync(rs.final_anchor, p.final_anchor.data(), p.final_anchor.size() * 4, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(rs.final_lat_anchor, p.final_lat_anchor.data(), p.final_lat_anchor.size() * 4, cudaMemcpyHostToDevice, s));
    }
    if (!p.delta_seg.empty())
      CK(cudaMemcpyAsync(rs.segs, p.delta_seg.data(), p.delta_seg.size() * 8, cudaMemcpyHostToDevice, s));
    for (size_t i = 0; i < p.peers.size(); i++) {
      const auto& pp = p.peers[i];
      if (!pp.send_idx.empty())
        CK(cudaMemcpyAsync(rs.send_idx + rs.send_off[i], pp.send_idx.data(), pp.send_idx.size() * 4, cudaMemcpyHostToDevice, s));
      if (!pp.recv_idx.empty())
        CK(cudaMemcpyAsync(rs.recv_idx + rs.recv_off[i], pp.recv_idx.data(), pp.recv_idx.size() * 4, cudaMemcpyHostToDevice, s));
    }
    CK(cudaMemsetAsync(rs.lat, 0, p.lat.cells * sizeof(float), s));
  }
  if (cfg->subsolver == MFP_SDNET) {
    CK(cudaMemcpyAsync(c->params, params, n_params * sizeof(float), cudaMemcpyHostToDevice, s));
    {
      // the tensor-core embed's constant-bank conv weights in channel-PAIR order
      // (kernels_embed_tc.cu conv_stack): [40) conv1 (w[2c][t], w[2c+1][t]) by
      // (c, t), [40, 48) conv1 biases, [48, 88) conv2 pairs likewise, [88] conv2
      // bias; conv2 weights halved when the channel activation yields 2 GELU
      // (gelu 1 / 2; exact power-of-two scaling)
      const float* c1w = params; const float* c1b = params + 40;
      const float* c2w = params + 48;
      const float h2 = net->gelu >= 1 ? 0.5f : 1.0f;
      for (int cp = 0; cp < kC1 / 2; cp++) {
        for (int t = 0; t < kK; t++)
          for (int u = 0; u < 2; u++) {
            c->dn.convw[2 * (cp * kK + t) + u] = c1w[(2 * cp + u) * kK + t];
            c->dn.convw[48 + 2 * (cp * kK + t) + u] = h2 * c2w[(2 * cp + u) * kK + t];
          }
        c->dn.convw[40 + 2 * cp] = c1b[2 * cp];
        c->dn.convw[40 + 2 * cp + 1] = c1b[2 * cp + 1];
      }
      c->dn.convw[88] = params[88];
    }
    {
      const int dd = net->d;   // 128 or 256 (check_net)
      const float* W2h = params + 89 + (int64_t)dd * kNB;   // [d][2]
      for (int n = 0; n < dd; n++) {
        c->dn.w2c[n] = W2h[2 * n];
        c->dn.w2c[dd + n] = W2h[2 * n + 1];
      }
    }
    CK(cudaMemsetAsync((void*)c->dn.Wh_sw2, 0, wimg_elems(net->d, net->n_hidden) * 2, s));
    PrepArgs a;
    a.P = c->params; a.n_hidden = net->n_hidden; a.d = net->d; a.f16 = (cfg->precision == MFP_FP16 || cfg->precision == MFP_FP16X) ? 1 : 0;
    a.oW1 = 89; a.oW2 = 89 + (int64_t)net->d * kNB; a.oWh0 = a.oW2 + 3 * (int64_t)net->d;
    a.W1T = (float*)c->dn.W1T; a.WhT = (float*)c->dn.WhT; a.bh = (float*)c->dn.bh;
    a.QTc = (float*)c->dn.QTc; a.QTf = (float*)c->dn.QTf;
    a.Wsw2 = (uint16_t*)c->dn.Wh_sw2;
    a.W1img = (uint16_t*)c->dn.W1img;
    launch_prep(a, s);
  } else {
    launch_harmonic(kQC, (float*)c->dn.HcT, s);
    launch_harmonic(kQF, (float*)c->dn.HfT, s);
  }
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  // MFP_PERSIST=1 (read per context): the exact subsolver on one rank runs each
  // iteration as ONE persistent dataflow kernel instead of four phase kernels
  // (NEXT-2; measured slower on one B200, so opt-in)
  const char* pe = getenv("MFP_PERSIST");
  if (cfg->subsolver == MFP_EXACT_LAPLACE && c->R == 1 && c->ranks.size() == 1 && pe && pe[0] == '1')
    if (mfp_status st2 = build_exact_persist(c)) return st2;
  return MFP_OK;
}

void mfp_destroy(mfp_ctx* c) {
  if (c)
    for (auto& e : c->ev_band)
      if (e) cudaEventDestroy(e);
  if (!c) return;
  for (auto e : c->evpool) cudaEventDestroy(e);
  if (c->hdelta) cudaFreeHost(c->hdelta);
  if (c->hloop) cudaFreeHost(c->hloop);
  if (c->gloop) cudaGraphExecDestroy(c->gloop);
  if (c->side) {
    cudaStreamSynchronize(c->side);
    cudaStreamDestroy(c->side);
  }
  for (auto& g : c->gexec)
    if (g) cudaGraphExecDestroy(g);
  if (c->ev_packed) cudaEventDestroy(c->ev_packed);
  if (c->ev_unpacked) cudaEventDestroy(c->ev_unpacked);
  if (c->p2p) {
    cudaStreamSynchronize(c->stream);
    if (c->rank != MFP_ALL_RANKS) p2p_quiesce(c);
  }
  for (void* p : c->p2p_opened) cudaIpcCloseMemHandle(p);
  for (void* q : {(void*)c->xargs.dep_off, (void*)c->xargs.dep_ids, (void*)c->xargs.done})
    if (q) cudaFree(q);
  for (auto& rs : c->ranks) {
    if (rs.p2p) cudaFree(rs.p2p);
    if (rs.p2p_tab) cudaFree(rs.p2p_tab);
    for (void* q : {(void*)rs.putmap, (void*)rs.putdst, (void*)rs.putbufs, (void*)rs.pu_idx, (void*)rs.pu_slot})
      if (q) cudaFree(q);
  }
  delete c;
}

// u pointers: the final phase runs iff the caller passes a non-NULL field
// pointer; the call is collective, so with NCCL every rank passes non-NULL
// (only rank 0's buffer is written) or every rank passes NULL.
mfp_status mfp_solve_device(mfp_ctx* c, const float* g_dev, int32_t max_iters, float tol, float* u_dev,
                            mfp_report* rep) {
  if (!c) return MFP_ERR_INVALID;
  if (c->poisoned) return MFP_ERR_STATE;
  const bool root = (c->rank == 0 || c->rank == MFP_ALL_RANKS);
  float* u = u_dev ? (root ? u_dev : c->ranks[0].block) : nullptr;
  return solve_impl(c, g_dev, max_iters, tol, u, u_dev != nullptr, rep);
}

mfp_status mfp_solve(mfp_ctx* c, const float* g, int32_t max_iters, float tol, float* u_out, mfp_report* rep) {
  if (!c) return MFP_ERR_INVALID;
  if (c->poisoned) return MFP_ERR_STATE;
  const size_t ng = 2 * (size_t)(c->cfg.nx + c->cfg.ny);
  const float* gd = nullptr;
  if (g) {
    bool bad = false;
    for (size_t i = 0; i < ng; i++)
      if (!std::isfinite(g[i])) bad = true;
    // collective: every rank returns NONFINITE together, none is left
    // waiting in the first exchange of a solve its peers abandoned
    if (mfp_status st = agree(c, 0, bad ? 1 : 0, MFP_ERR_NONFINITE, "non-finite boundary value (S:121)")) return st;
    CK(cudaMemcpyAsync(c->gstage, g, ng * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    gd = c->gstage;
  }
  const bool root = (c->rank == 0 || c->rank == MFP_ALL_RANKS);
  float* u = u_out ? (root ? c->full : c->ranks[0].block) : nullptr;
  const bool banded = u_out && root && c->R == 1 && c->cfg.subsolver == MFP_SDNET;
  c->pipe_host = banded ? u_out : nullptr;
  mfp_status st = solve_impl(c, gd, max_iters, tol, u, u_out != nullptr, rep);
  c->pipe_host = nullptr;
  if (banded) {
    CK(cudaStreamSynchronize(c->side));   // the band copies (also on error paths: no copy left in flight)
    return st;
  }
  if (st != MFP_OK && st != MFP_NOT_CONVERGED) return st;
  if (root && u_out) {
    const size_t nu = (size_t)(c->cfg.nx + 1) * (c->cfg.ny + 1);
    CK(cudaMemcpyAsync(u_out, c->full, nu * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  return st;
}

mfp_status mfp_sdnet_batch(mfp_ctx* c, const float* gb, int64_t B, int32_t query_set, float* out, void* stream) {
  if (!c) return MFP_ERR_INVALID;
  Nvtx nv("mfp_sdnet_batch");
  if (c->poisoned) return MFP_ERR_STATE;
  if (B < 0 || (B > 0 && (!gb || !out)) || (query_set != MFP_QUERY_CENTRE && query_set != MFP_QUERY_INTERIOR))
    return fail(c, MFP_ERR_INVALID, "bad sdnet_batch arguments");
  cudaStream_t saved = c->stream;
  if (stream) c->stream = (cudaStream_t)stream;
  const int q = query_set == MFP_QUERY_CENTRE ? kQC : kQF;
  RankState& rs = c->ranks[0];
  for (int64_t s0 = 0; s0 < B; s0 += rs.zcap) {
    const int64_t nb = std::min(rs.zcap, B - s0);
    Sink sk{};
    sk.mode = 2; sk.q = q; sk.out = out + s0 * q;
    if (c->cfg.subsolver == MFP_EXACT_LAPLACE) {
      launch_exact_general(nullptr, rs.plan.lat, nullptr, gb + s0 * kNB, nb, q,
                           q == kQC ? c->dn.HcT : c->dn.HfT, sk, c->stream);
    } else {
      {
        SpanGuard g(c, kKindGather, nb);
        embed(c, nullptr, rs.plan.lat, nullptr, gb + s0 * kNB, nb, rs.z);
      }
      chain(c, rs.z, nb, q, sk);
    }
  }
  cudaError_t e = cudaGetLastError();
  c->stream = saved;
  if (e != cudaSuccess) return fail(c, MFP_ERR_CUDA, cudaGetErrorString(e));
  return MFP_OK;
}

static mfp_status io_args(mfp_ctx* c, int32_t rank, int32_t phase, RankState** out) {
  if (!c) return MFP_ERR_INVALID;
  if (c->poisoned) return MFP_ERR_STATE;
  if (phase < 0 || phase > 3) return fail(c, MFP_ERR_INVALID, "phase must be 0..3");
  const int idx = c->rank == MFP_ALL_RANKS ? rank : 0;
  if ((c->rank != MFP_ALL_RANKS && rank != 0 && rank != c->rank) || idx < 0 || idx >= (int)c->ranks.size())
    return fail(c, MFP_ERR_INVALID, "rank out of range");
  *out = &c->ranks[idx];
  return MFP_OK;
}

mfp_status mfp_gather_phase(mfp_ctx* c, int32_t rank, int32_t phase, float* gb, int64_t cap, int64_t* B_out,
                            int32_t* ax_out, int32_t* ay_out) {
  RankState* rs = nullptr;
  if (mfp_status st = io_args(c, rank, phase, &rs)) return st;
  const RankPlan& p = rs->plan;
  const int64_t B = (int64_t)p.phase_anchor[phase].size();
  if (B_out) *B_out = B;
  if (!gb && !ax_out && !ay_out) return MFP_OK;   // size query
  if (cap < B) return fail(c, MFP_ERR_INVALID, "gather_phase: cap < number of subdomains");
  if ((ax_out == nullptr) != (ay_out == nullptr)) return fail(c, MFP_ERR_INVALID, "ax_out/ay_out: both or neither");
  if (ax_out)
    for (int64_t i = 0; i < B; i++) {
      const uint32_t pk = p.phase_anchor[phase][(size_t)i];
      ax_out[i] = p.lat.RX0 + kH * (int32_t)(pk & 0xffffu);
      ay_out[i] = p.lat.RY0 + kH * (int32_t)(pk >> 16);
    }
  if (gb) {
    launch_gather_phase(rs->lat, p.lat, rs->anchors[phase], B, gb, c->stream);
    c->launches++;
    CK(cudaGetLastError());
  }
  return MFP_OK;
}

mfp_status mfp_scatter_phase(mfp_ctx* c, int32_t rank, int32_t phase, const float* pred, int64_t B,
                             float* update_max) {
  RankState* rs = nullptr;
  if (mfp_status st = io_args(c, rank, phase, &rs)) return st;
  const RankPlan& p = rs->plan;
  if (B != (int64_t)p.phase_anchor[phase].size() || (B > 0 && !pred))
    return fail(c, MFP_ERR_INVALID, "scatter_phase: B must equal the phase's subdomain count");
  launch_scatter_phase(rs->lat, p.lat, rs->anchors[phase], B, pred, c->iomax, c->ioout, c->stream);
  c->launches += B > 0 ? 1 : 0;
  CK(cudaGetLastError());
  if (update_max) {
    unsigned int h[2];
    CK(cudaMemcpyAsync(h, c->ioout, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float v;
    memcpy(&v, &h[0], sizeof(v));
    *update_max = v;
    if (h[1]) return fail(c, MFP_ERR_NONFINITE, "scatter_phase: non-finite prediction");
  }
  return MFP_OK;
}

mfp_status mfp_set_exchange_every(mfp_ctx* c, int32_t s) {
  if (!c) return MFP_ERR_INVALID;
  if (c->poisoned) return MFP_ERR_STATE;
  if (s < 1 || c->cfg.check_every % s != 0)
    return fail(c, MFP_ERR_INVALID, "exchange_every must be >= 1 and divide check_every");
  if (s != c->exchange_every) {
    for (auto& g : c->gexec)
      if (g) { cudaGraphExecDestroy(g); g = nullptr; }
    if (c->gloop) { cudaGraphExecDestroy(c->gloop); c->gloop = nullptr; }
    c->exchange_every = s;
  }
  return MFP_OK;
}

namespace {
mfp_status p2p_alloc_own(mfp_ctx* c) {
  for (auto& rs : c->ranks)
    if (!rs.p2p) {
      const size_t bytes = p2p_region_bytes(rs.nsend, rs.nrecv);
      CK(cudaMalloc((void**)&rs.p2p, bytes));
      CK(cudaMemset(rs.p2p, 0, bytes));
    }
  CK(cudaDeviceSynchronize());
  return MFP_OK;
}
}  // namespace

mfp_status mfp_p2p_export(mfp_ctx* c, void* handle_out) {
  if (!c || !handle_out) return MFP_ERR_INVALID;
  if (c->poisoned) return MFP_ERR_STATE;
  if (c->rank == MFP_ALL_RANKS || c->R == 1)
    return fail(c, MFP_ERR_INVALID, "p2p_export: only for one-process-per-GPU contexts with R > 1");
  mfp_status st = p2p_alloc_own(c);
  if (st) return st;
  CK(cudaIpcGetMemHandle((cudaIpcMemHandle_t*)handle_out, c->ranks[0].p2p));
  return MFP_OK;
}

mfp_status mfp_p2p_open(mfp_ctx* c, const void* handles, int32_t n_handles) {
  if (!c) return MFP_ERR_INVALID;
  if (c->poisoned) return MFP_ERR_STATE;
  if (c->R == 1) return fail(c, MFP_ERR_INVALID, "p2p_open: a 1x1 grid has no halo");
  if (c->R > kP2PMaxRanks) return fail(c, MFP_ERR_INVALID, "p2p_open: more than 256 ranks");
  if (c->p2p) return fail(c, MFP_ERR_INVALID, "p2p_open: already open");
  if (c->pending) return fail(c, MFP_ERR_INVALID, "p2p_open: an exchange is in flight");
  const bool all = (c->rank == MFP_ALL_RANKS);
  if (all != (handles == nullptr))
    return fail(c, MFP_ERR_INVALID, "p2p_open: handles must be NULL exactly for MFP_ALL_RANKS");
  if (n_handles != (all ? 0 : c->R))
    return fail(c, MFP_ERR_INVALID, "p2p_open: n_handles must be R (0 for MFP_ALL_RANKS)");
  if (!all && !c->ranks[0].p2p) return fail(c, MFP_ERR_INVALID, "p2p_open: call mfp_p2p_export first");
  mfp_status st = p2p_alloc_own(c);
  if (st) return st;
  GlobalPlan gp;
  std::string err;
  if ((st = build_plan(&c->cfg, MFP_ALL_RANKS, &gp, &err))) return fail(c, st, err);
  std::vector<char*> base(c->R, nullptr);
  if (all) {
    for (auto& rs : c->ranks) base[rs.plan.rank] = rs.p2p;
  } else {
    // `handles` holds R 64-byte handles in rank order (the caller checks the count)
    base[c->rank] = c->ranks[0].p2p;
    for (const auto& pp : c->ranks[0].plan.peers) {
      if (base[pp.rank]) continue;
      void* p = nullptr;
      cudaIpcMemHandle_t h;
      memcpy(&h, (const char*)handles + (size_t)pp.rank * sizeof(cudaIpcMemHandle_t), sizeof(h));
      const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {   // roll back: a later retry starts from a clean state
        for (void* q : c->p2p_opened) cudaIpcCloseMemHandle(q);
        c->p2p_opened.clear();
        return fail(c, MFP_ERR_CUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
      }
      c->p2p_opened.push_back(p);
      base[pp.rank] = (char*)p;
    }
  }
  auto rollback = [&](mfp_status st, const std::string& msg) {
    for (auto& rs : c->ranks)
      if (rs.p2p_tab) { cudaFree(rs.p2p_tab); rs.p2p_tab = nullptr; rs.p2p_np = 0; }
    for (void* q : c->p2p_opened) cudaIpcCloseMemHandle(q);
    c->p2p_opened.clear();
    return fail(c, st, msg);
  };
  for (auto& rs : c->ranks) {
    std::vector<P2PPeer> tab;
    for (size_t i = 0; i < rs.plan.peers.size(); i++) {
      const int q = rs.plan.peers[i].rank;
      const RankPlan& qp = gp.ranks[q];
      int64_t off = 0, nq = 0, len = -1;
      for (const auto& x : qp.peers) {
        if (x.rank == rs.plan.rank) { len = (int64_t)x.send_idx.size(); off = nq; }
        nq += (int64_t)x.send_idx.size();
      }
      if (len != (int64_t)rs.plan.peers[i].recv_idx.size())
        return rollback(MFP_ERR_INVALID, "p2p_open: send/recv segment mismatch");
      P2PPeer e{};
      e.rank = q;
      e.flags = (unsigned long long*)base[q];
      e.sendbuf[0] = (const float*)(base[q] + kP2PHeader);
      e.sendbuf[1] = (const float*)(base[q] + kP2PHeader + p2p_parity_bytes(nq));
      e.send_off = off;
      e.recv_off = rs.recv_off[i];
      tab.push_back(e);
    }
    rs.p2p_np = (int)tab.size();
    cudaError_t e = cudaMalloc((void**)&rs.p2p_tab, std::max<size_t>(1, tab.size()) * sizeof(P2PPeer));
    if (e == cudaSuccess && !tab.empty())
      e = cudaMemcpy(rs.p2p_tab, tab.data(), tab.size() * sizeof(P2PPeer), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return rollback(MFP_ERR_CUDA, std::string("p2p_open: ") + cudaGetErrorString(e));
  }
  for (auto& g : c->gexec)
    if (g) { cudaGraphExecDestroy(g); g = nullptr; }
  if (c->gloop) { cudaGraphExecDestroy(c->gloop); c->gloop = nullptr; }
  c->p2p = true;
  return MFP_OK;
}

mfp_status mfp_p2p_set_mode(mfp_ctx* c, int32_t mode) {
  if (!c) return MFP_ERR_INVALID;
  if (c->poisoned) return MFP_ERR_STATE;
  if (mode != MFP_P2P_PULL && mode != MFP_P2P_PUT) return fail(c, MFP_ERR_INVALID, "p2p_set_mode: bad mode");
  if (!c->p2p) return fail(c, MFP_ERR_INVALID, "p2p_set_mode: call mfp_p2p_open first");
  if (c->pending) return fail(c, MFP_ERR_INVALID, "p2p_set_mode: an exchange is in flight");
  if ((mode == MFP_P2P_PUT) == c->p2p_put) return MFP_OK;
  if (mode == MFP_P2P_PUT && c->cfg.subsolver != MFP_SDNET)
    return fail(c, MFP_ERR_INVALID, "p2p_set_mode: puts come from the SDNet chain epilogue (MFP_SDNET only)");
  // switching resets the epochs: both transports start from a clean region
  // (collective: every rank switches at the same iteration boundary)
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaStreamSynchronize(c->side));
  auto free_put = [&](RankState& rs) {
    for (void* q : {(void*)rs.putmap, (void*)rs.putdst, (void*)rs.putbufs, (void*)rs.pu_idx, (void*)rs.pu_slot})
      if (q) cudaFree(q);
    rs.putmap = rs.putdst = rs.pu_idx = rs.pu_slot = nullptr;
    rs.putbufs = nullptr;
    rs.npu = 0;
  };
  for (auto& rs : c->ranks) free_put(rs);
  if (mode == MFP_P2P_PUT) {
    GlobalPlan gp;
    std::string err;
    if (mfp_status st = build_plan(&c->cfg, MFP_ALL_RANKS, &gp, &err)) return fail(c, st, err);
    const int nx = c->cfg.nx, ny = c->cfg.ny;
    auto on_boundary = [&](int x, int y) { return x == 0 || x == nx || y == 0 || y == ny; };
    std::vector<P2PPeer> tab;
    for (auto& rs : c->ranks) {
      const RankPlan& p = rs.plan;
      // sender: owned cell -> (peer i, slot in peer q's recv numbering); the
      // peer's recv segment from this rank has the same order as this rank's
      // send list to it (the pull transport relies on the same fact)
      std::vector<std::vector<int32_t>> dst((size_t)p.lat.cells);
      for (size_t i = 0; i < p.peers.size(); i++) {
        const RankPlan& qp = gp.ranks[p.peers[i].rank];
        int64_t base = 0;
        bool found = false;
        for (const auto& x : qp.peers) {
          if (x.rank == p.rank) { found = true; break; }
          base += (int64_t)x.recv_idx.size();
        }
        if (!found) return fail(c, MFP_ERR_INVALID, "p2p_set_mode: asymmetric stencil");
        if (base + (int64_t)p.peers[i].send_idx.size() >= (1 << 24) || p.peers.size() > 127)
          return fail(c, MFP_ERR_INVALID, "p2p_set_mode: put slot / peer index out of the 24 / 7-bit encoding");
        const auto& sp = p.peers[i];
        for (size_t k = 0; k < sp.send_idx.size(); k++) {
          if (on_boundary(sp.send_x[k], sp.send_y[k])) continue;   // never rewritten: no put
          dst[(size_t)sp.send_idx[k]].push_back((int32_t)((i << 24) | (size_t)(base + (int64_t)k)));
        }
      }
      std::vector<int32_t> map((size_t)p.lat.cells, -1), lst;
      for (size_t cell = 0; cell < dst.size(); cell++) {
        if (dst[cell].empty()) continue;
        if (dst[cell].size() > 3) return fail(c, MFP_ERR_INVALID, "p2p_set_mode: a cell in more than 3 halos");
        map[cell] = (int32_t)((lst.size() << 2) | dst[cell].size());
        lst.insert(lst.end(), dst[cell].begin(), dst[cell].end());
      }
      // receiver: every recv slot except the domain-boundary cells (their halo
      // copy is g, written by every rank's own init)
      std::vector<int32_t> uidx, uslot;
      int64_t o = 0;
      for (const auto& rp : p.peers)
        for (size_t k = 0; k < rp.recv_idx.size(); k++, o++)
          if (!on_boundary(rp.recv_x[k], rp.recv_y[k])) {
            uidx.push_back(rp.recv_idx[k]);
            uslot.push_back((int32_t)o);
          }
      // the peers' put buffers, parity 0 / 1
      tab.resize(p.peers.size());
      if (!p.peers.empty())
        CK(cudaMemcpy(tab.data(), rs.p2p_tab, p.peers.size() * sizeof(P2PPeer), cudaMemcpyDeviceToHost));
      std::vector<float*> bufs;
      for (size_t i = 0; i < p.peers.size(); i++) {
        const RankPlan& qp = gp.ranks[p.peers[i].rank];
        int64_t qs = 0, qr = 0;
        for (const auto& x : qp.peers) { qs += (int64_t)x.send_idx.size(); qr += (int64_t)x.recv_idx.size(); }
        char* qbase = (char*)tab[i].flags;   // the peer's region base
        bufs.push_back((float*)(qbase + kP2PHeader + 2 * p2p_parity_bytes(qs)));
        bufs.push_back((float*)(qbase + kP2PHeader + 2 * p2p_parity_bytes(qs) + p2p_parity_bytes(qr)));
      }
      auto up = [&](auto** dptr, const auto& v) -> cudaError_t {
        using T = typename std::remove_reference<decltype(v)>::type::value_type;
        cudaError_t e = cudaMalloc((void**)dptr, std::max<size_t>(1, v.size()) * sizeof(T));
        if (e == cudaSuccess && !v.empty()) e = cudaMemcpy(*dptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
        return e;
      };
      cudaError_t e = up(&rs.putmap, map);
      if (e == cudaSuccess) e = up(&rs.putdst, lst);
      if (e == cudaSuccess) e = up(&rs.putbufs, bufs);
      if (e == cudaSuccess) e = up(&rs.pu_idx, uidx);
      if (e == cudaSuccess) e = up(&rs.pu_slot, uslot);
      if (e != cudaSuccess) {
        for (auto& r2 : c->ranks) free_put(r2);
        return fail(c, MFP_ERR_CUDA, std::string("p2p_set_mode: ") + cudaGetErrorString(e));
      }
      rs.npu = (int64_t)uidx.size();
    }
  }
  // anchors: bit 31 marks the subdomains whose centre-line cells feed a peer's
  // halo (the epilogue looks up the put map only for those); plain in pull mode
  for (auto& rs : c->ranks) {
    const RankPlan& p = rs.plan;
    std::vector<int32_t> map;
    if (mode == MFP_P2P_PUT) {
      map.resize((size_t)p.lat.cells);
      CK(cudaMemcpy(map.data(), rs.putmap, map.size() * 4, cudaMemcpyDeviceToHost));
    }
    for (int k = 0; k < 4; k++) {
      std::vector<uint32_t> an = p.phase_anchor[k];
      if (mode == MFP_P2P_PUT)
        for (auto& pk : an) {
          const int a = (int)(pk & 0xffffu), b = (int)(pk >> 16), lx = kH * a, ly = kH * b;
          bool feeds = false;
          for (int t = 1; t < kM && !feeds; t++)
            feeds = map[(size_t)(p.lat.offV + (int64_t)(a + 1) * p.lat.strideV + ly + t)] >= 0 ||
                    map[(size_t)((int64_t)(b + 1) * p.lat.strideH + lx + t)] >= 0;
          if (feeds) pk |= 0x80000000u;
        }
      if (!an.empty()) CK(cudaMemcpy(rs.anchors[k], an.data(), an.size() * 4, cudaMemcpyHostToDevice));
    }
  }
  // fresh flags, epochs and tickets for the new protocol
  for (auto& rs : c->ranks) CK(cudaMemset(rs.p2p, 0, kP2PHeader));
  CK(cudaDeviceSynchronize());
  for (auto& g : c->gexec)
    if (g) { cudaGraphExecDestroy(g); g = nullptr; }
  if (c->gloop) { cudaGraphExecDestroy(c->gloop); c->gloop = nullptr; }
  c->p2p_put = (mode == MFP_P2P_PUT);
  return MFP_OK;
}

mfp_status mfp_step_phase(mfp_ctx* c, int32_t phase) {
  if (!c) return MFP_ERR_INVALID;
  if (c->poisoned) return MFP_ERR_STATE;
  if (phase < 0 || phase > 3) return fail(c, MFP_ERR_INVALID, "phase must be 0..3");
  for (auto& rs : c->ranks) run_phase(c, rs, phase);
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaGetLastError());
  return MFP_OK;
}

static mfp_status lines_io(mfp_ctx* c, int32_t rank, float* hl, float* vl, const float* hin, const float* vin) {
  if (!c) return MFP_ERR_INVALID;
  if (c->poisoned) return MFP_ERR_STATE;
  int idx = c->rank == MFP_ALL_RANKS ? rank : 0;
  if (idx < 0 || idx >= (int)c->ranks.size()) return fail(c, MFP_ERR_INVALID, "rank out of range");
  RankState& rs = c->ranks[idx];
  const LatticeGeom& L = rs.plan.lat;
  if (hl || hin) {
    if (hin) CK(cudaMemcpy2DAsync(rs.lat, L.strideH * 4, hin, L.lenH * 4, L.lenH * 4, L.nH, cudaMemcpyHostToDevice, c->stream));
    else CK(cudaMemcpy2DAsync(hl, L.lenH * 4, rs.lat, L.strideH * 4, L.lenH * 4, L.nH, cudaMemcpyDeviceToHost, c->stream));
  }
  if (vl || vin) {
    if (vin) CK(cudaMemcpy2DAsync(rs.lat + L.offV, L.strideV * 4, vin, L.lenV * 4, L.lenV * 4, L.nV, cudaMemcpyHostToDevice, c->stream));
    else CK(cudaMemcpy2DAsync(vl, L.lenV * 4, rs.lat + L.offV, L.strideV * 4, L.lenV * 4, L.nV, cudaMemcpyDeviceToHost, c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));
  return MFP_OK;
}

mfp_status mfp_export_lines(mfp_ctx* c, int32_t rank, float* hl, float* vl) {
  return lines_io(c, rank, hl, vl, nullptr, nullptr);
}
mfp_status mfp_import_lines(mfp_ctx* c, int32_t rank, const float* hl, const float* vl) {
  if (!hl || !vl) return MFP_ERR_INVALID;
  return lines_io(c, rank, nullptr, nullptr, hl, vl);
}

mfp_status mfp_profile_iterations(mfp_ctx* c, int32_t iters, mfp_profile* o) {
  if (!c || !o || iters < 1) return MFP_ERR_INVALID;
  if (c->poisoned) return MFP_ERR_STATE;
  memset(o, 0, sizeof(*o));
  c->profiling = true;
  c->spans.clear();
  c->evnext = 0;
  c->launches = 0;
  cudaEvent_t a = ev(c), b = ev(c);
  CK(cudaEventRecord(a, c->stream));
  for (int it = 0; it < iters; it++) {
    mfp_status st = iterate(c, (it + 1) % c->exchange_every == 0);
    if (st) { c->profiling = false; return st; }
  }
  {
    mfp_status st = exchange_wait(c);
    if (st) { c->profiling = false; return st; }
  }
  CK(cudaEventRecord(b, c->stream));
  CK(cudaEventSynchronize(b));
  c->profiling = false;
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  o->iterations = iters;
  o->ms_per_iter = ms / iters;
  o->launches_per_iter = c->launches / iters;
  double tg = 0, tc = 0, te = 0, th = 0, td = 0;
  int64_t ng = 0, nc = 0, ne = 0, nhh = 0, nd = 0;
  for (auto& sp : c->spans) {
    cudaEventElapsedTime(&ms, sp.a, sp.b);
    switch (sp.kind) {
      case kKindGather: tg += ms; ng++; o->gather_subdomains += sp.units; break;
      case kKindChain: tc += ms; nc++; o->chain_rows += sp.units; break;
      case kKindExact: te += ms; ne++; break;
      case kKindHalo: th += ms; nhh++; break;
      default: td += ms; nd++; break;
    }
  }
  o->ms_gather_embed = ng ? tg / ng : 0;
  o->ms_chain = nc ? tc / nc : 0;
  o->ms_exact = ne ? te / ne : 0;
  o->ms_halo = nhh ? th / nhh : 0;
  o->ms_delta = nd ? td / nd : 0;
  o->chain_launches = nc; o->chain_ms_total = tc;
  o->gather_launches = ng; o->gather_ms_total = tg;
  c->spans.clear();
  c->evnext = 0;
  CK(cudaGetLastError());
  return MFP_OK;
}

// ------------------------------------------------------------ NCCL bootstrap
mfp_status mfp_nccl_get_unique_id(void* id_out) {
  if (!id_out) return MFP_ERR_INVALID;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return MFP_ERR_NCCL;
  memcpy(id_out, &id, sizeof(id));
  return MFP_OK;
}

mfp_status mfp_nccl_comm_init(int32_t nranks, const void* id, int32_t rank, void** comm_out) {
  if (!id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) return MFP_ERR_INVALID;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm;
  if (ncclCommInitRank(&comm, nranks, uid, rank) != ncclSuccess) return MFP_ERR_NCCL;
  *comm_out = comm;
  return MFP_OK;
}

mfp_status mfp_nccl_comm_destroy(void* comm) {
  if (!comm) return MFP_ERR_INVALID;
  return ncclCommDestroy((ncclComm_t)comm) == ncclSuccess ? MFP_OK : MFP_ERR_NCCL;
}

}  // extern "C"
