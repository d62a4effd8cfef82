// NEXT-2: device-initiated halo exchange over peer memory (the
// paper points at NVSHMEM for direct GPU-GPU transfers).  Replaces the
// grouped ncclSend/ncclRecv + unpack of communicate_new_boundaries with
// two kernels and no host-side collective:
//   k_pack_p2p  (main stream): snapshots the owned send cells into
//               sendbuf[e & 1] ("new boundaries"; the previous pull made
//               sure every peer has consumed that buffer's exchange e - 2),
//               and the last block publishes packed = e (fence.sc.sys + relaxed store);
//   k_pull_p2p  (side stream): waits for each peer's packed >= e, loads the
//               peer's sendbuf[e & 1] segment addressed to this rank straight
//               over NVLink (or from the same device when every rank lives in
//               one process) into the halo cells of this rank's lattice (the
//               unpack is fused), and the last block publishes consumed[me] = e
//               on every peer, waits until every peer has consumed exchange
//               e - 1 (so pack(e + 1) may overwrite that parity buffer; the host
//               orders every pack after the previous pull, exchange_wait) and
//               advances this rank's epoch.
// The epoch lives in device memory, so both kernels replay unchanged inside
// the CUDA graphs of §8.  Deadlock freedom: pull(e) waits on
// peers' pack(e) and pull(e - 1), pack never waits; neither depends on a later
// kernel of the waiting rank.
#include "mfp_internal.h"

namespace mfp {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Relaxed system-scope store; preceded by one __threadfence_system() (fence.sc.sys)
// it forms the release pattern, so a block publishing to 8 peers pays one system
// membar instead of the one st.release.sys emits per store (MEMBAR.ALL.SYS each).
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Thread i < npeers spins until flag(i) >= want (all peers polled in parallel,
// one system-scope round trip instead of npeers); the block then proceeds.
template <class F>
__device__ __forceinline__ void block_wait_peers(int npeers, F flag, unsigned long long want) {
  if (threadIdx.x < npeers) {
    const unsigned long long* f = flag(threadIdx.x);
    while (ld_acquire_sys(f) < want) __nanosleep(64);
  }
  __syncthreads();
}

// Returns true in exactly one thread of the last block to finish (classic
// threadfence reduction); the counter is re-armed for the next launch.
__device__ __forceinline__ bool last_block(unsigned int* counter) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int t = atomicAdd(counter, 1u);
    am_last = (t == gridDim.x - 1);
    if (am_last) *counter = 0;
  }
  __syncthreads();
  return am_last && threadIdx.x == 0;
}

__global__ void k_pack_p2p(const float* __restrict__ lat, const int32_t* __restrict__ idx, int64_t n,
                           P2PSelf self, int npeers, const P2PPeer* __restrict__ peers) {
  // sendbuf[e & 1] was last read by the peers' pull(e - 2); this rank's pull(e - 1)
  // saw them consume it, and the host orders pack(e) after pull(e - 1)
  const unsigned long long e = *self.epoch + 1;
  float* buf = self.sendbuf[e & 1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = lat[__ldg(idx + i)];
  if (last_block(self.counter + 0)) {
    __threadfence_system();
    st_relaxed_sys(self.flags + kP2PPacked, e);
  }
}

__global__ void k_pull_p2p(float* __restrict__ lat, const int32_t* __restrict__ idx, int64_t n,
                           P2PSelf self, int npeers, const P2PPeer* __restrict__ peers) {
  const unsigned long long e = *self.epoch + 1;
  block_wait_peers(npeers, [&](int i) { return (const unsigned long long*)peers[i].flags + kP2PPacked; }, e);
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    int i = 0;
    while (i + 1 < npeers && j >= peers[i + 1].recv_off) i++;
    const P2PPeer& p = peers[i];
    // plain (weak) load is ordered after the acquire above by the block barrier
    lat[__ldg(idx + j)] = p.sendbuf[e & 1][p.send_off + (j - p.recv_off)];
  }
  if (last_block(self.counter + 1)) {
    __threadfence_system();
    for (int i = 0; i < npeers; i++) st_relaxed_sys(peers[i].flags + kP2PConsumed + self.rank, e);
    // free sendbuf[(e + 1) & 1] for pack(e + 1): the peers' pull(e - 1) has read it
    for (int i = 0; i < npeers; i++)
      while (ld_acquire_sys(self.flags + kP2PConsumed + peers[i].rank) + 1 < e) __nanosleep(64);
    *self.epoch = e;
  }
}

// ---- put mode (device-initiated halo from the chain epilogue, SURVEY NEXT-2:
// "the scatter epilogue puts strips into neighbours' halos").  During the
// phases of exchange e the chain epilogues of the SENDER store every owned cell
// a peer holds as a halo cell straight into the peer's putbuf[e & 1]
// (device_common.cuh put_halo; the last write of the iteration wins, so the
// buffer ends with the owner's end-of-iteration values, as a pack would).
//   k_put_publish (sender, main stream, after the iteration's last phase):
//     one system fence, put_done[me] = e on every peer; then wait until every
//     peer has unpacked exchange e - 1 (so the next iteration's puts, parity
//     (e + 1) & 1, overwrite a buffer nobody still reads), and advance the put
//     epoch the epilogues read.
//   k_put_unpack (receiver, side stream): wait for put_done >= e of every peer,
//     copy putbuf[e & 1] into the halo cells (local reads), publish
//     consumed[me] = e on every peer, advance the unpack epoch.
// No cycle: publish(e) waits on unpack(e - 1), unpack(e) on publish(e).
__global__ void k_put_publish(P2PSelf self, int npeers, const P2PPeer* __restrict__ peers) {
  if (threadIdx.x != 0) return;
  const unsigned long long e = self.epoch[1] + 1;
  // the chain kernels that stored the puts precede this kernel in stream order
  // (kernel boundary: their writes happen before this thread's operations), and
  // fence.sc.sys is cumulative: the flag below is ordered after those puts, as
  // after this thread's own writes — no fence in the 148 x 576 epilogue threads
  __threadfence_system();
  for (int i = 0; i < npeers; i++) st_relaxed_sys(peers[i].flags + kP2PPutDone + self.rank, e);
  for (int i = 0; i < npeers; i++)
    while (ld_acquire_sys(self.flags + kP2PConsumed + peers[i].rank) + 1 < e) __nanosleep(64);
  self.epoch[1] = e;
}

__global__ void k_put_unpack(float* __restrict__ lat, const int32_t* __restrict__ idx,
                             const int32_t* __restrict__ slot, int64_t n, P2PSelf self, int npeers,
                             const P2PPeer* __restrict__ peers) {
  const unsigned long long e = self.epoch[2] + 1;
  block_wait_peers(npeers, [&](int i) { return (const unsigned long long*)self.flags + kP2PPutDone + peers[i].rank; },
                   e);
  const float* buf = self.putbuf[e & 1];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    lat[__ldg(idx + j)] = buf[__ldg(slot + j)];
  if (last_block(self.counter + 2)) {
    __threadfence_system();
    for (int i = 0; i < npeers; i++) st_relaxed_sys(peers[i].flags + kP2PConsumed + self.rank, e);
    self.epoch[2] = e;
  }
}

static int grid_p2p(int64_t n) {
  int64_t b = (n + 255) / 256;
  // every pull block polls the <= 8 peer flags (one thread per peer, nanosleep
  // back-off) before copying; capping the grid at the SM count bounds that
  // spinning.  Blocks may still co-reside on an SM (nothing reserves one SM per
  // block) and share it with the main stream's persistent chain kernel.
  if (b > num_sms()) b = num_sms();
  return b < 1 ? 1 : (int)b;
}

void launch_pack_p2p(const float* lat, const int32_t* idx, int64_t n, const P2PSelf& self, int npeers,
                     const P2PPeer* peers, cudaStream_t s) {
  k_pack_p2p<<<grid_p2p(n), 256, 0, s>>>(lat, idx, n, self, npeers, peers);
}
void launch_pull_p2p(float* lat, const int32_t* idx, int64_t n, const P2PSelf& self, int npeers,
                     const P2PPeer* peers, cudaStream_t s) {
  k_pull_p2p<<<grid_p2p(n), 256, 0, s>>>(lat, idx, n, self, npeers, peers);
}
void launch_put_publish(const P2PSelf& self, int npeers, const P2PPeer* peers, cudaStream_t s) {
  k_put_publish<<<1, 32, 0, s>>>(self, npeers, peers);
}
void launch_put_unpack(float* lat, const int32_t* idx, const int32_t* slot, int64_t n, const P2PSelf& self,
                       int npeers, const P2PPeer* peers, cudaStream_t s) {
  k_put_unpack<<<grid_p2p(n), 256, 0, s>>>(lat, idx, slot, n, self, npeers, peers);
}

}  // namespace mfp
