/*
 * mfp.h — C ABI of the B200-native distributed Mosaic Flow Predictor (MFP).
 *
 * The library implements ONE thing: the data-parallel hot path of arXiv 2308.14258
 * ("Physics-informed neural PDE solvers at scale", the distributed MF predictor):
 *
 *   iterate  { for each of the 4 subdomain classes (phases):
 *                gather the boundaries of every non-overlapping atomic subdomain of
 *                the class, run ONE batched SDNet forward, scatter the centre-line
 *                predictions back onto the line lattice }
 *              exchange halo strips with the 3x3 stencil of neighbour ranks (once)
 *              every c iterations: global max-norm update test }
 *   final phase: predict every interior point of each atomic subdomain, gather.
 *
 * Paper passages (PAPER.md line numbers, "P:n"):
 *   P:23  (§4.1)  atomic subdomains of one iteration do not overlap -> one batch
 *   P:29  (§4.2)  Cartesian grid of subdomain boundaries with spacing m/2
 *   P:39-40       row-major 2-D processor grid, processor subdomain + halo
 *   P:43  (§4.2)  Algorithm 2: inputs t, eps, g, SDNet, n; predict only centre
 *                 lines; pack overlap boundaries into a contiguous buffer; send
 *   P:44          final phase: predict every grid point, all_gather, average
 *   P:48          relaxed synchronisation: communicate once per iteration,
 *                 immediate updates inside a processor subdomain
 *   P:53-61 (§4.3) alpha-beta cost model
 *   P:239-241 (§3.1) SDNet: 1-D convolutions over g, split layer, GELU MLP
 *   P:261-274 (§3.2, Eq. 5) U = phi(g W1^T (+) X W2^T), broadcasted sum
 *   P:512-519 (§2.1) Dirichlet Laplace BVP (defines the exact subsolver)
 *
 * Readings where the paper is silent are fixed in DESIGN.md §2 (G1..G7 of
 * SURVEY.md §0.3): m = 32 intervals per subdomain side (33 points), perimeter
 * of 4m = 128 values walked counter-clockwise from the lower-left corner
 * (bottom L->R, right B->T, top R->L, left T->B), 2m-3 = 61 centre-line
 * queries per prediction (vertical line bottom->top, then horizontal line
 * left->right without the centre), class order (0,0),(1,0),(0,1),(1,1),
 * distributed convention D1 (a rank computes every subdomain whose centre lies
 * in its CLOSED block; owner values overwrite halo copies once per iteration),
 * convergence delta = max over owned interior line points of |U_k - U_{k-1}|.
 *
 * Conventions for every entry point
 *   - Every call returns mfp_status; 0 == MFP_OK.  Errors other than
 *     MFP_NOT_CONVERGED leave a message readable with mfp_last_error().
 *   - CUDA/NCCL failures are sticky: the context enters MFP_ERR_STATE and every
 *     later call except mfp_destroy/mfp_last_error returns MFP_ERR_STATE.
 *   - Host pointers are read (copied) during the call; the caller keeps them.
 *   - Device buffers (workspace, g_dev, u_dev, gb, out) are caller-owned
 *     (allocated with torch); the context only keeps views into the workspace
 *     and never frees them.  The NCCL communicator is caller-owned as well.
 *   - All fields are fp32, row-major with x fastest: u[y*(nx+1)+x].
 *   - There is no CPU fallback: every numeric step runs in the library's
 *     sm_100a kernels; without a CUDA device calls return MFP_ERR_CUDA.
 */
#ifndef MFP_H
#define MFP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MFP_ABI_VERSION 1u
/* rank argument meaning "this process drives every rank of the processor grid
 * on its one device" (exchange by device copies instead of NCCL). */
#define MFP_ALL_RANKS (-1)
#define MFP_NCCL_UNIQUE_ID_BYTES 128

typedef enum {
  MFP_OK = 0,
  MFP_ERR_INVALID = 1,      /* bad argument / config / length mismatch            */
  MFP_ERR_NOT_TILEABLE = 2, /* nx or ny not a multiple of m, or grid not aligned  */
  MFP_ERR_NONFINITE = 3,    /* NaN/Inf in g, params, or in a prediction           */
  MFP_NOT_CONVERGED = 4,    /* non-fatal: u is written, report filled             */
  MFP_ERR_CUDA = 5,
  MFP_ERR_NCCL = 6,
  MFP_ERR_WORKSPACE = 7,    /* workspace too small or misaligned (256 B)          */
  MFP_ERR_STATE = 8         /* context poisoned by an earlier CUDA/NCCL error     */
} mfp_status;

/* Arithmetic of the SDNet MLP chain: FP32 = SIMT fp32 with exact-erf GELU (the
 * parity twin); BF16 / FP16 = tcgen05 tensor cores with operands rounded to
 * bf16 / fp16 and fp32 accumulation in TMEM (same throughput; fp16 has 8x
 * smaller unit roundoff); FP16X = the accuracy mode of the
 * tensor-core path (d = 128): every activation feeding an MMA is split
 * h = h_hi + h_lo into two fp16 operands and both products are accumulated
 * against the fp16 weights, so only the weights are rounded (
 * with trained weights and gelu = 2 it holds the 3e-3 per-field bar that the
 * single-rounding modes miss). */
enum { MFP_FP32 = 0, MFP_BF16 = 1, MFP_FP16 = 2, MFP_FP16X = 3 };
enum { MFP_SDNET = 0, MFP_EXACT_LAPLACE = 1 };  /* subdomain solver   */
enum { MFP_QUERY_CENTRE = 0, MFP_QUERY_INTERIOR = 1 };

/* Problem + decomposition.  P:39 (row-major processor grid), P:29 (stride m/2). */
typedef struct {
  uint32_t abi;        /* must be MFP_ABI_VERSION                                   */
  int32_t nx, ny;      /* global grid intervals per side; (nx+1)x(ny+1) points      */
  int32_t m;           /* subdomain intervals per side; must be 32 (G1)             */
  int32_t stride;      /* must be m/2 (paper d = 2)                           */
  int32_t grid_rows;   /* Py: processor rows    ((ny/m) % Py == 0)                  */
  int32_t grid_cols;   /* Px: processor columns ((nx/m) % Px == 0)                  */
  int32_t precision;   /* MFP_FP32 | MFP_BF16 | MFP_FP16 | MFP_FP16X                 */
  int32_t subsolver;   /* MFP_SDNET | MFP_EXACT_LAPLACE                              */
  int32_t check_every; /* c >= 1: convergence test every c iterations                */
} mfp_config;

/* SDNet shape (sizes are reading G7).  Supported:
 * n_conv = 2, conv_k = {5,5}, conv_ch = {1,8,1}, d = 128 or 256 (
 * MFP_FP16X: d = 128), 1 <= n_hidden <= 3. */
typedef struct {
  int32_t n_conv;
  int32_t conv_k[4];
  int32_t conv_ch[5];
  int32_t d;
  int32_t n_hidden;
  int32_t gelu;        /* 0: erff-based GELU; 1: fast GELU on the tensor-core paths —
                        * the classic tanh form of x Phi(x), |error of 2 GELU| <= 9.5e-4;
                        * 2: accurate tanh form tanh(x (c0 + t (c1 + t c2))),
                        * t = min(x^2, 16), |error of 2 GELU| <= 5e-5 (DESIGN.md
                        * reading GELU).  The fp32 chain always uses erff.          */
} mfp_sdnet_desc;

typedef struct {
  int32_t iterations;          /* iterations executed                                */
  int32_t converged;           /* 1 if delta <= tol was observed                     */
  float last_delta;            /* last computed delta (max over ranks)               */
  float pad_;
  double predictions;          /* UNIQUE subdomain predictions, (2Kx-1)(2Ky-1)/iter  */
  double predictions_computed; /* including D1's redundant straddlers, all ranks     */
  double ms_total;             /* device time of the solve (events), this rank       */
  double ms_final;             /* device time of the final phase + gather            */
  int64_t halo_bytes_sent;     /* this rank (all ranks for MFP_ALL_RANKS), whole run */
  int32_t halo_msgs_per_iter;  /* messages sent per iteration by this rank (max)     */
  int32_t gpu_launches;        /* kernels launched by the library during the solve   */
} mfp_report;

/* Per-kernel device time, measured with CUDA events on the launching stream. */
typedef struct {
  int32_t iterations;
  int32_t launches_per_iter;
  double ms_per_iter;          /* whole iteration (4 phases + exchange)              */
  double ms_gather_embed;      /* per launch average                                 */
  double ms_chain;             /* per launch average (SDNet chain, incl. scatter)    */
  double ms_exact;             /* per launch average (exact subsolver phase kernel)  */
  double ms_halo;              /* per iteration (pack + exchange + unpack)           */
  double ms_delta;             /* per launch                                         */
  int64_t chain_launches, chain_rows; /* rows = predictions * queries, all launches */
  double chain_ms_total;
  int64_t gather_launches, gather_subdomains;
  double gather_ms_total;
} mfp_profile;

typedef struct mfp_ctx mfp_ctx;

/* Host-only view of a rank's plan (no GPU needed).  P:39-43.  Coordinates are
 * global grid indices.  Owned block: X0 <= x < X1 (x <= nx for the last column),
 * same in y.  Read region (block + m/2 halo, clipped): RX0..RX1 closed. */
typedef struct {
  int32_t rank, ry, rx;
  int32_t X0, X1, Y0, Y1;
  int32_t RX0, RX1, RY0, RY1;
  int64_t phase_count[4];      /* subdomains computed per phase (D1, closed block)   */
  int64_t final_count;         /* owned atomic subdomains (final phase)              */
  int32_t n_peers;
  int32_t peers[8];            /* neighbour ranks in row-major order                 */
  int64_t send_count[8];       /* lattice cells sent to peers[i] per iteration       */
  int64_t recv_count[8];       /* lattice cells received from peers[i]               */
  int64_t lattice_cells;       /* horizontal + vertical line cells held locally      */
  int32_t n_hlines, n_vlines;  /* local line counts (y = RY0 + 16 i, x = RX0 + 16 j)  */
  int32_t hline_len, vline_len;/* RX1-RX0+1, RY1-RY0+1                               */
  int64_t phase0_interior;     /* phase-0 subdomains touching no halo cell: they run  */
                               /* while the previous exchange is in flight           */
} mfp_plan_info;

/* ---- sizing / lifetime ------------------------------------------------------ */

/* Bytes of device workspace mfp_init needs for `rank` (or MFP_ALL_RANKS). */
mfp_status mfp_workspace_size(const mfp_config* cfg, const mfp_sdnet_desc* net,
                              int rank, size_t* bytes);

/* Number of fp32 parameters `params` must hold, in SPEC MFCK declaration order
 * (S:387): for each conv layer l: w_l (cout,cin,k), b_l (cout); W1 (d, 4m*ch_last);
 * W2 (d,2); b1 (d); for each hidden layer: Wh (d,d), bh (d); wo (d); bo (1). */
mfp_status mfp_param_count(const mfp_sdnet_desc* net, int32_t m, size_t* n);

/* Validate, build the plan (N1), carve `workspace`, upload weights (and the
 * exact-solver matrices when subsolver == MFP_EXACT_LAPLACE), precompute the
 * per-query tables Q = X W2^T + b1 (Eq. 5).  `params` may be NULL iff
 * subsolver == MFP_EXACT_LAPLACE.  rank in [0, Py*Px) with a caller-owned
 * ncclComm_t (`nccl_comm`; required for Py*Px > 1, optional — a 1-rank communicator that
 * exercises the collective paths — for Py*Px == 1), or MFP_ALL_RANKS with
 * nccl_comm == NULL.  `stream` is a caller-owned cudaStream_t (NULL = legacy).
 * Errors: INVALID, NOT_TILEABLE, NONFINITE (params), WORKSPACE, CUDA. */
mfp_status mfp_init(const mfp_config* cfg, const mfp_sdnet_desc* net,
                    const float* params, size_t n_params,
                    int rank, void* nccl_comm,
                    void* workspace, size_t ws_bytes,
                    void* stream, mfp_ctx** out);

void mfp_destroy(mfp_ctx* ctx);
const char* mfp_last_error(const mfp_ctx* ctx);  /* never NULL */

/* ---- the hot path ----------------------------------------------------------- */

/* Algorithm 2.  g: HOST, 2(nx+ny) fp32 values walked counter-clockwise
 * from (0,0) (bottom x=0..nx-1, right y=0..ny-1, top x=nx..1, left y=ny..1;
 * reading G6).  g == NULL resumes from the current lattice (no init).
 * max_iters = t >= 1.  tol = eps >= 0.  delta_k (reading G5: max over owned
 * interior line points of |U_k - U_{k-1}|, allreduce-MAX over ranks) is
 * evaluated every check_every iterations and after the last one; the solve
 * stops at the first such k with delta_k <= tol.  tol == 0 runs exactly
 * max_iters iterations (parity mode; delta is still evaluated and reported in
 * rep->last_delta).  u_out: HOST (ny+1)*(nx+1) fp32, required on rank 0
 * (and for MFP_ALL_RANKS), ignored elsewhere; may be NULL to skip the final
 * phase.  rep nullable.  Collective over the communicator.
 * Execution: whole blocks of check_every iterations replay captured CUDA graphs;
 * with tol > 0 on a single-process context (one rank or MFP_ALL_RANKS) the
 * stopping rule itself runs on the device — one graph with a WHILE node repeats
 * the block until delta <= tol, a non-finite prediction or the budget — so a
 * converging solve makes no host round trip per block (same field bit for bit).
 * Returns OK, NOT_CONVERGED (u written), NONFINITE, CUDA, NCCL, STATE. */
mfp_status mfp_solve(mfp_ctx* ctx, const float* g, int32_t max_iters, float tol,
                     float* u_out, mfp_report* rep);

/* Same as mfp_solve with DEVICE g_dev / u_dev (inputs already resident). */
mfp_status mfp_solve_device(mfp_ctx* ctx, const float* g_dev, int32_t max_iters,
                            float tol, float* u_dev, mfp_report* rep);

/* Batched SDNet forward only (P:23 batching; forward_many).
 * gb: DEVICE B x 4m boundary vectors (G1 order); out: DEVICE B x q with
 * q = 61 (MFP_QUERY_CENTRE, G3 order) or 961 (MFP_QUERY_INTERIOR, row-major
 * (i/m, j/m), i,j = 1..31, i fastest).  Uses the context's weights and
 * precision; `stream` NULL = the context stream.  No communication. */
mfp_status mfp_sdnet_batch(mfp_ctx* ctx, const float* gb, int64_t B,
                           int32_t query_set, float* out, void* stream);

/* Standalone "Boundaries IO" of one phase — the unfused form of the
 * solve's gather (fused there into the embed) and scatter (fused into the chain
 * epilogue): mfp_gather_phase -> mfp_sdnet_batch -> mfp_scatter_phase is one
 * phase of Algorithm 2.  `rank`: 0 for single-rank contexts, the rank
 * index for MFP_ALL_RANKS contexts.  Both run asynchronously on the context
 * stream unless a host result is requested.
 *
 * mfp_gather_phase (a1, P:23 / P:43): gb (DEVICE, cap x 4m fp32) receives the
 * perimeter (G1 order) of every subdomain the rank computes in `phase` (0..3,
 * G2 order), read from its current lattice; *B_out = their number (required
 * rows).  ax_out / ay_out (HOST, cap int32 each, both or neither) receive the
 * global lower-left anchors in row order — mfp_plan_anchors' order, except that
 * with R > 1 phase 0 lists its phase0_interior subdomains first.  gb, ax_out and
 * ay_out all NULL = size query.  INVALID if cap < B. */
mfp_status mfp_gather_phase(mfp_ctx* ctx, int32_t rank, int32_t phase, float* gb, int64_t cap,
                            int64_t* B_out, int32_t* ax_out, int32_t* ay_out);
/* mfp_scatter_phase (a6 + a8, "the center lines of one subdomain are the
 * boundary of another"): pred (DEVICE, B x 61 fp32, G3 order, rows in
 * mfp_gather_phase's order; B must equal the phase's count) overwrite the
 * centre-line cells of the rank's lattice (the centre point in both line
 * arrays).  The kernel also reduces the update norm max |new - old| over the
 * written cells (per-block warp-shuffle max, then one reduction kernel); if
 * update_max (HOST, nullable) is given the call waits and stores it, and returns
 * NONFINITE when a prediction is NaN/Inf (the lattice is written regardless). */
mfp_status mfp_scatter_phase(mfp_ctx* ctx, int32_t rank, int32_t phase, const float* pred, int64_t B,
                             float* update_max);

/* Communication-avoiding variant (the paper's open problem
 * P:196 "reducing the communication frequency"): exchange halos after every s-th
 * iteration only (and always after the last), so halo copies are up to s - 1
 * iterations stale; s = 1 (default) is Algorithm 2.  s must divide
 * check_every (CUDA-graph blocks replay one pattern).  Collective in the sense
 * that every rank must use the same s.  Errors: INVALID. */
mfp_status mfp_set_exchange_every(mfp_ctx* ctx, int32_t s);

/* Device-initiated halo transport (the paper names
 * direct GPU-GPU transfers via NVSHMEM as the way past its MPI exchange).
 * communicate_new_boundaries then runs as two kernels and no NCCL call:
 * the pack snapshots the owned send cells into one of two parity buffers of the
 * rank's peer-memory region and publishes an epoch flag; the pull kernel waits
 * for each stencil peer's flag, loads the peer's segment straight from the
 * peer's region (NVLink P2P) into this rank's halo cells and signals
 * "consumed" back.  The convergence allreduce and the final gather stay NCCL.
 *
 * mfp_p2p_export (one process per GPU, R > 1): allocates this rank's region
 *   (cudaMalloc, owned by the context, freed by mfp_destroy) and writes its
 *   64-byte cudaIpcMemHandle_t to handle_out (HOST).  The caller all-gathers the
 *   handles (e.g. torch.distributed over any backend).
 * mfp_p2p_open: handles (HOST) = n_handles = R handles of 64 B in rank order
 *   for one process per GPU (every rank must have exported), or NULL with
 *   n_handles = 0 for MFP_ALL_RANKS (every rank's region on this device, no
 *   IPC).  Switches the context to the peer transport for the rest of its
 *   life; collective (every rank calls it at the same iteration boundary, no
 *   solve in flight).  On any error nothing stays opened (a retry starts
 *   clean).  mfp_destroy waits (<= 30 s) until every stencil peer has consumed
 *   this rank's last exchange before it frees the region.
 * Errors: INVALID (wrong mode, NULL/non-NULL handles, n_handles != R, already
 *   open, exchange in flight), CUDA (allocation, IPC). */
mfp_status mfp_p2p_export(mfp_ctx* ctx, void* handle_out);
mfp_status mfp_p2p_open(mfp_ctx* ctx, const void* handles, int32_t n_handles);

/* NEXT-2, device-initiated halo from the epilogue ("the scatter
 * epilogue puts strips into neighbours' halos"; P:193 NVSHMEM-style direct
 * GPU-GPU transfers).  After mfp_p2p_open, mode MFP_P2P_PUT makes the SDNet
 * chain's epilogue store every owned cell a stencil peer holds as a halo cell
 * straight into that peer's put buffer (peer memory; parity by exchange epoch)
 * as it writes the cell; the iteration's exchange is then one publish kernel
 * per rank (system fence + put-done flag to each peer; waits until every peer
 * has unpacked the previous exchange) and a local unpack on the receiver,
 * overlapped with the interior phase-0 subdomains as before — no pack kernel
 * and no remote reads.  MFP_P2P_PULL restores pack + pull.  Same results as
 * every other transport, bit for bit (the last write of the iteration wins in
 * the put buffer, as the pack would read it).  Collective, at an iteration
 * boundary; resets the region's flags and epochs.
 * Errors: INVALID (p2p not open, exchange in flight, bad mode, PUT with the
 * exact subsolver), CUDA. */
enum { MFP_P2P_PULL = 0, MFP_P2P_PUT = 1 };
mfp_status mfp_p2p_set_mode(mfp_ctx* ctx, int32_t mode);

/* Run ONE phase (class 0..3 in G2 order) on the current lattice of every local
 * rank, without exchange (debug / sampled parity at full size). */
mfp_status mfp_step_phase(mfp_ctx* ctx, int32_t phase);

/* Copy the local line lattice of `rank` (0 for single-rank contexts) to/from
 * HOST buffers: hl[n_hlines][hline_len], vl[n_vlines][vline_len] (plan info). */
mfp_status mfp_export_lines(mfp_ctx* ctx, int32_t rank, float* hl, float* vl);
mfp_status mfp_import_lines(mfp_ctx* ctx, int32_t rank, const float* hl, const float* vl);

/* Run `iters` iterations from the current lattice with CUDA events around each
 * kernel (bench roofline).  Not collective-free: exchanges like mfp_solve. */
mfp_status mfp_profile_iterations(mfp_ctx* ctx, int32_t iters, mfp_profile* out);

/* ---- host-only plan introspection (no GPU) ----------------------------------- */

mfp_status mfp_plan_query(const mfp_config* cfg, int32_t rank, mfp_plan_info* out);
/* Anchors (lower-left corners, global) computed by `rank` in `phase` (0..3) or
 * owned atomic subdomains (phase == 4), sorted by (ay, ax).  cap = array size. */
mfp_status mfp_plan_anchors(const mfp_config* cfg, int32_t rank, int32_t phase,
                            int32_t* ax, int32_t* ay, int64_t cap, int64_t* count);
/* Halo cells exchanged with peers[peer_idx] in canonical order: kind 0 = cell of
 * a horizontal line, 1 = vertical line; (x, y) global.  dir 0 = sent, 1 = recv. */
mfp_status mfp_plan_halo(const mfp_config* cfg, int32_t rank, int32_t peer_idx,
                         int32_t dir, int32_t* kind, int32_t* x, int32_t* y,
                         int64_t cap, int64_t* count);

/* alpha-beta model of §4.3: subdomains per processor (dN)^2/(m^2 P),
 * C_comm = 8 I alpha + (I/beta) 16 N d / sqrt(P), C_comp = c (dN)^2/(m^2 P). */
mfp_status mfp_cost_model(double N, double P, double m, double d, double I,
                          double alpha, double beta, double c,
                          double* subdomains_per_proc, double* c_comm, double* c_comp);

/* ---- NCCL bootstrap (the unique id travels through torch.distributed) -------- */
mfp_status mfp_nccl_get_unique_id(void* id_out /* MFP_NCCL_UNIQUE_ID_BYTES */);
mfp_status mfp_nccl_comm_init(int32_t nranks, const void* id, int32_t rank, void** comm_out);
mfp_status mfp_nccl_comm_destroy(void* comm);

#ifdef __cplusplus
}
#endif
#endif /* MFP_H */
