// plan.cpp — host geometry and decomposition plan (N1), plus the host-only
// plan-introspection entry points of include/mfp.h.
//
// PAPER.md passages: P:29 (subdomain-boundary grid with spacing m/2)
// (classes of non-overlapping atomic subdomains batched together)
// (row-major processor grid, processor subdomain + halo), P:43 (boundaries in the
// overlap region packed into contiguous buffers and sent to the neighbours),
// P:53-61 (cost model).  Readings G1-G6 and D1 are fixed in DESIGN.md §2.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "mfp_internal.h"

namespace mfp {

static int round_up(int v, int a) { return (v + a - 1) / a * a; }

mfp_status validate_config(const mfp_config* c, std::string* err) {
  if (!c) { *err = "cfg is NULL"; return MFP_ERR_INVALID; }
  if (c->abi != MFP_ABI_VERSION) { *err = "abi mismatch"; return MFP_ERR_INVALID; }
  if (c->m != kM) { *err = "m must be 32 (reading G1)"; return MFP_ERR_INVALID; }
  if (c->stride != c->m / 2) { *err = "stride must be m/2 (P:29)"; return MFP_ERR_INVALID; }
  if (c->nx < c->m || c->ny < c->m || c->nx > 32768 || c->ny > 32768) {
    *err = "nx, ny must be in [m, 32768]"; return MFP_ERR_INVALID;
  }
  if (c->nx % c->m || c->ny % c->m) { *err = "domain not tileable by m (S:56)"; return MFP_ERR_NOT_TILEABLE; }
  if (c->grid_rows < 1 || c->grid_cols < 1 || c->grid_rows * c->grid_cols > 4096) {
    *err = "bad processor grid"; return MFP_ERR_INVALID;
  }
  if ((c->nx / c->m) % c->grid_cols || (c->ny / c->m) % c->grid_rows) {
    *err = "processor grid does not divide the atomic-subdomain grid (S:75)";
    return MFP_ERR_NOT_TILEABLE;
  }
  if (c->precision < MFP_FP32 || c->precision > MFP_FP16X) { *err = "bad precision"; return MFP_ERR_INVALID; }
  if (c->subsolver != MFP_SDNET && c->subsolver != MFP_EXACT_LAPLACE) { *err = "bad subsolver"; return MFP_ERR_INVALID; }
  if (c->check_every < 1) { *err = "check_every must be >= 1"; return MFP_ERR_INVALID; }
  return MFP_OK;
}

static int owner(const mfp_config* c, int x, int y) {
  int Lx = c->nx / c->grid_cols, Ly = c->ny / c->grid_rows;
  int rx = std::min(x / Lx, c->grid_cols - 1), ry = std::min(y / Ly, c->grid_rows - 1);
  return ry * c->grid_cols + rx;
}

static void block_of(const mfp_config* c, int r, int* X0, int* X1, int* Y0, int* Y1) {
  int Lx = c->nx / c->grid_cols, Ly = c->ny / c->grid_rows;
  int ry = r / c->grid_cols, rx = r % c->grid_cols;
  *X0 = rx * Lx; *X1 = *X0 + Lx; *Y0 = ry * Ly; *Y1 = *Y0 + Ly;
}

static void read_region(const mfp_config* c, int r, int* RX0, int* RX1, int* RY0, int* RY1) {
  int X0, X1, Y0, Y1;
  block_of(c, r, &X0, &X1, &Y0, &Y1);
  *RX0 = std::max(0, X0 - kH); *RX1 = std::min(c->nx, X1 + kH);
  *RY0 = std::max(0, Y0 - kH); *RY1 = std::min(c->ny, Y1 + kH);
}

static void build_rank(const mfp_config* c, int r, RankPlan* p) {
  const int nx = c->nx, ny = c->ny, Px = c->grid_cols, Py = c->grid_rows;
  p->rank = r; p->ry = r / Px; p->rx = r % Px;
  block_of(c, r, &p->X0, &p->X1, &p->Y0, &p->Y1);
  p->bw = p->X1 - p->X0 + (p->rx == Px - 1 ? 1 : 0);
  p->bh = p->Y1 - p->Y0 + (p->ry == Py - 1 ? 1 : 0);
  LatticeGeom& L = p->lat;
  read_region(c, r, &L.RX0, &L.RX1, &L.RY0, &L.RY1);
  L.nH = (L.RY1 - L.RY0) / kH + 1;
  L.nV = (L.RX1 - L.RX0) / kH + 1;
  L.lenH = L.RX1 - L.RX0 + 1;
  L.lenV = L.RY1 - L.RY0 + 1;
  L.strideH = round_up(L.lenH, 32);
  L.strideV = round_up(L.lenV, 32);
  L.offV = (int64_t)L.nH * L.strideH;
  L.cells = L.offV + (int64_t)L.nV * L.strideV;

  // Phase compute sets (D1): centre (ax+h, ay+h) in the CLOSED block.
  for (int cls = 0; cls < 4; cls++) {
    int cx = cls & 1, cy = (cls >> 1) & 1;
    p->phase_anchor[cls].clear(); p->phase_ax[cls].clear(); p->phase_ay[cls].clear();
    for (int ay = 0; ay + kM <= ny; ay += kH) {
      if ((ay / kH) % 2 != cy) continue;
      int cyy = ay + kH;
      if (cyy < p->Y0 || cyy > p->Y1) continue;
      for (int ax = 0; ax + kM <= nx; ax += kH) {
        if ((ax / kH) % 2 != cx) continue;
        int cxx = ax + kH;
        if (cxx < p->X0 || cxx > p->X1) continue;
        uint32_t a = (uint32_t)((ax - L.RX0) / kH), b = (uint32_t)((ay - L.RY0) / kH);
        p->phase_anchor[cls].push_back(a | (b << 16));
        p->phase_ax[cls].push_back(ax);
        p->phase_ay[cls].push_back(ay);
      }
    }
  }
  // Final phase: owned atomic subdomains.
  p->final_anchor.clear(); p->final_lat_anchor.clear(); p->final_ax.clear(); p->final_ay.clear();
  for (int ay = p->Y0; ay + kM <= p->Y1; ay += kM)
    for (int ax = p->X0; ax + kM <= p->X1; ax += kM) {
      p->final_anchor.push_back((uint32_t)(ax - p->X0) | ((uint32_t)(ay - p->Y0) << 16));
      p->final_lat_anchor.push_back((uint32_t)((ax - L.RX0) / kH) |
                                    ((uint32_t)((ay - L.RY0) / kH) << 16));
      p->final_ax.push_back(ax); p->final_ay.push_back(ay);
    }
  // Convergence segments: owned interior line cells (reading G5).
  p->delta_seg.clear();
  int oxl = std::max(p->X0, 1), oxh = std::min(p->X0 + p->bw - 1, nx - 1);
  int oyl = std::max(p->Y0, 1), oyh = std::min(p->Y0 + p->bh - 1, ny - 1);
  for (int i = 0; i < L.nH; i++) {
    int y = L.RY0 + i * kH;
    if (y < oyl || y > oyh || oxl > oxh) continue;
    int64_t off = (int64_t)i * L.strideH + (oxl - L.RX0);
    p->delta_seg.push_back((off << 20) | (int64_t)(oxh - oxl + 1));
  }
  for (int j = 0; j < L.nV; j++) {
    int x = L.RX0 + j * kH;
    if (x < oxl || x > oxh || oyl > oyh) continue;
    int64_t off = L.offV + (int64_t)j * L.strideV + (oyl - L.RY0);
    p->delta_seg.push_back((off << 20) | (int64_t)(oyh - oyl + 1));
  }
  // Halo exchange with the 3x3 stencil: cells of points owned by
  // the sender that lie in the receiver's read region, canonical order: all
  // horizontal-line cells by (y, x), then all vertical-line cells by (x, y).
  p->peers.clear();
  for (int dy = -1; dy <= 1; dy++)
    for (int dx = -1; dx <= 1; dx++) {
      if (!dx && !dy) continue;
      int sy = p->ry + dy, sx = p->rx + dx;
      if (sy < 0 || sy >= Py || sx < 0 || sx >= Px) continue;
      int s = sy * Px + sx;
      PeerPlan pp;
      pp.rank = s;
      int SX0, SX1, SY0, SY1;
      read_region(c, s, &SX0, &SX1, &SY0, &SY1);
      // send: my owned points inside s's read region
      for (int pass = 0; pass < 2; pass++) {
        // pass 0: send, pass 1: recv (points owned by s inside my read region)
        int src = pass == 0 ? r : s;
        int qX0 = pass == 0 ? SX0 : L.RX0, qX1 = pass == 0 ? SX1 : L.RX1;
        int qY0 = pass == 0 ? SY0 : L.RY0, qY1 = pass == 0 ? SY1 : L.RY1;
        std::vector<int32_t>& idx = pass == 0 ? pp.send_idx : pp.recv_idx;
        std::vector<int32_t>& kk = pass == 0 ? pp.send_kind : pp.recv_kind;
        std::vector<int32_t>& kx = pass == 0 ? pp.send_x : pp.recv_x;
        std::vector<int32_t>& ky = pass == 0 ? pp.send_y : pp.recv_y;
        for (int i = 0; i < L.nH; i++) {
          int y = L.RY0 + i * kH;
          if (y < qY0 || y > qY1) continue;
          for (int x = std::max(L.RX0, qX0); x <= std::min(L.RX1, qX1); x++) {
            if (owner(c, x, y) != src) continue;
            idx.push_back((int32_t)((int64_t)i * L.strideH + (x - L.RX0)));
            kk.push_back(0); kx.push_back(x); ky.push_back(y);
          }
        }
        for (int j = 0; j < L.nV; j++) {
          int x = L.RX0 + j * kH;
          if (x < qX0 || x > qX1) continue;
          for (int y = std::max(L.RY0, qY0); y <= std::min(L.RY1, qY1); y++) {
            if (owner(c, x, y) != src) continue;
            idx.push_back((int32_t)(L.offV + (int64_t)j * L.strideV + (y - L.RY0)));
            kk.push_back(1); kx.push_back(x); ky.push_back(y);
          }
        }
      }
      if (!pp.send_idx.empty() || !pp.recv_idx.empty()) p->peers.push_back(std::move(pp));
    }
  // Overlap split of phase 0 (north_star: halo exchange overlapped with interior
  // subdomain batches): interior = no perimeter cell and no centre-line cell is
  // a received halo cell.  Within a class every order is equivalent.
  {
    std::vector<uint8_t> halo((size_t)L.cells, 0);
    for (auto& pp : p->peers)
      for (int32_t c : pp.recv_idx) halo[(size_t)c] = 1;
    std::vector<uint32_t> inner, outer;
    for (uint32_t pk : p->phase_anchor[0]) {
      const int a = (int)(pk & 0xffffu), b = (int)(pk >> 16);
      const int lx = kH * a, ly = kH * b;
      bool touches = false;
      for (int t = 0; t < kM && !touches; t++) {
        // perimeter (G1): bottom, right, top, left edges
        touches |= halo[(size_t)b * L.strideH + lx + t] || halo[(size_t)(b + 2) * L.strideH + lx + kM - t] ||
                   halo[(size_t)(L.offV + (int64_t)(a + 2) * L.strideV + ly + t)] ||
                   halo[(size_t)(L.offV + (int64_t)a * L.strideV + ly + kM - t)];
        // centre lines (G3)
        if (t >= 1)
          touches |= halo[(size_t)(L.offV + (int64_t)(a + 1) * L.strideV + ly + t)] ||
                     halo[(size_t)(b + 1) * L.strideH + lx + t];
      }
      (touches ? outer : inner).push_back(pk);
    }
    p->n0_interior = (int64_t)inner.size();
    p->phase_anchor[0] = inner;
    p->phase_anchor[0].insert(p->phase_anchor[0].end(), outer.begin(), outer.end());
  }
}

mfp_status build_plan(const mfp_config* cfg, int rank, GlobalPlan* out, std::string* err) {
  mfp_status st = validate_config(cfg, err);
  if (st != MFP_OK) return st;
  int R = cfg->grid_rows * cfg->grid_cols;
  if (rank >= R || rank < MFP_ALL_RANKS) { *err = "rank out of range"; return MFP_ERR_INVALID; }
  out->cfg = *cfg;
  out->R = R;
  out->ranks.clear();
  if (rank == MFP_ALL_RANKS) {
    out->ranks.resize(R);
    for (int r = 0; r < R; r++) build_rank(cfg, r, &out->ranks[r]);
  } else {
    out->ranks.resize(1);
    build_rank(cfg, rank, &out->ranks[0]);
  }
  return MFP_OK;
}

}  // namespace mfp

using namespace mfp;

extern "C" mfp_status mfp_plan_query(const mfp_config* cfg, int32_t rank, mfp_plan_info* o) {
  if (!o || rank < 0) return MFP_ERR_INVALID;
  GlobalPlan gp;
  std::string err;
  mfp_status st = build_plan(cfg, rank, &gp, &err);
  if (st) return st;
  const RankPlan& p = gp.ranks[0];
  memset(o, 0, sizeof(*o));
  o->rank = p.rank; o->ry = p.ry; o->rx = p.rx;
  o->X0 = p.X0; o->X1 = p.X1; o->Y0 = p.Y0; o->Y1 = p.Y1;
  o->RX0 = p.lat.RX0; o->RX1 = p.lat.RX1; o->RY0 = p.lat.RY0; o->RY1 = p.lat.RY1;
  for (int c = 0; c < 4; c++) o->phase_count[c] = (int64_t)p.phase_anchor[c].size();
  o->final_count = (int64_t)p.final_anchor.size();
  o->n_peers = (int32_t)p.peers.size();
  for (size_t i = 0; i < p.peers.size(); i++) {
    o->peers[i] = p.peers[i].rank;
    o->send_count[i] = (int64_t)p.peers[i].send_idx.size();
    o->recv_count[i] = (int64_t)p.peers[i].recv_idx.size();
  }
  o->lattice_cells = (int64_t)p.lat.nH * p.lat.lenH + (int64_t)p.lat.nV * p.lat.lenV;
  o->n_hlines = p.lat.nH; o->n_vlines = p.lat.nV;
  o->hline_len = p.lat.lenH; o->vline_len = p.lat.lenV;
  o->phase0_interior = p.n0_interior;
  return MFP_OK;
}

extern "C" mfp_status mfp_plan_anchors(const mfp_config* cfg, int32_t rank, int32_t phase,
                                       int32_t* ax, int32_t* ay, int64_t cap, int64_t* count) {
  if (rank < 0 || phase < 0 || phase > 4 || !count) return MFP_ERR_INVALID;
  GlobalPlan gp;
  std::string err;
  mfp_status st = build_plan(cfg, rank, &gp, &err);
  if (st) return st;
  const RankPlan& p = gp.ranks[0];
  const std::vector<int32_t>& X = phase < 4 ? p.phase_ax[phase] : p.final_ax;
  const std::vector<int32_t>& Y = phase < 4 ? p.phase_ay[phase] : p.final_ay;
  *count = (int64_t)X.size();
  if (ax && ay) {
    if (cap < (int64_t)X.size()) return MFP_ERR_INVALID;
    std::copy(X.begin(), X.end(), ax);
    std::copy(Y.begin(), Y.end(), ay);
  }
  return MFP_OK;
}

extern "C" mfp_status mfp_plan_halo(const mfp_config* cfg, int32_t rank, int32_t peer_idx,
                                    int32_t dir, int32_t* kind, int32_t* x, int32_t* y,
                                    int64_t cap, int64_t* count) {
  if (rank < 0 || !count || (dir != 0 && dir != 1)) return MFP_ERR_INVALID;
  GlobalPlan gp;
  std::string err;
  mfp_status st = build_plan(cfg, rank, &gp, &err);
  if (st) return st;
  const RankPlan& p = gp.ranks[0];
  if (peer_idx < 0 || peer_idx >= (int)p.peers.size()) return MFP_ERR_INVALID;
  const PeerPlan& pp = p.peers[peer_idx];
  const std::vector<int32_t>& K = dir ? pp.recv_kind : pp.send_kind;
  const std::vector<int32_t>& X = dir ? pp.recv_x : pp.send_x;
  const std::vector<int32_t>& Y = dir ? pp.recv_y : pp.send_y;
  *count = (int64_t)K.size();
  if (kind && x && y) {
    if (cap < (int64_t)K.size()) return MFP_ERR_INVALID;
    std::copy(K.begin(), K.end(), kind);
    std::copy(X.begin(), X.end(), x);
    std::copy(Y.begin(), Y.end(), y);
  }
  return MFP_OK;
}

extern "C" mfp_status mfp_cost_model(double N, double P, double m, double d, double I,
                                     double alpha, double beta, double c,
                                     double* spp, double* c_comm, double* c_comp) {
  if (!(N > 0 && P > 0 && m > 0 && d > 0 && I >= 0 && beta > 0) || !spp || !c_comm || !c_comp)
    return MFP_ERR_INVALID;
  // §4.3
  *spp = (d * N) * (d * N) / (m * m * P);
  *c_comm = 8.0 * I * alpha + (I / beta) * (16.0 * N * d / std::sqrt(P));
  *c_comp = c * (*spp);
  return MFP_OK;
}
