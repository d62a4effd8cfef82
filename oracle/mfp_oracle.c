/*
 * oracle/mfp_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 CPU implementation of the distributed
 * Mosaic Flow Predictor of arXiv 2308.14258.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library.  It
 * shares no code, header, table or constant generator with the CUDA product
 * (paper_2308_14258_b200/); neither side includes or links the other.
 *
 * Every function cites the passage it follows ("P:n" = PAPER.md line n, "S:n" =
 * SPEC.md line n) and the reading it takes where the paper is silent
 * (G1..G7, D1 — listed in DESIGN.md §2).  Arithmetic is double precision,
 * naive loops, in the order the paper states the method; OpenMP only spreads the
 * (mutually disjoint) subdomains of one class over threads, which cannot
 * change any result.
 *
 * Pins (tests/test_oracle_*.py): geometry by brute force and SPEC's worked
 * examples; harmonic-extension matrices against an
 * independent numpy LU and their invariants; the exact-subsolver MFP against
 * scipy DST-I / numpy LU global discrete solutions and the discrete-harmonic
 * closed forms x^2-y^2, xy; the SDNet forward against torch fp64 library ops
 * (conv1d circular, linear, gelu); split == concat (Eq. 5); batched ==
 * sequential; P=1 emulation == plain MFP and P>1 converging to the same
 * global discrete solution (Lions).  The SDNet trajectory at scale with
 * random weights has no paper value: "parity unpinned" beyond those checks.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_MAXLAYERS 8

/* ------------------------------------------------------------------------- */
/* Geometry ("distance between neighboring grid points is m/2";           */
/* readings G1 (perimeter), G2 (classes), G3 (centre-line write set)).          */
/* ------------------------------------------------------------------------- */

/* Perimeter of the subdomain with lower-left corner (ax, ay), m intervals per
 * side, 4m points, counter-clockwise from the lower-left corner (G1): bottom
 * left->right (ax+i, ay), right bottom->top (ax+m, ay+i), top right->left
 * (ax+m-i, ay+m), left top->bottom (ax, ay+m-i), i = 0..m-1.  Each corner once.
 * Generalises SPEC's m=2-interval example. */
int orc_perimeter(int m, int ax, int ay, int *px, int *py) {
  int n = 0;
  for (int i = 0; i < m; i++) { px[n] = ax + i;     py[n] = ay;         n++; }
  for (int i = 0; i < m; i++) { px[n] = ax + m;     py[n] = ay + i;     n++; }
  for (int i = 0; i < m; i++) { px[n] = ax + m - i; py[n] = ay + m;     n++; }
  for (int i = 0; i < m; i++) { px[n] = ax;         py[n] = ay + m - i; n++; }
  return n;
}

/* Centre-line write set, "predicts the values only along the center
 * lines" (G3): vertical line x = ax+m/2, y = ay+k (k = 1..m-1, bottom->top),
 * then horizontal line y = ay+m/2, x = ax+k (k = 1..m-1, k != m/2).
 * Local normalised query coordinates (x/m, y/m) in the subdomain's [0,1]^2
 * frame.  Returns 2m-3. */
int orc_writeset(int m, int ax, int ay, int *px, int *py, double *qx, double *qy) {
  int h = m / 2, n = 0;
  for (int k = 1; k < m; k++) {
    if (px) { px[n] = ax + h; py[n] = ay + k; }
    if (qx) { qx[n] = (double)h / m; qy[n] = (double)k / m; }
    n++;
  }
  for (int k = 1; k < m; k++) {
    if (k == h) continue;
    if (px) { px[n] = ax + k; py[n] = ay + h; }
    if (qx) { qx[n] = (double)k / m; qy[n] = (double)h / m; }
    n++;
  }
  return n;
}

/* Final-phase query set, "predict the values at every grid point within
 * each atomic subdomain": interior points (i, j), i, j = 1..m-1, i fastest. */
int orc_interior_queries(int m, double *qx, double *qy) {
  int n = 0;
  for (int j = 1; j < m; j++)
    for (int i = 1; i < m; i++) {
      qx[n] = (double)i / m; qy[n] = (double)j / m; n++;
    }
  return n;
}

/* Anchors of class cls (0..3 = (0,0),(1,0),(0,1),(1,1), G2 order) on an
 * nx x ny-interval grid, sorted by (ay, ax).  Class = (ax/(m/2) mod 2,
 * ay/(m/2) mod 2), anchors at every multiple of m/2 that fits. */
int orc_anchors(int nx, int ny, int m, int cls, int *ax, int *ay) {
  int h = m / 2, cx = cls & 1, cy = (cls >> 1) & 1, n = 0;
  for (int y = 0; y + m <= ny; y += h) {
    if ((y / h) % 2 != cy) continue;
    for (int x = 0; x + m <= nx; x += h) {
      if ((x / h) % 2 != cx) continue;
      if (ax) { ax[n] = x; ay[n] = y; }
      n++;
    }
  }
  return n;
}

/* ------------------------------------------------------------------------- */
/* SDNet forward, fp64 (Eq. 5; reading G7).            */
/* ------------------------------------------------------------------------- */

/* GELU ([hendrycks2016gelu]): x * Phi(x) with the exact error function. */
static double gelu(double x) { return 0.5 * x * (1.0 + erf(x / sqrt(2.0))); }

typedef struct {
  int n_conv, conv_k[ORC_MAXLAYERS], conv_ch[ORC_MAXLAYERS + 1];
  int d, n_hidden, nb; /* nb = 4m boundary length */
} orc_net;

/* Parameter offsets in SPEC MFCK declaration order: per conv layer
 * w (cout,cin,k), b (cout); W1 (d, ch_last*nb); W2 (d,2); b1 (d);
 * per hidden layer Wh (d,d), bh (d); wo (d); bo (1). */
typedef struct {
  size_t cw[ORC_MAXLAYERS], cb[ORC_MAXLAYERS], W1, W2, b1, Wh[ORC_MAXLAYERS],
      bh[ORC_MAXLAYERS], wo, bo, total;
} orc_offsets;

static orc_offsets offsets_of(const orc_net *n) {
  orc_offsets o;
  size_t p = 0;
  for (int l = 0; l < n->n_conv; l++) {
    o.cw[l] = p; p += (size_t)n->conv_ch[l + 1] * n->conv_ch[l] * n->conv_k[l];
    o.cb[l] = p; p += (size_t)n->conv_ch[l + 1];
  }
  o.W1 = p; p += (size_t)n->d * n->conv_ch[n->n_conv] * n->nb;
  o.W2 = p; p += (size_t)n->d * 2;
  o.b1 = p; p += (size_t)n->d;
  for (int l = 0; l < n->n_hidden; l++) {
    o.Wh[l] = p; p += (size_t)n->d * n->d;
    o.bh[l] = p; p += (size_t)n->d;
  }
  o.wo = p; p += (size_t)n->d;
  o.bo = p; p += 1;
  o.total = p;
  return o;
}

size_t orc_param_count(int n_conv, const int *conv_k, const int *conv_ch, int d,
                       int n_hidden, int m) {
  orc_net n;
  n.n_conv = n_conv; n.d = d; n.n_hidden = n_hidden; n.nb = 4 * m;
  for (int l = 0; l < n_conv; l++) n.conv_k[l] = conv_k[l];
  for (int l = 0; l <= n_conv; l++) n.conv_ch[l] = conv_ch[l];
  return offsets_of(&n).total;
}

/* Boundary embedding ("apply 1D convolutions to the input boundary
 * conditions to create a high-dimensional embedding"): conv1d layers with
 * circular padding (k-1)/2 (the perimeter is a closed loop), GELU
 * after every conv layer (G7), flattened channel-major, then the boundary half
 * of the split layer z = W1 e + b1 (Eq. 5: g W1^T, computed once per boundary,
 * P:273).  PyTorch conv1d convention (cross-correlation):
 *   out[o][i] = b[o] + sum_c sum_t w[o][c][t] * in[c][(i + t - pad) mod nb]. */
static void embed(const orc_net *n, const orc_offsets *o, const double *P,
                  const double *g, double *z, double *buf0, double *buf1) {
  int nb = n->nb;
  double *in = buf0, *out = buf1;
  memcpy(in, g, sizeof(double) * nb);
  for (int l = 0; l < n->n_conv; l++) {
    int cin = n->conv_ch[l], cout = n->conv_ch[l + 1], k = n->conv_k[l], pad = (k - 1) / 2;
    const double *w = P + o->cw[l], *b = P + o->cb[l];
    for (int oc = 0; oc < cout; oc++)
      for (int i = 0; i < nb; i++) {
        double s = b[oc];
        for (int c = 0; c < cin; c++)
          for (int t = 0; t < k; t++) {
            int j = ((i + t - pad) % nb + nb) % nb;
            s += w[((size_t)oc * cin + c) * k + t] * in[(size_t)c * nb + j];
          }
        out[(size_t)oc * nb + i] = gelu(s);
      }
    double *tmp = in; in = out; out = tmp;
  }
  int ne = n->conv_ch[n->n_conv] * nb;
  const double *W1 = P + o->W1, *b1 = P + o->b1;
  for (int r = 0; r < n->d; r++) {
    double s = 0.0;
    for (int c = 0; c < ne; c++) s += W1[(size_t)r * ne + c] * in[c];
    z[r] = s + b1[r];
  }
}

/* One query of the MLP ("a stack of linear layers, each followed by a
 * nonlinear activation function"; Eq. 5 first layer U = phi(gW1^T (+) XW2^T)):
 *   h = GELU(z + W2 x);  h = GELU(Wh_l h + bh_l) for each hidden l;  y = wo.h + bo. */
static double mlp_query(const orc_net *n, const orc_offsets *o, const double *P,
                        const double *z, double qx, double qy, double *h, double *h2) {
  int d = n->d;
  const double *W2 = P + o->W2;
  for (int r = 0; r < d; r++) h[r] = gelu(z[r] + (W2[2 * r] * qx + W2[2 * r + 1] * qy));
  for (int l = 0; l < n->n_hidden; l++) {
    const double *W = P + o->Wh[l], *b = P + o->bh[l];
    for (int r = 0; r < d; r++) {
      double s = 0.0;
      for (int c = 0; c < d; c++) s += W[(size_t)r * d + c] * h[c];
      h2[r] = gelu(s + b[r]);
    }
    memcpy(h, h2, sizeof(double) * d);
  }
  const double *wo = P + o->wo;
  double y = 0.0;
  for (int c = 0; c < d; c++) y += wo[c] * h[c];
  return y + P[o->bo];
}

typedef struct {
  orc_net net;
  orc_offsets off;
  const double *P;
} orc_sdnet;

static void sdnet_predict(const orc_sdnet *s, const double *g, int q, const double *qx,
                          const double *qy, double *out) {
  int nb = s->net.nb, d = s->net.d, cmax = 1;
  for (int l = 0; l <= s->net.n_conv; l++)
    if (s->net.conv_ch[l] > cmax) cmax = s->net.conv_ch[l];
  double *b0 = malloc(sizeof(double) * (size_t)cmax * nb);
  double *b1 = malloc(sizeof(double) * (size_t)cmax * nb);
  double *z = malloc(sizeof(double) * d), *h = malloc(sizeof(double) * d),
         *h2 = malloc(sizeof(double) * d);
  embed(&s->net, &s->off, s->P, g, z, b0, b1);
  for (int p = 0; p < q; p++) out[p] = mlp_query(&s->net, &s->off, s->P, z, qx[p], qy[p], h, h2);
  free(b0); free(b1); free(z); free(h); free(h2);
}

static orc_sdnet make_sdnet(int n_conv, const int *conv_k, const int *conv_ch, int d,
                            int n_hidden, int m, const double *P) {
  orc_sdnet s;
  s.net.n_conv = n_conv; s.net.d = d; s.net.n_hidden = n_hidden; s.net.nb = 4 * m;
  for (int l = 0; l < n_conv; l++) s.net.conv_k[l] = conv_k[l];
  for (int l = 0; l <= n_conv; l++) s.net.conv_ch[l] = conv_ch[l];
  s.off = offsets_of(&s.net);
  s.P = P;
  return s;
}

/* Batched SDNet forward (SPEC forward_many S:350): B boundaries x q
 * queries, out[b*q + p]. */
void orc_sdnet_forward(int n_conv, const int *conv_k, const int *conv_ch, int d, int n_hidden,
                       int m, const double *P, int64_t B, const double *g, int q,
                       const double *qx, const double *qy, double *out) {
  orc_sdnet s = make_sdnet(n_conv, conv_k, conv_ch, d, n_hidden, m, P);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t b = 0; b < B; b++)
    sdnet_predict(&s, g + (size_t)b * 4 * m, q, qx, qy, out + (size_t)b * q);
}

/* Input-concat first layer (Eq. 3): U = phi(I W^T), I = [G X],
 * W = [W1 W2] — kept only to check Eq. 5's algebraic identity. embed e given. */
void orc_first_layer_concat(int d, int ne, const double *W1, const double *W2, const double *b1,
                            const double *e, int q, const double *qx, const double *qy,
                            double *U) {
  for (int p = 0; p < q; p++)
    for (int r = 0; r < d; r++) {
      double s = 0.0;
      for (int c = 0; c < ne; c++) s += e[c] * W1[(size_t)r * ne + c]; /* row of I: [g, x] */
      s += qx[p] * W2[2 * r] + qy[p] * W2[2 * r + 1];
      U[(size_t)p * d + r] = gelu(s + b1[r]);
    }
}

/* Input-split first layer (Eq. 5): U = phi(g W1^T (+) X W2^T). */
void orc_first_layer_split(int d, int ne, const double *W1, const double *W2, const double *b1,
                           const double *e, int q, const double *qx, const double *qy,
                           double *U) {
  double *gw = malloc(sizeof(double) * d);
  for (int r = 0; r < d; r++) {
    double s = 0.0;
    for (int c = 0; c < ne; c++) s += e[c] * W1[(size_t)r * ne + c];
    gw[r] = s + b1[r];
  }
  for (int p = 0; p < q; p++)
    for (int r = 0; r < d; r++)
      U[(size_t)p * d + r] = gelu(gw[r] + (qx[p] * W2[2 * r] + qy[p] * W2[2 * r + 1]));
  free(gw);
}

/* ------------------------------------------------------------------------- */
/* Exact discrete-Laplace subsolver (the ASM local solve of §2.3;   */
/* A1: 5-point stencil).  H[q][k] = value at query q of the discrete     */
/* harmonic function on the (m+1)^2 patch whose boundary is unit vector e_k.   */
/* ------------------------------------------------------------------------- */

/* Dense LU with partial pivoting, A (n x n, row-major) overwritten, perm out. */
static int lu_factor(int n, double *A, int *perm) {
  for (int i = 0; i < n; i++) perm[i] = i;
  for (int k = 0; k < n; k++) {
    int piv = k;
    double best = fabs(A[(size_t)k * n + k]);
    for (int i = k + 1; i < n; i++)
      if (fabs(A[(size_t)i * n + k]) > best) { best = fabs(A[(size_t)i * n + k]); piv = i; }
    if (best == 0.0) return -1;
    if (piv != k) {
      for (int j = 0; j < n; j++) {
        double t = A[(size_t)k * n + j]; A[(size_t)k * n + j] = A[(size_t)piv * n + j];
        A[(size_t)piv * n + j] = t;
      }
      int t = perm[k]; perm[k] = perm[piv]; perm[piv] = t;
    }
    for (int i = k + 1; i < n; i++) {
      double f = A[(size_t)i * n + k] / A[(size_t)k * n + k];
      A[(size_t)i * n + k] = f;
      if (f != 0.0)
        for (int j = k + 1; j < n; j++) A[(size_t)i * n + j] -= f * A[(size_t)k * n + j];
    }
  }
  return 0;
}

static void lu_solve(int n, const double *LU, const int *perm, const double *b, double *x) {
  double *y = malloc(sizeof(double) * n);
  for (int i = 0; i < n; i++) {
    double s = b[perm[i]];
    for (int j = 0; j < i; j++) s -= LU[(size_t)i * n + j] * y[j];
    y[i] = s;
  }
  for (int i = n - 1; i >= 0; i--) {
    double s = y[i];
    for (int j = i + 1; j < n; j++) s -= LU[(size_t)i * n + j] * x[j];
    x[i] = s / LU[(size_t)i * n + i];
  }
  free(y);
}

/* H (q x 4m) for query_set 0 (G3 centre lines, q = 2m-3) or 1 (all interior,
 * q = (m-1)^2).  Interior unknowns u(i,j), i,j = 1..m-1; equations
 * 4u(i,j) - u(i-1,j) - u(i+1,j) - u(i,j-1) - u(i,j+1) = 0 with boundary terms
 * moved to the right-hand side.  Returns q, or -1 on failure. */
int orc_harmonic_matrix(int m, int query_set, double *H) {
  int ni = m - 1, n = ni * ni, nb = 4 * m;
  double *A = calloc((size_t)n * n, sizeof(double));
  int *perm = malloc(sizeof(int) * n);
  int *bx = malloc(sizeof(int) * nb), *by = malloc(sizeof(int) * nb);
  orc_perimeter(m, 0, 0, bx, by);
  /* boundary index of local point (x, y), or -1 */
  int *bidx = malloc(sizeof(int) * (m + 1) * (m + 1));
  for (int i = 0; i < (m + 1) * (m + 1); i++) bidx[i] = -1;
  for (int k = 0; k < nb; k++) bidx[by[k] * (m + 1) + bx[k]] = k;
  for (int j = 1; j < m; j++)
    for (int i = 1; i < m; i++) {
      int r = (j - 1) * ni + (i - 1);
      A[(size_t)r * n + r] = 4.0;
      int nbr[4][2] = {{i - 1, j}, {i + 1, j}, {i, j - 1}, {i, j + 1}};
      for (int t = 0; t < 4; t++) {
        int x = nbr[t][0], y = nbr[t][1];
        if (x >= 1 && x <= m - 1 && y >= 1 && y <= m - 1)
          A[(size_t)r * n + (y - 1) * ni + (x - 1)] = -1.0;
      }
    }
  if (lu_factor(n, A, perm) != 0) return -1;
  int q;
  int *qi, *qj;
  if (query_set == 0) {
    q = 2 * m - 3;
    qi = malloc(sizeof(int) * q); qj = malloc(sizeof(int) * q);
    orc_writeset(m, 0, 0, qi, qj, NULL, NULL);
  } else {
    q = n;
    qi = malloc(sizeof(int) * q); qj = malloc(sizeof(int) * q);
    int c = 0;
    for (int j = 1; j < m; j++)
      for (int i = 1; i < m; i++) { qi[c] = i; qj[c] = j; c++; }
  }
  double *rhs = malloc(sizeof(double) * n), *sol = malloc(sizeof(double) * n);
  for (int k = 0; k < nb; k++) {
    /* right-hand side of e_k: each interior equation adjacent to boundary
     * point k gets +1 (corners are adjacent to no interior point). */
    for (int r = 0; r < n; r++) rhs[r] = 0.0;
    for (int j = 1; j < m; j++)
      for (int i = 1; i < m; i++) {
        int nbr[4][2] = {{i - 1, j}, {i + 1, j}, {i, j - 1}, {i, j + 1}};
        for (int t = 0; t < 4; t++)
          if (bidx[nbr[t][1] * (m + 1) + nbr[t][0]] == k) rhs[(j - 1) * ni + (i - 1)] += 1.0;
      }
    lu_solve(n, A, perm, rhs, sol);
    for (int p = 0; p < q; p++) H[(size_t)p * nb + k] = sol[(qj[p] - 1) * ni + (qi[p] - 1)];
  }
  free(A); free(perm); free(bx); free(by); free(bidx); free(qi); free(qj); free(rhs); free(sol);
  return q;
}

/* ------------------------------------------------------------------------- */
/* Distributed MFP, Algorithm 2 with relaxed synchronisation, */
/* emulating a Py x Px row-major processor grid in one process under    */
/* convention D1: owner of (x,y) = (min(y/Ly,Py-1),             */
/* min(x/Lx,Px-1)); a rank computes every subdomain whose centre lies in its   */
/* CLOSED block [X0,X1]x[Y0,Y1]; each rank keeps its own copy of the field;   */
/* after the 4 phases owners' values overwrite every halo copy (one exchange   */
/* per iteration); delta_k = max over owned interior line points |U_k-U_k-1|.  */
/* ------------------------------------------------------------------------- */

typedef struct {
  int nx, ny, m, Py, Px;
  int subsolver;   /* 0 = SDNet, 1 = exact discrete Laplace                       */
  int check_every; /* c                                                           */
  int sequential;  /* 1: baseline MFP, one subdomain at a time (A4)         */
  int n_conv, conv_k[ORC_MAXLAYERS], conv_ch[ORC_MAXLAYERS + 1], d, n_hidden;
  int exchange_every; /* s: exchange after every s-th iteration and the last one
                       * (communication-avoiding variant); 1 = Algorithm 2 */
} orc_cfg;

typedef struct {
  const orc_cfg *c;
  orc_sdnet net;
  double *Hc, *Hf;      /* exact subsolver matrices                              */
  double *qxc, *qyc, *qxf, *qyf;
  int qc, qf;
} solver_t;

static void subsolve(const solver_t *s, int final, const double *g, double *out) {
  int nb = 4 * s->c->m;
  if (s->c->subsolver == 1) {
    const double *H = final ? s->Hf : s->Hc;
    int q = final ? s->qf : s->qc;
    for (int p = 0; p < q; p++) {
      double acc = 0.0;
      for (int k = 0; k < nb; k++) acc += H[(size_t)p * nb + k] * g[k];
      out[p] = acc;
    }
  } else {
    if (final) sdnet_predict(&s->net, g, s->qf, s->qxf, s->qyf, out);
    else sdnet_predict(&s->net, g, s->qc, s->qxc, s->qyc, out);
  }
}

static int owner_of(const orc_cfg *c, int x, int y) {
  int Lx = c->nx / c->Px, Ly = c->ny / c->Py;
  int rx = x / Lx, ry = y / Ly;
  if (rx > c->Px - 1) rx = c->Px - 1;
  if (ry > c->Py - 1) ry = c->Py - 1;
  return ry * c->Px + rx;
}

static int is_line_point(int m, int x, int y) { return (x % (m / 2)) == 0 || (y % (m / 2)) == 0; }

/* g (2(nx+ny), reading G6): bottom x=0..nx-1 at y=0, right y=0..ny-1 at x=nx,
 * top x=nx..1 at y=ny, left y=ny..1 at x=0. */
static void write_global_boundary(const orc_cfg *c, const double *g, double *U) {
  int nx = c->nx, ny = c->ny, W = nx + 1, k = 0;
  for (int x = 0; x < nx; x++) U[0 * W + x] = g[k++];
  for (int y = 0; y < ny; y++) U[(size_t)y * W + nx] = g[k++];
  for (int x = nx; x > 0; x--) U[(size_t)ny * W + x] = g[k++];
  for (int y = ny; y > 0; y--) U[(size_t)y * W + 0] = g[k++];
}

/* Run the MFP.  params: SDNet parameters (MFCK order) when subsolver == 0.
 * g: global boundary.  t: max iterations; tol: eps (0 => exactly t).
 * Outputs (nullable): lines_out (nx+1)(ny+1) owner view of every point after
 * the last iteration (line points meaningful, g on the boundary); u_out final
 * field; delta_log[t]: delta_k of every iteration.  *iters_out.
 * Returns 0, or -1 on allocation/solver failure. */
int orc_mfp_run(const orc_cfg *cfg, const double *params, const double *g, int t, double tol,
                double *lines_out, double *u_out, double *delta_log, int *iters_out) {
  const orc_cfg *c = cfg;
  int nx = c->nx, ny = c->ny, m = c->m, h = m / 2, W = nx + 1, H_ = ny + 1;
  int R = c->Py * c->Px, nb = 4 * m;
  size_t npts = (size_t)W * H_;
  solver_t s;
  memset(&s, 0, sizeof(s));
  s.c = c;
  s.qc = 2 * m - 3;
  s.qf = (m - 1) * (m - 1);
  s.qxc = malloc(sizeof(double) * s.qc); s.qyc = malloc(sizeof(double) * s.qc);
  s.qxf = malloc(sizeof(double) * s.qf); s.qyf = malloc(sizeof(double) * s.qf);
  orc_writeset(m, 0, 0, NULL, NULL, s.qxc, s.qyc);
  orc_interior_queries(m, s.qxf, s.qyf);
  if (c->subsolver == 1) {
    s.Hc = malloc(sizeof(double) * s.qc * nb);
    s.Hf = malloc(sizeof(double) * (size_t)s.qf * nb);
    if (orc_harmonic_matrix(m, 0, s.Hc) < 0 || orc_harmonic_matrix(m, 1, s.Hf) < 0) return -1;
  } else {
    s.net = make_sdnet(c->n_conv, c->conv_k, c->conv_ch, c->d, c->n_hidden, m, params);
  }
  /* per-rank copies of the field (only line points and ∂Ω are ever touched) */
  double **U = malloc(sizeof(double *) * R), **Uprev = malloc(sizeof(double *) * R);
  for (int r = 0; r < R; r++) {
    U[r] = calloc(npts, sizeof(double));
    Uprev[r] = calloc(npts, sizeof(double));
    write_global_boundary(c, g, U[r]);  /* init_state: interior 0, ∂Ω = g */
  }
  int Lx = nx / c->Px, Ly = ny / c->Py;
  /* class anchor lists */
  int *cax[4], *cay[4], cn[4];
  for (int cl = 0; cl < 4; cl++) {
    cn[cl] = orc_anchors(nx, ny, m, cl, NULL, NULL);
    cax[cl] = malloc(sizeof(int) * (cn[cl] + 1)); cay[cl] = malloc(sizeof(int) * (cn[cl] + 1));
    orc_anchors(nx, ny, m, cl, cax[cl], cay[cl]);
  }
  int *wpx = malloc(sizeof(int) * s.qc), *wpy = malloc(sizeof(int) * s.qc);
  int *ppx = malloc(sizeof(int) * nb), *ppy = malloc(sizeof(int) * nb);
  int maxn = 0;
  for (int cl = 0; cl < 4; cl++) if (cn[cl] > maxn) maxn = cn[cl];
  double *gb = malloc(sizeof(double) * (size_t)(maxn + 1) * nb);
  double *yb = malloc(sizeof(double) * (size_t)(maxn + 1) * s.qc);
  int it = 0;
  for (it = 1; it <= t; it++) {
    for (int r = 0; r < R; r++) memcpy(Uprev[r], U[r], sizeof(double) * npts);
    for (int cl = 0; cl < 4; cl++) {          /* the 4 phases of one iteration (G2) */
      for (int r = 0; r < R; r++) {
        int ry = r / c->Px, rx = r % c->Px;
        int X0 = rx * Lx, X1 = X0 + Lx, Y0 = ry * Ly, Y1 = Y0 + Ly;
        /* compute set of rank r in this class: centre in the closed block (D1) */
        int *sel = malloc(sizeof(int) * (cn[cl] + 1)), ns = 0;
        for (int i = 0; i < cn[cl]; i++) {
          int cxp = cax[cl][i] + h, cyp = cay[cl][i] + h;
          if (cxp >= X0 && cxp <= X1 && cyp >= Y0 && cyp <= Y1) sel[ns++] = i;
        }
        double *Ur = U[r];
        if (c->sequential) {
          /* baseline MFP: each prediction sees all earlier updates */
          for (int k = 0; k < ns; k++) {
            int ax = cax[cl][sel[k]], ay = cay[cl][sel[k]];
            double gl[4 * 64 + 8], yl[2 * 64];
            int ppx_l[4 * 64 + 8], ppy_l[4 * 64 + 8], wx[2 * 64], wy[2 * 64];
            orc_perimeter(m, ax, ay, ppx_l, ppy_l);
            for (int j = 0; j < nb; j++) gl[j] = Ur[(size_t)ppy_l[j] * W + ppx_l[j]];
            subsolve(&s, 0, gl, yl);
            orc_writeset(m, ax, ay, wx, wy, NULL, NULL);
            for (int p = 0; p < s.qc; p++) Ur[(size_t)wy[p] * W + wx[p]] = yl[p];
          }
        } else {
          /* batched (§4.1): gather the whole class, one forward, scatter */
#pragma omp parallel for schedule(dynamic, 4)
          for (int k = 0; k < ns; k++) {
            int lx[4 * 64 + 8], ly[4 * 64 + 8];
            orc_perimeter(m, cax[cl][sel[k]], cay[cl][sel[k]], lx, ly);
            for (int j = 0; j < nb; j++) gb[(size_t)k * nb + j] = Ur[(size_t)ly[j] * W + lx[j]];
          }
#pragma omp parallel for schedule(dynamic, 1)
          for (int k = 0; k < ns; k++) subsolve(&s, 0, gb + (size_t)k * nb, yb + (size_t)k * s.qc);
#pragma omp parallel for schedule(dynamic, 4)
          for (int k = 0; k < ns; k++) {
            int wx[2 * 64], wy[2 * 64];
            orc_writeset(m, cax[cl][sel[k]], cay[cl][sel[k]], wx, wy, NULL, NULL);
            for (int p = 0; p < s.qc; p++) Ur[(size_t)wy[p] * W + wx[p]] = yb[(size_t)k * s.qc + p];
          }
        }
        free(sel);
      }
    }
    /* communicate_new_boundaries: owners overwrite every halo copy of
     * a line point, once per iteration — or, in the communication-
     * avoiding variant, after every s-th iteration and the last. */
    const int s_ex = c->exchange_every > 1 ? c->exchange_every : 1;
    if (R > 1 && (it % s_ex == 0 || it == t)) {
      for (int r = 0; r < R; r++) {
        int ry = r / c->Px, rx = r % c->Px;
        int X0 = rx * Lx, X1 = X0 + Lx, Y0 = ry * Ly, Y1 = Y0 + Ly;
        int RX0 = X0 - h < 0 ? 0 : X0 - h, RX1 = X1 + h > nx ? nx : X1 + h;
        int RY0 = Y0 - h < 0 ? 0 : Y0 - h, RY1 = Y1 + h > ny ? ny : Y1 + h;
        for (int y = RY0; y <= RY1; y++)
          for (int x = RX0; x <= RX1; x++) {
            if (!is_line_point(m, x, y)) continue;
            int o = owner_of(c, x, y);
            if (o != r) U[r][(size_t)y * W + x] = U[o][(size_t)y * W + x];
          }
      }
    }
    /* convergence (reading G5): max over owned interior line points */
    double delta = 0.0;
    for (int y = 1; y < ny; y++)
      for (int x = 1; x < nx; x++) {
        if (!is_line_point(m, x, y)) continue;
        int o = owner_of(c, x, y);
        double dd = fabs(U[o][(size_t)y * W + x] - Uprev[o][(size_t)y * W + x]);
        if (dd > delta || dd != dd) delta = dd;
      }
    if (delta_log) delta_log[it - 1] = delta;
    if (tol > 0.0 && it % c->check_every == 0 && delta <= tol) break;
  }
  if (it > t) it = t;
  if (iters_out) *iters_out = it;
  if (lines_out) {
    for (int y = 0; y <= ny; y++)
      for (int x = 0; x <= nx; x++) {
        int o = owner_of(c, x, y);
        lines_out[(size_t)y * W + x] = U[o][(size_t)y * W + x];
      }
  }
  if (u_out) {
    /* final phase: every interior point of each atomic subdomain from
     * one SDNet evaluation on its most recent boundary, computed by the rank
     * owning it (its interior lies in one block, blocks align to m); the
     * atomic-subdomain boundary lines (x or y multiple of m) keep the owner's
     * line values; ∂Ω = g.  Every point has exactly one prediction, so the
     * overlap "average of the predictions" is over one value (D1). */
    for (int y = 0; y <= ny; y++)
      for (int x = 0; x <= nx; x++) {
        int o = owner_of(c, x, y);
        u_out[(size_t)y * W + x] = U[o][(size_t)y * W + x];
      }
    int na = orc_anchors(nx, ny, m, 0, NULL, NULL);
    int *fax = malloc(sizeof(int) * na), *fay = malloc(sizeof(int) * na);
    orc_anchors(nx, ny, m, 0, fax, fay);
#pragma omp parallel for schedule(dynamic, 1)
    for (int k = 0; k < na; k++) {
      int ax = fax[k], ay = fay[k];
      int o = owner_of(c, ax + 1, ay + 1);
      int lx[4 * 64 + 8], ly[4 * 64 + 8];
      double gl[4 * 64 + 8];
      double *yl = malloc(sizeof(double) * s.qf);
      orc_perimeter(m, ax, ay, lx, ly);
      for (int j = 0; j < nb; j++) gl[j] = U[o][(size_t)ly[j] * W + lx[j]];
      subsolve(&s, 1, gl, yl);
      for (int jj = 1; jj < m; jj++)
        for (int ii = 1; ii < m; ii++)
          u_out[(size_t)(ay + jj) * W + (ax + ii)] = yl[(jj - 1) * (m - 1) + (ii - 1)];
      free(yl);
    }
    free(fax); free(fay);
  }
  for (int r = 0; r < R; r++) { free(U[r]); free(Uprev[r]); }
  free(U); free(Uprev);
  for (int cl = 0; cl < 4; cl++) { free(cax[cl]); free(cay[cl]); }
  free(wpx); free(wpy); free(ppx); free(ppy); free(gb); free(yb);
  free(s.qxc); free(s.qyc); free(s.qxf); free(s.qyf);
  free(s.Hc); free(s.Hf);
  return 0;
}

/* Predict n subdomains (anchors ax, ay) of a given global field U (one phase
 * worth of predictions without writing back) — for sampled parity checks at
 * full size.  query_set 0: centre lines (2m-3 values), 1: interior. */
int orc_predict_from_field(const orc_cfg *cfg, const double *params, const double *U, int64_t n,
                           const int *ax, const int *ay, int query_set, double *out) {
  const orc_cfg *c = cfg;
  int m = c->m, nb = 4 * m, W = c->nx + 1;
  int qc = 2 * m - 3, qf = (m - 1) * (m - 1);
  int q = query_set ? qf : qc;
  double *qx = malloc(sizeof(double) * qf), *qy = malloc(sizeof(double) * qf);
  if (query_set) orc_interior_queries(m, qx, qy);
  else orc_writeset(m, 0, 0, NULL, NULL, qx, qy);
  double *H = NULL;
  orc_sdnet net;
  if (c->subsolver == 1) {
    H = malloc(sizeof(double) * (size_t)q * nb);
    if (orc_harmonic_matrix(m, query_set, H) < 0) return -1;
  } else {
    net = make_sdnet(c->n_conv, c->conv_k, c->conv_ch, c->d, c->n_hidden, m, params);
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t k = 0; k < n; k++) {
    int lx[4 * 64 + 8], ly[4 * 64 + 8];
    double gl[4 * 64 + 8];
    orc_perimeter(m, ax[k], ay[k], lx, ly);
    for (int j = 0; j < nb; j++) gl[j] = U[(size_t)ly[j] * W + lx[j]];
    double *o = out + (size_t)k * q;
    if (H) {
      for (int p = 0; p < q; p++) {
        double acc = 0.0;
        for (int j = 0; j < nb; j++) acc += H[(size_t)p * nb + j] * gl[j];
        o[p] = acc;
      }
    } else {
      sdnet_predict(&net, gl, q, qx, qy, o);
    }
  }
  free(qx); free(qy); free(H);
  return 0;
}

/* alpha-beta cost model, §4.3 written out:
 * subdomains per processor (dN)^2/(m^2 P); C_comm = 8 I alpha + (I/beta)(16 N d/sqrt(P));
 * C_comp = c (dN)^2/(m^2 P). */
void orc_cost_model(double N, double P, double m, double d, double I, double alpha, double beta,
                    double c, double *spp, double *ccomm, double *ccomp) {
  *spp = (d * N) * (d * N) / (m * m * P);
  *ccomm = 8.0 * I * alpha + (I / beta) * (16.0 * N * d / sqrt(P));
  *ccomp = c * (*spp);
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
