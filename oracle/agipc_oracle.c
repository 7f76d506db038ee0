/*
 * AGIPC CPU ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously correct single-threaded C99 implementation of what
 * the per-Newton-step coarsening path of AGIPC (arXiv 2605.04773) computes.
 * It exists only to check the CUDA library.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / `--impl reference` leg may load or execute it.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2605_04773_b200/csrc, include/agipc.h); neither includes the other.
 *
 * Citations: "P:n" = line n of the paper text (PAPER.md; supplement = P:1-574,
 * main paper = P:574-1164).  Readings of ambiguous passages are the ones listed
 * in DESIGN.md ("Readings of the paper"), tagged here as [Rk].
 *
 * Build: gcc -O2 -std=c99 -ffp-contract=off -fPIC -shared (no FMA contraction:
 * the tag step must reproduce one fixed operation order, [R12]).
 *
 * Parity pins (tests/test_oracle_*.py): every function below is pinned against
 * the paper's worked examples, closed forms, invariants or brute force; none is
 * "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ERANGE 2
#define ORC_ENOMEM 3
#define ORC_EDEGENERATE 6
#define ORC_ESINGULAR 7
#define ORC_EINDEFINITE 8
#define ORC_EBREAKDOWN 9
#define ORC_NOT_CONVERGED 10

/* ========================================================================== */
/* Step 1 -- edge tags from the Green-strain increment (main Sec 4.2, Eq 3,    */
/* P:834-838; supp Sec 1.1).                                         */
/* ========================================================================== */

/* D = [P_b - P_a | P_c - P_a | P_d - P_a]  (columns are the tet edges). */
static void edge_matrix(const double *P, const int32_t *t, double D[3][3]) {
  for (int r = 0; r < 3; ++r) {
    D[r][0] = P[3 * (int64_t)t[1] + r] - P[3 * (int64_t)t[0] + r];
    D[r][1] = P[3 * (int64_t)t[2] + r] - P[3 * (int64_t)t[0] + r];
    D[r][2] = P[3 * (int64_t)t[3] + r] - P[3 * (int64_t)t[0] + r];
  }
}

/* Inverse by the adjugate divided by the determinant: Minv = adj(D) * (1/det). */
static int inverse3(const double D[3][3], double M[3][3]) {
  double cof[3][3];
  cof[0][0] = D[1][1] * D[2][2] - D[1][2] * D[2][1];
  cof[0][1] = D[1][2] * D[2][0] - D[1][0] * D[2][2];
  cof[0][2] = D[1][0] * D[2][1] - D[1][1] * D[2][0];
  cof[1][0] = D[0][2] * D[2][1] - D[0][1] * D[2][2];
  cof[1][1] = D[0][0] * D[2][2] - D[0][2] * D[2][0];
  cof[1][2] = D[0][1] * D[2][0] - D[0][0] * D[2][1];
  cof[2][0] = D[0][1] * D[1][2] - D[0][2] * D[1][1];
  cof[2][1] = D[0][2] * D[1][0] - D[0][0] * D[1][2];
  cof[2][2] = D[0][0] * D[1][1] - D[0][1] * D[1][0];
  double det = D[0][0] * cof[0][0] + D[0][1] * cof[0][1] + D[0][2] * cof[0][2];
  if (det == 0.0 || !isfinite(det)) return 1;
  double inv_det = 1.0 / det;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) M[r][c] = cof[c][r] * inv_det;
  return 0;
}

/* G = 1/2 (F^T F - I) with F = Ds Dm^-1. */
static void green_strain(const double Ds[3][3], const double Minv[3][3], double G[3][3]) {
  double F[3][3], C[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      F[r][c] = Ds[r][0] * Minv[0][c] + Ds[r][1] * Minv[1][c] + Ds[r][2] * Minv[2][c];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      C[r][c] = F[0][r] * F[0][c] + F[1][r] * F[1][c] + F[2][r] * F[2][c];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) G[r][c] = 0.5 * (C[r][c] - (r == c ? 1.0 : 0.0));
}

/*
 * n_t = || G(x_cur) - G(x_prev) ||_F ; flag_t = n_t > theta (strict, [R11]);
 * tau_e = 0 iff some tet containing e is flagged, else 1.
 * slot_tags[2E] gets both directed slots of each edge (tet_slots[T][12]).
 * Returns ORC_EDEGENERATE (and *bad = tet index) if det(Dm) == 0.
 */
int orc_tag_edges(int64_t n_tets, const int32_t *tets, const int32_t *tet_slots, const double *X,
                  const double *x_prev, const double *x_cur, double theta, int64_t n_slots,
                  uint8_t *slot_tags, double *tet_norm, uint8_t *tet_flag, int64_t *bad) {
  for (int64_t s = 0; s < n_slots; ++s) slot_tags[s] = 1; /* default: collapsible */
  for (int64_t t = 0; t < n_tets; ++t) {
    const int32_t *tt = tets + 4 * t;
    double Dm[3][3], Minv[3][3], Dp[3][3], Dc[3][3], Gp[3][3], Gc[3][3];
    edge_matrix(X, tt, Dm);
    if (inverse3(Dm, Minv)) {
      if (bad) *bad = t;
      return ORC_EDEGENERATE;
    }
    edge_matrix(x_prev, tt, Dp);
    edge_matrix(x_cur, tt, Dc);
    green_strain(Dp, Minv, Gp);
    green_strain(Dc, Minv, Gc);
    double s2 = 0.0;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        double d = Gc[r][c] - Gp[r][c];
        s2 = s2 + d * d;
      }
    double n = sqrt(s2);
    int flag = n > theta;
    if (tet_norm) tet_norm[t] = n;
    if (tet_flag) tet_flag[t] = (uint8_t)flag;
    if (flag)
      for (int k = 0; k < 12; ++k) slot_tags[tet_slots[12 * t + k]] = 0;
  }
  return ORC_OK;
}

/* ========================================================================== */
/* Step 2 -- the fine-to-coarse map (supp Alg S1/S2, recursion P:217) */
/* Definition [R1,R5,R6]: at each level, the components of the tagged edges     */
/* that lie inside one group (contiguous index range of gs nodes within a       */
/* segment) are merged; components are numbered by ascending minimum member    */
/* (== O[group] + rank of the first set bit among elected lanes,   */
/* P:191-195).  The next level's graph is the surviving edges mapped through    */
/* the level map with self-loops dropped.  Stop at the     */
/* first level without a merge or after max_levels levels.                      */
/* ========================================================================== */

static int64_t uf_find(int64_t *parent, int64_t v) {
  int64_t r = v;
  while (parent[r] != r) r = parent[r];
  while (parent[v] != r) {
    int64_t nx = parent[v];
    parent[v] = r;
    v = nx;
  }
  return r;
}

/* segment of index v at the current level: largest s with B[s] <= v */
static int seg_of(const int64_t *B, int n_seg, int64_t v) {
  int lo = 0, hi = n_seg - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) / 2;
    if (B[mid] <= v) lo = mid; else hi = mid - 1;
  }
  return lo;
}

/*
 * adj_ptr/adj_nbr: symmetric adjacency of the fine nodes; slot_tags per
 * directed slot.  The undirected edge {u,v} (u<v) is collapsible iff the slot
 * (u->v) in row u is tagged 1 (tags are symmetric, [R8]).
 * seg_begin: n_seg+1 ascending fine-node bounds (NULL => one segment [0,N)).
 * Outputs: map[N], agg_size[n_coarse] (nullable, capacity N), *n_coarse,
 * *n_levels, level_n[level_cap] (nullable): node count after each level.
 */
int orc_build_map(int64_t N, const int64_t *adj_ptr, const int32_t *adj_nbr, const uint8_t *slot_tags,
                  int gs, int n_seg, const int64_t *seg_begin, int max_levels, int32_t *map,
                  int64_t *agg_size, int64_t *n_coarse, int *n_levels, int64_t *level_n, int level_cap) {
  if (gs < 1 || gs > 32 || N < 0 || n_seg < 1) return ORC_EINVAL;
  if (N >= INT32_MAX) return ORC_ERANGE;
  int64_t ne = 0;
  for (int64_t u = 0; u < N; ++u)
    for (int64_t k = adj_ptr[u]; k < adj_ptr[u + 1]; ++k)
      if (adj_nbr[k] > u && slot_tags[k]) ++ne;
  int64_t *eu = (int64_t *)malloc(sizeof(int64_t) * (ne + 1));
  int64_t *ev = (int64_t *)malloc(sizeof(int64_t) * (ne + 1));
  int64_t *parent = (int64_t *)malloc(sizeof(int64_t) * (N + 1));
  int64_t *mk = (int64_t *)malloc(sizeof(int64_t) * (N + 1));
  int64_t *B = (int64_t *)malloc(sizeof(int64_t) * (n_seg + 1));
  if (!eu || !ev || !parent || !mk || !B) return ORC_ENOMEM;
  ne = 0;
  for (int64_t u = 0; u < N; ++u)
    for (int64_t k = adj_ptr[u]; k < adj_ptr[u + 1]; ++k)
      if (adj_nbr[k] > u && slot_tags[k]) { eu[ne] = u; ev[ne] = adj_nbr[k]; ++ne; }
  for (int s = 0; s <= n_seg; ++s) B[s] = seg_begin ? seg_begin[s] : (s == 0 ? 0 : N);
  for (int64_t f = 0; f < N; ++f) map[f] = (int32_t)f;
  int64_t n = N;
  int level = 0;
  for (;;) {
    for (int64_t v = 0; v < n; ++v) parent[v] = v;
    /* union the tagged edges that lie inside one group (Alg S1 l.11-15) */
    for (int64_t e = 0; e < ne; ++e) {
      int64_t u = eu[e], v = ev[e];
      int su = seg_of(B, n_seg, u), sv = seg_of(B, n_seg, v);
      if (su != sv) continue;
      if ((u - B[su]) / gs != (v - B[sv]) / gs) continue;
      int64_t ru = uf_find(parent, u), rv = uf_find(parent, v);
      if (ru == rv) continue;
      if (ru < rv) parent[rv] = ru; else parent[ru] = rv; /* root = minimum member */
    }
    /* number components by ascending minimum member ([R1]) */
    int64_t nn = 0;
    for (int64_t v = 0; v < n; ++v)
      if (uf_find(parent, v) == v) mk[v] = nn++;
    for (int64_t v = 0; v < n; ++v) mk[v] = mk[uf_find(parent, v)];
    for (int64_t f = 0; f < N; ++f) map[f] = (int32_t)mk[map[f]];
    /* next level graph: surviving edges mapped through mk, self-loops dropped */
    int64_t ne2 = 0;
    for (int64_t e = 0; e < ne; ++e) {
      int64_t a = mk[eu[e]], b = mk[ev[e]];
      if (a != b) { eu[ne2] = a; ev[ne2] = b; ++ne2; }
    }
    ne = ne2;
    for (int s = 0; s < n_seg; ++s) B[s] = (B[s] < n) ? mk[B[s]] : nn;
    B[n_seg] = nn;
    if (level_n && level < level_cap) level_n[level] = nn;
    ++level;
    int done = (nn == n) || (max_levels > 0 && level >= max_levels);
    n = nn;
    if (done) break;
  }
  *n_coarse = n;
  *n_levels = level;
  if (agg_size) {
    for (int64_t c = 0; c < n; ++c) agg_size[c] = 0;
    for (int64_t f = 0; f < N; ++f) agg_size[map[f]] += 1;
  }
  free(eu); free(ev); free(parent); free(mk); free(B);
  return ORC_OK;
}

/* ========================================================================== */
/* Step 3 -- DoF classification + reorder (supp Alg S3) and the     */
/* Galerkin coarse Hessian / gradient (supp Alg S4 + Eq S2/S3;      */
/* main Eq 4; H_c = U H_f U^T, g_c = U g_f).                  */
/* ========================================================================== */

typedef struct {
  int64_t n3, n12, n_slots, nnzb;
  int32_t *new_map;   /* [N] reordered coarse node of each fine node */
  int32_t *dof;       /* [n_coarse] 3 or 12, indexed by the reordered id */
  int64_t *row_ptr;   /* [n_slots+1] */
  int32_t *col;       /* [nnzb] ascending per row */
  double *val;        /* [nnzb*9] Neumaier-compensated sums, row-major 3x3 */
  double *bound;      /* [nnzb*9] sum |w_i[p] w_j[q]| |B_ij| (|.|-Galerkin bound, [R19]) */
  double *g_c;        /* [n_slots*3] or NULL */
  double *g_bound;    /* [n_slots*3] or NULL */
} orc_coarse;

static void neumaier_add(double *s, double *c, double x) {
  double t = *s + x;
  if (fabs(*s) >= fabs(x)) *c += (*s - t) + x;
  else *c += (x - t) + *s;
  *s = t;
}

void orc_coarse_free(orc_coarse *o) {
  if (!o) return;
  free(o->new_map); free(o->dof); free(o->row_ptr); free(o->col); free(o->val);
  free(o->bound); free(o->g_c); free(o->g_bound); free(o);
}

/* weight w_f[p] of fine node f in slot p of its coarse node: X_bar = (x,y,z,1)
 * for a 12-DoF node (A_f = X_bar (x) I3), else 1. */
static double weight(const double *X, int64_t f, int ncb, int p) {
  if (ncb == 1) return 1.0;
  return p < 3 ? X[3 * f + p] : 1.0;
}

orc_coarse *orc_assemble(int64_t N, const int32_t *map, int64_t n_c, int64_t thr, const double *X,
                         const int64_t *row_ptr, const int32_t *col, const double *val,
                         const double *g_f, int *status) {
  *status = ORC_OK;
  orc_coarse *o = (orc_coarse *)calloc(1, sizeof(orc_coarse));
  int64_t *size = (int64_t *)calloc((size_t)n_c + 1, sizeof(int64_t));
  int64_t *newid = (int64_t *)malloc(sizeof(int64_t) * ((size_t)n_c + 1));
  if (!o || !size || !newid) { *status = ORC_ENOMEM; return NULL; }
  for (int64_t f = 0; f < N; ++f) {
    if (map[f] < 0 || map[f] >= n_c) { *status = ORC_EINVAL; free(size); free(newid); orc_coarse_free(o); return NULL; }
    size[map[f]] += 1;
  }
  /* Alg S3: dof 12 iff the aggregate has more than thr fine nodes ([R15]);
   * stable reorder, 3-DoF nodes first ([R13]). */
  int64_t n12 = 0;
  for (int64_t c = 0; c < n_c; ++c) n12 += size[c] > thr;
  int64_t n3 = n_c - n12, c3 = 0, c12 = n3;
  for (int64_t c = 0; c < n_c; ++c) newid[c] = (size[c] > thr) ? c12++ : c3++;
  o->n3 = n3; o->n12 = n12; o->n_slots = n3 + 4 * n12;
  o->new_map = (int32_t *)malloc(sizeof(int32_t) * ((size_t)N + 1));
  o->dof = (int32_t *)malloc(sizeof(int32_t) * ((size_t)n_c + 1));
  for (int64_t f = 0; f < N; ++f) o->new_map[f] = (int32_t)newid[map[f]];
  for (int64_t c = 0; c < n_c; ++c) o->dof[newid[c]] = size[c] > thr ? 12 : 3;
  const int32_t *nm = o->new_map;
  /* slot(c,p) = c for c < n3; n3 + 4(c - n3) + p otherwise (Eq S2/S3, [R14]) */
#define NCB(c) ((c) < n3 ? 1 : 4)
#define SLOT(c, p) ((c) < n3 ? (int64_t)(c) : n3 + 4 * ((int64_t)(c) - n3) + (p))
  /* children of every reordered coarse node, ascending fine id */
  int64_t *cptr = (int64_t *)calloc((size_t)n_c + 2, sizeof(int64_t));
  int64_t *clist = (int64_t *)malloc(sizeof(int64_t) * ((size_t)N + 1));
  for (int64_t f = 0; f < N; ++f) cptr[nm[f] + 1] += 1;
  for (int64_t c = 0; c < n_c; ++c) cptr[c + 1] += cptr[c];
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * ((size_t)n_c + 1));
  for (int64_t c = 0; c < n_c; ++c) fill[c] = cptr[c];
  for (int64_t f = 0; f < N; ++f) clist[fill[nm[f]]++] = f;
  /* sparse accumulator over coarse column slots, one coarse slot row at a time */
  int64_t ns = o->n_slots;
  double *acc = (double *)calloc((size_t)ns * 9 + 1, sizeof(double));
  double *cmp = (double *)calloc((size_t)ns * 9 + 1, sizeof(double));
  double *bnd = (double *)calloc((size_t)ns * 9 + 1, sizeof(double));
  int64_t *stamp = (int64_t *)malloc(sizeof(int64_t) * ((size_t)ns + 1));
  int64_t *touched = (int64_t *)malloc(sizeof(int64_t) * ((size_t)ns + 1));
  for (int64_t s = 0; s < ns; ++s) stamp[s] = -1;
  int64_t cap = 1024, nnzb = 0;
  o->row_ptr = (int64_t *)malloc(sizeof(int64_t) * ((size_t)ns + 1));
  o->col = (int32_t *)malloc(sizeof(int32_t) * cap);
  o->val = (double *)malloc(sizeof(double) * 9 * cap);
  o->bound = (double *)malloc(sizeof(double) * 9 * cap);
  o->row_ptr[0] = 0;
  for (int64_t c = 0; c < n_c; ++c) {
    int ncb_a = NCB(c);
    for (int p = 0; p < ncb_a; ++p) {
      int64_t r = SLOT(c, p), nt = 0;
      for (int64_t ci = cptr[c]; ci < cptr[c + 1]; ++ci) {
        int64_t i = clist[ci];
        double wi = weight(X, i, ncb_a, p);
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
          int64_t j = col[k], b = nm[j];
          int ncb_b = NCB(b);
          for (int q = 0; q < ncb_b; ++q) {
            int64_t cs = SLOT(b, q);
            double coef = wi * weight(X, j, ncb_b, q);
            if (stamp[cs] != r) {
              stamp[cs] = r;
              touched[nt++] = cs;
              for (int e = 0; e < 9; ++e) acc[9 * cs + e] = cmp[9 * cs + e] = bnd[9 * cs + e] = 0.0;
            }
            for (int e = 0; e < 9; ++e) {
              double v = val[9 * k + e];
              neumaier_add(&acc[9 * cs + e], &cmp[9 * cs + e], coef * v);
              bnd[9 * cs + e] += fabs(coef) * fabs(v);
            }
          }
        }
      }
      /* emit the row with ascending columns (insertion sort of touched slots) */
      for (int64_t a = 1; a < nt; ++a) {
        int64_t key = touched[a], b = a - 1;
        while (b >= 0 && touched[b] > key) { touched[b + 1] = touched[b]; --b; }
        touched[b + 1] = key;
      }
      if (nnzb + nt > cap) {
        while (nnzb + nt > cap) cap *= 2;
        o->col = (int32_t *)realloc(o->col, sizeof(int32_t) * cap);
        o->val = (double *)realloc(o->val, sizeof(double) * 9 * cap);
        o->bound = (double *)realloc(o->bound, sizeof(double) * 9 * cap);
      }
      for (int64_t a = 0; a < nt; ++a) {
        int64_t cs = touched[a];
        o->col[nnzb] = (int32_t)cs;
        for (int e = 0; e < 9; ++e) {
          o->val[9 * nnzb + e] = acc[9 * cs + e] + cmp[9 * cs + e];
          o->bound[9 * nnzb + e] = bnd[9 * cs + e];
        }
        ++nnzb;
      }
      o->row_ptr[r + 1] = nnzb;
    }
  }
  o->nnzb = nnzb;
  /* g_c = U g_f : g_c[slot(nm f, p)] += w_f[p] g_f[f] (Eq 4) */
  if (g_f) {
    o->g_c = (double *)calloc((size_t)ns * 3 + 1, sizeof(double));
    o->g_bound = (double *)calloc((size_t)ns * 3 + 1, sizeof(double));
    double *gc = (double *)calloc((size_t)ns * 3 + 1, sizeof(double));
    for (int64_t f = 0; f < N; ++f) {
      int64_t c = nm[f];
      int ncb = NCB(c);
      for (int p = 0; p < ncb; ++p) {
        double w = weight(X, f, ncb, p);
        int64_t s = SLOT(c, p);
        for (int d = 0; d < 3; ++d) {
          neumaier_add(&o->g_c[3 * s + d], &gc[3 * s + d], w * g_f[3 * f + d]);
          o->g_bound[3 * s + d] += fabs(w) * fabs(g_f[3 * f + d]);
        }
      }
    }
    for (int64_t s = 0; s < 3 * ns; ++s) o->g_c[s] += gc[s];
    free(gc);
  }
#undef NCB
#undef SLOT
  free(size); free(newid); free(cptr); free(clist); free(fill);
  free(acc); free(cmp); free(bnd); free(stamp); free(touched);
  return o;
}

/* ========================================================================== */
/* Step 4 -- coarse PCG with 3x3 block-Jacobi;    */
/* textbook preconditioned CG (Saad, Iterative Methods, Alg 9.1), [R20].        */
/* ========================================================================== */

static void bsr_spmv(int64_t n, const int64_t *rp, const int32_t *col, const double *val,
                     const double *x, double *y) {
  for (int64_t r = 0; r < n; ++r) {
    double y0 = 0.0, y1 = 0.0, y2 = 0.0;
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
      const double *B = val + 9 * k;
      const double *xc = x + 3 * (int64_t)col[k];
      y0 += B[0] * xc[0] + B[1] * xc[1] + B[2] * xc[2];
      y1 += B[3] * xc[0] + B[4] * xc[1] + B[5] * xc[2];
      y2 += B[6] * xc[0] + B[7] * xc[1] + B[8] * xc[2];
    }
    y[3 * r] = y0; y[3 * r + 1] = y1; y[3 * r + 2] = y2;
  }
}

static double dot(int64_t n, const double *a, const double *b) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* D^-1: inverse of each row's diagonal 3x3 block (ESINGULAR if missing/singular). */
int orc_block_jacobi(int64_t n, const int64_t *rp, const int32_t *col, const double *val, double *Dinv,
                     int64_t *bad) {
  for (int64_t r = 0; r < n; ++r) {
    const double *B = NULL;
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k)
      if (col[k] == r) B = val + 9 * k;
    double D[3][3], M[3][3];
    if (!B) { if (bad) *bad = r; return ORC_ESINGULAR; }
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) D[a][b] = B[3 * a + b];
    if (inverse3(D, M)) { if (bad) *bad = r; return ORC_ESINGULAR; }
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) Dinv[9 * r + 3 * a + b] = M[a][b];
  }
  return ORC_OK;
}

static void apply_block_diag(int64_t n, const double *Dinv, const double *r, double *z) {
  for (int64_t i = 0; i < n; ++i) {
    const double *M = Dinv + 9 * i;
    const double *v = r + 3 * i;
    z[3 * i] = M[0] * v[0] + M[1] * v[1] + M[2] * v[2];
    z[3 * i + 1] = M[3] * v[0] + M[4] * v[1] + M[5] * v[2];
    z[3 * i + 2] = M[6] * v[0] + M[7] * v[1] + M[8] * v[2];
  }
}

/*
 * Solve A x = b from the given x0.  Stop when ||r||_2 <= rel_tol ||b||_2 on the
 * recurrence residual ("relative residual-norm tolerance").  res_hist
 * (nullable, capacity max_iters+1) receives ||r_k||_2.
 */
int orc_pcg(int64_t n, const int64_t *rp, const int32_t *col, const double *val, const double *b,
            double *x, double rel_tol, int max_iters, int *iters, double *rel_res, double *res_hist) {
  int64_t m = 3 * n;
  double *r = (double *)malloc(sizeof(double) * (m + 1));
  double *z = (double *)malloc(sizeof(double) * (m + 1));
  double *p = (double *)malloc(sizeof(double) * (m + 1));
  double *q = (double *)malloc(sizeof(double) * (m + 1));
  double *Dinv = (double *)malloc(sizeof(double) * (9 * n + 1));
  int st = orc_block_jacobi(n, rp, col, val, Dinv, NULL);
  *iters = 0;
  *rel_res = 0.0;
  if (st != ORC_OK) goto out;
  bsr_spmv(n, rp, col, val, x, q);
  for (int64_t i = 0; i < m; ++i) r[i] = b[i] - q[i];
  double bn = sqrt(dot(m, b, b));
  double rn = sqrt(dot(m, r, r));
  if (res_hist) res_hist[0] = rn;
  *rel_res = bn > 0.0 ? rn / bn : rn;
  if (rn <= rel_tol * bn) goto out;
  apply_block_diag(n, Dinv, r, z);
  for (int64_t i = 0; i < m; ++i) p[i] = z[i];
  double rz = dot(m, r, z);
  st = ORC_NOT_CONVERGED;
  for (int k = 1; k <= max_iters; ++k) {
    bsr_spmv(n, rp, col, val, p, q);
    double pq = dot(m, p, q);
    if (!isfinite(pq) || !isfinite(rz)) { st = ORC_EBREAKDOWN; *iters = k; break; }
    if (pq <= 0.0) { st = ORC_EINDEFINITE; *iters = k; break; }
    double alpha = rz / pq;
    for (int64_t i = 0; i < m; ++i) x[i] += alpha * p[i];
    for (int64_t i = 0; i < m; ++i) r[i] -= alpha * q[i];
    rn = sqrt(dot(m, r, r));
    if (res_hist) res_hist[k] = rn;
    *iters = k;
    *rel_res = bn > 0.0 ? rn / bn : rn;
    if (rn <= rel_tol * bn) { st = ORC_OK; break; }
    apply_block_diag(n, Dinv, r, z);
    double rz2 = dot(m, r, z);
    double beta = rz2 / rz;
    for (int64_t i = 0; i < m; ++i) p[i] = z[i] + beta * p[i];
    rz = rz2;
  }
out:
  free(r); free(z); free(p); free(q); free(Dinv);
  return st;
}

/* ||A x - b||_2 / ||b||_2 with Neumaier-compensated row sums and norms. */
double orc_rel_residual(int64_t n, const int64_t *rp, const int32_t *col, const double *val,
                        const double *x, const double *b) {
  double rs = 0.0, rc = 0.0, bs = 0.0, bc = 0.0;
  for (int64_t r = 0; r < n; ++r) {
    for (int d = 0; d < 3; ++d) {
      double s = 0.0, c = 0.0;
      neumaier_add(&s, &c, -b[3 * r + d]);
      for (int64_t k = rp[r]; k < rp[r + 1]; ++k)
        for (int e = 0; e < 3; ++e) neumaier_add(&s, &c, val[9 * k + 3 * d + e] * x[3 * (int64_t)col[k] + e]);
      double v = s + c;
      neumaier_add(&rs, &rc, v * v);
      neumaier_add(&bs, &bc, b[3 * r + d] * b[3 * r + d]);
    }
  }
  double bn = sqrt(bs + bc);
  double rn = sqrt(rs + rc);
  return bn > 0.0 ? rn / bn : rn;
}

/* y = A x (plain row order) -- used by tests to build right-hand sides. */
void orc_spmv(int64_t n, const int64_t *rp, const int32_t *col, const double *val, const double *x,
              double *y) {
  bsr_spmv(n, rp, col, val, x, y);
}

/* ========================================================================== */
/* NEXT#2 -- symmetric storage (main Sec 6: "we store and accumulate   */
/* only the diagonal and upper-triangular entries").  Upper storage U of a    */
/* full BSR A keeps the blocks with col >= row in order; the product of the   */
/* symmetric operator from U is y_i = sum_{j>=i} U_ij x_j + sum_{j<i} U_ji^T x_j */
/* written out literally.  orc_bsr_upper returns the block count (urp/ucol/   */
/* uval may be NULL to count only).                                           */
/* ========================================================================== */
int64_t orc_bsr_upper(int64_t n, const int64_t *rp, const int32_t *col, const double *val, int64_t *urp,
                      int32_t *ucol, double *uval) {
  int64_t k = 0;
  if (urp) urp[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      if (col[e] < i) continue;
      if (ucol) ucol[k] = col[e];
      if (uval) memcpy(uval + 9 * k, val + 9 * e, 9 * sizeof(double));
      ++k;
    }
    if (urp) urp[i + 1] = k;
  }
  return k;
}

void orc_spmv_upper(int64_t n, const int64_t *urp, const int32_t *ucol, const double *uval, const double *x,
                    double *y) {
  for (int64_t t = 0; t < 3 * n; ++t) y[t] = 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = urp[i]; e < urp[i + 1]; ++e) {
      const int64_t j = ucol[e];
      const double *B = uval + 9 * e;
      for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) {
          y[3 * i + a] += B[3 * a + c] * x[3 * j + c];   /* U_ij x_j            */
          if (j != i) y[3 * j + c] += B[3 * a + c] * x[3 * i + a]; /* (U_ij^T x_i)_c */
        }
    }
}

/* Full storage from upper storage (the inverse of orc_bsr_upper on a symmetric */
/* pattern): full(i,j) = U(i,j) for j >= i and U(j,i)^T for j < i.  The full    */
/* pattern (rp, col) is given; returns the number of full blocks with no source */
/* in U (0 for a consistent pair of patterns).                                  */
int64_t orc_bsr_expand_upper(int64_t n, const int64_t *rp, const int32_t *col, const int64_t *urp,
                             const int32_t *ucol, const double *uval, double *val) {
  int64_t missing = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      const int64_t j = col[e];
      const int64_t r = j >= i ? i : j, c = j >= i ? j : i; /* stored as U(r, c) */
      int64_t f = -1;
      for (int64_t k = urp[r]; k < urp[r + 1]; ++k)
        if (ucol[k] == c) { f = k; break; }
      if (f < 0) { ++missing; memset(val + 9 * e, 0, 9 * sizeof(double)); continue; }
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          val[9 * e + 3 * a + b] = j >= i ? uval[9 * f + 3 * a + b] : uval[9 * f + 3 * b + a];
    }
  return missing;
}

/* ========================================================================== */
/* NEXT#1 -- prolongation d_f = U^T d_c (main Sec 4.3: "we mathematically */
/* prolongate the displacement to the fine mesh using the transpose of the     */
/* restriction operator").  For a 3-DoF parent d_f = d_c[c]; for a 12-DoF parent */
/* d_f = sum_p X_bar_f[p] d_c[slot(c,p)] (A_f^T d_c, A_f = X_bar (x) I3). */
/* ========================================================================== */
void orc_prolongate(int64_t N, const int32_t *new_map, int64_t n3, const double *X, const double *x_c,
                    double *d_f) {
  for (int64_t f = 0; f < N; ++f) {
    int64_t c = new_map[f];
    for (int d = 0; d < 3; ++d) {
      double s = 0.0;
      if (c < n3) {
        s = x_c[3 * c + d];
      } else {
        for (int p = 0; p < 4; ++p) {
          double w = p < 3 ? X[3 * f + p] : 1.0;
          s += w * x_c[3 * (n3 + 4 * (c - n3) + p) + d];
        }
      }
      d_f[3 * f + d] = s;
    }
  }
}

/* ========================================================================== */
/* NEXT#4 -- step 1 for shells and rods (main Sec 4.2: "applicable to various  */
/* element types (shells, volumes, rods)").       */
/* Triangle (a,b,c): rest tangent basis t1 = e1/|e1|, n = (e1 x e2)/|e1 x e2|, */
/* t2 = n x t1 (e1 = X_b - X_a, e2 = X_c - X_a); D_m = [t_r . e_c] (2x2);       */
/* F = D_s D_m^-1 (3x2), D_s = [x_b - x_a | x_c - x_a]; G = 1/2 (F^T F - I_2). */
/* Edge (a,b): F = l / L (current / rest length), G = 1/2 (F^2 - 1).           */
/* n = ||G(x_cur) - G(x_prev)||_F (|.| for edges), flagged iff n > theta;     */
/* every directed slot of a flagged element's edges gets tag 0.  The caller's  */
/* slot_tags are NOT reset (tets, shells and rods accumulate; reset_tags = 1   */
/* first sets every slot to 1).  Fixed operation order, no FMA [R12].          */
/* ========================================================================== */
static double dot3(const double *u, const double *v) { return u[0] * v[0] + u[1] * v[1] + u[2] * v[2]; }

static void cross3(const double *u, const double *v, double *w) {
  w[0] = u[1] * v[2] - u[2] * v[1];
  w[1] = u[2] * v[0] - u[0] * v[2];
  w[2] = u[0] * v[1] - u[1] * v[0];
}

/* G (2x2) of triangle t at positions P, with the rest inverse Minv */
static void tri_green(const double *P, const int32_t *t, const double Minv[2][2], double G[2][2]) {
  double d1[3], d2[3], F[3][2];
  for (int r = 0; r < 3; ++r) {
    d1[r] = P[3 * (int64_t)t[1] + r] - P[3 * (int64_t)t[0] + r];
    d2[r] = P[3 * (int64_t)t[2] + r] - P[3 * (int64_t)t[0] + r];
  }
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 2; ++c) F[r][c] = d1[r] * Minv[0][c] + d2[r] * Minv[1][c];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c) {
      double C = F[0][r] * F[0][c] + F[1][r] * F[1][c] + F[2][r] * F[2][c];
      G[r][c] = 0.5 * (C - (r == c ? 1.0 : 0.0));
    }
}

int orc_tag_shells(int64_t n_tris, const int32_t *tris, const int32_t *tri_slots, const double *X,
                   const double *x_prev, const double *x_cur, double theta, int64_t n_slots, int reset_tags,
                   uint8_t *slot_tags, double *tri_norm, int64_t *bad) {
  if (reset_tags)
    for (int64_t s = 0; s < n_slots; ++s) slot_tags[s] = 1;
  for (int64_t t = 0; t < n_tris; ++t) {
    const int32_t *tt = tris + 3 * t;
    double e1[3], e2[3], nr[3], t1[3], t2[3];
    for (int r = 0; r < 3; ++r) {
      e1[r] = X[3 * (int64_t)tt[1] + r] - X[3 * (int64_t)tt[0] + r];
      e2[r] = X[3 * (int64_t)tt[2] + r] - X[3 * (int64_t)tt[0] + r];
    }
    double L1 = sqrt(dot3(e1, e1));
    cross3(e1, e2, nr);
    double Ln = sqrt(dot3(nr, nr));
    if (L1 == 0.0 || Ln == 0.0 || !isfinite(L1) || !isfinite(Ln)) {
      if (bad) *bad = t;
      return ORC_EDEGENERATE;
    }
    double i1 = 1.0 / L1, in = 1.0 / Ln;
    for (int r = 0; r < 3; ++r) {
      t1[r] = e1[r] * i1;
      nr[r] = nr[r] * in;
    }
    cross3(nr, t1, t2);
    double Dm[2][2] = {{dot3(t1, e1), dot3(t1, e2)}, {dot3(t2, e1), dot3(t2, e2)}};
    double det = Dm[0][0] * Dm[1][1] - Dm[0][1] * Dm[1][0];
    if (det == 0.0 || !isfinite(det)) {
      if (bad) *bad = t;
      return ORC_EDEGENERATE;
    }
    double id = 1.0 / det;
    double Minv[2][2] = {{Dm[1][1] * id, -Dm[0][1] * id}, {-Dm[1][0] * id, Dm[0][0] * id}};
    double Gp[2][2], Gc[2][2];
    tri_green(x_prev, tt, Minv, Gp);
    tri_green(x_cur, tt, Minv, Gc);
    double s2 = 0.0;
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < 2; ++c) {
        double d = Gc[r][c] - Gp[r][c];
        s2 = s2 + d * d;
      }
    double n = sqrt(s2);
    if (tri_norm) tri_norm[t] = n;
    if (n > theta)
      for (int k = 0; k < 6; ++k)
        if (tri_slots[6 * t + k] >= 0) slot_tags[tri_slots[6 * t + k]] = 0;
  }
  return ORC_OK;
}

int orc_tag_rods(int64_t n_segs, const int32_t *segs, const int32_t *seg_slots, const double *X,
                 const double *x_prev, const double *x_cur, double theta, int64_t n_slots, int reset_tags,
                 uint8_t *slot_tags, double *seg_norm, int64_t *bad) {
  if (reset_tags)
    for (int64_t s = 0; s < n_slots; ++s) slot_tags[s] = 1;
  for (int64_t t = 0; t < n_segs; ++t) {
    const int64_t a = segs[2 * t], b = segs[2 * t + 1];
    double dR[3], dp[3], dc[3];
    for (int r = 0; r < 3; ++r) {
      dR[r] = X[3 * b + r] - X[3 * a + r];
      dp[r] = x_prev[3 * b + r] - x_prev[3 * a + r];
      dc[r] = x_cur[3 * b + r] - x_cur[3 * a + r];
    }
    double L = sqrt(dot3(dR, dR));
    if (L == 0.0 || !isfinite(L)) {
      if (bad) *bad = t;
      return ORC_EDEGENERATE;
    }
    double Fp = sqrt(dot3(dp, dp)) / L, Fc = sqrt(dot3(dc, dc)) / L;
    double Gp = 0.5 * (Fp * Fp - 1.0), Gc = 0.5 * (Fc * Fc - 1.0);
    double n = fabs(Gc - Gp);
    if (seg_norm) seg_norm[t] = n;
    if (n > theta)
      for (int k = 0; k < 2; ++k)
        if (seg_slots[2 * t + k] >= 0) slot_tags[seg_slots[2 * t + k]] = 0;
  }
  return ORC_OK;
}

/* ========================================================================== */
/* NEXT#3 -- fine-level hash reduction (supp Sec 2): triplets      */
/* (i, j, B_ij) keyed by (i << 32) | j, sorted by key (stable: equal keys keep */
/* input order), each group of equal keys summed in that order.  Output: the  */
/* unique triplets as BSR (rows ascending, columns ascending within a row).   */
/* ========================================================================== */
static const uint64_t *g_trip_key;

static int trip_cmp(const void *pa, const void *pb) {
  const int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
  if (g_trip_key[a] != g_trip_key[b]) return g_trip_key[a] < g_trip_key[b] ? -1 : 1;
  return a < b ? -1 : (a > b ? 1 : 0); /* stable */
}

/* returns nnzb (>= 0) or -ORC_EINVAL; row_ptr[n_rows+1], col/val sized n (worst case) */
int64_t orc_reduce_triplets(int64_t n_rows, int64_t n, const int32_t *ti, const int32_t *tj, const double *tval,
                            int64_t *row_ptr, int32_t *col, double *val) {
  uint64_t *key = (uint64_t *)malloc(sizeof(uint64_t) * (n + 1));
  int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
  for (int64_t t = 0; t < n; ++t) {
    if (ti[t] < 0 || tj[t] < 0 || ti[t] >= n_rows) {
      free(key);
      free(idx);
      return -ORC_EINVAL;
    }
    key[t] = ((uint64_t)(uint32_t)ti[t] << 32) | (uint32_t)tj[t]; /* hash key */
    idx[t] = t;
  }
  g_trip_key = key;
  qsort(idx, (size_t)n, sizeof(int64_t), trip_cmp);
  for (int64_t r = 0; r <= n_rows; ++r) row_ptr[r] = 0;
  int64_t u = -1;
  for (int64_t s = 0; s < n; ++s) {
    const int64_t t = idx[s];
    if (s == 0 || key[t] != key[idx[s - 1]]) {
      ++u;
      col[u] = tj[t];
      row_ptr[ti[t] + 1] += 1;
      for (int e = 0; e < 9; ++e) val[9 * u + e] = tval[9 * t + e];
    } else {
      for (int e = 0; e < 9; ++e) val[9 * u + e] = val[9 * u + e] + tval[9 * t + e];
    }
  }
  for (int64_t r = 0; r < n_rows; ++r) row_ptr[r + 1] += row_ptr[r];
  free(key);
  free(idx);
  return u + 1;
}
