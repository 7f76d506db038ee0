/*
 * Fast seeded-input generation for the AGIPC coarsening path -- INPUT GENERATION ONLY.
 *
 * Part of `synth/`, the one module shared by the CPU oracle and the CUDA path.  Like the
 * Python in synth/__init__.py it holds none of the method's arithmetic (no Green strain,
 * no tags, no hashing, no Galerkin products, no PCG): it builds the static Kuhn tet mesh
 * (adjacency, tet->slot table, BSR pattern) and the fine Hessian input
 * H_f = M_lumped (x) I3 + dt^2 K_lin, which the numpy versions build too slowly at the
 * 20M-node configuration (BASELINE.json configs[4]).  tests/test_synth_fast.py pins every
 * array against the numpy generator (synth.kuhn_grid_py / fine_hessian_py) on small grids.
 *
 * Build: gcc -O3 -fopenmp -ffp-contract=off -shared -fPIC (synth.build()).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* spread the low 10 bits of x so that bit b lands at bit 3b */
static inline int64_t spread3(int64_t x) {
  int64_t r = 0;
  for (int b = 0; b < 21; ++b) r |= ((x >> b) & 1) << (3 * b);
  return r;
}

/* Morton key with the x (i) bit lowest, as synth._morton_key */
static inline int64_t morton(int64_t i, int64_t j, int64_t k) { return spread3(i) | (spread3(j) << 1) | (spread3(k) << 2); }

/* The 7 positive Kuhn edge offsets (every component in {0,1}, not all 0); an edge joins v and
 * v + d or v - d.  Local tet edge order (0,1),(0,2),(0,3),(1,2),(1,3),(2,3). */
static const int TE[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
static const int PERMS[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

/* position of nb in the ascending row [p0, p1) of cols (linear: rows hold <= 15 entries) */
static inline int64_t find_in_row(const int32_t *cols, int64_t p0, int64_t p1, int32_t nb) {
  for (int64_t p = p0; p < p1; ++p)
    if (cols[p] == nb) return p;
  return -1;
}

/*
 * Kuhn/Freudenthal 6-tet grid with n nodes per side (synth.kuhn_grid, order='morton').
 * Sizes: N = n^3, T = 6 (n-1)^3, E = 3n^2(n-1) + 3n(n-1)^2 + (n-1)^3 (caller allocates).
 * Returns 0, or -1 if the sizes do not match the enumeration.
 */
int syn_kuhn_grid(int64_t n, double side, double ox, double oy, double oz, int64_t N, int64_t T, int64_t E,
                  double *X, int32_t *ijk, int32_t *tets, int64_t *adj_ptr, int32_t *adj_nbr, int32_t *tet_slots,
                  int32_t *edges, int64_t *edge_of_slot, int64_t *bsr_ptr, int32_t *bsr_col, int64_t *diag_slot) {
  if (n < 2 || N != n * n * n) return -1;
  /* new id of every lex node = rank of its Morton key (keys unique, so the order is total) */
  int64_t bits = 0;
  while ((1LL << bits) < n) ++bits;
  const int64_t nkeys = 1LL << (3 * bits);
  int32_t *new_of_lex = (int32_t *)malloc(sizeof(int32_t) * N);
  if (!new_of_lex) return -2;
  {
    int64_t r = 0;
    for (int64_t key = 0; key < nkeys; ++key) {
      int64_t i = 0, j = 0, k = 0;
      for (int b = 0; b < bits; ++b) {
        i |= ((key >> (3 * b)) & 1) << b;
        j |= ((key >> (3 * b + 1)) & 1) << b;
        k |= ((key >> (3 * b + 2)) & 1) << b;
      }
      if (i < n && j < n && k < n) {
        const int64_t lex = (i * n + j) * n + k;
        new_of_lex[lex] = (int32_t)r;
        ijk[3 * r] = (int32_t)i;
        ijk[3 * r + 1] = (int32_t)j;
        ijk[3 * r + 2] = (int32_t)k;
        ++r;
      }
    }
    if (r != N) {
      free(new_of_lex);
      return -1;
    }
  }
  const double h = side / (double)(n - 1);
  const double o[3] = {ox, oy, oz};
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < N; ++v)
    for (int d = 0; d < 3; ++d) X[3 * v + d] = ((double)ijk[3 * v + d] * h - 0.5 * side) + o[d];

  /* adjacency rows: v +- d for the 7 offsets, inside the grid, ascending by new id */
  static const int OFF[14][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 0}, {1, 0, 1}, {0, 1, 1}, {1, 1, 1},
                                 {-1, 0, 0}, {0, -1, 0}, {0, 0, -1}, {-1, -1, 0}, {-1, 0, -1}, {0, -1, -1}, {-1, -1, -1}};
  int64_t *upcnt = (int64_t *)malloc(sizeof(int64_t) * (N + 1));
  if (!upcnt) {
    free(new_of_lex);
    return -2;
  }
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < N; ++v) {
    const int i = ijk[3 * v], j = ijk[3 * v + 1], k = ijk[3 * v + 2];
    int c = 0, up = 0;
    for (int q = 0; q < 14; ++q) {
      const int a = i + OFF[q][0], b = j + OFF[q][1], cc = k + OFF[q][2];
      if (a < 0 || b < 0 || cc < 0 || a >= n || b >= n || cc >= n) continue;
      ++c;
      up += new_of_lex[((int64_t)a * n + b) * n + cc] > v;
    }
    adj_ptr[v + 1] = c;
    upcnt[v] = up;
  }
  adj_ptr[0] = 0;
  for (int64_t v = 0; v < N; ++v) adj_ptr[v + 1] += adj_ptr[v];
  if (adj_ptr[N] != 2 * E) {
    free(new_of_lex);
    free(upcnt);
    return -1;
  }
  /* edge id base of each row's upper neighbours (edges sorted by (lo, hi)) */
  {
    int64_t run = 0;
    for (int64_t v = 0; v < N; ++v) {
      const int64_t c = upcnt[v];
      upcnt[v] = run;
      run += c;
    }
    upcnt[N] = run;
    if (run != E) {
      free(new_of_lex);
      free(upcnt);
      return -1;
    }
  }
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < N; ++v) {
    const int i = ijk[3 * v], j = ijk[3 * v + 1], k = ijk[3 * v + 2];
    int32_t nb[14];
    int c = 0;
    for (int q = 0; q < 14; ++q) {
      const int a = i + OFF[q][0], b = j + OFF[q][1], cc = k + OFF[q][2];
      if (a < 0 || b < 0 || cc < 0 || a >= n || b >= n || cc >= n) continue;
      nb[c++] = new_of_lex[((int64_t)a * n + b) * n + cc];
    }
    for (int x = 1; x < c; ++x) { /* insertion sort */
      int32_t t = nb[x];
      int y = x - 1;
      while (y >= 0 && nb[y] > t) {
        nb[y + 1] = nb[y];
        --y;
      }
      nb[y + 1] = t;
    }
    const int64_t p0 = adj_ptr[v];
    int below = 0;
    for (int x = 0; x < c; ++x) {
      adj_nbr[p0 + x] = nb[x];
      below += nb[x] < v;
    }
    /* fine Hessian pattern: the adjacency row with the diagonal inserted */
    const int64_t b0 = p0 + v;
    bsr_ptr[v] = b0;
    for (int x = 0; x < below; ++x) bsr_col[b0 + x] = nb[x];
    bsr_col[b0 + below] = (int32_t)v;
    diag_slot[v] = b0 + below;
    for (int x = below; x < c; ++x) bsr_col[b0 + x + 1] = nb[x];
    /* upper neighbours: consecutive edge ids */
    int64_t e = upcnt[v];
    for (int x = below; x < c; ++x, ++e) {
      edges[2 * e] = (int32_t)v;
      edges[2 * e + 1] = nb[x];
      edge_of_slot[p0 + x] = e;
    }
  }
  bsr_ptr[N] = adj_ptr[N] + N;
  /* lower neighbours: the edge id of (u, v), u < v, from row u */
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < N; ++v) {
    for (int64_t p = adj_ptr[v]; p < adj_ptr[v + 1]; ++p) {
      const int32_t u = adj_nbr[p];
      if (u > v) break;
      int64_t below_u = 0;
      for (int64_t q = adj_ptr[u]; q < adj_ptr[u + 1] && adj_nbr[q] < u; ++q) ++below_u;
      const int64_t pos = find_in_row(adj_nbr, adj_ptr[u], adj_ptr[u + 1], (int32_t)v);
      edge_of_slot[p] = upcnt[u] + (pos - adj_ptr[u] - below_u);
    }
  }
  free(upcnt);
  /* tets: cubes in order of the new id of their min corner (== the min node of each of its 6
   * tets, Morton being monotone in every coordinate), types in PERMS order -- the stable sort
   * by min node of the numpy generator */
  const int64_t nc = n - 1;
  int64_t *cube_base = (int64_t *)malloc(sizeof(int64_t) * (N + 1));
  if (!cube_base) {
    free(new_of_lex);
    return -2;
  }
  {
    int64_t run = 0;
    for (int64_t v = 0; v < N; ++v) {
      cube_base[v] = run;
      run += (ijk[3 * v] < nc && ijk[3 * v + 1] < nc && ijk[3 * v + 2] < nc) ? 6 : 0;
    }
    if (run != T) {
      free(new_of_lex);
      free(cube_base);
      return -1;
    }
  }
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < N; ++v) {
    const int i = ijk[3 * v], j = ijk[3 * v + 1], k = ijk[3 * v + 2];
    if (i >= nc || j >= nc || k >= nc) continue;
    for (int ty = 0; ty < 6; ++ty) {
      int c[3] = {i, j, k};
      int32_t vs[4];
      vs[0] = (int32_t)v;
      for (int s = 0; s < 3; ++s) {
        c[PERMS[ty][s]] += 1;
        vs[s + 1] = new_of_lex[((int64_t)c[0] * n + c[1]) * n + c[2]];
      }
      const int64_t t = cube_base[v] + ty;
      for (int a = 0; a < 4; ++a) tets[4 * t + a] = vs[a];
      for (int e = 0; e < 6; ++e) {
        const int32_t a = vs[TE[e][0]], b = vs[TE[e][1]];
        tet_slots[12 * t + 2 * e] = (int32_t)find_in_row(adj_nbr, adj_ptr[a], adj_ptr[a + 1], b);
        tet_slots[12 * t + 2 * e + 1] = (int32_t)find_in_row(adj_nbr, adj_ptr[b], adj_ptr[b + 1], a);
      }
    }
  }
  free(cube_base);
  free(new_of_lex);
  return 0;
}

/* 3x3 inverse by the adjugate (input generation; any correct inverse will do) */
static void inv3(const double m[9], double r[9], double *det_out) {
  const double c00 = m[4] * m[8] - m[5] * m[7], c01 = m[5] * m[6] - m[3] * m[8], c02 = m[3] * m[7] - m[4] * m[6];
  const double det = m[0] * c00 + m[1] * c01 + m[2] * c02;
  const double id = 1.0 / det;
  r[0] = c00 * id;
  r[1] = (m[2] * m[7] - m[1] * m[8]) * id;
  r[2] = (m[1] * m[5] - m[2] * m[4]) * id;
  r[3] = c01 * id;
  r[4] = (m[0] * m[8] - m[2] * m[6]) * id;
  r[5] = (m[2] * m[3] - m[0] * m[5]) * id;
  r[6] = c02 * id;
  r[7] = (m[1] * m[6] - m[0] * m[7]) * id;
  r[8] = (m[0] * m[4] - m[1] * m[3]) * id;
  *det_out = det;
}

/* P1 shape-function gradients of tet t scaled by sqrt(V) (g[a][d]) and the volume V */
static void tet_grads(const double *X, const int32_t *tv, double g[4][3], double *V) {
  const double *xa = X + 3 * (int64_t)tv[0];
  double Dm[9];
  for (int c = 0; c < 3; ++c) {
    const double *xc = X + 3 * (int64_t)tv[c + 1];
    for (int d = 0; d < 3; ++d) Dm[3 * d + c] = xc[d] - xa[d]; /* column c = X_c - X_a */
  }
  double Mi[9], det;
  inv3(Dm, Mi, &det);
  const double vol = fabs(det) / 6.0;
  const double s = sqrt(vol);
  for (int a = 1; a < 4; ++a)
    for (int d = 0; d < 3; ++d) g[a][d] = Mi[3 * (a - 1) + d] * s; /* rows of D_m^-1 = grad N_1..3 */
  for (int d = 0; d < 3; ++d) g[0][d] = -(Mi[d] + Mi[3 + d] + Mi[6 + d]) * s;
  *V = vol;
}

/* raw (unsymmetrised) linear-elastic block R_ab[i][j] = mu g_b[i] g_a[j] + lam g_a[i] g_b[j]
 * + mu (g_a.g_b) delta_ij, with E = 1 (synth.stiffness_blocks) */
static void raw_block(double g[4][3], int a, int b, double mu, double lam, double R[9]) {
  const double gg = g[a][0] * g[b][0] + g[a][1] * g[b][1] + g[a][2] * g[b][2];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[3 * i + j] = g[b][i] * (mu * g[a][j]) + (lam * g[a][i]) * g[b][j] + (i == j ? mu * gg : 0.0);
}

/*
 * Fine Hessian values on a given BSR pattern (synth.fine_hessian): for every stored block (u, w),
 * H_uw = sum over the tets containing u and w, in ascending tet order, of dt^2 E_t K_t[a][b]
 * (K = the symmetrised linear-elastic tet stiffness, K_ba = K_ab^T bit for bit), plus
 * m_u I3 on the diagonal (m_u = sum rho V_t / 4 over the tets of u, ascending).  Both (u, w)
 * and (w, u) sum the same tets in the same order, so H is bitwise symmetric (R22).
 * E_tet: [T] (or NULL: E_const).  Returns the number of (tet, a, b) pairs whose block is
 * missing from the pattern (0 on success).
 */
int64_t syn_fine_hessian(int64_t N, int64_t T, const int32_t *tets, const double *X, const double *E_tet, double E_const,
                         double nu, double rho, double dt, int mass, int stiffness, const int64_t *bsr_ptr,
                         const int32_t *bsr_col, const int64_t *diag_slot, double *H) {
  const double mu = 1.0 / (2.0 * (1.0 + nu));
  const double lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  const double dt2 = dt * dt;
  /* node -> incident tets, ascending */
  int64_t *ip = (int64_t *)calloc((size_t)N + 1, sizeof(int64_t));
  int64_t *it = (int64_t *)malloc(sizeof(int64_t) * (size_t)(4 * T > 0 ? 4 * T : 1));
  if (!ip || !it) {
    free(ip);
    free(it);
    return -1;
  }
  for (int64_t q = 0; q < 4 * T; ++q) ip[tets[q] + 1] += 1;
  for (int64_t v = 0; v < N; ++v) ip[v + 1] += ip[v];
  {
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
    memcpy(cur, ip, sizeof(int64_t) * (size_t)N);
    for (int64_t t = 0; t < T; ++t)
      for (int a = 0; a < 4; ++a) it[cur[tets[4 * t + a]]++] = t;
    free(cur);
  }
  memset(H, 0, sizeof(double) * 9 * (size_t)bsr_ptr[N]);
  int64_t missing = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : missing)
  for (int64_t u = 0; u < N; ++u) {
    double m = 0.0;
    const int64_t r0 = bsr_ptr[u], r1 = bsr_ptr[u + 1];
    for (int64_t q = ip[u]; q < ip[u + 1]; ++q) {
      const int64_t t = it[q];
      const int32_t *tv = tets + 4 * t;
      double g[4][3], V;
      tet_grads(X, tv, g, &V);
      m += rho * V / 4.0;
      if (!stiffness) continue;
      int a = 0;
      while (tv[a] != u) ++a;
      const double Ev = E_tet ? E_tet[t] : E_const;
      for (int b = 0; b < 4; ++b) {
        const int64_t s = find_in_row(bsr_col, r0, r1, tv[b]);
        if (s < 0) {
          ++missing;
          continue;
        }
        double Rab[9], Rba[9];
        raw_block(g, a, b, mu, lam, Rab);
        raw_block(g, b, a, mu, lam, Rba);
        double *dst = H + 9 * s;
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            const double k = 0.5 * (Rab[3 * i + j] + Rba[3 * j + i]);
            dst[3 * i + j] += dt2 * (k * Ev);
          }
      }
    }
    if (mass) {
      double *d = H + 9 * diag_slot[u];
      d[0] += m;
      d[4] += m;
      d[8] += m;
    }
  }
  free(ip);
  free(it);
  return missing;
}

/*
 * Merge extra symmetric pattern entries into a BSR pattern (contact pairs of C4: Hessian-only
 * blocks, synth.mesh_from_tets(extra_pairs=...)).  extra: [P][2] (u, v), both (u,v) and (v,u)
 * are added unless already present.  Pass 1 (out_col == NULL) counts the merged row lengths
 * into out_ptr[1..N]; pass 2 fills out_ptr / out_col / diag_slot.  Rows ascending.
 */
int64_t syn_merge_pattern(int64_t N, const int64_t *ptr, const int32_t *col, int64_t P, const int32_t *extra,
                          int64_t *out_ptr, int32_t *out_col, int64_t *diag_slot) {
  /* extras per row (both directions), as an auxiliary CSR */
  int64_t *ep = (int64_t *)calloc((size_t)N + 1, sizeof(int64_t));
  int32_t *ec = (int32_t *)malloc(sizeof(int32_t) * (size_t)(2 * P > 0 ? 2 * P : 1));
  for (int64_t p = 0; p < P; ++p) {
    ep[extra[2 * p] + 1] += 1;
    ep[extra[2 * p + 1] + 1] += 1;
  }
  for (int64_t v = 0; v < N; ++v) ep[v + 1] += ep[v];
  {
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
    memcpy(cur, ep, sizeof(int64_t) * (size_t)N);
    for (int64_t p = 0; p < P; ++p) {
      ec[cur[extra[2 * p]]++] = extra[2 * p + 1];
      ec[cur[extra[2 * p + 1]]++] = extra[2 * p];
    }
    free(cur);
  }
  if (!out_col) {
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < N; ++v) {
      int64_t c = ptr[v + 1] - ptr[v];
      for (int64_t x = ep[v]; x < ep[v + 1]; ++x) {
        int dup = find_in_row(col, ptr[v], ptr[v + 1], ec[x]) >= 0;
        for (int64_t y = ep[v]; y < x && !dup; ++y) dup = ec[y] == ec[x];
        c += !dup;
      }
      out_ptr[v + 1] = c;
    }
    out_ptr[0] = 0;
    for (int64_t v = 0; v < N; ++v) out_ptr[v + 1] += out_ptr[v];
  } else {
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < N; ++v) {
      int64_t o = out_ptr[v];
      for (int64_t q = ptr[v]; q < ptr[v + 1]; ++q) out_col[o++] = col[q];
      for (int64_t x = ep[v]; x < ep[v + 1]; ++x) {
        int dup = 0;
        for (int64_t q = out_ptr[v]; q < o && !dup; ++q) dup = out_col[q] == ec[x];
        if (!dup) out_col[o++] = ec[x];
      }
      for (int64_t x = out_ptr[v] + 1; x < o; ++x) { /* insertion sort of the short row */
        int32_t t = out_col[x];
        int64_t y = x - 1;
        while (y >= out_ptr[v] && out_col[y] > t) {
          out_col[y + 1] = out_col[y];
          --y;
        }
        out_col[y + 1] = t;
      }
      diag_slot[v] = find_in_row(out_col, out_ptr[v], o, (int32_t)v);
    }
  }
  free(ep);
  free(ec);
  return out_ptr[N];
}

/* BSR slot of (u[k], v[k]) (-1 if absent) */
void syn_bsr_slots(int64_t K, const int64_t *ptr, const int32_t *col, const int64_t *u, const int64_t *v, int64_t *out) {
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < K; ++k) out[k] = find_in_row(col, ptr[u[k]], ptr[u[k] + 1], (int32_t)v[k]);
}
