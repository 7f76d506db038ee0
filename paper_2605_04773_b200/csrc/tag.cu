// Step 1 -- edge tags from the Green-strain increment (main Sec 4.2 Eq 3, PAPER.md P:834-838;
// supp Sec 1.1).
//
// One thread per tet.  The fp64 arithmetic follows ONE fixed operation order with explicit
// round-to-nearest intrinsics (no FMA contraction, reading R12) so that the norm --
// and therefore the integer tag decision -- is reproducible bit for bit:
//   D_m^-1 = adj(D_m) * (1/det D_m),  F = D_s D_m^-1,  G = 0.5 (F^T F - I),
//   n_t = sqrt(sum_rc (G_cur - G_prev)_rc^2) (row-major order),  flag = n_t > theta (strict).
// tau_e = 0 iff some tet containing e is flagged: the slots are pre-filled with 1 and every
// flagged tet stores 0 into the 12 directed slots of its 6 edges (idempotent, race-free).
#include "agipc_internal.cuh"

#define TAG_THREADS 256

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ void load3(const double *__restrict__ P, int v, double out[3]) {
  const double *p = P + 3 * (int64_t)v;
  out[0] = __ldg(p);
  out[1] = __ldg(p + 1);
  out[2] = __ldg(p + 2);
}

// D[r][c] = P_{n_{c+1}}[r] - P_{n_0}[r]
__device__ __forceinline__ void edge_matrix(const double *__restrict__ P, int4 t, double D[3][3]) {
  double a[3], b[3], c[3], d[3];
  load3(P, t.x, a);
  load3(P, t.y, b);
  load3(P, t.z, c);
  load3(P, t.w, d);
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    D[r][0] = ds(b[r], a[r]);
    D[r][1] = ds(c[r], a[r]);
    D[r][2] = ds(d[r], a[r]);
  }
}

__device__ __forceinline__ bool inverse3(const double D[3][3], double M[3][3]) {
  double c00 = ds(dm(D[1][1], D[2][2]), dm(D[1][2], D[2][1]));
  double c01 = ds(dm(D[1][2], D[2][0]), dm(D[1][0], D[2][2]));
  double c02 = ds(dm(D[1][0], D[2][1]), dm(D[1][1], D[2][0]));
  double c10 = ds(dm(D[0][2], D[2][1]), dm(D[0][1], D[2][2]));
  double c11 = ds(dm(D[0][0], D[2][2]), dm(D[0][2], D[2][0]));
  double c12 = ds(dm(D[0][1], D[2][0]), dm(D[0][0], D[2][1]));
  double c20 = ds(dm(D[0][1], D[1][2]), dm(D[0][2], D[1][1]));
  double c21 = ds(dm(D[0][2], D[1][0]), dm(D[0][0], D[1][2]));
  double c22 = ds(dm(D[0][0], D[1][1]), dm(D[0][1], D[1][0]));
  double det = da(da(dm(D[0][0], c00), dm(D[0][1], c01)), dm(D[0][2], c02));
  if (det == 0.0 || !isfinite(det)) return false;
  double inv = __ddiv_rn(1.0, det);
  // M[r][c] = cof[c][r] * inv
  M[0][0] = dm(c00, inv); M[0][1] = dm(c10, inv); M[0][2] = dm(c20, inv);
  M[1][0] = dm(c01, inv); M[1][1] = dm(c11, inv); M[1][2] = dm(c21, inv);
  M[2][0] = dm(c02, inv); M[2][1] = dm(c12, inv); M[2][2] = dm(c22, inv);
  return true;
}

__device__ __forceinline__ void green(const double Ds[3][3], const double M[3][3], double G[3][3]) {
  double F[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      F[r][c] = da(da(dm(Ds[r][0], M[0][c]), dm(Ds[r][1], M[1][c])), dm(Ds[r][2], M[2][c]));
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double C = da(da(dm(F[0][r], F[0][c]), dm(F[1][r], F[1][c])), dm(F[2][r], F[2][c]));
      G[r][c] = dm(0.5, ds(C, r == c ? 1.0 : 0.0));
    }
}

// (launch bounds without a minimum: 64 registers, no spills; 3 / 4 / 5 CTAs per SM pinned gave
// 80 / 64 + spill / 48 + spill registers and were slower, profiles/r02v)
#ifdef TAG_MINB
__global__ void __launch_bounds__(TAG_THREADS, TAG_MINB) k_tag(int64_t n_tets,
#else
__global__ void __launch_bounds__(TAG_THREADS) k_tag(int64_t n_tets,
#endif
                                                     const int4 *__restrict__ tets,
                                                     const int4 *__restrict__ tet_slots,
                                                     const double *__restrict__ X,
                                                     const double *__restrict__ xp,
                                                     const double *__restrict__ xc, double theta,
                                                     uint8_t *__restrict__ slot_tags,
                                                     double *__restrict__ tet_norm,
                                                     unsigned long long *__restrict__ counters) {
  int64_t t = (int64_t)blockIdx.x * TAG_THREADS + threadIdx.x;
  bool flag = false, degenerate = false;
  if (t < n_tets) {
    int4 q = __ldg(tets + t);
    double Dm[3][3], M[3][3], Dp[3][3], Dc[3][3], Gp[3][3], Gc[3][3];
    edge_matrix(X, q, Dm);
    if (!inverse3(Dm, M)) {
      degenerate = true;
      flag = true;
      if (tet_norm) tet_norm[t] = __longlong_as_double(0x7ff8000000000000ll);  // NaN
    } else {
      edge_matrix(xp, q, Dp);
      edge_matrix(xc, q, Dc);
      green(Dp, M, Gp);
      green(Dc, M, Gc);
      double s2 = 0.0;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double d = ds(Gc[r][c], Gp[r][c]);
          s2 = da(s2, dm(d, d));
        }
      double n = __dsqrt_rn(s2);
      flag = n > theta;
      if (tet_norm) tet_norm[t] = n;
    }
    if (flag) {
      const int4 *s = tet_slots + 3 * t;
      int4 s0 = __ldg(s), s1 = __ldg(s + 1), s2v = __ldg(s + 2);
      // slot -1: the edge is not owned at both ends on this rank (partitioned mesh, 8(e))
      const int sl[12] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w, s2v.x, s2v.y, s2v.z, s2v.w};
#pragma unroll
      for (int k = 0; k < 12; ++k)
        if (sl[k] >= 0) slot_tags[sl[k]] = 0;
    }
  }
  if (counters) {
    unsigned fb = __ballot_sync(FULL_MASK, flag);
    unsigned db = __ballot_sync(FULL_MASK, degenerate);
    if (lane_id() == 0) {
      if (fb) atomicAdd(counters, (unsigned long long)__popc(fb));
      if (db) atomicAdd(counters + 1, (unsigned long long)__popc(db));
    }
  }
}

extern "C" agipc_status agipc_tag_edges(agipc_handle h, const agipc_mesh *mesh, const double *x_prev,
                                        const double *x_cur, double threshold, uint8_t *slot_tags,
                                        double *tet_norm, int64_t *n_flagged) {
  if (!h) return AGIPC_EINVAL;
  if (!mesh || mesh->n_tets < 0 || mesh->nnz_adj < 0 || mesh->n_nodes < 0)
    return set_err(h, AGIPC_EINVAL, "tag_edges: bad mesh");
  if (mesh->n_tets > 0 && (!mesh->tets || !mesh->tet_slots || !mesh->x_rest || !x_prev || !x_cur))
    return set_err(h, AGIPC_EINVAL, "tag_edges: null input");
  if (mesh->nnz_adj > 0 && !slot_tags) return set_err(h, AGIPC_EINVAL, "tag_edges: null slot_tags");
  if (((uintptr_t)mesh->tets & 15) || ((uintptr_t)mesh->tet_slots & 15))
    return set_err(h, AGIPC_EINVAL, "tag_edges: tets/tet_slots must be 16-byte aligned");
  if (mesh->n_nodes >= INT32_MAX || mesh->nnz_adj >= INT32_MAX)
    return set_err(h, AGIPC_ERANGE, "tag_edges: index exceeds int32");
  CU_TRY(h, cudaSetDevice(h->device));
  ProfScope prof_scope(h, PROF_TAG, h->stream);
  if (mesh->nnz_adj > 0) CU_TRY(h, cudaMemsetAsync(slot_tags, 1, (size_t)mesh->nnz_adj, h->stream));
  unsigned long long *counters = nullptr;
  if (n_flagged) {
    WS(h, c, unsigned long long, "tag_counters", 2);
    counters = c;
    CU_TRY(h, cudaMemsetAsync(counters, 0, 2 * sizeof(unsigned long long), h->stream));
  }
  int64_t blocks = cdiv(mesh->n_tets, TAG_THREADS);
  LAUNCH(h, k_tag, (unsigned)blocks, TAG_THREADS, 0, mesh->n_tets, (const int4 *)mesh->tets,
         (const int4 *)mesh->tet_slots, mesh->x_rest, x_prev, x_cur, threshold, slot_tags, tet_norm, counters);
  if (n_flagged) {
    agipc_status st;
    unsigned long long *hc = (unsigned long long *)pinned_get(h, 16, &st);
    if (st != AGIPC_OK) return st;
    CU_TRY(h, cudaMemcpyAsync(hc, counters, 16, cudaMemcpyDeviceToHost, h->stream));
    CU_TRY(h, cudaStreamSynchronize(h->stream));
    *n_flagged = (int64_t)hc[0];
    if (hc[1]) return set_err(h, AGIPC_EDEGENERATE, "tag_edges: %llu tets with det(D_m) == 0", hc[1]);
  }
  return AGIPC_OK;
}

// ---------------------------------------------------------------------------------------------
// NEXT#4 -- shells (triangles) and rods (edges), "applicable to various element types
// (shells, volumes, rods)".  Same fixed operation order as the oracle (R12):
//   triangle: t1 = e1 (1/|e1|), n = (e1 x e2)(1/|e1 x e2|), t2 = n x t1, D_m = [t_r . e_c],
//             D_m^-1 = adj(D_m) (1/det), F = D_s D_m^-1 (3x2), G = 0.5 (F^T F - I_2);
//   rod:      F = |x_b - x_a| / |X_b - X_a|, G = 0.5 (F F - 1);
// n = ||G_cur - G_prev||_F; flagged iff n > theta; flags ACCUMULATE into slot_tags (the caller
// resets them once per Newton step: reset_tags, or agipc_tag_edges for a mixed mesh).
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ double dot3d(const double u[3], const double v[3]) {
  return da(da(dm(u[0], v[0]), dm(u[1], v[1])), dm(u[2], v[2]));
}
__device__ __forceinline__ void cross3d(const double u[3], const double v[3], double w[3]) {
  w[0] = ds(dm(u[1], v[2]), dm(u[2], v[1]));
  w[1] = ds(dm(u[2], v[0]), dm(u[0], v[2]));
  w[2] = ds(dm(u[0], v[1]), dm(u[1], v[0]));
}

__device__ __forceinline__ void tri_green_d(const double *__restrict__ P, int a, int b, int c, const double Mi[2][2],
                                            double G[2][2]) {
  double pa[3], pb[3], pc[3], d1[3], d2[3], F[3][2];
  load3(P, a, pa);
  load3(P, b, pb);
  load3(P, c, pc);
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    d1[r] = ds(pb[r], pa[r]);
    d2[r] = ds(pc[r], pa[r]);
  }
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 2; ++k) F[r][k] = da(dm(d1[r], Mi[0][k]), dm(d2[r], Mi[1][k]));
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double C = da(da(dm(F[0][r], F[0][k]), dm(F[1][r], F[1][k])), dm(F[2][r], F[2][k]));
      G[r][k] = dm(0.5, ds(C, r == k ? 1.0 : 0.0));
    }
}

__global__ void __launch_bounds__(TAG_THREADS) k_tag_shells(int64_t n_tris, const int32_t *__restrict__ tris,
                                                            const int32_t *__restrict__ tri_slots,
                                                            const double *__restrict__ X, const double *__restrict__ xp,
                                                            const double *__restrict__ xc, double theta,
                                                            uint8_t *__restrict__ slot_tags, double *__restrict__ norm,
                                                            unsigned long long *__restrict__ counters) {
  const int64_t t = (int64_t)blockIdx.x * TAG_THREADS + threadIdx.x;
  bool flag = false, degenerate = false;
  if (t < n_tris) {
    const int a = __ldg(tris + 3 * t), b = __ldg(tris + 3 * t + 1), c = __ldg(tris + 3 * t + 2);
    double Xa[3], Xb[3], Xc[3], e1[3], e2[3], nr[3], t1[3], t2[3];
    load3(X, a, Xa);
    load3(X, b, Xb);
    load3(X, c, Xc);
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      e1[r] = ds(Xb[r], Xa[r]);
      e2[r] = ds(Xc[r], Xa[r]);
    }
    const double L1 = __dsqrt_rn(dot3d(e1, e1));
    cross3d(e1, e2, nr);
    const double Ln = __dsqrt_rn(dot3d(nr, nr));
    double det = 0.0;
    double Dm[2][2];
    if (L1 != 0.0 && Ln != 0.0 && isfinite(L1) && isfinite(Ln)) {
      const double i1 = __ddiv_rn(1.0, L1), in = __ddiv_rn(1.0, Ln);
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        t1[r] = dm(e1[r], i1);
        nr[r] = dm(nr[r], in);
      }
      cross3d(nr, t1, t2);
      Dm[0][0] = dot3d(t1, e1); Dm[0][1] = dot3d(t1, e2);
      Dm[1][0] = dot3d(t2, e1); Dm[1][1] = dot3d(t2, e2);
      det = ds(dm(Dm[0][0], Dm[1][1]), dm(Dm[0][1], Dm[1][0]));
    }
    if (det == 0.0 || !isfinite(det)) {
      degenerate = true;
      flag = true;
      if (norm) norm[t] = __longlong_as_double(0x7ff8000000000000ll);
    } else {
      const double id = __ddiv_rn(1.0, det);
      const double Mi[2][2] = {{dm(Dm[1][1], id), dm(-Dm[0][1], id)}, {dm(-Dm[1][0], id), dm(Dm[0][0], id)}};
      double Gp[2][2], Gc[2][2];
      tri_green_d(xp, a, b, c, Mi, Gp);
      tri_green_d(xc, a, b, c, Mi, Gc);
      double s2 = 0.0;
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const double d = ds(Gc[r][k], Gp[r][k]);
          s2 = da(s2, dm(d, d));
        }
      const double n = __dsqrt_rn(s2);
      flag = n > theta;
      if (norm) norm[t] = n;
    }
    if (flag)
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const int sl = __ldg(tri_slots + 6 * t + k);
        if (sl >= 0) slot_tags[sl] = 0;
      }
  }
  if (counters) {
    const unsigned fb = __ballot_sync(FULL_MASK, flag), db = __ballot_sync(FULL_MASK, degenerate);
    if (lane_id() == 0) {
      if (fb) atomicAdd(counters, (unsigned long long)__popc(fb));
      if (db) atomicAdd(counters + 1, (unsigned long long)__popc(db));
    }
  }
}

__global__ void __launch_bounds__(TAG_THREADS) k_tag_rods(int64_t n_segs, const int32_t *__restrict__ segs,
                                                          const int32_t *__restrict__ seg_slots,
                                                          const double *__restrict__ X, const double *__restrict__ xp,
                                                          const double *__restrict__ xc, double theta,
                                                          uint8_t *__restrict__ slot_tags, double *__restrict__ norm,
                                                          unsigned long long *__restrict__ counters) {
  const int64_t t = (int64_t)blockIdx.x * TAG_THREADS + threadIdx.x;
  bool flag = false, degenerate = false;
  if (t < n_segs) {
    const int a = __ldg(segs + 2 * t), b = __ldg(segs + 2 * t + 1);
    double A[3], B[3], dR[3], dp[3], dc[3];
    load3(X, a, A);
    load3(X, b, B);
#pragma unroll
    for (int r = 0; r < 3; ++r) dR[r] = ds(B[r], A[r]);
    load3(xp, a, A);
    load3(xp, b, B);
#pragma unroll
    for (int r = 0; r < 3; ++r) dp[r] = ds(B[r], A[r]);
    load3(xc, a, A);
    load3(xc, b, B);
#pragma unroll
    for (int r = 0; r < 3; ++r) dc[r] = ds(B[r], A[r]);
    const double L = __dsqrt_rn(dot3d(dR, dR));
    if (L == 0.0 || !isfinite(L)) {
      degenerate = true;
      flag = true;
      if (norm) norm[t] = __longlong_as_double(0x7ff8000000000000ll);
    } else {
      const double Fp = __ddiv_rn(__dsqrt_rn(dot3d(dp, dp)), L), Fc = __ddiv_rn(__dsqrt_rn(dot3d(dc, dc)), L);
      const double Gp = dm(0.5, ds(dm(Fp, Fp), 1.0)), Gc = dm(0.5, ds(dm(Fc, Fc), 1.0));
      const double n = fabs(ds(Gc, Gp));
      flag = n > theta;
      if (norm) norm[t] = n;
    }
    if (flag)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int sl = __ldg(seg_slots + 2 * t + k);
        if (sl >= 0) slot_tags[sl] = 0;
      }
  }
  if (counters) {
    const unsigned fb = __ballot_sync(FULL_MASK, flag), db = __ballot_sync(FULL_MASK, degenerate);
    if (lane_id() == 0) {
      if (fb) atomicAdd(counters, (unsigned long long)__popc(fb));
      if (db) atomicAdd(counters + 1, (unsigned long long)__popc(db));
    }
  }
}

template <typename K>
static agipc_status tag_elements(agipc_handle h, const char *who, K kernel, int64_t n_el, const int32_t *el,
                                 const int32_t *el_slots, const double *x_rest, const double *x_prev,
                                 const double *x_cur, double threshold, int64_t nnz_adj, int reset_tags,
                                 uint8_t *slot_tags, double *norm, int64_t *n_flagged) {
  if (!h) return AGIPC_EINVAL;
  if (n_el < 0 || nnz_adj < 0) return set_err(h, AGIPC_EINVAL, "%s: negative size", who);
  if ((nnz_adj > 0 && !slot_tags) || (n_el > 0 && (!el || !el_slots || !x_rest || !x_prev || !x_cur)))
    return set_err(h, AGIPC_EINVAL, "%s: null input", who);
  if (nnz_adj >= INT32_MAX) return set_err(h, AGIPC_ERANGE, "%s: index exceeds int32", who);
  CU_TRY(h, cudaSetDevice(h->device));
  ProfScope prof_scope(h, PROF_TAG, h->stream);
  if (reset_tags && nnz_adj > 0) CU_TRY(h, cudaMemsetAsync(slot_tags, 1, (size_t)nnz_adj, h->stream));
  if (n_flagged) *n_flagged = 0;
  if (n_el == 0) return AGIPC_OK;
  unsigned long long *counters = nullptr;
  if (n_flagged) {
    WS(h, c, unsigned long long, "tag_counters", 2);
    counters = c;
    CU_TRY(h, cudaMemsetAsync(counters, 0, 2 * sizeof(unsigned long long), h->stream));
  }
  LAUNCH(h, kernel, (unsigned)cdiv(n_el, TAG_THREADS), TAG_THREADS, 0, n_el, el, el_slots, x_rest, x_prev, x_cur,
         threshold, slot_tags, norm, counters);
  if (n_flagged) {
    agipc_status st;
    unsigned long long *hc = (unsigned long long *)pinned_get(h, 16, &st);
    if (st != AGIPC_OK) return st;
    CU_TRY(h, cudaMemcpyAsync(hc, counters, 16, cudaMemcpyDeviceToHost, h->stream));
    CU_TRY(h, cudaStreamSynchronize(h->stream));
    *n_flagged = (int64_t)hc[0];
    if (hc[1]) return set_err(h, AGIPC_EDEGENERATE, "%s: %llu degenerate elements", who, hc[1]);
  }
  return AGIPC_OK;
}

extern "C" agipc_status agipc_tag_shells(agipc_handle h, int64_t n_tris, const int32_t *tris, const int32_t *tri_slots,
                                         const double *x_rest, const double *x_prev, const double *x_cur,
                                         double threshold, int64_t nnz_adj, int reset_tags, uint8_t *slot_tags,
                                         double *tri_norm, int64_t *n_flagged) {
  return tag_elements(h, "tag_shells", k_tag_shells, n_tris, tris, tri_slots, x_rest, x_prev, x_cur, threshold,
                      nnz_adj, reset_tags, slot_tags, tri_norm, n_flagged);
}

extern "C" agipc_status agipc_tag_rods(agipc_handle h, int64_t n_segs, const int32_t *segs, const int32_t *seg_slots,
                                       const double *x_rest, const double *x_prev, const double *x_cur,
                                       double threshold, int64_t nnz_adj, int reset_tags, uint8_t *slot_tags,
                                       double *seg_norm, int64_t *n_flagged) {
  return tag_elements(h, "tag_rods", k_tag_rods, n_segs, segs, seg_slots, x_rest, x_prev, x_cur, threshold, nnz_adj,
                      reset_tags, slot_tags, seg_norm, n_flagged);
}
