// NEXT#1 -- prolongation d_f = alpha * U^T x_c (main Sec 4.3; the adjoint of the
// restriction g_c = U g of assemble.cu, supp Eq S2/S3 P:298-319, main Eq 4).
//
// One thread per fine node: read new_map[f] and (for a 12-DoF parent) X_bar_f, gather the parent's
// 1 or 4 coarse 3-vectors, write the 3-vector d_f[f].  HBM-bound, 28 B read + 24 B written per
// node plus the coarse gathers (L2-resident: the coarse vector is n_slots*24 B ~ 6 MB at C3).
// The summation order is w0*x0 + w1*x1 + w2*x2 + x3 with explicit rn intrinsics.
#include "agipc_internal.cuh"

#define PROLONG_THREADS 256

__global__ void __launch_bounds__(PROLONG_THREADS) k_prolongate(int64_t N, const int32_t *__restrict__ nm,
                                                                 int64_t n3, int64_t n_par,
                                                                 const double *__restrict__ X,
                                                                 const double *__restrict__ xc, double alpha,
                                                                 double *__restrict__ df, int *__restrict__ bad) {
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= N) return;
  int64_t c = __ldg(nm + f);
  double s0, s1, s2;
  if (c < 0 || c >= n_par) {
    atomicOr(bad, 1);
    return;
  }
  if (c < n3) {
    const double *p = xc + 3 * c;
    s0 = __ldg(p); s1 = __ldg(p + 1); s2 = __ldg(p + 2);
  } else {
    const double *p = xc + 3 * (n3 + 4 * (c - n3));
    double w0 = __ldg(X + 3 * f), w1 = __ldg(X + 3 * f + 1), w2 = __ldg(X + 3 * f + 2);
    s0 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(w0, __ldg(p)), __dmul_rn(w1, __ldg(p + 3))),
                             __dmul_rn(w2, __ldg(p + 6))), __ldg(p + 9));
    s1 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(w0, __ldg(p + 1)), __dmul_rn(w1, __ldg(p + 4))),
                             __dmul_rn(w2, __ldg(p + 7))), __ldg(p + 10));
    s2 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(w0, __ldg(p + 2)), __dmul_rn(w1, __ldg(p + 5))),
                             __dmul_rn(w2, __ldg(p + 8))), __ldg(p + 11));
  }
  double *o = df + 3 * f;
  o[0] = __dmul_rn(alpha, s0);
  o[1] = __dmul_rn(alpha, s1);
  o[2] = __dmul_rn(alpha, s2);
}

extern "C" agipc_status agipc_prolongate(agipc_handle h, const agipc_mesh *mesh, const int32_t *new_map,
                                         int64_t n3, int64_t n_slots, const double *x_c, double alpha,
                                         double *d_f) {
  if (!h) return AGIPC_EINVAL;
  if (!mesh || mesh->n_nodes < 0) return set_err(h, AGIPC_EINVAL, "prolongate: bad mesh");
  if (n3 < 0 || n_slots < n3 || (n_slots - n3) % 4) return set_err(h, AGIPC_EINVAL, "prolongate: bad n3/n_slots");
  int64_t N = mesh->n_nodes;
  if (N == 0) return AGIPC_OK;
  if (!new_map || !x_c || !d_f || (n_slots > n3 && !mesh->x_rest))
    return set_err(h, AGIPC_EINVAL, "prolongate: null input");
  if (N >= INT32_MAX || n_slots >= INT32_MAX) return set_err(h, AGIPC_ERANGE, "prolongate: index exceeds int32");
  CU_TRY(h, cudaSetDevice(h->device));
  ProfScope prof_scope(h, PROF_PROLONG, h->stream);
  WS(h, bad, int, "prolong_bad", 1);
  CU_TRY(h, cudaMemsetAsync(bad, 0, sizeof(int), h->stream));
  int64_t n_par = n3 + (n_slots - n3) / 4;
  LAUNCH(h, k_prolongate, (unsigned)cdiv(N, PROLONG_THREADS), PROLONG_THREADS, 0, N, new_map, n3, n_par,
         mesh->x_rest, x_c, alpha, d_f, bad);
  agipc_status st;
  int *hb = (int *)pinned_get(h, sizeof(int), &st);
  if (st != AGIPC_OK) return st;
  CU_TRY(h, cudaMemcpyAsync(hb, bad, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  if (*hb) return set_err(h, AGIPC_EINVAL, "prolongate: new_map entry outside [0, %lld)", (long long)n_par);
  return AGIPC_OK;
}
