// Multi-GPU partitioned path: the rank-local pieces of the
// three exchanges around the coarsening step.  Communication itself is done by the caller
// (torch.distributed / NCCL); these kernels produce and consume its buffers.
//
//  agipc_gather_rows     pack rows of a device array by index (halo send buffers: x_prev /
//                        x_cur of exchange 1, ghost column codes of exchange 3)
//  agipc_coarse_halo     owner side of exchange 3: the coarse slots a peer needs, derived from
//                        the fine nodes sent to it (first-appearance order, no sort), and the
//                        column code of every sent fine node
//  agipc_assemble_halo   the Galerkin blocks of the rank's coarse rows x ghost coarse columns,
//                        H_c[slot(a,p), gslot(b)+q] = sum w_i[p] w_j[q] B_ij over fine blocks
//                        (i owned, j ghost) with new_map(i) = a and j in ghost aggregate b
//                        (supp Alg S4 + Eq 4 restricted to the cross-rank blocks, P:258-319,
//                        P:851-855; == the corresponding block of U H U^T)
#include <climits>

#include "agipc_internal.cuh"

#define GH_12 (1 << 30)         // column-code flag: the ghost aggregate is 12-DoF
#define GH_MASK (GH_12 - 1)

__global__ void k_gather_words(int64_t m, int w, const int32_t *__restrict__ idx, const uint32_t *__restrict__ src,
                               uint32_t *__restrict__ dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m * w) {
    const int64_t k = i / w, c = i - k * w;
    dst[i] = src[(int64_t)idx[k] * w + c];
  }
}

extern "C" agipc_status agipc_gather_rows(agipc_handle h, const void *src, const int32_t *idx, int64_t n,
                                          int row_bytes, void *dst) {
  if (!h) return AGIPC_EINVAL;
  if (n < 0 || row_bytes <= 0 || (row_bytes & 3)) return set_err(h, AGIPC_EINVAL, "gather_rows: bad sizes");
  if (n == 0) return AGIPC_OK;
  if (!src || !idx || !dst) return set_err(h, AGIPC_EINVAL, "gather_rows: null pointer");
  if (((uintptr_t)src & 3) || ((uintptr_t)dst & 3)) return set_err(h, AGIPC_EINVAL, "gather_rows: misaligned");
  CU_TRY(h, cudaSetDevice(h->device));
  const int w = row_bytes / 4;
  LAUNCH(h, k_gather_words, (unsigned)cdiv(n * w, 256), 256, 0, n, w, idx, (const uint32_t *)src, (uint32_t *)dst);
  return AGIPC_OK;
}

// ---------------------------------------------------------------------------------------------
// owner side of exchange 3
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ int ncb_c(int c, int64_t n3) { return c < n3 ? 1 : 4; }
__device__ __forceinline__ int64_t slot_c(int c, int p, int64_t n3) { return c < n3 ? c : n3 + 4 * ((int64_t)c - n3) + p; }

__global__ void k_ch_first(int64_t m, const int32_t *__restrict__ S, const int32_t *__restrict__ nm,
                           int *__restrict__ first) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) atomicMin(first + nm[S[k]], (int)k);
}

__global__ void k_ch_size(int64_t m, const int32_t *__restrict__ S, const int32_t *__restrict__ nm, int64_t n3,
                          const int *__restrict__ first, int32_t *__restrict__ sz) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) {
    const int c = nm[S[k]];
    sz[k] = first[c] == (int)k ? ncb_c(c, n3) : 0;
  }
}

__global__ void k_ch_emit(int64_t m, const int32_t *__restrict__ S, const int32_t *__restrict__ nm, int64_t n3,
                          const int *__restrict__ first, const int64_t *__restrict__ off, int32_t *__restrict__ info,
                          int32_t *__restrict__ slots) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) {
    const int c = nm[S[k]];
    const int f = first[c];
    info[k] = (int32_t)off[f] | (c >= n3 ? GH_12 : 0);
    if (f == (int)k)
      for (int p = 0; p < ncb_c(c, n3); ++p) slots[off[k] + p] = (int32_t)slot_c(c, p, n3);
  }
}

__global__ void k_ch_reset(int64_t m, const int32_t *__restrict__ S, const int32_t *__restrict__ nm,
                           int *__restrict__ first) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) first[nm[S[k]]] = INT_MAX;
}

__global__ void k_fill_int(int64_t n, int *p, int v) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

extern "C" agipc_status agipc_coarse_halo(agipc_handle h, const int32_t *new_map, int64_t n3, int64_t n_coarse,
                                          const int32_t *send_idx, int64_t n_send, int32_t *ghost_code,
                                          int32_t *send_slots, int64_t cap_slots, int64_t *n_slots) {
  if (!h) return AGIPC_EINVAL;
  if (!n_slots || n_send < 0 || n3 < 0 || n_coarse < n3) return set_err(h, AGIPC_EINVAL, "coarse_halo: bad arguments");
  *n_slots = 0;
  if (n_send == 0) return AGIPC_OK;
  if (!new_map || !send_idx || !ghost_code) return set_err(h, AGIPC_EINVAL, "coarse_halo: null pointer");
  if (n_send >= INT32_MAX || n3 + 4 * (n_coarse - n3) >= GH_12)
    return set_err(h, AGIPC_ERANGE, "coarse_halo: index exceeds the column code range");
  CU_TRY(h, cudaSetDevice(h->device));
  ProfScope prof(h, PROF_DIST, h->stream);
  // first[c] = first position of aggregate c in the send list; kept at INT_MAX between calls
  const size_t need = sizeof(int) * (size_t)(n_coarse + 1);
  int *first = nullptr;
  {
    agipc_status st;
    bool fresh = false;
    first = (int *)ws_get(h, "dist_first", need, &st, &fresh);
    if (st != AGIPC_OK) return st;
    const int64_t cap = (int64_t)(h->ws["dist_first"].bytes / sizeof(int));
    if (fresh) LAUNCH(h, k_fill_int, (unsigned)cdiv(cap, 256), 256, 0, cap, first, INT_MAX);
  }
  WS(h, sz, int32_t, "dist_ch_size", n_send);
  WS(h, off, int64_t, "dist_ch_off", n_send + 1);
  const unsigned G = (unsigned)cdiv(n_send, 256);
  LAUNCH(h, k_ch_first, G, 256, 0, n_send, send_idx, new_map, first);
  LAUNCH(h, k_ch_size, G, 256, 0, n_send, send_idx, new_map, n3, (const int *)first, sz);
  agipc_status st = scan_exclusive_i64(h, SCAN_SRC_I32, sz, n_send, off);
  if (st != AGIPC_OK) return st;
  int64_t *hoff = (int64_t *)pinned_get(h, sizeof(int64_t), &st);
  if (st != AGIPC_OK) return st;
  CU_TRY(h, cudaMemcpyAsync(hoff, off + n_send, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  *n_slots = *hoff;
  if (*n_slots > cap_slots || !send_slots) {
    LAUNCH(h, k_ch_reset, G, 256, 0, n_send, send_idx, new_map, first);
    return set_err(h, AGIPC_ENOSPACE, "coarse_halo: %lld slots > capacity %lld", (long long)*n_slots,
                   (long long)cap_slots);
  }
  LAUNCH(h, k_ch_emit, G, 256, 0, n_send, send_idx, new_map, n3, (const int *)first, (const int64_t *)off, ghost_code,
         send_slots);
  LAUNCH(h, k_ch_reset, G, 256, 0, n_send, send_idx, new_map, first);
  return AGIPC_OK;
}

// ---------------------------------------------------------------------------------------------
// halo-matrix assembly
// ---------------------------------------------------------------------------------------------
// ghost g of peer q (ghost range [gptr[q], gptr[q+1])) -> local column code: the peer's slot
// offset within its list + this rank's base for that peer's ghost slots
__global__ void k_ghost_cols(int64_t n_ghost, int n_peers, const int64_t *__restrict__ gptr,
                             const int64_t *__restrict__ gbase, const int32_t *__restrict__ code,
                             int32_t *__restrict__ gcol) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < n_ghost) {
    int q = 0;
    while (q + 1 < n_peers && gptr[q + 1] <= g) ++q;
    const int32_t c = code[g];
    gcol[g] = (int32_t)(gbase[q] + (c & GH_MASK)) | (c & GH_12);
  }
}

__device__ __forceinline__ unsigned long long hh_hash(unsigned long long key, unsigned long long mask) {
  return (key * 0x9E3779B97F4A7C15ull >> 17) & mask;
}

// thread per owned fine row: insert (a, column code) of every halo block into the pair set
__global__ void k_hh_insert(int64_t N, const int64_t *__restrict__ hrp, const int32_t *__restrict__ hcol,
                            const int32_t *__restrict__ nm, const int32_t *__restrict__ gcol,
                            unsigned long long *__restrict__ keys, unsigned long long mask,
                            int32_t *__restrict__ ent) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const unsigned long long a = (unsigned)nm[i];
  for (int64_t k = hrp[i]; k < hrp[i + 1]; ++k) {
    const unsigned long long key = ((a << 32) | (unsigned)gcol[hcol[k]]) + 1ull;
    unsigned long long s = hh_hash(key, mask);
    while (true) {
      const unsigned long long prev = atomicCAS(keys + s, 0ull, key);
      if (prev == 0ull || prev == key) break;
      s = (s + 1) & mask;
    }
    ent[k] = (int32_t)s;
  }
}

__global__ void k_hh_compact(unsigned long long cap, const unsigned long long *__restrict__ keys,
                             int32_t *__restrict__ pid_of, int32_t *__restrict__ pa, int32_t *__restrict__ pb,
                             int *__restrict__ cnt, unsigned long long *__restrict__ npairs) {
  unsigned long long s = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= cap) return;
  const unsigned long long key = keys[s];
  if (!key) return;
  const unsigned long long kk = key - 1ull;
  const int a = (int)(kk >> 32);
  const int id = (int)atomicAdd(npairs, 1ull);
  pid_of[s] = id;
  pa[id] = a;
  pb[id] = (int32_t)(kk & 0xffffffffull);
  atomicAdd(cnt + a, 1);
}

__global__ void k_hh_scatter(const unsigned long long *__restrict__ npairs, const int32_t *__restrict__ pa,
                             const int64_t *__restrict__ pstart, int *__restrict__ cur, int32_t *__restrict__ plist) {
  const long long np = (long long)*npairs;
  for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < np; id += (long long)gridDim.x * blockDim.x) {
    const int a = pa[id];
    plist[pstart[a] + atomicAdd(cur + a, 1)] = (int32_t)id;
  }
}

// thread per coarse node: sort its pairs by column code (insertion sort; lists are short),
// column position of each pair, row lengths of the node's 1 or 4 rows
__global__ void k_hh_rows(int64_t n_c, int64_t n3, const int64_t *__restrict__ pstart, int32_t *__restrict__ plist,
                          const int32_t *__restrict__ pb, int32_t *__restrict__ ppos, int32_t *__restrict__ rl) {
  int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n_c) return;
  const int64_t s0 = pstart[a], s1 = pstart[a + 1];
  for (int64_t u = s0 + 1; u < s1; ++u) {
    const int32_t id = plist[u];
    const int32_t key = pb[id] & GH_MASK;
    int64_t v = u - 1;
    while (v >= s0 && (pb[plist[v]] & GH_MASK) > key) {
      plist[v + 1] = plist[v];
      --v;
    }
    plist[v + 1] = id;
  }
  int32_t cp = 0;
  for (int64_t u = s0; u < s1; ++u) {
    const int32_t id = plist[u];
    ppos[id] = cp;
    cp += (pb[id] & GH_12) ? 4 : 1;
  }
  for (int p = 0; p < ncb_c((int)a, n3); ++p) rl[slot_c((int)a, p, n3)] = cp;
}

__global__ void k_hh_cols(int64_t n_c, int64_t n3, const int64_t *__restrict__ pstart, const int32_t *__restrict__ plist,
                          const int32_t *__restrict__ pb, const int64_t *__restrict__ rp, int32_t *__restrict__ col) {
  int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n_c) return;
  const int64_t s0 = pstart[a], s1 = pstart[a + 1];
  if (s0 == s1) return;
  for (int p = 0; p < ncb_c((int)a, n3); ++p) {
    int64_t o = rp[slot_c((int)a, p, n3)];
    for (int64_t u = s0; u < s1; ++u) {
      const int32_t b = pb[plist[u]];
      const int nq = (b & GH_12) ? 4 : 1;
      for (int q = 0; q < nq; ++q) col[o++] = (b & GH_MASK) + q;
    }
  }
}

// thread per halo block: add (w_i[p] w_j[q]) B into every coarse sub-block it feeds
__global__ void k_hh_numeric(int64_t N, int64_t n3, const int64_t *__restrict__ hrp, const int32_t *__restrict__ hcol,
                             const double *__restrict__ hval, const int32_t *__restrict__ nm,
                             const int32_t *__restrict__ gcol, const double *__restrict__ X,
                             const int32_t *__restrict__ ent, const int32_t *__restrict__ pid_of,
                             const int32_t *__restrict__ ppos, const int64_t *__restrict__ rp,
                             double *__restrict__ val) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int a = nm[i];
  const int na = ncb_c(a, n3);
  double wi[4] = {1.0, 0.0, 0.0, 0.0};
  if (na == 4) {
    wi[0] = X[3 * i]; wi[1] = X[3 * i + 1]; wi[2] = X[3 * i + 2]; wi[3] = 1.0;
  }
  for (int64_t k = hrp[i]; k < hrp[i + 1]; ++k) {
    const int j = hcol[k];
    const int32_t code = gcol[j];
    const int nb = (code & GH_12) ? 4 : 1;
    double wj[4] = {1.0, 0.0, 0.0, 0.0};
    if (nb == 4) {
      const int64_t jj = N + j;
      wj[0] = X[3 * jj]; wj[1] = X[3 * jj + 1]; wj[2] = X[3 * jj + 2]; wj[3] = 1.0;
    }
    const int32_t cp = ppos[pid_of[ent[k]]];
    double B[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) B[e] = hval[9 * k + e];
    for (int p = 0; p < na; ++p) {
      const int64_t o = rp[slot_c(a, p, n3)] + cp;
      for (int q = 0; q < nb; ++q) {
        const double c = wi[p] * wj[q];
        double *dst = val + 9 * (o + q);
#pragma unroll
        for (int e = 0; e < 9; ++e) atomicAdd(dst + e, c * B[e]);
      }
    }
  }
}

extern "C" agipc_status agipc_assemble_halo(agipc_handle h, const agipc_mesh *mesh, const int32_t *new_map, int64_t n3,
                                            int64_t n_coarse, const agipc_bsr *H_halo, int64_t n_ghost,
                                            const int32_t *ghost_code, int n_peers, const int64_t *peer_ghost_ptr,
                                            const int64_t *peer_slot_base, agipc_halo_matrix *out) {
  if (!h) return AGIPC_EINVAL;
  if (!mesh || !H_halo || !out || n3 < 0 || n_coarse < n3 || n_ghost < 0 || n_peers < 0 ||
      H_halo->n_rows != mesh->n_nodes)
    return set_err(h, AGIPC_EINVAL, "assemble_halo: bad arguments");
  const int64_t N = mesh->n_nodes, nh = H_halo->nnzb;
  const int64_t n_slots = n3 + 4 * (n_coarse - n3);
  out->n_rows = n_slots;
  out->nnzb = 0;
  if (N == 0) return AGIPC_OK;
  if (n_ghost > 0 && (!ghost_code || n_peers < 1 || !peer_ghost_ptr || !peer_slot_base))
    return set_err(h, AGIPC_EINVAL, "assemble_halo: ghost description missing");
  if (!new_map || !H_halo->row_ptr || (nh > 0 && (!H_halo->col || !H_halo->val || !mesh->x_rest)) || !out->row_ptr)
    return set_err(h, AGIPC_EINVAL, "assemble_halo: null pointer");
  if (nh >= INT32_MAX || n_slots >= GH_12) return set_err(h, AGIPC_ERANGE, "assemble_halo: too large");
  CU_TRY(h, cudaSetDevice(h->device));
  ProfScope prof(h, PROF_DIST, h->stream);
  cudaStream_t s = h->stream;
  agipc_status st;
  if (nh == 0) {
    CU_TRY(h, cudaMemsetAsync(out->row_ptr, 0, sizeof(int64_t) * (n_slots + 1), s));
    return AGIPC_OK;
  }
  for (int q = 0; q < n_peers; ++q)
    if (peer_slot_base[q] + (peer_ghost_ptr[q + 1] - peer_ghost_ptr[q]) * 4 >= GH_12)
      return set_err(h, AGIPC_ERANGE, "assemble_halo: ghost slot index too large");
  WS(h, gcol, int32_t, "dist_gcol", n_ghost + 1);
  WS(h, dptr, int64_t, "dist_peer_tab", 2 * n_peers + 2);
  {
    int64_t *ht = (int64_t *)pinned_get(h, sizeof(int64_t) * (2 * n_peers + 2), &st);
    if (st != AGIPC_OK) return st;
    for (int q = 0; q <= n_peers; ++q) ht[q] = peer_ghost_ptr[q];
    for (int q = 0; q < n_peers; ++q) ht[n_peers + 1 + q] = peer_slot_base[q];
    CU_TRY(h, cudaMemcpyAsync(dptr, ht, sizeof(int64_t) * (2 * n_peers + 1), cudaMemcpyHostToDevice, s));
    LAUNCH(h, k_ghost_cols, (unsigned)cdiv(n_ghost, 256), 256, 0, n_ghost, n_peers, (const int64_t *)dptr,
           (const int64_t *)(dptr + n_peers + 1), ghost_code, gcol);
    CU_TRY(h, cudaStreamSynchronize(s));  // the pinned table is reused below
  }
  unsigned long long cap = 1024;
  while (cap < 2ull * (unsigned long long)nh) cap <<= 1;
  WS(h, keys, unsigned long long, "dist_hh_keys", cap);
  WS(h, pid_of, int32_t, "dist_hh_pid", cap);
  WS(h, ent, int32_t, "dist_hh_ent", nh);
  WS(h, pa, int32_t, "dist_hh_pa", nh);
  WS(h, pb, int32_t, "dist_hh_pb", nh);
  WS(h, ppos, int32_t, "dist_hh_ppos", nh);
  WS(h, plist, int32_t, "dist_hh_plist", nh);
  WS(h, cnt, int, "dist_hh_cnt", 2 * (n_coarse + 1));
  WS(h, pstart, int64_t, "dist_hh_pstart", n_coarse + 1);
  WS(h, rl, int32_t, "dist_hh_rl", n_slots + 1);
  WS(h, np, unsigned long long, "dist_hh_np", 1);
  int *cur = cnt + (n_coarse + 1);
  CU_TRY(h, cudaMemsetAsync(keys, 0, sizeof(unsigned long long) * cap, s));
  CU_TRY(h, cudaMemsetAsync(cnt, 0, sizeof(int) * 2 * (n_coarse + 1), s));
  CU_TRY(h, cudaMemsetAsync(rl, 0, sizeof(int32_t) * (n_slots + 1), s));
  CU_TRY(h, cudaMemsetAsync(np, 0, sizeof(unsigned long long), s));
  const unsigned GN = (unsigned)cdiv(N, 256), GC = (unsigned)cdiv(n_coarse, 256);
  LAUNCH(h, k_hh_insert, GN, 256, 0, N, H_halo->row_ptr, H_halo->col, new_map, (const int32_t *)gcol, keys, cap - 1, ent);
  LAUNCH(h, k_hh_compact, (unsigned)cdiv((int64_t)cap, 256), 256, 0, cap, (const unsigned long long *)keys, pid_of, pa,
         pb, cnt, np);
  st = scan_exclusive_i64(h, SCAN_SRC_I32, cnt, n_coarse, pstart);
  if (st != AGIPC_OK) return st;
  LAUNCH(h, k_hh_scatter, (unsigned)std::min<int64_t>(cdiv(nh, 256), 8 * h->sm_count), 256, 0,
         (const unsigned long long *)np, (const int32_t *)pa, (const int64_t *)pstart, cur, plist);
  LAUNCH(h, k_hh_rows, GC, 256, 0, n_coarse, n3, (const int64_t *)pstart, plist, (const int32_t *)pb, ppos, rl);
  st = scan_exclusive_i64(h, SCAN_SRC_I32, rl, n_slots, out->row_ptr);
  if (st != AGIPC_OK) return st;
  int64_t *hn = (int64_t *)pinned_get(h, sizeof(int64_t), &st);
  if (st != AGIPC_OK) return st;
  CU_TRY(h, cudaMemcpyAsync(hn, out->row_ptr + n_slots, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CU_TRY(h, cudaStreamSynchronize(s));
  out->nnzb = *hn;
  if (out->nnzb > out->cap_nnzb || !out->col || !out->val)
    return set_err(h, AGIPC_ENOSPACE, "assemble_halo: %lld blocks > capacity %lld", (long long)out->nnzb,
                   (long long)out->cap_nnzb);
  LAUNCH(h, k_hh_cols, GC, 256, 0, n_coarse, n3, (const int64_t *)pstart, (const int32_t *)plist, (const int32_t *)pb,
         (const int64_t *)out->row_ptr, out->col);
  CU_TRY(h, cudaMemsetAsync(out->val, 0, sizeof(double) * 9 * out->nnzb, s));
  LAUNCH(h, k_hh_numeric, GN, 256, 0, N, n3, H_halo->row_ptr, H_halo->col, H_halo->val, new_map,
         (const int32_t *)gcol, mesh->x_rest, (const int32_t *)ent, (const int32_t *)pid_of, (const int32_t *)ppos,
         (const int64_t *)out->row_ptr, out->val);
  return AGIPC_OK;
}
