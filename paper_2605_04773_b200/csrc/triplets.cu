// NEXT#3 -- fine-level hash reduction (supp Sec 2): unreduced Hessian
// triplets (i, j, B_ij), key (i << 32) | j, sorted by key with equal keys in input order, each
// run of equal keys summed in that order -> unique BSR.
//
// B200 design: the topology is static, so the key sort is done ONCE per mesh as a plan
// and every Newton step only streams the values:
//   plan:   counting sort of the triplet ids by row (histogram, scan, scatter), then one warp
//           per row sorts its bucket by (j, id) in shared memory (bitonic; a CTA-wide
//           global-memory sort for rows longer than TP_WARP_CAP), marks the runs of equal j and
//           writes the row's unique columns and the run starts (seg_ptr); the sorted buckets
//           ARE seg_idx;
//   reduce: thread per unique block, sequential in-order sum of its triplets (bit-identical
//           to the oracle's order, no atomics).
#include <climits>

#include "agipc_internal.cuh"

#define TP_WARPS 8
#define TP_WARP_CAP 512

__global__ void k_tp_hist(int64_t n, const int32_t *__restrict__ ti, const int32_t *__restrict__ tj, int64_t n_rows,
                          int *__restrict__ cnt, int *__restrict__ bad) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = ti[t], j = tj[t];
    if (i < 0 || i >= n_rows || j < 0) {
      atomicOr(bad, 1);
      continue;
    }
    atomicAdd(cnt + i, 1);
  }
}

__global__ void k_tp_scatter(int64_t n, int64_t n_rows, const int32_t *__restrict__ ti, const int64_t *__restrict__ rstart,
                             int *__restrict__ cur, int32_t *__restrict__ bucket) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = ti[t];
    if (i < 0 || i >= n_rows) continue;  // flagged by k_tp_hist (EINVAL before any use)
    bucket[rstart[i] + atomicAdd(cur + i, 1)] = (int32_t)t;
  }
}

// sort the row's bucket by key (j << 32 | id); count unique j.  PASS 0: rowlen; PASS 1: col,
// seg_ptr (and the sorted bucket, written back in pass 0 already).
template <int PASS>
__global__ void __launch_bounds__(TP_WARPS * 32) k_tp_rows(int64_t n_rows, const int64_t *__restrict__ rstart,
                                                          int32_t *__restrict__ bucket, const int32_t *__restrict__ tj,
                                                          int32_t *__restrict__ rowlen, const int64_t *__restrict__ row_ptr,
                                                          int32_t *__restrict__ col, int64_t *__restrict__ seg_ptr,
                                                          int32_t *__restrict__ big_rows, int *__restrict__ n_big) {
  __shared__ unsigned long long s_key[TP_WARPS][TP_WARP_CAP];
  const int w = threadIdx.x >> 5, l = lane_id();
  unsigned long long *key = s_key[w];
  for (int64_t r = (int64_t)blockIdx.x * TP_WARPS + w; r < n_rows; r += (int64_t)gridDim.x * TP_WARPS) {
    const int64_t b0 = rstart[r];
    const int n = (int)(rstart[r + 1] - b0);
    if (n > TP_WARP_CAP) {
      if (PASS == 0 && l == 0) big_rows[atomicAdd(n_big, 1)] = (int32_t)r;
      continue;
    }
    int P = 1;
    while (P < n) P <<= 1;
    if (PASS == 0) {
      for (int e = l; e < P; e += 32) {
        unsigned long long k = ~0ull;
        if (e < n) {
          const int t = bucket[b0 + e];
          k = ((unsigned long long)(unsigned)tj[t] << 32) | (unsigned)t;
        }
        key[e] = k;
      }
      __syncwarp();
      for (int kk = 2; kk <= P; kk <<= 1)
        for (int j = kk >> 1; j > 0; j >>= 1) {
          for (int i = l; i < P; i += 32) {
            const int ixj = i ^ j;
            if (ixj > i) {
              const unsigned long long x = key[i], y = key[ixj];
              if ((x > y) == ((i & kk) == 0)) {
                key[i] = y;
                key[ixj] = x;
              }
            }
          }
          __syncwarp();
        }
      int u = 0;
      for (int e0 = 0; e0 < n; e0 += 32) {
        const int e = e0 + l;
        const bool head = e < n && (e == 0 || (key[e - 1] >> 32) != (key[e] >> 32));
        u += __popc(__ballot_sync(FULL_MASK, head));
        if (e < n) bucket[b0 + e] = (int32_t)(key[e] & 0xffffffffull);
      }
      if (l == 0) rowlen[r] = u;
    } else {
      int base = 0;
      for (int e0 = 0; e0 < n; e0 += 32) {
        const int e = e0 + l;
        bool head = false;
        int j = 0;
        if (e < n) {
          j = tj[bucket[b0 + e]];
          head = e == 0 || tj[bucket[b0 + e - 1]] != j;
        }
        const unsigned hb = __ballot_sync(FULL_MASK, head);
        if (head) {
          const int64_t u = row_ptr[r] + base + __popc(hb & ((1u << l) - 1u));
          col[u] = j;
          seg_ptr[u] = b0 + e;
        }
        base += __popc(hb);
      }
    }
    __syncwarp();
  }
}

// rows longer than TP_WARP_CAP: one CTA, bitonic sort in global memory (a scratch copy of keys)
__global__ void __launch_bounds__(1024) k_tp_big(const int32_t *__restrict__ big_rows, const int *__restrict__ n_big,
                                                 const int64_t *__restrict__ rstart, int32_t *__restrict__ bucket,
                                                 const int32_t *__restrict__ tj, unsigned long long *__restrict__ scratch,
                                                 int32_t *__restrict__ rowlen) {
  __shared__ int s_u;
  for (int q = blockIdx.x; q < *n_big; q += gridDim.x) {
    const int64_t r = big_rows[q];
    const int64_t b0 = rstart[r];
    const int n = (int)(rstart[r + 1] - b0);
    int P = 1;
    while (P < n) P <<= 1;
    unsigned long long *key = scratch + b0 * 2;  // scratch holds 2 * n_trip keys: room for P <= 2n
    for (int e = threadIdx.x; e < P; e += blockDim.x) {
      unsigned long long k = ~0ull;
      if (e < n) {
        const int t = bucket[b0 + e];
        k = ((unsigned long long)(unsigned)tj[t] << 32) | (unsigned)t;
      }
      key[e] = k;
    }
    __syncthreads();
    for (int kk = 2; kk <= P; kk <<= 1)
      for (int j = kk >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < P; i += blockDim.x) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const unsigned long long x = key[i], y = key[ixj];
            if ((x > y) == ((i & kk) == 0)) {
              key[i] = y;
              key[ixj] = x;
            }
          }
        }
        __syncthreads();
      }
    if (threadIdx.x == 0) s_u = 0;
    __syncthreads();
    int u = 0;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      if (e == 0 || (key[e - 1] >> 32) != (key[e] >> 32)) ++u;
      bucket[b0 + e] = (int32_t)(key[e] & 0xffffffffull);
    }
    atomicAdd(&s_u, u);
    __syncthreads();
    if (threadIdx.x == 0) rowlen[r] = s_u;
    __syncthreads();
  }
}

__global__ void k_tp_big_cols(const int32_t *__restrict__ big_rows, const int *__restrict__ n_big,
                              const int64_t *__restrict__ rstart, const int32_t *__restrict__ bucket,
                              const int32_t *__restrict__ tj, const int64_t *__restrict__ row_ptr,
                              int32_t *__restrict__ col, int64_t *__restrict__ seg_ptr) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < *n_big; q += gridDim.x * blockDim.x) {
    const int64_t r = big_rows[q];
    const int64_t b0 = rstart[r];
    const int n = (int)(rstart[r + 1] - b0);
    int64_t u = row_ptr[r];
    for (int e = 0; e < n; ++e) {
      const int j = tj[bucket[b0 + e]];
      if (e == 0 || tj[bucket[b0 + e - 1]] != j) {
        col[u] = j;
        seg_ptr[u] = b0 + e;
        ++u;
      }
    }
  }
}

__global__ void k_tp_last(const int64_t *__restrict__ row_ptr, int64_t n_rows, int64_t n, int64_t *__restrict__ seg_ptr) {
  seg_ptr[row_ptr[n_rows]] = n;
}

extern "C" agipc_status agipc_triplet_plan(agipc_handle h, int64_t n_rows, int64_t n_trip, const int32_t *ti,
                                           const int32_t *tj, agipc_triplet_plan_t *plan) {
  if (!h) return AGIPC_EINVAL;
  if (!plan || n_rows < 0 || n_trip < 0) return set_err(h, AGIPC_EINVAL, "triplet_plan: bad arguments");
  plan->n_rows = n_rows;
  plan->n_trip = n_trip;
  plan->nnzb = 0;
  if (!plan->row_ptr) return set_err(h, AGIPC_EINVAL, "triplet_plan: null row_ptr");
  if (n_trip >= INT32_MAX || n_rows >= INT32_MAX) return set_err(h, AGIPC_ERANGE, "triplet_plan: too large");
  CU_TRY(h, cudaSetDevice(h->device));
  ProfScope prof(h, PROF_TRIPLETS, h->stream);
  cudaStream_t s = h->stream;
  if (n_trip == 0) {
    CU_TRY(h, cudaMemsetAsync(plan->row_ptr, 0, sizeof(int64_t) * (n_rows + 1), s));
    return AGIPC_OK;
  }
  if (!ti || !tj || !plan->seg_idx) return set_err(h, AGIPC_EINVAL, "triplet_plan: null pointer");
  WS(h, cnt, int, "tp_cnt", 2 * (n_rows + 1) + 2);
  WS(h, rstart, int64_t, "tp_rstart", n_rows + 1);
  WS(h, rowlen, int32_t, "tp_rowlen", n_rows + 1);
  WS(h, big, int32_t, "tp_big", n_rows + 1);
  int *cur = cnt + (n_rows + 1);
  int *flags = cnt + 2 * (n_rows + 1);  // [0] bad index, [1] number of big rows
  CU_TRY(h, cudaMemsetAsync(cnt, 0, sizeof(int) * (2 * (n_rows + 1) + 2), s));
  const unsigned G = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n_trip, 256), 16 * h->sm_count));
  LAUNCH(h, k_tp_hist, G, 256, 0, n_trip, ti, tj, n_rows, cnt, flags);
  agipc_status st = scan_exclusive_i64(h, SCAN_SRC_I32, cnt, n_rows, rstart);
  if (st != AGIPC_OK) return st;
  int32_t *bucket = plan->seg_idx;  // the sorted buckets are seg_idx
  LAUNCH(h, k_tp_scatter, G, 256, 0, n_trip, n_rows, ti, (const int64_t *)rstart, cur, bucket);
  const unsigned GR = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n_rows, TP_WARPS), 64 * h->sm_count));
  LAUNCH(h, k_tp_rows<0>, GR, TP_WARPS * 32, 0, n_rows, (const int64_t *)rstart, bucket, tj, rowlen,
         (const int64_t *)nullptr, (int32_t *)nullptr, (int64_t *)nullptr, big, flags + 1);
  int *hf = (int *)pinned_get(h, 2 * sizeof(int), &st);
  if (st != AGIPC_OK) return st;
  CU_TRY(h, cudaMemcpyAsync(hf, flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  CU_TRY(h, cudaStreamSynchronize(s));
  if (hf[0]) return set_err(h, AGIPC_EINVAL, "triplet_plan: a row index outside [0, n_rows) or a negative column");
  const int nbig = hf[1];
  if (nbig > 0) {
    WS(h, scratch, unsigned long long, "tp_scratch", 2 * n_trip + 64);
    LAUNCH(h, k_tp_big, (unsigned)std::min(nbig, 4 * h->sm_count), 1024, 0, (const int32_t *)big,
           (const int *)(flags + 1), (const int64_t *)rstart, bucket, tj, scratch, rowlen);
  }
  st = scan_exclusive_i64(h, SCAN_SRC_I32, rowlen, n_rows, plan->row_ptr);
  if (st != AGIPC_OK) return st;
  int64_t *hn = (int64_t *)pinned_get(h, sizeof(int64_t), &st);
  if (st != AGIPC_OK) return st;
  CU_TRY(h, cudaMemcpyAsync(hn, plan->row_ptr + n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CU_TRY(h, cudaStreamSynchronize(s));
  plan->nnzb = *hn;
  if (plan->nnzb > plan->cap_nnzb || !plan->col || !plan->seg_ptr)
    return set_err(h, AGIPC_ENOSPACE, "triplet_plan: %lld unique blocks > capacity %lld", (long long)plan->nnzb,
                   (long long)plan->cap_nnzb);
  LAUNCH(h, k_tp_rows<1>, GR, TP_WARPS * 32, 0, n_rows, (const int64_t *)rstart, bucket, tj, rowlen,
         (const int64_t *)plan->row_ptr, plan->col, plan->seg_ptr, big, flags + 1);
  if (nbig > 0)
    LAUNCH(h, k_tp_big_cols, (unsigned)cdiv(nbig, 128), 128, 0, (const int32_t *)big, (const int *)(flags + 1),
           (const int64_t *)rstart, (const int32_t *)bucket, tj, (const int64_t *)plan->row_ptr, plan->col,
           plan->seg_ptr);
  LAUNCH(h, k_tp_last, 1, 1, 0, (const int64_t *)plan->row_ptr, n_rows, n_trip, plan->seg_ptr);
  return AGIPC_OK;
}

// thread per unique block: in-order sum (same order as the oracle's stable sort)
__global__ void k_tp_reduce(int64_t nnzb, const int64_t *__restrict__ seg_ptr, const int32_t *__restrict__ seg_idx,
                            const double *__restrict__ tval, double *__restrict__ val) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nnzb; u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s0 = seg_ptr[u], s1 = seg_ptr[u + 1];
    double acc[9];
    const double *B = tval + 9 * (int64_t)seg_idx[s0];
#pragma unroll
    for (int e = 0; e < 9; ++e) acc[e] = __ldg(B + e);
    for (int64_t s = s0 + 1; s < s1; ++s) {
      B = tval + 9 * (int64_t)seg_idx[s];
#pragma unroll
      for (int e = 0; e < 9; ++e) acc[e] = __dadd_rn(acc[e], __ldg(B + e));
    }
#pragma unroll
    for (int e = 0; e < 9; ++e) val[9 * u + e] = acc[e];
  }
}

extern "C" agipc_status agipc_triplet_reduce(agipc_handle h, const agipc_triplet_plan_t *plan, const double *tval,
                                             double *val) {
  if (!h) return AGIPC_EINVAL;
  if (!plan) return set_err(h, AGIPC_EINVAL, "triplet_reduce: null plan");
  if (plan->nnzb == 0) return AGIPC_OK;
  if (!tval || !val || !plan->seg_ptr || !plan->seg_idx) return set_err(h, AGIPC_EINVAL, "triplet_reduce: null pointer");
  CU_TRY(h, cudaSetDevice(h->device));
  ProfScope prof(h, PROF_TRIPLETS, h->stream);
  const unsigned G = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(plan->nnzb, 256), 16 * h->sm_count));
  LAUNCH(h, k_tp_reduce, G, 256, 0, plan->nnzb, (const int64_t *)plan->seg_ptr, (const int32_t *)plan->seg_idx, tval,
         val);
  return AGIPC_OK;
}
