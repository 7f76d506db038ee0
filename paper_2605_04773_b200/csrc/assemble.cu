// Step 3 -- DoF classification + reorder (supp Alg S3) and the Galerkin
// coarse Hessian / gradient with affine 12-DoF nodes (supp Alg S4 + Eq S2/S3, P:258-319;
// main Eq 4; H_c = U H_f U^T, g_c = U g_f).
//
// The paper flattens every transformed fine block into 1/4/16 BCOO triplets, sorts them by a
// 64-bit key and segment-reduces.  On B200 the sort and the
// flattened triplet array are the dominant HBM traffic, so this implementation is sort-free
// and row-centric:
//   A  classify: aggregate sizes, 12-DoF iff size > threshold, stable 3-DoF-first reorder by
//      a prefix sum (no SortPairs), new_map, children lists (CSR over coarse nodes);
//   B  symbolic: the sorted set of coarse neighbours of every coarse node.
//      Small nodes (<= 32 children, <= 2048 candidate entries): one warp gathers
//      new_map[col] of its children's rows into shared memory, bitonic-sorts and uniques it.
//      Large nodes: 32-children chunks emit their large-node neighbours; small nodes emit the
//      transposed (large, small) pairs; a per-node sort-unique merges them;
//   C  slot row pointer by a prefix sum of expanded row lengths (Eq S2/S3: 12-DoF columns
//      take 4 consecutive slots);
//   D  numeric: one warp per small coarse row accumulates w_i[p] w_j[q] B_ij in shared memory
//      and writes its row, and the mirrored blocks of its (small,large) pairs into the large
//      rows (B_ji = B_ij^T: each mixed pair is read once); large rows are processed by 32-child
//      chunks that keep the 12x12 diagonal block in registers (lane = (block group, p)) and
//      flush it with one fp64 atomic per entry per chunk.
#include <climits>

#include "agipc_internal.cuh"

#define SMALL_CHILDREN 32
#define SMALL_ENTRIES 2048
#define SYM_WARPS 4
#define NUM_WARPS 4
#define LIST_CAP 512
#define ACC_CAP 1024
#define LARGE_CHUNK 32

struct AsmScal {
  long long n3, n12, n_slots, nnzb;
  long long nbs_count;   // entries used in the small-node neighbour buffer
  long long pair_count;  // (large, x) pairs
  long long big_groups;  // large lists that need the CTA sort
  int err_map;           // map value outside [0, n_c)
  int err_overflow;      // a buffer capacity was exceeded
};

__device__ __forceinline__ int slot_of(int c, int p, long long n3) {
  return c < n3 ? c : (int)(n3 + 4 * ((long long)c - n3) + p);
}
__device__ __forceinline__ int ncb_of(int c, long long n3) { return c < n3 ? 1 : 4; }
__device__ __forceinline__ double wgt(const double *__restrict__ X, int f, int ncb, int p) {
  return ncb == 1 ? 1.0 : (p < 3 ? __ldg(X + 3 * (int64_t)f + p) : 1.0);
}
template <typename T>
__device__ __forceinline__ int lower_bound_dev(const T *a, int n, T key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}
// column position (in blocks) of list entry idx: every 12-DoF column before it expands to 4
__device__ __forceinline__ int colpos(int idx, int first12) { return idx + 3 * max(0, idx - first12); }

// ------------------------------------------------------------------------------------
// A. classification
// ------------------------------------------------------------------------------------
__global__ void k_size_hist(int64_t N, const int32_t *__restrict__ map, int64_t n_c, int32_t *__restrict__ size,
                            AsmScal *sc) {
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int key = -1;
  if (f < N) {
    key = map[f];
    if (key < 0 || key >= n_c) {
      sc->err_map = 1;
      key = -1;
    }
  }
  unsigned peers = __match_any_sync(FULL_MASK, key);
  if (key >= 0 && (__ffs(peers) - 1) == lane_id()) atomicAdd(size + key, __popc(peers));
}

__global__ void k_is12(int64_t n_c, const int32_t *__restrict__ size, int64_t thr, int32_t *__restrict__ is12) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n_c) is12[c] = (int64_t)size[c] > thr;  // "exceeds 32", strict
}

// stable partition: 3-DoF nodes keep ascending order first, then 12-DoF (Alg S3 l.10-13)
__global__ void k_newid(int64_t n_c, const int64_t *__restrict__ ex12, const int32_t *__restrict__ is12,
                        const int32_t *__restrict__ size, int32_t *__restrict__ newid,
                        int32_t *__restrict__ size_new, AsmScal *sc) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n12 = ex12[n_c];
  const long long n3 = n_c - n12;
  if (c == 0) {
    sc->n3 = n3;
    sc->n12 = n12;
    sc->n_slots = n3 + 4 * n12;
  }
  if (c < n_c) {
    long long id = is12[c] ? n3 + ex12[c] : c - ex12[c];
    newid[c] = (int32_t)id;
    size_new[id] = size[c];
  }
}

__global__ void k_new_map(int64_t N, const int32_t *__restrict__ map, const int32_t *__restrict__ newid,
                          int32_t *__restrict__ nm) {
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f < N) nm[f] = newid[map[f]];
}

// children lists (order inside an aggregate is arbitrary) and per-node candidate counts
__global__ void k_children(int64_t N, const int32_t *__restrict__ nm, const int64_t *__restrict__ rp,
                           unsigned long long *__restrict__ cursor, int32_t *__restrict__ child_list,
                           unsigned long long *__restrict__ rowsum) {
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int key = f < N ? nm[f] : -1;
  long long len = f < N ? rp[f + 1] - rp[f] : 0;
  unsigned peers = __match_any_sync(FULL_MASK, key);
  int leader = __ffs(peers) - 1;
  int rank = __popc(peers & ((1u << lane_id()) - 1u));
  // segmented sum of row lengths over the peers
  long long tot = 0;
  unsigned m = peers;
  while (m) {
    int src = __ffs(m) - 1;
    m &= m - 1;
    long long v = __shfl_sync(peers, len, src);
    tot += v;
  }
  unsigned long long base = 0;
  if (key >= 0 && lane_id() == leader) {
    base = atomicAdd(cursor + key, (unsigned long long)__popc(peers));
    atomicAdd(rowsum + key, (unsigned long long)tot);
  }
  if (key >= 0) {
    base = __shfl_sync(peers, base, leader);
    child_list[base + rank] = (int32_t)f;
  }
}

__global__ void k_classify(int64_t n_c, const int32_t *__restrict__ size_new,
                           const unsigned long long *__restrict__ rowsum, uint8_t *__restrict__ is_small,
                           int32_t *__restrict__ ntasks) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n_c) {
    bool s = size_new[c] <= SMALL_CHILDREN && rowsum[c] <= SMALL_ENTRIES;
    is_small[c] = s;
    ntasks[c] = s ? 0 : (int32_t)((size_new[c] + LARGE_CHUNK - 1) / LARGE_CHUNK);
  }
}

// ------------------------------------------------------------------------------------
// Warp helpers: children table, entry lookup, bitonic sort + unique in shared memory
// ------------------------------------------------------------------------------------
struct ChildTab {
  int ci[32];
  long long rb[32];
  int off[33];
};

// Loads up to 32 children [cbase, cbase+s) and the exclusive offsets of their rows.
__device__ __forceinline__ int load_children(ChildTab &tab, const int32_t *__restrict__ child_list, int64_t cbase,
                                             int s, const int64_t *__restrict__ rp) {
  const int l = lane_id();
  int len = 0;
  if (l < s) {
    int i = child_list[cbase + l];
    long long b = rp[i];
    tab.ci[l] = i;
    tab.rb[l] = b;
    len = (int)(rp[i + 1] - b);
  }
  int incl = warp_incl_scan(len);
  tab.off[l + 1] = incl;
  if (l == 0) tab.off[0] = 0;
  __syncwarp();
  return __shfl_sync(FULL_MASK, incl, 31);
}

// entry e of the flattened children rows -> (child slot c, fine block k)
__device__ __forceinline__ void entry_of(const ChildTab &tab, int s, int e, int &c, long long &k) {
  int lo = 0, hi = s;  // largest c with off[c] <= e
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (tab.off[mid] <= e) lo = mid; else hi = mid;
  }
  c = lo;
  k = tab.rb[lo] + (e - tab.off[lo]);
}

__device__ __forceinline__ void warp_bitonic_sort(int *buf, int P) {
  const int l = lane_id();
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = l; i < P; i += 32) {
        int ixj = i ^ j;
        if (ixj > i) {
          int a = buf[i], b = buf[ixj];
          bool up = (i & k) == 0;
          if ((a > b) == up) {
            buf[i] = b;
            buf[ixj] = a;
          }
        }
      }
      __syncwarp();
    }
  }
}

__device__ __forceinline__ int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Unique of sorted buf[0,n) written to out[] (may alias buf); returns the count and, in u12,
// the number of unique entries >= n3 (12-DoF columns).
__device__ __forceinline__ int warp_unique_store(const int *buf, int n, int32_t *out, long long n3, int &u12) {
  const int l = lane_id();
  int cnt = 0, c12 = 0;
  for (int e0 = 0; e0 < n; e0 += 32) {
    const int e = e0 + l;
    const int v = e < n ? buf[e] : 0;
    const int prev = (e > 0 && e < n) ? buf[e - 1] : 0;
    const bool keep = e < n && (e == 0 || v != prev);
    const unsigned b = __ballot_sync(FULL_MASK, keep);
    c12 += __popc(__ballot_sync(FULL_MASK, keep && v >= n3));
    __syncwarp();  // every read of this chunk precedes the (possibly aliasing) writes
    if (keep) out[cnt + __popc(b & ((1u << l) - 1u))] = v;
    __syncwarp();
    cnt += __popc(b);
  }
  u12 = c12;
  return cnt;
}

// ------------------------------------------------------------------------------------
// B. symbolic
// ------------------------------------------------------------------------------------
struct SymArgs {
  int64_t n_c;
  const int32_t *child_list;
  const int64_t *child_ptr;
  const int32_t *size_new;
  const uint8_t *is_small;
  const int64_t *rp;
  const int32_t *col;
  const int32_t *nm;
  int32_t *nbs;          // neighbour lists of small nodes
  long long nbs_cap;
  long long *nb_off;     // per node: offset of its list (nbs for small, gbuf for large)
  int32_t *nb_cnt;       // per node: list length
  int32_t *rowlen;       // per node: expanded row length in blocks
  int2 *pairs;           // (large node, neighbour) pairs
  long long pair_cap;
  const int64_t *task_ptr;
  int64_t n_tasks;
  AsmScal *sc;
};

__global__ void __launch_bounds__(SYM_WARPS * 32) k_sym_small(SymArgs A) {
  __shared__ int s_buf[SYM_WARPS][SMALL_ENTRIES];
  __shared__ ChildTab s_tab[SYM_WARPS];
  const int w = threadIdx.x >> 5, l = lane_id();
  const long long n3 = A.sc->n3;
  int *buf = s_buf[w];
  ChildTab &tab = s_tab[w];
  for (int64_t a = (int64_t)blockIdx.x * SYM_WARPS + w; a < A.n_c; a += (int64_t)gridDim.x * SYM_WARPS) {
    if (!A.is_small[a]) continue;
    const int s = A.size_new[a];
    const int T = load_children(tab, A.child_list, A.child_ptr[a], s, A.rp);
    for (int e = l; e < T; e += 32) {
      int c;
      long long k;
      entry_of(tab, s, e, c, k);
      buf[e] = A.nm[A.col[k]];
    }
    const int P = next_pow2(T);
    for (int e = T + l; e < P; e += 32) buf[e] = INT_MAX;
    __syncwarp();
    warp_bitonic_sort(buf, P);
    // count uniques first to reserve space
    int cnt = 0;
    for (int e0 = 0; e0 < T; e0 += 32) {
      int e = e0 + l;
      cnt += __popc(__ballot_sync(FULL_MASK, e < T && (e == 0 || buf[e] != buf[e - 1])));
    }
    long long off = 0;
    if (l == 0) off = atomicAdd((unsigned long long *)&A.sc->nbs_count, (unsigned long long)cnt);
    off = __shfl_sync(FULL_MASK, off, 0);
    if (off + cnt > A.nbs_cap) {
      if (l == 0) A.sc->err_overflow = 1;
      continue;
    }
    int u12;
    int U = warp_unique_store(buf, T, A.nbs + off, n3, u12);
    if (l == 0) {
      A.nb_off[a] = off;
      A.nb_cnt[a] = U;
      A.rowlen[a] = U + 3 * u12;
    }
    __syncwarp();
    // transposed pairs (large neighbour b, this small node a)
    const int32_t *lst = A.nbs + off;
    for (int t0 = 0; t0 < U; t0 += 32) {
      int t = t0 + l;
      int b = t < U ? lst[t] : 0;
      bool emit = t < U && !A.is_small[b];
      unsigned m = __ballot_sync(FULL_MASK, emit);
      if (!m) continue;
      long long pb = 0;
      if (l == 0) pb = atomicAdd((unsigned long long *)&A.sc->pair_count, (unsigned long long)__popc(m));
      pb = __shfl_sync(FULL_MASK, pb, 0);
      if (emit) {
        long long pos = pb + __popc(m & ((1u << l) - 1u));
        if (pos < A.pair_cap) A.pairs[pos] = make_int2(b, (int)a);
        else A.sc->err_overflow = 1;
      }
    }
    __syncwarp();
  }
}

// 32-children chunks of large nodes: emit (a, b) for every large neighbour b (a itself once).
__global__ void __launch_bounds__(SYM_WARPS * 32) k_sym_large(SymArgs A) {
  __shared__ int s_buf[SYM_WARPS][SMALL_ENTRIES];
  __shared__ ChildTab s_tab[SYM_WARPS];
  const int w = threadIdx.x >> 5, l = lane_id();
  int *buf = s_buf[w];
  ChildTab &tab = s_tab[w];
  const int64_t n_tasks = A.task_ptr[A.n_c];
  for (int64_t t = (int64_t)blockIdx.x * SYM_WARPS + w; t < n_tasks; t += (int64_t)gridDim.x * SYM_WARPS) {
    const int a = lower_bound_dev<int64_t>(A.task_ptr, (int)A.n_c + 1, t + 1) - 1;
    const int chunk = (int)(t - A.task_ptr[a]);
    const int s = min(LARGE_CHUNK, A.size_new[a] - chunk * LARGE_CHUNK);
    const int T = load_children(tab, A.child_list, A.child_ptr[a] + (int64_t)chunk * LARGE_CHUNK, s, A.rp);
    for (int e0 = 0; e0 < T; e0 += SMALL_ENTRIES) {
      const int n = min(SMALL_ENTRIES, T - e0);
      for (int e = l; e < n; e += 32) {
        int c;
        long long k;
        entry_of(tab, s, e0 + e, c, k);
        int b = A.nm[A.col[k]];
        buf[e] = (b == a || A.is_small[b]) ? INT_MAX : b;  // only large, off-diagonal columns
      }
      const int P = next_pow2(n);
      for (int e = n + l; e < P; e += 32) buf[e] = INT_MAX;
      __syncwarp();
      warp_bitonic_sort(buf, P);
      for (int e1 = 0; e1 < n; e1 += 32) {
        int e = e1 + l;
        bool keep = e < n && buf[e] != INT_MAX && (e == 0 || buf[e] != buf[e - 1]);
        unsigned m = __ballot_sync(FULL_MASK, keep);
        if (!m) continue;
        long long pb = 0;
        if (l == 0) pb = atomicAdd((unsigned long long *)&A.sc->pair_count, (unsigned long long)__popc(m));
        pb = __shfl_sync(FULL_MASK, pb, 0);
        if (keep) {
          long long pos = pb + __popc(m & ((1u << l) - 1u));
          if (pos < A.pair_cap) A.pairs[pos] = make_int2(a, buf[e]);
          else A.sc->err_overflow = 1;
        }
      }
      __syncwarp();
    }
    if (chunk == 0 && l == 0) {  // the diagonal block (a, a) always exists
      long long pos = (long long)atomicAdd((unsigned long long *)&A.sc->pair_count, 1ull);
      if (pos < A.pair_cap) A.pairs[pos] = make_int2(a, a);
      else A.sc->err_overflow = 1;
    }
  }
}

__global__ void k_pair_count(const AsmScal *sc, long long cap, const int2 *__restrict__ pairs,
                             int32_t *__restrict__ gcnt) {
  const long long np = min(sc->pair_count, cap);
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < np; p += (long long)gridDim.x * blockDim.x)
    atomicAdd(gcnt + pairs[p].x, 1);
}

// padded group sizes: next power of two (so every group can be sorted in place)
__global__ void k_pow2(int64_t n, const int32_t *__restrict__ cnt, int32_t *__restrict__ out) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n) out[c] = cnt[c] ? next_pow2(cnt[c]) : 0;
}

__global__ void k_pair_scatter(const AsmScal *sc, long long cap, const int2 *__restrict__ pairs,
                               unsigned long long *__restrict__ cursor, int32_t *__restrict__ gbuf) {
  const long long np = min(sc->pair_count, cap);
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < np; p += (long long)gridDim.x * blockDim.x) {
    int2 q = pairs[p];
    gbuf[atomicAdd(cursor + q.x, 1ull)] = q.y;
  }
}

// sort + unique of each large node's list in place (padded to a power of two)
__global__ void __launch_bounds__(SYM_WARPS * 32) k_group_unique(int64_t n_c, const uint8_t *__restrict__ is_small,
                                                                 const int64_t *__restrict__ gptr, int32_t *gbuf,
                                                                 const int32_t *__restrict__ gcnt, long long *nb_off,
                                                                 int32_t *nb_cnt, int32_t *rowlen, int32_t *big_list,
                                                                 AsmScal *sc) {
  __shared__ int s_buf[SYM_WARPS][SMALL_ENTRIES];
  const int w = threadIdx.x >> 5, l = lane_id();
  const long long n3 = sc->n3;
  int *buf = s_buf[w];
  for (int64_t a = (int64_t)blockIdx.x * SYM_WARPS + w; a < n_c; a += (int64_t)gridDim.x * SYM_WARPS) {
    if (is_small[a]) continue;
    const int n = gcnt[a];
    const int P = next_pow2(n);
    int32_t *g = gbuf + gptr[a];
    if (P > SMALL_ENTRIES) {
      if (l == 0) big_list[atomicAdd((unsigned long long *)&sc->big_groups, 1ull)] = (int32_t)a;
      continue;
    }
    for (int e = l; e < P; e += 32) buf[e] = e < n ? g[e] : INT_MAX;
    __syncwarp();
    warp_bitonic_sort(buf, P);
    int u12;
    int U = warp_unique_store(buf, n, g, n3, u12);
    if (l == 0) {
      nb_off[a] = gptr[a];
      nb_cnt[a] = U;
      rowlen[a] = U + 3 * u12;
    }
    __syncwarp();
  }
}

// CTA-wide global-memory bitonic sort for the (rare) large lists of more than 2048 entries.
__global__ void __launch_bounds__(1024) k_group_unique_big(const AsmScal *sc, const int32_t *__restrict__ big_list,
                                                           const int64_t *__restrict__ gptr, int32_t *gbuf,
                                                           const int32_t *__restrict__ gcnt, long long *nb_off,
                                                           int32_t *nb_cnt, int32_t *rowlen) {
  const long long nb = sc->big_groups;
  const long long n3 = sc->n3;
  for (long long q = blockIdx.x; q < nb; q += gridDim.x) {
    const int a = big_list[q];
    const int n = gcnt[a];
    const int P = next_pow2(n);
    int32_t *g = gbuf + gptr[a];
    for (int e = n + threadIdx.x; e < P; e += blockDim.x) g[e] = INT_MAX;
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < P; i += blockDim.x) {
          int ixj = i ^ j;
          if (ixj > i) {
            int x = g[i], y = g[ixj];
            bool up = (i & k) == 0;
            if ((x > y) == up) {
              g[i] = y;
              g[ixj] = x;
            }
          }
        }
        __syncthreads();
      }
    // unique: mark into the padding-free prefix by a sequential-per-warp compaction
    if (threadIdx.x < 32) {
      int u12;
      int U = warp_unique_store(g, n, g, n3, u12);  // in place: writes never overtake reads
      if (threadIdx.x == 0) {
        nb_off[a] = gptr[a];
        nb_cnt[a] = U;
        rowlen[a] = U + 3 * u12;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------
// C. slot row lengths
// ------------------------------------------------------------------------------------
__global__ void k_slot_rowlen(int64_t n_c, const AsmScal *sc, const int32_t *__restrict__ rowlen,
                              int32_t *__restrict__ rl) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n3 = sc->n3;
  if (c < n_c) {
    int ncb = ncb_of((int)c, n3);
    for (int p = 0; p < ncb; ++p) rl[slot_of((int)c, p, n3)] = rowlen[c];
  }
}

__global__ void k_final_scalars(AsmScal *sc, const int64_t *__restrict__ row_ptr) {
  sc->nnzb = row_ptr[sc->n_slots];
}

// ------------------------------------------------------------------------------------
// D. numeric
// ------------------------------------------------------------------------------------
struct NumArgs {
  int64_t n_c;
  const AsmScal *sc;
  const int32_t *child_list;
  const int64_t *child_ptr;
  const int32_t *size_new;
  const uint8_t *is_small;
  const int64_t *rp;
  const int32_t *col;
  const double *val;
  const int32_t *nm;
  const double *X;
  const double *g_f;
  const int32_t *nbs;
  const int32_t *gbuf;
  const long long *nb_off;
  const int32_t *nb_cnt;
  const int32_t *rowlen;
  const int64_t *task_ptr;
  int64_t n_tasks;
  const int64_t *crp;  // coarse row_ptr (slots)
  int32_t *ccol;
  double *cval;
  double *g_c;
};

__device__ __forceinline__ const int32_t *list_of(const NumArgs &A, int a) {
  return (A.is_small[a] ? A.nbs : A.gbuf) + A.nb_off[a];
}

// Large rows: write their column ids and zero their values (blocks are then filled by the
// mirrored writes of small rows and by the atomics of the large-row chunks).
__global__ void k_large_rows_init(NumArgs A) {
  const int w = threadIdx.x >> 5, l = lane_id();
  const int wpb = blockDim.x >> 5;
  const long long n3 = A.sc->n3;
  for (int64_t a = (int64_t)blockIdx.x * wpb + w; a < A.n_c; a += (int64_t)gridDim.x * wpb) {
    if (A.is_small[a]) continue;
    const int U = A.nb_cnt[a], rl = A.rowlen[a];
    const int32_t *lst = list_of(A, (int)a);
    const int first12 = lower_bound_dev<int32_t>(lst, U, (int32_t)n3);
    const int ncb_a = ncb_of((int)a, n3);
    for (int p = 0; p < ncb_a; ++p) {
      const long long rs = A.crp[slot_of((int)a, p, n3)];
      for (int t = l; t < U; t += 32) {
        int b = lst[t];
        int cp = colpos(t, first12);
        int ncb_b = ncb_of(b, n3);
        for (int q = 0; q < ncb_b; ++q) A.ccol[rs + cp + q] = slot_of(b, q, n3);
      }
      double *v = A.cval + 9 * rs;
      for (int x = l; x < 9 * rl; x += 32) v[x] = 0.0;
    }
  }
}

__global__ void __launch_bounds__(NUM_WARPS * 32) k_num_small(NumArgs A) {
  __shared__ int s_list[NUM_WARPS][LIST_CAP];
  __shared__ double s_acc[NUM_WARPS][ACC_CAP];
  __shared__ ChildTab s_tab[NUM_WARPS];
  const int w = threadIdx.x >> 5, l = lane_id();
  const long long n3 = A.sc->n3;
  ChildTab &tab = s_tab[w];
  for (int64_t a64 = (int64_t)blockIdx.x * NUM_WARPS + w; a64 < A.n_c; a64 += (int64_t)gridDim.x * NUM_WARPS) {
    const int a = (int)a64;
    if (!A.is_small[a]) continue;
    const int ncb_a = ncb_of(a, n3);
    const int U = A.nb_cnt[a], rl = A.rowlen[a];
    const int32_t *glist = A.nbs + A.nb_off[a];
    const bool in_smem = U <= LIST_CAP && ncb_a * rl * 9 <= ACC_CAP;
    const int32_t *lst = glist;
    if (in_smem) {
      for (int t = l; t < U; t += 32) s_list[w][t] = glist[t];
      for (int x = l; x < ncb_a * rl * 9; x += 32) s_acc[w][x] = 0.0;
      lst = s_list[w];
    } else {
      for (int p = 0; p < ncb_a; ++p) {
        double *v = A.cval + 9 * A.crp[slot_of(a, p, n3)];
        for (int x = l; x < 9 * rl; x += 32) v[x] = 0.0;
      }
    }
    __syncwarp();
    const int first12 = lower_bound_dev<int32_t>(lst, U, (int32_t)n3);
    const int s = A.size_new[a];
    const int T = load_children(tab, A.child_list, A.child_ptr[a], s, A.rp);
    // entries in batches of 32; lanes with the same target column form a peer group whose
    // leader sums the peers' contributions (shuffles) and updates the accumulator with a plain
    // read-modify-write -- no floating-point atomics (shared fp64 atomicAdd is a CAS loop)
    for (int e0 = 0; e0 < T; e0 += 32) {
      const int e = e0 + l;
      const bool act = e < T;
      int c = 0, i = 0, j = 0, b = 0, idx = -1;
      long long k = 0;
      if (act) {
        entry_of(tab, s, e, c, k);
        i = tab.ci[c];
        j = A.col[k];
        b = A.nm[j];
        idx = lower_bound_dev<int32_t>(lst, U, b);
      }
      const unsigned peers = __match_any_sync(FULL_MASK, idx);
      if (act) {
      const int leader = __ffs(peers) - 1;
      const bool solo = (peers & (peers - 1)) == 0;
      const int cp = colpos(idx, first12);
      const int ncb_b = ncb_of(b, n3);
      double B[9];
#pragma unroll
      for (int x = 0; x < 9; ++x) B[x] = __ldg(A.val + 9 * k + x);
      for (int p = 0; p < ncb_a; ++p) {
        const double wi = wgt(A.X, i, ncb_a, p);
        for (int q = 0; q < ncb_b; ++q) {
          const double coef = wi * wgt(A.X, j, ncb_b, q);
          double v[9];
#pragma unroll
          for (int x = 0; x < 9; ++x) v[x] = coef * B[x];
          if (!solo) {  // sum the peers' v into the leader (fixed lane order)
            double sum[9];
#pragma unroll
            for (int x = 0; x < 9; ++x) sum[x] = 0.0;
            unsigned m = peers;
            while (m) {
              const int src = __ffs(m) - 1;
              m &= m - 1;
#pragma unroll
              for (int x = 0; x < 9; ++x) sum[x] += __shfl_sync(peers, v[x], src);
            }
#pragma unroll
            for (int x = 0; x < 9; ++x) v[x] = sum[x];
          }
          if (l == leader) {
            double *dst = in_smem ? s_acc[w] + ((p * rl) + cp + q) * 9
                                  : A.cval + 9 * (A.crp[slot_of(a, p, n3)] + cp + q);
#pragma unroll
            for (int x = 0; x < 9; ++x) dst[x] += v[x];
          }
        }
      }
      }  // act
      __syncwarp();  // the next batch's leaders read what this batch's leaders wrote
    }
    __syncwarp();
    if (!in_smem) __threadfence();
    // write the row(s): values (flat, coalesced) and column ids
    for (int p = 0; p < ncb_a; ++p) {
      const long long rs = A.crp[slot_of(a, p, n3)];
      if (in_smem) {
        double *v = A.cval + 9 * rs;
        const double *src = s_acc[w] + p * rl * 9;
        for (int x = l; x < 9 * rl; x += 32) v[x] = src[x];
      }
      for (int t = l; t < U; t += 32) {
        int b = lst[t];
        int cp = colpos(t, first12);
        int ncb_b = ncb_of(b, n3);
        for (int q = 0; q < ncb_b; ++q) A.ccol[rs + cp + q] = slot_of(b, q, n3);
      }
    }
    // mirrored (large row, small column) blocks: H_c(slot(b,q), slot(a,p)) = H_c(slot(a,p), slot(b,q))^T
    for (int t = l; t < U; t += 32) {
      const int b = lst[t];
      if (A.is_small[b]) continue;
      const int cp = colpos(t, first12);
      const int ncb_b = ncb_of(b, n3);
      const int32_t *lb_ = A.gbuf + A.nb_off[b];
      const int Ub = A.nb_cnt[b];
      const int idxb = lower_bound_dev<int32_t>(lb_, Ub, (int32_t)a);
      const int cpb = colpos(idxb, lower_bound_dev<int32_t>(lb_, Ub, (int32_t)n3));
      for (int p = 0; p < ncb_a; ++p)
        for (int q = 0; q < ncb_b; ++q) {
          double m[9];
          if (in_smem) {
            const double *src = s_acc[w] + ((p * rl) + cp + q) * 9;
#pragma unroll
            for (int x = 0; x < 9; ++x) m[x] = src[x];
          } else {  // values were produced by L2 atomics: read them from L2
            const double *src = A.cval + 9 * (A.crp[slot_of(a, p, n3)] + cp + q);
#pragma unroll
            for (int x = 0; x < 9; ++x) m[x] = __ldcg(src + x);
          }
          double *dst = A.cval + 9 * (A.crp[slot_of(b, q, n3)] + cpb + p);
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) dst[3 * r + cc] = m[3 * cc + r];
        }
    }
    // g_c[slot(a,p)] = sum_children w_i[p] g_f[i]  (Eq 4)
    if (A.g_f) {
      for (int p = 0; p < ncb_a; ++p) {
        double g0 = 0, g1 = 0, g2 = 0;
        if (l < s) {
          int i = tab.ci[l];
          double wi = wgt(A.X, i, ncb_a, p);
          g0 = wi * A.g_f[3 * (int64_t)i];
          g1 = wi * A.g_f[3 * (int64_t)i + 1];
          g2 = wi * A.g_f[3 * (int64_t)i + 2];
        }
        g0 = warp_sum(g0);
        g1 = warp_sum(g1);
        g2 = warp_sum(g2);
        if (l == 0) {
          double *gc = A.g_c + 3 * (int64_t)slot_of(a, p, n3);
          gc[0] = g0;
          gc[1] = g1;
          gc[2] = g2;
        }
      }
    }
    __syncwarp();
  }
}

// Large rows, one warp per 32-children chunk.  lane = (g, p): G = 32/NCB block groups, NCB
// lanes per fine block.  The diagonal block (a,a) accumulates in registers (NCB x 9 doubles
// per lane) and is flushed once per chunk; (a, b) with b large and b != a uses fp64 atomics;
// (a, b) with b small is skipped here (mirrored by the small row b).
template <int NCB>
__global__ void __launch_bounds__(NUM_WARPS * 32) k_num_large(NumArgs A) {
  __shared__ ChildTab s_tab[NUM_WARPS];
  const int w = threadIdx.x >> 5, l = lane_id();
  const int gq = l / NCB, p = l % NCB;
  constexpr int G = 32 / NCB;
  const long long n3 = A.sc->n3;
  ChildTab &tab = s_tab[w];
  const int64_t n_tasks = A.task_ptr[A.n_c];
  for (int64_t t = (int64_t)blockIdx.x * NUM_WARPS + w; t < n_tasks; t += (int64_t)gridDim.x * NUM_WARPS) {
    const int a = lower_bound_dev<int64_t>(A.task_ptr, (int)A.n_c + 1, t + 1) - 1;
    if (ncb_of(a, n3) != NCB) continue;
    const int chunk = (int)(t - A.task_ptr[a]);
    const int s = min(LARGE_CHUNK, A.size_new[a] - chunk * LARGE_CHUNK);
    const int T = load_children(tab, A.child_list, A.child_ptr[a] + (int64_t)chunk * LARGE_CHUNK, s, A.rp);
    const int32_t *lst = A.gbuf + A.nb_off[a];
    const int U = A.nb_cnt[a];
    const int first12 = lower_bound_dev<int32_t>(lst, U, (int32_t)n3);
    const long long rs_p = A.crp[slot_of(a, p, n3)];
    double acc[NCB][9];
#pragma unroll
    for (int q = 0; q < NCB; ++q)
#pragma unroll
      for (int x = 0; x < 9; ++x) acc[q][x] = 0.0;
    for (int e0 = 0; e0 < T; e0 += G) {
      const int e = e0 + gq;
      if (e >= T) continue;
      int c;
      long long k;
      entry_of(tab, s, e, c, k);
      const int j = A.col[k];
      const int b = A.nm[j];
      if (b != a && A.is_small[b]) continue;
      const int i = tab.ci[c];
      double B[9];
#pragma unroll
      for (int x = 0; x < 9; ++x) B[x] = __ldg(A.val + 9 * k + x);
      const double wi = wgt(A.X, i, NCB, p);
      if (b == a) {
#pragma unroll
        for (int q = 0; q < NCB; ++q) {
          const double coef = wi * wgt(A.X, j, NCB, q);
#pragma unroll
          for (int x = 0; x < 9; ++x) acc[q][x] += coef * B[x];
        }
      } else {
        const int idx = lower_bound_dev<int32_t>(lst, U, b);
        const int cp = colpos(idx, first12);
        const int ncb_b = ncb_of(b, n3);
        for (int q = 0; q < ncb_b; ++q) {
          const double coef = wi * wgt(A.X, j, ncb_b, q);
          double *dst = A.cval + 9 * (rs_p + cp + q);
#pragma unroll
          for (int x = 0; x < 9; ++x) atomicAdd(dst + x, coef * B[x]);
        }
      }
    }
    // reduce the diagonal accumulators over the block groups (lanes with the same p)
#pragma unroll
    for (int o = NCB; o < 32; o <<= 1)
#pragma unroll
      for (int q = 0; q < NCB; ++q)
#pragma unroll
        for (int x = 0; x < 9; ++x) acc[q][x] += __shfl_xor_sync(FULL_MASK, acc[q][x], o);
    if (gq == 0) {
      const int idx = lower_bound_dev<int32_t>(lst, U, a);
      const int cp = colpos(idx, first12);
#pragma unroll
      for (int q = 0; q < NCB; ++q) {
        double *dst = A.cval + 9 * (rs_p + cp + q);
#pragma unroll
        for (int x = 0; x < 9; ++x) atomicAdd(dst + x, acc[q][x]);
      }
    }
    if (A.g_f) {
      for (int pp = 0; pp < NCB; ++pp) {
        double g0 = 0, g1 = 0, g2 = 0;
        if (l < s) {
          int i = tab.ci[l];
          double wi = wgt(A.X, i, NCB, pp);
          g0 = wi * A.g_f[3 * (int64_t)i];
          g1 = wi * A.g_f[3 * (int64_t)i + 1];
          g2 = wi * A.g_f[3 * (int64_t)i + 2];
        }
        g0 = warp_sum(g0);
        g1 = warp_sum(g1);
        g2 = warp_sum(g2);
        if (l == 0) {
          double *gc = A.g_c + 3 * (int64_t)slot_of(a, pp, n3);
          atomicAdd(gc, g0);
          atomicAdd(gc + 1, g1);
          atomicAdd(gc + 2, g2);
        }
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------
// host orchestration
// ------------------------------------------------------------------------------------
extern "C" agipc_status agipc_assemble_coarse(agipc_handle h, const agipc_mesh *mesh, const int32_t *map,
                                              int64_t n_coarse, int64_t affine_threshold, const agipc_bsr *H,
                                              const double *g_fine, agipc_coarse *out) {
  if (!h) return AGIPC_EINVAL;
  if (!mesh || !H || !out) return set_err(h, AGIPC_EINVAL, "assemble_coarse: null argument");
  const int64_t N = mesh->n_nodes, n_c = n_coarse;
  if (N < 0 || n_c < 0 || (N > 0 && n_c < 1) || n_c > N) return set_err(h, AGIPC_EINVAL, "assemble_coarse: bad sizes");
  if (H->n_rows != N) return set_err(h, AGIPC_EINVAL, "assemble_coarse: H_fine has %lld rows, mesh %lld nodes",
                                     (long long)H->n_rows, (long long)N);
  if (N >= INT32_MAX / 4 || H->nnzb >= ((int64_t)1 << 40)) return set_err(h, AGIPC_ERANGE, "assemble_coarse: too large");
  out->n3 = out->n12 = out->n_slots = out->nnzb = 0;
  if (N == 0) return AGIPC_OK;
  if (!map || !mesh->x_rest || !H->row_ptr || !H->col || !H->val || !out->new_map)
    return set_err(h, AGIPC_EINVAL, "assemble_coarse: null pointer");
  CU_TRY(h, cudaSetDevice(h->device));
  ProfScope prof_scope(h, PROF_ASSEMBLE, h->stream);
  cudaStream_t st_ = h->stream;
  const int64_t nnzb_f = H->nnzb;
  agipc_status st;

  WS(h, sc, AsmScal, "asm_scal", 1);
  CU_TRY(h, cudaMemsetAsync(sc, 0, sizeof(AsmScal), st_));
  // ---- A. classification ----
  WS(h, size, int32_t, "asm_size", n_c);
  WS(h, is12, int32_t, "asm_is12", n_c);
  WS(h, ex12, int64_t, "asm_ex12", n_c + 1);
  WS(h, newid, int32_t, "asm_newid", n_c);
  WS(h, size_new, int32_t, "asm_size_new", n_c);
  WS(h, child_ptr, int64_t, "asm_child_ptr", n_c + 1);
  WS(h, cursor, unsigned long long, "asm_cursor", n_c + 1);
  WS(h, rowsum, unsigned long long, "asm_rowsum", n_c);
  WS(h, child_list, int32_t, "asm_child_list", N);
  WS(h, is_small, uint8_t, "asm_is_small", n_c);
  WS(h, ntasks, int32_t, "asm_ntasks", n_c);
  WS(h, task_ptr, int64_t, "asm_task_ptr", n_c + 1);
  CU_TRY(h, cudaMemsetAsync(size, 0, sizeof(int32_t) * n_c, st_));
  CU_TRY(h, cudaMemsetAsync(rowsum, 0, sizeof(unsigned long long) * n_c, st_));
  const unsigned gN = (unsigned)cdiv(N, 256), gC = (unsigned)cdiv(n_c, 256);
  LAUNCH(h, k_size_hist, gN, 256, 0, N, map, n_c, size, sc);
  LAUNCH(h, k_is12, gC, 256, 0, n_c, size, affine_threshold, is12);
  if ((st = scan_exclusive_i64(h, SCAN_SRC_I32, is12, n_c, ex12)) != AGIPC_OK) return st;
  LAUNCH(h, k_newid, gC, 256, 0, n_c, ex12, is12, size, newid, size_new, sc);
  LAUNCH(h, k_new_map, gN, 256, 0, N, map, newid, out->new_map);
  if ((st = scan_exclusive_i64(h, SCAN_SRC_I32, size_new, n_c, child_ptr)) != AGIPC_OK) return st;
  CU_TRY(h, cudaMemcpyAsync(cursor, child_ptr, sizeof(int64_t) * n_c, cudaMemcpyDeviceToDevice, st_));
  LAUNCH(h, k_children, gN, 256, 0, N, out->new_map, H->row_ptr, cursor, child_list, rowsum);
  LAUNCH(h, k_classify, gC, 256, 0, n_c, size_new, rowsum, is_small, ntasks);
  if ((st = scan_exclusive_i64(h, SCAN_SRC_I32, ntasks, n_c, task_ptr)) != AGIPC_OK) return st;

  // ---- B. symbolic ----
  const long long nbs_cap = nnzb_f + 32;
  const long long pair_cap = nnzb_f + n_c + 32;
  WS(h, nbs, int32_t, "asm_nbs", nbs_cap);
  WS(h, nb_off, long long, "asm_nb_off", n_c);
  WS(h, nb_cnt, int32_t, "asm_nb_cnt", n_c);
  WS(h, rowlen, int32_t, "asm_rowlen", n_c);
  WS(h, pairs, int2, "asm_pairs", pair_cap);
  WS(h, gcnt, int32_t, "asm_gcnt", n_c);
  WS(h, gpad, int32_t, "asm_gpad", n_c);
  WS(h, gptr, int64_t, "asm_gptr", n_c + 1);
  WS(h, gbuf, int32_t, "asm_gbuf", 2 * pair_cap);
  WS(h, big_list, int32_t, "asm_big_list", n_c);
  // n_tasks is needed on the host for the grid only as an upper bound: sum of ceil(size/32) <= N/32 + n_c
  const int64_t task_bound = N / LARGE_CHUNK + n_c;
  SymArgs SA;
  SA.n_c = n_c; SA.child_list = child_list; SA.child_ptr = child_ptr; SA.size_new = size_new;
  SA.is_small = is_small; SA.rp = H->row_ptr; SA.col = H->col; SA.nm = out->new_map;
  SA.nbs = nbs; SA.nbs_cap = nbs_cap; SA.nb_off = nb_off; SA.nb_cnt = nb_cnt; SA.rowlen = rowlen;
  SA.pairs = pairs; SA.pair_cap = pair_cap; SA.task_ptr = task_ptr; SA.n_tasks = task_bound; SA.sc = sc;
  const unsigned gsym = (unsigned)std::min<int64_t>(cdiv(n_c, SYM_WARPS), 64 * h->sm_count);
  LAUNCH(h, k_sym_small, gsym, SYM_WARPS * 32, 0, SA);
  // the exact task count task_ptr[n_c] is read on the device; task_bound only sizes the grid
  LAUNCH(h, k_sym_large, (unsigned)std::min<int64_t>(std::max<int64_t>(1, cdiv(task_bound, SYM_WARPS)), 64 * h->sm_count),
         SYM_WARPS * 32, 0, SA);
  CU_TRY(h, cudaMemsetAsync(gcnt, 0, sizeof(int32_t) * n_c, st_));
  LAUNCH(h, k_pair_count, (unsigned)(8 * h->sm_count), 256, 0, sc, pair_cap, pairs, gcnt);
  LAUNCH(h, k_pow2, gC, 256, 0, n_c, gcnt, gpad);
  if ((st = scan_exclusive_i64(h, SCAN_SRC_I32, gpad, n_c, gptr)) != AGIPC_OK) return st;
  CU_TRY(h, cudaMemcpyAsync(cursor, gptr, sizeof(int64_t) * n_c, cudaMemcpyDeviceToDevice, st_));
  LAUNCH(h, k_pair_scatter, (unsigned)(8 * h->sm_count), 256, 0, sc, pair_cap, pairs, cursor, gbuf);
  LAUNCH(h, k_group_unique, gsym, SYM_WARPS * 32, 0, n_c, is_small, gptr, gbuf, gcnt, nb_off, nb_cnt, rowlen,
         big_list, sc);
  LAUNCH(h, k_group_unique_big, (unsigned)h->sm_count, 1024, 0, sc, big_list, gptr, gbuf, gcnt, nb_off, nb_cnt, rowlen);

  // ---- C. slot row pointer (upper bound 4 n_c slots; entries past n_slots are 0) ----
  const int64_t slot_bound = 4 * n_c;
  WS(h, rl, int32_t, "asm_rl", slot_bound);
  WS(h, crp_ws, int64_t, "asm_crp", slot_bound + 1);
  CU_TRY(h, cudaMemsetAsync(rl, 0, sizeof(int32_t) * slot_bound, st_));
  LAUNCH(h, k_slot_rowlen, gC, 256, 0, n_c, sc, rowlen, rl);
  if ((st = scan_exclusive_i64(h, SCAN_SRC_I32, rl, slot_bound, crp_ws)) != AGIPC_OK) return st;
  LAUNCH(h, k_final_scalars, 1, 1, 0, sc, crp_ws);
  AsmScal *hsc = (AsmScal *)pinned_get(h, sizeof(AsmScal), &st);
  if (st != AGIPC_OK) return st;
  CU_TRY(h, cudaMemcpyAsync(hsc, sc, sizeof(AsmScal), cudaMemcpyDeviceToHost, st_));
  CU_TRY(h, cudaStreamSynchronize(st_));
  if (hsc->err_map) return set_err(h, AGIPC_EINVAL, "assemble_coarse: map value outside [0, n_coarse)");
  if (hsc->err_overflow) return set_err(h, AGIPC_ECUDA, "assemble_coarse: internal buffer overflow");
  out->n3 = hsc->n3;
  out->n12 = hsc->n12;
  out->n_slots = hsc->n_slots;
  out->nnzb = hsc->nnzb;
  if (out->n_slots >= INT32_MAX) return set_err(h, AGIPC_ERANGE, "assemble_coarse: n_slots exceeds int32");
  if (out->cap_slots < out->n_slots || out->cap_nnzb < out->nnzb)
    return set_err(h, AGIPC_ENOSPACE, "assemble_coarse: need %lld slots / %lld blocks", (long long)out->n_slots,
                   (long long)out->nnzb);
  if (!out->row_ptr || (out->nnzb > 0 && (!out->col || !out->val)))
    return set_err(h, AGIPC_EINVAL, "assemble_coarse: null output arrays");
  CU_TRY(h, cudaMemcpyAsync(out->row_ptr, crp_ws, sizeof(int64_t) * (out->n_slots + 1), cudaMemcpyDeviceToDevice, st_));

  // ---- D. numeric ----
  NumArgs NA;
  NA.n_c = n_c; NA.sc = sc; NA.child_list = child_list; NA.child_ptr = child_ptr; NA.size_new = size_new;
  NA.is_small = is_small; NA.rp = H->row_ptr; NA.col = H->col; NA.val = H->val; NA.nm = out->new_map;
  NA.X = mesh->x_rest; NA.g_f = (g_fine && out->g_c) ? g_fine : nullptr; NA.nbs = nbs; NA.gbuf = gbuf;
  NA.nb_off = nb_off; NA.nb_cnt = nb_cnt; NA.rowlen = rowlen; NA.task_ptr = task_ptr; NA.n_tasks = task_bound;
  NA.crp = out->row_ptr; NA.ccol = out->col; NA.cval = out->val; NA.g_c = out->g_c;
  if (NA.g_f) CU_TRY(h, cudaMemsetAsync(out->g_c, 0, sizeof(double) * 3 * out->n_slots, st_));
  LAUNCH(h, k_large_rows_init, gsym, 128, 0, NA);
  LAUNCH(h, k_num_small, gsym, NUM_WARPS * 32, 0, NA);
  const unsigned glarge = (unsigned)std::min<int64_t>(std::max<int64_t>(1, cdiv(task_bound, NUM_WARPS)), 64 * h->sm_count);
  LAUNCH(h, k_num_large<4>, glarge, NUM_WARPS * 32, 0, NA);
  LAUNCH(h, k_num_large<1>, glarge, NUM_WARPS * 32, 0, NA);
  return AGIPC_OK;
}
