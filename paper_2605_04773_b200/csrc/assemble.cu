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
#include <memory>

#include "agipc_internal.cuh"

#define SMALL_CHILDREN 32
#define SMALL_ENTRIES 2048
#define SYM_WARPS 4
#define NUM_WARPS 4
#define LIST_CAP 512
#define ACC_CAP 1024
#define LARGE_CHUNK 32
#define SMALL_T 1024           // small nodes: <= 32 children and <= 1024 candidate entries
// CTAs per SM requested by the launch bounds (experiment knobs, defaults = measured best)
#ifndef SMALL_MINB_N
#define SMALL_MINB_N 4  // numeric small rows: 64 registers
#endif
#ifndef MID_MINB_N
#define MID_MINB_N 1    // numeric mid nodes: 128 registers
#endif
#ifndef SMALL_MINB_S
#define SMALL_MINB_S 6  // symbolic small rows: 40 registers, 6 x 8 warps per SM (profiles/r02v)
#endif
#ifndef MID_MINB_S
#define MID_MINB_S 6    // symbolic mid nodes: 80 registers (the register sort), 6 x 4 warps per SM
#endif

struct AsmScal {
  long long n3, n12, n_slots, nnzb;
  long long nbs_count;   // entries used in the small-node neighbour buffer
  long long list_top;    // entries allocated in the large-row entry lists (k_sym_large)
  long long n_w32;       // nodes of the 32-entry small list (k_sym_finish)
  long long pair_count;  // (large, x) pairs
  long long big_groups;  // large lists that need the CTA sort
  long long n_large3;    // large nodes with 3 DoF (affine threshold > 32)
  long long rec_total;   // interface records of the large-row chunks (k_num_large)
  long long n_tasks;     // large-row chunks
  int err_map;           // map value outside [0, n_c)
  int err_overflow;      // a buffer capacity was exceeded
  int err_cap;           // the numeric pass must not write: an error above, a slot count past
                         // int32 or outputs larger than the caller's capacity (k_sym_finish)
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
    if (key < 0 || key >= n_c) {  // reported as EINVAL after the symbolic phase; until then the
      sc->err_map = 1;             // node counts as a child of aggregate 0, so every later kernel
      key = 0;                     // stays in bounds (k_new_map applies the same substitution)
    }
  }
  unsigned peers = __match_any_sync(FULL_MASK, key);
  if (key >= 0 && (__ffs(peers) - 1) == lane_id()) atomicAdd(size + key, __popc(peers));
}

// stable partition: 3-DoF nodes keep ascending order first, then 12-DoF (Alg S3 l.10-13)
__global__ void k_newid(int64_t n_c, const int64_t *__restrict__ ex12, int64_t thr,
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
    long long id = (int64_t)size[c] > thr ? n3 + ex12[c] : c - ex12[c];  // is12 (k_is12 semantics)
    newid[c] = (int32_t)id;
    size_new[id] = size[c];
  }
}

__global__ void k_new_map(int64_t N, int64_t n_c, const int32_t *__restrict__ map, const int32_t *__restrict__ newid,
                          int32_t *__restrict__ nm) {
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f < N) {
    const int m = map[f];
    nm[f] = newid[(m >= 0 && m < n_c) ? m : 0];  // out-of-range: see k_size_hist
  }
}

// R22 precondition check (AGIPC_OPT_CHECK_SYMMETRY): every stored block (i, j) has a stored
// (j, i) with B_ji == B_ij^T bit for bit; warp per row, binary search in row j.
__global__ void k_check_sym(int64_t N, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                            const double *__restrict__ val, unsigned long long *bad) {
  unsigned long long nb = 0;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    for (int64_t k = rp[i] + lane_id(); k < rp[i + 1]; k += 32) {
      const int64_t j = col[k];
      if (j < 0 || j >= N) {
        ++nb;
        continue;
      }
      int64_t lo = rp[j], hi = rp[j + 1];
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (col[mid] < i) lo = mid + 1; else hi = mid;
      }
      if (lo >= rp[j + 1] || col[lo] != i) {
        ++nb;
        continue;
      }
      const double *a = val + 9 * k, *b = val + 9 * lo;
      bool ok = true;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) ok &= __double_as_longlong(a[3 * r + c]) == __double_as_longlong(b[3 * c + r]);
      nb += !ok;
    }
  }
  nb = warp_sum(nb);
  if (lane_id() == 0 && nb) atomicAdd(bad, nb);
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
                           int32_t *__restrict__ ntasks, AsmScal *sc, int32_t *__restrict__ f16,
                           int32_t *__restrict__ f32, int32_t *__restrict__ ft, int64_t *__restrict__ ecount) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n_c) {
    const unsigned long long rs = rowsum[c];
    bool s = size_new[c] <= SMALL_CHILDREN && rs <= SMALL_T;
    is_small[c] = s;
    ntasks[c] = s ? 0 : (int32_t)((size_new[c] + LARGE_CHUNK - 1) / LARGE_CHUNK);
    if (!s && c < sc->n3) atomicAdd((unsigned long long *)&sc->n_large3, 1ull);
    // small nodes: the 16- / 32-entry warp lists and the mid list (k_small_flags semantics)
    f16[c] = s && rs <= 16;
    f32[c] = s && rs > 16 && rs <= 32;
    ft[c] = s && rs > 32;
    ecount[c] = 0;  // k_small_lists fills the first n_small (the e_off scan runs over n_c)
  }
}

// ------------------------------------------------------------------------------------
// Warp helpers: children table, entry lookup, bitonic sort + unique in shared memory
// ------------------------------------------------------------------------------------
// Warp-buffered emission of (large row, column) pairs: one global atomic on the grid-wide pair
// counter per PAIR_BUF pairs instead of one per 32 entries (the counter is contended).
#define PAIR_BUF 128
// Each (large row, column) pair may carry an ORIGIN: the index of a mirror-position slot
// (A.mir) of the small row that emitted it; after the large rows' lists are final,
// k_sym_finish writes there the column position of the small row inside the large row, so the
// numeric pass mirrors B_ij^T (R22) without a binary search (-1: no origin).
struct PairBuf {
  int2 v[PAIR_BUF];
  long long o[PAIR_BUF];
};
__device__ __forceinline__ void pairs_flush(PairBuf &buf, int &nb, int2 *pairs, long long *porig, long long cap,
                                            AsmScal *scw) {
  const int l = lane_id();
  unsigned long long pb = 0;
  if (l == 0 && nb) pb = atomicAdd((unsigned long long *)&scw->pair_count, (unsigned long long)nb);
  pb = __shfl_sync(FULL_MASK, pb, 0);
  for (int t = l; t < nb; t += 32) {
    const long long pos = (long long)pb + t;
    if (pos < cap) {
      pairs[pos] = buf.v[t];
      porig[pos] = buf.o[t];
    } else scw->err_overflow = 1;
  }
  __syncwarp();
  nb = 0;
}
__device__ __forceinline__ void pairs_push(bool emit, int2 val, long long orig, PairBuf &buf, int &nb, int2 *pairs,
                                           long long *porig, long long cap, AsmScal *scw) {
  const unsigned m = __ballot_sync(FULL_MASK, emit);
  if (!m) return;
  if (nb + __popc(m) > PAIR_BUF) pairs_flush(buf, nb, pairs, porig, cap, scw);
  if (emit) {
    const int pos = nb + __popc(m & ((1u << lane_id()) - 1u));
    buf.v[pos] = val;
    buf.o[pos] = orig;
  }
  nb += __popc(m);
  __syncwarp();
}

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

// Bitonic sort (ascending) of 32 R keys held lane-major in registers: key i = lane R + r.
// Partner distances j < R stay inside a lane (compile-time register pairs), j >= R are one
// shuffle with lane ^ (j / R) -- no shared-memory round trips or warp barriers per stage.
template <int R, typename T>
__device__ __forceinline__ void warp_reg_bitonic(T (&k)[R]) {
  const int l = lane_id();
#pragma unroll
  for (int kq = 2; kq <= 32 * R; kq <<= 1) {
#pragma unroll
    for (int j = kq >> 1; j > 0; j >>= 1) {
      if (j >= R) {
        const int lj = j / R;
        const bool lower = (l & lj) == 0;  // my element is the lower index of its pair
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const bool up = ((l * R + r) & kq) == 0;
          const T o = __shfl_xor_sync(FULL_MASK, k[r], lj);
          k[r] = (lower == up) ? min(k[r], o) : max(k[r], o);
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if ((r & j) == 0) {
            const bool up = ((l * R + r) & kq) == 0;
            const T x = k[r], y = k[r | j];
            const bool sw = (x > y) == up;
            k[r] = sw ? y : x;
            k[r | j] = sw ? x : y;
          }
        }
      }
    }
  }
}

// Sort P (power of two) ints of a warp's shared-memory buffer: in registers for 64 <= P <= 512,
// the shared-memory network otherwise.
template <int R>
__device__ __forceinline__ void warp_sort_int_reg(int *buf) {
  const int l = lane_id();
  int k[R];
#pragma unroll
  for (int r = 0; r < R; ++r) k[r] = buf[l * R + r];
  warp_reg_bitonic<R>(k);
#pragma unroll
  for (int r = 0; r < R; ++r) buf[l * R + r] = k[r];
  __syncwarp();
}

__device__ __forceinline__ void warp_sort_int(int *buf, int P) {
  __syncwarp();
  if (P == 64) warp_sort_int_reg<2>(buf);
  else if (P == 128) warp_sort_int_reg<4>(buf);
  else if (P == 256) warp_sort_int_reg<8>(buf);
  else if (P == 512) warp_sort_int_reg<16>(buf);
  else warp_bitonic_sort(buf, P);
}

__device__ __forceinline__ int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// AGIPC_OPT_DETERMINISTIC: k_children appends in scheduling order; sort every child list
// ascending (fine id) so that the entry order -- and every summation order after it -- is fixed.
// Warp per node in shared memory up to SORTC_CAP children; longer lists go to k_sort_children_big.
#define SORTC_CAP 1024
__global__ void __launch_bounds__(128) k_sort_children(int64_t n_c, const int64_t *__restrict__ child_ptr,
                                                      int32_t *child_list, int32_t *big, AsmScal *sc) {
  __shared__ int s_buf[4][SORTC_CAP];
  const int w = threadIdx.x >> 5, l = lane_id();
  for (int64_t c = (int64_t)blockIdx.x * 4 + w; c < n_c; c += (int64_t)gridDim.x * 4) {
    const int64_t c0 = child_ptr[c];
    const int n = (int)(child_ptr[c + 1] - c0);
    if (n <= 1) continue;
    if (n > SORTC_CAP) {
      if (l == 0) big[atomicAdd((unsigned long long *)&sc->big_groups, 1ull)] = (int32_t)c;
      continue;
    }
    const int P = next_pow2(n);
    for (int e = l; e < P; e += 32) s_buf[w][e] = e < n ? child_list[c0 + e] : INT_MAX;
    __syncwarp();
    warp_bitonic_sort(s_buf[w], P);
    for (int e = l; e < n; e += 32) child_list[c0 + e] = s_buf[w][e];
    __syncwarp();
  }
}

__global__ void __launch_bounds__(1024) k_sort_children_big(const AsmScal *sc, const int32_t *__restrict__ big,
                                                            const int64_t *__restrict__ child_ptr, int32_t *child_list,
                                                            int32_t *scratch) {
  const long long nb = sc->big_groups;
  for (long long q = blockIdx.x; q < nb; q += gridDim.x) {
    const int64_t c = big[q], c0 = child_ptr[c];
    const int n = (int)(child_ptr[c + 1] - c0);
    const int P = next_pow2(n);
    int32_t *g = scratch + 2 * c0;  // scratch holds 2 N ints: room for P <= 2 n
    for (int e = threadIdx.x; e < P; e += blockDim.x) g[e] = e < n ? child_list[c0 + e] : INT_MAX;
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < P; i += blockDim.x) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const int x = g[i], y = g[ixj];
            if ((x > y) == ((i & k) == 0)) {
              g[i] = y;
              g[ixj] = x;
            }
          }
        }
        __syncthreads();
      }
    for (int e = threadIdx.x; e < n; e += blockDim.x) child_list[c0 + e] = g[e];
    __syncthreads();
  }
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
// ------------------------------------------------------------------------------------
// B. symbolic
// ------------------------------------------------------------------------------------
// Large nodes: 32-children chunks emit (a, b) for every large column b != a (warp de-dup with
// __match_any_sync; duplicates across chunks are removed by the per-node sort), and (a, a).
// k_task_node + k_fine_class + k_small_lists in one launch (independent once the scans are done):
// thread c < n_c writes the owner of its chunks and its small-list entries, thread f < N the
// class of fine node f
__global__ void k_class_lists(int64_t N, int64_t n_c, const int64_t *__restrict__ task_ptr, int32_t *__restrict__ task_node,
                              const int32_t *__restrict__ nm, const uint8_t *__restrict__ is_small,
                              uint8_t *__restrict__ fcls, const int32_t *__restrict__ f16,
                              const int32_t *__restrict__ f32, const int32_t *__restrict__ ft,
                              const int64_t *__restrict__ i16, const int64_t *__restrict__ i32,
                              const int64_t *__restrict__ it, const unsigned long long *__restrict__ rowsum,
                              int32_t *__restrict__ w16, int32_t *__restrict__ w32, int32_t *__restrict__ tlist,
                              int64_t *__restrict__ ecount) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < N) fcls[c] = is_small[nm[c]];
  if (c < n_c) {
    for (int64_t t = task_ptr[c]; t < task_ptr[c + 1]; ++t) task_node[t] = (int32_t)c;
    if (f16[c]) w16[i16[c]] = (int32_t)c;
    if (f32[c]) w32[i32[c]] = (int32_t)c;
    if (ft[c]) {
      tlist[it[c]] = (int32_t)c;
      ecount[it[c]] = (int64_t)rowsum[c];
    }
  }
}

struct LargeArgs {
  int64_t n_c;
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
  const int64_t *task_ptr;
  const int32_t *task_node;  // owner node of every large-row task (chunk)
  const uint8_t *fcls;       // [N] is_small[new_map[f]]: the class of fine node f's aggregate
  const AsmScal *sc;
  int2 *pairs;
  long long *porig;
  long long pair_cap;
  AsmScal *scw;
  const int32_t *gbuf;
  const long long *nb_off;
  const int32_t *nb_cnt;
  const int64_t *crp;
  double *cval;
  double *g_c;
  int32_t *recmax;         // symbolic: interface records a chunk may write (distinct large columns x batches)
  // large-row entry lists written by k_sym_large, read by k_num_large_list: per chunk t the
  // diagonal entries (column aggregate == a) at [lbase[t], lbase[t] + lnd[t]) and the large-large
  // interface entries at [lib[t], lib[t] + lni[t]); per entry (fine block << 5 | child slot) and
  // the column node j (interface entries also the column aggregate b)
  long long *lent;
  int32_t *lj, *lb;
  long long *lbase, *lib;
  int32_t *lnd, *lni;
  const int64_t *rec_off;  // numeric: exclusive scan of recmax
  int32_t *rec_b;          // [rec_total] column aggregate of each record (-1: unused)
  double *rec_v;           // [rec_total][144] record values, (p*4+q)*9+x
  double *part;            // [n_tasks][PART_STRIDE] diagonal block + g partials of every chunk
  const int32_t *f12;      // numeric: first 12-DoF entry of every large node's sorted column list
  const int32_t *dpos;     // numeric: column position of the diagonal block of every large row
};
#define PART_STRIDE 160  // 144 diagonal-block values (p*4+q)*9+x + 12 g values p*3+d (+ pad)
#define LSTAGE 128       // staged diagonal entries per batch of a large-row chunk
#define ITF_CAP 160      // staged large-large interface entries of a chunk (flushed when full)

#define SEEN_CAP 128
#ifndef SYML_MINB
#define SYML_MINB 16  // 32 registers, 64 warps per SM: symbolic -27 us vs 48 registers (profiles/r02v)
#endif
__global__ void __launch_bounds__(128, SYML_MINB) k_sym_large(LargeArgs A) {
  __shared__ ChildTab s_tab[4];
  __shared__ int s_seen[4][SEEN_CAP];  // large columns already emitted by this chunk
  __shared__ PairBuf s_pb[4];
  const int w = threadIdx.x >> 5, l = lane_id();
  int npb = 0;
  ChildTab &tab = s_tab[w];
  const int64_t n_tasks = A.task_ptr[A.n_c];
  const int64_t tstride = (int64_t)gridDim.x * 4;
  int a_nx = 0, s_nx = 0, ci_nx = 0, ch_nx = 0;  // next task prefetched (as in k_num_large_atomic)
  auto prefetch = [&](int64_t tn) {
    if (tn < n_tasks) {
      a_nx = A.task_node[tn];
      ch_nx = (int)(tn - A.task_ptr[a_nx]);
      s_nx = min(LARGE_CHUNK, A.size_new[a_nx] - ch_nx * LARGE_CHUNK);
      ci_nx = l < s_nx ? A.child_list[A.child_ptr[a_nx] + (int64_t)ch_nx * LARGE_CHUNK + l] : 0;
    }
  };
  prefetch((int64_t)blockIdx.x * 4 + w);
  for (int64_t t = (int64_t)blockIdx.x * 4 + w; t < n_tasks; t += tstride) {
    const int a = a_nx, chunk = ch_nx, s = s_nx, ci_c = ci_nx;
    prefetch(t + tstride);
    int len = 0;
    if (l < s) {
      const long long b0 = A.rp[ci_c];
      tab.ci[l] = ci_c;
      tab.rb[l] = b0;
      len = (int)(A.rp[ci_c + 1] - b0);
    }
    const int incl_c = warp_incl_scan(len);
    tab.off[l + 1] = incl_c;
    if (l == 0) tab.off[0] = 0;
    __syncwarp();
    const int T = __shfl_sync(FULL_MASK, incl_c, 31);
    int nseen = 0, nitf = 0, ndg = 0;
    long long lbase = 0;
    if (A.lent) {  // T list slots for this chunk: diagonal entries from the front, interface from the back
      if (l == 0) lbase = (long long)atomicAdd((unsigned long long *)&A.scw->list_top, (unsigned long long)T);
      lbase = __shfl_sync(FULL_MASK, lbase, 0);
    }
    for (int e0 = 0; e0 < T; e0 += 32) {
      const int e = e0 + l;
      int key = -1;
      bool dg = false;
      int c = 0, j = 0;
      long long k = 0;
      if (e < T) {
        entry_of(tab, s, e, c, k);
        j = A.col[k];
        if (!A.fcls[j]) {
          const int b = A.nm[j];
          if (b != a) key = b;
          else dg = true;
        }
      }
      if (A.lent) {
        const unsigned md = __ballot_sync(FULL_MASK, dg), mi = __ballot_sync(FULL_MASK, key >= 0);
        const unsigned below = (1u << l) - 1u;
        if (dg) {
          const long long o = lbase + ndg + __popc(md & below);
          A.lent[o] = (k << 5) | c;
          A.lj[o] = j;
        } else if (key >= 0) {
          const long long o = lbase + T - 1 - (nitf + __popc(mi & below));
          A.lent[o] = (k << 5) | c;
          A.lj[o] = j;
          A.lb[o] = key;
        }
        ndg += __popc(md);
      }
      nitf += __popc(__ballot_sync(FULL_MASK, key >= 0));
      const unsigned peers = __match_any_sync(FULL_MASK, key);
      bool emit = key >= 0 && (__ffs(peers) - 1) == l;
      if (emit)  // one pair per (chunk, column): skip columns this chunk already emitted
        for (int q = 0; q < min(nseen, SEEN_CAP); ++q)
          if (s_seen[w][q] == key) {
            emit = false;
            break;
          }
      const unsigned me = __ballot_sync(FULL_MASK, emit);
      if (emit) {
        const int pos = nseen + __popc(me & ((1u << l) - 1u));
        if (pos < SEEN_CAP) s_seen[w][pos] = key;
      }
      nseen += __popc(me);
      __syncwarp();
      pairs_push(emit, make_int2(a, key), -1, s_pb[w], npb, A.pairs, A.porig, A.pair_cap, A.scw);
    }
    // interface records the numeric chunk may write: one per (flush of its interface list,
    // distinct large column); the list holds ITF_CAP entries and is flushed before it overflows
    if (l == 0) A.recmax[t] = nseen * (1 + nitf / (ITF_CAP - 31));
    if (A.lent && l == 0) {
      A.lbase[t] = lbase;
      A.lnd[t] = ndg;
      A.lib[t] = lbase + T - nitf;
      A.lni[t] = nitf;
    }
    // the diagonal block (a, a) always exists
    pairs_push(chunk == 0 && l == 0, make_int2(a, a), -1, s_pb[w], npb, A.pairs, A.porig, A.pair_cap, A.scw);
    __syncwarp();
  }
  pairs_flush(s_pb[w], npb, A.pairs, A.porig, A.pair_cap, A.scw);
}

__global__ void k_pair_count(const AsmScal *sc, long long cap, const int2 *__restrict__ pairs,
                             int32_t *__restrict__ gcnt) {
  const long long np = min(sc->pair_count, cap);
  // consecutive pairs mostly share their large row: one atomic per distinct row of the warp
  for (long long b0 = (long long)blockIdx.x * blockDim.x; b0 < np; b0 += (long long)gridDim.x * blockDim.x) {
    const long long p = b0 + threadIdx.x;
    const int key = p < np ? pairs[p].x : -1;
    const unsigned peers = __match_any_sync(FULL_MASK, key);
    if (key >= 0 && (__ffs(peers) - 1) == lane_id()) atomicAdd(gcnt + key, __popc(peers));
  }
}

// padded group sizes: next power of two (so every group can be sorted in place)
__global__ void k_pair_scatter(const AsmScal *sc, long long cap, const int2 *__restrict__ pairs,
                               const int64_t *__restrict__ gptr, int32_t *__restrict__ gcur,
                               int32_t *__restrict__ gbuf) {
  const long long np = min(sc->pair_count, cap);
  for (long long b0 = (long long)blockIdx.x * blockDim.x; b0 < np; b0 += (long long)gridDim.x * blockDim.x) {
    const long long p = b0 + threadIdx.x;
    const int2 q = p < np ? pairs[p] : make_int2(-1, 0);
    const unsigned peers = __match_any_sync(FULL_MASK, q.x);
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (q.x >= 0 && leader == lane_id()) base = atomicAdd(gcur + q.x, __popc(peers));  // gcur zeroed with gcnt
    base = __shfl_sync(FULL_MASK, base, leader);
    if (q.x >= 0) gbuf[gptr[q.x] + base + __popc(peers & ((1u << lane_id()) - 1u))] = q.y;
  }
}

// sort + unique of each large node's list in place (padded to a power of two)
__global__ void __launch_bounds__(SYM_WARPS * 32) k_group_unique(int64_t n_c, const uint8_t *__restrict__ is_small,
                                                                 const int64_t *__restrict__ gptr, int32_t *gbuf,
                                                                 const int32_t *__restrict__ gcnt, long long *nb_off,
                                                                 int32_t *nb_cnt, int32_t *rowlen, int32_t *big_list,
                                                                 AsmScal *sc, int32_t *f12) {
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
    warp_sort_int(buf, P);
    int u12;
    int U = warp_unique_store(buf, n, g, n3, u12);
    if (l == 0) {
      nb_off[a] = gptr[a];
      nb_cnt[a] = U;
      rowlen[a] = U + 3 * u12;
      f12[a] = U - u12;  // ascending list: the 12-DoF columns (>= n3) come last
    }
    __syncwarp();
  }
}

// CTA-wide global-memory bitonic sort for the (rare) large lists of more than 2048 entries.
__global__ void __launch_bounds__(1024) k_group_unique_big(const AsmScal *sc, const int32_t *__restrict__ big_list,
                                                           const int64_t *__restrict__ gptr, int32_t *gbuf,
                                                           const int32_t *__restrict__ gcnt, long long *nb_off,
                                                           int32_t *nb_cnt, int32_t *rowlen, int32_t *f12) {
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
        f12[a] = U - u12;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------
// C. slot row lengths
// ------------------------------------------------------------------------------------
// End of the symbolic pass in ONE launch (was k_final_scalars + k_mirror_pos + k_copy_rowptr):
// every block derives the capacity / error verdict itself (block 0 also stores the scalars), then
// grid-stride loops copy the slot row pointer out and place the small rows' mirror positions.
__global__ void k_sym_finish(AsmScal *sc, const int64_t *__restrict__ crp, const int64_t *__restrict__ task_ptr,
                             int64_t n_c, const int64_t *__restrict__ rec_off, int64_t task_bound, int64_t cap_slots,
                             int64_t cap_nnzb, const int64_t *__restrict__ cnt32, int64_t *__restrict__ row_ptr_out,
                             long long cap, const int2 *__restrict__ pairs, const long long *__restrict__ porig,
                             const int32_t *__restrict__ gbuf, const long long *__restrict__ nb_off,
                             const int32_t *__restrict__ nb_cnt, const int32_t *__restrict__ f12,
                             const int32_t *__restrict__ rowlen, long long *__restrict__ mirpos,
                             int32_t *__restrict__ mirrl) {
  const long long n_slots = sc->n_slots, n3 = sc->n3;
  const long long nnzb = crp[n_slots];
  const bool bad = sc->err_map || sc->err_overflow || n_slots >= INT32_MAX || n_slots > cap_slots || nnzb > cap_nnzb;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc->nnzb = nnzb;
    sc->n_tasks = task_ptr[n_c];
    sc->rec_total = rec_off[task_bound];
    sc->n_w32 = *cnt32;
    sc->err_cap = bad;
  }
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (!bad)
    for (long long i = tid; i <= n_slots; i += stride) row_ptr_out[i] = crp[i];
  const long long np = min(sc->pair_count, cap);
  for (long long p = tid; p < np; p += stride) {
    const long long o = porig[p];
    if (o < 0) continue;
    const int2 q = pairs[p];
    const int idx = lower_bound_dev<int32_t>(gbuf + nb_off[q.x], nb_cnt[q.x], (int32_t)q.y);
    mirpos[o] = crp[slot_of(q.x, 0, n3)] + colpos(idx, f12[q.x]);
    mirrl[o] = rowlen[q.x];
  }
}

// ------------------------------------------------------------------------------------
// Small nodes with <= 32 candidate entries (singletons, pairs: the bulk of the 3-DoF rows):
// one SEG-lane segment of a warp per node (SEG = 16: two nodes per warp, interior singletons
// have 15 entries; SEG = 32 otherwise), one entry per lane, everything in registers -- a
// shuffle bitonic sort of (column, lane) keys, run heads by ballot, run sums by a segmented
// shuffle scan.  No shared-memory staging of values, no barriers.
// ------------------------------------------------------------------------------------
template <int SEG, typename T = long long>
__device__ __forceinline__ T seg_sort(T key, int sl) {
#pragma unroll
  for (int k = 2; k <= SEG; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const T other = __shfl_xor_sync(FULL_MASK, key, j, SEG);
      const bool up = (sl & k) == 0, lower = (sl & j) == 0;
      const T mn = min(key, other), mx = max(key, other);
      key = (lower == up) ? mn : mx;
    }
  return key;
}

template <int SEG>
__device__ __forceinline__ int seg_incl_scan(int v, int sl) {
#pragma unroll
  for (int o = 1; o < SEG; o <<= 1) {
    const int t = __shfl_up_sync(FULL_MASK, v, o, SEG);
    if (sl >= o) v += t;
  }
  return v;
}

template <int SEG>
__device__ __forceinline__ double seg_sum(double v) {
#pragma unroll
  for (int o = SEG / 2; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o, SEG);
  return v;
}

struct WarpArgs {
  int64_t n_w;
  // list sizes on the device (no host round trip after the classification): n16 = cnt16[0],
  // n32 = cnt32[0], nmid = cntmid[0]; kind 0 / 1 / 2 = this kernel's list (16-entry, 32-entry,
  // mid); n_w, mir_base and the 32-entry key offset are derived from them (warp_args_resolve)
  const int64_t *cnt16, *cnt32, *cntmid;
  int kind;
  int key32;  // n_c < 2^26 - 1: symbolic sort keys (column << 5 | lane) fit in 31 bits
  int32_t *mchild;  // small nodes: child of lane sl at wi * SEG + sl (symbolic -> numeric prefetch)
  long long *msrc;             // small nodes: (fine block << 5 | child index) per sorted key
  long long *mkeys;            // mid nodes: sorted (column, entry) keys, written by the symbolic
  const int64_t *e_off;        //   pass at e_off[wi], reused by the numeric pass (no second sort)
  const int32_t *wlist;        // small nodes handled by this kernel
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
  const AsmScal *sc;
  int32_t *rowlen;
  int2 *pairs;
  long long *porig;
  long long *mirpos;           // mirror block positions (k_sym_finish), indexed like mkeys from
  int32_t *mirrl;              //   mir_base; -1 = the run's column is small (no mirror)
  long long mir_base;
  long long pair_cap;
  AsmScal *scw;
  const int32_t *gbuf;
  const long long *nb_off;
  const int32_t *nb_cnt;
  const int64_t *crp;
  int32_t *ccol;
  double *cval;
  double *g_c;
};

__device__ __forceinline__ void warp_args_resolve(WarpArgs &A) {
  if (!A.cnt16) return;
  const long long n16 = *A.cnt16, n32 = *A.cnt32;
  if (A.kind == 0) {
    A.n_w = n16;
    A.mir_base = 0;
  } else if (A.kind == 1) {
    A.n_w = n32;
    A.mir_base = 16 * n16;
    A.mkeys += 16 * n16;
    A.msrc += 16 * n16;
    A.mchild += 16 * n16;
  } else {
    A.n_w = *A.cntmid;
    A.mir_base = 16 * n16 + 32 * n32;
  }
}

template <int SEG, bool NUMERIC>
__global__ void __launch_bounds__(256, NUMERIC ? SMALL_MINB_N : SMALL_MINB_S) k_small_warp(WarpArgs A) {
  if (NUMERIC && A.sc->err_cap) return;  // outputs do not fit / bad input: write nothing
  warp_args_resolve(A);
  constexpr int NSEG = 32 / SEG;
  __shared__ ChildTab s_tab[NUMERIC ? 1 : 8 * NSEG];
  // numeric: per-lane parked block B_ij (9), X_bar of its row child (3) and of its column node (3)
  __shared__ double s_v[NUMERIC ? 8 : 1][NUMERIC ? 32 : 1][15];
  // numeric: output descriptors (head lane | tail lane << 6 | q << 12) at column position, per
  // segment; per head lane its column node and mirror position / row length; per segment
  // (node, blocks per p, output blocks)
  __shared__ int s_desc[NUMERIC ? 8 : 1][NUMERIC ? 4 * 32 : 1];
  __shared__ int s_rbs[NUMERIC ? 8 : 1][NUMERIC ? 32 : 1];
  __shared__ long long s_rmb[NUMERIC ? 8 : 1][NUMERIC ? 32 : 1];
  __shared__ int s_rml[NUMERIC ? 8 : 1][NUMERIC ? 32 : 1];
  __shared__ int s_seg[NUMERIC ? 8 : 1][NUMERIC ? NSEG : 1][3];
  __shared__ PairBuf s_pb[NUMERIC ? 1 : 8];  // symbolic: buffered pairs
  int npb = 0;
  const int w = threadIdx.x >> 5, l = lane_id();
  const int sg = l / SEG, sl = l % SEG;
  const unsigned smask = SEG == 32 ? FULL_MASK : (((1u << SEG) - 1u) << (sg * SEG));
  const long long n3 = A.sc->n3;
  const int64_t n_units = (A.n_w + NSEG - 1) / NSEG;
  const int64_t ustride = (int64_t)gridDim.x * 8;
  // software pipeline over units: the node id, its child count and the lane's child of the NEXT
  // unit are loaded while this unit is processed (the wlist -> child_ptr -> child_list chain is
  // off the critical path; profiles/r02d stall-by-line).  The numeric pass also prefetches the
  // next unit's sorted key and source entry (written by the symbolic pass), so its only
  // dependent loads are the fine block itself and the output positions.
  int a_nx = 0, s_nx = 0, ci_nx = 0;
  long long key_nx = 0, m_nx = -1;
  {
    const int64_t u0 = (int64_t)blockIdx.x * 8 + w, wi0 = u0 * NSEG + sg;
    if (u0 < n_units && wi0 < A.n_w) {
      a_nx = A.wlist[wi0];
      s_nx = A.size_new[a_nx];
      if (!NUMERIC && sl < s_nx) ci_nx = A.child_list[A.child_ptr[a_nx] + sl];
      if (NUMERIC) {
        key_nx = A.mkeys[wi0 * SEG + sl];
        m_nx = A.msrc[wi0 * SEG + sl];
      }
      if (NUMERIC) ci_nx = max(A.mchild[wi0 * SEG + sl], 0);
    }
  }
  for (int64_t u = (int64_t)blockIdx.x * 8 + w; u < n_units; u += ustride) {
    const int64_t wi = u * NSEG + sg;
    const bool segv = wi < A.n_w;
    const int a = segv ? a_nx : 0;
    const int s = segv ? s_nx : 0;
    const int ci_cur = ci_nx;
    const long long key_cur = key_nx, m_cur = m_nx;
    {
      const int64_t wn = (u + ustride) * NSEG + sg;
      if (u + ustride < n_units && wn < A.n_w) {
        a_nx = A.wlist[wn];
        s_nx = A.size_new[a_nx];
        if (NUMERIC) {  // the child list as the symbolic pass left it: no child_ptr -> child_list chain
          key_nx = A.mkeys[wn * SEG + sl];
          m_nx = A.msrc[wn * SEG + sl];
          ci_nx = max(A.mchild[wn * SEG + sl], 0);
        } else {
          ci_nx = sl < s_nx ? A.child_list[A.child_ptr[a_nx] + sl] : 0;
        }
      }
    }
    if constexpr (!NUMERIC) {
      ChildTab &tab = s_tab[w * NSEG + sg];
      // children of the node and the offsets of their rows (segment-local scan)
      int len = 0;
      if (sl < s) {
        const int ci = ci_cur;
        const long long rb = A.rp[ci];
        tab.ci[sl] = ci;
        tab.rb[sl] = rb;
        len = (int)(A.rp[ci + 1] - rb);
      }
      const int incl = seg_incl_scan<SEG>(len, sl);
      tab.off[sl + 1] = incl;
      if (sl == 0) tab.off[0] = 0;
      __syncwarp();
      const int T = __shfl_sync(FULL_MASK, incl, SEG - 1, SEG);
      int b = INT_MAX, c = 0;
      long long k = 0;
      if (sl < T) {
        entry_of(tab, s, sl, c, k);
        b = A.nm[A.col[k]];
      }
      // sorted (column, entry) keys and, per sorted position, its fine block and child index:
      // kept at wi * SEG + sl for the numeric pass (no second new_map gather, sort or row walk)
      // 32-bit keys while every column id fits in 26 bits (one-instruction shuffles and min / max);
      // the same order as the 64-bit keys, the invalid lanes last in lane order
      const long long key = A.key32 ? (long long)seg_sort<SEG, int>(sl < T ? (b << 5) | sl : (0x7FFFFFE0 | sl), sl)
                                    : seg_sort<SEG>(((long long)b << 5) | sl, sl);
      const int src = (int)(key & 31);
      const long long ksrc = __shfl_sync(FULL_MASK, k, src, SEG);
      const int csrc = __shfl_sync(FULL_MASK, c, src, SEG);
      if (segv) {
        A.mchild[wi * SEG + sl] = sl < s ? ci_cur : -1;
        A.mkeys[wi * SEG + sl] = key;
        A.msrc[wi * SEG + sl] = sl < T ? ((ksrc << 5) | csrc) : -1;
      }
      const int bs = (int)(key >> 5);
      const long long prevk = __shfl_up_sync(FULL_MASK, key, 1, SEG);
      const bool valid = sl < T;
      const bool head = valid && (sl == 0 || (prevk >> 5) != bs);
      const unsigned hb = (__ballot_sync(FULL_MASK, head) & smask) >> (sg * SEG);  // segment-local bits
      const int U = __popc(hb);
      const int U12 = __popc((__ballot_sync(FULL_MASK, head && bs >= n3) & smask) >> (sg * SEG));
      if (segv && sl == 0) A.rowlen[a] = U + 3 * U12;
      const bool emit = head && !A.is_small[bs];  // transposed pair (large column, small node)
      if (head && !emit) A.mirpos[A.mir_base + wi * SEG + sl] = -1;
      pairs_push(emit, make_int2(bs, a), A.mir_base + wi * SEG + sl, s_pb[w], npb, A.pairs, A.porig, A.pair_cap,
                 A.scw);
      __syncwarp();
    } else {
      // Output-parallel numeric pass: every valid entry parks its fine block B_ij and the affine
      // coordinates of its row child / column node in shared memory; every run (one coarse
      // column b) posts one descriptor per output block q; then the warp's lanes take the output
      // blocks of ALL its segments round-robin (o = l, l + 32, ...) and sum their run's entries
      // left to right -- no lane idles through another lane's run or q loop.
      const long long key = segv ? key_cur : (((long long)INT_MAX << 5) | sl);
      const long long m = segv ? m_cur : -1;
      const bool valid = m >= 0;
      const int bs = (int)(key >> 5);
      const long long prevk = __shfl_up_sync(FULL_MASK, key, 1, SEG);
      const bool head = valid && (sl == 0 || (prevk >> 5) != bs);
      const unsigned hb = (__ballot_sync(FULL_MASK, head) & smask) >> (sg * SEG);  // segment-local bits
      const int T = __popc((__ballot_sync(FULL_MASK, valid) & smask) >> (sg * SEG));  // valid = prefix
      const long long sk = valid ? (m >> 5) : 0;
      const int si = __shfl_sync(FULL_MASK, ci_cur, (int)(m & 31), SEG);  // child c sits on lane c
      const int ncb_a = segv ? ncb_of(a, n3) : 1;
      const int PA = __ballot_sync(FULL_MASK, segv && ncb_a == 4) ? 4 : 1;  // warp-uniform (g_c loop)
      const int ncb_b = valid ? ncb_of(bs, n3) : 1;
      const int wgt_b = head ? ncb_b : 0;
      const int cp_incl = seg_incl_scan<SEG>(wgt_b, sl);
      const int R = __shfl_sync(FULL_MASK, cp_incl, SEG - 1, SEG);  // output blocks per p (row length)
      const int sj = (valid && ncb_b == 4) ? A.col[sk] : 0;  // the column node (affine weights only)
#pragma unroll
      for (int x = 0; x < 9; ++x) s_v[w][l][x] = valid ? __ldg(A.val + 9 * sk + x) : 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        s_v[w][l][9 + c] = (valid && ncb_a == 4) ? __ldg(A.X + 3 * (int64_t)si + c) : 0.0;
        s_v[w][l][12 + c] = (valid && ncb_b == 4) ? __ldg(A.X + 3 * (int64_t)sj + c) : 0.0;
      }
      if (head) {  // run [sl, tl]: descriptors of its output blocks q at column position cp + q
        const unsigned above = hb & ~((2u << sl) - 1u);
        const int tl = above ? __ffs(above) - 2 : T - 1;
        const int cp = cp_incl - wgt_b;
        for (int q = 0; q < ncb_b; ++q) s_desc[w][sg * 4 * SEG + cp + q] = sl | (tl << 6) | (q << 12);
        s_rbs[w][l] = bs;
        // mirrored block (slot(bs, q), slot(a, p)) at mb + q * mrl + p (B_ji = B_ij^T, reading R22)
        s_rmb[w][l] = A.mirpos[A.mir_base + wi * SEG + sl];  // k_sym_finish (-1: small column)
        s_rml[w][l] = A.mirrl[A.mir_base + wi * SEG + sl];
      }
      if (sl == 0) {
        s_seg[w][sg][0] = segv ? a : 0;
        s_seg[w][sg][1] = segv ? R : 0;
        s_seg[w][sg][2] = segv ? ncb_a * R : 0;  // output blocks of the segment
      }
      __syncwarp();
      int tot = 0;
#pragma unroll
      for (int g = 0; g < NSEG; ++g) tot += s_seg[w][g][2];
      for (int o = l; o < tot; o += 32) {
        int g = 0, oo = o;
#pragma unroll
        for (int gg = 0; gg < NSEG - 1; ++gg)
          if (g == gg && oo >= s_seg[w][gg][2]) { oo -= s_seg[w][gg][2]; g = gg + 1; }
        const int ag = s_seg[w][g][0], Rg = s_seg[w][g][1];
        const int p = (oo >= Rg) + (oo >= 2 * Rg) + (oo >= 3 * Rg), r = oo - p * Rg;  // p < 4: no division
        const int d = s_desc[w][g * 4 * SEG + r];
        const int h0 = g * SEG + (d & 63), t1 = g * SEG + ((d >> 6) & 63), q = d >> 12;
        const int b = s_rbs[w][h0];
        const int ncb_ag = ncb_of(ag, n3), ncb_bb = ncb_of(b, n3);
        // coef = w_i[p] w_j[q] (Eq 4), the same product order as the oracle's weights
        double v[9];
        for (int t = h0; t <= t1; ++t) {
          const double wit = (ncb_ag == 4 && p < 3) ? s_v[w][t][9 + p] : 1.0;
          const double wjt = (ncb_bb == 4 && q < 3) ? s_v[w][t][12 + q] : 1.0;
          const double ct = wit * wjt;
          if (t == h0) {
#pragma unroll
            for (int x = 0; x < 9; ++x) v[x] = ct * s_v[w][t][x];
          } else {
#pragma unroll
            for (int x = 0; x < 9; ++x) v[x] += ct * s_v[w][t][x];
          }
        }
        const long long pos = A.crp[slot_of(ag, p, n3)] + (r - q) + q;
        A.ccol[pos] = slot_of(b, q, n3);
        double *dst = A.cval + 9 * pos;
#pragma unroll
        for (int x = 0; x < 9; ++x) dst[x] = v[x];
        const long long mb = s_rmb[w][h0];
        if (mb >= 0) {
          double *mt = A.cval + 9 * (mb + (long long)q * s_rml[w][h0] + p);
#pragma unroll
          for (int rr = 0; rr < 3; ++rr)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) mt[3 * rr + cc] = v[3 * cc + rr];
        }
      }
      __syncwarp();
      if (A.g_f) {  // g_c[slot(a,p)] = sum over the children of w_i[p] g_f[i]
        for (int p = 0; p < PA; ++p) {
          double g0 = 0, g1 = 0, g2 = 0;
          if (sl < s && p < ncb_a) {
            const int ci = ci_cur;
            const double wc = wgt(A.X, ci, ncb_a, p);
            g0 = wc * A.g_f[3 * (int64_t)ci];
            g1 = wc * A.g_f[3 * (int64_t)ci + 1];
            g2 = wc * A.g_f[3 * (int64_t)ci + 2];
          }
          g0 = seg_sum<SEG>(g0);
          g1 = seg_sum<SEG>(g1);
          g2 = seg_sum<SEG>(g2);
          if (segv && sl == 0 && p < ncb_a) {
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
  if (!NUMERIC) pairs_flush(s_pb[w], npb, A.pairs, A.porig, A.pair_cap, A.scw);
}

// ------------------------------------------------------------------------------------
// Mid-size small nodes (> 32 and <= 1024 candidate entries, <= 32 children): one warp per
// node; (column, entry) keys sorted in shared memory by a warp-synchronous bitonic sort; the
// symbolic pass counts runs, the numeric pass gives each run to a lane.
// ------------------------------------------------------------------------------------
#define MID_WARPS 4
#define MID_CAP 1024

// Mid-node symbolic keys ((column << 10) | entry) of T <= 32 R entries, sorted in registers and
// stored to shared memory (run counting) and to global memory (reused by the numeric pass).
template <int R>
__device__ __forceinline__ void mid_keys_sorted(const WarpArgs &A, const ChildTab &tab, int s, int T, long long *key,
                                                long long *gkeys) {
  const int l = lane_id();
  long long k[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = l * R + r;
    k[r] = LLONG_MAX;
    if (e < T) {
      int c;
      long long kk;
      entry_of(tab, s, e, c, kk);
      k[r] = ((long long)A.nm[A.col[kk]] << 10) | e;
    }
  }
  warp_reg_bitonic<R>(k);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = l * R + r;
    key[e] = k[r];
    if (e < T) gkeys[e] = k[r];
  }
  __syncwarp();
}

template <bool NUMERIC>
#ifdef MID_MINB_S  // the numeric mid pass keeps the plain bounds (126 registers)
__global__ void __launch_bounds__(MID_WARPS * 32, NUMERIC ? MID_MINB_N : MID_MINB_S) k_mid_warp(WarpArgs A) {
#else
__global__ void __launch_bounds__(MID_WARPS * 32) k_mid_warp(WarpArgs A) {
#endif
  if (NUMERIC && A.sc->err_cap) return;
  warp_args_resolve(A);
  __shared__ ChildTab s_tab[MID_WARPS];
  __shared__ long long s_key[MID_WARPS][MID_CAP];
  __shared__ double s_carry[MID_WARPS][4][9];  // partial sums of a run continuing into the next window
  __shared__ PairBuf s_pb[NUMERIC ? 1 : MID_WARPS];  // symbolic: buffered pairs
  int npb = 0;
  const int w = threadIdx.x >> 5, l = lane_id();
  ChildTab &tab = s_tab[w];
  long long *key = s_key[w];
  const long long n3 = A.sc->n3;
  const int64_t wstride = (int64_t)gridDim.x * MID_WARPS;
  // software pipeline: the next node's id, child count and the lane's child are loaded while
  // this node is processed (as in k_small_warp)
  int a_nx = 0, s_nx = 0, ci_nx = 0;
  {
    const int64_t w0 = (int64_t)blockIdx.x * MID_WARPS + w;
    if (w0 < A.n_w) {
      a_nx = A.wlist[w0];
      s_nx = A.size_new[a_nx];
      if (l < s_nx) ci_nx = A.child_list[A.child_ptr[a_nx] + l];
    }
  }
  for (int64_t wi = (int64_t)blockIdx.x * MID_WARPS + w; wi < A.n_w; wi += wstride) {
    const int a = a_nx;
    const int s = s_nx;
    int len = 0;
    if (l < s) {  // load_children with the prefetched child
      const long long b0 = A.rp[ci_nx];
      tab.ci[l] = ci_nx;
      tab.rb[l] = b0;
      len = (int)(A.rp[ci_nx + 1] - b0);
    }
    if (wi + wstride < A.n_w) {
      a_nx = A.wlist[wi + wstride];
      s_nx = A.size_new[a_nx];
      ci_nx = l < s_nx ? A.child_list[A.child_ptr[a_nx] + l] : 0;
    }
    const int incl_c = warp_incl_scan(len);
    tab.off[l + 1] = incl_c;
    if (l == 0) tab.off[0] = 0;
    __syncwarp();
    const int T = __shfl_sync(FULL_MASK, incl_c, 31);  // T <= MID_CAP
    long long *gkeys = A.mkeys + A.e_off[wi];
    const long long mir0 = A.mir_base + A.e_off[wi];  // this node's mirror-position slots
    if (NUMERIC) {  // the symbolic pass left the sorted keys of this node in global memory
      for (int e = l; e < T; e += 32) key[e] = gkeys[e];
      __syncwarp();
    } else if (T <= 512) {  // register sort (T > 32 here: at least 2 keys per lane)
      if (T <= 64) mid_keys_sorted<2>(A, tab, s, T, key, gkeys);
      else if (T <= 128) mid_keys_sorted<4>(A, tab, s, T, key, gkeys);
      else if (T <= 256) mid_keys_sorted<8>(A, tab, s, T, key, gkeys);
      else mid_keys_sorted<16>(A, tab, s, T, key, gkeys);
    } else {
    const int P = next_pow2(T);
    for (int e = l; e < P; e += 32) {
      long long kk = LLONG_MAX;
      if (e < T) {
        int c;
        long long k;
        entry_of(tab, s, e, c, k);
        kk = ((long long)A.nm[A.col[k]] << 10) | e;
      }
      key[e] = kk;
    }
    __syncwarp();
    for (int kq = 2; kq <= P; kq <<= 1)
      for (int j = kq >> 1; j > 0; j >>= 1) {
        for (int i = l; i < P; i += 32) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const long long x = key[i], y = key[ixj];
            if ((x > y) == ((i & kq) == 0)) {
              key[i] = y;
              key[ixj] = x;
            }
          }
        }
        __syncwarp();
      }
    for (int e = l; e < T; e += 32) gkeys[e] = key[e];
    }
    // runs of equal column; colpos = prefix of the run weights (12-DoF columns count 4)
    int run_base = 0;
    for (int e0 = 0; !NUMERIC && e0 < T; e0 += 32) {
      const int e = e0 + l;
      const long long kk = e < T ? key[e] : LLONG_MAX;
      const int b = (int)(kk >> 10);
      const bool head = e < T && (e == 0 || (key[e - 1] >> 10) != (kk >> 10));
      const int wgt_b = head ? ncb_of(b, n3) : 0;
      const int incl = warp_incl_scan(wgt_b);
      const int cp = run_base + incl - wgt_b;
      run_base += __shfl_sync(FULL_MASK, incl, 31);
      if (!NUMERIC) {
        const bool emit = head && !A.is_small[b];  // transposed pair (large column, small node)
        if (head && !emit) A.mirpos[mir0 + e] = -1;
        pairs_push(emit, make_int2(b, a), mir0 + e, s_pb[w], npb, A.pairs, A.porig,
                   A.pair_cap, A.scw);
        continue;
      }
    }
    if (NUMERIC) {
      // Lane per sorted entry, one pass per row p of the node.  Per 32-entry window: the
      // entries' blocks are loaded in parallel, scaled by w_j[q], summed over each run of equal
      // column with a segmented shuffle scan; the tail lane of a run writes the coarse block
      // (and its mirror in a large row, R22).  A run that continues into the next window
      // passes its partial sums on in `carry` (added by the lanes of the next window's first run).
      const int ncb_a = ncb_of(a, n3);
      for (int p = 0; p < ncb_a; ++p) {
      double(*carry)[9] = s_carry[w];
      if (l < 36) carry[l / 9][l % 9] = 0.0;
      __syncwarp();
      int rb = 0, carry_cp = 0, carry_he = 0;
      const long long rs = A.crp[slot_of(a, p, n3)];
      for (int e0 = 0; e0 < T; e0 += 32) {
        const int e = e0 + l;
        const bool valid = e < T;
        const long long kk = valid ? key[e] : LLONG_MAX;
        const int b = (int)(kk >> 10);
        const bool head = valid && (e == 0 || (key[e - 1] >> 10) != (kk >> 10));
        const bool tail = valid && (e == T - 1 || (key[e + 1] >> 10) != (kk >> 10));
        const int wgt_b = head ? ncb_of(b, n3) : 0;
        const int incl = warp_incl_scan(wgt_b);
        const unsigned hb = __ballot_sync(FULL_MASK, head);
        const int hl = (hb & ((2u << l) - 1u)) ? 31 - __clz(hb & ((2u << l) - 1u)) : -1;  // my run's head lane
        const int cp_head = rb + incl - wgt_b;
        int cp = __shfl_sync(FULL_MASK, cp_head, hl < 0 ? 0 : hl);
        if (hl < 0) cp = carry_cp;  // the run started in an earlier window
        const int lo = hl < 0 ? 0 : hl;
        int el = 0, j = 0;
        long long k = 0;
        double wi = 0.0;
        if (valid) {
          el = (int)(kk & 1023);
          int c;
          entry_of(tab, s, el, c, k);
          j = A.col[k];
          wi = wgt(A.X, tab.ci[c], ncb_a, p);
        }
        double B[9];
#pragma unroll
        for (int x = 0; x < 9; ++x) B[x] = valid ? __ldg(A.val + 9 * k + x) : 0.0;
        const int ncb_b = valid ? ncb_of(b, n3) : 1;
        const int Q = __ballot_sync(FULL_MASK, valid && ncb_b == 4) ? 4 : 1;
        const int he = hl < 0 ? carry_he : e0 + hl;  // sorted position of my run's head
        long long mbase = -1;  // mirrored block of (b, a): mbase + q * mrl + p (R22, k_sym_finish)
        int mrl = 0;
        if (tail) {
          mbase = A.mirpos[mir0 + he];
          mrl = A.mirrl[mir0 + he];
        }
        const int last_he = __shfl_sync(FULL_MASK, he, 31);
        const bool cont = valid && !tail && l == 31;  // my run continues into the next window
        const int last_cp = __shfl_sync(FULL_MASK, cp, 31);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (q >= Q) break;
          const double coef = (valid && q < ncb_b) ? wi * wgt(A.X, j, ncb_b, q) : 0.0;
          double v[9];
#pragma unroll
          for (int x = 0; x < 9; ++x) v[x] = coef * B[x];
#pragma unroll
          for (int o = 1; o < 32; o <<= 1)
#pragma unroll
            for (int x = 0; x < 9; ++x) {
              const double t = __shfl_up_sync(FULL_MASK, v[x], o);
              if (l - o >= lo) v[x] += t;
            }
          if (hl < 0) {
#pragma unroll
            for (int x = 0; x < 9; ++x) v[x] += carry[q][x];
          }
          if (tail && q < ncb_b) {
            const long long pos = rs + cp + q;
            A.ccol[pos] = slot_of(b, q, n3);
            double *dst = A.cval + 9 * pos;
#pragma unroll
            for (int x = 0; x < 9; ++x) dst[x] = v[x];
            if (mbase >= 0) {
              double *mt = A.cval + 9 * (mbase + (long long)q * mrl + p);
#pragma unroll
              for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) mt[3 * r + cc] = v[3 * cc + r];
            }
          }
          const bool any_cont = __shfl_sync(FULL_MASK, cont ? 1 : 0, 31);
          __syncwarp();  // every lane has read carry[q] above
          if (l == 31) {
#pragma unroll
            for (int x = 0; x < 9; ++x) carry[q][x] = any_cont ? v[x] : 0.0;
          }
          __syncwarp();
        }
        carry_cp = last_cp;
        carry_he = last_he;
        rb += __shfl_sync(FULL_MASK, incl, 31);
      }
      }
    }
    if (NUMERIC && A.g_f) {
      const int ncb_a = ncb_of(a, n3);
      for (int p = 0; p < ncb_a; ++p) {
        double g0 = 0, g1 = 0, g2 = 0;
        if (l < s) {
          const int ci = tab.ci[l];
          const double wc = wgt(A.X, ci, ncb_a, p);
          g0 = wc * A.g_f[3 * (int64_t)ci];
          g1 = wc * A.g_f[3 * (int64_t)ci + 1];
          g2 = wc * A.g_f[3 * (int64_t)ci + 2];
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
    if (!NUMERIC && l == 0) A.rowlen[a] = run_base;
    __syncwarp();
  }
  if (!NUMERIC) pairs_flush(s_pb[w], npb, A.pairs, A.porig, A.pair_cap, A.scw);
}

// split the small nodes into the warp list (<= 32 entries) and the tile list (> 32)
// ------------------------------------------------------------------------------------
// D. numeric
// ------------------------------------------------------------------------------------
// ------------------------------------------------------------------------------------
// D. numeric
// ------------------------------------------------------------------------------------
// Large rows: write their column ids and zero their values (blocks are then filled by the
// mirrored writes of small rows and by the atomics of the large-row chunks).
__global__ void k_large_rows_init(int64_t n_c, const AsmScal *sc, const uint8_t *__restrict__ is_small,
                                  const int32_t *__restrict__ gbuf, const long long *__restrict__ nb_off,
                                  const int32_t *__restrict__ nb_cnt, const int32_t *__restrict__ rowlen,
                                  const int64_t *__restrict__ crp, int32_t *__restrict__ ccol, double *__restrict__ cval,
                                  int32_t *__restrict__ dpos) {
  if (sc->err_cap) return;  // outputs do not fit / bad input: write nothing
  const int w = threadIdx.x >> 5, l = lane_id();
  const int wpb = blockDim.x >> 5;
  const long long n3 = sc->n3;
  for (int64_t a = (int64_t)blockIdx.x * wpb + w; a < n_c; a += (int64_t)gridDim.x * wpb) {
    if (is_small[a]) continue;
    const int U = nb_cnt[a], rl = rowlen[a];
    const int32_t *lst = gbuf + nb_off[a];
    const int first12 = lower_bound_dev<int32_t>(lst, U, (int32_t)n3);
    const int ncb_a = ncb_of((int)a, n3);
    if (l == 0) dpos[a] = -1;  // no stored diagonal block (then the chunks accumulate nothing there)
    __syncwarp();
    for (int p = 0; p < ncb_a; ++p) {
      const long long rs = crp[slot_of((int)a, p, n3)];
      for (int t = l; t < U; t += 32) {
        const int b = lst[t];
        const int cp = colpos(t, first12);
        const int ncb_b = ncb_of(b, n3);
        // blocks of a small column are written exactly once by the small row's mirror (R22);
        // only the blocks the large-row chunks accumulate into need zeroing
        const bool zero = !is_small[b];
        if (b == a && p == 0) dpos[a] = cp;
        for (int q = 0; q < ncb_b; ++q) {
          ccol[rs + cp + q] = slot_of(b, q, n3);
          if (zero) {
            double *v = cval + 9 * (rs + cp + q);
#pragma unroll
            for (int x = 0; x < 9; ++x) v[x] = 0.0;
          }
        }
      }
    }
  }
}

// Large rows, one warp per 32-children chunk (reading R22: the (large, small) blocks are mirrored
// by the small rows).  Phase 1 (lane per entry, coalesced): classify the chunk's stored blocks
// into the diagonal list (new_map(j) == a) and the large-large interface list (staged in shared
// memory as (child, offset) and the column node).  Phase 2: 64 diagonal blocks staged per warp
// (two independent 72-B loads per lane), then lane (g, p, q) -- two groups g of 16 lanes, one
// (p, q) sub-block per lane -- accumulates acc[x] += w_i[p] w_j[q] B_ij[x] (Eq 4) for every other
// staged block.  Phase 3: one pass per distinct interface column aggregate b0.  No atomics: the
// chunk writes its diagonal-block / g partials (part) and one record per (batch, b0) (rec_*)
// at positions fixed by the symbolic pass, and k_large_reduce sums them in chunk order, so H_c
// and g_c are bitwise reproducible.  <= 80 registers (6 CTAs of 4 warps per SM).
// Large rows, one warp per 32-children chunk -- the default (fast, fp64 atomics: H_c reproducible
// only up to rounding; AGIPC_OPT_DETERMINISTIC selects k_num_large + k_large_reduce).  Phase 1 (lane per entry, coalesced): classify the
// chunk's stored blocks into the diagonal list (new_map(j) == a, staged in shared memory),
// large-large interface blocks (direct fp64 atomics, rare) and small columns (skipped: mirrored
// by the small row, reading R22).  Phase 2: lane = (block group g, p) streams the diagonal list
// two blocks per group in flight and accumulates acc[q][x] += w_i[p] w_j[q] B_ij[x] (Eq 4) in
// registers; a final reduction over g and one fp64 atomic per entry per chunk.
#ifndef LIST_ISTAGE
#define LIST_ISTAGE 192  // k_num_large_list: interface entries staged per batch
#endif
#ifndef LIST_MINB
#define LIST_MINB 4  // k_num_large_list CTAs per SM (128 registers)
#endif
#ifndef LSTAGE_A
#define LSTAGE_A 192
#endif
#ifndef LARGE_MINB
#define LARGE_MINB 4
#endif

template <int NCB, int NB>
__global__ void __launch_bounds__(128, NB > 2 ? 3 : LARGE_MINB) k_num_large_atomic(LargeArgs A) {
  if (A.sc->err_cap || (NCB == 1 && A.sc->n_large3 == 0)) return;
  __shared__ ChildTab s_tab[4];
  __shared__ long long s_k[4][LSTAGE_A];
  __shared__ int s_i[4][LSTAGE_A];     // child slot c of the entry's row (weights in s_wc)
  __shared__ int s_b[4][LSTAGE_A];     // interface entries (staged from the top): column aggregate
  __shared__ double s_xj[4][LSTAGE_A][3];  // X_bar of the entry's column node (w_j)
  __shared__ double s_wc[4][32][3];      // X_bar of the chunk's children (w_i)
  __shared__ double s_B[4][32][9];       // phase 2: 32 diagonal blocks staged per warp (one per lane)
  __shared__ int s_ix[4][LSTAGE_A];      // phase 3: staged positions of the current column's entries
  const int w = threadIdx.x >> 5, l = lane_id();
  // lane = (block group, p, q half): NCB = 4 -> 8 lanes per block, 2 q per lane
  constexpr int LPB = NCB == 4 ? 8 : 1, QN = NCB == 4 ? 2 : 1, G = 32 / LPB;
  const int gq = l / LPB, p = NCB == 4 ? (l >> 1) & 3 : 0, q0 = NCB == 4 ? (l & 1) * 2 : 0;
  const long long n3 = A.sc->n3;
  ChildTab &tab = s_tab[w];
  const int64_t n_tasks = A.task_ptr[A.n_c];
  const int64_t tstride = (int64_t)gridDim.x * 4;
  // software pipeline: the next task's node, chunk size and the lane's child are loaded while
  // this task is processed (task_node -> task_ptr / child_ptr -> child_list off the critical path)
  int a_nx = 0, s_nx = 0, ci_nx = 0;
  auto prefetch = [&](int64_t tn) {
    if (tn < n_tasks) {
      a_nx = A.task_node[tn];
      const int ch = (int)(tn - A.task_ptr[a_nx]);
      s_nx = min(LARGE_CHUNK, A.size_new[a_nx] - ch * LARGE_CHUNK);
      ci_nx = l < s_nx ? A.child_list[A.child_ptr[a_nx] + (int64_t)ch * LARGE_CHUNK + l] : 0;
    }
  };
  prefetch((int64_t)blockIdx.x * 4 + w);
  for (int64_t t = (int64_t)blockIdx.x * 4 + w; t < n_tasks; t += tstride) {
    const int a = a_nx, s = s_nx, ci_c = ci_nx;
    prefetch(t + tstride);
    if (ncb_of(a, n3) != NCB) continue;
    int len = 0;
    if (l < s) {  // load_children with the prefetched child
      const long long b0 = A.rp[ci_c];
      tab.ci[l] = ci_c;
      tab.rb[l] = b0;
      len = (int)(A.rp[ci_c + 1] - b0);
    }
    const int incl_c = warp_incl_scan(len);
    tab.off[l + 1] = incl_c;
    if (l == 0) tab.off[0] = 0;
    __syncwarp();
    const int T = __shfl_sync(FULL_MASK, incl_c, 31);
    if (l < s) {
      const int64_t ci = tab.ci[l];
      s_wc[w][l][0] = __ldg(A.X + 3 * ci);
      s_wc[w][l][1] = __ldg(A.X + 3 * ci + 1);
      s_wc[w][l][2] = __ldg(A.X + 3 * ci + 2);
    }
    __syncwarp();
    const int32_t *lst = A.gbuf + A.nb_off[a];
    const int U = A.nb_cnt[a];
    const int first12 = A.f12[a];
    const int cpa = A.dpos[a];
    for (int base = 0; base < T; base += LSTAGE_A) {
      const int n = min(LSTAGE_A, T - base);
      int cnt = 0, icnt = 0;
      // two-stage software pipeline: while the entries e0 + l are classified, the column
      // aggregate / class / X_bar of e0 + 32 + l and the column of e0 + 64 + l are in flight
      int c1 = 0, j1 = 0;
      long long k1 = 0;
      int c0 = 0, j0 = 0, b0v = -1;
      long long k0 = 0;
      bool sm0 = true;
      double x0a = 0.0, x0b = 0.0, x0c = 0.0;
      if (l < n) {
        entry_of(tab, s, base + l, c0, k0);
        j0 = A.col[k0];
      }
      if (32 + l < n) {
        entry_of(tab, s, base + 32 + l, c1, k1);
        j1 = A.col[k1];
      }
      if (l < n) {
        b0v = A.nm[j0];
        sm0 = A.fcls[j0];
        x0a = __ldg(A.X + 3 * (int64_t)j0);
        x0b = __ldg(A.X + 3 * (int64_t)j0 + 1);
        x0c = __ldg(A.X + 3 * (int64_t)j0 + 2);
      }
      for (int e0 = 0; e0 < n; e0 += 32) {
        const bool valid = e0 + l < n;
        const long long k = k0;
        const int c = c0, b = valid ? b0v : -1;
        const bool small_col = valid ? sm0 : true;
        const double xj0 = x0a, xj1 = x0b, xj2 = x0c;
        if (e0 + 32 + l < n) {  // stage 1 -> stage 0
          b0v = A.nm[j1];
          sm0 = A.fcls[j1];
          x0a = __ldg(A.X + 3 * (int64_t)j1);
          x0b = __ldg(A.X + 3 * (int64_t)j1 + 1);
          x0c = __ldg(A.X + 3 * (int64_t)j1 + 2);
        }
        c0 = c1;
        k0 = k1;
        if (e0 + 64 + l < n) {  // new stage 1
          entry_of(tab, s, base + e0 + 64 + l, c1, k1);
          j1 = A.col[k1];
        }
        const bool diag = valid && b == a;
        const unsigned m = __ballot_sync(FULL_MASK, diag);
        if (diag) {
          const int pos = cnt + __popc(m & ((1u << l) - 1u));
          s_k[w][pos] = k;
          s_i[w][pos] = c;
          s_xj[w][pos][0] = xj0; s_xj[w][pos][1] = xj1; s_xj[w][pos][2] = xj2;
        }
        cnt += __popc(m);
        // large-large interface block: staged from the top, reduced per column aggregate below
        const bool itf = valid && b != a && !small_col;
        const unsigned mi = __ballot_sync(FULL_MASK, itf);
        if (itf) {
          const int pos = LSTAGE_A - 1 - (icnt + __popc(mi & ((1u << l) - 1u)));
          s_k[w][pos] = k;
          s_i[w][pos] = c;
          s_b[w][pos] = b;
          s_xj[w][pos][0] = xj0; s_xj[w][pos][1] = xj1; s_xj[w][pos][2] = xj2;
        }
        icnt += __popc(mi);
      }
      double acc[QN][9];
#pragma unroll
      for (int q = 0; q < QN; ++q)
#pragma unroll
        for (int x = 0; x < 9; ++x) acc[q][x] = 0.0;
      __syncwarp();
      // phase 2: every lane stages one diagonal block (32 independent 72-B loads in flight per
      // warp), then lane (group, p, q half) accumulates the staged blocks d = gq, gq + G, ...
      for (int d0 = 0; d0 < cnt; d0 += 32) {
        if (d0 + l < cnt) {
          const long long kk = s_k[w][d0 + l];
#pragma unroll
          for (int x = 0; x < 9; ++x) s_B[w][l][x] = __ldg(A.val + 9 * kk + x);
        }
        __syncwarp();
        const int dn = min(32, cnt - d0);
        for (int dd = gq; dd < dn; dd += G) {
          const int d = d0 + dd;
          const double wi = (NCB == 1 || p == 3) ? 1.0 : s_wc[w][s_i[w][d]][p];
#pragma unroll
          for (int qq = 0; qq < QN; ++qq) {
            const int q = q0 + qq;
            const double c = wi * ((NCB == 1 || q == 3) ? 1.0 : s_xj[w][d][q]);
#pragma unroll
            for (int x = 0; x < 9; ++x) acc[qq][x] += c * s_B[w][dd][x];
          }
        }
        __syncwarp();
      }
      __syncwarp();
      if (cnt > 0) {  // reduce over the block groups (lanes with the same p, q half), flush the batch's part
#pragma unroll
        for (int o = LPB; o < 32; o <<= 1)
#pragma unroll
          for (int qq = 0; qq < QN; ++qq)
#pragma unroll
            for (int x = 0; x < 9; ++x) acc[qq][x] += __shfl_xor_sync(FULL_MASK, acc[qq][x], o);
        if (gq == 0 && cpa >= 0) {
          const long long rs = A.crp[slot_of(a, p, n3)];
#pragma unroll
          for (int qq = 0; qq < QN; ++qq)
#pragma unroll
            for (int x = 0; x < 9; ++x) atomicAdd(A.cval + 9 * (rs + cpa + q0 + qq) + x, acc[qq][x]);
        }
      }
      // interface entries [LSTAGE_A - icnt, LSTAGE_A): one pass per distinct column aggregate b0,
      // lanes (block group, p, q half) accumulate its entries, one set of atomics per (a, b0)
      const int i0 = LSTAGE_A - icnt;
      int left = icnt;
      while (left > 0) {
        int f = -1;
        for (int d0 = 0; d0 < icnt && f < 0; d0 += 32) {
          const unsigned mb = __ballot_sync(FULL_MASK, d0 + l < icnt && s_b[w][i0 + d0 + l] >= 0);
          if (mb) f = d0 + __ffs(mb) - 1;
        }
        const int b0 = s_b[w][i0 + f];
        const int ncb_b = ncb_of(b0, n3);
        constexpr int QI = NCB == 4 ? 2 : 4;  // q values per lane (a 3-DoF row meets 12-DoF columns)
        double ac[QI][9];
#pragma unroll
        for (int qq = 0; qq < QI; ++qq)
#pragma unroll
          for (int x = 0; x < 9; ++x) ac[qq][x] = 0.0;
        // the entries of b0, compacted in order; their blocks are staged 32 at a time (one
        // independent 72-B load per lane) before the groups accumulate them
        int nb = 0;
        for (int d0 = f; d0 < icnt; d0 += 32) {
          const bool mine = d0 + l < icnt && s_b[w][i0 + d0 + l] == b0;
          const unsigned mm = __ballot_sync(FULL_MASK, mine);
          if (mine) s_ix[w][nb + __popc(mm & ((1u << l) - 1u))] = i0 + d0 + l;
          nb += __popc(mm);
        }
        __syncwarp();
        for (int s0 = 0; s0 < nb; s0 += 32) {
          if (s0 + l < nb) {
            const long long kk = s_k[w][s_ix[w][s0 + l]];
#pragma unroll
            for (int x = 0; x < 9; ++x) s_B[w][l][x] = __ldg(A.val + 9 * kk + x);
          }
          __syncwarp();
          const int dn = min(32, nb - s0);
          for (int dd = gq; dd < dn; dd += G) {
            const int d = s_ix[w][s0 + dd];
            const double wi = (NCB == 1 || p == 3) ? 1.0 : s_wc[w][s_i[w][d]][p];
#pragma unroll
            for (int qq = 0; qq < QI; ++qq) {
              const int q = q0 + qq;
              const double c = q < ncb_b ? wi * ((ncb_b == 1 || q == 3) ? 1.0 : s_xj[w][d][q]) : 0.0;
#pragma unroll
              for (int x = 0; x < 9; ++x) ac[qq][x] += c * s_B[w][dd][x];
            }
          }
          __syncwarp();
        }
        __syncwarp();
        int done_n = 0;
        for (int d0 = f; d0 < icnt; d0 += 32) {
          const bool mine = d0 + l < icnt && s_b[w][i0 + d0 + l] == b0;
          done_n += __popc(__ballot_sync(FULL_MASK, mine));
          if (mine) s_b[w][i0 + d0 + l] = -1;
        }
        __syncwarp();
        left -= done_n;
#pragma unroll
        for (int o = LPB; o < 32; o <<= 1)
#pragma unroll
          for (int qq = 0; qq < QI; ++qq)
#pragma unroll
            for (int x = 0; x < 9; ++x) ac[qq][x] += __shfl_xor_sync(FULL_MASK, ac[qq][x], o);
        const int cp = colpos(lower_bound_dev<int32_t>(lst, U, b0), first12);
        if (gq == 0) {
          const long long rs = A.crp[slot_of(a, p, n3)];
#pragma unroll
          for (int qq = 0; qq < QI; ++qq)
            if (q0 + qq < ncb_b) {
              double *dst = A.cval + 9 * (rs + cp + q0 + qq);
#pragma unroll
              for (int x = 0; x < 9; ++x) atomicAdd(dst + x, ac[qq][x]);
            }
        }
      }
    }
    if (A.g_f) {  // g_c[slot(a,pp)] += sum over the chunk of w_i[pp] g_f[i]
      for (int pp = 0; pp < NCB; ++pp) {
        double g0 = 0, g1 = 0, g2 = 0;
        if (l < s) {
          const int i = tab.ci[l];
          const double wi = wgt(A.X, i, NCB, pp);
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

// Large rows from the entry lists of k_sym_large (default numeric path): one warp per 32-children
// chunk as k_num_large_atomic, but no classification pass -- the chunk's diagonal entries come as
// a list (fine block, child slot, column node), read 32 per round one round ahead, so a round has
// ONE dependent latency (its 72-B blocks and X_bar of the column nodes); the interface entries
// are staged from their list and reduced per column aggregate as before.
template <int NCB>
__global__ void __launch_bounds__(128, LIST_MINB) k_num_large_list(LargeArgs A) {
  if (A.sc->err_cap || (NCB == 1 && A.sc->n_large3 == 0)) return;
  __shared__ long long s_k[4][LIST_ISTAGE];
  __shared__ int s_i[4][LIST_ISTAGE];
  __shared__ int s_b[4][LIST_ISTAGE];
  __shared__ double s_xj[4][LIST_ISTAGE][3];
  __shared__ double s_wc[4][32][3];      // X_bar of the chunk's children (w_i)
  __shared__ double s_B[4][32][9];       // 32 blocks staged per warp (one per lane)
  __shared__ int s_ix[4][LIST_ISTAGE];
  const int w = threadIdx.x >> 5, l = lane_id();
  constexpr int LPB = NCB == 4 ? 8 : 1, QN = NCB == 4 ? 2 : 1, G = 32 / LPB;
  const int gq = l / LPB, p = NCB == 4 ? (l >> 1) & 3 : 0, q0 = NCB == 4 ? (l & 1) * 2 : 0;
  const long long n3 = A.sc->n3;
  const int64_t n_tasks = A.task_ptr[A.n_c];
  const int64_t tstride = (int64_t)gridDim.x * 4;
  int a_nx = 0, s_nx = 0, ci_nx = 0;
  auto prefetch = [&](int64_t tn) {
    if (tn < n_tasks) {
      a_nx = A.task_node[tn];
      const int ch = (int)(tn - A.task_ptr[a_nx]);
      s_nx = min(LARGE_CHUNK, A.size_new[a_nx] - ch * LARGE_CHUNK);
      ci_nx = l < s_nx ? A.child_list[A.child_ptr[a_nx] + (int64_t)ch * LARGE_CHUNK + l] : 0;
    }
  };
  prefetch((int64_t)blockIdx.x * 4 + w);
  for (int64_t t = (int64_t)blockIdx.x * 4 + w; t < n_tasks; t += tstride) {
    const int a = a_nx, s = s_nx, ci_c = ci_nx;
    prefetch(t + tstride);
    if (ncb_of(a, n3) != NCB) continue;
    const long long lbase = A.lbase[t], lib = A.lib[t];
    const int nd = A.lnd[t], ni = A.lni[t];
    // first round of the diagonal list in flight with the children's X_bar
    long long ek_nx = 0;
    int ej_nx = 0;
    if (l < nd) {
      ek_nx = A.lent[lbase + l];
      ej_nx = A.lj[lbase + l];
    }
    if (l < s) {
      s_wc[w][l][0] = __ldg(A.X + 3 * (int64_t)ci_c);
      s_wc[w][l][1] = __ldg(A.X + 3 * (int64_t)ci_c + 1);
      s_wc[w][l][2] = __ldg(A.X + 3 * (int64_t)ci_c + 2);
    }
    const int first12 = A.f12[a];
    const int cpa = A.dpos[a];
    double acc[QN][9];
#pragma unroll
    for (int q = 0; q < QN; ++q)
#pragma unroll
      for (int x = 0; x < 9; ++x) acc[q][x] = 0.0;
    for (int d0 = 0; d0 < nd; d0 += 32) {
      const long long ek = ek_nx;
      const int ej = ej_nx;
      if (d0 + 32 + l < nd) {  // next round's entries
        ek_nx = A.lent[lbase + d0 + 32 + l];
        ej_nx = A.lj[lbase + d0 + 32 + l];
      }
      if (d0 + l < nd) {
        const long long kk = ek >> 5;
#pragma unroll
        for (int x = 0; x < 9; ++x) s_B[w][l][x] = __ldg(A.val + 9 * kk + x);
        s_i[w][l] = (int)(ek & 31);
        s_xj[w][l][0] = __ldg(A.X + 3 * (int64_t)ej);
        s_xj[w][l][1] = __ldg(A.X + 3 * (int64_t)ej + 1);
        s_xj[w][l][2] = __ldg(A.X + 3 * (int64_t)ej + 2);
      }
      __syncwarp();
      const int dn = min(32, nd - d0);
      for (int dd = gq; dd < dn; dd += G) {
        const double wi = (NCB == 1 || p == 3) ? 1.0 : s_wc[w][s_i[w][dd]][p];
#pragma unroll
        for (int qq = 0; qq < QN; ++qq) {
          const int q = q0 + qq;
          const double c = wi * ((NCB == 1 || q == 3) ? 1.0 : s_xj[w][dd][q]);
#pragma unroll
          for (int x = 0; x < 9; ++x) acc[qq][x] += c * s_B[w][dd][x];
        }
      }
      __syncwarp();
    }
    if (nd > 0) {  // reduce over the block groups (lanes with the same p, q half) and flush
#pragma unroll
      for (int o = LPB; o < 32; o <<= 1)
#pragma unroll
        for (int qq = 0; qq < QN; ++qq)
#pragma unroll
          for (int x = 0; x < 9; ++x) acc[qq][x] += __shfl_xor_sync(FULL_MASK, acc[qq][x], o);
      if (gq == 0 && cpa >= 0) {
        const long long rs = A.crp[slot_of(a, p, n3)];
#pragma unroll
        for (int qq = 0; qq < QN; ++qq)
#pragma unroll
          for (int x = 0; x < 9; ++x) atomicAdd(A.cval + 9 * (rs + cpa + q0 + qq) + x, acc[qq][x]);
      }
    }
    // interface entries: batches of LIST_ISTAGE staged from the list, one pass per distinct column
    // aggregate b0 (its entries compacted, their blocks staged 32 at a time), one set of atomics
    // per (a, b0, batch)
    const int32_t *lst = A.gbuf + A.nb_off[a];
    const int U = A.nb_cnt[a];
    for (int ibase = 0; ibase < ni; ibase += LIST_ISTAGE) {
      const int icnt = min(LIST_ISTAGE, ni - ibase);
      for (int e = l; e < icnt; e += 32) {
        const long long o = lib + ibase + e;
        const long long ek = A.lent[o];
        const int ej = A.lj[o];
        s_k[w][e] = ek >> 5;
        s_i[w][e] = (int)(ek & 31);
        s_b[w][e] = A.lb[o];
        s_xj[w][e][0] = __ldg(A.X + 3 * (int64_t)ej);
        s_xj[w][e][1] = __ldg(A.X + 3 * (int64_t)ej + 1);
        s_xj[w][e][2] = __ldg(A.X + 3 * (int64_t)ej + 2);
      }
      __syncwarp();
      int left = icnt;
      while (left > 0) {
        int f = -1;
        for (int d0 = 0; d0 < icnt && f < 0; d0 += 32) {
          const unsigned mb = __ballot_sync(FULL_MASK, d0 + l < icnt && s_b[w][d0 + l] >= 0);
          if (mb) f = d0 + __ffs(mb) - 1;
        }
        const int b0 = s_b[w][f];
        const int ncb_b = ncb_of(b0, n3);
        constexpr int QI = NCB == 4 ? 2 : 4;  // q values per lane (a 3-DoF row meets 12-DoF columns)
        double ac[QI][9];
#pragma unroll
        for (int qq = 0; qq < QI; ++qq)
#pragma unroll
          for (int x = 0; x < 9; ++x) ac[qq][x] = 0.0;
        int nb = 0;
        for (int d0 = f; d0 < icnt; d0 += 32) {
          const bool mine = d0 + l < icnt && s_b[w][d0 + l] == b0;
          const unsigned mm = __ballot_sync(FULL_MASK, mine);
          if (mine) s_ix[w][nb + __popc(mm & ((1u << l) - 1u))] = d0 + l;
          nb += __popc(mm);
        }
        __syncwarp();
        for (int s0 = 0; s0 < nb; s0 += 32) {
          if (s0 + l < nb) {
            const long long kk = s_k[w][s_ix[w][s0 + l]];
#pragma unroll
            for (int x = 0; x < 9; ++x) s_B[w][l][x] = __ldg(A.val + 9 * kk + x);
          }
          __syncwarp();
          const int dn = min(32, nb - s0);
          for (int dd = gq; dd < dn; dd += G) {
            const int d = s_ix[w][s0 + dd];
            const double wi = (NCB == 1 || p == 3) ? 1.0 : s_wc[w][s_i[w][d]][p];
#pragma unroll
            for (int qq = 0; qq < QI; ++qq) {
              const int q = q0 + qq;
              const double c = q < ncb_b ? wi * ((ncb_b == 1 || q == 3) ? 1.0 : s_xj[w][d][q]) : 0.0;
#pragma unroll
              for (int x = 0; x < 9; ++x) ac[qq][x] += c * s_B[w][dd][x];
            }
          }
          __syncwarp();
        }
        for (int d0 = f; d0 < icnt; d0 += 32)
          if (d0 + l < icnt && s_b[w][d0 + l] == b0) s_b[w][d0 + l] = -1;
        __syncwarp();
        left -= nb;
#pragma unroll
        for (int o = LPB; o < 32; o <<= 1)
#pragma unroll
          for (int qq = 0; qq < QI; ++qq)
#pragma unroll
            for (int x = 0; x < 9; ++x) ac[qq][x] += __shfl_xor_sync(FULL_MASK, ac[qq][x], o);
        const int cp = colpos(lower_bound_dev<int32_t>(lst, U, b0), first12);
        if (gq == 0) {
          const long long rs = A.crp[slot_of(a, p, n3)];
#pragma unroll
          for (int qq = 0; qq < QI; ++qq)
            if (q0 + qq < ncb_b) {
              double *dst = A.cval + 9 * (rs + cp + q0 + qq);
#pragma unroll
              for (int x = 0; x < 9; ++x) atomicAdd(dst + x, ac[qq][x]);
            }
        }
      }
      __syncwarp();
    }
    if (A.g_f) {  // g_c[slot(a,pp)] += sum over the chunk of w_i[pp] g_f[i]
      for (int pp = 0; pp < NCB; ++pp) {
        double g0 = 0, g1 = 0, g2 = 0;
        if (l < s) {
          const double wi = (NCB == 1 || pp == 3) ? 1.0 : s_wc[w][l][pp];
          g0 = wi * A.g_f[3 * (int64_t)ci_c];
          g1 = wi * A.g_f[3 * (int64_t)ci_c + 1];
          g2 = wi * A.g_f[3 * (int64_t)ci_c + 2];
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

// Interface flush: one record per distinct column aggregate b0 of the staged interface list
// (lanes (g, p, q) accumulate the entries of b0, the two groups are reduced, group 0 writes).
template <int NCB>
__device__ __forceinline__ void itf_flush(LargeArgs &A, int w, int l, int icnt, int *s_ice, int *s_ij, int *s_ib,
                                          const ChildTab &tab, const double (*s_wc)[3], long long n3, int64_t rbase,
                                          int64_t rcap, int &nrec) {
  const int gq = l >> 4, p = (l >> 2) & 3, q = l & 3;
  const bool pin = p < NCB;
  int left = icnt;
  while (left > 0) {
    int f = -1;
    for (int d0 = 0; d0 < icnt && f < 0; d0 += 32) {
      const unsigned mb = __ballot_sync(FULL_MASK, d0 + l < icnt && s_ib[d0 + l] >= 0);
      if (mb) f = d0 + __ffs(mb) - 1;
    }
    const int b0 = s_ib[f];
    const int ncb_b = ncb_of(b0, n3);
    double ac[9];
#pragma unroll
    for (int x = 0; x < 9; ++x) ac[x] = 0.0;
    if (pin && q < ncb_b) {
      for (int d = f + gq; d < icnt; d += 2) {
        if (s_ib[d] != b0) continue;
        const int ce = s_ice[d];
        const long long kk = tab.rb[ce >> 16] + (ce & 0xffff);
        const double wi = (NCB == 1 || p == 3) ? 1.0 : s_wc[ce >> 16][p];
        const double wj = (ncb_b == 1 || q == 3) ? 1.0 : __ldg(A.X + 3 * (int64_t)s_ij[d] + q);
        const double cf = wi * wj;
#pragma unroll
        for (int x = 0; x < 9; ++x) ac[x] += cf * __ldg(A.val + 9 * kk + x);
      }
    }
    __syncwarp();
    int done_n = 0;
    for (int d0 = f; d0 < icnt; d0 += 32) {
      const bool mine = d0 + l < icnt && s_ib[d0 + l] == b0;
      done_n += __popc(__ballot_sync(FULL_MASK, mine));
      if (mine) s_ib[d0 + l] = -1;
    }
    __syncwarp();
    left -= done_n;
#pragma unroll
    for (int x = 0; x < 9; ++x) ac[x] += __shfl_xor_sync(FULL_MASK, ac[x], 16);
    if (nrec < rcap) {
      const int64_t r = rbase + nrec;
      if (gq == 0 && pin && q < ncb_b) {
        double *dst = A.rec_v + 144 * r + 9 * (p * 4 + q);
#pragma unroll
        for (int x = 0; x < 9; ++x) dst[x] = ac[x];
      }
      if (l == 0) A.rec_b[r] = b0;
    } else if (l == 0) {
      A.scw->err_overflow = 1;
    }
    ++nrec;
  }
  __syncwarp();
}

template <int NCB>
__global__ void __launch_bounds__(128, 6) k_num_large(LargeArgs A) {
  if (A.sc->err_cap) return;
  __shared__ ChildTab s_tab[4];
  __shared__ int s_ce[4][LSTAGE];     // diagonal entries: (child c << 16) | entry offset in its row
  __shared__ int s_j[4][LSTAGE];      //   column node j (w_j = X_bar_j)
  __shared__ int s_ice[4][ITF_CAP];   // interface entries (kept across batches)
  __shared__ int s_ij[4][ITF_CAP];
  __shared__ int s_ib[4][ITF_CAP];    //   column aggregate b0 (-1 once summed)
  __shared__ double s_wc[4][32][3];   // X_bar of the chunk's children (w_i)
  __shared__ double s_B[4][64][9];    // phase 2: 64 diagonal blocks staged per warp
  const int w = threadIdx.x >> 5, l = lane_id();
  const int gq = l >> 4, p = (l >> 2) & 3, q = l & 3;
  const bool pin = p < NCB;  // lanes with p >= NCB idle (NCB = 1: 3-DoF large rows, rare)
  const long long n3 = A.sc->n3;
  ChildTab &tab = s_tab[w];
  const int64_t n_tasks = A.task_ptr[A.n_c];
  for (int64_t t = (int64_t)blockIdx.x * 4 + w; t < n_tasks; t += (int64_t)gridDim.x * 4) {
    const int a = A.task_node[t];
    if (ncb_of(a, n3) != NCB) continue;
    const int chunk = (int)(t - A.task_ptr[a]);
    const int s = min(LARGE_CHUNK, A.size_new[a] - chunk * LARGE_CHUNK);
    const int T = load_children(tab, A.child_list, A.child_ptr[a] + (int64_t)chunk * LARGE_CHUNK, s, A.rp);
    if (l < s) {
      const int64_t ci = tab.ci[l];
      s_wc[w][l][0] = __ldg(A.X + 3 * ci);
      s_wc[w][l][1] = __ldg(A.X + 3 * ci + 1);
      s_wc[w][l][2] = __ldg(A.X + 3 * ci + 2);
    }
    __syncwarp();
    const int64_t rbase = A.rec_off[t], rcap = A.rec_off[t + 1] - rbase;
    int nrec = 0, icnt = 0;
    double acc[9];
#pragma unroll
    for (int x = 0; x < 9; ++x) acc[x] = 0.0;
    int c_nx = 0, j_nx = 0;
    long long k_nx = 0;
    if (l < T) {
      entry_of(tab, s, l, c_nx, k_nx);
      j_nx = A.col[k_nx];
    }
    for (int base = 0; base < T; base += LSTAGE) {
      const int n = min(LSTAGE, T - base);
      int cnt = 0;
      for (int e0 = 0; e0 < n; e0 += 32) {
        const bool valid = e0 + l < n;
        const long long k = k_nx;
        const int c = c_nx, j = j_nx;
        int b = -1;
        bool small_col = true;
        if (valid) {
          b = A.nm[j];
          small_col = A.fcls[j];
        }
        if (base + e0 + 32 + l < T) {  // the next 32 entries' columns in flight
          entry_of(tab, s, base + e0 + 32 + l, c_nx, k_nx);
          j_nx = A.col[k_nx];
        }
        const int ce = (c << 16) | (int)(k - tab.rb[c]);
        const bool diag = valid && b == a;
        const unsigned m = __ballot_sync(FULL_MASK, diag);
        if (diag) {
          const int pos = cnt + __popc(m & ((1u << l) - 1u));
          s_ce[w][pos] = ce;
          s_j[w][pos] = j;
        }
        cnt += __popc(m);
        const bool itf = valid && b != a && !small_col;
        const unsigned mi = __ballot_sync(FULL_MASK, itf);
        if (mi && icnt + __popc(mi) > ITF_CAP) {  // list full: emit its records first
          itf_flush<NCB>(A, w, l, icnt, s_ice[w], s_ij[w], s_ib[w], tab, s_wc[w], n3, rbase, rcap, nrec);
          icnt = 0;
        }
        if (itf) {
          const int pos = icnt + __popc(mi & ((1u << l) - 1u));
          s_ice[w][pos] = ce;
          s_ij[w][pos] = j;
          s_ib[w][pos] = b;
        }
        icnt += __popc(mi);
      }
      __syncwarp();
      // phase 2: the diagonal list, 64 blocks in flight per warp
      for (int d0 = 0; d0 < cnt; d0 += 64) {
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int d = d0 + h2 * 32 + l;
          if (d < cnt) {
            const int ce = s_ce[w][d];
            const long long kk = tab.rb[ce >> 16] + (ce & 0xffff);
#pragma unroll
            for (int x = 0; x < 9; ++x) s_B[w][h2 * 32 + l][x] = __ldg(A.val + 9 * kk + x);
          }
        }
        __syncwarp();
        const int dn = min(64, cnt - d0);
        if (pin) {
          for (int dd = gq; dd < dn; dd += 2) {
            const int d = d0 + dd;
            const int c = s_ce[w][d] >> 16;
            const double wi = (NCB == 1 || p == 3) ? 1.0 : s_wc[w][c][p];
            const double wj = (NCB == 1 || q == 3) ? 1.0 : __ldg(A.X + 3 * (int64_t)s_j[w][d] + q);
            const double cf = (NCB == 1 && q > 0) ? 0.0 : wi * wj;
#pragma unroll
            for (int x = 0; x < 9; ++x) acc[x] += cf * s_B[w][dd][x];
          }
        }
        __syncwarp();
      }
    }
    if (icnt > 0) itf_flush<NCB>(A, w, l, icnt, s_ice[w], s_ij[w], s_ib[w], tab, s_wc[w], n3, rbase, rcap, nrec);
    for (int r = nrec + l; r < rcap; r += 32) A.rec_b[rbase + r] = -1;  // unused record slots
    // the chunk's diagonal-block partial: reduce over the two groups, one (p, q) per lane
#pragma unroll
    for (int x = 0; x < 9; ++x) acc[x] += __shfl_xor_sync(FULL_MASK, acc[x], 16);
    double *pt = A.part + PART_STRIDE * t;
    if (gq == 0 && pin && (NCB == 4 || q == 0)) {
#pragma unroll
      for (int x = 0; x < 9; ++x) pt[9 * (p * 4 + q) + x] = acc[x];
    }
    if (A.g_f) {  // the chunk's g partial: sum over its children of w_i[pp] g_f[i]
      for (int pp = 0; pp < NCB; ++pp) {
        double g0 = 0, g1 = 0, g2 = 0;
        if (l < s) {
          const int i = tab.ci[l];
          const double wi = (NCB == 1 || pp == 3) ? 1.0 : s_wc[w][l][pp];
          g0 = wi * A.g_f[3 * (int64_t)i];
          g1 = wi * A.g_f[3 * (int64_t)i + 1];
          g2 = wi * A.g_f[3 * (int64_t)i + 2];
        }
        g0 = warp_sum(g0);
        g1 = warp_sum(g1);
        g2 = warp_sum(g2);
        if (l == 0) {
          pt[144 + 3 * pp] = g0;
          pt[144 + 3 * pp + 1] = g1;
          pt[144 + 3 * pp + 2] = g2;
        }
      }
    }
    __syncwarp();
  }
}

// CTA per large coarse node a: sums its chunks' partials in chunk order (fixed order: H_c, g_c
// bitwise reproducible).  The diagonal block (a, a) and g_c are written; the interface records
// are grouped by column aggregate b0 (first occurrence order) and each (a, b0) block is the sum
// of its records in record order -- every coarse value is written once, no read-modify-write.
#define RED_REC 256  // records of one node handled in shared memory (more: a second pass)
__global__ void __launch_bounds__(128) k_large_reduce(LargeArgs A, const int32_t *__restrict__ f12) {
  if (A.sc->err_cap) return;
  __shared__ int s_rb[RED_REC];
  __shared__ int s_first[RED_REC];  // record index of the first record of each distinct b0
  __shared__ int s_cp[RED_REC];     // column position of that b0 in row a
  __shared__ int s_nd;
  const long long n3 = A.sc->n3;
  for (int64_t a = blockIdx.x; a < A.n_c; a += gridDim.x) {
    if (A.is_small[a]) continue;
    const int ncb = ncb_of((int)a, n3);
    const int32_t *lst = A.gbuf + A.nb_off[a];
    const int U = A.nb_cnt[a], F = f12[a];
    const int64_t t0 = A.task_ptr[a], t1 = A.task_ptr[a + 1];
    const int cpa = colpos(lower_bound_dev<int32_t>(lst, U, (int32_t)a), F);
    for (int o = threadIdx.x; o < 9 * ncb * ncb; o += blockDim.x) {
      const int pp = o / (9 * ncb), qq = (o / 9) % ncb, x = o % 9;
      double v = 0.0;
      for (int64_t t = t0; t < t1; ++t) v += A.part[PART_STRIDE * t + 9 * (pp * 4 + qq) + x];
      A.cval[9 * (A.crp[slot_of((int)a, pp, n3)] + cpa + qq) + x] = v;
    }
    if (A.g_f && (int)threadIdx.x < 3 * ncb) {
      double v = 0.0;
      for (int64_t t = t0; t < t1; ++t) v += A.part[PART_STRIDE * t + 144 + threadIdx.x];
      A.g_c[3 * (int64_t)slot_of((int)a, threadIdx.x / 3, n3) + threadIdx.x % 3] = v;
    }
    const int64_t r0 = A.rec_off[t0], r1 = A.rec_off[t1];
    for (int64_t rb = r0; rb < r1; rb += RED_REC) {  // records in windows of RED_REC (one window typically)
      const int R = (int)min((int64_t)RED_REC, r1 - rb);
      __syncthreads();
      for (int r = threadIdx.x; r < R; r += blockDim.x) s_rb[r] = A.rec_b[rb + r];
      if (threadIdx.x == 0) s_nd = 0;
      __syncthreads();
      for (int r = threadIdx.x; r < R; r += blockDim.x) {
        const int b0 = s_rb[r];
        bool first = b0 >= 0;
        for (int u = 0; u < r && first; ++u) first = s_rb[u] != b0;
        // a b0 already seen in an earlier window is folded in there (windows past the first are
        // rare; the later window's records of that b0 then add onto the stored value below)
        if (first) {
          const int k = atomicAdd(&s_nd, 1);
          s_first[k] = r;
          s_cp[k] = colpos(lower_bound_dev<int32_t>(lst, U, (int32_t)b0), F);
        }
      }
      __syncthreads();
      const int nd = s_nd;
      for (int k = 0; k < nd; ++k) {
        const int f = s_first[k], b0 = s_rb[f];
        const int ncb_b = ncb_of(b0, n3);
        for (int o = threadIdx.x; o < 9 * ncb * ncb_b; o += blockDim.x) {
          const int pp = o / (9 * ncb_b), qq = (o / 9) % ncb_b, x = o % 9;
          double v = rb > r0 ? A.cval[9 * (A.crp[slot_of((int)a, pp, n3)] + s_cp[k] + qq) + x] : 0.0;
          for (int r = f; r < R; ++r)
            if (s_rb[r] == b0) v += A.rec_v[144 * (rb + r) + 9 * (pp * 4 + qq) + x];
          A.cval[9 * (A.crp[slot_of((int)a, pp, n3)] + s_cp[k] + qq) + x] = v;
        }
      }
    }
  }
}

__global__ void k_small_list(int64_t n_c, const uint8_t *__restrict__ is_small, const int64_t *__restrict__ sidx,
                             const unsigned long long *__restrict__ rowsum, int32_t *__restrict__ small_list,
                             int64_t *__restrict__ ecount) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n_c && is_small[c]) {
    small_list[sidx[c]] = (int32_t)c;
    ecount[sidx[c]] = (int64_t)rowsum[c];
  }
}

__global__ void k_is_small_i32(int64_t n_c, const uint8_t *__restrict__ is_small, int32_t *__restrict__ out) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n_c) out[c] = is_small[c];
}

// ------------------------------------------------------------------------------------
// host orchestration
// ------------------------------------------------------------------------------------
extern "C" agipc_status agipc_assemble_coarse(agipc_handle h, const agipc_mesh *mesh, const int32_t *map,
                                              int64_t n_coarse, int64_t affine_threshold, const agipc_bsr *H,
                                              const double *g_fine, agipc_coarse *out) {
  if (!h) return AGIPC_EINVAL;
  if (h->trace) trace_mark(h, "@assemble_enter");
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
  if (out->cap_slots < 0 || out->cap_nnzb < 0 || (out->cap_slots > 0 && !out->row_ptr) ||
      (out->cap_nnzb > 0 && (!out->col || !out->val)))
    return set_err(h, AGIPC_EINVAL, "assemble_coarse: null output arrays");
  CU_TRY(h, cudaSetDevice(h->device));
  ProfScope prof_scope(h, PROF_ASSEMBLE, h->stream);
  cudaStream_t st_ = h->stream;
  const int64_t nnzb_f = H->nnzb;
  agipc_status st;

  if (h->opt_check_sym) {  // DESIGN.md R22: the mixed-pair mirroring below relies on it
    WS(h, bad, unsigned long long, "asm_symcheck", 1);
    CU_TRY(h, cudaMemsetAsync(bad, 0, sizeof(unsigned long long), st_));
    LAUNCH(h, k_check_sym, (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(N, 8), 16 * h->sm_count)), 256, 0, N,
           H->row_ptr, H->col, H->val, bad);
    unsigned long long *hb = (unsigned long long *)pinned_get(h, sizeof(unsigned long long), &st);
    if (st != AGIPC_OK) return st;
    CU_TRY(h, cudaMemcpyAsync(hb, bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st_));
    CU_TRY(h, cudaStreamSynchronize(st_));
    if (*hb) return set_err(h, AGIPC_EINVAL, "assemble_coarse: H_fine is not bitwise symmetric (%llu blocks without "
                            "a stored B_ji == B_ij^T, DESIGN.md R22)", *hb);
  }
  WS(h, sc, AsmScal, "asm_scal", 1);
  std::unique_ptr<ProfScope> ps_classify(new ProfScope(h, PROF_ASM_CLASSIFY, st_));
  CU_TRY(h, cudaMemsetAsync(sc, 0, sizeof(AsmScal), st_));
  // ---- A. classification ----
  WS(h, size, int32_t, "asm_size", n_c);
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
  WS(h, small_i32, int32_t, "asm_small_i32", n_c);
  WS(h, sidx, int64_t, "asm_sidx", n_c + 1);
  WS(h, small_list, int32_t, "asm_small_list", n_c);
  WS(h, ecount, int64_t, "asm_ecount", n_c);
  WS(h, e_off, int64_t, "asm_e_off", n_c + 1);
  CU_TRY(h, cudaMemsetAsync(size, 0, sizeof(int32_t) * n_c, st_));
  CU_TRY(h, cudaMemsetAsync(rowsum, 0, sizeof(unsigned long long) * n_c, st_));
  const unsigned gN = (unsigned)cdiv(N, 256), gC = (unsigned)cdiv(n_c, 256);
  LAUNCH(h, k_size_hist, gN, 256, 0, N, map, n_c, size, sc);
  // ex12 = exclusive count of 12-DoF nodes: the scan evaluates size > threshold itself
  if ((st = scan_exclusive_i64(h, SCAN_SRC_GT, size, n_c, ex12, 1, affine_threshold)) != AGIPC_OK) return st;
  LAUNCH(h, k_newid, gC, 256, 0, n_c, ex12, affine_threshold, size, newid, size_new, sc);
  LAUNCH(h, k_new_map, gN, 256, 0, N, n_c, map, newid, out->new_map);
  if ((st = scan_exclusive_i64(h, SCAN_SRC_I32, size_new, n_c, child_ptr)) != AGIPC_OK) return st;
  CU_TRY(h, cudaMemcpyAsync(cursor, child_ptr, sizeof(int64_t) * n_c, cudaMemcpyDeviceToDevice, st_));
  LAUNCH(h, k_children, gN, 256, 0, N, out->new_map, H->row_ptr, cursor, child_list, rowsum);
  if (h->opt_deterministic) {  // fixed child order => fixed summation order downstream
    WS(h, sbig, int32_t, "asm_sortc_big", n_c + 1);
    LAUNCH(h, k_sort_children, (unsigned)std::min<int64_t>(cdiv(n_c, 4), 64 * h->sm_count), 128, 0, n_c,
           (const int64_t *)child_ptr, child_list, sbig, sc);
    WS(h, sscr, int32_t, "asm_sortc_scratch", 2 * N + 64);
    LAUNCH(h, k_sort_children_big, (unsigned)h->sm_count, 1024, 0, (const AsmScal *)sc, (const int32_t *)sbig,
           (const int64_t *)child_ptr, child_list, sscr);
    CU_TRY(h, cudaMemsetAsync(&sc->big_groups, 0, sizeof(long long), st_));  // reused by the symbolic phase
  }
  // small nodes: the warp list (<= 32 candidate entries) and the tile list (> 32, with the
  // prefix of their entries)
  WS(h, f16, int32_t, "asm_f16", n_c);
  WS(h, f32, int32_t, "asm_f32", n_c);
  WS(h, i16, int64_t, "asm_i16", n_c + 1);
  WS(h, i32, int64_t, "asm_i32", n_c + 1);
  WS(h, w16, int32_t, "asm_w16", n_c);
  WS(h, w32, int32_t, "asm_w32", n_c);
  LAUNCH(h, k_classify, gC, 256, 0, n_c, size_new, rowsum, is_small, ntasks, sc, f16, f32, small_i32, ecount);
  {  // chunk offsets and the three small-node list positions: one launch
    ScanJobs jobs;
    memset(&jobs, 0, sizeof(jobs));
    jobs.njobs = 4;
    jobs.j[0] = scan_job(SCAN_SRC_I32, ntasks, n_c, task_ptr);
    jobs.j[1] = scan_job(SCAN_SRC_I32, f16, n_c, i16);
    jobs.j[2] = scan_job(SCAN_SRC_I32, f32, n_c, i32);
    jobs.j[3] = scan_job(SCAN_SRC_I32, small_i32, n_c, sidx);
    if ((st = scan_multi(h, jobs)) != AGIPC_OK) return st;
  }
  WS(h, task_node, int32_t, "asm_task_node", N / LARGE_CHUNK + n_c + 1);
  WS(h, fcls, uint8_t, "asm_fcls", N);
  LAUNCH(h, k_class_lists, gN, 256, 0, N, n_c, (const int64_t *)task_ptr, task_node, (const int32_t *)out->new_map,
         (const uint8_t *)is_small, fcls, f16, f32, small_i32, i16, i32, sidx, rowsum, w16, w32, small_list, ecount);
  AsmScal *hsc = (AsmScal *)pinned_get(h, sizeof(AsmScal) + 64, &st);
  if (st != AGIPC_OK) return st;
  // the list sizes stay on the device (i16[n_c], i32[n_c], sidx[n_c]): the symbolic and numeric
  // kernels read them (warp_args_resolve); buffers and grids use the bound n_c.  ecount is zero
  // past the mid list, so its scan over n_c entries is exact on the first n_small + 1.
  if ((st = scan_exclusive_i64(h, SCAN_SRC_I64, ecount, n_c, e_off)) != AGIPC_OK) return st;

  ps_classify.reset();
  std::unique_ptr<ProfScope> ps_sym(new ProfScope(h, PROF_ASM_SYMBOLIC, st_));
  // ---- B. symbolic ----
  const long long pair_cap = nnzb_f + n_c + 32;
  WS(h, nb_off, long long, "asm_nb_off", n_c);
  WS(h, nb_cnt, int32_t, "asm_nb_cnt", n_c);
  WS(h, rowlen, int32_t, "asm_rowlen", n_c);
  WS(h, pairs, int2, "asm_pairs", pair_cap);
  WS(h, porig, long long, "asm_pair_orig", pair_cap);
  WS(h, f12, int32_t, "asm_first12", n_c);
  WS(h, gcnt, int32_t, "asm_gcnt", 2 * n_c);  // [count | scatter cursor]
  WS(h, gptr, int64_t, "asm_gptr", n_c + 1);
  WS(h, gbuf, int32_t, "asm_gbuf", 2 * pair_cap);
  WS(h, big_list, int32_t, "asm_big_list", n_c);
  const int64_t task_bound = N / LARGE_CHUNK + n_c;
  WS(h, recmax, int32_t, "asm_recmax", task_bound + 1);
  WS(h, rec_off, int64_t, "asm_rec_off", task_bound + 1);
  CU_TRY(h, cudaMemsetAsync(recmax, 0, sizeof(int32_t) * (task_bound + 1), st_));
  const double *gfp = (g_fine && out->g_c) ? g_fine : nullptr;
  WarpArgs WA;
  WA.n_w = 0; WA.wlist = w16; WA.child_list = child_list; WA.child_ptr = child_ptr; WA.size_new = size_new;
  WA.is_small = is_small; WA.rp = H->row_ptr; WA.col = H->col; WA.val = H->val; WA.nm = out->new_map;
  WA.X = mesh->x_rest; WA.g_f = gfp; WA.sc = sc; WA.rowlen = rowlen; WA.pairs = pairs; WA.pair_cap = pair_cap;
  WA.porig = porig; WA.mirpos = nullptr; WA.mirrl = nullptr; WA.mir_base = 0;
  WA.scw = sc; WA.gbuf = gbuf; WA.nb_off = nb_off; WA.nb_cnt = nb_cnt; WA.crp = nullptr; WA.ccol = nullptr;
  WA.cval = nullptr; WA.g_c = out->g_c;
  WA.mkeys = nullptr; WA.e_off = nullptr; WA.msrc = nullptr;
  WA.cnt16 = i16 + n_c; WA.cnt32 = i32 + n_c; WA.cntmid = sidx + n_c; WA.kind = 0;
  WA.key32 = n_c < (1 << 26) - 1;
  WarpArgs WB = WA, WM;
  WB.wlist = w32; WB.kind = 1;
  // mirror positions: [16 n_w16 | 32 n_w32 | mid entries], indexed like the sorted keys (the
  // list sizes are on the device: buffers use 16 n_w16 + 32 n_w32 <= 32 n_c)
  WS(h, mirpos, long long, "asm_mirror_pos", 32 * n_c + nnzb_f + 1);
  WS(h, mirrl, int32_t, "asm_mirror_rl", 32 * n_c + nnzb_f + 1);
  {  // small nodes: SEG key slots per node of the 16- and 32-entry lists
    WS(h, skeys, long long, "asm_small_keys", 32 * n_c + 1);
    WS(h, ssrc, long long, "asm_small_src", 32 * n_c + 1);
    WS(h, schild, int32_t, "asm_small_child", 32 * n_c + 1);
    WA.mchild = schild;
    WB.mchild = schild;  // + 16 n_w16 (warp_args_resolve)
    WA.mkeys = skeys;
    WB.mkeys = skeys;  // + 16 n_w16 (warp_args_resolve)
    WA.msrc = ssrc;
    WB.msrc = ssrc;
    WA.mirpos = mirpos;
    WA.mirrl = mirrl;
    WB.mirpos = mirpos;
    WB.mirrl = mirrl;
  }
  // grid-stride kernels; the 32-entry list is usually short or empty (persistent grid)
#ifndef SMALL_GRID
#define SMALL_GRID 32  // CTAs per SM of the 16-entry small-row kernels
#endif
  const unsigned g16 = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n_c, 16), SMALL_GRID * h->sm_count));
  const unsigned g32 = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n_c, 8), 4 * h->sm_count));
  // the large-row symbolic pass runs on the aux stream next to the small / mid rows' (both
  // latency-bound at partial occupancy; they only share the atomic pair counter)
  if ((st = aux_fork(h)) != AGIPC_OK) return st;
  // the 32-entry list first: usually short or empty, it then does not wait for free SM slots
  // behind the large-row symbolic pass
  LAUNCH(h, (k_small_warp<32, false>), g32, 256, 0, WB);
  LAUNCH(h, (k_small_warp<16, false>), g16, 256, 0, WA);
  WM = WA;
  WM.wlist = small_list; WM.kind = 2;
  {  // mid-node entries: sum of their candidate entries <= the fine blocks
    WS(h, mkeys, long long, "asm_mid_keys", nnzb_f + 1);
    WM.mkeys = mkeys;
    WM.e_off = e_off;
  }
#ifndef MID_GRID
#define MID_GRID 12  // CTAs per SM of the mid-node kernels
#endif
  const unsigned gmid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n_c, MID_WARPS), MID_GRID * h->sm_count));
  LargeArgs LA;
  LA.n_c = n_c; LA.child_list = child_list; LA.child_ptr = child_ptr; LA.size_new = size_new; LA.is_small = is_small;
  LA.rp = H->row_ptr; LA.col = H->col; LA.val = H->val; LA.nm = out->new_map; LA.X = mesh->x_rest;
  LA.g_f = gfp; LA.task_ptr = task_ptr; LA.task_node = task_node; LA.fcls = fcls; LA.sc = sc; LA.pairs = pairs; LA.porig = porig; LA.pair_cap = pair_cap; LA.scw = sc;
  LA.gbuf = gbuf; LA.nb_off = nb_off; LA.nb_cnt = nb_cnt; LA.crp = nullptr; LA.cval = nullptr; LA.g_c = out->g_c;
  LA.recmax = recmax; LA.rec_off = rec_off; LA.rec_b = nullptr; LA.rec_v = nullptr; LA.part = nullptr;
  const unsigned glarge = (unsigned)std::min<int64_t>(std::max<int64_t>(1, cdiv(task_bound, 4)), 64 * h->sm_count);
  // large-row entry lists for the numeric pass (default, non-deterministic mode; AGIPC_LARGE_LIST=0
  // selects the classifying k_num_large_atomic for experiments)
  static const bool large_list = !(getenv("AGIPC_LARGE_LIST") && atoi(getenv("AGIPC_LARGE_LIST")) == 0);
  LA.lent = nullptr; LA.lj = nullptr; LA.lb = nullptr; LA.lbase = nullptr; LA.lib = nullptr;
  LA.lnd = nullptr; LA.lni = nullptr;
  if (large_list && !h->opt_deterministic) {
    WS(h, lent, long long, "asm_lent", nnzb_f + 1);
    WS(h, lj, int32_t, "asm_lj", nnzb_f + 1);
    WS(h, lb, int32_t, "asm_lb", nnzb_f + 1);
    WS(h, lbase, long long, "asm_lbase", task_bound + 1);
    WS(h, lib, long long, "asm_lib", task_bound + 1);
    WS(h, lnd, int32_t, "asm_lnd", task_bound + 1);
    WS(h, lni, int32_t, "asm_lni", task_bound + 1);
    LA.lent = lent; LA.lj = lj; LA.lb = lb; LA.lbase = lbase; LA.lib = lib; LA.lnd = lnd; LA.lni = lni;
  }
#ifndef SYML_GRID
#define SYML_GRID 64  // CTAs per SM of the large-row symbolic pass
#endif
  LAUNCH_S(h, h->aux, k_sym_large, (unsigned)std::min<int64_t>(std::max<int64_t>(1, cdiv(task_bound, 4)), SYML_GRID * h->sm_count),
           128, 0, LA);
  // the mid nodes follow the large rows on the aux stream: the small rows alone are the longer stream
  LAUNCH_S(h, h->aux, k_mid_warp<false>, gmid, MID_WARPS * 32, 0, WM);
  if ((st = aux_join(h)) != AGIPC_OK) return st;
  CU_TRY(h, cudaMemsetAsync(gcnt, 0, sizeof(int32_t) * 2 * n_c, st_));
  LAUNCH(h, k_pair_count, (unsigned)(8 * h->sm_count), 256, 0, sc, pair_cap, pairs, gcnt);
  // bucket offsets: power-of-two padded counts (k_group_unique sorts in place), evaluated by the scan
  if ((st = scan_exclusive_i64(h, SCAN_SRC_POW2, gcnt, n_c, gptr)) != AGIPC_OK) return st;
  LAUNCH(h, k_pair_scatter, (unsigned)(8 * h->sm_count), 256, 0, sc, pair_cap, pairs, (const int64_t *)gptr,
         gcnt + n_c, gbuf);
  const unsigned gsym = (unsigned)std::min<int64_t>(cdiv(n_c, SYM_WARPS), 64 * h->sm_count);
  LAUNCH(h, k_group_unique, gsym, SYM_WARPS * 32, 0, n_c, is_small, gptr, gbuf, gcnt, nb_off, nb_cnt, rowlen,
         big_list, sc, f12);
  LAUNCH(h, k_group_unique_big, (unsigned)h->sm_count, 1024, 0, sc, big_list, gptr, gbuf, gcnt, nb_off, nb_cnt, rowlen,
         f12);


  // ---- C. slot row pointer (upper bound 4 n_c slots; entries past n_slots are 0) ----
  const int64_t slot_bound = 4 * n_c;
  WS(h, crp_ws, int64_t, "asm_crp", slot_bound + 1);
  {  // slot row pointer (the scan reads each slot's node row length) and the chunk record offsets
    ScanJobs jobs;
    memset(&jobs, 0, sizeof(jobs));
    jobs.njobs = 2;
    jobs.j[0] = scan_job(SCAN_SRC_SLOTRL, rowlen, slot_bound, crp_ws);
    jobs.j[0].dev_n3 = &sc->n3;
    jobs.j[0].dev_nslots = &sc->n_slots;
    jobs.j[1] = scan_job(SCAN_SRC_I32, recmax, task_bound, rec_off);
    if ((st = scan_multi(h, jobs)) != AGIPC_OK) return st;
  }
  // one host round trip per call, after this: the sizes and error flags come back while the
  // numeric pass is still to be enqueued (it then runs asynchronously to the caller); the capacity
  // check is also on the device (err_cap: every numeric kernel writes nothing)
  LAUNCH(h, k_sym_finish, (unsigned)(8 * h->sm_count), 256, 0, sc, (const int64_t *)crp_ws, (const int64_t *)task_ptr,
         n_c, (const int64_t *)rec_off, task_bound, out->cap_slots, out->cap_nnzb, (const int64_t *)(i32 + n_c),
         out->row_ptr, pair_cap, (const int2 *)pairs, (const long long *)porig, (const int32_t *)gbuf,
         (const long long *)nb_off, (const int32_t *)nb_cnt, (const int32_t *)f12, (const int32_t *)rowlen, mirpos,
         mirrl);
  CU_TRY(h, cudaMemcpyAsync(hsc, sc, sizeof(AsmScal), cudaMemcpyDeviceToHost, st_));
  CU_TRY(h, host_wait(h, st_));
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

  ps_sym.reset();
  if (h->values_event) {  // H_fine / g_fine values uploaded on another stream (one-shot)
    cudaEvent_t ev = h->values_event;
    h->values_event = nullptr;
    CU_TRY(h, cudaStreamWaitEvent(st_, ev, 0));
  }
  ProfScope ps_num(h, PROF_ASM_NUMERIC, st_);
  // ---- D. numeric ----
  if (gfp) CU_TRY(h, cudaMemsetAsync(out->g_c, 0, sizeof(double) * 3 * out->n_slots, st_));
  WS(h, dpos, int32_t, "asm_dpos", n_c);
  LA.f12 = f12;
  LA.dpos = dpos;
  // the 12-DoF chunks and the small / mid rows write disjoint blocks -- (large, large) by the
  // chunks, own rows and the mirrored (large, small) blocks by the small rows.  AGIPC_NUM_MODE
  // (experiments): 0 = chunks on the aux stream next to the small rows, 1 = chunks first then
  // the small rows on one stream, 2 = small rows first then the chunks
  static const int num_mode = getenv("AGIPC_NUM_MODE") ? atoi(getenv("AGIPC_NUM_MODE")) : 0;
  const bool fork = num_mode == 0;
  cudaStream_t ls = fork ? h->aux : st_;
  if (fork && (st = aux_fork(h)) != AGIPC_OK) return st;
  // the large rows' column ids / zeroed blocks only gate the 12-DoF chunks: on their stream, so the
  // small rows start at once (the small rows' mirrored values go to other words of those rows)
  LAUNCH_S(h, ls, k_large_rows_init, gsym, 128, 0, n_c, sc, is_small, gbuf, nb_off, nb_cnt, rowlen, out->row_ptr,
           out->col, out->val, dpos);
  auto launch_large = [&]() -> agipc_status {
    LA.crp = out->row_ptr; LA.cval = out->val;
    // (a factorised variant -- lane per child, C_i[q] = sum_j w_j[q] B_ij, then sum_i w_i[p] C_i[q] --
    // cuts the FMAs 4x but measured 2.03 vs 0.54 ms at C3: divergent per-lane row walks, 17% warps
    // active; profiles/r02f)
    if (!h->opt_deterministic) {  // 2 diagonal blocks per group in flight: 3 or 4 measured slower (r01h)
      if (LA.lent) {
#ifndef LIST_GRID
#define LIST_GRID 8  // CTAs per SM: persistent warps with the next-chunk prefetch (64 / 16 / 4 measured slower, profiles/r02v)
#endif
        const unsigned glist = (unsigned)std::min<int64_t>(std::max<int64_t>(1, cdiv(task_bound, 4)), LIST_GRID * h->sm_count);
        LAUNCH_S(h, ls, k_num_large_list<4>, glist, 128, 0, LA);
        if (hsc->n_large3 > 0) LAUNCH_S(h, ls, k_num_large_list<1>, glist, 128, 0, LA);
      } else {
        LAUNCH_S(h, ls, (k_num_large_atomic<4, 2>), glarge, 128, 0, LA);
        if (hsc->n_large3 > 0) LAUNCH_S(h, ls, (k_num_large_atomic<1, 2>), glarge, 128, 0, LA);
      }
    } else {  // large rows: per-chunk partials + records, then the fixed-order reduction (no atomics)
      // sizes vary between Newton steps: ask for 1.5x so that the buffers rarely grow
      WS(h, part, double, "asm_large_part", PART_STRIDE * (3 * hsc->n_tasks / 2 + 64));
      WS(h, rec_b, int32_t, "asm_rec_b", 3 * hsc->rec_total / 2 + 64);
      WS(h, rec_v, double, "asm_rec_v", 144 * (3 * hsc->rec_total / 2 + 64));
      LA.part = part;
      LA.rec_b = rec_b;
      LA.rec_v = rec_v;
      LAUNCH_S(h, ls, k_num_large<4>, glarge, 128, 0, LA);
      if (hsc->n_large3 > 0) LAUNCH_S(h, ls, k_num_large<1>, glarge, 128, 0, LA);
      LAUNCH_S(h, ls, k_large_reduce, (unsigned)std::min<int64_t>(n_c, 16 * h->sm_count), 128, 0, LA,
               (const int32_t *)f12);
    }
    return AGIPC_OK;
  };
  if (num_mode == 1 && (st = launch_large()) != AGIPC_OK) return st;
  WM.crp = out->row_ptr; WM.ccol = out->col; WM.cval = out->val;
  WA.crp = out->row_ptr; WA.ccol = out->col; WA.cval = out->val;
  WB.crp = out->row_ptr; WB.ccol = out->col; WB.cval = out->val;
  // (5 CTAs/SM at 48 registers measured slower: 1.35 vs 1.26 ms numeric at C3, profiles/r02k)
  LAUNCH(h, (k_small_warp<16, true>), g16, 256, 0, WA);
  if (hsc->n_w32 > 0) LAUNCH(h, (k_small_warp<32, true>), g32, 256, 0, WB);
  if (num_mode != 1 && (st = launch_large()) != AGIPC_OK) return st;
  LAUNCH_S(h, ls, k_mid_warp<true>, gmid, MID_WARPS * 32, 0, WM);  // after the large rows (aux stream)
  return fork ? aux_join(h) : AGIPC_OK;
}
