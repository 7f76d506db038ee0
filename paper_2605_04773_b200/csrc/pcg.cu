// Step 4 -- coarse PCG with 3x3 block-Jacobi (PAPER.md P:752 d_c = -H_c^-1 g_c; P:879 relative
// residual tolerance; "3x3 block Jacobi"; textbook preconditioned CG, reading R20).
//
// B200 design:
//  * once per solve the BSR matrix is re-laid out for streaming: rows longer than 64 blocks are
//    split into segments ("virtual rows"), virtual rows are sorted by length inside windows of
//    4096 and packed 32 per slice (SELL-32-sigma); a slice stores, for each block column j, a
//    9 x 32 component-major tile of doubles and 32 column ids, so every value load of the SpMV
//    is one fully used 256-byte line.  The conversion costs one pass over the matrix and is
//    amortised over the hundreds of iterations of a solve;
//  * per iteration two kernels, all scalars on the device:
//      K1  p_new = z + beta p_old formed on the fly for every gathered column (bit-identical to
//          the value the owner stores), q-segment = A p_new per virtual row (thread per row,
//          ~30 independent loads in flight), partial p_new.q; the last CTA reduces the partials
//          in a fixed order and computes alpha or flags EINDEFINITE / EBREAKDOWN;
//      K2  q = sum of the row's segments (fixed order), x += alpha p, r -= alpha q, z = D^-1 r,
//          partial r.z and r.r; the last CTA tests ||r|| <= tol ||b|| and computes beta;
//  * check_every iterations are one CUDA graph on an internal stream (ordered after the caller's
//    stream by events); the host polls the device done flag between graph launches.
#include <cmath>
#include <vector>

#include "agipc_internal.cuh"

#define PCG_THREADS 256
#define PCG_WARPS (PCG_THREADS / 32)
#define SEG_MAX 64          // blocks per virtual row
#define SORT_WIN 8192       // virtual rows per sorting window (sigma = 256 slices)
#define PROF_EVERY 8        // profiling: time the kernels of every 8th iteration
#define HALO_BIT (1 << 30)  // v_len flag: the virtual row is a segment of the halo matrix (8(e))
#define VLEN(x) ((x) & (HALO_BIT - 1))

struct PcgState {
  double rz, alpha, beta, bn2, rr, pq;
  int it, done, status, max_iters;
  double tol;
  unsigned int arrive;  // last-block counter
  int pad;
  long long nv, ns, sell_blocks;  // virtual rows, slices, stored SELL blocks (incl. padding)
};

struct PcgGraph {
  cudaGraphExec_t exec = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  const void *key[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int64_t n = -1, ns = -1;
  int chunk = 0;
  int grid1 = 0, grid2 = 0;
  bool prof = false;
  bool sym = false;
  int win = 0, all_red = 0, upd_u = 0, spmv_un = 0;
  const void *yext = nullptr;
  uint64_t ws_gen = 0;
  bool flat = false;
  int64_t n_flat = -1;
  bool l2on = false;  // captured with the persisting access-policy window
  std::vector<cudaEvent_t> ev;  // profiling: 3 events per iteration of the chunk
};

void pcg_graph_free(PcgGraph *g) {
  if (!g) return;
  for (auto e : g->ev) cudaEventDestroy(e);
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->ev_in) cudaEventDestroy(g->ev_in);
  if (g->ev_out) cudaEventDestroy(g->ev_out);
  if (g->stream) cudaStreamDestroy(g->stream);
  delete g;
}

// Block-wide sum of one double (fixed order: warp shuffles then warp 0), result in thread 0.
// NT = threads per CTA (s_red holds NT / 32 entries).
template <int NT = PCG_THREADS>
__device__ __forceinline__ double block_sum(double v, double *s_red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) s_red[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = l < NT / 32 ? s_red[l] : 0.0;
    r = warp_sum(r);
  }
  __syncthreads();
  return r;
}

// Returns true in the last CTA to arrive (all partials of the grid are then visible).
__device__ __forceinline__ bool last_block(PcgState *st) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev = atomicAdd(&st->arrive, 1u);
    s_last = prev == gridDim.x - 1;
    if (s_last) st->arrive = 0;
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

// fixed-order reduction of nparts partials by one CTA
// (four independent partial sums per thread keep four loads in flight; the order is fixed)
template <int NT = PCG_THREADS>
__device__ __forceinline__ double reduce_parts(const double *parts, int nparts, double *s_red) {
  double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
  int i = threadIdx.x;
  for (; i + 3 * NT < nparts; i += 4 * NT) {
    v0 += __ldcg(parts + i);
    v1 += __ldcg(parts + i + NT);
    v2 += __ldcg(parts + i + 2 * NT);
    v3 += __ldcg(parts + i + 3 * NT);
  }
  for (; i < nparts; i += NT) v0 += __ldcg(parts + i);
  return block_sum<NT>((v0 + v1) + (v2 + v3), s_red);
}

__device__ __forceinline__ void dinv_apply(const double *__restrict__ D, const double r0, const double r1,
                                           const double r2, double &z0, double &z1, double &z2) {
  z0 = D[0] * r0 + D[1] * r1 + D[2] * r2;
  z1 = D[3] * r0 + D[4] * r1 + D[5] * r2;
  z2 = D[6] * r0 + D[7] * r1 + D[8] * r2;
}

// ------------------------------------------------------------------------------------
// setup: block-Jacobi and the SELL layout
// ------------------------------------------------------------------------------------
// D^-1 of every row's 3x3 diagonal block (adjugate / determinant).
// ub != nullptr (symmetric solve): ub[r] = first position of row r with col >= r, i.e. where the
// diagonal + upper half of the row starts (NEXT#2).
__global__ void k_dinv(int64_t n, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                       const double *__restrict__ val, double *__restrict__ Dinv, PcgState *st,
                       int64_t *__restrict__ ub, int upper_only) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int64_t lo = rp[r], hi = rp[r + 1];
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (col[mid] < r) lo = mid + 1; else hi = mid;
  }
  if (ub) ub[r] = lo;
  if (upper_only && lo != rp[r]) {  // AGIPC_STORAGE_UPPER input with a block below the diagonal
    st->status = AGIPC_EINVAL;
    st->done = 1;
    return;
  }
  bool ok = lo < rp[r + 1] && col[lo] == r;
  double M[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (ok) {
    const double *B = val + 9 * lo;
    double c00 = B[4] * B[8] - B[5] * B[7], c01 = B[5] * B[6] - B[3] * B[8], c02 = B[3] * B[7] - B[4] * B[6];
    double c10 = B[2] * B[7] - B[1] * B[8], c11 = B[0] * B[8] - B[2] * B[6], c12 = B[1] * B[6] - B[0] * B[7];
    double c20 = B[1] * B[5] - B[2] * B[4], c21 = B[2] * B[3] - B[0] * B[5], c22 = B[0] * B[4] - B[1] * B[3];
    double det = B[0] * c00 + B[1] * c01 + B[2] * c02;
    if (det == 0.0 || !isfinite(det)) ok = false;
    else {
      double inv = 1.0 / det;
      M[0] = c00 * inv; M[1] = c10 * inv; M[2] = c20 * inv;
      M[3] = c01 * inv; M[4] = c11 * inv; M[5] = c21 * inv;
      M[6] = c02 * inv; M[7] = c12 * inv; M[8] = c22 * inv;
    }
  }
  if (!ok) {
    st->status = AGIPC_ESINGULAR;
    st->done = 1;
  }
#pragma unroll
  for (int i = 0; i < 9; ++i) Dinv[9 * r + i] = M[i];
}

// segments of row r: max(1, ceil(len/64)) of the matrix, then ceil(len_h/64) of the halo matrix
// (distributed solve: the rank's rows x ghost columns); hrp == nullptr: none
__device__ __forceinline__ int64_t nseg_local(int64_t len) { return len <= SEG_MAX ? 1 : (len + SEG_MAX - 1) / SEG_MAX; }

// rows are [rb[r], re[r]) of the matrix: rb = row_ptr, re = row_ptr + 1 for the full matrix;
// rb = ub (k_dinv) for the diagonal + upper half streamed by the symmetric solve (NEXT#2)
__global__ void k_seg_count(int64_t n, const int64_t *__restrict__ rb, const int64_t *__restrict__ re,
                            const int64_t *__restrict__ hrp, int32_t *__restrict__ nseg) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) {
    int64_t ns = nseg_local(re[r] - rb[r]);
    if (hrp) ns += (hrp[r + 1] - hrp[r] + SEG_MAX - 1) / SEG_MAX;
    nseg[r] = (int32_t)ns;
  }
}

// virtual row v = segment k of row r: blocks [rp[r] + 64k, ...) of length <= 64 (halo segments
// carry HALO_BIT and index hrp)
__global__ void k_seg_fill(int64_t n, const int64_t *__restrict__ rb, const int64_t *__restrict__ re,
                           const int64_t *__restrict__ hrp, const int64_t *__restrict__ vr_ptr,
                           int32_t *__restrict__ v_row, int32_t *__restrict__ v_len, PcgState *st) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r == 0) st->nv = vr_ptr[n];
  if (r < n) {
    const int64_t len = re[r] - rb[r];
    const int64_t nl = nseg_local(len);
    const int64_t v0 = vr_ptr[r], nv = vr_ptr[r + 1] - v0;
    for (int64_t k = 0; k < nv; ++k) {
      v_row[v0 + k] = (int32_t)r;
      if (k < nl) v_len[v0 + k] = (int32_t)min((int64_t)SEG_MAX, len - SEG_MAX * k);
      else v_len[v0 + k] = (int32_t)min((int64_t)SEG_MAX, hrp[r + 1] - hrp[r] - SEG_MAX * (k - nl)) | HALO_BIT;
    }
  }
}

// sort the virtual rows of each window of `win` (power of two <= SORT_WIN) by decreasing length
// (ties: ascending id)
__global__ void __launch_bounds__(1024) k_window_sort(const PcgState *st, const int32_t *__restrict__ v_len,
                                                      int32_t *__restrict__ perm, int win) {
  extern __shared__ unsigned long long s_key[];  // [win] (dynamic: up to 64 KB)
  const long long nv = st->nv;
  const long long w0 = (long long)blockIdx.x * win;
  if (w0 >= nv) return;
  for (int i = threadIdx.x; i < win; i += blockDim.x) {
    long long v = w0 + i;
    s_key[i] = v < nv ? ((unsigned long long)(SEG_MAX - VLEN(v_len[v])) << 32) | (unsigned long long)i : ~0ull;
  }
  __syncthreads();
  for (int k = 2; k <= win; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < win; i += blockDim.x) {
        int ixj = i ^ j;
        if (ixj > i) {
          unsigned long long a = s_key[i], b = s_key[ixj];
          bool up = (i & k) == 0;
          if ((a > b) == up) {
            s_key[i] = b;
            s_key[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < win; i += blockDim.x) {
    long long v = w0 + i;
    if (v < nv) perm[v] = (int32_t)(w0 + (long long)(s_key[i] & 0xffffffffull));
  }
}

// slice length (x32, for the scan) = longest virtual row among the slice's 32
__global__ void k_slice_len(int64_t ns_bound, const PcgState *st, const int32_t *__restrict__ perm,
                            const int32_t *__restrict__ v_len, int32_t *__restrict__ slen) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nv = st->nv;
  if (s < ns_bound) {
    int L = 0;
    for (int t = 0; t < 32 && 32 * s + t < nv; ++t) L = max(L, VLEN(v_len[perm[32 * s + t]]));
    slen[s] = 32 * L;
  }
}

// processing order of the slices: longest first (LPT), via a counting sort over lengths 0..64
__global__ void __launch_bounds__(1024) k_slice_order(const PcgState *st, const int32_t *__restrict__ slen,
                                                      int32_t *__restrict__ order) {
  __shared__ int s_cnt[SEG_MAX + 2];
  __shared__ int s_off[SEG_MAX + 2];
  const long long ns = st->ns;
  for (int i = threadIdx.x; i < SEG_MAX + 2; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  for (long long s = threadIdx.x; s < ns; s += blockDim.x) atomicAdd(&s_cnt[SEG_MAX - slen[s] / 32], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int i = 0; i < SEG_MAX + 2; ++i) {
      s_off[i] = run;
      run += s_cnt[i];
    }
  }
  __syncthreads();
  for (long long s = threadIdx.x; s < ns; s += blockDim.x) order[atomicAdd(&s_off[SEG_MAX - slen[s] / 32], 1)] = (int32_t)s;
}

__global__ void k_sell_scalars(int64_t ns_bound, const int64_t *__restrict__ sptr, PcgState *st) {
  st->ns = (st->nv + 31) / 32;
  st->sell_blocks = sptr[ns_bound];
}

// Position of component e of lane l's block inside a 288-double block-column tile: components
// are paired, (0,1) (2,3) (4,5) (6,7) as [pair][lane][2], component 8 as [lane] -- so the SpMV
// reads a block with four 16-B loads and one 8-B load, every warp access fully coalesced.
__host__ __device__ __forceinline__ int tile_off(int e, int l) { return e < 8 ? 64 * (e >> 1) + 2 * l + (e & 1) : 256 + l; }

// warp per slice: block-column tiles (tile_off); padding = zero blocks pointing at the row itself
#ifndef FILL_PIPE
#define FILL_PIPE 1
#endif
__global__ void k_sell_fill(const PcgState *st, const int64_t *__restrict__ rb, const int64_t *__restrict__ re,
                            const int32_t *__restrict__ col,
                            const double *__restrict__ val, const int64_t *__restrict__ hrp,
                            const int32_t *__restrict__ hcol, const double *__restrict__ hval,
                            const int64_t *__restrict__ vr_ptr,
                            const int32_t *__restrict__ perm, const int32_t *__restrict__ v_row,
                            const int32_t *__restrict__ v_len, const int64_t *__restrict__ sptr,
                            int32_t *__restrict__ scol, double *__restrict__ sval, int32_t *__restrict__ s_vrow,
                            const double *__restrict__ x0, double *__restrict__ qx) {
  // x0 != nullptr: also the virtual row's part of A x0 into qx[v] (k_init sums a row's parts:
  // the initial residual r = b - A x0 without a second pass over the matrix)
  const long long ns = st->ns, nv = st->nv;
  const int l = lane_id();
  for (long long s = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < ns;
       s += ((long long)gridDim.x * blockDim.x) >> 5) {
    const long long vi = 32 * s + l;
    const int v = vi < nv ? perm[vi] : -1;
    s_vrow[vi] = v;
    int row = 0, len = 0;
    long long k0 = 0;
    bool halo = false;
    if (v >= 0) {
      row = v_row[v];
      const int vl = v_len[v];
      len = VLEN(vl);
      halo = (vl & HALO_BIT) != 0;
      const long long k = v - vr_ptr[row];
      if (!halo) k0 = rb[row] + (long long)SEG_MAX * k;
      else k0 = hrp[row] + (long long)SEG_MAX * (k - nseg_local(re[row] - rb[row]));
    }
    const int32_t *cs = halo ? hcol : col;
    const double *vs = halo ? hval : val;
    const long long base = sptr[s];
    const int L = (int)((sptr[s + 1] - base) / 32);
    double y0 = 0.0, y1 = 0.0, y2 = 0.0;
#if FILL_PIPE
    // software pipeline: block j + 1 (and its column / x0 entry) is loaded before block j is
    // stored, so every lane keeps two independent 72-B reads in flight
    double vn[9];
    int cn = row;
    {
      const bool real = 0 < len;
      if (real) cn = cs[k0];
#pragma unroll
      for (int e = 0; e < 9; ++e) vn[e] = real ? vs[9 * k0 + e] : 0.0;
    }
    for (int j = 0; j < L; ++j) {
      const long long t = base + 32LL * j;
      const bool real = j < len;
      const int c = cn;
      double v[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) v[e] = vn[e];
      if (j + 1 < L) {
        const bool rn = j + 1 < len;
        cn = rn ? cs[k0 + j + 1] : row;
        const double *src = vs + 9 * (k0 + j + 1);
#pragma unroll
        for (int e = 0; e < 9; ++e) vn[e] = rn ? src[e] : 0.0;
      }
      scol[t + l] = c;
      double *dst = sval + 9 * t;  // tile of the block column (see blk_load for the layout)
#pragma unroll
      for (int pp = 0; pp < 4; ++pp)  // one 16-B store per component pair: 512 B per warp
        *reinterpret_cast<double2 *>(dst + tile_off(2 * pp, l)) = make_double2(v[2 * pp], v[2 * pp + 1]);
      dst[tile_off(8, l)] = v[8];
      if (x0 && real) {
        const double a0 = x0[3 * (int64_t)c], a1 = x0[3 * (int64_t)c + 1], a2 = x0[3 * (int64_t)c + 2];
        y0 += v[0] * a0 + v[1] * a1 + v[2] * a2;
        y1 += v[3] * a0 + v[4] * a1 + v[5] * a2;
        y2 += v[6] * a0 + v[7] * a1 + v[8] * a2;
      }
    }
#else
    for (int j = 0; j < L; ++j) {
      const long long t = base + 32LL * j;
      const bool real = j < len;
      const int c = real ? cs[k0 + j] : row;
      scol[t + l] = c;
      double *dst = sval + 9 * t;  // tile of the block column (see blk_load for the layout)
      const double *src = vs + 9 * (k0 + j);
      double v[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) v[e] = real ? src[e] : 0.0;
#pragma unroll
      for (int pp = 0; pp < 4; ++pp)  // one 16-B store per component pair: 512 B per warp
        *reinterpret_cast<double2 *>(dst + tile_off(2 * pp, l)) = make_double2(v[2 * pp], v[2 * pp + 1]);
      dst[tile_off(8, l)] = v[8];
      if (x0 && real) {
        const double a0 = x0[3 * (int64_t)c], a1 = x0[3 * (int64_t)c + 1], a2 = x0[3 * (int64_t)c + 2];
        y0 += v[0] * a0 + v[1] * a1 + v[2] * a2;
        y1 += v[3] * a0 + v[4] * a1 + v[5] * a2;
        y2 += v[6] * a0 + v[7] * a1 + v[8] * a2;
      }
    }
#endif
    if (x0 && v >= 0) {
      qx[3 * (int64_t)v] = y0;
      qx[3 * (int64_t)v + 1] = y1;
      qx[3 * (int64_t)v + 2] = y2;
    }
  }
}

// y = A x for A given as its diagonal + upper blocks (NEXT#2, x0 != 0 only): warp per row,
// y_i += A_ij x_j and y_j += A_ij^T x_i (j > i) by fp64 reductions into y (zeroed by the caller).
__global__ void k_ax_upper(int64_t n, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                           const double *__restrict__ val, const double *__restrict__ x, double *y) {
  const int l = lane_id();
  for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < n;
       row += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const double xi0 = x[3 * row], xi1 = x[3 * row + 1], xi2 = x[3 * row + 2];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int64_t k = rp[row] + l; k < rp[row + 1]; k += 32) {
      const int64_t c = col[k];
      const double *m = val + 9 * k;
      const double x0 = x[3 * c], x1 = x[3 * c + 1], x2 = x[3 * c + 2];
      a0 += m[0] * x0 + m[1] * x1 + m[2] * x2;
      a1 += m[3] * x0 + m[4] * x1 + m[5] * x2;
      a2 += m[6] * x0 + m[7] * x1 + m[8] * x2;
      if (c != row) {
        atomicAdd(y + 3 * c, m[0] * xi0 + m[3] * xi1 + m[6] * xi2);
        atomicAdd(y + 3 * c + 1, m[1] * xi0 + m[4] * xi1 + m[7] * xi2);
        atomicAdd(y + 3 * c + 2, m[2] * xi0 + m[5] * xi1 + m[8] * xi2);
      }
    }
    a0 = warp_sum(a0);
    a1 = warp_sum(a1);
    a2 = warp_sum(a2);
    if (l == 0) {
      atomicAdd(y + 3 * row, a0);
      atomicAdd(y + 3 * row + 1, a1);
      atomicAdd(y + 3 * row + 2, a2);
    }
  }
}

// r = b - A x (or b); z = D^-1 r; rz = r.z, rr = r.r, bb = b.b; p_old = 0 and beta = 0, so the
// first K1 forms p = z exactly
__global__ void __launch_bounds__(PCG_THREADS) k_init(int64_t n, const int64_t *__restrict__ rp,
                                                      const int32_t *__restrict__ col, const double *__restrict__ val,
                                                      const double *__restrict__ b, double *__restrict__ x,
                                                      const double *__restrict__ Dinv, double *__restrict__ r,
                                                      double *__restrict__ z, double *__restrict__ p, double *parts,
                                                      PcgState *st, int zero_x0, double *red,
                                                      const double *__restrict__ ax,
                                                      const int64_t *__restrict__ vr_ptr = nullptr,
                                                      const double *__restrict__ qx = nullptr) {
  __shared__ double s_red[PCG_WARPS];
  const int w = threadIdx.x >> 5, l = lane_id();
  double rz = 0.0, rr = 0.0, bb = 0.0;
  auto finish_row = [&](int64_t row, double y0, double y1, double y2) {
    if (zero_x0) {
      x[3 * row] = 0.0; x[3 * row + 1] = 0.0; x[3 * row + 2] = 0.0;
    }
    double b0 = b[3 * row], b1 = b[3 * row + 1], b2 = b[3 * row + 2];
    double r0 = b0 - y0, r1 = b1 - y1, r2 = b2 - y2;
    double z0, z1, z2;
    dinv_apply(Dinv + 9 * row, r0, r1, r2, z0, z1, z2);
    r[3 * row] = r0; r[3 * row + 1] = r1; r[3 * row + 2] = r2;
    z[3 * row] = z0; z[3 * row + 1] = z1; z[3 * row + 2] = z2;
    p[3 * row] = 0.0; p[3 * row + 1] = 0.0; p[3 * row + 2] = 0.0;
    rz += r0 * z0 + r1 * z1 + r2 * z2;
    rr += r0 * r0 + r1 * r1 + r2 * r2;
    bb += b0 * b0 + b1 * b1 + b2 * b2;
  };
  if (zero_x0 || ax || qx) {  // thread per row: (A x0)_row is 0, precomputed, or the sum of the
    // row's virtual-row parts (usually one) -- every row independent, no warp reduction
    const int64_t tstride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n; row += tstride) {
      double y0 = 0.0, y1 = 0.0, y2 = 0.0;
      if (!zero_x0 && ax) {  // (A x)_row precomputed from upper storage (k_ax_upper)
        y0 = ax[3 * row]; y1 = ax[3 * row + 1]; y2 = ax[3 * row + 2];
      } else if (!zero_x0) {  // (A x)_row = sum of its virtual rows' parts (k_sell_fill)
        for (int64_t v = vr_ptr[row]; v < vr_ptr[row + 1]; ++v) {
          y0 += qx[3 * v];
          y1 += qx[3 * v + 1];
          y2 += qx[3 * v + 2];
        }
      }
      finish_row(row, y0, y1, y2);
    }
  } else {
    for (int64_t row = (int64_t)blockIdx.x * PCG_WARPS + w; row < n; row += (int64_t)gridDim.x * PCG_WARPS) {
      // (A x)_row, one warp, lane per block (consecutive 72-B blocks)
      double y0 = 0.0, y1 = 0.0, y2 = 0.0;
      for (int64_t k = rp[row] + l; k < rp[row + 1]; k += 32) {
        const double *B = val + 9 * k;
        const int64_t c = 3 * (int64_t)col[k];
        const double x0 = x[c], x1 = x[c + 1], x2 = x[c + 2];
        y0 += B[0] * x0 + B[1] * x1 + B[2] * x2;
        y1 += B[3] * x0 + B[4] * x1 + B[5] * x2;
        y2 += B[6] * x0 + B[7] * x1 + B[8] * x2;
      }
      y0 = warp_sum(y0);
      y1 = warp_sum(y1);
      y2 = warp_sum(y2);
      if (l == 0) finish_row(row, y0, y1, y2);
    }
  }
  const int G = gridDim.x;
  rz = block_sum(rz, s_red);
  rr = block_sum(rr, s_red);
  bb = block_sum(bb, s_red);
  if (threadIdx.x == 0) {
    parts[blockIdx.x] = rz;
    parts[G + blockIdx.x] = rr;
    parts[2 * G + blockIdx.x] = bb;
  }
  if (last_block(st)) {
    double RZ = reduce_parts(parts, G, s_red);
    double RR = reduce_parts(parts + G, G, s_red);
    double BB = reduce_parts(parts + 2 * G, G, s_red);
    if (threadIdx.x == 0 && red) {  // distributed: rank partials, the caller all-reduces them
      red[0] = RZ; red[1] = RR; red[2] = BB;
      red[3] = st->status == AGIPC_ESINGULAR ? 1.0 : 0.0;  // k_dinv ran before: stops every rank
    } else if (threadIdx.x == 0) {
      st->rz = RZ;
      st->rr = RR;
      st->bn2 = BB;
      st->it = 0;
      st->beta = 0.0;
      if (!st->done && sqrt(RR) <= st->tol * sqrt(BB)) st->done = 1;
    }
  }
}

// ------------------------------------------------------------------------------------
// K1: SELL SpMV, thread per virtual row, fused p update and p.q
// ------------------------------------------------------------------------------------
// loads of one 3x3 block column tile (9 values) and its gathered p_new = z + beta p_old entries
struct BlkLoad {
  double m[9], z[3], p[3];
};
__device__ __forceinline__ void blk_load(BlkLoad &b, const double *__restrict__ tile, int l, int64_t c0,
                                         const double *__restrict__ z, const double *__restrict__ pold) {
  // components (0,1) (2,3) (4,5) (6,7): one 16-B load per lane (512 contiguous bytes per warp);
  // component 8: one 8-B load (256 bytes per warp)
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const double2 v = __ldcs(reinterpret_cast<const double2 *>(tile + 64 * p + 2 * l));
    b.m[2 * p] = v.x;
    b.m[2 * p + 1] = v.y;
  }
  b.m[8] = __ldcs(tile + 256 + l);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    b.z[k] = __ldg(z + c0 + k);
    b.p[k] = __ldg(pold + c0 + k);
  }
}
__device__ __forceinline__ void blk_fma(const BlkLoad &b, double beta, double &a0, double &a1, double &a2) {
  const double x0 = b.z[0] + beta * b.p[0], x1 = b.z[1] + beta * b.p[1], x2 = b.z[2] + beta * b.p[2];
  a0 += b.m[0] * x0 + b.m[1] * x1 + b.m[2] * x2;
  a1 += b.m[3] * x0 + b.m[4] * x1 + b.m[5] * x2;
  a2 += b.m[6] * x0 + b.m[7] * x1 + b.m[8] * x2;
}

// Persistent grid (resident CTAs only); every warp repeatedly claims the next slice of the
// longest-first order from counter[parity] (reset by K2 for the next iteration).  p.q is kept
// per SLICE (pqs[s]) and the last CTA sums the slice partials in slice order, so the result does
// not depend on which warp took which slice: the solve is bit-for-bit reproducible run to run.
// (A static round-robin of the slices, which would also be reproducible, measured 20% slower at
// C3: 103 vs 83 us per SpMV, profiles/r02b.)
template <int UN, int MINB>
__global__ void __launch_bounds__(PCG_THREADS, MINB) k_spmv_sell(const int64_t *__restrict__ sptr,
                                                           const int32_t *__restrict__ scol,
                                                           const double *__restrict__ sval,
                                                           const int32_t *__restrict__ s_vrow,
                                                           const int32_t *__restrict__ order,
                                                           const int32_t *__restrict__ v_row,
                                                           const int64_t *__restrict__ vr_ptr,
                                                           const double *__restrict__ z, const double *__restrict__ pold,
                                                           double *__restrict__ pnew, double *__restrict__ qseg,
                                                           int *counter, double *pqs, PcgState *st,
                                                           double *red) {
  if (*(volatile int *)&st->done) return;
  __shared__ double s_red[PCG_WARPS];
  const double beta = st->beta;
  const long long ns = st->ns;
  const int l = lane_id();
  while (true) {
    int si = 0;
    if (l == 0) si = atomicAdd(counter, 1);
    si = __shfl_sync(FULL_MASK, si, 0);
    if (si >= ns) break;
    const long long s = order[si];
    const long long base = sptr[s];
    const int L = (int)((sptr[s + 1] - base) >> 5);
    const int32_t *cp = scol + base + l;
    const double *vp = sval + 9 * base;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    int64_t nc[UN];  // column offsets of the next UN blocks (prefetched one group ahead)
#pragma unroll
    for (int u = 0; u < UN; ++u) nc[u] = u < L ? 3 * (int64_t)__ldcs(cp + 32 * u) : 0;
    int j = 0;
    for (; j + UN - 1 < L; j += UN) {
      BlkLoad b[UN];  // all 15 UN loads of the group are issued before any FMA
#pragma unroll
      for (int u = 0; u < UN; ++u) blk_load(b[u], vp + 288 * (int64_t)(j + u), l, nc[u], z, pold);
#pragma unroll
      for (int u = 0; u < UN; ++u)
        if (j + UN + u < L) nc[u] = 3 * (int64_t)__ldcs(cp + 32 * (j + UN + u));
#pragma unroll
      for (int u = 0; u < UN; ++u) blk_fma(b[u], beta, a0, a1, a2);  // blocks in column order
    }
#pragma unroll
    for (int u = 0; u < UN - 1; ++u)
      if (j + u < L) {
        BlkLoad b0;
        blk_load(b0, vp + 288 * (int64_t)(j + u), l, nc[u], z, pold);
        blk_fma(b0, beta, a0, a1, a2);
      }
    const int v = s_vrow[32 * s + l];
    double pq = 0.0;
    if (v >= 0) {
      const int64_t row = v_row[v];
      const int64_t i = 3 * row;
      const double pn0 = z[i] + beta * pold[i], pn1 = z[i + 1] + beta * pold[i + 1],
                   pn2 = z[i + 2] + beta * pold[i + 2];
      if (vr_ptr[row] == v) {  // the first segment stores the row's new direction
        pnew[i] = pn0; pnew[i + 1] = pn1; pnew[i + 2] = pn2;
      }
      qseg[3 * (int64_t)v] = a0; qseg[3 * (int64_t)v + 1] = a1; qseg[3 * (int64_t)v + 2] = a2;
      pq = pn0 * a0 + pn1 * a1 + pn2 * a2;  // p.q is linear in the segments
    }
    pq = warp_sum(pq);  // the slice's partial (fixed lane order)
    if (l == 0) pqs[s] = pq;
  }
  if (last_block(st)) {
    double PQ = reduce_parts(pqs, (int)ns, s_red);
    if (threadIdx.x == 0 && red) {
      red[0] = PQ;
    } else if (threadIdx.x == 0) {
      st->pq = PQ;
      if (!isfinite(PQ) || !isfinite(st->rz)) {
        st->status = AGIPC_EBREAKDOWN;
        st->done = 1;
        st->it += 1;
      } else if (PQ <= 0.0) {
        st->status = AGIPC_EINDEFINITE;
        st->done = 1;
        st->it += 1;
      } else {
        st->alpha = st->rz / PQ;
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// K1 on the caller's BSR as it is (no SELL re-layout): warp per row, the row's 9 x nblocks values
// read flat and coalesced (a 15-block fine row is 1,080 contiguous bytes), p_new = z + beta p_old
// formed for every gathered column, segmented sums over the row's 3 output components by warp
// shuffles.  For SHORT solves -- NEXT#1's <= 10 post-coarsening fine iterations -- where
// the per-solve re-layout of the 1.1 GB fine matrix (two extra passes) costs more than the tiling
// gains.  Static row -> warp assignment, so the p.q partials (and the solve) are reproducible.
// ------------------------------------------------------------------------------------
template <int SW>
__global__ void __launch_bounds__(PCG_THREADS) k_spmv_flat(int64_t n, const int64_t *__restrict__ rp,
                                                         const int32_t *__restrict__ col,
                                                         const double *__restrict__ val,
                                                         const double *__restrict__ z, const double *__restrict__ pold,
                                                         double *__restrict__ pnew, double *__restrict__ q,
                                                         double *parts, PcgState *st, double *red) {
  if (*(volatile int *)&st->done) return;
  __shared__ double s_red[PCG_WARPS];
  const double beta = st->beta;
  // SW-lane segment per row, lane per block (consecutive 72-B blocks); 32 / SW rows per warp
  constexpr int RPW = 32 / SW;
  const int l = lane_id(), sl = l % SW, sg = l / SW;
  double pq = 0.0;
  const int64_t W = RPW * (int64_t)gridDim.x * PCG_WARPS;
  for (int64_t row = RPW * ((int64_t)blockIdx.x * PCG_WARPS + (threadIdx.x >> 5)) + sg; row - sg < n; row += W) {
    const bool rv = row < n;
    const int64_t k0 = rv ? rp[row] : 0, k1 = rv ? rp[row + 1] : 0;
    double y0 = 0.0, y1 = 0.0, y2 = 0.0;
    for (int64_t k = k0 + sl; k < k1; k += SW) {
      const double *B = val + 9 * k;
      const int64_t c = 3 * (int64_t)__ldg(col + k);
      double m[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) m[e] = __ldcs(B + e);
      const double x0 = __ldg(z + c) + beta * __ldg(pold + c), x1 = __ldg(z + c + 1) + beta * __ldg(pold + c + 1),
                   x2 = __ldg(z + c + 2) + beta * __ldg(pold + c + 2);
      y0 += m[0] * x0 + m[1] * x1 + m[2] * x2;
      y1 += m[3] * x0 + m[4] * x1 + m[5] * x2;
      y2 += m[6] * x0 + m[7] * x1 + m[8] * x2;
    }
#pragma unroll
    for (int o = SW / 2; o > 0; o >>= 1) {  // sums over the segment (fixed order)
      y0 += __shfl_xor_sync(FULL_MASK, y0, o);
      y1 += __shfl_xor_sync(FULL_MASK, y1, o);
      y2 += __shfl_xor_sync(FULL_MASK, y2, o);
    }
    if (sl == 0 && rv) {
      const int64_t i = 3 * row;
      const double pn0 = z[i] + beta * pold[i], pn1 = z[i + 1] + beta * pold[i + 1], pn2 = z[i + 2] + beta * pold[i + 2];
      pnew[i] = pn0; pnew[i + 1] = pn1; pnew[i + 2] = pn2;
      q[i] = y0; q[i + 1] = y1; q[i + 2] = y2;
      pq += pn0 * y0 + pn1 * y1 + pn2 * y2;
    }
  }
  pq = block_sum(pq, s_red);
  if (threadIdx.x == 0) parts[blockIdx.x] = pq;
  if (last_block(st)) {
    double PQ = reduce_parts(parts, gridDim.x, s_red);
    if (threadIdx.x == 0 && red) {
      red[0] = PQ;
    } else if (threadIdx.x == 0) {
      st->pq = PQ;
      if (!isfinite(PQ) || !isfinite(st->rz)) {
        st->status = AGIPC_EBREAKDOWN;
        st->done = 1;
        st->it += 1;
      } else if (PQ <= 0.0) {
        st->status = AGIPC_EINDEFINITE;
        st->done = 1;
        st->it += 1;
      } else {
        st->alpha = st->rz / PQ;
      }
    }
  }
}

__global__ void k_iota64(int64_t n, int64_t *__restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= n) out[i] = i;
}

// ------------------------------------------------------------------------------------
// K1 of the symmetric solve (NEXT#2, "store ... only the diagonal and upper-triangular
// entries ... reduces memory traffic ... for the subsequent coarse system").  The SELL layout
// holds only the blocks with col >= row, so every stored block is streamed once per iteration
// and used twice: q_i += A_ij p_j (gather, as in k_spmv_sell) and q_j += A_ij^T p_i (scatter,
// j > i).  Persistent CTAs claim whole windows of `win` virtual rows; a window covers the
// contiguous row range [lo, hi] (virtual rows are numbered by row), so a scatter target inside
// it is summed in shared memory and written once by this CTA (y_tin); a target outside, or a
// row whose segments straddle two windows, goes to y_ext by fp64 reductions in L2 (zeroed by
// K2 after use).  p.q = sum_i p_i.(A_ii p_i) + 2 sum_{i<j} p_i.(A_ij p_j) from the gather part.
// Reduction order in shared memory / L2 is not fixed: q is deterministic only up to rounding.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void red_f64(double *p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

__device__ __forceinline__ void sym_blk(const BlkLoad &b, int64_t c3, int64_t i3, double beta, double pi0, double pi1,
                                        double pi2, int64_t lo3, int64_t nr3, double *s_acc, double *yext,
                                        double &d0, double &d1, double &d2, double &o0, double &o1, double &o2) {
  const double x0 = b.z[0] + beta * b.p[0], x1 = b.z[1] + beta * b.p[1], x2 = b.z[2] + beta * b.p[2];
  const double g0 = b.m[0] * x0 + b.m[1] * x1 + b.m[2] * x2;
  const double g1 = b.m[3] * x0 + b.m[4] * x1 + b.m[5] * x2;
  const double g2 = b.m[6] * x0 + b.m[7] * x1 + b.m[8] * x2;
  if (c3 == i3) {  // diagonal block (or SELL padding: zero block pointing at the row)
    d0 += g0; d1 += g1; d2 += g2;
  } else {
    o0 += g0; o1 += g1; o2 += g2;
    const double t0 = b.m[0] * pi0 + b.m[3] * pi1 + b.m[6] * pi2;
    const double t1 = b.m[1] * pi0 + b.m[4] * pi1 + b.m[7] * pi2;
    const double t2 = b.m[2] * pi0 + b.m[5] * pi1 + b.m[8] * pi2;
    const int64_t off = c3 - lo3;
    if ((uint64_t)off < (uint64_t)nr3) {
      atomicAdd(s_acc + off, t0);
      atomicAdd(s_acc + off + 1, t1);
      atomicAdd(s_acc + off + 2, t2);
    } else {
      red_f64(yext + c3, t0);
      red_f64(yext + c3 + 1, t1);
      red_f64(yext + c3 + 2, t2);
    }
  }
}

__global__ void __launch_bounds__(PCG_THREADS, 2) k_spmv_sym(const int64_t *__restrict__ sptr,
                                                          const int32_t *__restrict__ scol,
                                                          const double *__restrict__ sval,
                                                          const int32_t *__restrict__ s_vrow,
                                                          const int32_t *__restrict__ v_row,
                                                          const int64_t *__restrict__ vr_ptr,
                                                          const double *__restrict__ z, const double *__restrict__ pold,
                                                          double *__restrict__ pnew, double *__restrict__ qseg,
                                                          double *__restrict__ ytin, double *yext, int win,
                                                          int *counter, double *parts, PcgState *st, int all_red) {
  if (*(volatile int *)&st->done) return;
  extern __shared__ double s_acc[];  // [3 * win]
  __shared__ double s_red[PCG_WARPS];
  __shared__ int s_w;
  const double beta = st->beta;
  const long long ns = st->ns, nv = st->nv;
  const long long nwin = (nv + win - 1) / win;
  const int l = lane_id(), w = threadIdx.x >> 5;
  const int spw = win >> 5;  // slices per window
  double pq = 0.0;
  while (true) {
    if (threadIdx.x == 0) s_w = atomicAdd(counter, 1);
    __syncthreads();
    const long long W = s_w;
    if (W >= nwin) break;
    const long long v0 = W * win, v1 = min(v0 + win, nv);
    const int64_t lo = v_row[v0], hi = v_row[v1 - 1];
    const int nr = (int)(hi - lo + 1);
    const int64_t nr3 = all_red ? 0 : 3 * (int64_t)nr;  // all_red: every scatter target through L2
    for (int t = threadIdx.x; t < 3 * nr; t += PCG_THREADS) s_acc[t] = 0.0;
    __syncthreads();
    const long long s_end = min((W + 1) * spw, ns);
    for (long long s = W * spw + w; s < s_end; s += PCG_WARPS) {
      const long long base = sptr[s];
      const int L = (int)((sptr[s + 1] - base) >> 5);
      const int32_t *cp = scol + base + l;
      const double *vp = sval + 9 * base;
      const int v = s_vrow[32 * s + l];
      const int64_t row = v >= 0 ? v_row[v] : -1;
      const int64_t i3 = 3 * row;
      double pi0 = 0.0, pi1 = 0.0, pi2 = 0.0;
      if (v >= 0) {
        pi0 = z[i3] + beta * pold[i3];
        pi1 = z[i3 + 1] + beta * pold[i3 + 1];
        pi2 = z[i3 + 2] + beta * pold[i3 + 2];
      }
      double d0 = 0.0, d1 = 0.0, d2 = 0.0, o0 = 0.0, o1 = 0.0, o2 = 0.0;
      // padding lanes (v < 0) hold zero blocks pointing at row 0: treat them as diagonal
      const int64_t ii3 = v >= 0 ? i3 : -1;
      int64_t n0 = L > 0 ? 3 * (int64_t)__ldcs(cp) : 0, n1 = L > 1 ? 3 * (int64_t)__ldcs(cp + 32) : 0;
      int j = 0;
      for (; j + 1 < L; j += 2) {
        BlkLoad b0, b1;
        const int64_t c0 = n0, c1 = n1;
        blk_load(b0, vp + 288 * (int64_t)j, l, c0, z, pold);
        blk_load(b1, vp + 288 * (int64_t)(j + 1), l, c1, z, pold);
        if (j + 2 < L) n0 = 3 * (int64_t)__ldcs(cp + 32 * (j + 2));
        if (j + 3 < L) n1 = 3 * (int64_t)__ldcs(cp + 32 * (j + 3));
        sym_blk(b0, v >= 0 ? c0 : -1, ii3, beta, pi0, pi1, pi2, 3 * lo, nr3, s_acc, yext, d0, d1, d2, o0, o1, o2);
        sym_blk(b1, v >= 0 ? c1 : -1, ii3, beta, pi0, pi1, pi2, 3 * lo, nr3, s_acc, yext, d0, d1, d2, o0, o1, o2);
      }
      if (j < L) {
        BlkLoad b0;
        const int64_t c0 = n0;
        blk_load(b0, vp + 288 * (int64_t)j, l, c0, z, pold);
        sym_blk(b0, v >= 0 ? c0 : -1, ii3, beta, pi0, pi1, pi2, 3 * lo, nr3, s_acc, yext, d0, d1, d2, o0, o1, o2);
      }
      if (v >= 0) {
        if (vr_ptr[row] == v) {  // the first segment stores the row's new direction
          pnew[i3] = pi0; pnew[i3 + 1] = pi1; pnew[i3 + 2] = pi2;
        }
        qseg[3 * (int64_t)v] = d0 + o0;
        qseg[3 * (int64_t)v + 1] = d1 + o1;
        qseg[3 * (int64_t)v + 2] = d2 + o2;
        pq += pi0 * d0 + pi1 * d1 + pi2 * d2 + 2.0 * (pi0 * o0 + pi1 * o1 + pi2 * o2);
      }
    }
    __syncthreads();
    // flush: rows whose virtual rows all lie in this window are owned here (plain stores);
    // a straddling row receives scatter from two windows and goes through L2 reductions
    for (int t = threadIdx.x; t < nr; t += PCG_THREADS) {
      const int64_t row = lo + t;
      const double a0 = s_acc[3 * t], a1 = s_acc[3 * t + 1], a2 = s_acc[3 * t + 2];
      if (vr_ptr[row] >= v0 && vr_ptr[row + 1] <= v1) {
        ytin[3 * row] = a0; ytin[3 * row + 1] = a1; ytin[3 * row + 2] = a2;
      } else {
        red_f64(yext + 3 * row, a0);
        red_f64(yext + 3 * row + 1, a1);
        red_f64(yext + 3 * row + 2, a2);
      }
    }
    __syncthreads();
  }
  pq = block_sum(pq, s_red);
  if (threadIdx.x == 0) parts[blockIdx.x] = pq;
  if (last_block(st)) {
    double PQ = reduce_parts(parts, gridDim.x, s_red);
    if (threadIdx.x == 0) {
      st->pq = PQ;
      if (!isfinite(PQ) || !isfinite(st->rz)) {
        st->status = AGIPC_EBREAKDOWN;
        st->done = 1;
        st->it += 1;
      } else if (PQ <= 0.0) {
        st->status = AGIPC_EINDEFINITE;
        st->done = 1;
        st->it += 1;
      } else {
        st->alpha = st->rz / PQ;
      }
    }
  }
}

// K2: thread per slot; q = sum of the row's segments (fixed order); x += alpha p; r -= alpha q;
// z = D^-1 r; last CTA: ||r|| <= tol ||b||, iteration count, beta.  Each thread takes U
// slots per pass and issues all their independent loads before the arithmetic (the kernel is
// latency-bound at 2 CTAs per SM, the grid size that keeps the last-block reduction cheap).
template <int U, int NT = PCG_THREADS>
__global__ void __launch_bounds__(NT) k_update(int64_t n, const int64_t *__restrict__ vr_ptr,
                                                        double *__restrict__ x, double *__restrict__ r,
                                                        double *__restrict__ z, const double *__restrict__ p,
                                                        const double *__restrict__ qseg,
                                                        const double *__restrict__ Dinv, int *next_counter,
                                                        double *parts, PcgState *st, double *red,
                                                        const double *__restrict__ ytin, double *__restrict__ yext) {
  if (*(volatile int *)&st->done) return;
  __shared__ double s_red[NT / 32];
  const double alpha = st->alpha;
  if (blockIdx.x == 0 && threadIdx.x == 0) *next_counter = 0;
  double rz = 0.0, rr = 0.0;
  const int64_t stride = (int64_t)gridDim.x * NT;
  for (int64_t i0 = (int64_t)blockIdx.x * NT + threadIdx.x; i0 < n; i0 += U * stride) {
    int64_t v0[U], v1[U];
    double q[U][3], xv[U][3], rv[U][3], pv[U][3], D[U][9];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) {
        v0[u] = vr_ptr[i]; v1[u] = vr_ptr[i + 1];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          xv[u][c] = x[3 * i + c]; rv[u][c] = r[3 * i + c]; pv[u][c] = p[3 * i + c];
        }
#pragma unroll
        for (int e = 0; e < 9; ++e) D[u][e] = Dinv[9 * i + e];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) {
        q[u][0] = qseg[3 * v0[u]]; q[u][1] = qseg[3 * v0[u] + 1]; q[u][2] = qseg[3 * v0[u] + 2];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= n) continue;
      for (int64_t v = v0[u] + 1; v < v1[u]; ++v) {
        q[u][0] += qseg[3 * v];
        q[u][1] += qseg[3 * v + 1];
        q[u][2] += qseg[3 * v + 2];
      }
      const int64_t k = 3 * i;
      if (yext) {  // symmetric solve: the scattered A_ji^T p_j parts (NEXT#2); y_ext is re-zeroed
        q[u][0] += ytin[k] + yext[k];
        q[u][1] += ytin[k + 1] + yext[k + 1];
        q[u][2] += ytin[k + 2] + yext[k + 2];
        yext[k] = 0.0; yext[k + 1] = 0.0; yext[k + 2] = 0.0;
      }
      x[k] = xv[u][0] + alpha * pv[u][0];
      x[k + 1] = xv[u][1] + alpha * pv[u][1];
      x[k + 2] = xv[u][2] + alpha * pv[u][2];
      const double r0 = rv[u][0] - alpha * q[u][0], r1 = rv[u][1] - alpha * q[u][1], r2 = rv[u][2] - alpha * q[u][2];
      r[k] = r0; r[k + 1] = r1; r[k + 2] = r2;
      double z0, z1, z2;
      dinv_apply(D[u], r0, r1, r2, z0, z1, z2);
      z[k] = z0; z[k + 1] = z1; z[k + 2] = z2;
      rz += r0 * z0 + r1 * z1 + r2 * z2;
      rr += r0 * r0 + r1 * r1 + r2 * r2;
    }
  }
  const int G = gridDim.x;
  rz = block_sum<NT>(rz, s_red);
  rr = block_sum<NT>(rr, s_red);
  if (threadIdx.x == 0) {
    parts[G + blockIdx.x] = rz;
    parts[2 * G + blockIdx.x] = rr;
  }
  if (last_block(st)) {
    double RZ = reduce_parts<NT>(parts + G, G, s_red);
    double RR = reduce_parts<NT>(parts + 2 * G, G, s_red);
    if (threadIdx.x == 0 && red) {
      red[0] = RZ; red[1] = RR;
    } else if (threadIdx.x == 0) {
      st->it += 1;
      st->rr = RR;
      if (sqrt(RR) <= st->tol * sqrt(st->bn2)) {
        st->done = 1;
        st->status = AGIPC_OK;
      } else if (st->it >= st->max_iters) {
        st->done = 1;
        st->status = AGIPC_NOT_CONVERGED;
      } else {
        st->beta = RZ / st->rz;
        st->rz = RZ;
      }
    }
  }
}

__global__ void k_copy_out(int64_t n3, const double *__restrict__ src, double *__restrict__ dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n3) dst[i] = src[i];
}

typedef void (*SpmvKernel)(const int64_t *, const int32_t *, const double *, const int32_t *, const int32_t *,
                           const int32_t *, const int64_t *, const double *, const double *, double *, double *,
                           int *, double *, PcgState *, double *);
// k_spmv_sell variants: UN blocks per thread in flight at MINB CTAs per SM (register budget)
static SpmvKernel spmv_kernel(int un) {
  return un == 4 ? k_spmv_sell<4, 2> : un == 3 ? k_spmv_sell<3, 2> : k_spmv_sell<2, 3>;
}

struct PcgBufs {
  double *x, *r, *z, *P[2], *qseg, *Dinv, *parts, *sval;
  double *pqs;  // per-slice p.q partials of K1 (summed in slice order by its last CTA)
  int64_t *vr_ptr, *sptr;
  int32_t *v_row, *v_len, *perm, *scol, *s_vrow, *order;
  int *counters;  // two slice counters, used by alternate iterations
  PcgState *st;
  int64_t ns_bound;
  int G1, G2;
  // symmetric solve (NEXT#2): windows of `win` virtual rows, scatter targets y_tin / y_ext
  bool sym = false;
  int win = SORT_WIN;
  double *ytin = nullptr, *yext = nullptr;
  int all_red = 0;
  int upd_u = 1;  // slots per K2 thread pass
  double *arena = nullptr;  // x, r, z, p0, p1, qseg, Dinv (+ ytin, yext): one L2 window
  int spmv_un = 3;          // blocks per thread in flight in k_spmv_sell
  size_t arena_bytes = 0;
  bool flat = false;        // K1 = k_spmv_flat on the caller's BSR (short solves, no re-layout)
  const int64_t *A_rp = nullptr;
  const int32_t *A_col = nullptr;
  const double *A_val = nullptr;
  int64_t n = 0;
};


// L2 residency of the PCG vectors (B200: 126 MB L2), opt-in (agipc_set_option AGIPC_OPT_L2_PERSIST):
// the matrix is streamed with evict-first loads; when the whole vector arena fits in the requested
// persisting size, the solve stream gets a persisting access-policy window over it (the captured
// kernel nodes inherit it) and the device's persisting carve-out is set to the arena for the
// solve and restored afterwards (pcg_l2_release).  A window larger than the carve-out thrashes and
// a carve-out without a window only shrinks the normal L2 (C4, 1.1M slots: SpMV 386 -> 273 us,
// K2 107 -> 54 us without either, profiles/r02f), so neither is set then.
struct L2Win {
  bool on = false;
  size_t prev_limit = 0;
};

static L2Win pcg_l2_window(agipc_handle h, cudaStream_t s, const void *base, size_t bytes) {
  L2Win r;
  cudaStreamAttrValue v;
  memset(&v, 0, sizeof(v));
  int max_win = 0;
  cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, h->device);
  const bool on = h->opt_l2_persist > 0 && base && bytes > 0 && bytes <= h->opt_l2_persist && max_win > 0 &&
                  bytes <= (size_t)max_win;
  if (on && cudaDeviceGetLimit(&r.prev_limit, cudaLimitPersistingL2CacheSize) == cudaSuccess &&
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes) == cudaSuccess) {
    v.accessPolicyWindow.base_ptr = const_cast<void *>(base);
    v.accessPolicyWindow.num_bytes = bytes;
    v.accessPolicyWindow.hitRatio = 1.0f;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    r.on = true;
  }
  cudaGetLastError();
  if (cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess) cudaGetLastError();
  return r;
}

static void pcg_l2_release(cudaStream_t s, const L2Win &w) {
  if (!w.on) return;
  cudaStreamAttrValue v;
  memset(&v, 0, sizeof(v));
  if (cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess) cudaGetLastError();
  if (cudaCtxResetPersistingL2Cache() != cudaSuccess) cudaGetLastError();
  if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, w.prev_limit) != cudaSuccess) cudaGetLastError();
}

// iteration j reads p_old = P[j&1] and writes p_new = P[(j+1)&1] (the chunk length is even)
static agipc_status enqueue_iters(agipc_handle h, cudaStream_t s, int iters, int64_t n, const PcgBufs &B,
                                  cudaEvent_t *ev) {
  for (int k = 0; k < iters; ++k) {
    double *pold = B.P[k & 1], *pnew = B.P[(k + 1) & 1];
    const bool sample = ev && (k % PROF_EVERY) == 0;  // sampled kernel timing (low overhead)
    if (sample) cudaEventRecordWithFlags(ev[3 * k], s, cudaEventRecordExternal);
    if (B.flat)
      k_spmv_flat<8><<<B.G1, PCG_THREADS, 0, s>>>(B.n, B.A_rp, B.A_col, B.A_val, B.z, pold, pnew, B.qseg, B.parts, B.st,
                                               nullptr);
    else if (B.sym)
      k_spmv_sym<<<B.G1, PCG_THREADS, 3 * sizeof(double) * B.win, s>>>(
          B.sptr, B.scol, B.sval, B.s_vrow, B.v_row, B.vr_ptr, B.z, pold, pnew, B.qseg, B.ytin, B.yext, B.win,
          B.counters + (k & 1), B.parts, B.st, B.all_red);
    else
      spmv_kernel(B.spmv_un)<<<B.G1, PCG_THREADS, 0, s>>>(B.sptr, B.scol, B.sval, B.s_vrow, B.order, B.v_row,
                                                          B.vr_ptr, B.z, pold, pnew, B.qseg, B.counters + (k & 1),
                                                          B.pqs, B.st, nullptr);
    if (sample) cudaEventRecordWithFlags(ev[3 * k + 1], s, cudaEventRecordExternal);
    k_update<1, PCG_THREADS><<<B.G2, PCG_THREADS, 0, s>>>(n, B.vr_ptr, B.x, B.r, B.z, pnew, B.qseg, B.Dinv, B.counters + ((k + 1) & 1),
                                          B.parts, B.st, nullptr, B.ytin, B.yext);
    if (sample) cudaEventRecordWithFlags(ev[3 * k + 2], s, cudaEventRecordExternal);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(h, AGIPC_ECUDA, "pcg launch: %s", cudaGetErrorString(e));
  return AGIPC_OK;
}

// Block-Jacobi + SELL layout + k_init, shared by the 1-GPU solve and the distributed solve.
// Ah (nullable): halo matrix of the rank's rows x ghost columns (columns >= n index the ghost
// region of the vectors, n_gs slots).  red != nullptr: k_init leaves rank partials in red.
// storage (1-GPU solve only): AGIPC_STORAGE_FULL streams every block (k_spmv_sell);
// AGIPC_STORAGE_SYM keeps only the diagonal + upper blocks of a full-storage A in the SELL copy
// and AGIPC_STORAGE_UPPER takes A already stored that way; both run k_spmv_sym (NEXT#2).
static agipc_status pcg_setup(agipc_handle h, const agipc_bsr *A, const agipc_bsr *Ah, int64_t n_gs, const double *b,
                              const double *x, int zero_x0, double rel_tol, int max_iters, PcgBufs &B,
                              PcgState *hst, double *red, int storage = AGIPC_STORAGE_FULL,
                              const char *pfx = "pcg_", bool flat = false, bool stat = false) {
#define PN(x) (std::string(pfx) + (x)).c_str()  // the distributed solve has its own buffers
  const int64_t n = A->n_rows;
  B.sym = storage != AGIPC_STORAGE_FULL;
  B.flat = flat && !B.sym && !Ah;
  B.n = n;
  B.A_rp = A->row_ptr;
  B.A_col = A->col;
  B.A_val = A->val;
  B.win = SORT_WIN;
  if (B.sym) {
    B.win = 1024;
    if (const char *e = getenv("AGIPC_SYM_WIN")) {  // experiments: 128 .. 4096, power of two
      int w = atoi(e);
      if (w >= 128 && w <= SORT_WIN && (w & (w - 1)) == 0) B.win = w;
    }
    B.all_red = getenv("AGIPC_SYM_RED") ? 1 : 0;
  }
  const int64_t nh = Ah ? Ah->nnzb : 0;
  cudaStream_t s0 = h->stream;
  const int64_t nv_bound = n + (A->nnzb + nh) / SEG_MAX + (Ah ? n : 0) + 1;  // virtual rows
  const int64_t nx = n + n_gs;  // owned + ghost slots (z and p carry the ghost region)
  B.ns_bound = cdiv(nv_bound, 32);
  // the per-iteration vectors live in one arena so that one L2 access-policy window (persisting)
  // covers them: the SpMV streams the matrix with evict-first loads, K2 and the gathers then hit
  // L2 instead of HBM (pcg_l2_window)
  {
    const int64_t len[9] = {3 * n + 2, 3 * n + 2, 3 * nx + 2, 3 * nx + 2, 3 * nx + 2, 3 * nv_bound + 2, 9 * n + 2,
                            storage != AGIPC_STORAGE_FULL ? 3 * n + 2 : 0, storage != AGIPC_STORAGE_FULL ? 3 * n + 2 : 0};
    int64_t off[10];
    off[0] = 0;
    for (int i = 0; i < 9; ++i) off[i + 1] = off[i] + ((len[i] + 31) & ~(int64_t)31);  // 256-B aligned
    WS(h, arena, double, PN("vec_arena"), off[9]);
    B.x = arena + off[0]; B.r = arena + off[1]; B.z = arena + off[2];
    B.P[0] = arena + off[3]; B.P[1] = arena + off[4]; B.qseg = arena + off[5]; B.Dinv = arena + off[6];
    B.ytin = len[7] ? arena + off[7] : nullptr;
    B.yext = len[8] ? arena + off[8] : nullptr;
    B.arena = arena;
    B.arena_bytes = sizeof(double) * (size_t)off[9];
  }
  WS(h, vr, int64_t, PN("vr_ptr"), n + 1); B.vr_ptr = vr;
  WS(h, nseg, int32_t, PN("nseg"), n);
  WS(h, vrow, int32_t, PN("v_row"), nv_bound); B.v_row = vrow;
  WS(h, vlen, int32_t, PN("v_len"), nv_bound); B.v_len = vlen;
  WS(h, perm, int32_t, PN("perm"), nv_bound); B.perm = perm;
  WS(h, slen, int32_t, PN("slen"), B.ns_bound);
  WS(h, sptr, int64_t, PN("sptr"), B.ns_bound + 1); B.sptr = sptr;
  WS(h, svr, int32_t, PN("s_vrow"), 32 * B.ns_bound); B.s_vrow = svr;
  WS(h, stp, PcgState, PN("state"), 1); B.st = stp;
  WS(h, order, int32_t, PN("order"), B.ns_bound); B.order = order;
  WS(h, ctr, int, PN("counters"), 2); B.counters = ctr;
  WS(h, pqs, double, PN("pqs"), B.ns_bound + 1); B.pqs = pqs;
  int occ = 0;
  if (B.sym) {
    const size_t smem = 3 * sizeof(double) * B.win;
    CU_TRY(h, cudaFuncSetAttribute(k_spmv_sym, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_spmv_sym, PCG_THREADS, smem));
    B.G1 = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(nv_bound, B.win), (int64_t)std::max(1, occ) * h->sm_count));
  } else {
    // 3 blocks per thread in flight at 2 CTAs/SM: 82.0 -> 76.7 us per SpMV at C3 vs 2 at 3 CTAs/SM
    // (4 at 2 CTAs/SM: 77.9 us; profiles/r01o/un*.txt).  AGIPC_SPMV_UN selects another variant.
    B.spmv_un = 3;
    if (const char *e = getenv("AGIPC_SPMV_UN")) B.spmv_un = atoi(e) == 4 ? 4 : atoi(e) == 2 ? 2 : 3;
    CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spmv_kernel(B.spmv_un), PCG_THREADS, 0));
    B.G1 = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(B.ns_bound, PCG_WARPS), (int64_t)std::max(1, occ) * h->sm_count));
  }
  if (B.flat) B.G1 = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 4 * PCG_WARPS), 8 * (int64_t)h->sm_count));
  // K2: 2 CTAs of 256 threads per SM, 1 slot per thread pass (profiles/r01h/update_exp.jsonl,
  // upd_nt.jsonl: 3-8 CTAs per SM, 2 slots per pass or 512-thread CTAs are not faster)
  B.upd_u = 1;
  B.G2 = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, PCG_THREADS), 2 * (int64_t)h->sm_count));
  const int Gi = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, PCG_WARPS), 8 * (int64_t)h->sm_count));
  const int Gp = std::max(std::max(B.G1, B.G2), Gi);
  WS(h, parts, double, PN("parts"), 3 * Gp); B.parts = parts;
  // static pattern (agipc_pcg_set_static): the SELL layout of the previous solve on the same
  // row_ptr / col is reused when its buffers are still in place; only the values are refilled
  const void *pat_bufs[8] = {B.vr_ptr, B.v_row, B.v_len, B.perm, B.sptr, B.s_vrow, B.order, nullptr};
  bool reuse = stat && h->spat.built;
  for (int i = 0; i < 7 && reuse; ++i) reuse = h->spat.bufs[i] == pat_bufs[i];
  PcgState init;
  memset(&init, 0, sizeof(init));
  init.tol = rel_tol;
  init.max_iters = max_iters;
  init.status = AGIPC_OK;
  if (reuse) {
    init.nv = h->spat.nv;
    init.ns = h->spat.ns;
    init.sell_blocks = h->spat.sell_blocks;
  }
  *hst = init;
  ProfScope prof_setup(h, PROF_PCG_SETUP, s0);
  CU_TRY(h, cudaMemcpyAsync(stp, hst, sizeof(PcgState), cudaMemcpyHostToDevice, s0));
  if (!zero_x0) CU_TRY(h, cudaMemcpyAsync(B.x, x, sizeof(double) * 3 * n, cudaMemcpyDeviceToDevice, s0));
  if (n_gs > 0) {  // ghost p starts at 0 like the owned p (beta = 0 in the first iteration)
    CU_TRY(h, cudaMemsetAsync(B.P[0] + 3 * n, 0, sizeof(double) * 3 * n_gs, s0));
    CU_TRY(h, cudaMemsetAsync(B.P[1] + 3 * n, 0, sizeof(double) * 3 * n_gs, s0));
  }
  const int64_t *rb = A->row_ptr, *re = A->row_ptr + 1;
  int64_t *ub = nullptr;
  if (storage == AGIPC_STORAGE_SYM) {
    WS(h, ubw, int64_t, PN("ub"), n + 1); ub = ubw; rb = ubw;
  }
  LAUNCH(h, k_dinv, (unsigned)cdiv(n, 256), 256, 0, n, A->row_ptr, A->col, A->val, B.Dinv, stp, ub,
         storage == AGIPC_STORAGE_UPPER ? 1 : 0);
  if (B.flat) {  // one "segment" per row: K2 sums q[vr_ptr[i] .. vr_ptr[i+1]) = q[i]
    LAUNCH(h, k_iota64, (unsigned)cdiv(n + 1, 256), 256, 0, n, B.vr_ptr);
    LAUNCH(h, k_init, (unsigned)Gi, PCG_THREADS, 0, n, A->row_ptr, A->col, A->val, b, B.x, B.Dinv, B.r, B.z, B.P[0],
           parts, stp, zero_x0, red, (const double *)nullptr);
    CU_TRY(h, cudaMemcpyAsync(hst, stp, sizeof(PcgState), cudaMemcpyDeviceToHost, s0));
    return AGIPC_OK;
  }
  // SELL layout (once per solve, or once per static pattern)
  const int64_t *hrp = Ah ? Ah->row_ptr : nullptr;
  // A x0 of a full-storage, halo-free solve from x0 != 0 rides on the value fill
  const bool fuse_ax = !zero_x0 && !Ah && !B.sym && storage == AGIPC_STORAGE_FULL;
  if (!reuse) {
    LAUNCH(h, k_seg_count, (unsigned)cdiv(n, 256), 256, 0, n, rb, re, hrp, nseg);
    agipc_status sst = scan_exclusive_i64(h, SCAN_SRC_I32, nseg, n, B.vr_ptr);
    if (sst != AGIPC_OK) return sst;
    LAUNCH(h, k_seg_fill, (unsigned)cdiv(n, 256), 256, 0, n, rb, re, hrp, B.vr_ptr, B.v_row, B.v_len, stp);
    CU_TRY(h, cudaFuncSetAttribute(k_window_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(sizeof(unsigned long long) * SORT_WIN)));
    LAUNCH(h, k_window_sort, (unsigned)cdiv(nv_bound, B.win), 1024, sizeof(unsigned long long) * B.win, stp, B.v_len,
           B.perm, B.win);
    LAUNCH(h, k_slice_len, (unsigned)cdiv(B.ns_bound, 256), 256, 0, B.ns_bound, stp, B.perm, B.v_len, slen);
    sst = scan_exclusive_i64(h, SCAN_SRC_I32, slen, B.ns_bound, B.sptr);
    if (sst != AGIPC_OK) return sst;
    LAUNCH(h, k_sell_scalars, 1, 1, 0, B.ns_bound, B.sptr, stp);
    LAUNCH(h, k_slice_order, 1, 1024, 0, stp, slen, B.order);
    CU_TRY(h, cudaMemcpyAsync(hst, stp, sizeof(PcgState), cudaMemcpyDeviceToHost, s0));
    CU_TRY(h, cudaStreamSynchronize(s0));
    if (stat) {
      h->spat.built = true;
      h->spat.nv = hst->nv;
      h->spat.ns = hst->ns;
      h->spat.sell_blocks = hst->sell_blocks;
      for (int i = 0; i < 8; ++i) h->spat.bufs[i] = pat_bufs[i];
    }
  }
  CU_TRY(h, cudaMemsetAsync(B.counters, 0, 2 * sizeof(int), s0));
  const long long sell_blocks = hst->sell_blocks;
  WS(h, scol, int32_t, PN("scol"), sell_blocks + 32); B.scol = scol;
  WS(h, sval, double, PN("sval"), 9 * sell_blocks + 288); B.sval = sval;
  LAUNCH(h, k_sell_fill, (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(hst->ns, 8), 16 * h->sm_count)), 256,
         0, stp, rb, re, A->col, A->val, hrp, Ah ? Ah->col : nullptr, Ah ? Ah->val : nullptr, B.vr_ptr, B.perm,
         B.v_row, B.v_len, B.sptr, B.scol, B.sval, B.s_vrow, fuse_ax ? (const double *)B.x : nullptr, B.qseg);
  const double *ax = nullptr;
  if (B.sym) {
    CU_TRY(h, cudaMemsetAsync(B.ytin, 0, sizeof(double) * 3 * n, s0));  // straddling rows keep 0
    CU_TRY(h, cudaMemsetAsync(B.yext, 0, sizeof(double) * 3 * n, s0));
    if (storage == AGIPC_STORAGE_UPPER && !zero_x0) {  // r = b - A x0 from the upper half
      WS(h, axw, double, PN("ax"), 3 * n + 2);
      CU_TRY(h, cudaMemsetAsync(axw, 0, sizeof(double) * 3 * n, s0));
      LAUNCH(h, k_ax_upper, (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 8), 16 * h->sm_count)), 256, 0, n,
             A->row_ptr, A->col, A->val, B.x, axw);
      ax = axw;
    }
  }
  LAUNCH(h, k_init, (unsigned)Gi, PCG_THREADS, 0, n, A->row_ptr, A->col, A->val, b, B.x, B.Dinv, B.r, B.z, B.P[0],
         parts, stp, zero_x0, red, ax, (const int64_t *)B.vr_ptr, fuse_ax ? (const double *)B.qseg : nullptr);
  return AGIPC_OK;
#undef PN
}

static agipc_status pcg_solve_impl(agipc_handle h, const agipc_bsr *A, int storage, const double *b, double *x,
                                   int zero_x0, double rel_tol, int max_iters, int check_every,
                                   agipc_pcg_stats *stats) {
  if (!h) return AGIPC_EINVAL;
  if (!A || !stats || max_iters < 0 || A->n_rows < 0 || !(rel_tol >= 0.0))
    return set_err(h, AGIPC_EINVAL, "pcg_solve: bad arguments");
  const int64_t n = A->n_rows;
  memset(stats, 0, sizeof(*stats));
  if (n == 0) return AGIPC_OK;
  if (!A->row_ptr || !A->col || !A->val || !b || !x) return set_err(h, AGIPC_EINVAL, "pcg_solve: null pointer");
  if (n >= INT32_MAX / 4 || A->nnzb >= ((int64_t)1 << 40)) return set_err(h, AGIPC_ERANGE, "pcg_solve: too large");
  if (check_every <= 0) check_every = 16;
  CU_TRY(h, cudaSetDevice(h->device));
  cudaStream_t s0 = h->stream;
  agipc_status ast;
  PcgState *hst = (PcgState *)pinned_get(h, sizeof(PcgState), &ast);
  if (ast != AGIPC_OK) return ast;
  PcgBufs B;
  // short solves (NEXT#1: <= 10 post-coarsening fine iterations) stream the caller's BSR
  // flat instead of re-laying it out; AGIPC_PCG_FLAT=0/1 forces a variant (A/B runs)
  const bool stat = storage == AGIPC_STORAGE_FULL && h->spat.rp == A->row_ptr && h->spat.col == A->col &&
                    h->spat.n == n && h->spat.nnzb == A->nnzb;
  bool flat = storage == AGIPC_STORAGE_FULL && max_iters <= 32 && !stat;
  if (const char *e = getenv("AGIPC_PCG_FLAT")) flat = storage == AGIPC_STORAGE_FULL && atoi(e) != 0;
  ast = pcg_setup(h, A, nullptr, 0, b, x, zero_x0, rel_tol, max_iters, B, hst, nullptr, storage,
                  stat && !flat ? "pcgs_" : "pcg_", flat, stat && !flat);
  if (ast != AGIPC_OK) return ast;
  if (max_iters == 0) {
    CU_TRY(h, cudaMemcpyAsync(hst, B.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s0));
    CU_TRY(h, cudaStreamSynchronize(s0));
  } else {
    PcgGraph *&gslot = (stat && !flat) ? h->pcg_static : h->pcg;  // one cached graph per kind
    PcgGraph *g = gslot;
    if (!g) {
      g = gslot = new PcgGraph();
      CU_TRY(h, cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
      CU_TRY(h, cudaEventCreateWithFlags(&g->ev_in, cudaEventDisableTiming));
      CU_TRY(h, cudaEventCreateWithFlags(&g->ev_out, cudaEventDisableTiming));
    }
    int chunk = std::max(2, std::min(check_every, max_iters));
    chunk += chunk & 1;  // even: the p ping-pong parity is the same at every graph launch
    const L2Win l2win = pcg_l2_window(h, g->stream, B.arena, B.arena_bytes);
    const void *key[8] = {B.flat ? (const void *)B.A_val : B.sval, B.flat ? (const void *)B.A_col : B.scol, B.x, B.qseg,
                          B.Dinv, B.flat ? (const void *)B.A_rp : B.sptr, B.P[0], B.parts};
    // ws_gen changes whenever any named buffer moved (every pointer baked into the graph is one)
    bool same = g->exec && g->ws_gen == h->ws_gen && g->n == n && g->ns == B.ns_bound && g->chunk == chunk && g->grid1 == B.G1 &&
                g->grid2 == B.G2 && g->prof == h->prof && g->sym == B.sym && g->win == B.win && g->yext == B.yext &&
                g->all_red == B.all_red && g->upd_u == B.upd_u &&
                g->spmv_un == B.spmv_un && g->flat == B.flat && g->n_flat == B.n && g->l2on == l2win.on;
    for (int i = 0; i < 8 && same; ++i) same = g->key[i] == key[i];
    if (!same) {
      if (g->exec) {
        cudaGraphExecDestroy(g->exec);
        g->exec = nullptr;
      }
      while (h->prof && (int)g->ev.size() < 3 * chunk) {
        cudaEvent_t e;
        CU_TRY(h, cudaEventCreate(&e));
        g->ev.push_back(e);
      }
      cudaGraph_t graph;
      CU_TRY(h, cudaStreamBeginCapture(g->stream, cudaStreamCaptureModeThreadLocal));
      agipc_status es = enqueue_iters(h, g->stream, chunk, n, B, h->prof ? g->ev.data() : nullptr);
      cudaError_t ce = cudaStreamEndCapture(g->stream, &graph);
      if (es != AGIPC_OK) return es;
      if (ce != cudaSuccess) return set_err(h, AGIPC_ECUDA, "pcg capture: %s", cudaGetErrorString(ce));
      CU_TRY(h, cudaGraphInstantiate(&g->exec, graph, 0));
      cudaGraphDestroy(graph);
      g->n = n;
      g->ns = B.ns_bound;
      g->chunk = chunk;
      g->grid1 = B.G1;
      g->grid2 = B.G2;
      g->prof = h->prof;
      g->sym = B.sym;
      g->win = B.win;
      g->yext = B.yext;
      g->all_red = B.all_red;
      g->upd_u = B.upd_u;
      g->spmv_un = B.spmv_un;
      g->ws_gen = h->ws_gen;
      g->flat = B.flat;
      g->n_flat = B.n;
      g->l2on = l2win.on;
      for (int i = 0; i < 8; ++i) g->key[i] = key[i];
    }
    CU_TRY(h, cudaEventRecord(g->ev_in, s0));
    CU_TRY(h, cudaStreamWaitEvent(g->stream, g->ev_in, 0));
    {
      ProfScope prof_solve(h, PROF_PCG_SOLVE, g->stream);
      int launched = 0, it_before = 0;
      while (true) {
        CU_TRY(h, cudaGraphLaunch(g->exec, g->stream));
        launched += chunk;
        CU_TRY(h, cudaMemcpyAsync(hst, B.st, sizeof(PcgState), cudaMemcpyDeviceToHost, g->stream));
        CU_TRY(h, host_wait(h, g->stream));
        const int ran = hst->it - it_before;  // iterations whose K1/K2 did work in this chunk
        h->launches += 2 * (int64_t)ran;
        if (h->prof) {
          for (int k = 0; k < ran && k < chunk; k += PROF_EVERY) {
            float a = 0.f, b2 = 0.f;
            if (cudaEventElapsedTime(&a, g->ev[3 * k], g->ev[3 * k + 1]) == cudaSuccess) prof_add(h, PROF_PCG_SPMV, a, 1);
            if (cudaEventElapsedTime(&b2, g->ev[3 * k + 1], g->ev[3 * k + 2]) == cudaSuccess)
              prof_add(h, PROF_PCG_UPDATE, b2, 1);
          }
          cudaGetLastError();
        }
        it_before = hst->it;
        if (hst->done || launched >= max_iters) break;
      }
    }
    // the solve's vectors were persisting L2 lines; release them so the next Newton step's
    // coarsen/assemble kernels get the whole L2 (the loop above has synchronised the solve)
    pcg_l2_release(g->stream, l2win);
    CU_TRY(h, cudaEventRecord(g->ev_out, g->stream));
    CU_TRY(h, cudaStreamWaitEvent(s0, g->ev_out, 0));
  }
  LAUNCH(h, k_copy_out, (unsigned)cdiv(3 * n, 256), 256, 0, 3 * n, B.x, x);
  stats->iters = hst->it;
  stats->status = hst->done ? hst->status : AGIPC_NOT_CONVERGED;
  stats->b_norm = sqrt(hst->bn2);
  stats->rel_residual = hst->bn2 > 0 ? sqrt(hst->rr) / sqrt(hst->bn2) : sqrt(hst->rr);
  if (stats->status == AGIPC_EINVAL) return set_err(h, AGIPC_EINVAL, "pcg_solve: upper storage has a block below the diagonal");
  if (stats->status == AGIPC_ESINGULAR) return set_err(h, AGIPC_ESINGULAR, "pcg_solve: singular diagonal block");
  if (stats->status == AGIPC_EINDEFINITE) return set_err(h, AGIPC_EINDEFINITE, "pcg_solve: p^T A p <= 0");
  if (stats->status == AGIPC_EBREAKDOWN) return set_err(h, AGIPC_EBREAKDOWN, "pcg_solve: NaN/Inf");
  if (stats->status == AGIPC_NOT_CONVERGED) return AGIPC_NOT_CONVERGED;
  return AGIPC_OK;
}

extern "C" agipc_status agipc_pcg_set_static(agipc_handle h, const agipc_bsr *A) {
  if (!h) return AGIPC_EINVAL;
  h->spat = agipc_handle_s::StaticPattern();
  if (A) {
    if (!A->row_ptr || !A->col || A->n_rows < 0 || A->nnzb < 0) return set_err(h, AGIPC_EINVAL, "pcg_set_static: bad matrix");
    h->spat.rp = A->row_ptr;
    h->spat.col = A->col;
    h->spat.n = A->n_rows;
    h->spat.nnzb = A->nnzb;
  }
  return AGIPC_OK;
}

extern "C" agipc_status agipc_pcg_solve(agipc_handle h, const agipc_bsr *A, const double *b, double *x,
                                        int zero_x0, double rel_tol, int max_iters, int check_every,
                                        agipc_pcg_stats *stats) {
  return pcg_solve_impl(h, A, AGIPC_STORAGE_FULL, b, x, zero_x0, rel_tol, max_iters, check_every, stats);
}

extern "C" agipc_status agipc_pcg_solve_sym(agipc_handle h, const agipc_bsr *A, int storage, const double *b,
                                            double *x, int zero_x0, double rel_tol, int max_iters, int check_every,
                                            agipc_pcg_stats *stats) {
  if (!h) return AGIPC_EINVAL;
  if (storage != AGIPC_STORAGE_FULL && storage != AGIPC_STORAGE_SYM && storage != AGIPC_STORAGE_UPPER)
    return set_err(h, AGIPC_EINVAL, "pcg_solve_sym: bad storage %d", storage);
  return pcg_solve_impl(h, A, storage, b, x, zero_x0, rel_tol, max_iters, check_every, stats);
}

// ------------------------------------------------------------------------------------
// Distributed PCG: the rank's rows of H_c (matrix A, columns = owned slots) and
// of its halo matrix Ah (columns n + g = ghost slot g).  The iteration is the 1-GPU one split
// at its three reductions; after every dpcg call the caller sums `red` over the ranks
// (all-reduce) and, after update, exchanges the ghost slots of z (pack -> send/recv -> the
// recv buffer of the next spmv).  The scalar logic that the last CTA runs in the 1-GPU solve
// (alpha, convergence, beta) then runs on the reduced sums in k_dscalars, identically on every
// rank, so all ranks take the same decisions and stop at the same iteration.
// ------------------------------------------------------------------------------------
enum { DP_INIT = 0, DP_ALPHA = 1, DP_UPDATE = 2, DP_NONE = 3 };

struct DPcg {
  PcgGraph *g = nullptr;  // agipc_dpcg_solve: captured iterations (NCCL calls included)
  std::vector<int64_t> gkey;
  PcgBufs B;
  int64_t n = 0, n_gs = 0;
  int k = 0;            // iterations launched (p ping-pong parity)
  int pending = DP_NONE;  // which reduced sums in red the next call must consume
  bool active = false;
};

void dpcg_free(DPcg *d) {
  if (d) pcg_graph_free(d->g);
  delete d;
}
bool dpcg_active(agipc_handle h) { return h->dpcg && h->dpcg->active; }

__global__ void k_dscalars(PcgState *st, const double *red, int phase) {
  if (phase == DP_INIT) {
    st->rz = red[0];
    st->rr = red[1];
    st->bn2 = red[2];
    st->it = 0;
    st->beta = 0.0;
    if (red[3] > 0.0) {  // some rank has a singular diagonal block: every rank stops
      st->status = AGIPC_ESINGULAR;
      st->done = 1;
    }
    if (!st->done && sqrt(red[1]) <= st->tol * sqrt(red[2])) st->done = 1;
    return;
  }
  if (st->done) return;
  if (phase == DP_ALPHA) {
    const double PQ = red[0];
    st->pq = PQ;
    if (!isfinite(PQ) || !isfinite(st->rz)) {
      st->status = AGIPC_EBREAKDOWN;
      st->done = 1;
      st->it += 1;
    } else if (PQ <= 0.0) {
      st->status = AGIPC_EINDEFINITE;
      st->done = 1;
      st->it += 1;
    } else {
      st->alpha = st->rz / PQ;
    }
  } else {  // DP_UPDATE
    const double RZ = red[0], RR = red[1];
    st->it += 1;
    st->rr = RR;
    if (sqrt(RR) <= st->tol * sqrt(st->bn2)) {
      st->done = 1;
      st->status = AGIPC_OK;
    } else if (st->it >= st->max_iters) {
      st->done = 1;
      st->status = AGIPC_NOT_CONVERGED;
    } else {
      st->beta = RZ / st->rz;
      st->rz = RZ;
    }
  }
}

// ghost slots: z from the owners; p_new = z + beta p_old (the owner's value, bit for bit)
__global__ void k_ghost_in(int64_t n, int64_t n_gs, const double *__restrict__ recv, double *__restrict__ z,
                           const double *__restrict__ pold, double *__restrict__ pnew, const PcgState *st) {
  if (*(volatile int *)&st->done) return;
  const double beta = st->beta;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 3 * n_gs; i += (int64_t)gridDim.x * blockDim.x) {
    const double zv = recv[i];
    z[3 * n + i] = zv;
    pnew[3 * n + i] = zv + beta * pold[3 * n + i];
  }
}

__global__ void k_pack3(int64_t m, const int32_t *__restrict__ idx, const double *__restrict__ src,
                        double *__restrict__ dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 3 * m) {
    const int64_t k = i / 3, c = i - 3 * k;
    dst[i] = src[3 * (int64_t)idx[k] + c];
  }
}

static agipc_status dpcg_get(agipc_handle h, DPcg **d, const char *who) {
  if (!h) return AGIPC_EINVAL;
  if (!h->dpcg || !h->dpcg->active) return set_err(h, AGIPC_EINVAL, "%s: no distributed solve in progress", who);
  *d = h->dpcg;
  return AGIPC_OK;
}

extern "C" agipc_status agipc_dpcg_setup(agipc_handle h, const agipc_bsr *A, const agipc_bsr *A_halo,
                                         int64_t n_ghost_slots, const double *b, double rel_tol, int max_iters,
                                         double *red) {
  if (!h) return AGIPC_EINVAL;
  if (!A || !red || !b || max_iters < 0 || A->n_rows <= 0 || n_ghost_slots < 0 || !(rel_tol >= 0.0))
    return set_err(h, AGIPC_EINVAL, "dpcg_setup: bad arguments");
  if (!A->row_ptr || !A->col || !A->val) return set_err(h, AGIPC_EINVAL, "dpcg_setup: null matrix");
  if (A_halo && (A_halo->n_rows != A->n_rows || !A_halo->row_ptr || (A_halo->nnzb > 0 && (!A_halo->col || !A_halo->val))))
    return set_err(h, AGIPC_EINVAL, "dpcg_setup: bad halo matrix");
  const int64_t n = A->n_rows;
  if (n + n_ghost_slots >= INT32_MAX / 4) return set_err(h, AGIPC_ERANGE, "dpcg_setup: too large");
  CU_TRY(h, cudaSetDevice(h->device));
  if (!h->dpcg) h->dpcg = new DPcg();
  DPcg *d = h->dpcg;
  agipc_status ast;
  PcgState *hst = (PcgState *)pinned_get(h, sizeof(PcgState), &ast);
  if (ast != AGIPC_OK) return ast;
  ast = pcg_setup(h, A, A_halo, n_ghost_slots, b, nullptr, 1, rel_tol, max_iters, d->B, hst, red, AGIPC_STORAGE_FULL,
                  "dpcg_");
  if (ast != AGIPC_OK) return ast;
  d->n = n;
  d->n_gs = n_ghost_slots;
  d->k = 0;
  d->pending = DP_INIT;
  d->active = true;
  return AGIPC_OK;
}

extern "C" agipc_status agipc_dpcg_pack(agipc_handle h, const int32_t *send_slots, int64_t n_send, double *sendbuf) {
  DPcg *d;
  agipc_status st = dpcg_get(h, &d, "dpcg_pack");
  if (st != AGIPC_OK) return st;
  if (n_send <= 0) return AGIPC_OK;
  if (!send_slots || !sendbuf) return set_err(h, AGIPC_EINVAL, "dpcg_pack: null pointer");
  LAUNCH(h, k_pack3, (unsigned)cdiv(3 * n_send, 256), 256, 0, n_send, send_slots, d->B.z, sendbuf);
  return AGIPC_OK;
}

extern "C" agipc_status agipc_dpcg_spmv(agipc_handle h, const double *recvbuf, double *red) {
  DPcg *d;
  agipc_status st = dpcg_get(h, &d, "dpcg_spmv");
  if (st != AGIPC_OK) return st;
  if (d->pending != DP_INIT && d->pending != DP_UPDATE) return set_err(h, AGIPC_EINVAL, "dpcg_spmv: out of order");
  if (!red || (d->n_gs > 0 && !recvbuf)) return set_err(h, AGIPC_EINVAL, "dpcg_spmv: null pointer");
  const PcgBufs &B = d->B;
  double *pold = B.P[d->k & 1], *pnew = B.P[(d->k + 1) & 1];
  ProfScope prof(h, PROF_PCG_SPMV, h->stream);
  LAUNCH(h, k_dscalars, 1, 1, 0, B.st, (const double *)red, d->pending);
  if (d->n_gs > 0)
    LAUNCH(h, k_ghost_in, (unsigned)std::min<int64_t>(cdiv(3 * d->n_gs, 256), 4 * h->sm_count), 256, 0, d->n, d->n_gs,
           recvbuf, B.z, (const double *)pold, pnew, (const PcgState *)B.st);
  LAUNCH(h, spmv_kernel(B.spmv_un), (unsigned)B.G1, PCG_THREADS, 0, B.sptr, B.scol, B.sval, B.s_vrow, B.order, B.v_row,
         B.vr_ptr, B.z, pold, pnew, B.qseg, B.counters + (d->k & 1), B.pqs, B.st, red);
  d->pending = DP_ALPHA;
  return AGIPC_OK;
}

extern "C" agipc_status agipc_dpcg_update(agipc_handle h, double *red) {
  DPcg *d;
  agipc_status st = dpcg_get(h, &d, "dpcg_update");
  if (st != AGIPC_OK) return st;
  if (d->pending != DP_ALPHA) return set_err(h, AGIPC_EINVAL, "dpcg_update: out of order");
  if (!red) return set_err(h, AGIPC_EINVAL, "dpcg_update: null pointer");
  const PcgBufs &B = d->B;
  double *pnew = B.P[(d->k + 1) & 1];
  ProfScope prof(h, PROF_PCG_UPDATE, h->stream);
  LAUNCH(h, k_dscalars, 1, 1, 0, B.st, (const double *)red, (int)DP_ALPHA);
  LAUNCH(h, (k_update<1, PCG_THREADS>), (unsigned)B.G2, PCG_THREADS, 0, d->n, B.vr_ptr, B.x, B.r, B.z, (const double *)pnew, B.qseg,
         B.Dinv, B.counters + ((d->k + 1) & 1), B.parts, B.st, red, (const double *)nullptr, (double *)nullptr);
  d->k += 1;
  d->pending = DP_UPDATE;
  return AGIPC_OK;
}

static void dpcg_fill_stats(const PcgState *hst, agipc_pcg_stats *stats) {
  stats->iters = hst->it;
  stats->status = hst->done ? hst->status : AGIPC_NOT_CONVERGED;
  stats->b_norm = sqrt(hst->bn2);
  stats->rel_residual = hst->bn2 > 0 ? sqrt(hst->rr) / sqrt(hst->bn2) : sqrt(hst->rr);
}

extern "C" agipc_status agipc_dpcg_status(agipc_handle h, int *done, agipc_pcg_stats *stats) {
  DPcg *d;
  agipc_status st = dpcg_get(h, &d, "dpcg_status");
  if (st != AGIPC_OK) return st;
  PcgState *hst = (PcgState *)pinned_get(h, sizeof(PcgState), &st);
  if (st != AGIPC_OK) return st;
  CU_TRY(h, cudaMemcpyAsync(hst, d->B.st, sizeof(PcgState), cudaMemcpyDeviceToHost, h->stream));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  if (done) *done = hst->done;
  if (stats) dpcg_fill_stats(hst, stats);
  return AGIPC_OK;
}

extern "C" agipc_status agipc_dpcg_finish(agipc_handle h, const double *red, double *x, agipc_pcg_stats *stats) {
  DPcg *d;
  agipc_status st = dpcg_get(h, &d, "dpcg_finish");
  if (st != AGIPC_OK) return st;
  if (!x || !stats) return set_err(h, AGIPC_EINVAL, "dpcg_finish: null pointer");
  if (d->pending == DP_ALPHA) return set_err(h, AGIPC_EINVAL, "dpcg_finish: out of order (after spmv)");
  if (d->pending == DP_INIT || d->pending == DP_UPDATE) {
    if (!red) return set_err(h, AGIPC_EINVAL, "dpcg_finish: null red");
    LAUNCH(h, k_dscalars, 1, 1, 0, d->B.st, red, d->pending);
  }
  d->pending = DP_NONE;
  d->active = false;
  LAUNCH(h, k_copy_out, (unsigned)cdiv(3 * d->n, 256), 256, 0, 3 * d->n, d->B.x, x);
  PcgState *hst = (PcgState *)pinned_get(h, sizeof(PcgState), &st);
  if (st != AGIPC_OK) return st;
  CU_TRY(h, cudaMemcpyAsync(hst, d->B.st, sizeof(PcgState), cudaMemcpyDeviceToHost, h->stream));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  dpcg_fill_stats(hst, stats);
  if (stats->status == AGIPC_ESINGULAR) return set_err(h, AGIPC_ESINGULAR, "dpcg: singular diagonal block");
  if (stats->status == AGIPC_EINDEFINITE) return set_err(h, AGIPC_EINDEFINITE, "dpcg: p^T A p <= 0");
  if (stats->status == AGIPC_EBREAKDOWN) return set_err(h, AGIPC_EBREAKDOWN, "dpcg: NaN/Inf");
  if (stats->status == AGIPC_NOT_CONVERGED) return AGIPC_NOT_CONVERGED;
  return AGIPC_OK;
}

// ------------------------------------------------------------------------------------
// agipc_dpcg_solve: the split-phase iteration above with the exchanges inside the library
// (SURVEY 8(e) exchange 4): per iteration
//   k_ghost_in (ghost z, p)  K1 (rank's p.q partial)  AllReduce(1)  k_dscalars(alpha)
//   K2 (rank's r.z, r.r partials)  AllReduce(2)  k_dscalars(beta, stop)  pack z  send/recv
// -- the same kernels in the same order as the split-phase calls driven by dist.py over gloo, so
// every rank takes the same decisions from the same reduced sums; check_every iterations are one
// CUDA graph with the NCCL calls captured in it.
// ------------------------------------------------------------------------------------
agipc_status comm_check(agipc_handle h, const char *who);                          // comm.cu
agipc_status comm_allreduce_f64(agipc_handle h, double *buf, int64_t n, cudaStream_t s);
agipc_status comm_sendrecv_f64(agipc_handle h, int n_peers, const int *peer_rank, const double *sendbuf,
                               const int64_t *soff, double *recvbuf, const int64_t *roff, cudaStream_t s);

struct DHalo {  // the PCG halo as the graph sees it (stable workspace pointers)
  int P = 0;
  std::vector<int> peer;
  std::vector<int64_t> soff, roff;  // element (double) offsets per peer
  int64_t n_send = 0;
  const int32_t *send_idx = nullptr;
  double *sendbuf = nullptr, *recvbuf = nullptr;
};

static agipc_status dpcg_enqueue(agipc_handle h, cudaStream_t s, int iters, DPcg *d, const DHalo &X, double *red) {
  const PcgBufs &B = d->B;
  for (int k = 0; k < iters; ++k) {
    double *pold = B.P[k & 1], *pnew = B.P[(k + 1) & 1];
    if (d->n_gs > 0)
      k_ghost_in<<<(unsigned)std::min<int64_t>(cdiv(3 * d->n_gs, 256), 4 * h->sm_count), 256, 0, s>>>(
          d->n, d->n_gs, X.recvbuf, B.z, pold, pnew, B.st);
    spmv_kernel(B.spmv_un)<<<B.G1, PCG_THREADS, 0, s>>>(B.sptr, B.scol, B.sval, B.s_vrow, B.order, B.v_row, B.vr_ptr, B.z,
                                                       pold, pnew, B.qseg, B.counters + (k & 1), B.pqs, B.st, red);
    agipc_status st = comm_allreduce_f64(h, red, 1, s);
    if (st != AGIPC_OK) return st;
    k_dscalars<<<1, 1, 0, s>>>(B.st, red, (int)DP_ALPHA);
    k_update<1, PCG_THREADS><<<B.G2, PCG_THREADS, 0, s>>>(d->n, B.vr_ptr, B.x, B.r, B.z, pnew, B.qseg, B.Dinv,
                                                           B.counters + ((k + 1) & 1), B.parts, B.st, red, nullptr,
                                                           nullptr);
    if ((st = comm_allreduce_f64(h, red, 2, s)) != AGIPC_OK) return st;
    k_dscalars<<<1, 1, 0, s>>>(B.st, red, (int)DP_UPDATE);
    if (X.n_send > 0)
      k_pack3<<<(unsigned)cdiv(3 * X.n_send, 256), 256, 0, s>>>(X.n_send, X.send_idx, B.z, X.sendbuf);
    if ((st = comm_sendrecv_f64(h, X.P, X.peer.data(), X.sendbuf, X.soff.data(), X.recvbuf, X.roff.data(), s)) !=
        AGIPC_OK)
      return st;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(h, AGIPC_ECUDA, "dpcg launch: %s", cudaGetErrorString(e));
  return AGIPC_OK;
}

extern "C" agipc_status agipc_dpcg_solve(agipc_handle h, const agipc_bsr *A, const agipc_bsr *A_halo,
                                         int64_t n_ghost_slots, const agipc_halo *slots, const double *b, double *x,
                                         double rel_tol, int max_iters, int check_every, agipc_pcg_stats *stats) {
  if (!h) return AGIPC_EINVAL;
  agipc_status ast = comm_check(h, "dpcg_solve");
  if (ast != AGIPC_OK) return ast;
  if (!A || !b || !x || !stats || max_iters < 0 || A->n_rows <= 0 || n_ghost_slots < 0 || !(rel_tol >= 0.0))
    return set_err(h, AGIPC_EINVAL, "dpcg_solve: bad arguments");
  if (dpcg_active(h)) return set_err(h, AGIPC_EINVAL, "dpcg_solve: a split-phase distributed solve is in progress");
  const int P = slots ? slots->n_peers : 0;
  if (P > 0 && (!slots->peer_rank || !slots->send_ptr || !slots->recv_ptr))
    return set_err(h, AGIPC_EINVAL, "dpcg_solve: null halo arrays");
  memset(stats, 0, sizeof(*stats));
  CU_TRY(h, cudaSetDevice(h->device));
  if (check_every <= 0) check_every = 16;
  if (!h->dpcg) h->dpcg = new DPcg();
  DPcg *d = h->dpcg;
  cudaStream_t s0 = h->stream;
  PcgState *hst = (PcgState *)pinned_get(h, sizeof(PcgState), &ast);
  if (ast != AGIPC_OK) return ast;
  // halo of the PCG vectors in stable workspace buffers (the graph keeps their addresses)
  DHalo X;
  X.P = P;
  X.soff.assign(P + 1, 0);
  X.roff.assign(P + 1, 0);
  for (int q = 0; q < P; ++q) {
    X.peer.push_back(slots->peer_rank[q]);
    X.soff[q + 1] = X.soff[q] + 3 * (slots->send_ptr[q + 1] - slots->send_ptr[q]);
    X.roff[q + 1] = X.roff[q] + 3 * (slots->recv_ptr[q + 1] - slots->recv_ptr[q]);
  }
  X.n_send = X.soff[P] / 3;
  if (X.roff[P] / 3 != n_ghost_slots) return set_err(h, AGIPC_EINVAL, "dpcg_solve: recv ranges != n_ghost_slots");
  WS(h, red, double, "dpcg_red", 4);
  WS(h, sidx, int32_t, "dpcg_send_idx", X.n_send + 1);
  WS(h, sbuf, double, "dpcg_sendbuf", 3 * X.n_send + 3);
  WS(h, rbuf, double, "dpcg_recvbuf", 3 * n_ghost_slots + 3);
  X.send_idx = sidx;
  X.sendbuf = sbuf;
  X.recvbuf = rbuf;
  if (X.n_send > 0) {
    if (!slots->send_idx) return set_err(h, AGIPC_EINVAL, "dpcg_solve: null send_idx");
    CU_TRY(h, cudaMemcpyAsync(sidx, slots->send_idx + slots->send_ptr[0], sizeof(int32_t) * X.n_send,
                              cudaMemcpyDeviceToDevice, s0));
  }
  ast = pcg_setup(h, A, A_halo, n_ghost_slots, b, nullptr, 1, rel_tol, max_iters, d->B, hst, red, AGIPC_STORAGE_FULL,
                  "dpcg_");
  if (ast != AGIPC_OK) return ast;
  d->n = A->n_rows;
  d->n_gs = n_ghost_slots;
  const PcgBufs &B = d->B;
  // setup sums [r.z, r.r, b.b, singular] over the ranks, then the first halo of z
  if ((ast = comm_allreduce_f64(h, red, 4, s0)) != AGIPC_OK) return ast;
  LAUNCH(h, k_dscalars, 1, 1, 0, B.st, (const double *)red, (int)DP_INIT);
  if (X.n_send > 0) LAUNCH(h, k_pack3, (unsigned)cdiv(3 * X.n_send, 256), 256, 0, X.n_send, (const int32_t *)sidx, B.z, sbuf);
  if ((ast = comm_sendrecv_f64(h, P, X.peer.data(), sbuf, X.soff.data(), rbuf, X.roff.data(), s0)) != AGIPC_OK)
    return ast;
  if (max_iters > 0) {
    PcgGraph *g = d->g;
    if (!g) {
      g = d->g = new PcgGraph();
      CU_TRY(h, cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
      CU_TRY(h, cudaEventCreateWithFlags(&g->ev_in, cudaEventDisableTiming));
      CU_TRY(h, cudaEventCreateWithFlags(&g->ev_out, cudaEventDisableTiming));
    }
    int chunk = std::max(2, std::min(check_every, max_iters));
    chunk += chunk & 1;
    const L2Win l2win = pcg_l2_window(h, g->stream, B.arena, B.arena_bytes);  // before capture: nodes inherit it
    std::vector<int64_t> key = {(int64_t)h->ws_gen, d->n, d->n_gs, chunk, B.G1, B.G2, B.spmv_un, P,
                                (int64_t)(intptr_t)h->comm, (int64_t)l2win.on};
    for (int q = 0; q < P; ++q) {
      key.push_back(X.peer[q]);
      key.push_back(X.soff[q + 1]);
      key.push_back(X.roff[q + 1]);
    }
    if (!g->exec || key != d->gkey) {
      if (g->exec) {
        cudaGraphExecDestroy(g->exec);
        g->exec = nullptr;
      }
      cudaGraph_t graph;
      CU_TRY(h, cudaStreamBeginCapture(g->stream, cudaStreamCaptureModeThreadLocal));
      agipc_status es = dpcg_enqueue(h, g->stream, chunk, d, X, red);
      cudaError_t ce = cudaStreamEndCapture(g->stream, &graph);
      if (es != AGIPC_OK) return es;
      if (ce != cudaSuccess) return set_err(h, AGIPC_ECUDA, "dpcg capture: %s", cudaGetErrorString(ce));
      CU_TRY(h, cudaGraphInstantiate(&g->exec, graph, 0));
      cudaGraphDestroy(graph);
      d->gkey = key;
    }
    CU_TRY(h, cudaEventRecord(g->ev_in, s0));
    CU_TRY(h, cudaStreamWaitEvent(g->stream, g->ev_in, 0));
    {
      ProfScope prof_solve(h, PROF_PCG_SOLVE, g->stream);
      int launched = 0, it_before = 0;
      while (true) {
        CU_TRY(h, cudaGraphLaunch(g->exec, g->stream));
        launched += chunk;
        CU_TRY(h, cudaMemcpyAsync(hst, B.st, sizeof(PcgState), cudaMemcpyDeviceToHost, g->stream));
        CU_TRY(h, host_wait(h, g->stream));
        const int ran = hst->it - it_before;
        h->launches += (2 + (d->n_gs > 0) + (X.n_send > 0) + 2) * (int64_t)ran;
        it_before = hst->it;
        if (hst->done || launched >= max_iters) break;  // identical on every rank
      }
    }
    pcg_l2_release(g->stream, l2win);
    CU_TRY(h, cudaEventRecord(g->ev_out, g->stream));
    CU_TRY(h, cudaStreamWaitEvent(s0, g->ev_out, 0));
  }
  LAUNCH(h, k_copy_out, (unsigned)cdiv(3 * d->n, 256), 256, 0, 3 * d->n, B.x, x);
  CU_TRY(h, cudaMemcpyAsync(hst, B.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s0));
  CU_TRY(h, cudaStreamSynchronize(s0));
  dpcg_fill_stats(hst, stats);
  if (stats->status == AGIPC_ESINGULAR) return set_err(h, AGIPC_ESINGULAR, "dpcg_solve: singular diagonal block");
  if (stats->status == AGIPC_EINDEFINITE) return set_err(h, AGIPC_EINDEFINITE, "dpcg_solve: p^T A p <= 0");
  if (stats->status == AGIPC_EBREAKDOWN) return set_err(h, AGIPC_EBREAKDOWN, "dpcg_solve: NaN/Inf");
  if (stats->status == AGIPC_NOT_CONVERGED) return AGIPC_NOT_CONVERGED;
  return AGIPC_OK;
}

// ------------------------------------------------------------------------------------
// NEXT#2: diagonal + upper storage of a full-storage BSR.  Row r keeps the blocks
// with col >= r in their order; row pointers by a scan of the per-row counts.
// ------------------------------------------------------------------------------------
__global__ void k_upper_count(int64_t n, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                              int64_t *__restrict__ ub, int32_t *__restrict__ cnt) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int64_t lo = rp[r], hi = rp[r + 1];
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (col[mid] < r) lo = mid + 1; else hi = mid;
  }
  ub[r] = lo;
  cnt[r] = (int32_t)(rp[r + 1] - lo);
}

// warp per row: columns, then the 9 values of each block as a flat coalesced copy
__global__ void k_upper_copy(int64_t n, const int64_t *__restrict__ rp, const int64_t *__restrict__ ub,
                             const int32_t *__restrict__ col, const double *__restrict__ val,
                             const int64_t *__restrict__ urp, int32_t *__restrict__ ucol, double *__restrict__ uval) {
  const int l = lane_id();
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t s0 = ub[r], d0 = urp[r], len = urp[r + 1] - d0;
    for (int64_t k = l; k < len; k += 32) ucol[d0 + k] = col[s0 + k];
    for (int64_t k = l; k < 9 * len; k += 32) uval[9 * d0 + k] = val[9 * s0 + k];
  }
}

extern "C" agipc_status agipc_bsr_upper(agipc_handle h, const agipc_bsr *A, int64_t cap_nnzb, int64_t *row_ptr,
                                        int32_t *col, double *val, int64_t *nnzb_upper) {
  if (!h) return AGIPC_EINVAL;
  if (!A || !nnzb_upper || A->n_rows < 0 || cap_nnzb < 0) return set_err(h, AGIPC_EINVAL, "bsr_upper: bad arguments");
  const int64_t n = A->n_rows;
  *nnzb_upper = 0;
  if (!row_ptr || (n > 0 && (!A->row_ptr || (A->nnzb > 0 && (!A->col || !A->val)))))
    return set_err(h, AGIPC_EINVAL, "bsr_upper: null pointer");
  CU_TRY(h, cudaSetDevice(h->device));
  cudaStream_t s = h->stream;
  if (n == 0) {
    CU_TRY(h, cudaMemsetAsync(row_ptr, 0, sizeof(int64_t), s));
    return AGIPC_OK;
  }
  WS(h, ub, int64_t, "upper_ub", n + 1);
  WS(h, cnt, int32_t, "upper_cnt", n + 1);
  LAUNCH(h, k_upper_count, (unsigned)cdiv(n, 256), 256, 0, n, A->row_ptr, A->col, ub, cnt);
  agipc_status st = scan_exclusive_i64(h, SCAN_SRC_I32, cnt, n, row_ptr);
  if (st != AGIPC_OK) return st;
  int64_t *hn = (int64_t *)pinned_get(h, sizeof(int64_t), &st);
  if (st != AGIPC_OK) return st;
  CU_TRY(h, cudaMemcpyAsync(hn, row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CU_TRY(h, cudaStreamSynchronize(s));
  *nnzb_upper = *hn;
  if (*hn > cap_nnzb || (*hn > 0 && (!col || !val)))
    return set_err(h, AGIPC_ENOSPACE, "bsr_upper: %lld blocks > capacity %lld", (long long)*hn, (long long)cap_nnzb);
  LAUNCH(h, k_upper_copy, (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 8), 16 * h->sm_count)), 256, 0, n,
         A->row_ptr, (const int64_t *)ub, A->col, A->val, (const int64_t *)row_ptr, col, val);
  return AGIPC_OK;
}

// ------------------------------------------------------------------------------------
// NEXT#2 for the fine input: full-storage values from the diagonal + upper blocks (P:1126 --
// the Hessian is produced and shipped in symmetric storage; the assembly reads full rows).
// Warp per row i: the row's col >= i part is one contiguous run in both storages (flat,
// coalesced copy); each strict-upper block U_ij is mirrored as U_ij^T into row j, found by a
// binary search over row j's col < j part.  flags[0] counts pattern mismatches, flags[1] the
// blocks written.
// ------------------------------------------------------------------------------------
__global__ void k_expand_upper(int64_t n, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                               const int64_t *__restrict__ urp, const int32_t *__restrict__ ucol,
                               const double *__restrict__ uval, double *__restrict__ val,
                               unsigned long long *flags) {
  const int l = lane_id();
  unsigned long long bad = 0, wrote = 0;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t u0 = urp[i], ulen = urp[i + 1] - u0;
    const int64_t flen = rp[i + 1] - rp[i];
    const int64_t f0 = rp[i] + flen - ulen;  // where the row's col >= i part starts in full storage
    if (ulen > flen) {
      bad += l == 0;
      continue;
    }
    for (int64_t k = l; k < 9 * ulen; k += 32) val[9 * f0 + k] = uval[9 * u0 + k];
    for (int64_t e = l; e < ulen; e += 32) {
      const int32_t j = ucol[u0 + e];
      if (col[f0 + e] != j || j < i || (e == 0) != (j == i)) {
        ++bad;
        continue;
      }
      ++wrote;
      if (j == i) continue;
      // mirror: row j, column i, in the col < j part of row j
      int64_t lo = rp[j], hi = rp[j] + (rp[j + 1] - rp[j]) - (urp[j + 1] - urp[j]);
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (col[mid] < i) lo = mid + 1; else hi = mid;
      }
      if (lo >= rp[j + 1] || col[lo] != i) {
        ++bad;
        continue;
      }
      ++wrote;
      const double *s = uval + 9 * (u0 + e);
      double *d = val + 9 * lo;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) d[3 * r + c] = s[3 * c + r];
    }
  }
  bad = warp_sum(bad);
  wrote = warp_sum(wrote);
  if (l == 0) {
    if (bad) atomicAdd(flags, bad);
    if (wrote) atomicAdd(flags + 1, wrote);
  }
}

extern "C" agipc_status agipc_bsr_expand_upper(agipc_handle h, const agipc_bsr *full, const agipc_bsr *U,
                                               double *val, int check) {
  if (!h) return AGIPC_EINVAL;
  if (!full || !U || full->n_rows != U->n_rows || full->n_rows < 0)
    return set_err(h, AGIPC_EINVAL, "bsr_expand_upper: bad arguments");
  const int64_t n = full->n_rows;
  if (n == 0) return AGIPC_OK;
  if (!full->row_ptr || !U->row_ptr || (full->nnzb > 0 && (!full->col || !val)) || (U->nnzb > 0 && (!U->col || !U->val)))
    return set_err(h, AGIPC_EINVAL, "bsr_expand_upper: null pointer");
  CU_TRY(h, cudaSetDevice(h->device));
  cudaStream_t s = h->stream;
  WS(h, flags, unsigned long long, "expand_flags", 2);
  CU_TRY(h, cudaMemsetAsync(flags, 0, 2 * sizeof(unsigned long long), s));
  LAUNCH(h, k_expand_upper, (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 8), 16 * h->sm_count)), 256, 0,
         n, full->row_ptr, full->col, U->row_ptr, U->col, U->val, val, flags);
  if (!check) return AGIPC_OK;  // stream-ordered, no host round trip (pattern validated before)
  agipc_status st;
  unsigned long long *hf = (unsigned long long *)pinned_get(h, 2 * sizeof(unsigned long long), &st);
  if (st != AGIPC_OK) return st;
  CU_TRY(h, cudaMemcpyAsync(hf, flags, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  CU_TRY(h, cudaStreamSynchronize(s));
  if (hf[0] || (int64_t)hf[1] != full->nnzb)
    return set_err(h, AGIPC_EINVAL, "bsr_expand_upper: patterns disagree (%llu mismatches, %llu of %lld blocks written)",
                   hf[0], hf[1], (long long)full->nnzb);
  return AGIPC_OK;
}
