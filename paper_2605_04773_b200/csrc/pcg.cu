// Step 4 -- coarse PCG with 3x3 block-Jacobi (PAPER.md P:752 d_c = -H_c^-1 g_c; P:879 relative
// residual tolerance; "3x3 block Jacobi"; textbook preconditioned CG, reading R20).
//
// Per iteration three kernels, all scalars on the device (no host round trip):
//   K1  q = A p (one warp per block row, the row's 9*nnz values streamed flat and coalesced)
//       fused with the partial dot p.q; the last CTA reduces the partials in a fixed order
//       (deterministic) and computes alpha = rz / pq, or flags EINDEFINITE / EBREAKDOWN;
//   K2  x += alpha p, r -= alpha q, z = D^-1 r, partial r.z and r.r; the last CTA checks
//       ||r|| <= tol ||b||, counts the iteration, computes beta;
//   K3  p = z + beta p.
// The host enqueues check_every iterations as one CUDA graph (captured once per system on an
// internal stream ordered after the caller's stream by events) and polls the done flag.
#include <cmath>
#include <vector>

#include "agipc_internal.cuh"

#define PCG_THREADS 256
#define PCG_WARPS (PCG_THREADS / 32)

struct PcgState {
  double rz, alpha, beta, bn2, rr, pq;
  int it, done, status, max_iters;
  double tol;
  unsigned int arrive;  // last-block counter
  int pad;
};

struct PcgGraph {
  cudaGraphExec_t exec = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  const void *key[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int64_t n = -1;
  int chunk = 0;
  int grid = 0;
  bool prof = false;
  std::vector<cudaEvent_t> ev;  // profiling: 4 events per iteration of the chunk
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
__device__ __forceinline__ double block_sum(double v, double *s_red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) s_red[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = l < PCG_WARPS ? s_red[l] : 0.0;
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
__device__ __forceinline__ double reduce_parts(const double *parts, int nparts, double *s_red) {
  double v = 0.0;
  for (int i = threadIdx.x; i < nparts; i += PCG_THREADS) v += __ldcg(parts + i);
  return block_sum(v, s_red);
}

// y_r = (A x)_r for the row handled by this warp (all lanes receive the 3 sums)
__device__ __forceinline__ void row_spmv(const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                                         const double *__restrict__ val, const double *__restrict__ x, int64_t r,
                                         double &y0, double &y1, double &y2) {
  const int l = lane_id();
  const int64_t k0 = rp[r], k1 = rp[r + 1];
  const int64_t ne = 9 * (k1 - k0);
  const double *v = val + 9 * k0;
  const int32_t *c = col + k0;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int64_t e = l; e < ne; e += 32) {
    const int blk = (int)(e / 9);
    const int rem = (int)(e - 9 * (int64_t)blk);
    const int ii = rem / 3, jj = rem - 3 * ii;
    const double prod = __ldcs(v + e) * __ldg(x + 3 * (int64_t)__ldg(c + blk) + jj);
    a0 += ii == 0 ? prod : 0.0;
    a1 += ii == 1 ? prod : 0.0;
    a2 += ii == 2 ? prod : 0.0;
  }
  y0 = warp_sum(a0);
  y1 = warp_sum(a1);
  y2 = warp_sum(a2);
}

__device__ __forceinline__ void dinv_apply(const double *__restrict__ D, const double r0, const double r1,
                                           const double r2, double &z0, double &z1, double &z2) {
  z0 = D[0] * r0 + D[1] * r1 + D[2] * r2;
  z1 = D[3] * r0 + D[4] * r1 + D[5] * r2;
  z2 = D[6] * r0 + D[7] * r1 + D[8] * r2;
}

// D^-1 of every row's 3x3 diagonal block (adjugate / determinant).
__global__ void k_dinv(int64_t n, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                       const double *__restrict__ val, double *__restrict__ Dinv, PcgState *st) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int64_t lo = rp[r], hi = rp[r + 1];
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (col[mid] < r) lo = mid + 1; else hi = mid;
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

// r = b - A x; z = D^-1 r; p = z; rz = r.z, rr = r.r, bb = b.b
__global__ void __launch_bounds__(PCG_THREADS) k_init(int64_t n, const int64_t *__restrict__ rp,
                                                      const int32_t *__restrict__ col, const double *__restrict__ val,
                                                      const double *__restrict__ b, double *__restrict__ x,
                                                      const double *__restrict__ Dinv, double *__restrict__ r,
                                                      double *__restrict__ z, double *__restrict__ p, double *parts,
                                                      PcgState *st, int zero_x0) {
  __shared__ double s_red[PCG_WARPS];
  const int w = threadIdx.x >> 5, l = lane_id();
  double rz = 0.0, rr = 0.0, bb = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * PCG_WARPS + w; row < n; row += (int64_t)gridDim.x * PCG_WARPS) {
    double y0 = 0.0, y1 = 0.0, y2 = 0.0;
    if (!zero_x0) row_spmv(rp, col, val, x, row, y0, y1, y2);
    if (l == 0) {
      if (zero_x0) {
        x[3 * row] = 0.0; x[3 * row + 1] = 0.0; x[3 * row + 2] = 0.0;
      }
      double b0 = b[3 * row], b1 = b[3 * row + 1], b2 = b[3 * row + 2];
      double r0 = b0 - y0, r1 = b1 - y1, r2 = b2 - y2;
      double z0, z1, z2;
      dinv_apply(Dinv + 9 * row, r0, r1, r2, z0, z1, z2);
      r[3 * row] = r0; r[3 * row + 1] = r1; r[3 * row + 2] = r2;
      z[3 * row] = z0; z[3 * row + 1] = z1; z[3 * row + 2] = z2;
      p[3 * row] = z0; p[3 * row + 1] = z1; p[3 * row + 2] = z2;
      rz += r0 * z0 + r1 * z1 + r2 * z2;
      rr += r0 * r0 + r1 * r1 + r2 * r2;
      bb += b0 * b0 + b1 * b1 + b2 * b2;
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
    if (threadIdx.x == 0) {
      st->rz = RZ;
      st->rr = RR;
      st->bn2 = BB;
      st->it = 0;
      if (!st->done && sqrt(RR) <= st->tol * sqrt(BB)) st->done = 1;
    }
  }
}

// K1: q = A p, pq partials; last CTA: alpha
__global__ void __launch_bounds__(PCG_THREADS) k_spmv_pq(int64_t n, const int64_t *__restrict__ rp,
                                                         const int32_t *__restrict__ col,
                                                         const double *__restrict__ val, const double *__restrict__ p,
                                                         double *__restrict__ q, double *parts, PcgState *st) {
  if (*(volatile int *)&st->done) return;
  __shared__ double s_red[PCG_WARPS];
  const int w = threadIdx.x >> 5, l = lane_id();
  double pq = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * PCG_WARPS + w; row < n; row += (int64_t)gridDim.x * PCG_WARPS) {
    double y0, y1, y2;
    row_spmv(rp, col, val, p, row, y0, y1, y2);
    if (l == 0) {
      q[3 * row] = y0; q[3 * row + 1] = y1; q[3 * row + 2] = y2;
      pq += p[3 * row] * y0 + p[3 * row + 1] * y1 + p[3 * row + 2] * y2;
    }
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

// K2: x += alpha p; r -= alpha q; z = D^-1 r; partial rz, rr; last CTA: convergence, beta
__global__ void __launch_bounds__(PCG_THREADS) k_update(int64_t n, double *__restrict__ x, double *__restrict__ r,
                                                        double *__restrict__ z, const double *__restrict__ p,
                                                        const double *__restrict__ q, const double *__restrict__ Dinv,
                                                        double *parts, PcgState *st) {
  if (*(volatile int *)&st->done) return;
  __shared__ double s_red[PCG_WARPS];
  const double alpha = st->alpha;
  double rz = 0.0, rr = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * PCG_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * PCG_THREADS) {
    double p0 = p[3 * i], p1 = p[3 * i + 1], p2 = p[3 * i + 2];
    double q0 = q[3 * i], q1 = q[3 * i + 1], q2 = q[3 * i + 2];
    x[3 * i] += alpha * p0; x[3 * i + 1] += alpha * p1; x[3 * i + 2] += alpha * p2;
    double r0 = r[3 * i] - alpha * q0, r1 = r[3 * i + 1] - alpha * q1, r2 = r[3 * i + 2] - alpha * q2;
    r[3 * i] = r0; r[3 * i + 1] = r1; r[3 * i + 2] = r2;
    double z0, z1, z2;
    dinv_apply(Dinv + 9 * i, r0, r1, r2, z0, z1, z2);
    z[3 * i] = z0; z[3 * i + 1] = z1; z[3 * i + 2] = z2;
    rz += r0 * z0 + r1 * z1 + r2 * z2;
    rr += r0 * r0 + r1 * r1 + r2 * r2;
  }
  const int G = gridDim.x;
  rz = block_sum(rz, s_red);
  rr = block_sum(rr, s_red);
  if (threadIdx.x == 0) {
    parts[G + blockIdx.x] = rz;
    parts[2 * G + blockIdx.x] = rr;
  }
  if (last_block(st)) {
    double RZ = reduce_parts(parts + G, G, s_red);
    double RR = reduce_parts(parts + 2 * G, G, s_red);
    if (threadIdx.x == 0) {
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

// K3: p = z + beta p
__global__ void __launch_bounds__(PCG_THREADS) k_direction(int64_t n, const double *__restrict__ z,
                                                           double *__restrict__ p, const PcgState *st) {
  if (*(volatile const int *)&st->done) return;
  const double beta = st->beta;
  for (int64_t i = (int64_t)blockIdx.x * PCG_THREADS + threadIdx.x; i < 3 * n; i += (int64_t)gridDim.x * PCG_THREADS)
    p[i] = z[i] + beta * p[i];
}

static agipc_status enqueue_iters(agipc_handle h, cudaStream_t s, int iters, int G, int64_t n, const agipc_bsr *A,
                                  double *x, double *r, double *z, double *p, double *q, const double *Dinv,
                                  double *parts, PcgState *st, cudaEvent_t *ev) {
  for (int k = 0; k < iters; ++k) {
    if (ev) cudaEventRecordWithFlags(ev[4 * k], s, cudaEventRecordExternal);
    k_spmv_pq<<<G, PCG_THREADS, 0, s>>>(n, A->row_ptr, A->col, A->val, p, q, parts, st);
    if (ev) cudaEventRecordWithFlags(ev[4 * k + 1], s, cudaEventRecordExternal);
    k_update<<<G, PCG_THREADS, 0, s>>>(n, x, r, z, p, q, Dinv, parts, st);
    if (ev) cudaEventRecordWithFlags(ev[4 * k + 2], s, cudaEventRecordExternal);
    k_direction<<<G, PCG_THREADS, 0, s>>>(n, z, p, st);
    if (ev) cudaEventRecordWithFlags(ev[4 * k + 3], s, cudaEventRecordExternal);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(h, AGIPC_ECUDA, "pcg launch: %s", cudaGetErrorString(e));
  return AGIPC_OK;
}

extern "C" agipc_status agipc_pcg_solve(agipc_handle h, const agipc_bsr *A, const double *b, double *x,
                                        int zero_x0, double rel_tol, int max_iters, int check_every,
                                        agipc_pcg_stats *stats) {
  if (!h) return AGIPC_EINVAL;
  if (!A || !stats || max_iters < 0 || A->n_rows < 0 || !(rel_tol >= 0.0))
    return set_err(h, AGIPC_EINVAL, "pcg_solve: bad arguments");
  const int64_t n = A->n_rows;
  memset(stats, 0, sizeof(*stats));
  if (n == 0) return AGIPC_OK;
  if (!A->row_ptr || !A->col || !A->val || !b || !x) return set_err(h, AGIPC_EINVAL, "pcg_solve: null pointer");
  if (n >= INT32_MAX) return set_err(h, AGIPC_ERANGE, "pcg_solve: too many rows");
  if (check_every <= 0) check_every = 16;
  CU_TRY(h, cudaSetDevice(h->device));
  ProfScope prof_setup(h, PROF_PCG_SETUP, h->stream);
  WS(h, r, double, "pcg_r", 3 * n);
  WS(h, z, double, "pcg_z", 3 * n);
  WS(h, p, double, "pcg_p", 3 * n);
  WS(h, q, double, "pcg_q", 3 * n);
  WS(h, Dinv, double, "pcg_dinv", 9 * n);
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, PCG_WARPS), 8 * (int64_t)h->sm_count));
  WS(h, parts, double, "pcg_parts", 3 * G);
  WS(h, stp, PcgState, "pcg_state", 1);
  PcgState init;
  memset(&init, 0, sizeof(init));
  init.tol = rel_tol;
  init.max_iters = max_iters;
  init.status = AGIPC_OK;
  agipc_status ast;
  PcgState *hst = (PcgState *)pinned_get(h, sizeof(PcgState), &ast);
  if (ast != AGIPC_OK) return ast;
  *hst = init;
  CU_TRY(h, cudaMemcpyAsync(stp, hst, sizeof(PcgState), cudaMemcpyHostToDevice, h->stream));
  LAUNCH(h, k_dinv, (unsigned)cdiv(n, 256), 256, 0, n, A->row_ptr, A->col, A->val, Dinv, stp);
  LAUNCH(h, k_init, (unsigned)G, PCG_THREADS, 0, n, A->row_ptr, A->col, A->val, b, x, Dinv, r, z, p, parts, stp,
         zero_x0);
  if (max_iters == 0) {
    CU_TRY(h, cudaMemcpyAsync(hst, stp, sizeof(PcgState), cudaMemcpyDeviceToHost, h->stream));
    CU_TRY(h, cudaStreamSynchronize(h->stream));
  } else {
    // chunk graph on an internal stream, ordered after the caller's stream
    PcgGraph *g = h->pcg;
    if (!g) {
      g = h->pcg = new PcgGraph();
      CU_TRY(h, cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
      CU_TRY(h, cudaEventCreateWithFlags(&g->ev_in, cudaEventDisableTiming));
      CU_TRY(h, cudaEventCreateWithFlags(&g->ev_out, cudaEventDisableTiming));
    }
    const int chunk = std::min(check_every, max_iters);
    const void *key[6] = {A->row_ptr, A->col, A->val, x, r, Dinv};
    bool same = g->exec && g->n == n && g->chunk == chunk && g->grid == G && g->prof == h->prof;
    for (int i = 0; i < 6 && same; ++i) same = g->key[i] == key[i];
    if (!same) {
      if (g->exec) {
        cudaGraphExecDestroy(g->exec);
        g->exec = nullptr;
      }
      while (h->prof && (int)g->ev.size() < 4 * chunk) {
        cudaEvent_t e;
        CU_TRY(h, cudaEventCreate(&e));
        g->ev.push_back(e);
      }
      cudaGraph_t graph;
      CU_TRY(h, cudaStreamBeginCapture(g->stream, cudaStreamCaptureModeThreadLocal));
      agipc_status es = enqueue_iters(h, g->stream, chunk, G, n, A, x, r, z, p, q, Dinv, parts, stp,
                                      h->prof ? g->ev.data() : nullptr);
      cudaError_t ce = cudaStreamEndCapture(g->stream, &graph);
      if (es != AGIPC_OK) return es;
      if (ce != cudaSuccess) return set_err(h, AGIPC_ECUDA, "pcg capture: %s", cudaGetErrorString(ce));
      CU_TRY(h, cudaGraphInstantiate(&g->exec, graph, 0));
      cudaGraphDestroy(graph);
      g->n = n;
      g->chunk = chunk;
      g->grid = G;
      g->prof = h->prof;
      for (int i = 0; i < 6; ++i) g->key[i] = key[i];
    }
    CU_TRY(h, cudaEventRecord(g->ev_in, h->stream));
    CU_TRY(h, cudaStreamWaitEvent(g->stream, g->ev_in, 0));
    ProfScope prof_solve(h, PROF_PCG_SOLVE, g->stream);
    int launched = 0;
    int it_before = 0;
    bool first = true;
    while (true) {
      CU_TRY(h, cudaGraphLaunch(g->exec, g->stream));
      launched += chunk;
      CU_TRY(h, cudaMemcpyAsync(hst, stp, sizeof(PcgState), cudaMemcpyDeviceToHost, g->stream));
      CU_TRY(h, cudaStreamSynchronize(g->stream));
      if (first) {  // iterations already counted before this solve (none: k_init sets it = 0)
        first = false;
      }
      const int ran = hst->it - it_before;  // K1/K2 launches that did work in this chunk
      h->launches += 3 * (int64_t)ran;
      if (h->prof) {
        const bool conv = hst->done && hst->status == AGIPC_OK && ran > 0;
        for (int k = 0; k < ran && k < chunk; ++k) {
          float a = 0.f, b = 0.f, c = 0.f;
          cudaError_t e1 = cudaEventElapsedTime(&a, g->ev[4 * k], g->ev[4 * k + 1]);
          if (e1 != cudaSuccess && getenv("AGIPC_DEBUG"))
            fprintf(stderr, "libagipc[debug] elapsed: %s\n", cudaGetErrorString(e1));
          cudaEventElapsedTime(&b, g->ev[4 * k + 1], g->ev[4 * k + 2]);
          prof_add(h, PROF_PCG_SPMV, a, 1);
          prof_add(h, PROF_PCG_UPDATE, b, 1);
          if (!(conv && k == ran - 1)) {  // K3 of the converged iteration exits early
            cudaEventElapsedTime(&c, g->ev[4 * k + 2], g->ev[4 * k + 3]);
            prof_add(h, PROF_PCG_DIRECTION, c, 1);
          }
        }
      }
      it_before = hst->it;
      if (hst->done || launched >= max_iters) break;
    }
    CU_TRY(h, cudaEventRecord(g->ev_out, g->stream));
    CU_TRY(h, cudaStreamWaitEvent(h->stream, g->ev_out, 0));
  }
  stats->iters = hst->it;
  stats->status = hst->done ? hst->status : AGIPC_NOT_CONVERGED;
  stats->b_norm = sqrt(hst->bn2);
  stats->rel_residual = hst->bn2 > 0 ? sqrt(hst->rr) / sqrt(hst->bn2) : sqrt(hst->rr);
  if (stats->status == AGIPC_ESINGULAR) return set_err(h, AGIPC_ESINGULAR, "pcg_solve: singular diagonal block");
  if (stats->status == AGIPC_EINDEFINITE) return set_err(h, AGIPC_EINDEFINITE, "pcg_solve: p^T A p <= 0");
  if (stats->status == AGIPC_EBREAKDOWN) return set_err(h, AGIPC_EBREAKDOWN, "pcg_solve: NaN/Inf");
  if (stats->status == AGIPC_NOT_CONVERGED) return AGIPC_NOT_CONVERGED;
  return AGIPC_OK;
}
