// Handle management, errors, workspace and the generic device-wide scan of libagipc.
#include <algorithm>

#include "agipc_internal.cuh"

agipc_status set_err(agipc_handle h, agipc_status st, const char *fmt, ...) {
  if (h) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    h->err = buf;
  }
  return st;
}

static size_t ws_pad(size_t bytes) { return ((bytes + bytes / 8 + 256) + 255) & ~(size_t)255; }

void *ws_get(agipc_handle h, const char *name, size_t bytes, agipc_status *st, bool *fresh) {
  WsBuf &b = h->ws[name];
  if (fresh) *fresh = false;
  if (b.bytes < bytes) {
    const size_t want = ws_pad(bytes);  // headroom: sizes vary between Newton steps
    size_t &mx = h->ws_max[name];
    if (want > mx) {
      h->ws_high += want - mx;
      mx = want;
    }
    if (h->arena) {  // caller-owned workspace: bump allocation, never freed until set_workspace
      if (h->arena_top + want > h->arena_cap) {
        *st = set_err(h, AGIPC_ENOSPACE,
                      "workspace '%s' needs %zu bytes: %zu of the %zu registered are in use; "
                      "register at least agipc_workspace_size() bytes",
                      name, want, h->arena_top, h->arena_cap);
        return nullptr;
      }
      b.ptr = h->arena + h->arena_top;
      b.bytes = want;
      h->arena_top += want;
    } else {
      if (b.ptr) {
        cudaStreamSynchronize(h->stream);  // the old buffer may still be in use
        cudaFree(b.ptr);
        b.ptr = nullptr;
        b.bytes = 0;
      }
      cudaError_t e = cudaMalloc(&b.ptr, want);
      if (e != cudaSuccess) {
        b.ptr = nullptr;
        *st = set_err(h, AGIPC_ECUDA, "workspace '%s' (%zu bytes): %s", name, want, cudaGetErrorString(e));
        return nullptr;
      }
      b.bytes = want;
    }
    h->ws_gen += 1;
    if (fresh) *fresh = true;
  }
  *st = AGIPC_OK;
  return b.ptr;
}

agipc_status aux_fork(agipc_handle h) {
  if (!h->aux) {
    // the aux stream carries the longer half of each fork (large-row + mid-node passes): it gets
    // the highest priority, so its CTAs take the SM slots first (AGIPC_AUX_PRIO=0: default priority)
    int lo = 0, hi = 0;
    static const bool prio = !(getenv("AGIPC_AUX_PRIO") && atoi(getenv("AGIPC_AUX_PRIO")) == 0);
    if (prio && cudaDeviceGetStreamPriorityRange(&lo, &hi) == cudaSuccess)
      CU_TRY(h, cudaStreamCreateWithPriority(&h->aux, cudaStreamNonBlocking, hi));
    else
      CU_TRY(h, cudaStreamCreateWithFlags(&h->aux, cudaStreamNonBlocking));
    CU_TRY(h, cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    CU_TRY(h, cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  }
  CU_TRY(h, cudaEventRecord(h->ev_fork, h->stream));
  CU_TRY(h, cudaStreamWaitEvent(h->aux, h->ev_fork, 0));
  return AGIPC_OK;
}

cudaError_t host_wait(agipc_handle h, cudaStream_t s) {
  if (!h->ev_wait) {
    cudaError_t e = cudaEventCreateWithFlags(&h->ev_wait, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = cudaEventRecord(h->ev_wait, s);
  if (e != cudaSuccess) return e;
  while ((e = cudaEventQuery(h->ev_wait)) == cudaErrorNotReady) {
  }
  return e;
}

agipc_status aux_join(agipc_handle h) {
  CU_TRY(h, cudaEventRecord(h->ev_join, h->aux));
  CU_TRY(h, cudaStreamWaitEvent(h->stream, h->ev_join, 0));
  return AGIPC_OK;
}

void *pinned_get(agipc_handle h, size_t bytes, agipc_status *st) {
  if (h->pinned_bytes < bytes) {
    if (h->pinned) {
      cudaStreamSynchronize(h->stream);
      cudaFreeHost(h->pinned);
    }
    size_t want = bytes < 4096 ? 4096 : bytes;
    cudaError_t e = cudaMallocHost(&h->pinned, want);
    if (e != cudaSuccess) {
      h->pinned = nullptr;
      h->pinned_bytes = 0;
      *st = set_err(h, AGIPC_ECUDA, "pinned host buffer: %s", cudaGetErrorString(e));
      return nullptr;
    }
    h->pinned_bytes = want;
  }
  *st = AGIPC_OK;
  return h->pinned;
}

void pcg_graph_free(PcgGraph *g);  // pcg.cu
void dpcg_free(struct DPcg *d);    // pcg.cu
bool dpcg_active(agipc_handle h);  // pcg.cu
void comm_free(agipc_handle h);    // comm.cu

cudaEvent_t prof_event(agipc_handle h) {
  if (!h->prof_pool.empty()) {
    cudaEvent_t e = h->prof_pool.back();
    h->prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaError_t err = cudaEventCreate(&e);
  if (err != cudaSuccess) {
    fprintf(stderr, "libagipc: cudaEventCreate: %s\n", cudaGetErrorString(err));
    cudaGetLastError();
    return nullptr;
  }
  return e;
}

void prof_push(agipc_handle h, int phase, cudaEvent_t a, cudaEvent_t b) {
  h->prof_pending.push_back(ProfPending{phase, a, b});
}

void prof_add(agipc_handle h, int phase, double ms, int64_t n) {
  h->prof_ms[phase] += ms;
  h->prof_n[phase] += n;
}

static void prof_flush(agipc_handle h) {
  for (auto &p : h->prof_pending) {
    cudaEventSynchronize(p.b);
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) prof_add(h, p.phase, ms, 1);
    h->prof_pool.push_back(p.a);
    h->prof_pool.push_back(p.b);
  }
  h->prof_pending.clear();
}

// ---- launch trace (AGIPC_TRACE=<file>) ----
#include <chrono>
static double host_now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
void trace_pre(agipc_handle h, const char *name, cudaStream_t s) {
  if (h->trace_recs.size() >= 200000) return;
  agipc_handle_s::TraceRec r{name, s, nullptr, nullptr, host_now_us()};
  r.a = prof_event(h);
  if (r.a) cudaEventRecord(r.a, s);
  h->trace_recs.push_back(r);
}
void trace_mark(agipc_handle h, const char *name) {
  if (h->trace_recs.size() >= 200000) return;
  h->trace_recs.push_back(agipc_handle_s::TraceRec{name, nullptr, nullptr, nullptr, host_now_us()});
}
void trace_post(agipc_handle h, cudaStream_t s) {
  if (h->trace_recs.empty() || h->trace_recs.back().b || h->trace_recs.back().s != s) return;
  auto &r = h->trace_recs.back();
  r.b = prof_event(h);
  if (r.b) cudaEventRecord(r.b, s);
}
static void trace_dump(agipc_handle h) {
  const char *path = getenv("AGIPC_TRACE");
  if (!path || h->trace_recs.empty()) return;
  cudaDeviceSynchronize();
  FILE *f = fopen(path, "a");
  if (!f) return;
  const auto &r0 = h->trace_recs.front();
  fprintf(f, "# name stream gpu_start_us gpu_end_us host_submit_us\n");
  for (auto &r : h->trace_recs) {
    float t0 = -1.f, t1 = -1.f;
    if (r0.a && r.a) cudaEventElapsedTime(&t0, r0.a, r.a);
    if (r0.a && r.b) cudaEventElapsedTime(&t1, r0.a, r.b);
    fprintf(f, "%s %p %.2f %.2f %.2f\n", r.name, (void *)r.s, 1e3 * t0, 1e3 * t1, r.host_us - r0.host_us);
  }
  fclose(f);
  cudaGetLastError();
}

static const char *kPhaseNames[PROF_N] = {"tag_edges", "build_map", "assemble_coarse", "pcg_setup",
                                          "pcg_spmv", "pcg_update", "pcg_solve",
                                          "asm_classify", "asm_symbolic", "asm_numeric",
                                          "prolongate", "dist_halo", "triplets", "map_level0", "map_tail"};

extern "C" {

agipc_status agipc_create(agipc_handle *out, int cuda_device) {
  if (!out) return AGIPC_EINVAL;
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return AGIPC_ECUDA;
  if (cuda_device < 0 || cuda_device >= n) return AGIPC_EINVAL;
  e = cudaSetDevice(cuda_device);
  if (e != cudaSuccess) return AGIPC_ECUDA;
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, cuda_device);
  if (e != cudaSuccess) return AGIPC_ECUDA;
  if (prop.major != 10) return AGIPC_ECUDA;  // built for sm_100a only
  agipc_handle h = new agipc_handle_s();
  h->device = cuda_device;
  h->sm_count = prop.multiProcessorCount;
  h->trace = getenv("AGIPC_TRACE") != nullptr;
  *out = h;
  return AGIPC_OK;
}

agipc_status agipc_destroy(agipc_handle h) {
  if (!h) return AGIPC_EINVAL;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  if (!h->arena)
    for (auto &kv : h->ws)
      if (kv.second.ptr) cudaFree(kv.second.ptr);
  comm_free(h);
  if (h->pinned) cudaFreeHost(h->pinned);
  if (h->pcg) pcg_graph_free(h->pcg);
  if (h->pcg_static) pcg_graph_free(h->pcg_static);
  if (h->aux) {
    cudaStreamSynchronize(h->aux);
    cudaStreamDestroy(h->aux);
    cudaEventDestroy(h->ev_fork);
    cudaEventDestroy(h->ev_join);
  }
  if (h->dpcg) dpcg_free(h->dpcg);
  if (h->ev_wait) cudaEventDestroy(h->ev_wait);
  trace_dump(h);
  prof_flush(h);
  for (auto e : h->prof_pool) cudaEventDestroy(e);
  delete h;
  return AGIPC_OK;
}

agipc_status agipc_set_stream(agipc_handle h, void *stream) {
  if (!h) return AGIPC_EINVAL;
  h->stream = (cudaStream_t)stream;
  return AGIPC_OK;
}

agipc_status agipc_set_values_event(agipc_handle h, void *event) {
  if (!h) return AGIPC_EINVAL;
  h->values_event = (cudaEvent_t)event;
  return AGIPC_OK;
}

agipc_status agipc_set_option(agipc_handle h, int option, int64_t value) {
  if (!h) return AGIPC_EINVAL;
  switch (option) {
    case AGIPC_OPT_CHECK_SYMMETRY:
      h->opt_check_sym = value != 0;
      return AGIPC_OK;
    case AGIPC_OPT_COMM_ALWAYS:
      h->opt_comm_always = value != 0;
      return AGIPC_OK;
    case AGIPC_OPT_DETERMINISTIC:
      h->opt_deterministic = value != 0;
      return AGIPC_OK;
    case AGIPC_OPT_L2_PERSIST: {
      if (value < 0) return set_err(h, AGIPC_EINVAL, "set_option: negative L2 size");
      CU_TRY(h, cudaSetDevice(h->device));
      int max_persist = 0;
      CU_TRY(h, cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, h->device));
      h->opt_l2_persist = std::min((size_t)value, (size_t)std::max(0, max_persist));
      return AGIPC_OK;
    }
  }
  return set_err(h, AGIPC_EINVAL, "set_option: unknown option %d", option);
}

agipc_status agipc_workspace_size(agipc_handle h, int64_t n_nodes, int64_t n_tets, int64_t nnz_adj, int64_t nnzb_fine,
                                  size_t *bytes) {
  if (!h || !bytes) return AGIPC_EINVAL;
  if (n_nodes < 0 || n_tets < 0 || nnz_adj < 0 || nnzb_fine < 0)
    return set_err(h, AGIPC_EINVAL, "workspace_size: negative size");
  // a priori estimate of one Newton step (tag, map, assemble, coarse PCG):
  // per-node, per-adjacency-slot and per-fine-block bytes of the named buffers, the coarse system
  // taken as large as the fine one (the ENOSPACE retry covers the rare larger case)
  const double est = 1.25 * (160.0 * n_nodes + 12.0 * nnz_adj + 8.0 * n_tets + 220.0 * nnzb_fine) + (1 << 22);
  *bytes = std::max(h->ws_high, (size_t)est);
  return AGIPC_OK;
}

agipc_status agipc_set_workspace(agipc_handle h, void *ws, size_t bytes) {
  if (!h) return AGIPC_EINVAL;
  if (ws && ((uintptr_t)ws & 255)) return set_err(h, AGIPC_EINVAL, "set_workspace: base must be 256-byte aligned");
  if (dpcg_active(h)) return set_err(h, AGIPC_EINVAL, "set_workspace: a distributed solve is in progress");
  CU_TRY(h, cudaSetDevice(h->device));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  if (!h->arena)
    for (auto &kv : h->ws)
      if (kv.second.ptr) cudaFree(kv.second.ptr);
  h->ws.clear();  // every named buffer is re-placed (fresh) on its next use
  h->arena = (char *)ws;
  h->arena_cap = ws ? bytes : 0;
  h->arena_top = 0;
  h->ws_gen += 1;
  return AGIPC_OK;
}

const char *agipc_last_error(agipc_handle h) { return h ? h->err.c_str() : "null handle"; }

const char *agipc_status_string(agipc_status s) {
  switch (s) {
    case AGIPC_OK: return "AGIPC_OK";
    case AGIPC_EINVAL: return "AGIPC_EINVAL";
    case AGIPC_ERANGE: return "AGIPC_ERANGE";
    case AGIPC_ENOSPACE: return "AGIPC_ENOSPACE";
    case AGIPC_ECUDA: return "AGIPC_ECUDA";
    case AGIPC_ENCCL: return "AGIPC_ENCCL";
    case AGIPC_EDEGENERATE: return "AGIPC_EDEGENERATE";
    case AGIPC_ESINGULAR: return "AGIPC_ESINGULAR";
    case AGIPC_EINDEFINITE: return "AGIPC_EINDEFINITE";
    case AGIPC_EBREAKDOWN: return "AGIPC_EBREAKDOWN";
    case AGIPC_NOT_CONVERGED: return "AGIPC_NOT_CONVERGED";
  }
  return "unknown agipc_status";
}

void agipc_version(int *major, int *minor) {
  if (major) *major = AGIPC_VERSION_MAJOR;
  if (minor) *minor = AGIPC_VERSION_MINOR;
}

int64_t agipc_kernel_launches(agipc_handle h) { return h ? h->launches : -1; }

agipc_status agipc_profile(agipc_handle h, int enable) {
  if (!h) return AGIPC_EINVAL;
  prof_flush(h);
  for (int i = 0; i < PROF_N; ++i) {
    h->prof_ms[i] = 0.0;
    h->prof_n[i] = 0;
  }
  h->prof = enable != 0;
  return AGIPC_OK;
}

int agipc_profile_read(agipc_handle h, agipc_profile_entry *out, int cap) {
  if (!h) return -1;
  prof_flush(h);
  int n = 0;
  for (int i = 0; i < PROF_N && n < cap; ++i) {
    if (!out) break;
    snprintf(out[n].name, sizeof(out[n].name), "%s", kPhaseNames[i]);
    out[n].count = h->prof_n[i];
    out[n].total_ms = h->prof_ms[i];
    ++n;
  }
  return out ? n : PROF_N;
}

}  // extern "C"

// ------------------------------------------------------------------------------------
// Generic single-pass exclusive scan (decoupled look-back), 2048 items per CTA tile.
// ------------------------------------------------------------------------------------
#define SCAN_THREADS 256
#ifndef SCAN_ITEMS
#define SCAN_ITEMS 4  // 1024-item tiles (8: 2048 and 16: 4096 measured slower, profiles/r02v)
#endif
#define SCAN_TILE (SCAN_THREADS * SCAN_ITEMS)

// Several independent scans in ONE launch (scan_multi): tiles are claimed from one counter in
// job order, so every predecessor tile of a job belongs to a resident CTA; each job has its own
// look-back status region.  The item value is a functor of the job's kind (SCAN_SRC_*).
__device__ __forceinline__ long long scan_item(const ScanJob &J, int64_t i, long long n3, long long nslots) {
  switch (J.kind) {
    case SCAN_SRC_I32: return (long long)(J.mul * (int64_t)((const int32_t *)J.src)[i] + J.add);
    case SCAN_SRC_I64: return (long long)(J.mul * ((const int64_t *)J.src)[i] + J.add);
    case SCAN_SRC_GT: return ((const int32_t *)J.src)[i] > J.add ? 1 : 0;
    case SCAN_SRC_POW2: {
      const int x = ((const int32_t *)J.src)[i];
      return x > 0 ? (1ll << (32 - __clz(x - 1))) : 0;  // next power of two (1 -> 1)
    }
    default: {  // SCAN_SRC_SLOTRL: row length of slot i (a 12-DoF node's 4 slots share its row)
      if (i >= nslots) return 0;
      const long long c = i < n3 ? i : n3 + (i - n3) / 4;
      return ((const int32_t *)J.src)[c];
    }
  }
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_multi(ScanJobs Jobs, unsigned long long *status, int *counter) {
  __shared__ int s_tile;
  __shared__ long long s_warp[SCAN_THREADS / 32];
  __shared__ long long s_prefix;
  __shared__ long long s_items[SCAN_TILE];
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1);
  __syncthreads();
  int jb = 0;
  while (jb + 1 < Jobs.njobs && s_tile >= Jobs.j[jb + 1].tile0) ++jb;
  const ScanJob &J = Jobs.j[jb];
  const int tile = s_tile - J.tile0;
  long long n3 = 0, nslots = 0;
  if (J.kind == SCAN_SRC_SLOTRL) {
    n3 = *J.dev_n3;
    nslots = *J.dev_nslots;
  }
  const int64_t n = J.n;
  const int64_t base = (int64_t)tile * SCAN_TILE;
  for (int k = threadIdx.x; k < SCAN_TILE; k += SCAN_THREADS) {  // striped coalesced load
    int64_t i = base + k;
    s_items[k] = i < n ? scan_item(J, i, n3, nslots) : 0;
  }
  __syncthreads();
  long long v[SCAN_ITEMS];
  long long tsum = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    v[k] = s_items[threadIdx.x * SCAN_ITEMS + k];
    tsum += v[k];
  }
  long long incl = warp_incl_scan(tsum);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 31) s_warp[w] = incl;
  __syncthreads();
  if (w == 0) {
    long long ws = l < SCAN_THREADS / 32 ? s_warp[l] : 0;
    long long wi = warp_incl_scan(ws);
    long long agg = __shfl_sync(FULL_MASK, wi, SCAN_THREADS / 32 - 1);
    if (l < SCAN_THREADS / 32) s_warp[l] = wi - ws;  // exclusive warp offsets
    long long pfx = lb_exclusive(status + J.tile0, tile, agg);
    if (l == 0) s_prefix = pfx;
  }
  __syncthreads();
  long long run = s_prefix + s_warp[w] + incl - tsum;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    s_items[threadIdx.x * SCAN_ITEMS + k] = run;
    run += v[k];
  }
  __syncthreads();
  int64_t *out = J.out;
  for (int k = threadIdx.x; k < SCAN_TILE; k += SCAN_THREADS) {
    int64_t i = base + k;
    if (i <= n) out[i] = s_items[k];  // out[n] (the total) is the exclusive value at n
  }
}

agipc_status scan_multi(agipc_handle h, ScanJobs jobs) {
  if (jobs.njobs < 1 || jobs.njobs > SCAN_MAX_JOBS) return set_err(h, AGIPC_EINVAL, "scan_multi: bad job count");
  int64_t tiles = 0;
  for (int k = 0; k < jobs.njobs; ++k) {
    if (jobs.j[k].n < 0) return set_err(h, AGIPC_EINVAL, "scan of negative size");
    // one extra item so that out[n] (the total) is produced by the tile containing index n
    const int64_t t = cdiv(jobs.j[k].n + 1, SCAN_TILE);
    if (tiles + t >= INT32_MAX) return set_err(h, AGIPC_ERANGE, "scan too large");
    jobs.j[k].tile0 = (int)tiles;
    tiles += t;
  }
  WS(h, status, unsigned long long, "scan_status", tiles + 1);
  CU_TRY(h, cudaMemsetAsync(status, 0, sizeof(unsigned long long) * (tiles + 1), h->stream));
  int *counter = (int *)(status + tiles);
  LAUNCH(h, k_scan_multi, (unsigned)tiles, SCAN_THREADS, 0, jobs, status, counter);
  return AGIPC_OK;
}

ScanJob scan_job(int kind, const void *src, int64_t n, int64_t *out, int64_t mul, int64_t add) {
  ScanJob J;
  memset(&J, 0, sizeof(J));
  J.kind = kind;
  J.src = src;
  J.n = n;
  J.out = out;
  J.mul = mul;
  J.add = add;
  return J;
}

agipc_status scan_exclusive_i64(agipc_handle h, int kind, const void *src, int64_t n, int64_t *out,
                                int64_t mul, int64_t add) {
  ScanJobs jobs;
  memset(&jobs, 0, sizeof(jobs));
  jobs.njobs = 1;
  jobs.j[0] = scan_job(kind, src, n, out, mul, add);
  return scan_multi(h, jobs);
}
