// Internal definitions of libagipc (B200 / sm_100a).  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <unordered_map>
#include <vector>

#include "agipc.h"

#define AGIPC_WARP 32
#define FULL_MASK 0xffffffffu

// ------------------------------------------------------------------------------------
// Handle: device, stream, error text, grow-only workspace, pinned host scratch.
// ------------------------------------------------------------------------------------
struct WsBuf {
  void *ptr = nullptr;
  size_t bytes = 0;
};

struct PcgGraph;  // pcg.cu

// Profiling phases (agipc_profile_read names them)
enum ProfPhase {
  PROF_TAG = 0,
  PROF_MAP,
  PROF_ASSEMBLE,
  PROF_PCG_SETUP,
  PROF_PCG_SPMV,
  PROF_PCG_UPDATE,
  PROF_PCG_SOLVE,
  PROF_ASM_CLASSIFY,
  PROF_ASM_SYMBOLIC,
  PROF_ASM_NUMERIC,
  PROF_PROLONG,
  PROF_DIST,
  PROF_TRIPLETS,
  PROF_MAP_LEVEL0,
  PROF_MAP_TAIL,
  PROF_N
};

struct ProfPending {
  int phase;
  cudaEvent_t a, b;
};

struct agipc_handle_s {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches = 0;
  std::unordered_map<std::string, WsBuf> ws;
  // caller-owned workspace (agipc_set_workspace): named buffers are carved from [arena,
  // arena + arena_cap) by a bump pointer; nullptr = the library cudaMallocs them itself
  char *arena = nullptr;
  size_t arena_cap = 0, arena_top = 0;
  uint64_t ws_gen = 0;  // bumped whenever a named buffer moves (captured PCG graphs key on it)
  std::unordered_map<std::string, size_t> ws_max;  // largest (padded) size ever requested per name
  size_t ws_high = 0;                               // sum of ws_max: agipc_workspace_size
  // agipc_set_option
  int opt_check_sym = 0;     // AGIPC_OPT_CHECK_SYMMETRY
  size_t opt_l2_persist = 0;  // AGIPC_OPT_L2_PERSIST (bytes; 0 = no persisting window)
  int opt_comm_always = 0;    // AGIPC_OPT_COMM_ALWAYS
  int opt_deterministic = 0;  // AGIPC_OPT_DETERMINISTIC
  void *pinned = nullptr;  // small pinned host buffer for D2H of scalars
  size_t pinned_bytes = 0;
  PcgGraph *pcg = nullptr;
  PcgGraph *pcg_static = nullptr;  // graph of solves on the registered static pattern
  struct StaticPattern {           // agipc_pcg_set_static: SELL layout kept across solves
    const void *rp = nullptr, *col = nullptr;
    int64_t n = -1, nnzb = -1;
    bool built = false;
    long long nv = 0, ns = 0, sell_blocks = 0;
    const void *bufs[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  } spat;
  size_t tail_smem = 0;
  cudaEvent_t values_event = nullptr;  // agipc_set_values_event (one-shot, consumed by assemble)
  struct DPcg *dpcg = nullptr;  // distributed PCG in progress (pcg.cu)
  struct Comm *comm = nullptr;  // NCCL communicator (comm.cu, agipc_comm_init)
  cudaStream_t aux = nullptr;   // second stream for independent kernels of one call (fork / join)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_wait = nullptr;  // host_wait
  // profiling (CUDA events on the launching stream; off by default)
  bool prof = false;
  std::vector<ProfPending> prof_pending;
  std::vector<cudaEvent_t> prof_pool;
  double prof_ms[PROF_N] = {0};
  int64_t prof_n[PROF_N] = {0};
  // launch trace (env AGIPC_TRACE=<file>, diagnostics only): an event before and after every
  // LAUNCH on its stream plus the host submit time; written at agipc_destroy
  bool trace = false;
  struct TraceRec {
    const char *name;
    cudaStream_t s;
    cudaEvent_t a, b;
    double host_us;
  };
  std::vector<TraceRec> trace_recs;
};

cudaEvent_t prof_event(agipc_handle h);             // from the pool
void prof_push(agipc_handle h, int phase, cudaEvent_t a, cudaEvent_t b);
void prof_add(agipc_handle h, int phase, double ms, int64_t n);

// Records a start event on construction and an end event on destruction (if profiling).
struct ProfScope {
  agipc_handle h;
  int phase;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  ProfScope(agipc_handle h_, int phase_, cudaStream_t s_) : h(h_), phase(phase_), s(s_) {
    static const bool debug = getenv("AGIPC_DEBUG") != nullptr;
    if (debug) {
      cudaError_t e0 = cudaGetLastError();
      fprintf(stderr, "libagipc[debug] enter phase %d: pending=%s\n", phase, cudaGetErrorString(e0));
    }
    if (h->prof) {
      a = prof_event(h);
      cudaError_t e = a ? cudaEventRecord(a, s) : cudaErrorInvalidValue;
      if (e != cudaSuccess) {
        fprintf(stderr, "libagipc: profiling disabled, cudaEventRecord: %s\n", cudaGetErrorString(e));
        cudaGetLastError();
        h->prof = false;
        a = nullptr;
      }
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = prof_event(h);
      if (b && cudaEventRecord(b, s) == cudaSuccess) prof_push(h, phase, a, b);
      else cudaGetLastError();
    }
  }
};

agipc_status set_err(agipc_handle h, agipc_status st, const char *fmt, ...);

// Grow-only named device workspace (cudaMalloc only when a buffer must grow, or carved from the
// caller's arena).  *fresh (nullable) = the buffer was (re)placed, its content is undefined.
void *ws_get(agipc_handle h, const char *name, size_t bytes, agipc_status *st, bool *fresh = nullptr);
// Pinned host scratch of at least `bytes`.
void *pinned_get(agipc_handle h, size_t bytes, agipc_status *st);

#define CU_TRY(h, call)                                                                      \
  do {                                                                                       \
    cudaError_t _e = (call);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      return set_err((h), AGIPC_ECUDA, "%s failed at %s:%d: %s", #call, __FILE__, __LINE__,  \
                     cudaGetErrorString(_e));                                                \
  } while (0)

void trace_pre(agipc_handle h, const char *name, cudaStream_t s);
void trace_post(agipc_handle h, cudaStream_t s);
void trace_mark(agipc_handle h, const char *name);  // host-time marker (no GPU events)

// Every kernel launch goes through LAUNCH so that the handle counts it and errors surface.
// (one cudaGetLastError after the launch: it also reports an error left pending by an earlier
// asynchronous call; the host-side cost per launch is on the critical path after every sync)
#define LAUNCH(h, kernel, grid, block, smem, ...)                                            \
  do {                                                                                       \
    if ((grid) > 0) {                                                                        \
      if ((h)->trace) trace_pre((h), #kernel, (h)->stream);                                 \
      kernel<<<(grid), (block), (smem), (h)->stream>>>(__VA_ARGS__);                         \
      if ((h)->trace) trace_post((h), (h)->stream);                                         \
      (h)->launches += 1;                                                                    \
      cudaError_t _e = cudaGetLastError();                                                   \
      if (_e != cudaSuccess)                                                                 \
        return set_err((h), AGIPC_ECUDA, "launch %s failed: %s", #kernel,                    \
                       cudaGetErrorString(_e));                                              \
    }                                                                                        \
  } while (0)

// LAUNCH on an explicit stream (the handle's aux stream of a fork / join region)
#define LAUNCH_S(h, strm, kernel, grid, block, smem, ...)                                     \
  do {                                                                                       \
    if ((grid) > 0) {                                                                        \
      if ((h)->trace) trace_pre((h), #kernel, (strm));                                      \
      kernel<<<(grid), (block), (smem), (strm)>>>(__VA_ARGS__);                              \
      if ((h)->trace) trace_post((h), (strm));                                              \
      (h)->launches += 1;                                                                    \
      cudaError_t _e = cudaGetLastError();                                                   \
      if (_e != cudaSuccess)                                                                 \
        return set_err((h), AGIPC_ECUDA, "launch %s failed: %s", #kernel,                    \
                       cudaGetErrorString(_e));                                              \
    }                                                                                        \
  } while (0)

// Host wait for everything enqueued on s so far by spinning on an event (cudaEventQuery) instead
// of cudaStreamSynchronize: the calls that must return device-computed sizes pay no blocking-sync
// wake-up latency (the GPU idles until the host enqueues the next work).
cudaError_t host_wait(agipc_handle h, cudaStream_t s);

// Fork: work enqueued on h->aux after this starts once everything before on h->stream is done.
agipc_status aux_fork(agipc_handle h);
// Join: h->stream waits for everything enqueued on h->aux so far.
agipc_status aux_join(agipc_handle h);

#define WS(h, var, type, name, count)                                                        \
  type *var = nullptr;                                                                       \
  do {                                                                                       \
    agipc_status _st = AGIPC_OK;                                                             \
    var = (type *)ws_get((h), (name), sizeof(type) * (size_t)((count) > 0 ? (count) : 1), &_st); \
    if (_st != AGIPC_OK) return _st;                                                         \
  } while (0)

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ------------------------------------------------------------------------------------
// Device helpers
// ------------------------------------------------------------------------------------
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  return v;
}

// Inclusive warp scan (Kogge-Stone with shuffles).
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int l = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(FULL_MASK, v, o);
    if (l >= o) v += t;
  }
  return v;
}

// ---- single-pass decoupled look-back (chained scan) --------------------------------
// Status word per tile: bits 63..62 = flag (0 empty, 1 aggregate, 2 inclusive prefix),
// bits 61..0 = value (non-negative).  Tiles are claimed in order from a counter so that
// every predecessor tile belongs to a CTA that is already resident (forward progress).
#define LB_AGG 1ull
#define LB_PFX 2ull
__device__ __forceinline__ void lb_publish(unsigned long long *status, int tile, unsigned long long flag,
                                           long long value) {
  unsigned long long w = (flag << 62) | (unsigned long long)value;
  __threadfence();
  atomicExch(status + tile, w);
}

__device__ __forceinline__ unsigned long long lb_read(const unsigned long long *status, int idx) {
  return *((volatile const unsigned long long *)(status + idx));
}

// Called by ALL 32 lanes of one warp.  Returns the exclusive prefix of `tile`
// (to every lane) and publishes the inclusive prefix.
__device__ __forceinline__ long long lb_exclusive(unsigned long long *status, int tile, long long aggregate) {
  const int l = lane_id();
  if (tile == 0) {
    if (l == 0) lb_publish(status, 0, LB_PFX, aggregate);
    return 0;
  }
  if (l == 0) lb_publish(status, tile, LB_AGG, aggregate);
  long long excl = 0;
  int pred = tile - 1;
  while (true) {
    int idx = pred - l;
    unsigned long long s = idx >= 0 ? lb_read(status, idx) : (LB_PFX << 62);
    unsigned long long flag = s >> 62;
    if (__any_sync(FULL_MASK, flag == 0)) continue;  // a predecessor has not published yet
    unsigned pmask = __ballot_sync(FULL_MASK, flag == LB_PFX);
    long long v = (long long)(s & ((1ull << 62) - 1));
    int stop = pmask ? __ffs(pmask) - 1 : 31;
    long long part = (l <= stop) ? v : 0;
    excl += warp_sum(part);
    if (pmask) break;
    pred -= 32;
  }
  if (l == 0) lb_publish(status, tile, LB_PFX, excl + aggregate);
  return excl;
}

// Device-wide exclusive scan of int64 values given by a functor: out[i] = sum_{k<i} f(k),
// out[n] = total (out must hold n+1 entries).  Workspace: status[n_tiles] zeroed + counter.
agipc_status scan_exclusive_i64(agipc_handle h, int kind, const void *src, int64_t n, int64_t *out,
                                int64_t mul = 1, int64_t add = 0);
// kinds of source for scan_exclusive_i64: value(i) = mul * src[i] + add  (int32 or int64 source)
#define SCAN_SRC_I32 0
#define SCAN_SRC_I64 1
#define SCAN_SRC_GT 2      // int32 src[i] > add ? 1 : 0
#define SCAN_SRC_POW2 3    // int32 src[i] > 0 ? next power of two : 0
#define SCAN_SRC_SLOTRL 4  // slot i < *dev_nslots: int32 src[node of slot i] (12-DoF nodes: 4 slots)
#define SCAN_MAX_JOBS 4
struct ScanJob {
  const void *src;
  const long long *dev_n3, *dev_nslots;  // SCAN_SRC_SLOTRL
  int64_t n, mul, add;
  int64_t *out;
  int kind;
  int tile0;  // set by scan_multi
};
struct ScanJobs {
  ScanJob j[SCAN_MAX_JOBS];
  int njobs;
};
ScanJob scan_job(int kind, const void *src, int64_t n, int64_t *out, int64_t mul = 1, int64_t add = 0);
// up to SCAN_MAX_JOBS independent exclusive scans in one launch (out[k][n_k] = total)
agipc_status scan_multi(agipc_handle h, ScanJobs jobs);
