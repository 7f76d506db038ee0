// Library-owned communicator of the partitioned multi-GPU path (north star: "Ranks exchange PCG
// halo vectors over NVLink via NCCL send/recv, allreduce PCG dot products, and use an all-gather
// exclusive scan of per-rank super-node counts"; SURVEY 8(b) agipc_comm_init, 8(e) exchanges 1-4).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2 -- the copy torch has already loaded when
// there is one -- or $AGIPC_NCCL_LIB), so libagipc loads and every 1-GPU entry point works
// without it.  One communicator per handle, on the handle's device; every collective is enqueued
// on the caller's stream (or on the PCG graph's stream during capture: NCCL calls are captured
// into the distributed PCG graph, pcg.cu).  The caller only moves the 128-byte unique id between
// processes (e.g. a torch.distributed broadcast of bytes).
#include <dlfcn.h>
#include <nccl.h>

#include "agipc_internal.cuh"

struct NcclApi {
  void *so = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int *) = nullptr;
};

static NcclApi g_nccl;
static std::string g_nccl_err;

static bool nccl_load() {
  if (g_nccl.so) return true;
  const char *env = getenv("AGIPC_NCCL_LIB");
  const char *names[] = {env, "libnccl.so.2", "libnccl.so"};
  void *so = nullptr;
  for (const char *n : names)
    if (n && (so = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!so) {
    g_nccl_err = std::string("dlopen libnccl.so.2 failed: ") + (dlerror() ? dlerror() : "?");
    return false;
  }
#define NCCL_SYM(field, name)                                          \
  *(void **)&g_nccl.field = dlsym(so, name);                           \
  if (!g_nccl.field) {                                                 \
    g_nccl_err = std::string("libnccl has no symbol ") + name;         \
    dlclose(so);                                                       \
    return false;                                                      \
  }
  NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
  NCCL_SYM(CommInitRank, "ncclCommInitRank");
  NCCL_SYM(CommDestroy, "ncclCommDestroy");
  NCCL_SYM(CommAbort, "ncclCommAbort");
  NCCL_SYM(AllReduce, "ncclAllReduce");
  NCCL_SYM(AllGather, "ncclAllGather");
  NCCL_SYM(Send, "ncclSend");
  NCCL_SYM(Recv, "ncclRecv");
  NCCL_SYM(GroupStart, "ncclGroupStart");
  NCCL_SYM(GroupEnd, "ncclGroupEnd");
  NCCL_SYM(GetErrorString, "ncclGetErrorString");
  NCCL_SYM(GetVersion, "ncclGetVersion");
#undef NCCL_SYM
  g_nccl.so = so;
  return true;
}

struct Comm {
  ncclComm_t nc = nullptr;
  int nranks = 1, rank = 0;
};

// Handles are destroyed after their stream has been synchronised; ncclCommAbort (not Destroy)
// so that tearing down a handle -- e.g. at interpreter exit -- never waits on a peer.
void comm_free(agipc_handle h) {
  if (h && h->comm) {
    if (h->comm->nc) g_nccl.CommAbort(h->comm->nc);
    delete h->comm;
    h->comm = nullptr;
  }
}

#define NCCL_TRY(h, call)                                                                            \
  do {                                                                                               \
    ncclResult_t _r = (call);                                                                        \
    if (_r != ncclSuccess)                                                                           \
      return set_err((h), AGIPC_ENCCL, "%s failed: %s", #call, g_nccl.GetErrorString(_r));          \
  } while (0)

int comm_size(agipc_handle h) { return h->comm ? h->comm->nranks : 0; }
int comm_rank(agipc_handle h) { return h->comm ? h->comm->rank : 0; }

// In-place sum over the ranks of n doubles (PCG reductions; capturable).  A one-rank sum is the
// identity: no NCCL call unless AGIPC_OPT_COMM_ALWAYS asks for it (tests of the captured path).
agipc_status comm_allreduce_f64(agipc_handle h, double *buf, int64_t n, cudaStream_t s) {
  if (h->comm->nranks == 1 && !h->opt_comm_always) return AGIPC_OK;
  NCCL_TRY(h, g_nccl.AllReduce(buf, buf, (size_t)n, ncclFloat64, ncclSum, h->comm->nc, s));
  return AGIPC_OK;
}

// One grouped exchange with every peer: send sendbuf[soff[q] .. soff[q+1]) to peer_rank[q] and
// receive recvbuf[roff[q] .. roff[q+1]) from it (element counts of `dt`; capturable).
agipc_status comm_sendrecv(agipc_handle h, int n_peers, const int *peer_rank, const void *sendbuf,
                           const int64_t *soff, void *recvbuf, const int64_t *roff, ncclDataType_t dt, size_t esize,
                           cudaStream_t s) {
  if (n_peers == 0) return AGIPC_OK;
  NCCL_TRY(h, g_nccl.GroupStart());
  for (int q = 0; q < n_peers; ++q) {
    const int64_t ns = soff[q + 1] - soff[q], nr = roff[q + 1] - roff[q];
    if (ns > 0) {
      ncclResult_t r = g_nccl.Send((const char *)sendbuf + esize * soff[q], (size_t)ns, dt, peer_rank[q], h->comm->nc, s);
      if (r != ncclSuccess) {
        g_nccl.GroupEnd();
        return set_err(h, AGIPC_ENCCL, "ncclSend to %d: %s", peer_rank[q], g_nccl.GetErrorString(r));
      }
    }
    if (nr > 0) {
      ncclResult_t r = g_nccl.Recv((char *)recvbuf + esize * roff[q], (size_t)nr, dt, peer_rank[q], h->comm->nc, s);
      if (r != ncclSuccess) {
        g_nccl.GroupEnd();
        return set_err(h, AGIPC_ENCCL, "ncclRecv from %d: %s", peer_rank[q], g_nccl.GetErrorString(r));
      }
    }
  }
  NCCL_TRY(h, g_nccl.GroupEnd());
  return AGIPC_OK;
}

agipc_status comm_sendrecv_f64(agipc_handle h, int n_peers, const int *peer_rank, const double *sendbuf,
                               const int64_t *soff, double *recvbuf, const int64_t *roff, cudaStream_t s) {
  return comm_sendrecv(h, n_peers, peer_rank, sendbuf, soff, recvbuf, roff, ncclFloat64, 8, s);
}

agipc_status comm_check(agipc_handle h, const char *who) {
  if (!h->comm) return set_err(h, AGIPC_EINVAL, "%s: no communicator (agipc_comm_init)", who);
  return AGIPC_OK;
}

// out[k] (k < K) = sum over ranks r' < rank of all[r'][k]; out[K + k] = the total over all ranks
__global__ void k_rank_scan(int nranks, int rank, int K, const int64_t *__restrict__ all, int64_t *__restrict__ out) {
  const int k = threadIdx.x;
  if (k >= K) return;
  long long ex = 0, tot = 0;
  for (int r = 0; r < nranks; ++r) {
    const long long v = all[(int64_t)r * K + k];
    if (r < rank) ex += v;
    tot += v;
  }
  out[k] = ex;
  out[K + k] = tot;
}

// rows of row_bytes (multiple of 4) gathered by index: dst[k] = src[idx[k]]
__global__ void k_gather_rows4(int64_t n, int words, const uint32_t *__restrict__ src, const int32_t *__restrict__ idx,
                               uint32_t *__restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * words; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / words, w = i - k * words;
    dst[i] = src[(int64_t)idx[k] * words + w];
  }
}

extern "C" {

agipc_status agipc_comm_unique_id(void *id) {
  if (!id) return AGIPC_EINVAL;
  if (!nccl_load()) return AGIPC_ENCCL;
  ncclUniqueId u;
  if (g_nccl.GetUniqueId(&u) != ncclSuccess) return AGIPC_ENCCL;
  memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  return AGIPC_OK;
}

agipc_status agipc_comm_init(agipc_handle h, const void *unique_id, int nranks, int rank) {
  if (!h) return AGIPC_EINVAL;
  if (!unique_id || nranks < 1 || rank < 0 || rank >= nranks)
    return set_err(h, AGIPC_EINVAL, "comm_init: bad arguments (nranks %d, rank %d)", nranks, rank);
  if (!nccl_load()) return set_err(h, AGIPC_ENCCL, "comm_init: %s", g_nccl_err.c_str());
  CU_TRY(h, cudaSetDevice(h->device));
  comm_free(h);
  ncclUniqueId u;
  memcpy(u.internal, unique_id, NCCL_UNIQUE_ID_BYTES);
  Comm *c = new Comm();
  ncclResult_t r = g_nccl.CommInitRank(&c->nc, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return set_err(h, AGIPC_ENCCL, "ncclCommInitRank(%d of %d): %s", rank, nranks, g_nccl.GetErrorString(r));
  }
  c->nranks = nranks;
  c->rank = rank;
  h->comm = c;
  return AGIPC_OK;
}

agipc_status agipc_comm_info(agipc_handle h, int *nranks, int *rank, int *nccl_version) {
  if (!h) return AGIPC_EINVAL;
  if (nranks) *nranks = comm_size(h);
  if (rank) *rank = comm_rank(h);
  if (nccl_version) {
    *nccl_version = 0;
    if (g_nccl.so) g_nccl.GetVersion(nccl_version);
  }
  return AGIPC_OK;
}

agipc_status agipc_comm_allgather_scan(agipc_handle h, const int64_t *local, int k, int64_t *all, int64_t *scan) {
  if (!h) return AGIPC_EINVAL;
  agipc_status st = comm_check(h, "comm_allgather_scan");
  if (st != AGIPC_OK) return st;
  if (!local || !all || !scan || k < 1 || k > 1024) return set_err(h, AGIPC_EINVAL, "comm_allgather_scan: bad arguments");
  CU_TRY(h, cudaSetDevice(h->device));
  ProfScope prof(h, PROF_DIST, h->stream);
  NCCL_TRY(h, g_nccl.AllGather(local, all, (size_t)k, ncclInt64, h->comm->nc, h->stream));
  LAUNCH(h, k_rank_scan, 1, 1024, 0, h->comm->nranks, h->comm->rank, k, (const int64_t *)all, scan);
  return AGIPC_OK;
}

agipc_status agipc_comm_alltoall_i64(agipc_handle h, const int64_t *send, int64_t *recv) {
  if (!h) return AGIPC_EINVAL;
  agipc_status st = comm_check(h, "comm_alltoall_i64");
  if (st != AGIPC_OK) return st;
  if (!send || !recv) return set_err(h, AGIPC_EINVAL, "comm_alltoall_i64: null pointer");
  CU_TRY(h, cudaSetDevice(h->device));
  const int R = h->comm->nranks;
  NCCL_TRY(h, g_nccl.GroupStart());
  for (int q = 0; q < R; ++q) {
    ncclResult_t r1 = g_nccl.Send(send + q, 1, ncclInt64, q, h->comm->nc, h->stream);
    ncclResult_t r2 = g_nccl.Recv(recv + q, 1, ncclInt64, q, h->comm->nc, h->stream);
    if (r1 != ncclSuccess || r2 != ncclSuccess) {
      g_nccl.GroupEnd();
      return set_err(h, AGIPC_ENCCL, "comm_alltoall_i64: %s", g_nccl.GetErrorString(r1 != ncclSuccess ? r1 : r2));
    }
  }
  NCCL_TRY(h, g_nccl.GroupEnd());
  return AGIPC_OK;
}

agipc_status agipc_halo_exchange(agipc_handle h, const agipc_halo *halo, const void *src, int row_bytes, void *dst) {
  if (!h) return AGIPC_EINVAL;
  agipc_status st = comm_check(h, "halo_exchange");
  if (st != AGIPC_OK) return st;
  if (!halo || row_bytes <= 0 || (row_bytes & 3)) return set_err(h, AGIPC_EINVAL, "halo_exchange: bad arguments");
  if (halo->n_peers == 0) return AGIPC_OK;
  if (!halo->peer_rank || !halo->send_ptr || !halo->recv_ptr || !src || !dst)
    return set_err(h, AGIPC_EINVAL, "halo_exchange: null pointer");
  const int P = halo->n_peers;
  for (int q = 0; q < P; ++q)
    if (halo->peer_rank[q] < 0 || halo->peer_rank[q] >= h->comm->nranks || halo->send_ptr[q + 1] < halo->send_ptr[q] ||
        halo->recv_ptr[q + 1] < halo->recv_ptr[q])
      return set_err(h, AGIPC_EINVAL, "halo_exchange: bad peer %d", q);
  CU_TRY(h, cudaSetDevice(h->device));
  ProfScope prof(h, PROF_DIST, h->stream);
  const int64_t n_send = halo->send_ptr[P] - halo->send_ptr[0];
  const int words = row_bytes / 4;
  uint32_t *sendbuf = nullptr;
  if (n_send > 0) {
    if (!halo->send_idx) return set_err(h, AGIPC_EINVAL, "halo_exchange: null send_idx");
    WS(h, sb, uint32_t, "halo_sendbuf", n_send * words);
    sendbuf = sb;
    LAUNCH(h, k_gather_rows4, (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n_send * words, 256), 8 * h->sm_count)),
           256, 0, n_send, words, (const uint32_t *)src, halo->send_idx + halo->send_ptr[0], sendbuf);
  }
  std::vector<int64_t> so(P + 1), ro(P + 1);
  for (int q = 0; q <= P; ++q) {
    so[q] = (halo->send_ptr[q] - halo->send_ptr[0]) * words;
    ro[q] = (halo->recv_ptr[q] - halo->recv_ptr[0]) * words;
  }
  return comm_sendrecv(h, P, halo->peer_rank, sendbuf, so.data(), (uint32_t *)dst + halo->recv_ptr[0] * words,
                       ro.data(), ncclUint32, 4, h->stream);
}

}  // extern "C"
