// Step 2 -- the fine-to-coarse map (supp Alg S1/S2; recursion P:217).
//
// B200 design:
//  * one warp hosts floor(32/gs) groups of gs consecutive nodes ("a Warp may handle
//    multiple groups"); each lane owns one node and keeps its 32-bit connectivity hash in a
//    register (Alg S1's con_hashs) -- no shared-memory hash table;
//  * the OR-propagation of Alg S2 is a register Warshall closure: for k < gs,
//    h |= bit_k(h) ? shfl(h, lane k of my group) : 0 -- gs unconditional shuffles, all lanes
//    converged; it equals the BFS over the initial hashes (reachability inside the group);
//  * election is one __ballot_sync of "no set bit below my lane"; the local
//    index is the popcount of elected lanes below the FIRST SET BIT of the closed hash
//    (P:86, P:222 -- reading R1, which corrects the lane_id of P:183-184);
//  * the ExclusiveSum over per-group counts is fused into the same kernel with a
//    single-pass decoupled look-back over CTA tiles, and map = O[g] + P;
//  * level >= 1: the surviving tagged edges mapped through the level map (self loops
//    dropped) are the next level's graph; their intra-group part is OR-ed into per-node
//    hashes with atomicOr, then the same group kernel runs.  The final map composes the
//    level maps; the recursion stops at the first level without an intra-group edge.
#include "agipc_internal.cuh"

#define MAP_THREADS 256
#define MAP_WARPS (MAP_THREADS / 32)

struct GroupGeom {
  int gs;         // group size 1..32
  int gpw;        // groups per warp = 32 / gs
  unsigned gmask; // low gs bits
};

// One level of Alg S1/S2 over n nodes.  FROM_CSR: level 0 (hash from adjacency + tags, emits
// tagged cross-group edges); otherwise the intra-group hashes come from h_mem.
template <bool FROM_CSR>
__global__ void __launch_bounds__(MAP_THREADS)
    k_group_pass(int64_t n, GroupGeom geo, const int64_t *__restrict__ adj_ptr,
                 const int32_t *__restrict__ adj_nbr, const uint8_t *__restrict__ tags,
                 const uint32_t *__restrict__ h_mem, int32_t *__restrict__ map_out,
                 int2 *__restrict__ cross, unsigned long long *__restrict__ cross_count,
                 unsigned long long *status, int *tile_counter, long long *n_out) {
  __shared__ int s_tile;
  __shared__ long long s_warp[MAP_WARPS];
  __shared__ long long s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1);
  __syncthreads();
  const int tile = s_tile;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gs = geo.gs;
  const int gin = lane / gs;                 // group index inside the warp
  const int lig = lane - gin * gs;           // lane in group (Alg S1 lane_id)
  const int64_t g = ((int64_t)tile * MAP_WARPS + w) * geo.gpw + gin;
  const int64_t v = g * gs + lig;
  const bool active = (gin < geo.gpw) && (v < n);

  uint32_t h = 0;
  if (active) {
    h = 1u << lig;  // Alg S1 l.4
    if (FROM_CSR) {
      int64_t k0 = adj_ptr[v], k1 = adj_ptr[v + 1];
      int ncross = 0;
      for (int64_t k = k0; k < k1; ++k) {
        if (!tags[k]) continue;                   // protected edge (Alg S1 l.6-8)
        int64_t u = adj_nbr[k];
        if (u / gs == g) h |= 1u << (int)(u - g * gs);  // same group (l.10-13)
        else if (u > v) ++ncross;
      }
      // tagged cross-group edges (u > v): the level-1 graph ("remained neighbour")
      if (ncross) {
        unsigned long long base = atomicAdd(cross_count, (unsigned long long)ncross);
        int o = 0;
        for (int64_t k = k0; k < k1; ++k) {
          if (!tags[k]) continue;
          int64_t u = adj_nbr[k];
          if (u / gs != g && u > v) cross[base + o++] = make_int2((int)v, (int)u);
        }
      }
    } else {
      h |= h_mem[v];
    }
  }
  // Alg S2 OR-propagation == Warshall closure inside the group (registers + shuffles)
  const int base_lane = gin * gs;
  for (int k = 0; k < gs; ++k) {
    uint32_t t = __shfl_sync(FULL_MASK, h, (base_lane + k) & 31);
    if ((h >> k) & 1u) h |= t;
  }
  // election: lowest lane of each component
  const bool elected = active && ((h & ((1u << lig) - 1u)) == 0u);
  const unsigned bal = __ballot_sync(FULL_MASK, elected);
  // local index: elected lanes below the first set bit of my closed hash (R1)
  const unsigned gelect = (bal >> base_lane) & geo.gmask;
  const int first = active ? __ffs(h) - 1 : 0;
  const int local = __popc(gelect & ((1u << first) - 1u));
  const int warp_off = __popc(bal & ((1u << base_lane) - 1u));  // earlier groups of this warp
  if (lane == 0) s_warp[w] = __popc(bal);
  __syncthreads();
  if (w == 0) {
    long long c = lane < MAP_WARPS ? s_warp[lane] : 0;
    long long ci = warp_incl_scan(c);
    long long agg = __shfl_sync(FULL_MASK, ci, MAP_WARPS - 1);
    if (lane < MAP_WARPS) s_warp[lane] = ci - c;
    long long pfx = lb_exclusive(status, tile, agg);  // ExclusiveSum over groups
    if (lane == 0) {
      s_prefix = pfx;
      if (tile == (int)gridDim.x - 1) *n_out = pfx + agg;
    }
  }
  __syncthreads();
  if (active) map_out[v] = (int32_t)(s_prefix + s_warp[w] + warp_off + local);  // O[g] + P
}

// Level >= 1: OR the intra-group edges of the current graph into per-node hashes.
__global__ void k_edges_intra(const int2 *__restrict__ E, const unsigned long long *__restrict__ ne_ptr,
                              int gs, uint32_t *__restrict__ h, int *__restrict__ any) {
  const int64_t ne = (int64_t)*ne_ptr;
  bool hit = false;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    int2 uv = E[e];
    int gu = uv.x / gs, gv = uv.y / gs;
    if (gu == gv) {
      atomicOr(h + uv.x, 1u << (uv.y - gv * gs));
      atomicOr(h + uv.y, 1u << (uv.x - gu * gs));
      hit = true;
    }
  }
  if (__any_sync(FULL_MASK, hit) && lane_id() == 0) *any = 1;
}

// Map the edge list through map_k; drop self loops; compact into E_out.
__global__ void k_edges_remap(const int2 *__restrict__ E, const unsigned long long *__restrict__ ne_ptr,
                              const int32_t *__restrict__ mk, int2 *__restrict__ E_out,
                              unsigned long long *__restrict__ ne_out) {
  const int64_t ne = (int64_t)*ne_ptr;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < ne; base += stride) {
    int64_t e = base + threadIdx.x;
    int2 o = make_int2(0, 0);
    bool keep = false;
    if (e < ne) {
      int2 uv = E[e];
      o.x = mk[uv.x];
      o.y = mk[uv.y];
      keep = o.x != o.y;
    }
    unsigned b = __ballot_sync(FULL_MASK, keep);
    unsigned long long wbase = 0;
    if (lane_id() == 0 && b) wbase = atomicAdd(ne_out, (unsigned long long)__popc(b));
    wbase = __shfl_sync(FULL_MASK, wbase, 0);
    if (keep) E_out[wbase + __popc(b & ((1u << lane_id()) - 1u))] = o;
  }
}

// comp[c] = mk[comp[c]]  (compose the level maps on the level-1 index space)
__global__ void k_compose(int64_t n, int32_t *__restrict__ comp, const int32_t *__restrict__ mk, int first) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n) comp[c] = first ? mk[c] : mk[comp[c]];
}

// map[f] = comp[map[f]]
__global__ void k_apply(int64_t n, int32_t *__restrict__ map, const int32_t *__restrict__ comp) {
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f < n) map[f] = comp[map[f]];
}

// Aggregate sizes: histogram of the final map with warp-aggregated atomics.
__global__ void k_histogram(int64_t n, const int32_t *__restrict__ map, int32_t *__restrict__ cnt) {
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int key = f < n ? map[f] : -1;
  unsigned peers = __match_any_sync(FULL_MASK, key);
  if (key >= 0 && (__ffs(peers) - 1) == lane_id()) atomicAdd(cnt + key, __popc(peers));
}

static agipc_status group_pass(agipc_handle h, bool from_csr, int64_t n, GroupGeom geo, const agipc_mesh *mesh,
                               const uint8_t *tags, const uint32_t *hmem, int32_t *map_out, int2 *cross,
                               unsigned long long *cross_count, long long *n_out) {
  int64_t groups = cdiv(n, geo.gs);
  int64_t tiles = cdiv(groups, (int64_t)MAP_WARPS * geo.gpw);
  if (tiles == 0) tiles = 1;
  WS(h, status, unsigned long long, "map_status", tiles + 1);
  CU_TRY(h, cudaMemsetAsync(status, 0, sizeof(unsigned long long) * (tiles + 1), h->stream));
  int *counter = (int *)(status + tiles);
  if (from_csr)
    LAUNCH(h, k_group_pass<true>, (unsigned)tiles, MAP_THREADS, 0, n, geo, mesh->adj_ptr, mesh->adj_nbr, tags,
           hmem, map_out, cross, cross_count, status, counter, n_out);
  else
    LAUNCH(h, k_group_pass<false>, (unsigned)tiles, MAP_THREADS, 0, n, geo, nullptr, nullptr, nullptr, hmem,
           map_out, cross, cross_count, status, counter, n_out);
  return AGIPC_OK;
}

extern "C" agipc_status agipc_build_map(agipc_handle h, const agipc_mesh *mesh, const uint8_t *slot_tags,
                                        int group_size, int max_levels, int32_t *map, int32_t *agg_size,
                                        agipc_map_info *info) {
  if (!h) return AGIPC_EINVAL;
  if (!mesh || !info) return set_err(h, AGIPC_EINVAL, "build_map: null mesh/info");
  if (group_size < 1 || group_size > 32) return set_err(h, AGIPC_EINVAL, "build_map: group_size %d not in [1,32]", group_size);
  if (mesh->n_nodes < 0 || max_levels < 0) return set_err(h, AGIPC_EINVAL, "build_map: negative size");
  if (mesh->n_nodes >= INT32_MAX || mesh->nnz_adj >= INT32_MAX) return set_err(h, AGIPC_ERANGE, "build_map: index exceeds int32");
  const int64_t N = mesh->n_nodes;
  memset(info, 0, sizeof(*info));
  if (N == 0) {
    info->n_levels = 1;
    return AGIPC_OK;
  }
  if (!map || !mesh->adj_ptr || (mesh->nnz_adj > 0 && (!mesh->adj_nbr || !slot_tags)))
    return set_err(h, AGIPC_EINVAL, "build_map: null pointer");
  CU_TRY(h, cudaSetDevice(h->device));
  ProfScope prof_scope(h, PROF_MAP, h->stream);
  GroupGeom geo;
  geo.gs = group_size;
  geo.gpw = 32 / group_size;
  geo.gmask = group_size == 32 ? 0xffffffffu : ((1u << group_size) - 1u);

  // scalars: [0] n_out (level), [1] cross count, [2] edge count A, [3] edge count B, [4] any-intra flag
  WS(h, sc, long long, "map_scalars", 8);
  agipc_status st;
  long long *hs = (long long *)pinned_get(h, 64, &st);
  if (st != AGIPC_OK) return st;
  const int64_t ecap = mesh->nnz_adj / 2 + 1;
  WS(h, cross, int2, "map_cross", ecap);
  CU_TRY(h, cudaMemsetAsync(sc, 0, 8 * sizeof(long long), h->stream));

  // ---- level 0: warp-per-group hashing over the fine mesh (fused scan) ----
  st = group_pass(h, true, N, geo, mesh, slot_tags, nullptr, map, cross, (unsigned long long *)(sc + 1), sc + 0);
  if (st != AGIPC_OK) return st;
  CU_TRY(h, cudaMemcpyAsync(hs, sc, 2 * sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  int64_t n = hs[0];
  int64_t ncross = hs[1];
  info->n_cross_edges = ncross;
  info->level_n[0] = n;
  int level = 1;
  bool done = (n == N) || (max_levels == 1);

  if (!done) {
    const int64_t n1 = n;
    WS(h, EA, int2, "map_EA", ecap);
    WS(h, EB, int2, "map_EB", ecap);
    WS(h, hh, uint32_t, "map_h", n1);
    WS(h, mk, int32_t, "map_mk", n1);
    WS(h, comp, int32_t, "map_comp", n1);
    unsigned long long *neA = (unsigned long long *)(sc + 2), *neB = (unsigned long long *)(sc + 3);
    int *any = (int *)(sc + 4);
    // level-1 graph = tagged cross edges mapped through the level-0 map
    CU_TRY(h, cudaMemsetAsync(neA, 0, sizeof(long long), h->stream));
    LAUNCH(h, k_edges_remap, (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(ncross, 256), 8 * h->sm_count)), 256, 0,
           cross, (const unsigned long long *)(sc + 1), map, EA, neA);
    int first = 1;
    while (true) {
      ++level;
      CU_TRY(h, cudaMemsetAsync(hh, 0, sizeof(uint32_t) * n, h->stream));
      CU_TRY(h, cudaMemsetAsync(any, 0, sizeof(int), h->stream));
      LAUNCH(h, k_edges_intra, (unsigned)(8 * h->sm_count), 256, 0, EA, neA, group_size, hh, any);
      CU_TRY(h, cudaMemcpyAsync(hs, any, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
      CU_TRY(h, cudaStreamSynchronize(h->stream));
      if (*(int *)hs == 0) {  // no intra-group edge: this pass merges nothing (fixpoint)
        if (level <= 64) info->level_n[level - 1] = n;
        break;
      }
      st = group_pass(h, false, n, geo, mesh, nullptr, hh, mk, nullptr, nullptr, sc + 0);
      if (st != AGIPC_OK) return st;
      CU_TRY(h, cudaMemsetAsync(neB, 0, sizeof(long long), h->stream));
      LAUNCH(h, k_edges_remap, (unsigned)(8 * h->sm_count), 256, 0, EA, neA, mk, EB, neB);
      LAUNCH(h, k_compose, (unsigned)cdiv(n1, 256), 256, 0, n1, comp, mk, first);
      first = 0;
      CU_TRY(h, cudaMemcpyAsync(hs, sc, sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
      CU_TRY(h, cudaStreamSynchronize(h->stream));
      n = hs[0];
      if (level <= 64) info->level_n[level - 1] = n;
      std::swap(EA, EB);
      std::swap(neA, neB);
      if (max_levels > 0 && level >= max_levels) break;
    }
    if (!first) LAUNCH(h, k_apply, (unsigned)cdiv(N, 256), 256, 0, N, map, comp);
  }
  info->n_coarse = n;
  info->n_levels = level;
  if (agg_size) {
    CU_TRY(h, cudaMemsetAsync(agg_size, 0, sizeof(int32_t) * n, h->stream));
    LAUNCH(h, k_histogram, (unsigned)cdiv(N, 256), 256, 0, N, map, agg_size);
  }
  CU_TRY(h, cudaStreamSynchronize(h->stream));
  return AGIPC_OK;
}
