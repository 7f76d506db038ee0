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
//  * level >= 1 runs in ONE cooperative persistent kernel: per level, the surviving
//    tagged edges (mapped through the previous level, self loops dropped) OR their intra-group
//    part into per-node hashes (atomicOr), a grid barrier, the same group pass, a barrier, the
//    edge remap + compaction and the composition of the level maps, a barrier.  No host round
//    trip per level; the recursion stops at the first level without an intra-group edge.
#include <cooperative_groups.h>

#include <memory>

#include "agipc_internal.cuh"

namespace cg = cooperative_groups;

#define MAP_THREADS 256
#define MAP_WARPS (MAP_THREADS / 32)

struct GroupGeom {
  int gs;          // group size 1..32
  int gpw;         // groups per warp = 32 / gs
  unsigned gmask;  // low gs bits
};

struct TileSmem {
  int tile;
  long long warp[MAP_WARPS];
  long long prefix;
};

__device__ __forceinline__ int64_t tiles_of(int64_t n, const GroupGeom &geo) {
  return (((n + geo.gs - 1) / geo.gs) + (int64_t)MAP_WARPS * geo.gpw - 1) / ((int64_t)MAP_WARPS * geo.gpw);
}

// One CTA tile of one level of Alg S1/S2 over n nodes.  FROM_CSR: level 0 (hash from adjacency
// + tags, emits the tagged cross-group edges); otherwise the intra-group hashes come from h_mem
// (which is cleared after it is read, ready for the next level).
template <bool FROM_CSR>
__device__ __forceinline__ void group_tile(TileSmem &S, int tile, int64_t ntiles, int64_t n, const GroupGeom &geo,
                                           const int64_t *__restrict__ adj_ptr, const int32_t *__restrict__ adj_nbr,
                                           const uint8_t *__restrict__ tags, uint32_t *h_mem,
                                           int32_t *__restrict__ map_out, int2 *__restrict__ cross,
                                           unsigned long long *__restrict__ cross_count, unsigned long long *status,
                                           long long *n_out) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gs = geo.gs;
  const int gin = lane / gs;        // group index inside the warp
  const int lig = lane - gin * gs;  // lane in group (Alg S1 lane_id)
  const int64_t g = ((int64_t)tile * MAP_WARPS + w) * geo.gpw + gin;
  const int64_t v = g * gs + lig;
  const bool active = (gin < geo.gpw) && (v < n);

  uint32_t h = 0;
  if (active) {
    h = 1u << lig;  // Alg S1 l.4
    if (FROM_CSR) {
      const int64_t k0 = adj_ptr[v], k1 = adj_ptr[v + 1];
      int ncross = 0;
      for (int64_t k = k0; k < k1; ++k) {
        if (!tags[k]) continue;  // protected edge (Alg S1 l.6-8)
        const int64_t u = adj_nbr[k];
        if (u / gs == g) h |= 1u << (int)(u - g * gs);  // same group (l.10-13)
        else if (u > v) ++ncross;
      }
      // tagged cross-group edges (u > v): the level-1 graph ("remained neighbour")
      if (ncross) {
        unsigned long long base = atomicAdd(cross_count, (unsigned long long)ncross);
        int o = 0;
        for (int64_t k = k0; k < k1; ++k) {
          if (!tags[k]) continue;
          const int64_t u = adj_nbr[k];
          if (u / gs != g && u > v) cross[base + o++] = make_int2((int)v, (int)u);
        }
      }
    } else {
      h |= h_mem[v];
      h_mem[v] = 0u;
    }
  }
  // Alg S2 OR-propagation == Warshall closure inside the group (registers + shuffles)
  const int base_lane = gin * gs;
  for (int k = 0; k < gs; ++k) {
    const uint32_t t = __shfl_sync(FULL_MASK, h, (base_lane + k) & 31);
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
  if (lane == 0) S.warp[w] = __popc(bal);
  __syncthreads();
  if (w == 0) {
    const long long c = lane < MAP_WARPS ? S.warp[lane] : 0;
    const long long ci = warp_incl_scan(c);
    const long long agg = __shfl_sync(FULL_MASK, ci, MAP_WARPS - 1);
    if (lane < MAP_WARPS) S.warp[lane] = ci - c;
    const long long pfx = lb_exclusive(status, tile, agg);  // ExclusiveSum over groups
    if (lane == 0) {
      S.prefix = pfx;
      if (tile == ntiles - 1) *n_out = pfx + agg;
    }
  }
  __syncthreads();
  if (active) map_out[v] = (int32_t)(S.prefix + S.warp[w] + warp_off + local);  // O[g] + P
  __syncthreads();  // S is reused by the next tile of a persistent CTA
}

// Level 0 over the fine mesh.  A warp handles L0_CHUNKS consecutive chunks of gpw groups
// (<= 32 nodes); the adjacency entries of a chunk are read ENTRY-parallel (lane = entry,
// coalesced adj_nbr / tag loads, every load independent), each entry's row found by a binary
// search over the chunk's row pointers in shared memory; intra-group tagged edges set the row's
// hash bit with a shared atomicOr (Alg S1 l.10-13), tagged cross-group edges (u > v) are
// compacted warp-wide (one global atomic per 32 entries).  Then the register closure /
// election of group_tile per chunk, and one decoupled look-back per CTA tile.
#ifndef L0_CHUNKS
#define L0_CHUNKS 1  // chunks of groups per warp per tile (2 / 4 / 8 measured slower: 98 / 105 / 164 vs 94.5 us at C3, profiles/r02v)
#endif
#define L0_XCAP 256

#ifdef L0_MINB  // (6 / 8 CTAs per SM measured slower: 40 / 32 registers with spills, profiles/r02v)
__global__ void __launch_bounds__(MAP_THREADS, L0_MINB)
#else
__global__ void __launch_bounds__(MAP_THREADS)
#endif
    k_level0(int64_t n, GroupGeom geo, const int64_t *__restrict__ adj_ptr, const int32_t *__restrict__ adj_nbr,
             const uint8_t *__restrict__ tags, int32_t *__restrict__ map_out, int2 *__restrict__ cross,
             unsigned long long *__restrict__ cross_count, int32_t *__restrict__ tile_cnt, int *tile_counter) {
  __shared__ TileSmem S;
  __shared__ long long s_ptr[MAP_WARPS][33];
  __shared__ uint32_t s_h[MAP_WARPS][32];
  __shared__ int s_gb[MAP_WARPS][32];             // first node of the group of each chunk row
  __shared__ int2 s_cross[MAP_WARPS][L0_XCAP];    // per-warp buffer of tagged cross edges
  if (threadIdx.x == 0) S.tile = atomicAdd(tile_counter, 1);
  __syncthreads();
  const int tile = S.tile;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gs = geo.gs, cn = geo.gpw * gs;  // nodes per chunk
  const int gin = lane / gs, lig = lane - gin * gs, base_lane = gin * gs;
  int local[L0_CHUNKS], off[L0_CHUNKS];
  int wcount = 0, nx = 0;  // nx: cross edges buffered by this warp
  // flush the warp's buffered cross edges with ONE global atomic (a single counter shared by
  // the whole grid is the contended resource)
  auto flush = [&]() {
    __syncwarp();  // the lanes' s_cross writes are visible before other lanes read them
    unsigned long long cb = 0;
    if (lane == 0) cb = atomicAdd(cross_count, (unsigned long long)nx);
    cb = __shfl_sync(FULL_MASK, cb, 0);
    for (int t = lane; t < nx; t += 32) cross[cb + t] = s_cross[w][t];
    __syncwarp();
    nx = 0;
  };
#pragma unroll
  for (int c = 0; c < L0_CHUNKS; ++c) {
    const int64_t q = ((int64_t)tile * MAP_WARPS + w) * L0_CHUNKS + c;
    const int64_t v0 = q * cn;
    const int nn = v0 < n ? (int)min((int64_t)cn, n - v0) : 0;
    const int64_t v = v0 + lane;
    const bool active = lane < nn;
    if (lane <= nn) s_ptr[w][lane] = adj_ptr[v0 + lane];
    if (lane == 0 && nn == 32) s_ptr[w][32] = adj_ptr[v0 + 32];
    s_h[w][lane] = 0u;
    s_gb[w][lane] = (int)(v0 + (lane / gs) * gs);  // v0 is a multiple of gs
    __syncwarp();
    if (nn > 0) {
      const long long E0 = s_ptr[w][0], E1 = s_ptr[w][nn];
      // software pipeline: the next 32 entries' neighbour / tag loads are issued before this
      // batch's row search, hash OR and ballots
      int u_nx = 0, t_nx = 0;
      if (E0 + lane < E1) {
        u_nx = __ldg(adj_nbr + E0 + lane);
        t_nx = __ldg(tags + E0 + lane);
      }
      for (long long eb = E0; eb < E1; eb += 32) {
        const long long e = eb + lane;
        const bool valid = e < E1;
        const int u = u_nx, t = t_nx;
        if (e + 32 < E1) {
          u_nx = __ldg(adj_nbr + e + 32);
          t_nx = __ldg(tags + e + 32);
        }
        int lo = 0, hi = nn;  // row r: s_ptr[r] <= e < s_ptr[r+1]
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (s_ptr[w][mid] <= e) lo = mid; else hi = mid;
        }
        const int vv = (int)(v0 + lo);
        const int gb = s_gb[w][lo];
        const bool tg = valid && t;
        const bool intra = tg && u >= gb && u < gb + gs;
        const bool cr = tg && !intra && u > vv;
        if (intra) atomicOr(&s_h[w][lo], 1u << (u - gb));
        const unsigned b = __ballot_sync(FULL_MASK, cr);
        if (b) {
          if (nx + __popc(b) > L0_XCAP) flush();
          if (cr) s_cross[w][nx + __popc(b & ((1u << lane) - 1u))] = make_int2(vv, u);
          nx += __popc(b);
        }
      }
    }
    __syncwarp();
    uint32_t h = active ? ((1u << lig) | s_h[w][lane]) : 0u;
    for (int k = 0; k < gs; ++k) {  // Alg S2 OR-propagation == Warshall closure
      const uint32_t tt = __shfl_sync(FULL_MASK, h, (base_lane + k) & 31);
      if ((h >> k) & 1u) h |= tt;
    }
    const bool elected = active && gin < geo.gpw && ((h & ((1u << lig) - 1u)) == 0u);
    const unsigned bal = __ballot_sync(FULL_MASK, elected);
    const unsigned gelect = (bal >> base_lane) & geo.gmask;
    const int first = active ? __ffs(h) - 1 : 0;
    local[c] = __popc(gelect & ((1u << first) - 1u));
    off[c] = wcount + __popc(bal & ((1u << base_lane) - 1u));
    wcount += __popc(bal);
    __syncwarp();
  }
  __syncwarp();
  if (nx) flush();
  if (lane == 0) S.warp[w] = wcount;
  __syncthreads();
  if (w == 0) {
    const long long cc = lane < MAP_WARPS ? S.warp[lane] : 0;
    const long long ci = warp_incl_scan(cc);
    const long long agg = __shfl_sync(FULL_MASK, ci, MAP_WARPS - 1);
    if (lane < MAP_WARPS) S.warp[lane] = ci - cc;
    // the ExclusiveSum over groups is split: this tile's count now, the tile prefix by one
    // scan afterwards, added by the map's consumers (k_cross_to_level1, k_apply) -- no look-back
    // chain on this kernel's critical path (it cost ~40 of 140 us at C3, profiles/r02v)
    if (lane == 0) tile_cnt[tile] = (int32_t)agg;
  }
  __syncthreads();
  const long long wb = S.warp[w];  // tile-relative map
#pragma unroll
  for (int c = 0; c < L0_CHUNKS; ++c) {
    const int64_t q = ((int64_t)tile * MAP_WARPS + w) * L0_CHUNKS + c;
    const int64_t v = q * cn + lane;
    if (lane < cn && v < n) map_out[v] = (int32_t)(wb + off[c] + local[c]);  // O[g] + P, minus the tile prefix
  }
}

// CTA-wide stream compaction: returns this thread's output position for keep == true, with ONE
// global atomic per CTA (a single grid-wide counter is the contended resource).  All threads of
// the CTA must call it; s_w holds blockDim/32 ints, s_base one 64-bit word.
__device__ __forceinline__ unsigned long long cta_compact(bool keep, unsigned long long *counter, int *s_w,
                                                          unsigned long long *s_base) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  const unsigned b = __ballot_sync(FULL_MASK, keep);
  if (l == 0) s_w[w] = __popc(b);
  __syncthreads();
  if (w == 0) {
    const int c = l < nw ? s_w[l] : 0;
    const int ci = warp_incl_scan(c);
    if (l < nw) s_w[l] = ci - c;
    const int tot = __shfl_sync(FULL_MASK, ci, 31);
    if (l == 0) *s_base = tot ? atomicAdd(counter, (unsigned long long)tot) : 0ull;
  }
  __syncthreads();
  const unsigned long long pos = *s_base + s_w[w] + __popc(b & ((1u << l) - 1u));
  __syncthreads();  // s_w / s_base are reused by the next call
  return pos;
}

// Map the tagged fine cross edges through the level-0 map and de-duplicate them with an
// open-addressing hash set (key (a << 32 | b) + 1; a < b because the level-0 map is monotone
// across groups).  The slots a call fills are recorded and cleared again at the end.
__global__ void k_cross_to_level1(const int2 *__restrict__ E, const unsigned long long *__restrict__ ne_ptr,
                                  const int32_t *__restrict__ m0, unsigned long long *__restrict__ table,
                                  unsigned long long tmask, int2 *__restrict__ E_out,
                                  unsigned long long *__restrict__ ne_out, unsigned long long *__restrict__ used,
                                  const int64_t *__restrict__ tpref, int tn0, int64_t tiles0, long long *n1_out) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *n1_out = tpref[tiles0];  // level-1 node count
  __shared__ int s_w[32];
  __shared__ unsigned long long s_base;
  const int64_t ne = (int64_t)*ne_ptr;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < ne; base += stride) {
    const int64_t e = base + threadIdx.x;
    bool keep = false;
    int2 o = make_int2(0, 0);
    unsigned long long slot = 0;
    unsigned long long key = 0ull;  // 0: no edge
    if (e < ne) {
      const int2 uv = E[e];
      o = make_int2((int)(m0[uv.x] + tpref[uv.x / tn0]), (int)(m0[uv.y] + tpref[uv.y / tn0]));
      key = (((unsigned long long)(unsigned)o.x << 32) | (unsigned)o.y) + 1ull;
    }
    // neighbouring list entries mostly map to the same coarse pair: one probe per distinct key
    // of the warp (the lowest lane holding it)
    const unsigned same = __match_any_sync(FULL_MASK, key);
    if (key && (same & ((1u << (threadIdx.x & 31)) - 1u)) == 0u) {
      slot = (key * 0x9E3779B97F4A7C15ull) >> 20 & tmask;
      while (true) {
        const unsigned long long prev = atomicCAS(table + slot, 0ull, key);
        if (prev == 0ull) { keep = true; break; }
        if (prev == key) break;
        slot = (slot + 1) & tmask;
      }
    }
    const unsigned long long pos = cta_compact(keep, ne_out, s_w, &s_base);
    if (keep) {
      E_out[pos] = o;
      used[pos] = slot;
    }
  }
}

#ifndef TAIL_THREADS
#define TAIL_THREADS 1024
#endif
#define TAIL_WARPS (TAIL_THREADS / 32)
#ifndef TAIL_SUB
#define TAIL_SUB 2  // group blocks per warp per tile (a tile = TAIL_WARPS * TAIL_SUB * gpw * gs nodes)
#endif

struct TailArgs {
  GroupGeom geo;
  int max_levels;
  int64_t N;
  int tile_nodes;          // nodes per tile = TAIL_WARPS * TAIL_SUB * gpw * gs
  int2 *E[2];
  unsigned long long *ne;  // [2] edge counts of E[0], E[1]; ne[0] = level-1 edges on entry
  uint32_t *h;             // [>= n1], zero on entry
  int32_t *mk;             // tile-local rank of every node at the current level
  int32_t *comp;           // level-1 id -> current id
  int32_t *tcount;         // per-tile coarse-node count
  int *ctrl;               // [1] any intra edge, [2] levels run, [3] comp valid
  long long *nvals;        // [0] n1 on entry / final n on exit
  long long *level_n;      // [64]
  unsigned *bar;           // software grid barrier counter (zeroed before launch); nullptr =
                           // cooperative launch + cg grid.sync()
  unsigned long long *trace;  // AGIPC_TAIL_TRACE: CTA 0's %globaltimer at 7 points of each level
  // folded launches: the level-1 hash-set slots are cleared at the start (k_clear_slots) and the
  // fine map is finished at the end (k_apply: level-0 tile prefix, then the composed map)
  unsigned long long *table;
  const unsigned long long *used;
  int32_t *map;
  int64_t n_fine;
  const int64_t *tpref;
  int tn0;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Grid barrier of a persistent kernel whose CTAs are all resident (one per SM, checked by the
// occupancy query before launch): a monotone arrival counter, barrier i completes when it reaches
// (i + 1) * gridDim.x.  Lets k_tail go out as an ordinary launch (the host-side cost of
// cudaLaunchCooperativeKernel is paid while the GPU waits, once per Newton step).
#ifndef TAIL_BAR_ACQREL
#define TAIL_BAR_ACQREL 1
#endif
__device__ __forceinline__ void sw_grid_sync(unsigned *bar, unsigned &epoch) {
  __syncthreads();
  epoch += 1;
  if (threadIdx.x == 0) {
    const unsigned target = epoch * gridDim.x;
#if TAIL_BAR_ACQREL
    // release-add of the arrival (orders this CTA's writes, made visible to thread 0 by the
    // __syncthreads above, before it), acquire-load spin (orders every later read after the
    // other CTAs' releases): no full fences
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
#else
    __threadfence();
    atomicAdd(bar, 1u);
    while (*(volatile unsigned *)bar < target) __nanosleep(32);
    __threadfence();
#endif
  }
  __syncthreads();
}

// Levels >= 1 in one cooperative kernel, one 1024-thread CTA per SM, two grid barriers per
// level: (P2) closure/election per tile -> tile-local rank and per-tile count; (P3) every CTA
// scans the tile counts in shared memory, remaps + compacts the edges, composes the level maps
// and ORs the remapped intra-group edges into the next level's hashes (P1 of the next level;
// P1 of the first tail level runs on its own).  Stops at the first level without an
// intra-group edge.  The "any intra edge" flag alternates between ctrl[0] and ctrl[1].
__global__ void __launch_bounds__(TAIL_THREADS, 1) k_tail(TailArgs A) {
  unsigned epoch = 0;
  auto gsync = [&]() {
    if (A.bar) sw_grid_sync(A.bar, epoch);
    else cg::this_grid().sync();
  };
  extern __shared__ int32_t s_pref[];  // exclusive prefix of the tile counts
  __shared__ int s_w[TAIL_WARPS];
  __shared__ int s_red[TAIL_WARPS];
  __shared__ int s_total;
  __shared__ int s_cw[TAIL_WARPS];
  __shared__ unsigned long long s_cbase;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const GroupGeom geo = A.geo;
  const int gs = geo.gs;
  const int TN = A.tile_nodes;
  const int64_t n1 = A.nvals[0];
  int64_t n = n1;
  int level = 1, cur = 0;
  if (gtid == 0) A.level_n[0] = n1;
  {  // the level-1 de-duplication's hash slots, cleared for the next call (k_clear_slots)
    const int64_t ne0 = (int64_t)*(volatile unsigned long long *)A.ne;
    for (int64_t e = gtid; e < ne0; e += gstride) A.table[A.used[e]] = 0ull;
  }
  // fine map = level-0 id (tile-relative value + tile prefix), then the composed tail map (k_apply)
  auto apply = [&](bool composed) {
    for (int64_t f = gtid; f < A.n_fine; f += gstride) {
      const int g = (int)(A.map[f] + A.tpref[f / A.tn0]);
      A.map[f] = composed ? A.comp[g] : g;
    }
  };
  if (n1 == A.N) {  // level 0 merged nothing: fixpoint after one pass
    if (gtid == 0) A.ctrl[2] = 1;
    apply(false);
    return;
  }
  const int gin = lane / gs, lig = lane - gin * gs, base_lane = gin * gs;
  bool first_pass = true;
  bool composed = false;  // some level's P3 composed the level maps (ctrl[3])
  while (true) {
    ++level;
    const int fl = level & 1;
    const int64_t ne = (int64_t)*(volatile unsigned long long *)(A.ne + cur);
    const int2 *E = A.E[cur];
    if (first_pass) {  // ---- P1 of the first tail level: intra-group edges -> node hashes ----
      bool hit = false;
      for (int64_t e = gtid; e < ne; e += gstride) {
        const int2 uv = E[e];
        const int gu = uv.x / gs, gv = uv.y / gs;
        if (gu == gv) {
          atomicOr(A.h + uv.x, 1u << (uv.y - gv * gs));
          atomicOr(A.h + uv.y, 1u << (uv.x - gu * gs));
          hit = true;
        }
      }
      if (__any_sync(FULL_MASK, hit) && lane == 0) atomicOr(A.ctrl + fl, 1);
      gsync();
      first_pass = false;
    }
    if (*(volatile int *)(A.ctrl + fl) == 0) {  // no merge possible: this pass is the fixpoint
      if (gtid == 0) {
        if (level <= 64) A.level_n[level - 1] = n;
        A.ctrl[2] = level;
        A.nvals[0] = n;
      }
      break;
    }
    // ---- P2: Alg S1/S2 per tile (closure, election, tile-local rank); clears the hashes ----
    unsigned long long *tr = (A.trace && level <= 64 && blockIdx.x == 0 && threadIdx.x == 0) ? A.trace + 8 * (level - 1) : nullptr;
    if (tr) tr[0] = gtimer();
    const int64_t ntiles = (n + TN - 1) / TN;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      // a warp takes TAIL_SUB consecutive blocks of gpw groups (all hashes loaded up front)
      int64_t v[TAIL_SUB];
      bool active[TAIL_SUB];
      uint32_t hv[TAIL_SUB];
#pragma unroll
      for (int r = 0; r < TAIL_SUB; ++r) {
        v[r] = (((t * TAIL_WARPS + w) * TAIL_SUB + r) * geo.gpw + gin) * gs + lig;
        active[r] = (gin < geo.gpw) && (v[r] < n);
        hv[r] = active[r] ? (1u << lig) | A.h[v[r]] : 0u;
      }
      int local[TAIL_SUB], wcount = 0;
#pragma unroll
      for (int r = 0; r < TAIL_SUB; ++r) {
        if (active[r]) A.h[v[r]] = 0u;
        uint32_t x = hv[r];
        // most groups of the later levels have no intra-group edge: every lane is its own
        // component and the closure is the identity -- skip it warp-uniformly
        const unsigned nonisol = __ballot_sync(FULL_MASK, active[r] && x != (1u << lig));
        if (nonisol) {
          if (gs == 32) {  // Warshall over the non-isolated lanes only (an isolated vertex joins nothing)
            for (unsigned m = nonisol; m; m &= m - 1u) {
              const int k = __ffs(m) - 1;
              const uint32_t tt = __shfl_sync(FULL_MASK, x, k);
              if ((x >> k) & 1u) x |= tt;
            }
          } else {
            for (int k = 0; k < gs; ++k) {
              const uint32_t tt = __shfl_sync(FULL_MASK, x, (base_lane + k) & 31);
              if ((x >> k) & 1u) x |= tt;
            }
          }
        }
        const bool elected = active[r] && ((x & ((1u << lig) - 1u)) == 0u);
        const unsigned bal = __ballot_sync(FULL_MASK, elected);
        const unsigned gelect = (bal >> base_lane) & geo.gmask;
        const int first = active[r] ? __ffs(x) - 1 : 0;
        local[r] = wcount + __popc(gelect & ((1u << first) - 1u)) + __popc(bal & ((1u << base_lane) - 1u));
        wcount += __popc(bal);
      }
      if (lane == 0) s_w[w] = wcount;
      __syncthreads();
      if (w == 0) {
        const int c = s_w[lane];
        const int ci = warp_incl_scan(c);
        s_w[lane] = ci - c;
        if (lane == 31) A.tcount[t] = ci;
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < TAIL_SUB; ++r)
        if (active[r]) A.mk[v[r]] = s_w[w] + local[r];
      __syncthreads();
    }
    if (tr) tr[1] = gtimer();
    gsync();
    if (tr) tr[2] = gtimer();
    // ---- P3: scan the tile counts (every CTA, shared memory), remap, compose, reset ----
    {
      const int64_t per = (ntiles + TAIL_THREADS - 1) / TAIL_THREADS;
      const int64_t t0 = threadIdx.x * per, t1 = min(ntiles, t0 + per);
      int sum = 0;
      for (int64_t t = t0; t < t1; ++t) sum += A.tcount[t];
      const int wi = warp_incl_scan(sum);
      if (lane == 31) s_red[w] = wi;
      __syncthreads();
      if (w == 0) {
        const int c = s_red[lane];
        s_red[lane] = warp_incl_scan(c) - c;
      }
      __syncthreads();
      int run = s_red[w] + wi - sum;
      for (int64_t t = t0; t < t1; ++t) {
        s_pref[t] = run;
        run += A.tcount[t];
      }
      if (threadIdx.x == TAIL_THREADS - 1) s_total = run;
      __syncthreads();
    }
    const int64_t n2 = s_total;
    if (tr) tr[3] = gtimer();
    bool hit = false;
    // remap in place (each edge is read and written by one thread): a merged edge becomes dead
    // (-1, -1) instead of being compacted away -- no CTA-wide compaction (two barriers and a
    // global atomic) on the per-level critical path; later levels skip dead entries
    int2 *Ew = A.E[cur];
    for (int64_t e = gtid; e < ne; e += gstride) {
      const int2 uv = E[e];
      if (uv.x < 0) continue;
      int2 o;
      o.x = s_pref[uv.x / TN] + A.mk[uv.x];
      o.y = s_pref[uv.y / TN] + A.mk[uv.y];
      const bool keep = o.x != o.y;
      if (keep && o.x / gs == o.y / gs) {  // P1 of the next level
        atomicOr(A.h + o.x, 1u << (o.y - (o.y / gs) * gs));
        atomicOr(A.h + o.y, 1u << (o.x - (o.x / gs) * gs));
        hit = true;
      }
      Ew[e] = keep ? o : make_int2(-1, -1);
      if (A.trace && keep && level <= 64) atomicAdd(A.trace + 8 * (level - 1) + 7, 1ull);  // live edges
    }
    if (__any_sync(FULL_MASK, hit) && lane == 0) atomicOr(A.ctrl + (1 - fl), 1);
    if (tr) tr[4] = gtimer();
    for (int64_t c = gtid; c < n1; c += 2 * gstride) {  // two independent gathers in flight
      const int64_t c1 = c + gstride;
      const bool two = c1 < n1;
      const int32_t u0 = level == 2 ? (int32_t)c : A.comp[c];
      const int32_t u1 = !two ? 0 : level == 2 ? (int32_t)c1 : A.comp[c1];
      const int32_t m0 = A.mk[u0];
      const int32_t m1 = two ? A.mk[u1] : 0;
      A.comp[c] = s_pref[u0 / TN] + m0;
      if (two) A.comp[c1] = s_pref[u1 / TN] + m1;
    }
    composed = true;
    if (gtid == 0) {
      A.ctrl[fl] = 0;
      A.ctrl[3] = 1;
      if (level <= 64) A.level_n[level - 1] = n2;
    }
    if (tr) tr[5] = gtimer();
    gsync();
    if (tr) tr[6] = gtimer();
    n = n2;
    if (A.max_levels > 0 && level >= A.max_levels) {
      if (gtid == 0) {
        A.ctrl[2] = level;
        A.nvals[0] = n;
      }
      break;
    }
  }
  apply(composed);  // the last composition is behind a grid barrier
}

// map[f] = comp[map[f]] if any tail level merged
// map[f] = level-0 id (tile-relative value + tile prefix), then comp[] if any tail level merged
__global__ void k_apply(int64_t n, int32_t *__restrict__ map, const int32_t *__restrict__ comp,
                        const int *__restrict__ ctrl, const int64_t *__restrict__ tpref, int tn0, int64_t tiles0,
                        long long *n1_out) {
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n1_out && f == 0) *n1_out = tpref[tiles0];  // no tail launched (max_levels == 1)
  if (f < n) {
    const int g = (int)(map[f] + tpref[f / tn0]);
    map[f] = ctrl[3] ? comp[g] : g;
  }
}

// Aggregate sizes: histogram of the final map with warp-aggregated atomics.
__global__ void k_histogram(int64_t n, const int32_t *__restrict__ map, int32_t *__restrict__ cnt) {
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int key = f < n ? map[f] : -1;
  unsigned peers = __match_any_sync(FULL_MASK, key);
  if (key >= 0 && (__ffs(peers) - 1) == lane_id()) atomicAdd(cnt + key, __popc(peers));
}

struct MapScalars {
  long long nvals[2];
  unsigned long long cross;  // level-0 cross edges
  unsigned long long ne[2];
  int ctrl[4];
  long long level_n[64];
  unsigned bar;              // k_tail software grid barrier (zeroed with the struct)
  unsigned pad;
};

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
  cudaStream_t s0 = h->stream;
  GroupGeom geo;
  geo.gs = group_size;
  geo.gpw = 32 / group_size;
  geo.gmask = group_size == 32 ? 0xffffffffu : ((1u << group_size) - 1u);
  const int64_t tiles0 =
      std::max<int64_t>(1, cdiv(cdiv(N, (int64_t)geo.gpw * geo.gs), (int64_t)MAP_WARPS * L0_CHUNKS));
  const int64_t ecap = mesh->nnz_adj / 2 + 1;

  WS(h, sc, MapScalars, "map_scalars", 1);
  WS(h, tcnt, int32_t, "map_tile_cnt", tiles0 + 2);
  WS(h, tpref, int64_t, "map_tile_pref", tiles0 + 1);
  WS(h, cross, int2, "map_cross", ecap);
  CU_TRY(h, cudaMemsetAsync(sc, 0, sizeof(MapScalars), s0));
  int *tile_counter = (int *)(tcnt + tiles0 + 1);
  CU_TRY(h, cudaMemsetAsync(tile_counter, 0, sizeof(int), s0));
  const int tn0 = MAP_WARPS * L0_CHUNKS * geo.gpw * geo.gs;  // fine nodes per k_level0 tile

  // ---- level 0: warp-per-group hashing over the fine mesh (fused look-back scan) ----
  std::unique_ptr<ProfScope> ps_l0(new ProfScope(h, PROF_MAP_LEVEL0, s0));
  LAUNCH(h, k_level0, (unsigned)tiles0, MAP_THREADS, 0, N, geo, mesh->adj_ptr, mesh->adj_nbr, slot_tags, map, cross,
         &sc->cross, tcnt, tile_counter);
  agipc_status sst = scan_exclusive_i64(h, SCAN_SRC_I32, tcnt, tiles0, tpref);  // O[g] over the tiles
  if (sst != AGIPC_OK) return sst;

  ps_l0.reset();
  // ---- levels >= 1: one cooperative persistent kernel ----
  std::unique_ptr<ProfScope> ps_tail;
  if (max_levels != 1) {
    WS(h, EA, int2, "map_EA", ecap);
    WS(h, EB, int2, "map_EB", ecap);
    WS(h, used, unsigned long long, "map_used", ecap);
    WS(h, hh, uint32_t, "map_h", N);
    WS(h, mk, int32_t, "map_mk", N);
    WS(h, comp, int32_t, "map_comp", N);
    const int tile_nodes = TAIL_WARPS * TAIL_SUB * geo.gpw * geo.gs;
    const int64_t tiles_max = cdiv(N, tile_nodes) + 1;
    WS(h, tcount, int32_t, "map_tcount", tiles_max);
    // hash set for the level-1 edge de-duplication (zeroed once; used slots are cleared after use)
    int64_t tsize = 1024;
    while (tsize < 2 * ecap) tsize <<= 1;
    unsigned long long *table = nullptr;
    {
      bool fresh = false;
      agipc_status wst;
      table = (unsigned long long *)ws_get(h, "map_hash", sizeof(unsigned long long) * (size_t)tsize, &wst, &fresh);
      if (wst != AGIPC_OK) return wst;
      if (fresh) CU_TRY(h, cudaMemsetAsync(table, 0, h->ws["map_hash"].bytes, s0));
    }
    CU_TRY(h, cudaMemsetAsync(hh, 0, sizeof(uint32_t) * N, s0));
#ifndef CROSS_GRID
#define CROSS_GRID 8  // CTAs per SM of the level-1 edge de-duplication
#endif
    const unsigned gedge = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(ecap, 256), CROSS_GRID * h->sm_count));
    LAUNCH(h, k_cross_to_level1, gedge, 256, 0, cross, &sc->cross, map, table, (unsigned long long)(tsize - 1), EA,
           &sc->ne[0], used, (const int64_t *)tpref, tn0, tiles0, &sc->nvals[0]);
    TailArgs A;
    A.geo = geo;
    A.max_levels = max_levels;
    A.N = N;
    A.tile_nodes = tile_nodes;
    A.E[0] = EA;
    A.E[1] = EB;
    A.ne = sc->ne;
    A.h = hh;
    A.mk = mk;
    A.comp = comp;
    A.tcount = tcount;
    A.ctrl = sc->ctrl;
    A.nvals = sc->nvals;
    A.level_n = sc->level_n;
    static const bool trace_on = getenv("AGIPC_TAIL_TRACE") != nullptr;
    unsigned long long *trace = nullptr;
    if (trace_on) {
      WS(h, trw, unsigned long long, "map_tail_trace", 8 * 64);
      CU_TRY(h, cudaMemsetAsync(trw, 0, sizeof(unsigned long long) * 8 * 64, s0));
      trace = trw;
    }
    A.trace = trace;
    A.table = table;
    A.used = used;
    A.map = map;
    A.n_fine = N;
    A.tpref = tpref;
    A.tn0 = tn0;
    const size_t smem = sizeof(int32_t) * (size_t)tiles_max;
    if (smem > 200 * 1024) return set_err(h, AGIPC_ERANGE, "build_map: %lld nodes exceed the tail kernel", (long long)N);
    if (smem > h->tail_smem) {  // host-side attribute + residency check once per size (they cost
      // tens of microseconds of host time while the GPU waits for the cooperative launch)
      const size_t want = std::max(smem, (size_t)16 * 1024);
      CU_TRY(h, cudaFuncSetAttribute(k_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want));
      int occ = 0;
      CU_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tail, TAIL_THREADS, want));
      if (occ < 1) return set_err(h, AGIPC_ECUDA, "build_map: tail kernel cannot be resident");
      h->tail_smem = want;
    }
    const int grid = h->sm_count;  // one CTA per SM: cheap grid barriers
    void *args[] = {&A};
    cudaError_t pre = cudaGetLastError();
    if (pre != cudaSuccess) return set_err(h, AGIPC_ECUDA, "pending CUDA error before k_tail: %s", cudaGetErrorString(pre));
    static const bool coop = getenv("AGIPC_TAIL_COOP") && atoi(getenv("AGIPC_TAIL_COOP")) != 0;
    if (coop) {
      A.bar = nullptr;
      ps_tail.reset(new ProfScope(h, PROF_MAP_TAIL, s0));
      CU_TRY(h, cudaLaunchCooperativeKernel((const void *)k_tail, grid, TAIL_THREADS, args, smem, s0));
      h->launches += 1;
    } else {  // ordinary launch, software grid barrier (every CTA resident: 1 per SM, checked above)
      A.bar = (unsigned *)&sc->bar;
      ps_tail.reset(new ProfScope(h, PROF_MAP_TAIL, s0));
      LAUNCH(h, k_tail, (unsigned)grid, TAIL_THREADS, smem, A);
    }
    ps_tail.reset();  // (k_tail also cleared the hash slots and finished the fine map)
  } else {  // level 0 only: the tile prefixes still have to be added
    LAUNCH(h, k_apply, (unsigned)cdiv(N, 256), 256, 0, N, map, (const int32_t *)nullptr, sc->ctrl,
           (const int64_t *)tpref, tn0, tiles0, &sc->nvals[0]);
  }
  if (agg_size) {
    CU_TRY(h, cudaMemsetAsync(agg_size, 0, sizeof(int32_t) * N, s0));
    LAUNCH(h, k_histogram, (unsigned)cdiv(N, 256), 256, 0, N, map, agg_size);
  }
  agipc_status st;
  MapScalars *hs = (MapScalars *)pinned_get(h, sizeof(MapScalars), &st);
  if (st != AGIPC_OK) return st;
  CU_TRY(h, cudaMemcpyAsync(hs, sc, sizeof(MapScalars), cudaMemcpyDeviceToHost, s0));
  CU_TRY(h, host_wait(h, s0));
  if (h->trace) trace_mark(h, "@build_map_synced");
  if (getenv("AGIPC_TAIL_TRACE") && max_levels != 1) {  // per-phase time of the tail levels (CTA 0)
    unsigned long long t[8 * 64];
    if (cudaMemcpy(t, h->ws["map_tail_trace"].ptr, sizeof(t), cudaMemcpyDeviceToHost) == cudaSuccess) {
      double acc[6] = {0, 0, 0, 0, 0, 0};
      int nl = 0;
      for (int lv = 0; lv < 64; ++lv) {
        const unsigned long long *r = t + 8 * lv;
        if (!r[0] || !r[6]) continue;
        ++nl;
        for (int k = 0; k < 6; ++k) acc[k] += 1e-3 * (double)(r[k + 1] - r[k]);
      }
      fprintf(stderr, "libagipc[tail-trace] live edges per level:");
      for (int lv = 0; lv < 64; ++lv)
        if (t[8 * lv + 6]) fprintf(stderr, " %llu", t[8 * lv + 7]);
      fprintf(stderr, "\n");
      fprintf(stderr, "libagipc[tail-trace] levels %d, mean us per level: P2 closure %.2f | barrier %.2f | "
              "tile scan %.2f | edges %.2f | compose %.2f | barrier %.2f\n", nl, acc[0] / nl, acc[1] / nl,
              acc[2] / nl, acc[3] / nl, acc[4] / nl, acc[5] / nl);
    }
  }
  info->n_cross_edges = (int64_t)hs->cross;
  info->n_coarse = hs->nvals[0];
  if (max_levels == 1) {
    info->n_levels = 1;
    info->level_n[0] = hs->nvals[0];
  } else {
    info->n_levels = hs->ctrl[2];
    for (int l = 0; l < std::min(info->n_levels, 64); ++l) info->level_n[l] = hs->level_n[l];
  }
  return AGIPC_OK;
}
