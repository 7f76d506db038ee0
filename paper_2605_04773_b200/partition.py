"""Host-side partitioning for the multi-GPU path.

Rank r owns the contiguous global node range [bounds[r], bounds[r+1]) (the north star's
"partitioned ... by contiguous node groups": super-nodes never cross a rank because the
recursion of step 2 is rank-local, reading R24).  Its LOCAL mesh numbers the owned nodes
0..n_own-1 in global order, then the ghost nodes (non-owned nodes of the tets that touch an
owned node) n_own.. in ascending global id, so the ghosts of one peer form one contiguous
range.

  * ghosts      non-owned vertices of those tets and non-owned columns of the owned rows of the
                fine Hessian (contact couplings, C4);
  * tets        every tet with at least one owned vertex (boundary tets are evaluated on both
                sides); tet_slots is -1 for an edge that is not owned at both ends, so tags are
                written only into owned rows and cross-rank edges never merge;
  * adjacency   rows of owned nodes, owned neighbours only (what step 2 sees);
  * H_loc       fine BSR rows = owned nodes, columns = owned nodes (adjacency + diagonal);
  * H_halo      the same rows, columns = ghost index g (local id n_own + g);
  * halo        per peer q: recv = ghost range of q, send = the owned nodes q holds as ghosts
                (ordered like q's ghost range, i.e. by global id).

This is set-up logic (once per mesh), plain numpy, not a step of the hot path."""
from __future__ import annotations

import dataclasses

import numpy as np

TET_EDGES = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))


@dataclasses.dataclass
class LocalMesh:
    rank: int
    n_own: int
    n_ghost: int
    gid: np.ndarray          # int64 [n_own+n_ghost] global id of every local node
    X: np.ndarray            # float64 [n_own+n_ghost,3]
    tets: np.ndarray         # int32 [T,4] local ids
    tet_slots: np.ndarray    # int32 [T,12] local adjacency slot or -1
    adj_ptr: np.ndarray      # int64 [n_own+1]
    adj_nbr: np.ndarray      # int32 owned neighbours
    bsr_ptr: np.ndarray      # int64 [n_own+1]  H_loc
    bsr_col: np.ndarray      # int32
    loc_src: np.ndarray      # int64 source block (in the generating mesh's BSR) of every H_loc block
    hbsr_ptr: np.ndarray     # int64 [n_own+1]  H_halo
    hbsr_col: np.ndarray     # int32 ghost index
    halo_src: np.ndarray     # int64 source block of every H_halo block
    ghost_owner: np.ndarray  # int32 [n_ghost]
    peers: list              # ranks with a nonempty recv or send list, ascending
    recv_ptr: dict           # peer -> (g0, g1) ghost index range
    send_idx: dict           # peer -> int32 owned local ids (filled by attach_halo)
    slot_src: np.ndarray     # int64 [nnz_adj] source adjacency slot (generating mesh) of each local slot

    @property
    def n_nodes(self):
        return self.n_own


def owner_of(gids, bounds):
    return (np.searchsorted(np.asarray(bounds, np.int64), np.asarray(gids, np.int64), side="right") - 1).astype(np.int32)


def local_mesh(mesh, gid, lo, hi, bounds, rank) -> LocalMesh:
    """Local mesh of the rank owning global ids [lo, hi) from a mesh that contains all of its
    tets (the global mesh, or a sub-box around the slab).  `gid` maps mesh nodes to global
    ids and must be ascending.  Halo send lists are left empty (attach_halo fills them)."""
    gid = np.asarray(gid, np.int64)
    Nm = gid.shape[0]
    own = (gid >= lo) & (gid < hi)
    tet_own = own[mesh.tets].any(axis=1)
    tets_m = mesh.tets[tet_own]
    used = np.zeros(Nm, bool)
    used[tets_m.ravel()] = True
    used |= own
    # Hessian-only couplings of owned rows (contact blocks, C4) also need their columns
    brow_all = np.repeat(np.arange(Nm), np.diff(mesh.bsr_ptr))
    used[mesh.bsr_col[own[brow_all]]] = True
    ghost = used & ~own
    own_idx = np.nonzero(own)[0]
    ghost_idx = np.nonzero(ghost)[0]   # ascending mesh id == ascending gid
    n_own, n_ghost = own_idx.shape[0], ghost_idx.shape[0]
    loc_of = np.full(Nm, -1, np.int64)
    loc_of[own_idx] = np.arange(n_own)
    loc_of[ghost_idx] = n_own + np.arange(n_ghost)
    tets = loc_of[tets_m].astype(np.int32)
    # adjacency: owned rows, owned neighbours (mesh adjacency is ascending per row)
    rows_m = np.repeat(np.arange(Nm), np.diff(mesh.adj_ptr))
    keep = own[rows_m] & own[mesh.adj_nbr]
    slot_src = np.nonzero(keep)[0].astype(np.int64)
    r_loc = loc_of[rows_m[keep]]
    adj_nbr = loc_of[mesh.adj_nbr[keep]].astype(np.int32)
    adj_ptr = np.zeros(n_own + 1, np.int64)
    np.cumsum(np.bincount(r_loc, minlength=n_own), out=adj_ptr[1:])
    # tet slots: (u->v) exists locally iff both ends are owned.  The local slots are the kept
    # global slots in order, so a mesh tet-slot table translates by the rank of each kept slot
    # (checked edge by edge; otherwise the slots are found by search)
    ts = np.full((tets.shape[0], 12), -1, np.int32)
    if not _translate_tet_slots(mesh, tet_own, tets, n_own, rows_m, keep, ts):
        key = r_loc * (n_own + 1) + adj_nbr
        for e, (a, b) in enumerate(TET_EDGES):
            u = tets[:, a].astype(np.int64)
            v = tets[:, b].astype(np.int64)
            ok = (u < n_own) & (v < n_own)
            for col, (x, y) in ((2 * e, (u, v)), (2 * e + 1, (v, u))):
                q = x[ok] * (n_own + 1) + y[ok]
                pos = np.searchsorted(key, q)
                assert np.all(key[np.minimum(pos, key.shape[0] - 1)] == q)
                ts[np.nonzero(ok)[0], col] = pos
    # fine BSR split into owned / ghost columns
    brow = np.repeat(np.arange(Nm), np.diff(mesh.bsr_ptr))
    bo = own[brow]
    lc = loc_of[mesh.bsr_col]
    kl = bo & own[mesh.bsr_col]
    kh = bo & ghost[mesh.bsr_col]
    loc_src = np.nonzero(kl)[0].astype(np.int64)
    halo_src = np.nonzero(kh)[0].astype(np.int64)
    bsr_ptr = np.zeros(n_own + 1, np.int64)
    np.cumsum(np.bincount(loc_of[brow[kl]], minlength=n_own), out=bsr_ptr[1:])
    hbsr_ptr = np.zeros(n_own + 1, np.int64)
    np.cumsum(np.bincount(loc_of[brow[kh]], minlength=n_own), out=hbsr_ptr[1:])
    bsr_col = lc[kl].astype(np.int32)
    hbsr_col = (lc[kh] - n_own).astype(np.int32)
    ghost_owner = owner_of(gid[ghost_idx], bounds)
    recv_ptr = {}
    for q in np.unique(ghost_owner).tolist():
        sel = np.nonzero(ghost_owner == q)[0]
        recv_ptr[int(q)] = (int(sel[0]), int(sel[-1]) + 1)
    lid = np.concatenate([own_idx, ghost_idx])
    return LocalMesh(rank=rank, n_own=n_own, n_ghost=n_ghost, gid=gid[lid], X=np.ascontiguousarray(mesh.X[lid]),
                     tets=tets, tet_slots=ts, adj_ptr=adj_ptr, adj_nbr=adj_nbr, bsr_ptr=bsr_ptr, bsr_col=bsr_col,
                     loc_src=loc_src, hbsr_ptr=hbsr_ptr, hbsr_col=hbsr_col, halo_src=halo_src,
                     ghost_owner=ghost_owner, peers=sorted(recv_ptr), recv_ptr=recv_ptr, send_idx={},
                     slot_src=slot_src)


def _translate_tet_slots(mesh, tet_own, tets, n_own, rows_m, keep, ts) -> bool:
    """ts[:, col] = local slot of the mesh's tet slot when both ends are owned.  Returns False
    (ts untouched) if the mesh has no complete tet-slot table in TET_EDGES order."""
    mts = getattr(mesh, "tet_slots", None)
    if mts is None or mts.shape[1] != 12:
        return False
    mts = mts[tet_own]
    if mts.shape[0] != tets.shape[0] or np.any(mts < 0):
        return False
    rank_of = np.cumsum(keep, dtype=np.int64) - 1
    # convention check on (up to) 65536 evenly spaced tets: column 2e is u->v of TET_EDGES[e]
    smp = np.unique(np.linspace(0, mts.shape[0] - 1, min(mts.shape[0], 65536)).astype(np.int64))
    tm = mesh.tets[np.nonzero(tet_own)[0][smp]]
    out = np.full_like(ts, -1)
    for e, (a, b) in enumerate(TET_EDGES):
        ok = (tets[:, a] < n_own) & (tets[:, b] < n_own)
        for col, (x, y) in ((2 * e, (a, b)), (2 * e + 1, (b, a))):
            g = mts[:, col]
            gs = g[smp].astype(np.int64)
            if not (np.array_equal(rows_m[gs], tm[:, x]) and np.array_equal(mesh.adj_nbr[gs], tm[:, y])):
                return False
            out[ok, col] = rank_of[g[ok]]
    ts[:] = out
    return True


def send_lists_from_requests(lm: LocalMesh, requests: dict):
    """requests[q] = global ids (ascending) that peer q holds as ghosts owned by this rank.
    Returns peer -> owned local ids in the same order."""
    out = {}
    lo = int(lm.gid[0]) if lm.n_own else 0
    for q, g in requests.items():
        g = np.asarray(g, np.int64)
        if g.size:
            loc = g - lo
            assert np.all((loc >= 0) & (loc < lm.n_own)) and np.all(lm.gid[loc] == g)
            out[int(q)] = loc.astype(np.int32)
    return out


def attach_halo(lms):
    """Single-process helper: fill every rank's send lists from the others' ghost ranges."""
    for lm in lms:
        req = {}
        for other in lms:
            if other.rank != lm.rank and lm.rank in other.recv_ptr:
                g0, g1 = other.recv_ptr[lm.rank]
                req[other.rank] = other.gid[other.n_own + g0:other.n_own + g1]
        lm.send_idx = send_lists_from_requests(lm, req)
        lm.peers = sorted(set(lm.peers) | set(lm.send_idx))
    return lms


def exchange_requests(lm: LocalMesh, world: int, exchange):
    """Distributed variant of attach_halo.  `exchange(send: dict[int, np.ndarray]) -> dict` is the
    communicator's all-to-all of int64 arrays (paper_2605_04773_b200.dist.Comm.alltoall_i64)."""
    send = {}
    for q, (g0, g1) in lm.recv_ptr.items():
        send[q] = lm.gid[lm.n_own + g0:lm.n_own + g1]
    got = exchange(send)
    lm.send_idx = send_lists_from_requests(lm, got)
    lm.peers = sorted(set(lm.peers) | set(lm.send_idx))
    return lm


def slab_bounds(n: int, R: int, t: int | None = None):
    """Owned global id ranges of R slabs of n x n x t nodes (t = n: cubes)."""
    t = n if t is None else t
    return [r * n * n * t for r in range(R + 1)]
