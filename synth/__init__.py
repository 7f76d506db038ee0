"""Seeded synthetic inputs for the AGIPC coarsening path.

This module is the ONLY code shared by the CPU oracle (``oracle/``) and the
CUDA path (``paper_2605_04773_b200``).  It holds none of the method's
arithmetic: no Green strain, no tags derived from strain, no hashing, no
Galerkin products, no PCG.  It only builds the *inputs* the paper's problem
statement takes (Alg 1 lines 8-10):

* a static tetrahedral fine mesh (Kuhn 6-tet subdivision of an n^3 grid,
  centred on the origin, nodes in Morton order -- a stand-in for the METIS
  ordering of P:226), its symmetric CSR adjacency and the tet->directed-slot
  table ("the edge-element adjacency can be precomputed");
* iterates x_{i-1}, x_i (twist, walls) for the strain criterion;
* the fine Hessian H_f = M (x) I_3 + dt^2 K_lin in full-storage BSR and a
  gradient g_f (the paper's H(x), grad E(x) of Eq. 2; H is SPD);
* Bernoulli edge tags for map-only workloads.

Recipe: side 1 m, rho = 1000,
nu = 0.3, dt = 0.01, E per config, g_f ~ N(0,1).
"""
from __future__ import annotations

import ctypes as _C
import dataclasses
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_GEN_SRC = os.path.join(_HERE, "_gen.c")
_GEN_LIB = os.path.join(_HERE, "libsynthgen.so")
_gen = None


def build(force: bool = False) -> str:
    """Compile the fast input generator (_gen.c, gcc + OpenMP).  Input generation only."""
    if force or not os.path.exists(_GEN_LIB) or os.path.getmtime(_GEN_LIB) < os.path.getmtime(_GEN_SRC):
        tmp = _GEN_LIB + ".%d.tmp" % os.getpid()
        subprocess.check_call(["gcc", "-O3", "-std=gnu99", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", tmp, _GEN_SRC, "-lm"])
        os.replace(tmp, _GEN_LIB)
    return _GEN_LIB


def _lib():
    global _gen
    if _gen is None:
        build()
        L = _C.CDLL(_GEN_LIB)
        P, i64, f64 = _C.c_void_p, _C.c_int64, _C.c_double
        L.syn_kuhn_grid.argtypes = [i64, f64, f64, f64, f64, i64, i64, i64] + [P] * 11
        L.syn_kuhn_grid.restype = _C.c_int
        L.syn_fine_hessian.argtypes = [i64, i64, P, P, P, f64, f64, f64, f64, _C.c_int, _C.c_int, P, P, P, P]
        L.syn_fine_hessian.restype = i64
        L.syn_merge_pattern.argtypes = [i64, P, P, i64, P, P, P, P]
        L.syn_merge_pattern.restype = i64
        L.syn_bsr_slots.argtypes = [i64, P, P, P, P, P]
        L.syn_bsr_slots.restype = None
        _gen = L
    return _gen


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_C.c_void_p)

__all__ = [
    "Mesh", "kuhn_grid", "mesh_from_tets", "stiffness_blocks", "fine_hessian",
    "fine_gradient", "twist", "walls", "random_tags", "edge_tags_to_slots",
    "config_c1", "config_c2", "config_c3",
]

# Local edge order of a tet (a,b,c,d) = nodes 0..3.  tet_slots[t, 2e] is the
# CSR slot of the directed edge (u->v), tet_slots[t, 2e+1] that of (v->u).
TET_EDGES = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))


@dataclasses.dataclass
class Mesh:
    """Static fine mesh.  All index arrays are C-contiguous numpy arrays."""
    X: np.ndarray            # float64 [N,3] rest positions
    tets: np.ndarray         # int32  [T,4]
    adj_ptr: np.ndarray      # int64  [N+1]  symmetric adjacency, ascending
    adj_nbr: np.ndarray      # int32  [2E]
    tet_slots: np.ndarray    # int32  [T,12] directed CSR slot per tet edge
    edges: np.ndarray        # int32  [E,2] canonical (min,max), ascending
    edge_of_slot: np.ndarray  # int64 [2E] undirected edge id of each slot
    bsr_ptr: np.ndarray      # int64  [N+1] fine Hessian pattern (adjacency + diagonal)
    bsr_col: np.ndarray      # int32  [N+2E]
    diag_slot: np.ndarray    # int64  [N] BSR slot of the diagonal block of each row
    ijk: np.ndarray | None = None  # int32 [N,3] grid coordinates (grid meshes)
    n_side: int = 0
    n_extra: int = 0         # BSR blocks beyond adjacency + diagonal (contact pairs, C4)

    @property
    def n_nodes(self) -> int:
        return int(self.X.shape[0])

    @property
    def n_tets(self) -> int:
        return int(self.tets.shape[0])

    @property
    def n_edges(self) -> int:
        return int(self.edges.shape[0])


def _morton_key(ijk: np.ndarray) -> np.ndarray:
    """3-D bit interleave of non-negative grid coordinates (x bit lowest)."""
    key = np.zeros(ijk.shape[0], dtype=np.int64)
    for bit in range(21):
        for d in range(3):
            key |= ((ijk[:, d].astype(np.int64) >> bit) & 1) << (3 * bit + d)
    return key


def mesh_from_tets(X: np.ndarray, tets: np.ndarray, ijk=None, n_side=0, extra_pairs=None) -> Mesh:
    """Build adjacency, tet->slot table and the fine BSR pattern from tets.  `extra_pairs`
    (int [P,2]) adds symmetric Hessian-only blocks (contact, C4) to the BSR pattern; they are
    not mesh edges (never tagged, not in the adjacency)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    tets = np.ascontiguousarray(tets, dtype=np.int32)
    N = X.shape[0]
    T = tets.shape[0]
    t64 = tets.astype(np.int64)
    if T:
        u = np.concatenate([t64[:, a] for a, b in TET_EDGES])
        v = np.concatenate([t64[:, b] for a, b in TET_EDGES])
    else:
        u = v = np.zeros(0, np.int64)
    lo = np.minimum(u, v)
    hi = np.maximum(u, v)
    ekey, inv = np.unique(lo * N + hi, return_inverse=True)
    inv = inv.reshape(-1)
    E = ekey.shape[0]
    edges = np.stack([ekey // N, ekey % N], axis=1).astype(np.int32)
    allk = np.concatenate([ekey, (ekey % N) * N + ekey // N])
    order = np.argsort(allk, kind="stable")
    dkey = allk[order]
    pos = np.empty(2 * E, np.int64)
    pos[order] = np.arange(2 * E)
    rows = dkey // N
    adj_nbr = (dkey % N).astype(np.int32)
    adj_ptr = np.zeros(N + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=N), out=adj_ptr[1:])
    # tet edge -> both directed slots
    fwd = pos[inv]            # slot of (lo -> hi)
    bwd = pos[E + inv]        # slot of (hi -> lo)
    s_uv = np.where(u < v, fwd, bwd).reshape(6, T)
    s_vu = np.where(u < v, bwd, fwd).reshape(6, T)
    ts = np.empty((T, 12), np.int32)
    ts[:, 0::2] = s_uv.T
    ts[:, 1::2] = s_vu.T
    edge_of_slot = np.where(order < E, order, order - E).astype(np.int64)
    # fine Hessian pattern: adjacency + diagonal, ascending columns
    gt = (adj_nbr > rows).astype(np.int64)
    nbelow = np.bincount(rows[adj_nbr < rows], minlength=N)
    bsr_ptr = adj_ptr + np.arange(N + 1, dtype=np.int64)
    bsr_col = np.empty(N + 2 * E, np.int32)
    bsr_col[np.arange(2 * E, dtype=np.int64) + rows + gt] = adj_nbr
    diag_slot = adj_ptr[:-1] + np.arange(N, dtype=np.int64) + nbelow
    bsr_col[diag_slot] = np.arange(N, dtype=np.int32)
    n_extra = 0
    if extra_pairs is not None and len(extra_pairs):
        ep = np.asarray(extra_pairs, np.int64)
        brow = np.repeat(np.arange(N, dtype=np.int64), np.diff(bsr_ptr))
        key = np.unique(np.concatenate([brow * N + bsr_col, ep[:, 0] * N + ep[:, 1], ep[:, 1] * N + ep[:, 0]]))
        n_extra = int(key.shape[0] - bsr_col.shape[0])
        bsr_col = (key % N).astype(np.int32)
        bsr_ptr = np.zeros(N + 1, np.int64)
        np.cumsum(np.bincount(key // N, minlength=N), out=bsr_ptr[1:])
        diag_slot = np.searchsorted(key, np.arange(N, dtype=np.int64) * (N + 1))
    return Mesh(X=X, tets=tets, adj_ptr=adj_ptr, adj_nbr=adj_nbr, tet_slots=ts,
                edges=edges, edge_of_slot=edge_of_slot, bsr_ptr=bsr_ptr, bsr_col=bsr_col,
                diag_slot=diag_slot,
                ijk=None if ijk is None else np.ascontiguousarray(ijk, np.int32), n_side=n_side, n_extra=n_extra)


def bsr_slot(mesh: Mesh, u, v) -> np.ndarray:
    """BSR slot of blocks (u, v) (general lookup; -1 if absent)."""
    u = np.ascontiguousarray(np.asarray(u, np.int64).reshape(-1))
    v = np.ascontiguousarray(np.asarray(v, np.int64).reshape(-1))
    out = np.empty(u.shape[0], np.int64)
    _lib().syn_bsr_slots(u.shape[0], _ptr(mesh.bsr_ptr), _ptr(mesh.bsr_col), _ptr(u), _ptr(v), _ptr(out))
    return out


def bsr_slot_py(mesh: Mesh, u, v) -> np.ndarray:
    """numpy version of bsr_slot (pins the fast one in tests/test_synth_fast.py)."""
    N = mesh.n_nodes
    brow = np.repeat(np.arange(N, dtype=np.int64), np.diff(mesh.bsr_ptr))
    key = brow * N + mesh.bsr_col
    q = np.asarray(u, np.int64) * N + np.asarray(v, np.int64)
    pos = np.searchsorted(key, q)
    ok = (pos < key.shape[0]) & (key[np.minimum(pos, key.shape[0] - 1)] == q)
    return np.where(ok, pos, -1)


def kuhn_grid(n: int, order: str = "morton", side: float = 1.0, origin=(0.0, 0.0, 0.0)) -> Mesh:
    """Kuhn/Freudenthal 6-tet subdivision of an n^3 node grid on a cube of the
    given side centred on ``origin``.  Each cube is split along its
    (0,0,0)-(1,1,1) diagonal into the 6 path tets.  Nodes are renumbered in
    Morton order (``order='morton'``) or kept lexicographic (``'lex'``); tets
    are sorted by their smallest node id (stable).  The Morton grid is built by the
    C generator (_gen.c, O(N), OpenMP); kuhn_grid_py is the numpy definition it is pinned to."""
    if order != "morton":
        return kuhn_grid_py(n, order, side, origin)
    assert n >= 2
    N, T = n ** 3, 6 * (n - 1) ** 3
    E = 3 * n * n * (n - 1) + 3 * n * (n - 1) ** 2 + (n - 1) ** 3
    X = np.empty((N, 3), np.float64)
    ijk = np.empty((N, 3), np.int32)
    tets = np.empty((T, 4), np.int32)
    adj_ptr = np.empty(N + 1, np.int64)
    adj_nbr = np.empty(2 * E, np.int32)
    ts = np.empty((T, 12), np.int32)
    edges = np.empty((E, 2), np.int32)
    eos = np.empty(2 * E, np.int64)
    bsr_ptr = np.empty(N + 1, np.int64)
    bsr_col = np.empty(N + 2 * E, np.int32)
    diag = np.empty(N, np.int64)
    o = [float(v) for v in origin]
    rc = _lib().syn_kuhn_grid(n, float(side), o[0], o[1], o[2], N, T, E, *[_ptr(a) for a in (
        X, ijk, tets, adj_ptr, adj_nbr, ts, edges, eos, bsr_ptr, bsr_col, diag)])
    if rc != 0:
        raise RuntimeError(f"syn_kuhn_grid({n}) failed: {rc}")
    return Mesh(X=X, tets=tets, adj_ptr=adj_ptr, adj_nbr=adj_nbr, tet_slots=ts, edges=edges, edge_of_slot=eos,
                bsr_ptr=bsr_ptr, bsr_col=bsr_col, diag_slot=diag, ijk=ijk, n_side=n)


def kuhn_grid_py(n: int, order: str = "morton", side: float = 1.0, origin=(0.0, 0.0, 0.0)) -> Mesh:
    """numpy definition of kuhn_grid (any order)."""
    assert n >= 2
    g = np.arange(n)
    I, J, K = np.meshgrid(g, g, g, indexing="ij")
    ijk = np.stack([I.ravel(), J.ravel(), K.ravel()], axis=1).astype(np.int64)
    lex = (ijk[:, 0] * n + ijk[:, 1]) * n + ijk[:, 2]
    if order == "morton":
        perm = np.argsort(_morton_key(ijk), kind="stable")  # new id -> lex id
    elif order == "lex":
        perm = np.arange(n ** 3)
    else:
        raise ValueError(order)
    new_of_lex = np.empty(n ** 3, np.int64)
    new_of_lex[lex[perm]] = np.arange(n ** 3)
    ijk_new = ijk[perm]
    X = ijk_new.astype(np.float64) * (side / (n - 1)) - 0.5 * side + np.asarray(origin, np.float64)
    # tets
    c = np.arange(n - 1)
    CI, CJ, CK = np.meshgrid(c, c, c, indexing="ij")
    cubes = np.stack([CI.ravel(), CJ.ravel(), CK.ravel()], axis=1)
    unit = np.eye(3, dtype=np.int64)
    tl = []
    for s0, s1, s2 in ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)):
        v0 = cubes
        v1 = v0 + unit[s0]
        v2 = v1 + unit[s1]
        v3 = v2 + unit[s2]
        tl.append(np.stack([(v[:, 0] * n + v[:, 1]) * n + v[:, 2] for v in (v0, v1, v2, v3)], axis=1))
    tets = new_of_lex[np.concatenate(tl, axis=0)]
    tets = tets[np.argsort(tets.min(axis=1), kind="stable")].astype(np.int32)
    return mesh_from_tets(X, tets, ijk=ijk_new, n_side=n)


# ----------------------------------------------------------------------------
# Fine Hessian input: H_f = M_lumped (x) I_3 + dt^2 K_lin   (SPD)
# ----------------------------------------------------------------------------

def lame(E: float, nu: float):
    mu = E / (2.0 * (1.0 + nu))
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    return mu, lam


def stiffness_blocks(X: np.ndarray, tets: np.ndarray, E: float, nu: float):
    """Per-tet linear-elastic (StVK at rest) stiffness blocks K_ab [T,4,4,3,3]
    and volumes [T]: K_ab = V (mu (g_a.g_b) I + mu g_b g_a^T + lam g_a g_b^T),
    g_a the P1 shape-function gradients.  Symmetrised so that K_ba = K_ab^T
    holds bit-exactly.  Input generation only (torch CPU ops for speed)."""
    import torch
    mu, lam = lame(E, nu)
    Xt = torch.from_numpy(np.ascontiguousarray(X, np.float64))
    tt = torch.from_numpy(np.ascontiguousarray(tets, np.int64))
    Xa = Xt[tt[:, 0]]
    Dm = torch.stack([Xt[tt[:, 1]] - Xa, Xt[tt[:, 2]] - Xa, Xt[tt[:, 3]] - Xa], dim=2)
    V = torch.linalg.det(Dm).abs() / 6.0
    Minv = torch.linalg.inv(Dm)            # rows = grad N_1..3
    g = torch.empty((tets.shape[0], 4, 3), dtype=torch.float64)
    g[:, 1:, :] = Minv
    g[:, 0, :] = -Minv.sum(dim=1)
    g *= V.sqrt()[:, None, None]           # fold V into both gradients
    gg = torch.matmul(g, g.transpose(1, 2))  # [T,a,b] = g_a . g_b
    K = g[:, None, :, :, None] * (mu * g[:, :, None, None, :])   # mu g_b g_a^T
    K += (lam * g[:, :, None, :, None]) * g[:, None, :, None, :]  # lam g_a g_b^T
    d = mu * gg
    for i in range(3):
        K[:, :, :, i, i] += d
    K = 0.5 * (K + K.permute(0, 2, 1, 4, 3))
    return K.numpy(), V.numpy()


def _slot_index(mesh: Mesh, t0: int, t1: int) -> np.ndarray:
    """BSR slot of every (tet, a, b) pair -> int64 [t1-t0,4,4].  A row of the
    BSR pattern is the adjacency row with the diagonal inserted, so
    bsr_slot(u->v) = adj_slot(u->v) + u + [v > u]."""
    tets = mesh.tets[t0:t1].astype(np.int64)
    if mesh.n_extra:  # the pattern is not adjacency + diagonal: general lookup
        u = np.repeat(tets, 4, axis=1).reshape(-1)
        v = np.tile(tets, (1, 4)).reshape(-1)
        return bsr_slot(mesh, u, v).reshape(tets.shape[0], 4, 4)
    ts = mesh.tet_slots[t0:t1].astype(np.int64)
    S = np.empty((tets.shape[0], 4, 4), np.int64)
    for k in range(4):
        S[:, k, k] = mesh.diag_slot[tets[:, k]]
    for e, (a, b) in enumerate(TET_EDGES):
        u, v = tets[:, a], tets[:, b]
        S[:, a, b] = ts[:, 2 * e] + u + (v > u)
        S[:, b, a] = ts[:, 2 * e + 1] + v + (u > v)
    return S


def fine_hessian(mesh: Mesh, E: float = 1e5, nu: float = 0.3, rho: float = 1000.0,
                 dt: float = 0.01, mass: bool = True, stiffness: bool = True) -> np.ndarray:
    """Values of H_f in the mesh's BSR pattern: float64 [nnzb, 3, 3] row-major
    blocks.  ``E`` may be a per-tet array (multi-material scenes).  C generator (_gen.c):
    row-centric sums over each node's tets in ascending tet order, so H is bitwise symmetric;
    fine_hessian_py is the numpy definition it is pinned to (equal within rounding)."""
    N, T = mesh.n_nodes, mesh.n_tets
    nnzb = mesh.bsr_col.shape[0]
    H = np.empty((nnzb, 3, 3), np.float64)
    Earr = None
    if np.ndim(E) > 0:
        Earr = np.ascontiguousarray(np.broadcast_to(np.asarray(E, np.float64), (T,)))
    miss = _lib().syn_fine_hessian(N, T, _ptr(mesh.tets), _ptr(mesh.X), _ptr(Earr), float(E) if Earr is None else 0.0,
                                   float(nu), float(rho), float(dt), int(bool(mass)), int(bool(stiffness)),
                                   _ptr(mesh.bsr_ptr), _ptr(mesh.bsr_col), _ptr(mesh.diag_slot), _ptr(H))
    if miss != 0:
        raise RuntimeError(f"fine_hessian: {miss} tet blocks missing from the BSR pattern")
    return H


def fine_hessian_py(mesh: Mesh, E: float = 1e5, nu: float = 0.3, rho: float = 1000.0,
                    dt: float = 0.01, mass: bool = True, stiffness: bool = True,
                    chunk: int = 1 << 18) -> np.ndarray:
    """numpy/torch-CPU definition of fine_hessian (scatter in tet order)."""
    import torch  # index_add_ is only used as a fast scatter for input generation
    N = mesh.n_nodes
    nnzb = mesh.bsr_col.shape[0]
    out = torch.zeros((nnzb, 9), dtype=torch.float64)
    T = mesh.n_tets
    Earr = np.broadcast_to(np.asarray(E, np.float64), (T,))
    mnode = np.zeros(N)
    for t0 in range(0, T, chunk):
        tt = mesh.tets[t0:t0 + chunk]
        Ech = Earr[t0:t0 + chunk]
        uniq = np.unique(Ech)
        K = np.empty((tt.shape[0], 4, 4, 3, 3))
        V = None
        for Ev in uniq:  # E enters linearly: compute with E=1 and scale
            sel = Ech == Ev
            Ks, Vs = stiffness_blocks(mesh.X, tt[sel], 1.0, nu)
            K[sel] = Ks * Ev
            if V is None:
                V = np.empty(tt.shape[0])
            V[sel] = Vs
        mnode += np.bincount(tt.ravel(), weights=np.repeat(rho * V / 4.0, 4), minlength=N)
        if stiffness:
            idx = torch.from_numpy(_slot_index(mesh, t0, t0 + tt.shape[0]).reshape(-1))
            src = torch.from_numpy((dt * dt) * K.reshape(-1, 9))
            out.index_add_(0, idx, src)
    if mass:
        dslot = mesh.diag_slot
        eye = torch.tensor([1.0, 0, 0, 0, 1.0, 0, 0, 0, 1.0], dtype=torch.float64)
        out[torch.from_numpy(dslot)] += torch.from_numpy(mnode)[:, None] * eye[None, :]
    return out.numpy().reshape(nnzb, 3, 3)


def lumped_mass(mesh: Mesh, rho: float = 1000.0) -> np.ndarray:
    Xa = mesh.X[mesh.tets[:, 0]]
    Dm = np.stack([mesh.X[mesh.tets[:, k]] - Xa for k in (1, 2, 3)], axis=2)
    V = np.abs(np.linalg.det(Dm)) / 6.0
    m = np.zeros(mesh.n_nodes)
    np.add.at(m, mesh.tets.ravel(), np.repeat(rho * V / 4.0, 4))
    return m


def fine_gradient(n_nodes: int, seed: int = 0) -> np.ndarray:
    """g_f ~ N(0, 1) per component, float64 [N,3]."""
    return np.random.default_rng([seed, 7]).standard_normal((n_nodes, 3))


# ----------------------------------------------------------------------------
# Iterates for the strain criterion
# ----------------------------------------------------------------------------

def _smoothstep(t):
    t = np.clip(t, 0.0, 1.0)
    return t * t * (3.0 - 2.0 * t)


def twist(X: np.ndarray, alpha: float, w: float = 0.2, axis=(0.0, 0.0, 1.0), center=(0.0, 0.0, 0.0)):
    """Rotate each node about ``axis`` through ``center`` by
    phi(s) = alpha * S(s/w + 1/2), s = axial coordinate, S = clamped smoothstep."""
    a = np.asarray(axis, np.float64)
    a = a / np.linalg.norm(a)
    c = np.asarray(center, np.float64)
    r = X - c
    s = r @ a
    phi = alpha * _smoothstep(s / w + 0.5)
    cos, sin = np.cos(phi)[:, None], np.sin(phi)[:, None]
    # Rodrigues: r cos + (a x r) sin + a (a.r)(1-cos)
    axr = np.cross(a[None, :], r)
    return c + r * cos + axr * sin + a[None, :] * s[:, None] * (1.0 - cos)


def walls(mesh: Mesh, k: int, period: int = 16, rel_amp: float = 1e-2, seed: int = 0):
    """x_prev = X; x_cur = X + delta*xi on wall nodes (any grid coordinate
    = k mod period), delta = rel_amp * h, xi ~ N(0, I3)."""
    assert mesh.ijk is not None
    h = 1.0 / (mesh.n_side - 1)
    wall = np.any(mesh.ijk % period == (k % period), axis=1)
    xi = np.random.default_rng([seed, 11, k]).standard_normal((mesh.n_nodes, 3))
    x_cur = mesh.X + (rel_amp * h) * xi * wall[:, None]
    return mesh.X.copy(), x_cur


def random_tags(mesh: Mesh, p: float, seed: int = 0) -> np.ndarray:
    """tau_e ~ Bernoulli(p) per undirected edge in canonical (min,max) order,
    returned per directed CSR slot (uint8 [2E], both directions equal)."""
    tau = (np.random.default_rng([seed, 3]).random(mesh.n_edges) < p).astype(np.uint8)
    return edge_tags_to_slots(mesh, tau)


def edge_tags_to_slots(mesh: Mesh, tau_edge: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(tau_edge, np.uint8)[mesh.edge_of_slot])


# ----------------------------------------------------------------------------
# Named configurations (BASELINE.json configs)
# ----------------------------------------------------------------------------

def config_c1(seed: int = 0, p: float = 0.2):
    """C1: 10^3 grid, random tags p, gs=32, E=1e5 (one Newton step)."""
    m = kuhn_grid(10)
    return dict(mesh=m, slot_tags=random_tags(m, p, seed), E=1e5, group_size=32,
                x_prev=twist(m.X, 0.5), x_cur=twist(m.X, 0.501), theta=5e-5)


def config_c2(n: int = 47):
    """C2: 47^3 = 103,823 nodes, twist 0.5 -> 0.501, theta = 5e-5, E=1e5."""
    m = kuhn_grid(n)
    return dict(mesh=m, x_prev=twist(m.X, 0.5), x_cur=twist(m.X, 0.501), theta=5e-5,
                E=1e5, group_size=32)


def config_c3(n: int = 100, k: int = 0):
    """C3: 100^3 = 1,000,000 nodes, strain walls with phase k, theta = 5e-5."""
    m = kuhn_grid(n)
    xp, xc = walls(m, k)
    return dict(mesh=m, x_prev=xp, x_cur=xc, theta=5e-5, E=1e5, group_size=32)


# ----------------------------------------------------------------------------
# Partitioned workloads: a box of n x n x (R n) nodes ordered
# slab-major (slab s = nodes with s n <= k < (s+1) n), Morton inside each slab,
# so rank r of R owns the contiguous global range [r n^3, (r+1) n^3).  With
# R = 1 this is exactly kuhn_grid(n).
# ----------------------------------------------------------------------------

def kuhn_box(n: int, slabs: int = 1, z_lo: int = 0, z_hi: int | None = None, side: float = 1.0,
             t: int | None = None):
    """Kuhn 6-tet grid over nodes (i, j, k), 0 <= i, j < n, z_lo <= k <= z_hi (default: the
    whole box, k < slabs*t) of `slabs` slabs of n x n x t nodes (t = n: cubes).  Returns
    (mesh, gid): gid[v] = global slab-major Morton id of local node v; local ids are ascending
    in gid (so a sub-box keeps the global order).  Spacing h = side/(n-1); the whole box is
    centred on the origin."""
    t = n if t is None else t
    nz = slabs * t
    z_hi = nz - 1 if z_hi is None else z_hi
    assert n >= 2 and t >= 1 and 0 <= z_lo < z_hi < nz
    h = side / (n - 1)
    gi = np.arange(n)
    gk = np.arange(z_lo, z_hi + 1)
    I, J, K = np.meshgrid(gi, gi, gk, indexing="ij")
    ijk = np.stack([I.ravel(), J.ravel(), K.ravel()], axis=1).astype(np.int64)
    s = ijk[:, 2] // t
    loc = ijk.copy()
    loc[:, 2] -= s * t
    gid_all = s * (n * n * t) + _morton_rank(n, t)[_morton_key(loc)]
    perm = np.argsort(gid_all, kind="stable")
    gid = gid_all[perm]
    ijk_new = ijk[perm]
    nzl = z_hi - z_lo + 1
    lex = ((ijk[:, 0] * n + ijk[:, 1]) * nzl + (ijk[:, 2] - z_lo))
    new_of_lex = np.empty(lex.shape[0], np.int64)
    new_of_lex[lex[perm]] = np.arange(lex.shape[0])
    X = ijk_new.astype(np.float64) * h
    X[:, 0:2] -= 0.5 * side
    X[:, 2] -= 0.5 * h * (nz - 1)
    c = np.arange(n - 1)
    ck = np.arange(nzl - 1)
    CI, CJ, CK = np.meshgrid(c, c, ck, indexing="ij")
    cubes = np.stack([CI.ravel(), CJ.ravel(), CK.ravel()], axis=1)
    unit = np.eye(3, dtype=np.int64)
    tl = []
    for s0, s1, s2 in ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)):
        v0 = cubes
        v1 = v0 + unit[s0]
        v2 = v1 + unit[s1]
        v3 = v2 + unit[s2]
        tl.append(np.stack([(v[:, 0] * n + v[:, 1]) * nzl + v[:, 2] for v in (v0, v1, v2, v3)], axis=1))
    tets = new_of_lex[np.concatenate(tl, axis=0)]
    tets = tets[np.argsort(tets.min(axis=1), kind="stable")].astype(np.int32)
    return mesh_from_tets(X, tets, ijk=ijk_new, n_side=n), gid


_MR = {}


def _morton_rank(n: int, t: int | None = None):
    """Dense rank of every Morton key of the n x n x t grid (t = n: the cube; lookup table,
    key -> rank)."""
    t = n if t is None else t
    if (n, t) not in _MR:
        g = np.arange(n)
        I, J, K = np.meshgrid(g, g, np.arange(t), indexing="ij")
        keys = _morton_key(np.stack([I.ravel(), J.ravel(), K.ravel()], axis=1).astype(np.int64))
        tab = np.full(int(keys.max()) + 1, -1, np.int64)
        tab[np.sort(keys)] = np.arange(keys.shape[0])
        _MR[(n, t)] = tab
    return _MR[(n, t)]


def slab_walls(ijk: np.ndarray, gid: np.ndarray, n: int, k: int, period: int = 16, rel_amp: float = 1e-2,
               seed: int = 0):
    """C3's wall displacement on a slab-ordered box, drawn per GLOBAL node id (counter-based:
    one generator per node block of 2^16 ids) so that every rank reproduces the owner's value
    for its ghosts.  Returns the displacement [len(gid), 3] (x_prev = X, x_cur = X + disp)."""
    h = 1.0 / (n - 1)
    wall = np.any(ijk % period == (k % period), axis=1)
    disp = _per_block_normals(gid, lambda b: [seed, 11, k, b])
    return (rel_amp * h) * disp * wall[:, None]


def _per_block_normals(gid: np.ndarray, seed_of) -> np.ndarray:
    """xi[v] = row (gid[v] & 0xFFFF) of the N(0,1) [2^16, 3] draw of generator seed_of(gid[v] >> 16)
    (one pass over the nodes; the blocks' draws are made once each)."""
    gid = np.asarray(gid, np.int64)
    ub, inv = np.unique(gid >> 16, return_inverse=True)
    tab = np.empty((ub.shape[0], 1 << 16, 3))
    for t, b in enumerate(ub):
        tab[t] = np.random.default_rng(seed_of(int(b))).standard_normal((1 << 16, 3))
    return tab[inv.reshape(-1), gid & 0xFFFF]


def slab_gradient(gid: np.ndarray, seed: int = 0) -> np.ndarray:
    """g_f ~ N(0,1) per component, drawn per global node id (counter-based like slab_walls)."""
    return _per_block_normals(gid, lambda b: [seed, 7, b])


# ----------------------------------------------------------------------------
# C4: multi-object contact scene: k^3 objects of n^3 nodes on a lattice with
# gaps, E cycling {1e5, 1e6, 1e7}, contact blocks between facing boundary nodes of adjacent
# objects (Hessian entries, never tagged: coarsening stays inside objects)
# ----------------------------------------------------------------------------

def _replicate_with_extras(base: Mesh, nobj: int, X, tets, ijk, pairs) -> Mesh:
    """The mesh of nobj disjoint copies of `base` (object-major node ids) plus symmetric
    Hessian-only pattern entries `pairs` -- equal to mesh_from_tets(X, tets, extra_pairs=pairs)
    (pinned in tests/test_synth_fast.py), without its global sorts."""
    N0, E0, S0 = base.n_nodes, base.n_edges, base.adj_nbr.shape[0]
    N = N0 * nobj
    oN = np.arange(nobj, dtype=np.int64)
    adj_ptr = np.concatenate([[0], (base.adj_ptr[1:][None, :] + (oN * S0)[:, None]).reshape(-1)])
    adj_nbr = (base.adj_nbr[None, :].astype(np.int64) + (oN * N0)[:, None]).reshape(-1).astype(np.int32)
    ts = (base.tet_slots[None].astype(np.int64) + (oN * S0)[:, None, None]).reshape(-1, 12).astype(np.int32)
    edges = (base.edges[None].astype(np.int64) + (oN * N0)[:, None, None]).reshape(-1, 2).astype(np.int32)
    eos = (base.edge_of_slot[None, :] + (oN * E0)[:, None]).reshape(-1)
    nb0 = base.bsr_col.shape[0]
    bptr = np.concatenate([[0], (base.bsr_ptr[1:][None, :] + (oN * nb0)[:, None]).reshape(-1)])
    bcol = (base.bsr_col[None, :].astype(np.int64) + (oN * N0)[:, None]).reshape(-1).astype(np.int32)
    ex = np.ascontiguousarray(np.asarray(pairs, np.int32))
    L = _lib()
    optr = np.empty(N + 1, np.int64)
    L.syn_merge_pattern(N, _ptr(bptr), _ptr(bcol), ex.shape[0], _ptr(ex), _ptr(optr), None, None)
    ocol = np.empty(int(optr[N]), np.int32)
    diag = np.empty(N, np.int64)
    L.syn_merge_pattern(N, _ptr(bptr), _ptr(bcol), ex.shape[0], _ptr(ex), _ptr(optr), _ptr(ocol), _ptr(diag))
    return Mesh(X=np.ascontiguousarray(X), tets=np.ascontiguousarray(tets, np.int32), adj_ptr=adj_ptr,
                adj_nbr=adj_nbr, tet_slots=ts, edges=edges, edge_of_slot=eos, bsr_ptr=optr, bsr_col=ocol,
                diag_slot=diag, ijk=np.ascontiguousarray(ijk, np.int32), n_side=base.n_side,
                n_extra=int(ocol.shape[0] - bcol.shape[0]))


def c4_scene(n: int = 57, k: int = 3, gap: float = 1e-3, side: float = 1.0, seed: int = 0, fast: bool = True):
    base = kuhn_grid(n, side=side)
    N0 = base.n_nodes
    nobj = k ** 3
    pitch = side + gap
    offs = []
    for ox in range(k):
        for oy in range(k):
            for oz in range(k):
                offs.append(((ox - (k - 1) / 2) * pitch, (oy - (k - 1) / 2) * pitch, (oz - (k - 1) / 2) * pitch))
    offs = np.asarray(offs)
    X = np.concatenate([base.X + offs[o] for o in range(nobj)])
    tets = np.concatenate([base.tets.astype(np.int64) + o * N0 for o in range(nobj)]).astype(np.int32)
    ijk = np.tile(base.ijk, (nobj, 1))
    # facing boundary nodes of lattice neighbours: (max face of o, min face of o + e_d)
    lid = np.empty((n, n, n), np.int64)
    lid[base.ijk[:, 0], base.ijk[:, 1], base.ijk[:, 2]] = np.arange(N0)
    oid = np.arange(nobj).reshape(k, k, k)
    pairs, normals = [], []
    for d in range(3):
        hi = np.take(lid, n - 1, axis=d).reshape(-1)
        lo = np.take(lid, 0, axis=d).reshape(-1)
        a_obj = np.take(oid, np.arange(k - 1), axis=d).reshape(-1)
        b_obj = np.take(oid, np.arange(1, k), axis=d).reshape(-1)
        for oa, ob in zip(a_obj, b_obj):
            pairs.append(np.stack([hi + oa * N0, lo + ob * N0], axis=1))
            nrm = np.zeros(3)
            nrm[d] = 1.0
            normals.append(np.broadcast_to(nrm, (hi.shape[0], 3)))
    pairs = np.concatenate(pairs)
    normals = np.concatenate(normals)
    m = _replicate_with_extras(base, nobj, X, tets, ijk, pairs) if fast else \
        mesh_from_tets(X, tets, ijk=ijk, n_side=n, extra_pairs=pairs)
    E_tet = np.repeat(np.asarray([(1e5, 1e6, 1e7)[o % 3] for o in range(nobj)]), base.n_tets)
    rng = np.random.default_rng([seed, 41])
    axes = rng.standard_normal((nobj, 3))
    return dict(mesh=m, N0=N0, nobj=nobj, offs=offs, pairs=pairs, normals=normals, E_tet=E_tet, axes=axes,
                side=side)


def c4_hessian(sc: dict, dt: float = 0.01) -> np.ndarray:
    """H_f = M + dt^2 K (per-object E) + contact kappa n n^T couplings, kappa = the mean
    diagonal entry of the elastic H_f (PSD pair blocks)."""
    m = sc["mesh"]
    H = fine_hessian(m, E=sc["E_tet"], dt=dt)
    kappa = float(np.mean(np.einsum("bii->b", H[m.diag_slot]) / 3.0))
    i, j = sc["pairs"][:, 0], sc["pairs"][:, 1]
    nn = np.einsum("pa,pb->pab", sc["normals"], sc["normals"]) * kappa
    np.add.at(H, m.diag_slot[i], nn)
    np.add.at(H, m.diag_slot[j], nn)
    np.add.at(H, bsr_slot(m, i, j), -nn)
    np.add.at(H, bsr_slot(m, j, i), -nn)
    return H


def c4_iterates(sc: dict, alpha0: float = 0.5, alpha1: float = 0.501, w: float = 0.2):
    """Per object: twist about its seeded random axis through its centre, alpha0 -> alpha1."""
    m = sc["mesh"]
    N0 = sc["N0"]
    xp = np.empty_like(m.X)
    xc = np.empty_like(m.X)
    for o in range(sc["nobj"]):
        sl = slice(o * N0, (o + 1) * N0)
        c = sc["offs"][o]
        xp[sl] = twist(m.X[sl], alpha0, w=w * sc["side"], axis=sc["axes"][o], center=c)
        xc[sl] = twist(m.X[sl], alpha1, w=w * sc["side"], axis=sc["axes"][o], center=c)
    return xp, xc


# ----------------------------------------------------------------------------
# NEXT#4: shells (triangles) and rods (edges) for step 1
# ----------------------------------------------------------------------------

def adj_slot(adj_ptr: np.ndarray, adj_nbr: np.ndarray, u, v) -> np.ndarray:
    """Adjacency slot of the directed edge (u -> v) (-1 if absent)."""
    N = adj_ptr.shape[0] - 1
    rows = np.repeat(np.arange(N, dtype=np.int64), np.diff(adj_ptr))
    key = rows * N + adj_nbr.astype(np.int64)
    q = np.asarray(u, np.int64) * N + np.asarray(v, np.int64)
    pos = np.searchsorted(key, q)
    ok = (pos < key.shape[0]) & (key[np.minimum(pos, key.shape[0] - 1)] == q)
    return np.where(ok, pos, -1)


def element_slots(adj_ptr, adj_nbr, elems: np.ndarray, local_edges) -> np.ndarray:
    """int32 [n_el, 2*len(local_edges)]: slots of (u->v), (v->u) for each local edge."""
    out = np.empty((elems.shape[0], 2 * len(local_edges)), np.int32)
    for e, (a, b) in enumerate(local_edges):
        out[:, 2 * e] = adj_slot(adj_ptr, adj_nbr, elems[:, a], elems[:, b])
        out[:, 2 * e + 1] = adj_slot(adj_ptr, adj_nbr, elems[:, b], elems[:, a])
    return out


TRI_EDGES = ((0, 1), (0, 2), (1, 2))


def adjacency_from_edges(N: int, pairs: np.ndarray):
    """Symmetric ascending adjacency CSR from undirected pairs."""
    p = np.asarray(pairs, np.int64)
    lo, hi = np.minimum(p[:, 0], p[:, 1]), np.maximum(p[:, 0], p[:, 1])
    ek = np.unique(lo * N + hi)
    allk = np.sort(np.concatenate([ek, (ek % N) * N + ek // N]))
    adj_nbr = (allk % N).astype(np.int32)
    adj_ptr = np.zeros(N + 1, np.int64)
    np.cumsum(np.bincount(allk // N, minlength=N), out=adj_ptr[1:])
    return adj_ptr, adj_nbr


def sheet(n: int, side: float = 1.0, seed: int = 0, rods: bool = True):
    """An n x n cloth sheet (2 triangles per quad) in a seeded random plane, Morton order, plus
    (rods=True) rod strands along every third grid row sharing the sheet's nodes.  Returns
    dict(X, tris, tri_slots, segs, seg_slots, adj_ptr, adj_nbr, ij)."""
    g = np.arange(n)
    I, J = np.meshgrid(g, g, indexing="ij")
    ij = np.stack([I.ravel(), J.ravel()], axis=1).astype(np.int64)
    key = np.zeros(ij.shape[0], np.int64)
    for bit in range(21):
        for d in range(2):
            key |= ((ij[:, d] >> bit) & 1) << (2 * bit + d)
    perm = np.argsort(key, kind="stable")
    new_of = np.empty(n * n, np.int64)
    new_of[perm] = np.arange(n * n)
    ij = ij[perm]
    q, _ = np.linalg.qr(np.random.default_rng([seed, 17]).standard_normal((3, 3)))
    P2 = np.stack([ij[:, 0], ij[:, 1], np.zeros(n * n)], axis=1) * (side / (n - 1)) - np.array([side / 2, side / 2, 0])
    X = P2 @ q.T
    c = np.arange(n - 1)
    CI, CJ = np.meshgrid(c, c, indexing="ij")
    v00 = (CI * n + CJ).ravel()
    v10, v01, v11 = v00 + n, v00 + 1, v00 + n + 1
    tris = new_of[np.concatenate([np.stack([v00, v10, v11], 1), np.stack([v00, v11, v01], 1)])].astype(np.int32)
    tris = tris[np.argsort(tris.min(axis=1), kind="stable")]
    segs = np.zeros((0, 2), np.int32)
    if rods:
        rows = np.arange(0, n, 3)
        a = (rows[:, None] * n + np.arange(n - 1)[None, :]).ravel()
        segs = new_of[np.stack([a, a + 1], 1)].astype(np.int32)
    pairs = np.concatenate([tris[:, [0, 1]], tris[:, [0, 2]], tris[:, [1, 2]], segs])
    adj_ptr, adj_nbr = adjacency_from_edges(n * n, pairs)
    return dict(X=X, tris=tris, tri_slots=element_slots(adj_ptr, adj_nbr, tris, TRI_EDGES), segs=segs,
                seg_slots=element_slots(adj_ptr, adj_nbr, segs, ((0, 1),)), adj_ptr=adj_ptr, adj_nbr=adj_nbr,
                ij=ij, n=n, rot=q)


def boundary_triangles(mesh: Mesh) -> np.ndarray:
    """Boundary faces of a tet mesh (faces used by exactly one tet), int32 [F,3]."""
    t = mesh.tets.astype(np.int64)
    faces = np.concatenate([t[:, [0, 1, 2]], t[:, [0, 1, 3]], t[:, [0, 2, 3]], t[:, [1, 2, 3]]])
    fs = np.sort(faces, axis=1)
    N = mesh.n_nodes
    key = (fs[:, 0] * N + fs[:, 1]) * N + fs[:, 2]
    u, idx, cnt = np.unique(key, return_index=True, return_counts=True)
    return faces[idx[cnt == 1]].astype(np.int32)


def tet_triplets(mesh: Mesh, E: float = 1e5, nu: float = 0.3, dt: float = 0.01):
    """NEXT#3 input: the unreduced element Hessian triplets of dt^2 K_lin -- 16 (i, j, B) per tet
    in tet order (a, b row-major) -- as (ti int32, tj int32, val float64 [16T,3,3])."""
    K, _ = stiffness_blocks(mesh.X, mesh.tets, E, nu)
    t = mesh.tets.astype(np.int64)
    ti = np.repeat(t, 4, axis=1).reshape(-1).astype(np.int32)
    tj = np.tile(t, (1, 4)).reshape(-1).astype(np.int32)
    return ti, tj, (dt * dt) * K.reshape(-1, 3, 3)
