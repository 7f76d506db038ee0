"""CPU oracle loader -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_2605_04773_b200``) never imports it and fails loudly without its
CUDA library.  The oracle itself is plain C (``agipc_oracle.c``); this module
only compiles it with gcc and marshals numpy arrays through ctypes.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "agipc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

OK, EINVAL, ERANGE, ENOMEM = 0, 1, 2, 3
EDEGENERATE, ESINGULAR, EINDEFINITE, EBREAKDOWN, NOT_CONVERGED = 6, 7, 8, 9, 10


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu99", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P = C.c_void_p
        i64, i32, f64 = C.c_int64, C.c_int, C.c_double
        L.orc_tag_edges.argtypes = [i64, P, P, P, P, P, f64, i64, P, P, P, P]
        L.orc_tag_edges.restype = i32
        L.orc_build_map.argtypes = [i64, P, P, P, i32, i32, P, i32, P, P, P, P, P, i32]
        L.orc_build_map.restype = i32
        L.orc_assemble.argtypes = [i64, P, i64, i64, P, P, P, P, P, P]
        L.orc_assemble.restype = P
        L.orc_coarse_free.argtypes = [P]
        L.orc_pcg.argtypes = [i64, P, P, P, P, P, f64, i32, P, P, P]
        L.orc_pcg.restype = i32
        L.orc_rel_residual.argtypes = [i64, P, P, P, P, P]
        L.orc_rel_residual.restype = f64
        L.orc_spmv.argtypes = [i64, P, P, P, P, P]
        L.orc_bsr_upper.argtypes = [i64, P, P, P, P, P, P]
        L.orc_bsr_upper.restype = i64
        L.orc_spmv_upper.argtypes = [i64, P, P, P, P, P]
        L.orc_spmv_upper.restype = None
        L.orc_bsr_expand_upper.argtypes = [i64, P, P, P, P, P, P]
        L.orc_bsr_expand_upper.restype = i64
        L.orc_block_jacobi.argtypes = [i64, P, P, P, P, P]
        L.orc_block_jacobi.restype = i32
        L.orc_prolongate.argtypes = [i64, P, i64, P, P, P]
        L.orc_prolongate.restype = None
        L.orc_reduce_triplets.argtypes = [i64, i64, P, P, P, P, P, P]
        L.orc_reduce_triplets.restype = i64
        for nm in ("orc_tag_shells", "orc_tag_rods"):
            getattr(L, nm).argtypes = [i64, P, P, P, P, P, f64, i64, i32, P, P, P]
            getattr(L, nm).restype = i32
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class OracleError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"oracle status {status} {msg}")
        self.status = status


# ---------------------------------------------------------------------------
def tag_edges(tets, tet_slots, X, x_prev, x_cur, theta, n_slots):
    """Step 1 (Eq 3).  Returns (slot_tags u8[2E], tet_norm f64[T], tet_flag u8[T])."""
    tets = _c(tets, np.int32); ts = _c(tet_slots, np.int32)
    X = _c(X, np.float64); xp = _c(x_prev, np.float64); xc = _c(x_cur, np.float64)
    T = tets.shape[0]
    tags = np.empty(n_slots, np.uint8)
    norm = np.empty(T, np.float64)
    flag = np.empty(T, np.uint8)
    bad = np.zeros(1, np.int64)
    st = lib().orc_tag_edges(T, _p(tets), _p(ts), _p(X), _p(xp), _p(xc), float(theta), int(n_slots),
                             _p(tags), _p(norm), _p(flag), _p(bad))
    if st != OK:
        raise OracleError(st, f"degenerate tet {int(bad[0])}")
    return tags, norm, flag


def build_map(adj_ptr, adj_nbr, slot_tags, group_size, max_levels=0, seg_begin=None):
    """Step 2 (Alg S1/S2 + P:217, level-wise).  Returns dict(map, agg_size, n_coarse, n_levels, level_n)."""
    adj_ptr = _c(adj_ptr, np.int64); adj_nbr = _c(adj_nbr, np.int32); tags = _c(slot_tags, np.uint8)
    N = adj_ptr.shape[0] - 1
    mp = np.empty(max(N, 1), np.int32)
    sz = np.empty(max(N, 1), np.int64)
    nc = np.zeros(1, np.int64)
    nl = np.zeros(1, np.int32)
    cap = 4096
    ln = np.zeros(cap, np.int64)
    seg = None if seg_begin is None else _c(seg_begin, np.int64)
    nseg = 1 if seg is None else seg.shape[0] - 1
    st = lib().orc_build_map(N, _p(adj_ptr), _p(adj_nbr), _p(tags), int(group_size), nseg, _p(seg),
                             int(max_levels), _p(mp), _p(sz), _p(nc), _p(nl), _p(ln), cap)
    if st != OK:
        raise OracleError(st)
    n_c = int(nc[0]); L = int(nl[0])
    return dict(map=mp[:N].copy(), agg_size=sz[:n_c].copy(), n_coarse=n_c, n_levels=L,
                level_n=ln[:min(L, cap)].copy())


class _Coarse(C.Structure):
    _fields_ = [("n3", C.c_int64), ("n12", C.c_int64), ("n_slots", C.c_int64), ("nnzb", C.c_int64),
                ("new_map", C.POINTER(C.c_int32)), ("dof", C.POINTER(C.c_int32)),
                ("row_ptr", C.POINTER(C.c_int64)), ("col", C.POINTER(C.c_int32)),
                ("val", C.POINTER(C.c_double)), ("bound", C.POINTER(C.c_double)),
                ("g_c", C.POINTER(C.c_double)), ("g_bound", C.POINTER(C.c_double))]


def _arr(ptr, n, dt):
    if n == 0 or not ptr:
        return np.zeros(n, dt)
    return np.ctypeslib.as_array(ptr, shape=(n,)).copy()


def assemble(map_, n_coarse, affine_threshold, X, bsr_ptr, bsr_col, bsr_val, g_f=None):
    """Step 3 (Alg S3 + S4 + Eq 4).  Returns dict(n3, n12, n_slots, nnzb, new_map, dof,
    row_ptr, col, val[nnzb,3,3], bound[nnzb,3,3], g_c[n_slots,3] | None, g_bound)."""
    map_ = _c(map_, np.int32); X = _c(X, np.float64)
    rp = _c(bsr_ptr, np.int64); cl = _c(bsr_col, np.int32); vl = _c(bsr_val, np.float64)
    g = None if g_f is None else _c(g_f, np.float64)
    N = map_.shape[0]
    st = C.c_int(0)
    L = lib()
    L.orc_assemble.argtypes[-1] = C.POINTER(C.c_int)
    ptr = L.orc_assemble(N, _p(map_), int(n_coarse), int(affine_threshold), _p(X), _p(rp), _p(cl), _p(vl),
                         _p(g), C.byref(st))
    if not ptr:
        raise OracleError(st.value)
    o = C.cast(ptr, C.POINTER(_Coarse)).contents
    ns, nnzb = int(o.n_slots), int(o.nnzb)
    out = dict(n3=int(o.n3), n12=int(o.n12), n_slots=ns, nnzb=nnzb,
               new_map=_arr(o.new_map, N, np.int32), dof=_arr(o.dof, int(n_coarse), np.int32),
               row_ptr=_arr(o.row_ptr, ns + 1, np.int64), col=_arr(o.col, nnzb, np.int32),
               val=_arr(o.val, 9 * nnzb, np.float64).reshape(nnzb, 3, 3),
               bound=_arr(o.bound, 9 * nnzb, np.float64).reshape(nnzb, 3, 3),
               g_c=None if g is None else _arr(o.g_c, 3 * ns, np.float64).reshape(ns, 3),
               g_bound=None if g is None else _arr(o.g_bound, 3 * ns, np.float64).reshape(ns, 3))
    if ns == 0:
        out["row_ptr"] = np.zeros(1, np.int64)
    L.orc_coarse_free(ptr)
    return out


def pcg(row_ptr, col, val, b, x0=None, rel_tol=1e-3, max_iters=1000, history=False):
    """Step 4: block-Jacobi PCG.  Returns dict(x, iters, rel_res, status, res_hist)."""
    rp = _c(row_ptr, np.int64); cl = _c(col, np.int32); vl = _c(val, np.float64)
    n = rp.shape[0] - 1
    b = _c(b, np.float64).reshape(-1)
    x = np.zeros(3 * n) if x0 is None else _c(x0, np.float64).reshape(-1).copy()
    it = np.zeros(1, np.int32)
    rr = np.zeros(1, np.float64)
    hist = np.zeros(max_iters + 1) if history else None
    st = lib().orc_pcg(n, _p(rp), _p(cl), _p(vl), _p(b), _p(x), float(rel_tol), int(max_iters),
                       _p(it), _p(rr), _p(hist))
    out = dict(x=x.reshape(n, 3), iters=int(it[0]), rel_res=float(rr[0]), status=int(st))
    if history:
        out["res_hist"] = hist[:int(it[0]) + 1]
    return out


def rel_residual(row_ptr, col, val, x, b):
    rp = _c(row_ptr, np.int64); cl = _c(col, np.int32); vl = _c(val, np.float64)
    n = rp.shape[0] - 1
    return float(lib().orc_rel_residual(n, _p(rp), _p(cl), _p(vl), _p(_c(x, np.float64)), _p(_c(b, np.float64))))


def spmv(row_ptr, col, val, x):
    rp = _c(row_ptr, np.int64); cl = _c(col, np.int32); vl = _c(val, np.float64)
    n = rp.shape[0] - 1
    y = np.empty(3 * n)
    lib().orc_spmv(n, _p(rp), _p(cl), _p(vl), _p(_c(x, np.float64)), _p(y))
    return y.reshape(n, 3)


def bsr_upper(row_ptr, col, val):
    """NEXT#2: diagonal + upper blocks of a full-storage BSR -> (row_ptr, col, val)."""
    rp = _c(row_ptr, np.int64); cl = _c(col, np.int32); vl = _c(val, np.float64)
    n = rp.shape[0] - 1
    nb = int(lib().orc_bsr_upper(n, _p(rp), _p(cl), _p(vl), None, None, None))
    urp = np.zeros(n + 1, np.int64)
    ucol = np.zeros(max(nb, 1), np.int32)
    uval = np.zeros((max(nb, 1), 3, 3))
    lib().orc_bsr_upper(n, _p(rp), _p(cl), _p(vl), _p(urp), _p(ucol), _p(uval))
    return urp, ucol[:nb], uval[:nb]


def spmv_upper(urp, ucol, uval, x):
    """NEXT#2: y = A x for the symmetric A given by its diagonal + upper blocks."""
    rp = _c(urp, np.int64); cl = _c(ucol, np.int32); vl = _c(uval, np.float64)
    n = rp.shape[0] - 1
    y = np.empty(3 * n)
    lib().orc_spmv_upper(n, _p(rp), _p(cl), _p(vl), _p(_c(x, np.float64)), _p(y))
    return y.reshape(n, 3)


def bsr_expand_upper(row_ptr, col, urp, ucol, uval):
    """NEXT#2: full-storage values on the pattern (row_ptr, col) from upper storage.
    Returns (val, number of full blocks without a source block)."""
    rp = _c(row_ptr, np.int64); cl = _c(col, np.int32)
    n = rp.shape[0] - 1
    val = np.zeros((cl.shape[0], 3, 3))
    miss = int(lib().orc_bsr_expand_upper(n, _p(rp), _p(cl), _p(_c(urp, np.int64)), _p(_c(ucol, np.int32)),
                                          _p(_c(uval, np.float64)), _p(val)))
    return val, miss


def block_jacobi(row_ptr, col, val):
    rp = _c(row_ptr, np.int64); cl = _c(col, np.int32); vl = _c(val, np.float64)
    n = rp.shape[0] - 1
    D = np.empty(9 * n + 1)
    bad = np.zeros(1, np.int64)
    st = lib().orc_block_jacobi(n, _p(rp), _p(cl), _p(vl), _p(D), _p(bad))
    if st != OK:
        raise OracleError(st, f"row {int(bad[0])}")
    return D[:9 * n].reshape(n, 3, 3)


def prolongate(new_map, n3, X, x_c):
    """NEXT#1: d_f = U^T d_c.  Returns float64 [N,3]."""
    nm = _c(new_map, np.int32); X = _c(X, np.float64); xc = _c(x_c, np.float64)
    N = nm.shape[0]
    d = np.empty((N, 3))
    lib().orc_prolongate(N, _p(nm), int(n3), _p(X), _p(xc), _p(d))
    return d


def _tag_elems(fn, elems, slots, X, x_prev, x_cur, theta, n_slots, slot_tags=None):
    el = _c(elems, np.int32); sl = _c(slots, np.int32)
    X = _c(X, np.float64); xp = _c(x_prev, np.float64); xc = _c(x_cur, np.float64)
    T = el.shape[0]
    reset = slot_tags is None
    tags = np.empty(n_slots, np.uint8) if reset else np.ascontiguousarray(slot_tags, np.uint8).copy()
    norm = np.empty(T, np.float64)
    bad = np.zeros(1, np.int64)
    st = getattr(lib(), fn)(T, _p(el), _p(sl), _p(X), _p(xp), _p(xc), float(theta), int(n_slots), int(reset),
                            _p(tags), _p(norm), _p(bad))
    if st != OK:
        raise OracleError(st, f"degenerate element {int(bad[0])}")
    return tags, norm


def tag_shells(tris, tri_slots, X, x_prev, x_cur, theta, n_slots, slot_tags=None):
    """NEXT#4, triangles ("shells"): returns (slot_tags, tri_norm).  If slot_tags is given
    the flags are accumulated into a copy of it (tets + shells + rods), else all start at 1."""
    return _tag_elems("orc_tag_shells", tris, tri_slots, X, x_prev, x_cur, theta, n_slots, slot_tags)


def tag_rods(segs, seg_slots, X, x_prev, x_cur, theta, n_slots, slot_tags=None):
    """NEXT#4, edges ("rods"): G = 1/2 (F^2 - 1), F = l / L."""
    return _tag_elems("orc_tag_rods", segs, seg_slots, X, x_prev, x_cur, theta, n_slots, slot_tags)


def reduce_triplets(n_rows, ti, tj, tval):
    """NEXT#3 (supp Sec 2): stable key sort + in-order segmented sums.
    Returns (row_ptr int64 [n_rows+1], col int32 [nnzb], val float64 [nnzb,3,3])."""
    ti = _c(ti, np.int32); tj = _c(tj, np.int32); tv = _c(tval, np.float64)
    n = ti.shape[0]
    rp = np.zeros(n_rows + 1, np.int64)
    col = np.empty(max(n, 1), np.int32)
    val = np.empty((max(n, 1), 9))
    nb = lib().orc_reduce_triplets(int(n_rows), n, _p(ti), _p(tj), _p(tv), _p(rp), _p(col), _p(val))
    if nb < 0:
        raise OracleError(-nb)
    return rp, col[:nb].copy(), val[:nb].reshape(nb, 3, 3).copy()
