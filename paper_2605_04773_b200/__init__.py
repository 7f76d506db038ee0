"""Thin Python binding of libagipc -- the B200-native AGIPC coarsening path.

Argument marshalling only: every step of the path runs in the CUDA kernels of
``libagipc.so`` (built from ``csrc/`` for sm_100a).  PyTorch provides device
memory and streams.  There is no CPU fallback: if the library is missing or no
CUDA device is present the calls raise.

Entry points (same names as the C ABI, include/agipc.h):
  tag_edges        step 1, Eq 3
  build_map        step 2, supp Alg S1/S2 + recursion
  assemble_coarse  step 3, supp Alg S3/S4 + Eq 4
  pcg_solve        step 4, block-Jacobi PCG
  prolongate       NEXT#1, d_f = U^T d_c
Multi-GPU: the library-owned NCCL communicator (Handle.comm_init, comm_unique_id,
comm_allgather_scan, comm_alltoall_i64, halo_exchange, dpcg_solve) and the rank-local pieces
(gather_rows, coarse_halo, assemble_halo, DistPcg for the split-phase solve over gloo);
paper_2605_04773_b200.dist composes them.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AGIPC_LIB") or os.path.join(_HERE, "libagipc.so")
_lib = None

OK, EINVAL, ERANGE, ENOSPACE, ECUDA, ENCCL = 0, 1, 2, 3, 4, 5
EDEGENERATE, ESINGULAR, EINDEFINITE, EBREAKDOWN, NOT_CONVERGED = 6, 7, 8, 9, 10


class AgipcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_status_name(status)}: {msg}")
        self.status = status


class _Mesh(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("n_tets", C.c_int64), ("nnz_adj", C.c_int64),
                ("tets", C.c_void_p), ("adj_ptr", C.c_void_p), ("adj_nbr", C.c_void_p),
                ("tet_slots", C.c_void_p), ("x_rest", C.c_void_p)]


class _Bsr(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("nnzb", C.c_int64), ("row_ptr", C.c_void_p),
                ("col", C.c_void_p), ("val", C.c_void_p)]


class _MapInfo(C.Structure):
    _fields_ = [("n_coarse", C.c_int64), ("n_levels", C.c_int32), ("reserved", C.c_int32),
                ("level_n", C.c_int64 * 64), ("n_cross_edges", C.c_int64)]


class _Coarse(C.Structure):
    _fields_ = [("n3", C.c_int64), ("n12", C.c_int64), ("n_slots", C.c_int64), ("nnzb", C.c_int64),
                ("cap_slots", C.c_int64), ("cap_nnzb", C.c_int64), ("new_map", C.c_void_p),
                ("row_ptr", C.c_void_p), ("col", C.c_void_p), ("val", C.c_void_p), ("g_c", C.c_void_p)]


class _HaloMatrix(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("nnzb", C.c_int64), ("cap_nnzb", C.c_int64), ("row_ptr", C.c_void_p),
                ("col", C.c_void_p), ("val", C.c_void_p)]


class _Halo(C.Structure):
    _fields_ = [("n_peers", C.c_int), ("peer_rank", C.c_void_p), ("send_ptr", C.c_void_p), ("send_idx", C.c_void_p),
                ("recv_ptr", C.c_void_p)]


class _TripletPlan(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_trip", C.c_int64), ("nnzb", C.c_int64), ("cap_nnzb", C.c_int64),
                ("row_ptr", C.c_void_p), ("col", C.c_void_p), ("seg_ptr", C.c_void_p), ("seg_idx", C.c_void_p)]


class _ProfEntry(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("count", C.c_int64), ("total_ms", C.c_double)]


class _PcgStats(C.Structure):
    _fields_ = [("iters", C.c_int32), ("status", C.c_int32), ("rel_residual", C.c_double),
                ("b_norm", C.c_double)]


EXPORTS = ["agipc_create", "agipc_destroy", "agipc_set_stream", "agipc_last_error", "agipc_status_string",
           "agipc_version", "agipc_kernel_launches", "agipc_profile", "agipc_profile_read", "agipc_tag_edges",
           "agipc_build_map", "agipc_assemble_coarse", "agipc_pcg_solve", "agipc_prolongate",
           "agipc_gather_rows", "agipc_coarse_halo", "agipc_assemble_halo", "agipc_dpcg_setup", "agipc_dpcg_pack",
           "agipc_dpcg_spmv", "agipc_dpcg_update", "agipc_dpcg_status", "agipc_dpcg_finish", "agipc_tag_shells",
           "agipc_tag_rods", "agipc_triplet_plan", "agipc_triplet_reduce", "agipc_bsr_upper", "agipc_pcg_solve_sym",
           "agipc_bsr_expand_upper", "agipc_set_values_event", "agipc_set_option", "agipc_workspace_size",
           "agipc_set_workspace", "agipc_comm_unique_id", "agipc_comm_init", "agipc_comm_info",
           "agipc_comm_allgather_scan", "agipc_comm_alltoall_i64", "agipc_halo_exchange", "agipc_dpcg_solve",
           "agipc_pcg_set_static"]

OPT_CHECK_SYMMETRY, OPT_L2_PERSIST, OPT_COMM_ALWAYS, OPT_DETERMINISTIC = 1, 2, 3, 4  # include/agipc.h AGIPC_OPT_*


def lib():
    """Load libagipc.so (raises if it has not been built -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py build` "
                               "(nvcc, sm_100a); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        P, i64, i32, f64 = C.c_void_p, C.c_int64, C.c_int, C.c_double
        L.agipc_create.argtypes = [C.POINTER(C.c_void_p), i32]
        L.agipc_destroy.argtypes = [P]
        L.agipc_set_stream.argtypes = [P, P]
        L.agipc_last_error.argtypes = [P]
        L.agipc_last_error.restype = C.c_char_p
        L.agipc_status_string.argtypes = [i32]
        L.agipc_status_string.restype = C.c_char_p
        L.agipc_version.argtypes = [C.POINTER(i32), C.POINTER(i32)]
        L.agipc_version.restype = None
        L.agipc_kernel_launches.argtypes = [P]
        L.agipc_kernel_launches.restype = i64
        L.agipc_profile.argtypes = [P, i32]
        L.agipc_profile.restype = i32
        L.agipc_profile_read.argtypes = [P, C.POINTER(_ProfEntry), i32]
        L.agipc_profile_read.restype = i32
        L.agipc_tag_edges.argtypes = [P, C.POINTER(_Mesh), P, P, f64, P, P, C.POINTER(i64)]
        L.agipc_build_map.argtypes = [P, C.POINTER(_Mesh), P, i32, i32, P, P, C.POINTER(_MapInfo)]
        L.agipc_assemble_coarse.argtypes = [P, C.POINTER(_Mesh), P, i64, i64, C.POINTER(_Bsr), P,
                                            C.POINTER(_Coarse)]
        L.agipc_pcg_solve.argtypes = [P, C.POINTER(_Bsr), P, P, i32, f64, i32, i32, C.POINTER(_PcgStats)]
        L.agipc_pcg_solve_sym.argtypes = [P, C.POINTER(_Bsr), i32, P, P, i32, f64, i32, i32, C.POINTER(_PcgStats)]
        L.agipc_bsr_upper.argtypes = [P, C.POINTER(_Bsr), i64, P, P, P, C.POINTER(i64)]
        L.agipc_set_values_event.argtypes = [P, P]
        L.agipc_bsr_expand_upper.argtypes = [P, C.POINTER(_Bsr), C.POINTER(_Bsr), P, i32]
        L.agipc_prolongate.argtypes = [P, C.POINTER(_Mesh), P, i64, i64, P, f64, P]
        L.agipc_gather_rows.argtypes = [P, P, P, i64, i32, P]
        L.agipc_triplet_plan.argtypes = [P, i64, i64, P, P, C.POINTER(_TripletPlan)]
        L.agipc_triplet_reduce.argtypes = [P, C.POINTER(_TripletPlan), P, P]
        for nm in ("agipc_tag_shells", "agipc_tag_rods"):
            getattr(L, nm).argtypes = [P, i64, P, P, P, P, P, f64, i64, i32, P, P, C.POINTER(i64)]
        L.agipc_coarse_halo.argtypes = [P, P, i64, i64, P, i64, P, P, i64, C.POINTER(i64)]
        L.agipc_assemble_halo.argtypes = [P, C.POINTER(_Mesh), P, i64, i64, C.POINTER(_Bsr), i64, P, i32,
                                          C.POINTER(i64), C.POINTER(i64), C.POINTER(_HaloMatrix)]
        L.agipc_dpcg_setup.argtypes = [P, C.POINTER(_Bsr), C.POINTER(_Bsr), i64, P, f64, i32, P]
        L.agipc_dpcg_pack.argtypes = [P, P, i64, P]
        L.agipc_dpcg_spmv.argtypes = [P, P, P]
        L.agipc_dpcg_update.argtypes = [P, P]
        L.agipc_dpcg_status.argtypes = [P, C.POINTER(i32), C.POINTER(_PcgStats)]
        L.agipc_dpcg_finish.argtypes = [P, P, P, C.POINTER(_PcgStats)]
        L.agipc_set_option.argtypes = [P, i32, i64]
        L.agipc_pcg_set_static.argtypes = [P, C.POINTER(_Bsr)]
        L.agipc_workspace_size.argtypes = [P, i64, i64, i64, i64, C.POINTER(C.c_size_t)]
        L.agipc_set_workspace.argtypes = [P, P, C.c_size_t]
        L.agipc_comm_unique_id.argtypes = [P]
        L.agipc_comm_init.argtypes = [P, P, i32, i32]
        L.agipc_comm_info.argtypes = [P, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]
        L.agipc_comm_allgather_scan.argtypes = [P, P, i32, P, P]
        L.agipc_comm_alltoall_i64.argtypes = [P, P, P]
        L.agipc_halo_exchange.argtypes = [P, C.POINTER(_Halo), P, i32, P]
        L.agipc_dpcg_solve.argtypes = [P, C.POINTER(_Bsr), C.POINTER(_Bsr), i64, C.POINTER(_Halo), P, P, f64, i32, i32,
                                       C.POINTER(_PcgStats)]
        for name in EXPORTS:
            if name not in ("agipc_last_error", "agipc_status_string", "agipc_version", "agipc_kernel_launches",
                            "agipc_profile_read"):
                getattr(L, name).restype = i32
        _lib = L
    return _lib


def _status_name(s):
    try:
        return lib().agipc_status_string(int(s)).decode()
    except Exception:  # noqa: BLE001 - only used for messages
        return f"status {s}"


def version():
    a, b = C.c_int(), C.c_int()
    lib().agipc_version(C.byref(a), C.byref(b))
    return a.value, b.value


def _p(t):
    if t is None:
        return None
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("libagipc takes contiguous CUDA tensors")
    return C.c_void_p(t.data_ptr())


class Handle:
    """One libagipc handle bound to a CUDA device; kernels go on the current torch stream."""

    def __init__(self, device: int = 0):
        if not torch.cuda.is_available():
            raise RuntimeError("libagipc needs a CUDA device (no CPU fallback)")
        self.device = int(device)
        self._h = C.c_void_p()
        st = lib().agipc_create(C.byref(self._h), self.device)
        if st != OK:
            raise AgipcError(st, f"agipc_create(device={device}) failed")
        self.sync_stream()

    def sync_stream(self, stream: torch.cuda.Stream | None = None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._check(lib().agipc_set_stream(self._h, C.c_void_p(s.cuda_stream)))

    def _check(self, st, allow=()):
        if st != OK and st not in allow:
            raise AgipcError(st, lib().agipc_last_error(self._h).decode())
        return st

    def set_values_event(self, event: torch.cuda.Event | None):
        """One-shot: the next assemble_coarse's numeric phase waits for `event` (see
        agipc_set_values_event)."""
        self._check(lib().agipc_set_values_event(self._h, C.c_void_p(event.cuda_event if event is not None else 0)))

    @property
    def kernel_launches(self) -> int:
        return int(lib().agipc_kernel_launches(self._h))

    def profile(self, enable: bool = True):
        """Reset and enable/disable the library's CUDA-event timing (agipc_profile)."""
        self._check(lib().agipc_profile(self._h, int(bool(enable))))

    def profile_read(self) -> dict:
        """{phase: (count, total_ms)} from agipc_profile_read (synchronises pending events)."""
        buf = (_ProfEntry * 16)()
        n = lib().agipc_profile_read(self._h, buf, 16)
        return {buf[i].name.decode(): (int(buf[i].count), float(buf[i].total_ms)) for i in range(n)}

    def set_option(self, option: int, value: int):
        """agipc_set_option (OPT_CHECK_SYMMETRY, OPT_L2_PERSIST)."""
        self._check(lib().agipc_set_option(self._h, int(option), int(value)))

    def pcg_set_static(self, row_ptr=None, col=None):
        """agipc_pcg_set_static: solves on exactly this (row_ptr, col) keep their SELL layout and
        only refill values (the fine pattern is static).  No arguments clears."""
        if row_ptr is None:
            self._check(lib().agipc_pcg_set_static(self._h, None))
            return
        self._static_pattern = (row_ptr, col)  # the library holds the pointers: keep them alive
        bsr = _Bsr(row_ptr.shape[0] - 1, col.shape[0], _p(row_ptr), _p(col), None)
        self._check(lib().agipc_pcg_set_static(self._h, C.byref(bsr)))

    def workspace_size(self, n_nodes=0, n_tets=0, nnz_adj=0, nnzb_fine=0) -> int:
        """agipc_workspace_size: bytes of caller-owned scratch to register (set_workspace)."""
        b = C.c_size_t(0)
        self._check(lib().agipc_workspace_size(self._h, int(n_nodes), int(n_tets), int(nnz_adj), int(nnzb_fine),
                                               C.byref(b)))
        return int(b.value)

    def set_workspace(self, ws: torch.Tensor | None):
        """Hand the library a caller-owned device arena (uint8 CUDA tensor, kept alive here), or None
        to return to internal allocation (agipc_set_workspace)."""
        if ws is None:
            self._check(lib().agipc_set_workspace(self._h, None, 0))
        else:
            if ws.dtype != torch.uint8 or not ws.is_cuda or not ws.is_contiguous():
                raise ValueError("workspace must be a contiguous uint8 CUDA tensor")
            self._check(lib().agipc_set_workspace(self._h, C.c_void_p(ws.data_ptr()), ws.numel()))
        self._ws = ws

    def comm_init(self, unique_id: bytes, nranks: int, rank: int):
        """agipc_comm_init: the library's own NCCL communicator (unique_id from comm_unique_id() on
        rank 0, moved to the other ranks by the caller)."""
        if len(unique_id) != 128:
            raise ValueError("unique id must be 128 bytes")
        buf = C.create_string_buffer(bytes(unique_id), 128)
        self._check(lib().agipc_comm_init(self._h, buf, int(nranks), int(rank)))

    def comm_info(self):
        a, b, v = C.c_int(), C.c_int(), C.c_int()
        self._check(lib().agipc_comm_info(self._h, C.byref(a), C.byref(b), C.byref(v)))
        return dict(nranks=a.value, rank=b.value, nccl_version=v.value)

    def close(self):
        if self._h:
            lib().agipc_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


@dataclasses.dataclass
class DeviceMesh:
    """Static fine mesh resident on the GPU (layouts of include/agipc.h: agipc_mesh)."""
    tets: torch.Tensor       # int32 [T,4]
    adj_ptr: torch.Tensor    # int64 [N+1]
    adj_nbr: torch.Tensor    # int32 [2E]
    tet_slots: torch.Tensor  # int32 [T,12]
    x_rest: torch.Tensor     # float64 [N(+ghosts),3]
    n_own: int | None = None  # partitioned local mesh: owned nodes (x_rest also holds the ghosts)

    @property
    def n_nodes(self):
        return self.x_rest.shape[0] if self.n_own is None else self.n_own

    def c_struct(self):
        # cached per tensor identity: the struct is marshalled once, not at every call of a step
        key = (id(self.tets), id(self.adj_ptr), id(self.adj_nbr), id(self.tet_slots), id(self.x_rest), self.n_own)
        c = self.__dict__.get("_cstruct")
        if c is None or c[0] != key:
            c = (key, _Mesh(self.n_nodes, self.tets.shape[0], self.adj_nbr.shape[0], _p(self.tets), _p(self.adj_ptr),
                            _p(self.adj_nbr), _p(self.tet_slots), _p(self.x_rest)))
            self.__dict__["_cstruct"] = c
        return c[1]

    @staticmethod
    def from_arrays(tets, adj_ptr, adj_nbr, tet_slots, x_rest, device="cuda", n_own=None):
        t = lambda a, dt: torch.as_tensor(a).to(device=device, dtype=dt).contiguous()  # noqa: E731
        return DeviceMesh(t(tets, torch.int32), t(adj_ptr, torch.int64), t(adj_nbr, torch.int32),
                          t(tet_slots, torch.int32), t(x_rest, torch.float64), n_own)


# ---------------------------------------------------------------------------------------
# the four entry points
# ---------------------------------------------------------------------------------------
def tag_edges(h: Handle, mesh: DeviceMesh, x_prev, x_cur, threshold: float, slot_tags=None, tet_norm=None,
              count: bool = False):
    """Step 1 (Eq 3).  Returns (slot_tags uint8 [2E], n_flagged or None)."""
    if slot_tags is None:
        slot_tags = torch.empty(mesh.adj_nbr.shape[0], dtype=torch.uint8, device=mesh.x_rest.device)
    ms = mesh.c_struct()
    nf = C.c_int64(0)
    h._check(lib().agipc_tag_edges(h._h, C.byref(ms), _p(x_prev), _p(x_cur), float(threshold), _p(slot_tags),
                                   _p(tet_norm), C.byref(nf) if count else None))
    return slot_tags, (int(nf.value) if count else None)


def build_map(h: Handle, mesh: DeviceMesh, slot_tags, group_size: int = 32, max_levels: int = 0, map=None,
              agg_size=None):
    """Step 2 (Alg S1/S2 + P:217).  Returns (map int32 [N], info dict)."""
    N = mesh.n_nodes
    if map is None:
        map = torch.empty(N, dtype=torch.int32, device=mesh.x_rest.device)
    ms = mesh.c_struct()
    info = _MapInfo()
    h._check(lib().agipc_build_map(h._h, C.byref(ms), _p(slot_tags), int(group_size), int(max_levels), _p(map),
                                   _p(agg_size), C.byref(info)))
    L = info.n_levels
    return map, dict(n_coarse=int(info.n_coarse), n_levels=int(L),
                     level_n=list(info.level_n[:min(L, 64)]),
                     n_cross_edges=int(info.n_cross_edges))


@dataclasses.dataclass
class CoarseSystem:
    n3: int
    n12: int
    n_slots: int
    nnzb: int
    new_map: torch.Tensor
    row_ptr: torch.Tensor     # int64 [n_slots+1] (view)
    col: torch.Tensor         # int32 [nnzb] (view)
    val: torch.Tensor         # float64 [nnzb,3,3] (view)
    g_c: torch.Tensor | None  # float64 [n_slots,3] (view)


class CoarseBuffers:
    """Grow-only output buffers for assemble_coarse (capacity-retry convention)."""

    def __init__(self, device, n_nodes, cap_slots=0, cap_nnzb=0):
        self.device = device
        self.new_map = torch.empty(n_nodes, dtype=torch.int32, device=device)
        self.cap_slots = 0
        self.cap_nnzb = 0
        self.grow(cap_slots, cap_nnzb)

    def grow(self, slots, nnzb):
        if slots > self.cap_slots or not hasattr(self, "row_ptr"):
            self.cap_slots = max(int(slots * 1.25) + 16, self.cap_slots)
            self.row_ptr = torch.empty(self.cap_slots + 1, dtype=torch.int64, device=self.device)
            self.g_c = torch.empty((self.cap_slots, 3), dtype=torch.float64, device=self.device)
        if nnzb > self.cap_nnzb or not hasattr(self, "col"):
            self.cap_nnzb = max(int(nnzb * 1.25) + 64, self.cap_nnzb)
            self.col = torch.empty(self.cap_nnzb, dtype=torch.int32, device=self.device)
            self.val = torch.empty((self.cap_nnzb, 3, 3), dtype=torch.float64, device=self.device)


def assemble_coarse(h: Handle, mesh: DeviceMesh, map, n_coarse: int, affine_threshold: int, H_row_ptr, H_col,
                    H_val, g_fine=None, bufs: CoarseBuffers | None = None) -> CoarseSystem:
    """Step 3 (Alg S3/S4 + Eq 4).  Retries once with grown buffers on AGIPC_ENOSPACE."""
    N = mesh.n_nodes
    if bufs is None:
        bufs = CoarseBuffers(mesh.x_rest.device, N, 4 * n_coarse, H_col.shape[0])
    ms = mesh.c_struct()
    bsr = _Bsr(N, H_col.shape[0], _p(H_row_ptr), _p(H_col), _p(H_val))
    for attempt in range(2):
        out = _Coarse(0, 0, 0, 0, bufs.cap_slots, bufs.cap_nnzb, _p(bufs.new_map), _p(bufs.row_ptr),
                      _p(bufs.col), _p(bufs.val), _p(bufs.g_c) if g_fine is not None else None)
        st = lib().agipc_assemble_coarse(h._h, C.byref(ms), _p(map), int(n_coarse), int(affine_threshold),
                                         C.byref(bsr), _p(g_fine), C.byref(out))
        if st == ENOSPACE and attempt == 0:
            bufs.grow(out.n_slots, out.nnzb)
            continue
        h._check(st)
        break
    ns, nb = int(out.n_slots), int(out.nnzb)
    return CoarseSystem(int(out.n3), int(out.n12), ns, nb, bufs.new_map, bufs.row_ptr[:ns + 1], bufs.col[:nb],
                        bufs.val[:nb], bufs.g_c[:ns] if g_fine is not None else None)


STORAGE_FULL, STORAGE_SYM, STORAGE_UPPER = 0, 1, 2  # include/agipc.h AGIPC_STORAGE_* (NEXT#2)


def pcg_solve(h: Handle, row_ptr, col, val, b, x=None, rel_tol: float = 1e-3, max_iters: int = 10000,
              check_every: int = 16, zero_x0: bool = False, storage: int = STORAGE_FULL):
    """Step 4 (block-Jacobi PCG).  x is the initial guess; if None (or zero_x0) the solve starts
    from x0 = 0 in the kernels.  x is overwritten.  Returns (x, stats dict).  NOT_CONVERGED is
    reported in stats, not raised.  storage != STORAGE_FULL calls agipc_pcg_solve_sym (NEXT#2,
    P:1126): STORAGE_SYM streams the upper half of a full-storage matrix, STORAGE_UPPER takes a
    matrix that holds only its diagonal + upper blocks (see bsr_upper)."""
    n = row_ptr.shape[0] - 1
    zero_x0 = x is None or zero_x0
    if x is None:
        x = torch.empty((n, 3), dtype=torch.float64, device=b.device)
    bsr = _Bsr(n, col.shape[0], _p(row_ptr), _p(col), _p(val))
    stats = _PcgStats()
    if storage == STORAGE_FULL:
        st = lib().agipc_pcg_solve(h._h, C.byref(bsr), _p(b), _p(x), int(bool(zero_x0)), float(rel_tol),
                                   int(max_iters), int(check_every), C.byref(stats))
    else:
        st = lib().agipc_pcg_solve_sym(h._h, C.byref(bsr), int(storage), _p(b), _p(x), int(bool(zero_x0)),
                                       float(rel_tol), int(max_iters), int(check_every), C.byref(stats))
    h._check(st, allow=(NOT_CONVERGED,))
    return x, dict(iters=int(stats.iters), status=int(stats.status), rel_residual=float(stats.rel_residual),
                   b_norm=float(stats.b_norm))


def bsr_upper(h: Handle, row_ptr, col, val, cap_nnzb: int | None = None):
    """NEXT#2: the diagonal + upper blocks (col >= row) of a full-storage BSR.
    Returns (row_ptr, col, val) of the upper storage."""
    n = row_ptr.shape[0] - 1
    dev = row_ptr.device
    bsr = _Bsr(n, col.shape[0], _p(row_ptr), _p(col), _p(val))
    urp = torch.empty(n + 1, dtype=torch.int64, device=dev)
    cap = (col.shape[0] + n) // 2 + 1 if cap_nnzb is None else int(cap_nnzb)
    while True:
        ucol = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        uval = torch.empty((max(cap, 1), 3, 3), dtype=torch.float64, device=dev)
        nb = C.c_int64(0)
        st = lib().agipc_bsr_upper(h._h, C.byref(bsr), int(cap), _p(urp), _p(ucol), _p(uval), C.byref(nb))
        if st == ENOSPACE:
            cap = int(nb.value)
            continue
        h._check(st)
        return urp, ucol[:nb.value], uval[:nb.value]


def bsr_expand_upper(h: Handle, row_ptr, col, u_row_ptr, u_col, u_val, out=None, check: bool = True):
    """NEXT#2: full-storage values on the pattern (row_ptr, col) from the diagonal + upper
    blocks (u_row_ptr, u_col, u_val) -- the symmetric storage of P:1126.  check=False skips the
    pattern check and its host synchronisation (for a validated, static pattern).  Returns out."""
    n = row_ptr.shape[0] - 1
    if out is None:
        out = torch.empty((col.shape[0], 3, 3), dtype=torch.float64, device=u_val.device)
    full = _Bsr(n, col.shape[0], _p(row_ptr), _p(col), None)
    U = _Bsr(n, u_col.shape[0], _p(u_row_ptr), _p(u_col), _p(u_val))
    h._check(lib().agipc_bsr_expand_upper(h._h, C.byref(full), C.byref(U), _p(out), int(bool(check))))
    return out


def prolongate(h: Handle, mesh: DeviceMesh, new_map, n3: int, n_slots: int, x_c, alpha: float = 1.0, out=None):
    """NEXT#1: d_f = alpha * U^T x_c.  Returns out (float64 [N,3])."""
    N = mesh.n_nodes
    if out is None:
        out = torch.empty((N, 3), dtype=torch.float64, device=x_c.device)
    ms = mesh.c_struct()
    h._check(lib().agipc_prolongate(h._h, C.byref(ms), _p(new_map), int(n3), int(n_slots), _p(x_c),
                                    float(alpha), _p(out)))
    return out


# ---------------------------------------------------------------------------------------
# multi-GPU pieces (include/agipc.h "Multi-GPU partitioned path")
# ---------------------------------------------------------------------------------------
def gather_rows(h: Handle, src, idx, out=None):
    """out[k] = src[idx[k]] (rows of src; halo send buffers)."""
    n = idx.shape[0]
    if out is None:
        out = torch.empty((n,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    rb = src[0].numel() * src.element_size() if src.shape[0] else 4
    h._check(lib().agipc_gather_rows(h._h, _p(src), _p(idx), int(n), int(rb), _p(out)))
    return out


def coarse_halo(h: Handle, new_map, n3: int, n_coarse: int, send_idx, ghost_code=None, send_slots=None):
    """Owner side of exchange 3 for one peer.  Returns (ghost_code int32 [n_send], send_slots int32 [m])."""
    n = send_idx.shape[0]
    dev = new_map.device
    if ghost_code is None:
        ghost_code = torch.empty(n, dtype=torch.int32, device=dev)
    cap = 0 if send_slots is None else send_slots.shape[0]
    ns = C.c_int64(0)
    for attempt in range(2):
        st = lib().agipc_coarse_halo(h._h, _p(new_map), int(n3), int(n_coarse), _p(send_idx), int(n), _p(ghost_code),
                                     _p(send_slots), int(cap), C.byref(ns))
        if st == ENOSPACE and attempt == 0:
            cap = int(ns.value)
            send_slots = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
            continue
        h._check(st)
        break
    m = int(ns.value)
    if send_slots is None:
        send_slots = torch.empty(0, dtype=torch.int32, device=dev)
    return ghost_code, send_slots[:m]


def assemble_halo(h: Handle, mesh: DeviceMesh, new_map, n3: int, n_coarse: int, H_row_ptr, H_col, H_val,
                  ghost_code, peer_ghost_ptr, peer_slot_base, cap_nnzb: int = 0):
    """Halo matrix of this rank's coarse rows x ghost coarse columns.  Returns (row_ptr, col, val)."""
    n_slots = n3 + 4 * (n_coarse - n3)
    dev = new_map.device
    rp = torch.empty(n_slots + 1, dtype=torch.int64, device=dev)
    col = val = None
    P = len(peer_slot_base)
    gp = (C.c_int64 * (P + 1))(*[int(v) for v in peer_ghost_ptr])
    sb = (C.c_int64 * max(P, 1))(*[int(v) for v in peer_slot_base])
    ms = mesh.c_struct()
    bsr = _Bsr(mesh.n_nodes, H_col.shape[0], _p(H_row_ptr), _p(H_col), _p(H_val))
    n_ghost = ghost_code.shape[0] if ghost_code is not None else 0
    for attempt in range(2):
        out = _HaloMatrix(0, 0, cap_nnzb, _p(rp), _p(col), _p(val))
        st = lib().agipc_assemble_halo(h._h, C.byref(ms), _p(new_map), int(n3), int(n_coarse), C.byref(bsr),
                                       int(n_ghost), _p(ghost_code), P, gp, sb, C.byref(out))
        if st == ENOSPACE and attempt == 0:
            cap_nnzb = int(out.nnzb)
            col = torch.empty(max(cap_nnzb, 1), dtype=torch.int32, device=dev)
            val = torch.empty((max(cap_nnzb, 1), 3, 3), dtype=torch.float64, device=dev)
            continue
        h._check(st)
        break
    nb = int(out.nnzb)
    if col is None:
        col = torch.empty(0, dtype=torch.int32, device=dev)
        val = torch.empty((0, 3, 3), dtype=torch.float64, device=dev)
    return rp, col[:nb], val[:nb]


class DistPcg:
    """The rank-local half of the distributed PCG (agipc_dpcg_*).  `red` (device float64[4]) must
    be summed over the ranks after setup / spmv / update (see dist.Comm.allreduce_)."""

    def __init__(self, h: Handle, row_ptr, col, val, h_row_ptr, h_col, h_val, n_ghost_slots: int, b,
                 rel_tol: float, max_iters: int):
        self.h = h
        n = row_ptr.shape[0] - 1
        self.n = n
        self.red = torch.zeros(4, dtype=torch.float64, device=b.device)
        self._A = _Bsr(n, col.shape[0], _p(row_ptr), _p(col), _p(val))
        self._Ah = None if h_row_ptr is None else _Bsr(n, h_col.shape[0], _p(h_row_ptr), _p(h_col), _p(h_val))
        self._keep = (row_ptr, col, val, h_row_ptr, h_col, h_val, b)
        h._check(lib().agipc_dpcg_setup(h._h, C.byref(self._A), C.byref(self._Ah) if self._Ah is not None else None,
                                        int(n_ghost_slots), _p(b), float(rel_tol), int(max_iters), _p(self.red)))

    def pack(self, send_slots, sendbuf):
        self.h._check(lib().agipc_dpcg_pack(self.h._h, _p(send_slots), int(send_slots.shape[0]), _p(sendbuf)))

    def spmv(self, recvbuf):
        self.h._check(lib().agipc_dpcg_spmv(self.h._h, _p(recvbuf) if recvbuf is not None and recvbuf.numel() else None,
                                            _p(self.red)))

    def update(self):
        self.h._check(lib().agipc_dpcg_update(self.h._h, _p(self.red)))

    def status(self):
        d = C.c_int(0)
        s = _PcgStats()
        self.h._check(lib().agipc_dpcg_status(self.h._h, C.byref(d), C.byref(s)))
        return bool(d.value), dict(iters=int(s.iters), status=int(s.status), rel_residual=float(s.rel_residual))

    def finish(self, x):
        s = _PcgStats()
        self.h._check(lib().agipc_dpcg_finish(self.h._h, _p(self.red), _p(x), C.byref(s)), allow=(NOT_CONVERGED,))
        return dict(iters=int(s.iters), status=int(s.status), rel_residual=float(s.rel_residual),
                    b_norm=float(s.b_norm))


def comm_unique_id() -> bytes:
    """agipc_comm_unique_id: a fresh NCCL unique id (128 bytes) for agipc_comm_init."""
    buf = C.create_string_buffer(128)
    st = lib().agipc_comm_unique_id(buf)
    if st != OK:
        raise AgipcError(st, "agipc_comm_unique_id failed (libnccl.so.2 not loadable?)")
    return buf.raw


class Halo:
    """agipc_halo: per-peer send lists (device int32 indices) and receive row ranges."""

    def __init__(self, peer_rank, send_ptr, send_idx, recv_ptr):
        P = len(peer_rank)
        self.n_peers = P
        self._pr = (C.c_int * max(P, 1))(*[int(v) for v in peer_rank])
        self._sp = (C.c_int64 * (P + 1))(*[int(v) for v in send_ptr])
        self._rp = (C.c_int64 * (P + 1))(*[int(v) for v in recv_ptr])
        self.send_idx = send_idx
        self.c = _Halo(P, C.cast(self._pr, C.c_void_p), C.cast(self._sp, C.c_void_p),
                       _p(send_idx) if send_idx is not None and send_idx.numel() else None, C.cast(self._rp, C.c_void_p))


def comm_allgather_scan(h: Handle, local):
    """Exchange 2: local int64 [k] (device) -> (all [nranks, k], scan [2k]: exclusive prefix of this
    rank, then the totals)."""
    k = local.shape[0]
    nr = h.comm_info()["nranks"]
    all_ = torch.empty((nr, k), dtype=torch.int64, device=local.device)
    scan = torch.empty(2 * k, dtype=torch.int64, device=local.device)
    h._check(lib().agipc_comm_allgather_scan(h._h, _p(local), int(k), _p(all_), _p(scan)))
    return all_, scan


def comm_alltoall_i64(h: Handle, send):
    recv = torch.empty_like(send)
    h._check(lib().agipc_comm_alltoall_i64(h._h, _p(send), _p(recv)))
    return recv


def halo_exchange(h: Handle, halo: Halo, src, dst_ghost):
    """Rows of src (owned) to the peers; rows from the peers into dst_ghost (the ghost region)."""
    rb = src[0].numel() * src.element_size() if src.dim() > 1 else src.element_size()
    h._check(lib().agipc_halo_exchange(h._h, C.byref(halo.c), _p(src), int(rb), _p(dst_ghost)))


def dpcg_solve(h: Handle, row_ptr, col, val, h_row_ptr, h_col, h_val, n_ghost_slots: int, slots: Halo, b, x=None,
               rel_tol: float = 1e-3, max_iters: int = 10000, check_every: int = 32):
    """agipc_dpcg_solve: the distributed PCG with its NCCL exchanges inside the library."""
    n = row_ptr.shape[0] - 1
    if x is None:
        x = torch.empty((n, 3), dtype=torch.float64, device=b.device)
    A = _Bsr(n, col.shape[0], _p(row_ptr), _p(col), _p(val))
    Ah = None if h_row_ptr is None else _Bsr(n, h_col.shape[0], _p(h_row_ptr), _p(h_col) if h_col.numel() else None,
                                             _p(h_val) if h_val.numel() else None)
    stats = _PcgStats()
    st = lib().agipc_dpcg_solve(h._h, C.byref(A), C.byref(Ah) if Ah is not None else None, int(n_ghost_slots),
                                C.byref(slots.c) if slots is not None else None, _p(b), _p(x), float(rel_tol),
                                int(max_iters), int(check_every), C.byref(stats))
    h._check(st, allow=(NOT_CONVERGED,))
    return x, dict(iters=int(stats.iters), status=int(stats.status), rel_residual=float(stats.rel_residual),
                   b_norm=float(stats.b_norm))


def _tag_elems(fn, h, elems, el_slots, x_rest, x_prev, x_cur, threshold, slot_tags, reset, norm, count):
    nf = C.c_int64(0)
    h._check(getattr(lib(), fn)(h._h, int(elems.shape[0]), _p(elems), _p(el_slots), _p(x_rest), _p(x_prev), _p(x_cur),
                                float(threshold), int(slot_tags.shape[0]), int(bool(reset)), _p(slot_tags), _p(norm),
                                C.byref(nf) if count else None))
    return slot_tags, (int(nf.value) if count else None)


def tag_shells(h: Handle, tris, tri_slots, x_rest, x_prev, x_cur, threshold: float, slot_tags, reset: bool = False,
               tri_norm=None, count: bool = False):
    """NEXT#4: step 1 for triangles; flags accumulate into slot_tags unless reset."""
    return _tag_elems("agipc_tag_shells", h, tris, tri_slots, x_rest, x_prev, x_cur, threshold, slot_tags, reset,
                      tri_norm, count)


def tag_rods(h: Handle, segs, seg_slots, x_rest, x_prev, x_cur, threshold: float, slot_tags, reset: bool = False,
             seg_norm=None, count: bool = False):
    """NEXT#4: step 1 for rods (edges); flags accumulate into slot_tags unless reset."""
    return _tag_elems("agipc_tag_rods", h, segs, seg_slots, x_rest, x_prev, x_cur, threshold, slot_tags, reset,
                      seg_norm, count)


class TripletPlan:
    """NEXT#3 (supp Sec 2): the once-per-mesh key sort of the fine Hessian triplets;
    reduce(tval) -> the unique BSR values of one Newton step."""

    def __init__(self, h: Handle, n_rows: int, ti, tj, cap_nnzb: int | None = None):
        self.h = h
        dev = ti.device
        n = ti.shape[0]
        self.row_ptr = torch.empty(n_rows + 1, dtype=torch.int64, device=dev)
        self.seg_idx = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        cap = n if cap_nnzb is None else int(cap_nnzb)
        for attempt in range(2):
            self.col = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
            self.seg_ptr = torch.empty(cap + 1, dtype=torch.int64, device=dev)
            self._p = _TripletPlan(0, 0, 0, cap, _p(self.row_ptr), _p(self.col), _p(self.seg_ptr), _p(self.seg_idx))
            st = lib().agipc_triplet_plan(h._h, int(n_rows), int(n), _p(ti), _p(tj), C.byref(self._p))
            if st == ENOSPACE and attempt == 0:
                cap = int(self._p.nnzb)
                continue
            h._check(st)
            break
        self.nnzb = int(self._p.nnzb)
        self.col = self.col[:self.nnzb]

    def reduce(self, tval, out=None):
        if out is None:
            out = torch.empty((self.nnzb, 3, 3), dtype=torch.float64, device=tval.device)
        self.h._check(lib().agipc_triplet_reduce(self.h._h, C.byref(self._p), _p(tval), _p(out)))
        return out
