"""One Newton iteration of the coarsening path (main Alg 1 lines 8-10):
tag -> map -> assemble -> coarse PCG, composed from the four C-ABI calls, optionally followed
by NEXT#1: prolongation d_f = U^T d_c and <= refine_iters fine PCG iterations from d_f.  Plumbing only:
all arithmetic runs in libagipc's kernels."""
from __future__ import annotations

import dataclasses

import torch

from . import (STORAGE_FULL, CoarseBuffers, DeviceMesh, Handle, assemble_coarse, build_map, pcg_solve, prolongate,
               tag_edges)


@dataclasses.dataclass
class StepResult:
    n_flagged: int | None
    map_info: dict
    coarse: object
    x: torch.Tensor
    pcg: dict
    y_f: torch.Tensor | None = None   # refined fine solution of H_f y = g_f; direction d_f = -y_f (NEXT#1)
    refine: dict | None = None


class CoarseningStep:
    """Holds the device-resident static inputs and grow-only buffers of the path."""

    def __init__(self, h: Handle, mesh: DeviceMesh, H_row_ptr, H_col, H_val, group_size=32,
                 affine_threshold=32, theta=5e-5, rel_tol=1e-3, max_iters=10000, check_every=16,
                 refine_iters=0, pcg_storage=STORAGE_FULL):
        self.h, self.mesh = h, mesh
        self.pcg_storage = pcg_storage  # STORAGE_SYM: the coarse SpMV streams the upper half (NEXT#2)
        self.H = (H_row_ptr, H_col, H_val)
        self.group_size, self.affine_threshold, self.theta = group_size, affine_threshold, theta
        self.rel_tol, self.max_iters, self.check_every = rel_tol, max_iters, check_every
        dev = mesh.x_rest.device
        self.slot_tags = torch.empty(mesh.adj_nbr.shape[0], dtype=torch.uint8, device=dev)
        self.map = torch.empty(mesh.n_nodes, dtype=torch.int32, device=dev)
        self.bufs = CoarseBuffers(dev, mesh.n_nodes, 4 * mesh.n_nodes // 8 + 16, H_col.shape[0] // 2 + 64)
        self.x = None
        self.refine_iters = refine_iters
        if refine_iters > 0:  # the fine solve of every Newton step reuses one SELL layout of H_f
            h.pcg_set_static(H_row_ptr, H_col)
        self.y_f = torch.empty((mesh.n_nodes, 3), dtype=torch.float64, device=dev)

    def coarsen(self, x_prev, x_cur, g_fine, count=False, hessian_ready=None):
        """Steps 1-3.  Returns (n_flagged, map_info, CoarseSystem).  hessian_ready: optional CUDA
        event the numeric assembly waits for (steps 1-2 and the classification / symbolic parts of
        step 3 do not read H_f or g_f values, so their upload can overlap them on another stream)."""
        _, nf = tag_edges(self.h, self.mesh, x_prev, x_cur, self.theta, self.slot_tags, count=count)
        _, info = build_map(self.h, self.mesh, self.slot_tags, self.group_size, 0, self.map)
        if hessian_ready is not None:
            self.h.set_values_event(hessian_ready)
        cs = assemble_coarse(self.h, self.mesh, self.map, info["n_coarse"], self.affine_threshold, *self.H,
                             g_fine, self.bufs)
        return nf, info, cs

    def solve(self, cs):
        """Step 4: H_c y = g_c from y0 = 0; the coarse direction of P:752 is d_c = -y."""
        n = cs.n_slots
        if self.x is None or self.x.shape[0] < n:
            self.x = torch.empty((int(n * 1.25) + 16, 3), dtype=torch.float64, device=cs.val.device)
        x = self.x[:n]
        _, st = pcg_solve(self.h, cs.row_ptr, cs.col, cs.val, cs.g_c, x, self.rel_tol, self.max_iters,
                          self.check_every, zero_x0=True, storage=self.pcg_storage)
        return x, st

    def refine(self, cs, y_c, g_fine):
        """NEXT#1: y_f = U^T y_c, then <= refine_iters block-Jacobi PCG iterations on
        H_f y = g_f from y_f.  CG is linear in (b, x0), so the fine direction is d_f = -y_f."""
        y = prolongate(self.h, self.mesh, cs.new_map, cs.n3, cs.n_slots, y_c, 1.0, self.y_f)
        y, st = pcg_solve(self.h, *self.H, g_fine, y, self.rel_tol, self.refine_iters, self.check_every)
        return y, st

    def __call__(self, x_prev, x_cur, g_fine, count=False) -> StepResult:
        nf, info, cs = self.coarsen(x_prev, x_cur, g_fine, count)
        x, st = self.solve(cs)
        if self.refine_iters <= 0:
            return StepResult(nf, info, cs, x, st)
        y, rst = self.refine(cs, x, g_fine)
        return StepResult(nf, info, cs, x, st, y_f=y, refine=rst)
