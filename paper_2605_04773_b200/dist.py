"""Multi-GPU partitioned coarsening step (north star).

One process per GPU.  Rank r owns a contiguous range of fine nodes (partition.LocalMesh); every
step of the path runs in libagipc's kernels on the rank's own rows, and this module only moves
buffers between ranks with torch.distributed (plumbing):

  exchange 1  x_prev / x_cur of the ghost nodes (send/recv), before tagging
  exchange 2  all-gather of the per-rank coarse slot counts -> exclusive scan = global offsets
  exchange 3  column codes of the ghost nodes (send/recv) -> the halo matrix of the coarse rows
  PCG         per iteration: send/recv of z on the ghost slots, all-reduce of [p.q] and [r.z, r.r]

With the NCCL backend the buffers stay on the GPU (NVLink).  With gloo (tests: several processes
sharing one GPU, or CPU-only host logic) they are staged through host memory; the kernels and
the numbers are the same."""
from __future__ import annotations

import dataclasses

import numpy as np
import torch
import torch.distributed as dist

from . import (CoarseBuffers, DeviceMesh, DistPcg, Handle, assemble_coarse, assemble_halo, build_map, coarse_halo,
               gather_rows, tag_edges)
from .partition import LocalMesh


class Comm:
    """Point-to-point and collective plumbing over a torch.distributed process group."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.stage = dist.get_backend(group) != "nccl"   # gloo: through host memory

    def _dev_ok(self, t):
        return t.is_cuda and not self.stage

    def allreduce_(self, t: torch.Tensor):
        """In-place sum over the ranks."""
        if self.world == 1:
            return t
        if self._dev_ok(t) or not t.is_cuda:
            dist.all_reduce(t, group=self.group)
        else:
            c = t.cpu()
            dist.all_reduce(c, group=self.group)
            t.copy_(c)
        return t

    def allgather_i64(self, vals) -> np.ndarray:
        """[world, len(vals)] int64 on the host."""
        v = torch.tensor(list(vals), dtype=torch.int64)
        if self.world == 1:
            return v.numpy()[None, :]
        if not self.stage:
            v = v.cuda()
        out = [torch.empty_like(v) for _ in range(self.world)]
        dist.all_gather(out, v, group=self.group)
        return torch.stack(out).cpu().numpy()

    def exchange(self, sends: dict, recvs: dict):
        """sends[q] / recvs[q]: tensors to send to / receive from peer q (contiguous)."""
        if not sends and not recvs:
            return
        if self.stage:
            hs = {q: t.detach().cpu() if t.is_cuda else t for q, t in sends.items()}
            hr = {q: torch.empty(t.shape, dtype=t.dtype) for q, t in recvs.items()}
            reqs = [dist.isend(hs[q], q, group=self.group) for q in sorted(hs)]
            reqs += [dist.irecv(hr[q], q, group=self.group) for q in sorted(hr)]
            for r in reqs:
                r.wait()
            for q, t in recvs.items():
                t.copy_(hr[q])
        else:
            ops = [dist.P2POp(dist.isend, sends[q], q, group=self.group) for q in sorted(sends)]
            ops += [dist.P2POp(dist.irecv, recvs[q], q, group=self.group) for q in sorted(recvs)]
            for r in dist.batch_isend_irecv(ops):
                r.wait()

    def alltoall_i64(self, send: dict) -> dict:
        """Variable-length int64 arrays: send[q] -> returns {q: array received from q}."""
        cnt = np.zeros(self.world, np.int64)
        for q, a in send.items():
            cnt[q] = len(a)
        allc = self.allgather_i64(cnt.tolist())
        dev = "cpu" if self.stage else "cuda"
        sends = {q: torch.as_tensor(np.asarray(a, np.int64), device=dev) for q, a in send.items() if len(a)}
        recvs = {q: torch.empty(int(allc[q, self.rank]), dtype=torch.int64, device=dev)
                 for q in range(self.world) if q != self.rank and allc[q, self.rank] > 0}
        self.exchange(sends, recvs)
        return {q: t.cpu().numpy() for q, t in recvs.items()}


@dataclasses.dataclass
class DistCoarse:
    """This rank's share of the coarse system."""
    cs: object               # CoarseSystem: rows and owned columns (local slot ids)
    h_row_ptr: torch.Tensor  # halo matrix: same rows, columns n_slots + ghost slot
    h_col: torch.Tensor
    h_val: torch.Tensor
    slot_offset: int         # S_r: first global slot of this rank (rank-major numbering)
    coarse_offset: int       # first global coarse node id of this rank (map parity)
    n_slots_all: np.ndarray  # [world] slot counts
    n_ghost_slots: int
    send_slots: dict         # peer -> int32 local slots to pack (z halo)
    recv_slot_range: dict    # peer -> (s0, s1) in the ghost-slot region
    map_info: dict
    n_flagged: int | None


class DistCoarseningStep:
    """Rank-local driver of steps 1-4 on a partitioned mesh."""

    def __init__(self, h: Handle, comm: Comm, lm: LocalMesh, device, group_size=32, affine_threshold=32,
                 theta=5e-5, rel_tol=1e-3, max_iters=10000, check_every=32):
        self.h, self.comm, self.lm = h, comm, lm
        self.group_size, self.affine_threshold, self.theta = group_size, affine_threshold, theta
        self.rel_tol, self.max_iters, self.check_every = rel_tol, max_iters, check_every
        t = lambda a, dt: torch.as_tensor(a).to(device=device, dtype=dt).contiguous()  # noqa: E731
        self.dmesh = DeviceMesh(t(lm.tets, torch.int32), t(lm.adj_ptr, torch.int64), t(lm.adj_nbr, torch.int32),
                                t(lm.tet_slots, torch.int32), t(lm.X, torch.float64), lm.n_own)
        self.H_ptr, self.H_col = t(lm.bsr_ptr, torch.int64), t(lm.bsr_col, torch.int32)
        self.Hh_ptr, self.Hh_col = t(lm.hbsr_ptr, torch.int64), t(lm.hbsr_col, torch.int32)
        self.send_idx = {q: t(v, torch.int32) for q, v in lm.send_idx.items()}
        self.recv_peers = sorted(lm.recv_ptr)
        self.slot_tags = torch.empty(lm.adj_nbr.shape[0], dtype=torch.uint8, device=device)
        self.map = torch.empty(lm.n_own, dtype=torch.int32, device=device)
        self.bufs = CoarseBuffers(device, lm.n_own, 4 * lm.n_own // 8 + 16, lm.bsr_col.shape[0] // 2 + 64)
        self.ghost_code = torch.empty(lm.n_ghost, dtype=torch.int32, device=device)
        self.device = device

    # -- exchange 1 -------------------------------------------------------------------------
    def halo_positions(self, *xs):
        """Fill the ghost rows of each [n_own+n_ghost, 3] array from the owners."""
        lm = self.lm
        for x in xs:
            sends = {q: gather_rows(self.h, x, idx) for q, idx in self.send_idx.items()}
            recvs = {q: x[lm.n_own + g0:lm.n_own + g1] for q, (g0, g1) in lm.recv_ptr.items()}
            self.comm.exchange(sends, recvs)

    # -- steps 1-3 + exchanges 2, 3 -----------------------------------------------------------
    def coarsen(self, x_prev, x_cur, g_own, H_val, Hh_val, count=False) -> DistCoarse:
        h, lm, comm = self.h, self.lm, self.comm
        self.halo_positions(x_prev, x_cur)
        _, nf = tag_edges(h, self.dmesh, x_prev, x_cur, self.theta, self.slot_tags, count=count)
        _, info = build_map(h, self.dmesh, self.slot_tags, self.group_size, 0, self.map)
        cs = assemble_coarse(h, self.dmesh, self.map, info["n_coarse"], self.affine_threshold, self.H_ptr, self.H_col,
                             H_val, g_own, self.bufs)
        n_c = cs.n3 + cs.n12
        # exchange 2: counts -> rank-major offsets
        allc = comm.allgather_i64([cs.n_slots, n_c])
        slot_off = int(allc[:comm.rank, 0].sum())
        coarse_off = int(allc[:comm.rank, 1].sum())
        # exchange 3: column codes of the ghosts + the per-peer ghost slot counts
        codes, send_slots = {}, {}
        for q, idx in self.send_idx.items():
            codes[q], send_slots[q] = coarse_halo(h, cs.new_map, cs.n3, n_c, idx)
        cnt = np.zeros(comm.world, np.int64)
        for q, s in send_slots.items():
            cnt[q] = s.shape[0]
        allcnt = comm.allgather_i64(cnt.tolist())
        recvs = {q: self.ghost_code[g0:g1] for q, (g0, g1) in lm.recv_ptr.items()}
        comm.exchange(codes, recvs)
        base, gptr, sbase, rng = cs.n_slots, [], [], {}
        for q in self.recv_peers:
            g0, g1 = lm.recv_ptr[q]
            m = int(allcnt[q, comm.rank])
            gptr.append(g0)
            sbase.append(base)
            rng[q] = (base - cs.n_slots, base - cs.n_slots + m)
            base += m
        gptr.append(lm.n_ghost)
        if not self.recv_peers:
            gptr = [0]
        hrp, hcol, hval = assemble_halo(h, self.dmesh, cs.new_map, cs.n3, n_c, self.Hh_ptr, self.Hh_col, Hh_val,
                                        self.ghost_code, gptr, sbase)
        return DistCoarse(cs, hrp, hcol, hval, slot_off, coarse_off, allc[:, 0].copy(), base - cs.n_slots, send_slots,
                          rng, info, nf)

    # -- step 4 -------------------------------------------------------------------------------
    def solve(self, dc: DistCoarse, x=None):
        """Distributed block-Jacobi PCG on H_c y = g_c from y0 = 0 (d_c = -y)."""
        cs, comm = dc.cs, self.comm
        n = cs.n_slots
        if x is None:
            x = torch.empty((n, 3), dtype=torch.float64, device=self.device)
        pcg = DistPcg(self.h, cs.row_ptr, cs.col, cs.val, dc.h_row_ptr, dc.h_col, dc.h_val, dc.n_ghost_slots, cs.g_c,
                      self.rel_tol, self.max_iters)
        peers_s = sorted(dc.send_slots)
        tot = sum(int(dc.send_slots[q].shape[0]) for q in peers_s)
        sendbuf = torch.empty((max(tot, 1), 3), dtype=torch.float64, device=self.device)
        recvbuf = torch.empty((max(dc.n_ghost_slots, 1), 3), dtype=torch.float64, device=self.device)
        so, sviews = 0, {}
        for q in peers_s:
            m = int(dc.send_slots[q].shape[0])
            if m:
                sviews[q] = sendbuf[so:so + m]
            so += m
        rviews = {q: recvbuf[a:b] for q, (a, b) in dc.recv_slot_range.items() if b > a}
        send_all = torch.cat([dc.send_slots[q] for q in peers_s]) if tot else None

        def halo():
            if send_all is not None:
                pcg.pack(send_all, sendbuf)
            comm.exchange(sviews, rviews)

        comm.allreduce_(pcg.red)
        halo()
        it = 0
        while it < self.max_iters:
            pcg.spmv(recvbuf)
            comm.allreduce_(pcg.red)
            pcg.update()
            comm.allreduce_(pcg.red)
            halo()
            it += 1
            if it % self.check_every == 0 and pcg.status()[0]:
                break
        st = pcg.finish(x)
        return x, st

    def __call__(self, x_prev, x_cur, g_own, H_val, Hh_val, count=False):
        dc = self.coarsen(x_prev, x_cur, g_own, H_val, Hh_val, count)
        x, st = self.solve(dc)
        return dc, x, st
