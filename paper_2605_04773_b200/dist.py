"""Multi-GPU partitioned coarsening step (north star).

One process per GPU.  Rank r owns a contiguous range of fine nodes (partition.LocalMesh); every
step of the path runs in libagipc's kernels on the rank's own rows.  The exchanges:

  exchange 1  x_prev / x_cur of the ghost nodes (send/recv), before tagging
  exchange 2  all-gather of the per-rank coarse slot counts -> exclusive scan = global offsets
  exchange 3  column codes of the ghost nodes (send/recv) -> the halo matrix of the coarse rows
  PCG         per iteration: send/recv of z on the ghost slots, all-reduce of [p.q] and [r.z, r.r]

Two transports with the same kernels in the same order:
  LibComm  (GPU runs, one process per GPU): the library's own NCCL communicator
           (agipc_comm_init; torch.distributed only broadcasts its 128-byte unique id) -- every
           exchange is an agipc_* call (agipc_halo_exchange, agipc_comm_allgather_scan,
           agipc_comm_alltoall_i64) and the PCG is agipc_dpcg_solve, NCCL calls captured in its
           CUDA graph: no torch collective on the hot path;
  Comm     (tests: several processes sharing one GPU -- NCCL refuses two ranks on one device --
           or CPU-only host logic): torch.distributed over gloo staging through host memory,
           driving the split-phase agipc_dpcg_* calls."""
from __future__ import annotations

import dataclasses

import numpy as np
import torch
import torch.distributed as dist

from . import (CoarseBuffers, DeviceMesh, DistPcg, Halo, Handle, assemble_coarse, assemble_halo, build_map,
               coarse_halo, comm_allgather_scan, comm_alltoall_i64, comm_unique_id, dpcg_solve, gather_rows,
               halo_exchange, tag_edges)
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


class LibComm:
    """The library-owned NCCL communicator of handle h (agipc_comm_init).  The process group is used
    once, to broadcast rank 0's 128-byte unique id (plumbing)."""

    def __init__(self, h: Handle, group=None):
        self.h = h
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        uid = [comm_unique_id() if self.rank == 0 else None]
        dist.broadcast_object_list(uid, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        h.comm_init(uid[0], self.world, self.rank)


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

    def __init__(self, h: Handle, comm, lm: LocalMesh, device, group_size=32, affine_threshold=32,
                 theta=5e-5, rel_tol=1e-3, max_iters=10000, check_every=32):
        self.h, self.comm, self.lm = h, comm, lm
        self.lib = isinstance(comm, LibComm)
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
        if self.lib:  # node halo for agipc_halo_exchange: peers ascending, concatenated send lists
            peers = sorted(set(lm.send_idx) | set(lm.recv_ptr))
            sp, rp, idx = [0], [0], []
            for q in peers:
                si = lm.send_idx.get(q, np.zeros(0, np.int32))
                idx.append(np.asarray(si, np.int32))
                sp.append(sp[-1] + len(si))
                g0, g1 = lm.recv_ptr.get(q, (rp[-1], rp[-1]))
                assert g0 == rp[-1], "ghost ranges must follow the ascending peer order"
                rp.append(g1)
            self.peers = peers
            self.node_send_all = t(np.concatenate(idx) if idx else np.zeros(0, np.int32), torch.int32)
            self.node_halo = Halo(peers, sp, self.node_send_all, rp)
            n_send = sp[-1]
            self.code_send = torch.empty(max(n_send, 1), dtype=torch.int32, device=device)
            self.code_halo = Halo(peers, sp, torch.arange(n_send, dtype=torch.int32, device=device), rp)
            self.node_send_ptr = sp

    # -- exchange 1 -------------------------------------------------------------------------
    def halo_positions(self, *xs):
        """Fill the ghost rows of each [n_own+n_ghost, 3] array from the owners."""
        lm = self.lm
        if self.lib:
            for x in xs:
                halo_exchange(self.h, self.node_halo, x, x[lm.n_own:])
            return
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
        if self.lib:
            return self._coarsen_lib(cs, info, nf, H_val, Hh_val)
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

    def _coarsen_lib(self, cs, info, nf, H_val, Hh_val) -> DistCoarse:
        """Exchanges 2 and 3 through the library communicator (device buffers, NCCL)."""
        h, lm, comm = self.h, self.lm, self.comm
        n_c = cs.n3 + cs.n12
        dev = self.device
        # exchange 2: all-gather exclusive scan of (n_slots, n_coarse) on the device
        local = torch.tensor([cs.n_slots, n_c], dtype=torch.int64, device=dev)
        allc, scan = comm_allgather_scan(h, local)
        # exchange 3: column codes of the sent nodes (concatenated in peer order) and slot counts
        send_slots, cnt_send = {}, torch.zeros(comm.world, dtype=torch.int64)
        sp = self.node_send_ptr
        for k, q in enumerate(self.peers):
            if sp[k + 1] > sp[k]:
                code, sl = coarse_halo(h, cs.new_map, cs.n3, n_c, self.node_send_all[sp[k]:sp[k + 1]],
                                       ghost_code=self.code_send[sp[k]:sp[k + 1]])
                send_slots[q] = sl
                cnt_send[q] = sl.shape[0]
        halo_exchange(h, self.code_halo, self.code_send, self.ghost_code)
        cnt_recv = comm_alltoall_i64(h, cnt_send.to(dev)).cpu().numpy()
        sc = scan.cpu().numpy()
        allc_h = allc.cpu().numpy()
        base, gptr, sbase, rng = cs.n_slots, [], [], {}
        for q in self.recv_peers:
            g0, g1 = lm.recv_ptr[q]
            m = int(cnt_recv[q])
            gptr.append(g0)
            sbase.append(base)
            rng[q] = (base - cs.n_slots, base - cs.n_slots + m)
            base += m
        gptr.append(lm.n_ghost)
        if not self.recv_peers:
            gptr = [0]
        hrp, hcol, hval = assemble_halo(h, self.dmesh, cs.new_map, cs.n3, n_c, self.Hh_ptr, self.Hh_col, Hh_val,
                                        self.ghost_code, gptr, sbase)
        return DistCoarse(cs, hrp, hcol, hval, int(sc[0]), int(sc[1]), allc_h[:, 0].copy(), base - cs.n_slots,
                          send_slots, rng, info, nf)

    # -- step 4 -------------------------------------------------------------------------------
    def solve(self, dc: DistCoarse, x=None):
        """Distributed block-Jacobi PCG on H_c y = g_c from y0 = 0 (d_c = -y)."""
        cs, comm = dc.cs, self.comm
        n = cs.n_slots
        if x is None:
            x = torch.empty((n, 3), dtype=torch.float64, device=self.device)
        if self.lib:  # agipc_dpcg_solve: halo + all-reduces inside the library's CUDA graph
            peers = sorted(set(dc.send_slots) | set(dc.recv_slot_range))
            sp, rp, idx = [0], [0], []
            for q in peers:
                sl = dc.send_slots.get(q)
                idx.append(sl if sl is not None else torch.zeros(0, dtype=torch.int32, device=self.device))
                sp.append(sp[-1] + (sl.shape[0] if sl is not None else 0))
                a, b = dc.recv_slot_range.get(q, (rp[-1], rp[-1]))
                assert a == rp[-1]
                rp.append(b)
            send_all = torch.cat(idx) if idx else torch.zeros(0, dtype=torch.int32, device=self.device)
            slots = Halo(peers, sp, send_all, rp)
            return dpcg_solve(self.h, cs.row_ptr, cs.col, cs.val, dc.h_row_ptr, dc.h_col, dc.h_val, dc.n_ghost_slots,
                              slots, cs.g_c, x, self.rel_tol, self.max_iters, self.check_every)
        return split_phase_solve(self.h, comm, cs.row_ptr, cs.col, cs.val, dc.h_row_ptr, dc.h_col, dc.h_val,
                                 dc.n_ghost_slots, dc.send_slots, dc.recv_slot_range, cs.g_c, x, self.rel_tol,
                                 self.max_iters, self.check_every)

    def __call__(self, x_prev, x_cur, g_own, H_val, Hh_val, count=False):
        dc = self.coarsen(x_prev, x_cur, g_own, H_val, Hh_val, count)
        x, st = self.solve(dc)
        return dc, x, st


def split_phase_solve(h: Handle, comm: Comm, row_ptr, col, val, h_row_ptr, h_col, h_val, n_ghost_slots: int,
                      send_slots: dict, recv_slot_range: dict, b, x, rel_tol: float, max_iters: int, check_every: int):
    """The distributed PCG driven from the host over a torch.distributed Comm (the gloo transport of
    the tests): the split-phase agipc_dpcg_* calls with the all-reduces and the z halo in between --
    the kernel sequence agipc_dpcg_solve captures with NCCL.  Returns (x, stats); a library error
    (e.g. ESINGULAR on any rank: the setup sums carry the flag) raises on every rank alike."""
    dev = b.device
    pcg = DistPcg(h, row_ptr, col, val, h_row_ptr, h_col, h_val, n_ghost_slots, b, rel_tol, max_iters)
    peers_s = sorted(send_slots)
    tot = sum(int(send_slots[q].shape[0]) for q in peers_s)
    sendbuf = torch.empty((max(tot, 1), 3), dtype=torch.float64, device=dev)
    recvbuf = torch.empty((max(n_ghost_slots, 1), 3), dtype=torch.float64, device=dev)
    so, sviews = 0, {}
    for q in peers_s:
        m = int(send_slots[q].shape[0])
        if m:
            sviews[q] = sendbuf[so:so + m]
        so += m
    rviews = {q: recvbuf[a:b_] for q, (a, b_) in recv_slot_range.items() if b_ > a}
    send_all = torch.cat([send_slots[q] for q in peers_s]) if tot else None

    def halo():
        if send_all is not None:
            pcg.pack(send_all, sendbuf)
        comm.exchange(sviews, rviews)

    comm.allreduce_(pcg.red)
    halo()
    it = 0
    while it < max_iters:
        pcg.spmv(recvbuf)  # consumes the reduced sums of the previous call (k_dscalars) first
        comm.allreduce_(pcg.red)
        pcg.update()
        comm.allreduce_(pcg.red)
        halo()
        it += 1
        # the done flag is only read after the first spmv has applied the reduced setup sums, so
        # every rank sees the same flag (a singular block on one rank stops all of them)
        if it % check_every == 0 and pcg.status()[0]:
            break
    st = pcg.finish(x)
    return x, st
