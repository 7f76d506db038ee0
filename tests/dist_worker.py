"""Multi-process workers for the partitioned path.  Spawned by test_dist_host.py
(CPU, gloo: host logic) and test_dist_gpu.py (several ranks sharing one GPU, gloo staging:
the full distributed step through libagipc, checked against the oracle run with
segments = rank bounds, reading R24)."""
import os
import sys
import traceback

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)


def _init(rank, world, port):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)


def host_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    import synth
    from paper_2605_04773_b200 import partition as pt
    from paper_2605_04773_b200.dist import Comm
    try:
        _init(rank, world, port)
        comm = Comm()
        assert comm.rank == rank and comm.world == world and comm.stage
        # collectives
        t = torch.tensor([rank + 1.0, 2.0 * rank], dtype=torch.float64)
        comm.allreduce_(t)
        assert t.tolist() == [sum(range(1, world + 1)), 2.0 * sum(range(world))]
        g = comm.allgather_i64([rank, 10 * rank])
        assert g.tolist() == [[q, 10 * q] for q in range(world)]
        got = comm.alltoall_i64({q: np.arange(rank + q + 1) + 100 * rank for q in range(world) if q != rank})
        for q in range(world):
            if q != rank:
                assert got[q].tolist() == (np.arange(q + rank + 1) + 100 * q).tolist()
        # halo lists by request exchange == the single-process construction
        n = 5
        G, gid = synth.kuhn_box(n, slabs=world)
        b = pt.slab_bounds(n, world)
        ref = pt.attach_halo([pt.local_mesh(G, gid, b[r], b[r + 1], b, r) for r in range(world)])[rank]
        r = rank
        S, gs = synth.kuhn_box(n, slabs=world, z_lo=max(0, r * n - 1), z_hi=min(world * n - 1, (r + 1) * n))
        lm = pt.local_mesh(S, gs, b[r], b[r + 1], b, r)
        pt.exchange_requests(lm, world, comm.alltoall_i64)
        assert lm.peers == ref.peers and lm.recv_ptr == ref.recv_ptr
        for q in ref.send_idx:
            assert np.array_equal(lm.send_idx[q], ref.send_idx[q])
        # a halo exchange of positions (host tensors) fills exactly the ghost rows
        X = torch.as_tensor(lm.X.copy())
        X[lm.n_own:] = float("nan")
        sends = {q: X[torch.as_tensor(idx, dtype=torch.int64)] for q, idx in lm.send_idx.items()}
        recvs = {q: X[lm.n_own + g0:lm.n_own + g1] for q, (g0, g1) in lm.recv_ptr.items()}
        comm.exchange(sends, recvs)
        assert np.array_equal(X.numpy(), lm.X)
        dist.barrier()
        dist.destroy_process_group()
        open(os.path.join(out_dir, f"ok{rank}"), "w").write("ok")
    except Exception:
        open(os.path.join(out_dir, f"err{rank}"), "w").write(traceback.format_exc())
        raise


def gpu_worker(rank, world, port, out_dir, n, thr, kind):
    import torch
    import torch.distributed as dist
    import oracle
    import synth
    import paper_2605_04773_b200 as P
    from paper_2605_04773_b200 import partition as pt
    from paper_2605_04773_b200.dist import Comm, DistCoarseningStep
    try:
        _init(rank, world, port)
        torch.cuda.set_device(0)
        comm = Comm()
        h = P.Handle(0)
        if kind == "c4":  # multi-object contact scene split mid-object (contact blocks become halo)
            sc = synth.c4_scene(n=n, k=2)
            G = sc["mesh"]
            gid = np.arange(G.n_nodes)
            b = [int(round(r * G.n_nodes / world)) for r in range(world + 1)]
            H = synth.c4_hessian(sc)
        elif kind == "thin":  # bench --strong: ONE n^3 cube cut into world slabs of n x n x n/world
            G, gid = synth.kuhn_box(n, slabs=world, t=n // world)
            b = pt.slab_bounds(n, world, n // world)
            H = synth.fine_hessian(G)
        else:
            G, gid = synth.kuhn_box(n, slabs=world)
            b = pt.slab_bounds(n, world)
            H = synth.fine_hessian(G)
        lm = pt.local_mesh(G, gid, b[rank], b[rank + 1], b, rank)
        pt.exchange_requests(lm, world, comm.alltoall_i64)
        g = synth.fine_gradient(G.n_nodes, seed=1)
        if kind == "c4":
            xp, xc = synth.c4_iterates(sc)
            theta = 5e-5
        elif kind == "twist":
            xp, xc, theta = synth.twist(G.X, 0.5, w=0.2 * world), synth.twist(G.X, 0.501, w=0.2 * world), 5e-5
        else:
            rng = np.random.default_rng(3)
            xp = G.X + 1e-3 * rng.standard_normal(G.X.shape)
            xc = xp + 1e-4 * rng.standard_normal(G.X.shape)
            theta = float(np.quantile(oracle.tag_edges(G.tets, G.tet_slots, G.X, xp, xc, 1.0,
                                                       G.adj_nbr.shape[0])[1], 0.6))
        dev = torch.device("cuda:0")
        own = slice(b[rank], b[rank + 1])
        td = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        x_prev = torch.full((lm.n_own + lm.n_ghost, 3), float("nan"), dtype=torch.float64, device=dev)
        x_cur = x_prev.clone()
        x_prev[:lm.n_own] = td(xp[own])
        x_cur[:lm.n_own] = td(xc[own])
        step = DistCoarseningStep(h, comm, lm, dev, affine_threshold=thr, theta=theta, rel_tol=1e-8,
                                  max_iters=50000, check_every=8)
        dc = step.coarsen(x_prev, x_cur, td(g[own]), td(H[lm.loc_src]), td(H[lm.halo_src]))
        # exchange 1 filled the ghosts with the owners' values
        assert torch.equal(x_cur.cpu(), torch.as_tensor(xc[lm.gid]))
        # step 1: tags of the rank's slots == the oracle's global tags (bit-exact)
        ot, _, _ = oracle.tag_edges(G.tets, G.tet_slots, G.X, xp, xc, theta, G.adj_nbr.shape[0])
        assert np.array_equal(step.slot_tags.cpu().numpy(), ot[lm.slot_src])
        # step 2: rank-local recursion == the oracle with segments = rank bounds (R24)
        om = oracle.build_map(G.adj_ptr, G.adj_nbr, ot, 32, seg_begin=np.asarray(b, np.int64))
        assert np.array_equal(step.map.cpu().numpy() + dc.coarse_offset, om["map"][own])
        assert dc.coarse_offset + dc.map_info["n_coarse"] <= om["n_coarse"]
        # step 3: the rank's coarse rows (owned + halo columns) == oracle rows (1e-12 of the bound)
        oa = oracle.assemble(om["map"], om["n_coarse"], thr, G.X, G.bsr_ptr, G.bsr_col, H, g)
        cs = dc.cs
        nm_all = comm_allgather_obj(comm, (dc.slot_offset, cs.n3, cs.new_map.cpu().numpy().tolist()))
        # oracle slot -> distributed global slot, built from every fine node
        perm = -np.ones(oa["n_slots"], np.int64)
        for r in range(world):
            so, n3r, nmr = nm_all[r]
            nmr = np.asarray(nmr)
            o_nm = oa["new_map"][b[r]:b[r + 1]]
            for f in range(nmr.shape[0]):
                c, co = int(nmr[f]), int(o_nm[f])
                ob = co if co < oa["n3"] else oa["n3"] + 4 * (co - oa["n3"])
                db = so + (c if c < n3r else n3r + 4 * (c - n3r))
                for p in range(1 if co < oa["n3"] else 4):
                    perm[ob + p] = db + p
        assert np.all(perm >= 0) and np.array_equal(np.sort(perm), np.arange(oa["n_slots"]))
        inv = np.argsort(perm)
        # halo columns -> global slots via the owners' send lists
        sends = {q: (dc.slot_offset + s.cpu().numpy()).tolist() for q, s in dc.send_slots.items()}
        all_sends = comm_allgather_obj(comm, sends)
        hcol_g = np.empty(dc.n_ghost_slots, np.int64)
        for q, (a0, a1) in dc.recv_slot_range.items():
            lst = all_sends[q][rank]
            assert len(lst) == a1 - a0
            hcol_g[a0:a1] = lst
        rp, col, val = cs.row_ptr.cpu().numpy(), cs.col.cpu().numpy(), cs.val.cpu().numpy()
        hrp, hcol, hval = dc.h_row_ptr.cpu().numpy(), dc.h_col.cpu().numpy(), dc.h_val.cpu().numpy()
        for s in range(cs.n_slots):
            orow = inv[dc.slot_offset + s]
            ok0, ok1 = oa["row_ptr"][orow], oa["row_ptr"][orow + 1]
            ocols = perm[oa["col"][ok0:ok1]]
            order = np.argsort(ocols)
            mycols = np.concatenate([dc.slot_offset + col[rp[s]:rp[s + 1]],
                                     hcol_g[hcol[hrp[s]:hrp[s + 1]] - cs.n_slots]])
            myvals = np.concatenate([val[rp[s]:rp[s + 1]], hval[hrp[s]:hrp[s + 1]]])
            mo = np.argsort(mycols)
            assert np.array_equal(mycols[mo], ocols[order]), s
            dv = np.abs(myvals[mo] - oa["val"][ok0:ok1][order])
            assert np.all(dv <= 1e-12 * oa["bound"][ok0:ok1][order]), (s, dv.max())
            assert np.all(np.abs(cs.g_c[s].cpu().numpy() - oa["g_c"][orow]) <= 1e-12 * oa["g_bound"][orow])
        # step 4: distributed PCG; the oracle evaluates the residual of the gathered solution
        x, st = step.solve(dc)
        xs = comm_allgather_obj(comm, x.cpu().numpy().tolist())
        xd = np.concatenate([np.asarray(v).reshape(-1, 3) for v in xs])
        rr = oracle.rel_residual(oa["row_ptr"], oa["col"], oa["val"], xd[perm], oa["g_c"])
        assert st["status"] == P.OK and rr <= 1.01e-8, (st, rr)
        step.rel_tol = 1e-3
        _, st3 = step.solve(dc)
        from pcg_band import oracle_iteration_band  # reading R25
        lo, hi = oracle_iteration_band(oa["row_ptr"], oa["col"], oa["val"], oa["g_c"], 1e-3, n_pert=16, slack=4)
        assert lo <= st3["iters"] <= hi, (st3, lo, hi)
        ref = {"iters": (lo, hi)}
        dist.barrier()
        dist.destroy_process_group()
        open(os.path.join(out_dir, f"ok{rank}"), "w").write(f"{st} {st3['iters']} {ref['iters']} {rr}")
    except Exception:
        open(os.path.join(out_dir, f"err{rank}"), "w").write(traceback.format_exc())
        raise


def comm_allgather_obj(comm, obj):
    import torch.distributed as dist
    out = [None] * comm.world
    dist.all_gather_object(out, obj)
    return out


def singular_worker(rank, world, port, out_dir):
    """a singular diagonal block on ONE rank must stop every rank (no hang)."""
    import torch
    import torch.distributed as dist
    import paper_2605_04773_b200 as P
    from paper_2605_04773_b200.dist import Comm, split_phase_solve
    try:
        _init(rank, world, port)
        torch.cuda.set_device(0)
        comm = Comm()
        h = P.Handle(0)
        n = 6
        d = torch.device("cuda:0")
        rp = torch.arange(n + 1, dtype=torch.int64, device=d)
        col = torch.arange(n, dtype=torch.int32, device=d)
        val = torch.eye(3, dtype=torch.float64, device=d).repeat(n, 1, 1) * (rank + 2.0)
        if rank == world - 1:
            val[2] = 0.0
        b = torch.ones((n, 3), dtype=torch.float64, device=d)
        x = torch.empty_like(b)
        try:
            split_phase_solve(h, comm, rp, col, val, None, None, None, 0, {}, {}, b, x, 1e-8, 1000, 4)
            status = "ok"
        except P.AgipcError as e:
            status = P._status_name(e.status)
        dist.barrier()
        dist.destroy_process_group()
        open(os.path.join(out_dir, f"ok{rank}"), "w").write(status)
    except Exception:
        open(os.path.join(out_dir, f"err{rank}"), "w").write(traceback.format_exc())
        raise
