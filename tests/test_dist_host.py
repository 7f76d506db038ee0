"""Host-side logic of the partitioned path on CPU: partition invariants, the
segmented oracle == rank-local oracle runs (reading R24), and the communicator / halo-request
exchange in a world_size-2 gloo job."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import synth
from paper_2605_04773_b200 import partition as pt


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n,R,t", [(4, 2, None), (5, 3, None), (6, 2, 3), (6, 3, 2)])
def test_partition_invariants(n, R, t):
    G, gid = synth.kuhn_box(n, slabs=R, t=t)
    b = pt.slab_bounds(n, R, t)
    lms = pt.attach_halo([pt.local_mesh(G, gid, b[r], b[r + 1], b, r) for r in range(R)])
    assert sum(lm.n_own for lm in lms) == G.n_nodes
    # every global BSR block of a row appears exactly once, in H_loc or H_halo of its owner
    seen = np.concatenate([np.concatenate([lm.loc_src, lm.halo_src]) for lm in lms])
    assert np.array_equal(np.sort(seen), np.arange(G.bsr_col.shape[0]))
    for lm in lms:
        # local columns map back to the right global columns
        rows = np.repeat(np.arange(lm.n_own), np.diff(lm.bsr_ptr))
        assert np.array_equal(lm.gid[lm.bsr_col], G.bsr_col[lm.loc_src])
        assert np.array_equal(lm.gid[lm.n_own + lm.hbsr_col], G.bsr_col[lm.halo_src])
        assert np.array_equal(lm.gid[rows], np.repeat(np.arange(G.n_nodes), np.diff(G.bsr_ptr))[lm.loc_src])
        # tet slots point at the directed edge of the global mesh
        for e, (a, c) in enumerate(pt.TET_EDGES):
            s = lm.tet_slots[:, 2 * e]
            ok = s >= 0
            u = lm.gid[lm.tets[ok, a]]
            v = lm.gid[lm.tets[ok, c]]
            gs = lm.slot_src[s[ok]]
            gr = np.repeat(np.arange(G.n_nodes), np.diff(G.adj_ptr))
            assert np.array_equal(gr[gs], u) and np.array_equal(G.adj_nbr[gs], v)
        # every tet touching an owned node is present
        own = (gid >= b[lm.rank]) & (gid < b[lm.rank + 1])
        assert lm.tets.shape[0] == int(own[G.tets].any(axis=1).sum())
        # halo symmetry
        for q, (g0, g1) in lm.recv_ptr.items():
            assert np.array_equal(lms[q].gid[lms[q].send_idx[lm.rank]], lm.gid[lm.n_own + g0:lm.n_own + g1])


@pytest.mark.parametrize("p", [0.3, 0.6, 1.0])
def test_rank_local_oracle_equals_segmented_oracle(p):
    """R24: the map of the partitioned path (each rank runs the recursion on its own rows)
    equals the oracle run on the global mesh with segments = rank bounds."""
    n, R = 6, 3
    G, gid = synth.kuhn_box(n, slabs=R)
    b = pt.slab_bounds(n, R)
    tags = synth.random_tags(G, p, 5)
    og = oracle.build_map(G.adj_ptr, G.adj_nbr, tags, 32, seg_begin=np.asarray(b, np.int64))
    off = 0
    levels = 0
    for r in range(R):
        lm = pt.local_mesh(G, gid, b[r], b[r + 1], b, r)
        ol = oracle.build_map(lm.adj_ptr, lm.adj_nbr, tags[lm.slot_src], 32)
        assert np.array_equal(ol["map"] + off, og["map"][b[r]:b[r + 1]])
        off += ol["n_coarse"]
        levels = max(levels, ol["n_levels"])
    assert off == og["n_coarse"] and levels == og["n_levels"]


def test_comm_and_halo_requests_gloo_world2(tmp_path):
    from dist_worker import host_worker
    mp.start_processes(host_worker, args=(2, free_port(), str(tmp_path)), nprocs=2, start_method="spawn")
    errs = [f.read_text() for f in tmp_path.glob("err*")]
    assert not errs, errs
    assert sorted(os.listdir(tmp_path)) == ["ok0", "ok1"]


def _ijk_sets(m):
    ijk = m.ijk.astype(np.int64)
    tets = np.sort(ijk[m.tets] @ np.array([1 << 40, 1 << 20, 1]), axis=1)
    return ijk, tets[np.lexsort(tets.T[::-1])]


@pytest.mark.parametrize("n,R", [(6, 1), (6, 2), (6, 3), (8, 4)])
def test_thin_slab_box_is_the_cube(n, R):
    """--strong cuts ONE n^3 cube into R slabs of n x n x n/R: the slab box has the cube's nodes,
    positions and tets (as ijk sets); at R = 1 its numbering is the cube's Morton numbering."""
    C = synth.kuhn_grid(n)
    B, gid = synth.kuhn_box(n, slabs=R, t=n // R)
    assert np.array_equal(gid, np.arange(n ** 3))
    ci, ct = _ijk_sets(C)
    bi, bt = _ijk_sets(B)
    key = lambda a: (a[:, 0] * n + a[:, 1]) * n + a[:, 2]  # noqa: E731
    oc, ob = np.argsort(key(ci)), np.argsort(key(bi))
    assert np.array_equal(ci[oc], bi[ob])
    assert np.allclose(C.X[oc], B.X[ob], rtol=0, atol=1e-15)
    assert np.array_equal(ct, bt)
    if R == 1:
        assert np.array_equal(ci, bi)


def test_strong_partitions_solve_one_problem():
    """bench --strong: for every rank count the ranks' owned rows together hold the same
    physical problem (g_f, the wall displacements, the fine Hessian rows), keyed by the global
    lexicographic node (i n + j) n + k."""
    import bench
    n = 8
    ref = None
    for R in (1, 2, 4):
        gs, ds, hs = {}, {}, {}
        for r in range(R):
            lm, Hl, Hh, g, disp, _ = bench.build_partition(n, R, r, strong=True)
            # lexicographic key of every local node from its position (spacing 1/(n-1), centred)
            ijk = np.rint((lm.X + np.array([0.5, 0.5, 0.5])) * (n - 1)).astype(np.int64)
            key = (ijk[:, 0] * n + ijk[:, 1]) * n + ijk[:, 2]
            for v in range(lm.n_own):
                gs[key[v]] = g[v]
                ds[key[v]] = np.stack([d[v] for d in disp[:3]])
                for s in range(lm.bsr_ptr[v], lm.bsr_ptr[v + 1]):
                    hs[(key[v], key[lm.bsr_col[s]])] = Hl[s]
                for s in range(lm.hbsr_ptr[v], lm.hbsr_ptr[v + 1]):
                    hs[(key[v], key[lm.n_own + lm.hbsr_col[s]])] = Hh[s]
        assert len(gs) == n ** 3
        if ref is None:
            ref = (gs, ds, hs)
            continue
        assert all(np.array_equal(gs[k], ref[0][k]) and np.array_equal(ds[k], ref[1][k]) for k in gs)
        assert hs.keys() == ref[2].keys()
        assert all(np.allclose(hs[k], ref[2][k], rtol=1e-13, atol=0) for k in hs)
