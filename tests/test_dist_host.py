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


@pytest.mark.parametrize("n,R", [(4, 2), (5, 3)])
def test_partition_invariants(n, R):
    G, gid = synth.kuhn_box(n, slabs=R)
    b = pt.slab_bounds(n, R)
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
