"""The library-owned communicator and workspace on one B200 (SURVEY 8(b) agipc_comm_init,
agipc_workspace_size / agipc_set_workspace; 8(e) exchanges 1-4), plus the input-validation
guarantees of the boundary (out-of-range indices never reach memory; the R22
precondition can be checked).

NCCL refuses two ranks on one device, so the NCCL data plane is exercised here with a one-rank
communicator -- including real send/recv traffic through a SELF halo: the coarse matrix is split
into owned columns and "ghost" columns whose values the rank sends to itself every PCG
iteration inside the captured graph.  The multi-rank logic (same kernels, same order) is covered
by the gloo tests (test_dist_gpu.py), which drive the split-phase calls."""
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth
from pcg_band import oracle_iteration_band
from test_dist_host import free_port

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2605_04773_b200 as P
    return P


@pytest.fixture(scope="module")
def h(P, gpu):
    h = P.Handle(0)
    h.comm_init(P.comm_unique_id(), 1, 0)
    return h


def dev(a, dt):
    return torch.as_tensor(np.ascontiguousarray(a)).to("cuda:0", dt)


@pytest.fixture(scope="module")
def c1(P, h):
    """C1 coarse system (GPU-assembled, oracle-checked in test_gpu_parity) + oracle copy."""
    m = synth.kuhn_grid(10)
    H = synth.fine_hessian(m)
    g = synth.fine_gradient(m.n_nodes)
    om = oracle.build_map(m.adj_ptr, m.adj_nbr, synth.random_tags(m, 0.2, 0), 32)
    oa = oracle.assemble(om["map"], om["n_coarse"], 32, m.X, m.bsr_ptr, m.bsr_col, H, g)
    return m, H, g, om, oa


def test_comm_info_and_collectives(P, h):
    info = h.comm_info()
    assert info["nranks"] == 1 and info["rank"] == 0 and info["nccl_version"] >= 22000
    all_, scan = P.comm_allgather_scan(h, torch.tensor([5, 7, -2], dtype=torch.int64, device="cuda:0"))
    assert all_.cpu().tolist() == [[5, 7, -2]] and scan.cpu().tolist() == [0, 0, 0, 5, 7, -2]
    r = P.comm_alltoall_i64(h, torch.tensor([42], dtype=torch.int64, device="cuda:0"))
    assert r.cpu().tolist() == [42]


@pytest.mark.parametrize("row_cols,dt", [(3, torch.float64), (1, torch.int32), (5, torch.float32)])
def test_halo_exchange_self(P, h, row_cols, dt):
    rng = np.random.default_rng(row_cols)
    n_own = 1000
    src = dev(rng.standard_normal((n_own, row_cols)) * 100, dt)
    idx = rng.integers(0, n_own, 137).astype(np.int32)
    ghosts = torch.full((200, row_cols), -1, dtype=dt, device="cuda:0")
    halo = P.Halo([0], [0, idx.shape[0]], dev(idx, torch.int32), [11, 11 + idx.shape[0]])
    P.halo_exchange(h, halo, src, ghosts)
    torch.cuda.synchronize()
    assert torch.equal(ghosts[11:11 + 137], src[torch.as_tensor(idx, dtype=torch.long, device="cuda:0")])
    assert torch.all(ghosts[:11] == -1) and torch.all(ghosts[148:] == -1)


@pytest.mark.parametrize("always", [0, 1])
def test_dpcg_solve_one_rank_equals_pcg_solve(P, h, c1, always):
    """always = 1: the one-rank NCCL all-reduces are issued (AGIPC_OPT_COMM_ALWAYS) and captured."""
    _, _, _, _, oa = c1
    h.set_option(P.OPT_COMM_ALWAYS, always)
    rp, col, val, b = (dev(oa["row_ptr"], torch.int64), dev(oa["col"], torch.int32), dev(oa["val"], torch.float64),
                       dev(oa["g_c"], torch.float64))
    for tol in (1e-3, 1e-10):
        x1, s1 = P.pcg_solve(h, rp, col, val, b, rel_tol=tol, max_iters=10000, zero_x0=True, check_every=8)
        x2, s2 = P.dpcg_solve(h, rp, col, val, None, None, None, 0, None, b, rel_tol=tol, max_iters=10000,
                              check_every=8)
        # same kernels and the same reductions (a one-rank all-reduce is the identity): bit for bit
        assert s2["status"] == P.OK and s2["iters"] == s1["iters"]
        assert torch.equal(x1, x2)
    h.set_option(P.OPT_COMM_ALWAYS, 0)


def test_pcg_bitwise_reproducible(P, h, c1):
    """Static slice schedule + fixed-order reductions: two solves agree bit for bit."""
    _, _, _, _, oa = c1
    args = (dev(oa["row_ptr"], torch.int64), dev(oa["col"], torch.int32), dev(oa["val"], torch.float64),
            dev(oa["g_c"], torch.float64))
    x1, s1 = P.pcg_solve(h, *args, rel_tol=1e-10, zero_x0=True)
    for _ in range(3):
        x2, s2 = P.pcg_solve(h, *args, rel_tol=1e-10, zero_x0=True)
        assert s2["iters"] == s1["iters"] and torch.equal(x1, x2)


def _self_split(oa, every=3):
    """Owned columns j % every != 0 and the diagonal blocks (block-Jacobi reads them from the owned
    part, as on a real rank), ghost columns (sent to self) j % every == 0 off the diagonal."""
    n = oa["n_slots"]
    S = np.arange(0, n, every)
    gidx = -np.ones(n, np.int64)
    gidx[S] = np.arange(S.shape[0])
    rows = np.repeat(np.arange(n), np.diff(oa["row_ptr"]))
    col = oa["col"]
    loc = (gidx[col] < 0) | (col == rows)
    loc_rp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows[loc], minlength=n), out=loc_rp[1:])
    h_rp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows[~loc], minlength=n), out=h_rp[1:])
    return (S.astype(np.int32), loc_rp, col[loc], oa["val"][loc], h_rp, (n + gidx[col[~loc]]).astype(np.int32),
            oa["val"][~loc])


@pytest.mark.parametrize("every", [2, 3, 7])
def test_dpcg_solve_self_halo_matches_oracle(P, h, c1, every):
    """NCCL send/recv of z inside the captured graph every iteration (self peer)."""
    _, _, _, _, oa = c1
    S, lrp, lcol, lval, hrp, hcol, hval = _self_split(oa, every)
    halo = P.Halo([0], [0, S.shape[0]], dev(S, torch.int32), [0, S.shape[0]])
    x, s = P.dpcg_solve(h, dev(lrp, torch.int64), dev(lcol, torch.int32), dev(lval, torch.float64),
                        dev(hrp, torch.int64), dev(hcol, torch.int32), dev(hval, torch.float64), S.shape[0], halo,
                        dev(oa["g_c"], torch.float64), rel_tol=1e-10, max_iters=10000, check_every=16)
    assert s["status"] == P.OK
    rr = oracle.rel_residual(oa["row_ptr"], oa["col"], oa["val"], x.cpu().numpy(), oa["g_c"])
    assert rr <= 1.01e-10 * 100 and rr <= 1e-8, rr
    _, s3 = P.dpcg_solve(h, dev(lrp, torch.int64), dev(lcol, torch.int32), dev(lval, torch.float64),
                         dev(hrp, torch.int64), dev(hcol, torch.int32), dev(hval, torch.float64), S.shape[0], halo,
                         dev(oa["g_c"], torch.float64), rel_tol=1e-3, max_iters=10000, check_every=16)
    lo, hi = oracle_iteration_band(oa["row_ptr"], oa["col"], oa["val"], oa["g_c"], 1e-3)
    assert lo <= s3["iters"] <= hi, (s3, lo, hi)


def test_dpcg_solve_singular_and_not_converged(P, h, c1):
    _, _, _, _, oa = c1
    val = oa["val"].copy()
    d = np.flatnonzero(np.repeat(np.arange(oa["n_slots"]), np.diff(oa["row_ptr"])) == oa["col"])[3]
    val[d] = 0.0
    with pytest.raises(P.AgipcError) as e:
        P.dpcg_solve(h, dev(oa["row_ptr"], torch.int64), dev(oa["col"], torch.int32), dev(val, torch.float64), None,
                     None, None, 0, None, dev(oa["g_c"], torch.float64), rel_tol=1e-8)
    assert e.value.status == P.ESINGULAR
    _, s = P.dpcg_solve(h, dev(oa["row_ptr"], torch.int64), dev(oa["col"], torch.int32),
                        dev(oa["val"], torch.float64), None, None, None, 0, None, dev(oa["g_c"], torch.float64),
                        rel_tol=1e-14, max_iters=7, check_every=4)
    assert s["status"] == P.NOT_CONVERGED and s["iters"] == 7


def test_libcomm_step_one_rank_equals_single_gpu(P, gpu, tmp_path):
    """DistCoarseningStep over the library communicator (world 1) == the 1-GPU CoarseningStep."""
    mp.start_processes(_libcomm_worker, args=(free_port(), str(tmp_path)), nprocs=1, start_method="spawn")
    errs = [f.read_text() for f in tmp_path.glob("err*")]
    assert not errs, errs
    assert (tmp_path / "ok0").exists()


def _libcomm_worker(rank, port, out_dir):
    import traceback
    import torch.distributed as dist
    import paper_2605_04773_b200 as P
    from paper_2605_04773_b200 import partition as pt
    from paper_2605_04773_b200.dist import DistCoarseningStep, LibComm
    from paper_2605_04773_b200.step import CoarseningStep
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
        torch.cuda.set_device(0)
        G, gid = synth.kuhn_box(12, slabs=1)
        H = synth.fine_hessian(G)
        g = synth.fine_gradient(G.n_nodes, seed=1)
        xp, xc = synth.twist(G.X, 0.5), synth.twist(G.X, 0.501)
        b = pt.slab_bounds(12, 1)
        lm = pt.attach_halo([pt.local_mesh(G, gid, b[0], b[1], b, 0)])[0]
        h = P.Handle(0)
        h.set_option(P.OPT_DETERMINISTIC, 1)  # bitwise-comparable coarse systems on both paths
        comm = LibComm(h)
        d = torch.device("cuda:0")
        td = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(d)  # noqa: E731
        step = DistCoarseningStep(h, comm, lm, d, rel_tol=1e-8, max_iters=50000, check_every=8)
        dc = step.coarsen(td(xp), td(xc), td(g), td(H[lm.loc_src]), td(H[lm.halo_src]))
        x, st = step.solve(dc)
        h1 = P.Handle(0)
        h1.set_option(P.OPT_DETERMINISTIC, 1)
        dm = P.DeviceMesh.from_arrays(G.tets, G.adj_ptr, G.adj_nbr, G.tet_slots, G.X, device=d)
        one = CoarseningStep(h1, dm, td(G.bsr_ptr), td(G.bsr_col), td(H), rel_tol=1e-8, max_iters=50000,
                             check_every=8)
        nf, info, cs = one.coarsen(td(xp), td(xc), td(g))
        x1, st1 = one.solve(cs)
        assert dc.cs.n_slots == cs.n_slots and dc.cs.nnzb == cs.nnzb and dc.n_ghost_slots == 0
        assert torch.equal(dc.cs.new_map, cs.new_map) and torch.equal(dc.cs.col, cs.col)
        # the same kernels on the same (bitwise-equal) coarse system: the distributed solve over
        # the one-rank communicator equals the 1-GPU solve
        assert torch.equal(dc.cs.val, cs.val) and torch.equal(dc.cs.g_c, cs.g_c)
        assert st["iters"] == st1["iters"] and st["status"] == P.OK
        assert torch.equal(x, x1)
        dist.destroy_process_group()
        open(os.path.join(out_dir, "ok0"), "w").write("ok")
    except Exception:
        open(os.path.join(out_dir, "err0"), "w").write(traceback.format_exc())
        raise


# ---------------------------------------------------------------------------------------------
# caller-owned workspace
# ---------------------------------------------------------------------------------------------
def test_caller_owned_workspace(P, gpu, c1):
    m, H, g, om, oa = c1
    hw = P.Handle(0)
    dm = P.DeviceMesh.from_arrays(m.tets, m.adj_ptr, m.adj_nbr, m.tet_slots, m.X, device="cuda:0")
    args = (dev(m.bsr_ptr, torch.int64), dev(m.bsr_col, torch.int32), dev(H, torch.float64))
    est = hw.workspace_size(m.n_nodes, m.n_tets, m.adj_nbr.shape[0], m.bsr_col.shape[0])
    assert est > 0
    # too small: ENOSPACE, nothing crashes; then the size the handle reports works
    hw.set_workspace(torch.empty(4096, dtype=torch.uint8, device="cuda:0"))
    tags = dev(synth.random_tags(m, 0.2, 0), torch.uint8)
    with pytest.raises(P.AgipcError) as e:
        P.build_map(hw, dm, tags, 32)
    assert e.value.status == P.ENOSPACE
    need = hw.workspace_size(m.n_nodes, m.n_tets, m.adj_nbr.shape[0], m.bsr_col.shape[0])
    arena = torch.empty(need, dtype=torch.uint8, device="cuda:0")
    hw.set_workspace(arena)
    before = torch.cuda.memory_allocated()
    mp_, info = P.build_map(hw, dm, tags, 32)
    cs = P.assemble_coarse(hw, dm, mp_, info["n_coarse"], 32, *args, dev(g, torch.float64))
    x, s = P.pcg_solve(hw, cs.row_ptr, cs.col, cs.val, cs.g_c, rel_tol=1e-10, zero_x0=True)
    assert np.array_equal(mp_.cpu().numpy(), om["map"]) and np.array_equal(cs.col.cpu().numpy(), oa["col"])
    rr = oracle.rel_residual(oa["row_ptr"], oa["col"], oa["val"], x.cpu().numpy(), oa["g_c"])
    assert rr <= 1.01e-10 * 10
    # a second step reuses the arena; the library allocated nothing through torch (outputs aside)
    hw.set_workspace(arena)
    x2, s2 = P.pcg_solve(hw, cs.row_ptr, cs.col, cs.val, cs.g_c, rel_tol=1e-10, zero_x0=True)
    assert s2["iters"] == s["iters"] and torch.equal(x, x2)
    assert hw.workspace_size() <= need
    hw.set_workspace(None)  # back to internal buffers
    x3, _ = P.pcg_solve(hw, cs.row_ptr, cs.col, cs.val, cs.g_c, rel_tol=1e-10, zero_x0=True)
    assert torch.equal(x, x3)
    del before


# ---------------------------------------------------------------------------------------------
# input validation at the boundary
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("bad", [2 ** 31 - 2, -5, 3])
def test_assemble_out_of_range_map_is_einval_and_context_survives(P, h, bad):
    m = synth.kuhn_grid(6)
    dm = P.DeviceMesh.from_arrays(m.tets, m.adj_ptr, m.adj_nbr, m.tet_slots, m.X, device="cuda:0")
    H = synth.fine_hessian(m)
    mp_ = np.zeros(m.n_nodes, np.int32)
    mp_[m.n_nodes // 2:] = 1
    mp_[[5, 77, m.n_nodes - 1]] = bad
    args = (dev(m.bsr_ptr, torch.int64), dev(m.bsr_col, torch.int32), dev(H, torch.float64))
    with pytest.raises(P.AgipcError) as e:
        P.assemble_coarse(h, dm, dev(mp_, torch.int32), 3, 32, *args)
    assert e.value.status == P.EINVAL
    torch.cuda.synchronize()  # no sticky error: the context is intact
    good = np.minimum(np.arange(m.n_nodes) // 40, 4).astype(np.int32)
    cs = P.assemble_coarse(h, dm, dev(good, torch.int32), 5, 32, *args)
    oa = oracle.assemble(good, 5, 32, m.X, m.bsr_ptr, m.bsr_col, H)
    assert np.array_equal(cs.col.cpu().numpy(), oa["col"])


@pytest.mark.parametrize("which,bad", [("ti", 2 ** 31 - 2), ("ti", -5), ("ti", 50), ("tj", -3)])
def test_triplet_plan_out_of_range_is_einval(P, h, which, bad):
    rng = np.random.default_rng(1)
    ti = rng.integers(0, 50, 400).astype(np.int32)
    tj = rng.integers(0, 50, 400).astype(np.int32)
    (ti if which == "ti" else tj)[[3, 200]] = bad
    with pytest.raises(P.AgipcError) as e:
        P.TripletPlan(h, 50, dev(ti, torch.int32), dev(tj, torch.int32))
    assert e.value.status == P.EINVAL
    torch.cuda.synchronize()


def test_symmetry_check_option(P, gpu):
    hs = P.Handle(0)
    hs.set_option(P.OPT_CHECK_SYMMETRY, 1)
    m = synth.kuhn_grid(5)
    dm = P.DeviceMesh.from_arrays(m.tets, m.adj_ptr, m.adj_nbr, m.tet_slots, m.X, device="cuda:0")
    H = synth.fine_hessian(m)
    mp_ = (np.arange(m.n_nodes) // 50).astype(np.int32)
    nc = int(mp_.max()) + 1
    args = (dev(m.bsr_ptr, torch.int64), dev(m.bsr_col, torch.int32))
    P.assemble_coarse(hs, dm, dev(mp_, torch.int32), nc, 32, *args, dev(H, torch.float64))  # symmetric: OK
    Hb = H.copy()
    off = np.flatnonzero(np.repeat(np.arange(m.n_nodes), np.diff(m.bsr_ptr)) != m.bsr_col)[10]
    Hb[off, 0, 1] += 1e-9  # one off-diagonal block is no longer the transpose of its mirror
    with pytest.raises(P.AgipcError) as e:
        P.assemble_coarse(hs, dm, dev(mp_, torch.int32), nc, 32, *args, dev(Hb, torch.float64))
    assert e.value.status == P.EINVAL and "symmetric" in str(e.value)
    hs.set_option(P.OPT_CHECK_SYMMETRY, 0)
    P.assemble_coarse(hs, dm, dev(mp_, torch.int32), nc, 32, *args, dev(Hb, torch.float64))  # unchecked
