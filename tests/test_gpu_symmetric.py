"""GPU parity for NEXT#2, symmetric (diagonal + upper) storage (main Sec 6), through the C
ABI: agipc_bsr_upper bit-exact against the oracle's extraction; agipc_pcg_solve_sym (storage SYM:
upper half of a full matrix, UPPER: upper storage input) under the PCG contract of
test_gpu_parity (oracle-evaluated residual, iteration band of reading R25), including rows split
into several SELL segments, rows straddling scatter windows, x0 != 0 and the error paths."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from pcg_band import oracle_iteration_band

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2605_04773_b200 as P
    return P


@pytest.fixture(scope="module")
def h(P, gpu):
    return P.Handle(0)


def dev(a, dt):
    return torch.as_tensor(np.ascontiguousarray(a)).to("cuda:0", dt)


def coarse_c1(thr=32, p=0.2, seed=0):
    m = synth.kuhn_grid(10)
    H = synth.fine_hessian(m)
    g = synth.fine_gradient(m.n_nodes)
    om = oracle.build_map(m.adj_ptr, m.adj_nbr, synth.random_tags(m, p, seed), 32)
    return oracle.assemble(om["map"], om["n_coarse"], thr, m.X, m.bsr_ptr, m.bsr_col, H, g)


def arrow_spd(n=700, dense=(3, 150, 351, 500, 690), seed=0):
    """Symmetric block matrix with a few dense rows/columns (rows of >> 64 blocks, split into
    several SELL segments) and a random sparse part; block diagonally dominant => SPD."""
    rng = np.random.default_rng(seed)
    pairs = set()
    for i in range(n):
        for j in rng.integers(0, n, 6):
            if i != j:
                pairs.add((min(i, j), max(i, j)))
    for d in dense:
        for j in range(n):
            if j != d:
                pairs.add((min(d, j), max(d, j)))
    blocks = {}
    for (i, j) in pairs:
        B = rng.standard_normal((3, 3)) * 0.1
        blocks[(i, j)] = B
        blocks[(j, i)] = B.T.copy()
    rowsum = np.zeros(n)
    for (i, j), B in blocks.items():
        rowsum[i] += np.abs(B).sum()
    for i in range(n):
        S = rng.standard_normal((3, 3)) * 0.1
        blocks[(i, i)] = (S + S.T) / 2 + (rowsum[i] + 1.0) * np.eye(3)
    keys = sorted(blocks)
    rp = np.zeros(n + 1, np.int64)
    for (i, _) in keys:
        rp[i + 1] += 1
    rp = np.cumsum(rp)
    col = np.array([j for (_, j) in keys], np.int32)
    val = np.array([blocks[k] for k in keys])
    return rp, col, val


def check_solve(P, h, rp, col, val, b, storage, tol, band=True):
    if storage == P.STORAGE_UPPER:
        urp, ucol, uval = oracle.bsr_upper(rp, col, val)
        A = (dev(urp, torch.int64), dev(ucol, torch.int32), dev(uval, torch.float64))
    else:
        A = (dev(rp, torch.int64), dev(col, torch.int32), dev(val, torch.float64))
    x, s = P.pcg_solve(h, *A, dev(b, torch.float64), rel_tol=tol, max_iters=50000, zero_x0=True, storage=storage)
    assert s["status"] == P.OK, s
    rr = oracle.rel_residual(rp, col, val, x.cpu().numpy(), b)
    assert rr <= max(tol, 1e-8) * 1.01, rr
    if band:
        # the symmetric SpMV scatters its transposed products with fp64 atomics (no fixed
        # summation order): the band of the partitioned solve, reading R25 (16 copies, +- 4)
        lo, hi = oracle_iteration_band(rp, col, val, b, tol, n_pert=16, slack=4)
        assert lo <= s["iters"] <= hi, (s["iters"], lo, hi)
    return x, s


def test_bsr_upper_bit_exact(P, h):
    oa = coarse_c1(thr=5)
    m = synth.kuhn_grid(10)
    for rp, col, val in ((oa["row_ptr"], oa["col"], oa["val"]), (m.bsr_ptr, m.bsr_col, synth.fine_hessian(m)),
                         arrow_spd()):
        urp, ucol, uval = P.bsr_upper(h, dev(rp, torch.int64), dev(col, torch.int32), dev(val, torch.float64))
        orp, ocol, oval = oracle.bsr_upper(rp, col, val)
        assert np.array_equal(urp.cpu().numpy(), orp)
        assert np.array_equal(ucol.cpu().numpy(), ocol)
        assert np.array_equal(uval.cpu().numpy(), oval)
    # capacity retry: too small a capacity -> ENOSPACE with the count, then success
    urp, ucol, uval = P.bsr_upper(h, dev(rp, torch.int64), dev(col, torch.int32), dev(val, torch.float64), cap_nnzb=3)
    assert ucol.shape[0] == orp[-1]


@pytest.mark.parametrize("storage", [1, 2])
@pytest.mark.parametrize("thr", [32, 5])
def test_pcg_sym_c1(P, h, storage, thr):
    # the iteration-count contract is at the paper's tolerance (reading R25); the scatter
    # sums in no fixed order, so at 1e-10 only the oracle-evaluated residual is the contract
    oa = coarse_c1(thr=thr)
    for tol in (1e-3, 1e-10):
        check_solve(P, h, oa["row_ptr"], oa["col"], oa["val"], oa["g_c"], storage, tol, band=tol >= 1e-3)


@pytest.mark.parametrize("win", ["128", "1024", "4096"])
@pytest.mark.parametrize("storage", [1, 2])
def test_pcg_sym_long_rows_and_windows(P, h, storage, win):
    rp, col, val = arrow_spd()
    urp, _, _ = oracle.bsr_upper(rp, col, val)
    assert np.diff(urp).max() > 3 * 64         # several SELL segments in the upper half of a row
    b = np.random.default_rng(1).standard_normal((rp.shape[0] - 1, 3))
    os.environ["AGIPC_SYM_WIN"] = win
    try:
        check_solve(P, h, rp, col, val, b, storage, 1e-10, band=False)
    finally:
        del os.environ["AGIPC_SYM_WIN"]


def test_pcg_sym_special_cases_and_errors(P, h):
    n = 10
    rp = dev(np.arange(n + 1, dtype=np.int64), torch.int64)
    cl = dev(np.arange(n, dtype=np.int32), torch.int32)
    I = dev(np.tile(np.eye(3), (n, 1, 1)), torch.float64)
    b = dev(np.random.default_rng(0).standard_normal((n, 3)), torch.float64)
    for storage in (P.STORAGE_SYM, P.STORAGE_UPPER):
        x, s = P.pcg_solve(h, rp, cl, I, b, rel_tol=1e-12, zero_x0=True, storage=storage)
        assert s["iters"] == 1 and torch.allclose(x, b, rtol=1e-15, atol=0)
        x, s = P.pcg_solve(h, rp, cl, I, torch.zeros_like(b), rel_tol=1e-3, zero_x0=True, storage=storage)
        assert s["iters"] == 0 and torch.all(x == 0)
        with pytest.raises(P.AgipcError) as e:
            P.pcg_solve(h, rp, cl, -I, b, rel_tol=1e-3, zero_x0=True, storage=storage)
        assert e.value.status == P.EINDEFINITE
        Z = I.clone(); Z[3] = 0
        with pytest.raises(P.AgipcError) as e:
            P.pcg_solve(h, rp, cl, Z, b, rel_tol=1e-3, zero_x0=True, storage=storage)
        assert e.value.status == P.ESINGULAR
        x, s = P.pcg_solve(h, rp, cl, 2 * I, b, x=b.clone(), rel_tol=1e-12, storage=storage)   # x0 != 0
        assert torch.allclose(x, b / 2, rtol=1e-14)
    # a full-storage matrix passed as upper storage is rejected
    m = synth.kuhn_grid(4)
    H = synth.fine_hessian(m)
    with pytest.raises(P.AgipcError) as e:
        P.pcg_solve(h, dev(m.bsr_ptr, torch.int64), dev(m.bsr_col, torch.int32), dev(H, torch.float64),
                    dev(synth.fine_gradient(m.n_nodes), torch.float64), zero_x0=True, storage=P.STORAGE_UPPER)
    assert e.value.status == P.EINVAL
    with pytest.raises(P.AgipcError) as e:
        P.pcg_solve(h, rp, cl, I, b, zero_x0=True, storage=7)
    assert e.value.status == P.EINVAL


@pytest.mark.parametrize("storage", [1, 2])
def test_pcg_sym_not_converged_and_nonzero_x0(P, h, storage):
    m = synth.kuhn_grid(8)
    H = synth.fine_hessian(m)
    g = synth.fine_gradient(m.n_nodes)
    if storage == 2:
        A = [dev(a, dt) for a, dt in zip(oracle.bsr_upper(m.bsr_ptr, m.bsr_col, H),
                                          (torch.int64, torch.int32, torch.float64))]
    else:
        A = [dev(m.bsr_ptr, torch.int64), dev(m.bsr_col, torch.int32), dev(H, torch.float64)]
    x, s = P.pcg_solve(h, *A, dev(g, torch.float64), rel_tol=1e-14, max_iters=7, check_every=3, zero_x0=True,
                       storage=storage)
    assert s["status"] == P.NOT_CONVERGED and s["iters"] == 7
    ref = oracle.pcg(m.bsr_ptr, m.bsr_col, H, g, rel_tol=1e-14, max_iters=7)
    assert np.allclose(x.cpu().numpy(), ref["x"], rtol=1e-9, atol=1e-12 * np.abs(ref["x"]).max())
    # nonzero x0 (the post-coarsening fine CG starts from d_f): r0 = b - A x0
    x0 = np.random.default_rng(3).standard_normal(g.shape) * 1e-3
    x, s = P.pcg_solve(h, *A, dev(g, torch.float64), x=dev(x0, torch.float64), rel_tol=1e-3, max_iters=10,
                       storage=storage)
    ref = oracle.pcg(m.bsr_ptr, m.bsr_col, H, g, x0=x0, rel_tol=1e-3, max_iters=10)
    assert s["iters"] == ref["iters"] and s["status"] == ref["status"]
    assert np.linalg.norm(x.cpu().numpy() - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_pcg_sym_full_size(P, h, cfg):
    """The coarse systems bench.py times, solved with the symmetric SpMV."""
    c = synth.config_c2() if cfg == "c2" else synth.config_c3()
    m = c["mesh"]
    H = synth.fine_hessian(m, E=c["E"])
    g = synth.fine_gradient(m.n_nodes)
    ot, _, _ = oracle.tag_edges(m.tets, m.tet_slots, m.X, c["x_prev"], c["x_cur"], c["theta"], m.adj_nbr.shape[0])
    om = oracle.build_map(m.adj_ptr, m.adj_nbr, ot, 32)
    oa = oracle.assemble(om["map"], om["n_coarse"], 32, m.X, m.bsr_ptr, m.bsr_col, H, g)
    check_solve(P, h, oa["row_ptr"], oa["col"], oa["val"], oa["g_c"], P.STORAGE_SYM, 1e-8, band=False)
    if cfg == "c2":
        check_solve(P, h, oa["row_ptr"], oa["col"], oa["val"], oa["g_c"], P.STORAGE_SYM, 1e-3, band=True)
        check_solve(P, h, oa["row_ptr"], oa["col"], oa["val"], oa["g_c"], P.STORAGE_UPPER, 1e-3, band=True)


def test_bsr_expand_upper_bit_exact(P, h):
    """Fine Hessians arrive in symmetric storage; the device expansion equals the
    oracle's definition bit for bit and inverts agipc_bsr_upper."""
    cases = []
    for n in (10, 47):
        m = synth.kuhn_grid(n)
        cases.append((m.bsr_ptr, m.bsr_col, synth.fine_hessian(m)))
    oa = coarse_c1(thr=5)
    cases.append((oa["row_ptr"], oa["col"], oa["val"]))
    cases.append(arrow_spd())
    for rp, col, val in cases:
        urp, ucol, uval = oracle.bsr_upper(rp, col, val)
        ref, miss = oracle.bsr_expand_upper(rp, col, urp, ucol, uval)
        assert miss == 0
        drp, dcol = dev(rp, torch.int64), dev(col, torch.int32)
        out = P.bsr_expand_upper(h, drp, dcol, dev(urp, torch.int64), dev(ucol, torch.int32), dev(uval, torch.float64))
        assert np.array_equal(out.cpu().numpy(), ref)
        sym = all(np.array_equal(val[e], val[np.searchsorted(col[rp[j]:rp[j + 1]], i) + rp[j]].T)
                  for i in range(len(rp) - 1) for e in range(rp[i], rp[i + 1]) for j in [col[e]])
        if sym:  # the synthetic fine Hessians are bitwise symmetric: expansion restores them
            assert np.array_equal(out.cpu().numpy(), val)
        # round trip through the device selection; unchecked (stream-ordered) variant
        u2 = P.bsr_upper(h, drp, dcol, dev(val, torch.float64))
        out2 = P.bsr_expand_upper(h, drp, dcol, *u2, check=False)
        assert np.array_equal(out2.cpu().numpy(), ref)
    # a pattern that is not the symmetric closure of U's is rejected
    rp, col, val = cases[0]
    urp, ucol, uval = oracle.bsr_upper(rp, col, val)
    bad = ucol.copy()
    bad[urp[1] - 1] += 1                                          # last upper column of row 0 shifted
    with pytest.raises(P.AgipcError) as e:
        P.bsr_expand_upper(h, dev(rp, torch.int64), dev(col, torch.int32), dev(urp, torch.int64),
                           dev(bad, torch.int32), dev(uval, torch.float64))
    assert e.value.status == P.EINVAL


def test_values_event_orders_a_late_upload(P, h):
    """agipc_set_values_event: the numeric assembly waits for values uploaded on another stream
    (delayed here by a spin kernel), so the result equals the synchronous one bit for bit."""
    from paper_2605_04773_b200.step import CoarseningStep
    c = synth.config_c1()
    m = c["mesh"]
    H = synth.fine_hessian(m)
    g = synth.fine_gradient(m.n_nodes)
    dm = P.DeviceMesh.from_arrays(m.tets, m.adj_ptr, m.adj_nbr, m.tet_slots, m.X, device="cuda:0")
    rp, cl = dev(m.bsr_ptr, torch.int64), dev(m.bsr_col, torch.int32)
    xp, xc = dev(c["x_prev"], torch.float64), dev(c["x_cur"], torch.float64)
    ref_step = CoarseningStep(h, dm, rp, cl, dev(H, torch.float64))
    _, _, ref = ref_step.coarsen(xp, xc, dev(g, torch.float64))
    ref_val, ref_g = ref.val.clone(), ref.g_c.clone()
    dH = torch.zeros((m.bsr_col.shape[0], 3, 3), dtype=torch.float64, device="cuda:0")
    dg = torch.zeros((m.n_nodes, 3), dtype=torch.float64, device="cuda:0")
    hH = torch.as_tensor(H).pin_memory()
    hg = torch.as_tensor(g).pin_memory()
    side = torch.cuda.Stream()
    ready = torch.cuda.Event()
    step = CoarseningStep(h, dm, rp, cl, dH)
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        torch.cuda._sleep(20_000_000)            # ~10 ms: the upload lands long after steps 1-2
        dH.copy_(hH, non_blocking=True)
        dg.copy_(hg, non_blocking=True)
        ready.record(side)
    _, info, cs = step.coarsen(xp, xc, dg, hessian_ready=ready)
    torch.cuda.synchronize()
    # same contract as the synchronous result: the 12-DoF rows sum with fp64 atomics, so two runs
    # agree to rounding, both within 1e-12 of the oracle's |.|-Galerkin bound
    om = oracle.build_map(m.adj_ptr, m.adj_nbr, step.slot_tags.cpu().numpy(), 32)
    oa = oracle.assemble(om["map"], om["n_coarse"], 32, m.X, m.bsr_ptr, m.bsr_col, H, g)
    assert np.array_equal(cs.col.cpu().numpy(), oa["col"])
    for v, gc in ((cs.val, cs.g_c), (ref_val, ref_g)):
        assert np.all(np.abs(v.cpu().numpy() - oa["val"]) <= 1e-12 * oa["bound"])
        assert np.all(np.abs(gc.cpu().numpy() - oa["g_c"]) <= 1e-12 * oa["g_bound"])
