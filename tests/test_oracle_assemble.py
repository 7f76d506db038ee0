"""Pins for the oracle's DoF classification / reorder (supp Alg S3),
Galerkin coarse Hessian and gradient (supp Alg S4 + Eq S2/S3; main
Eq 4; H_c = U H_f U^T): dense U H U^T with an explicitly
built U, closed forms (affine rigid modes), special cases, SPEC/Table S1 fixtures."""
import numpy as np
import pytest

import oracle
import synth
from conftest import read_golden, read_golden_rows


def bsr_dense(rp, col, val, n):
    A = np.zeros((3 * n, 3 * n))
    for r in range(n):
        for k in range(rp[r], rp[r + 1]):
            A[3 * r:3 * r + 3, 3 * col[k]:3 * col[k] + 3] += val[k]
    return A


def explicit_U(new_map, n3, X):
    """U of shape (3 n_slots) x (3 N): I3 for a 3-DoF parent, X_bar_f[p] I3 in
    slot p of a 12-DoF parent (A_f = X_bar (x) I3)."""
    N = new_map.shape[0]
    n12 = (new_map.max() + 1 - n3) if N and new_map.max() >= n3 else 0
    ns = n3 + 4 * n12
    U = np.zeros((3 * ns, 3 * N))
    for f in range(N):
        c = new_map[f]
        if c < n3:
            U[3 * c:3 * c + 3, 3 * f:3 * f + 3] = np.eye(3)
        else:
            w = [X[f, 0], X[f, 1], X[f, 2], 1.0]
            for p in range(4):
                s = n3 + 4 * (c - n3) + p
                U[3 * s:3 * s + 3, 3 * f:3 * f + 3] = w[p] * np.eye(3)
    return U


def fine(m, **kw):
    return m.bsr_ptr, m.bsr_col, synth.fine_hessian(m, **kw)


@pytest.mark.parametrize("seed", range(6))
def test_dense_galerkin_random_maps(seed):
    """Random (not necessarily connected) maps and thresholds on <= 30-node meshes:
    oracle == dense U H_f U^T and U g_f within 1e-12 of the |.|-Galerkin bound,
    and the bound equals |U| |H_f| |U|^T."""
    rng = np.random.default_rng(seed)
    m = synth.kuhn_grid(3)  # 27 nodes
    N = m.n_nodes
    rp, cl, H = fine(m, E=10.0 ** rng.uniform(4, 7))
    g = rng.standard_normal((N, 3))
    n_c = int(rng.integers(1, N + 1))
    mp = np.concatenate([np.arange(n_c), rng.integers(0, n_c, N - n_c)])
    rng.shuffle(mp)
    thr = int(rng.integers(0, 6))
    o = oracle.assemble(mp, n_c, thr, m.X, rp, cl, H, g)
    sizes = np.bincount(mp, minlength=n_c)
    is12 = sizes > thr
    assert o["n12"] == is12.sum() and o["n3"] == n_c - is12.sum()
    # stable partition (Alg S3, R13): 3-DoF in ascending c, then 12-DoF ascending
    newid = np.empty(n_c, int)
    newid[~is12] = np.arange((~is12).sum())
    newid[is12] = (~is12).sum() + np.arange(is12.sum())
    assert np.array_equal(o["new_map"], newid[mp])
    U = explicit_U(o["new_map"], o["n3"], m.X)
    Hf = bsr_dense(rp, cl, H, N)
    Hc = U @ Hf @ U.T
    B = np.abs(U) @ np.abs(Hf) @ np.abs(U).T
    A = bsr_dense(o["row_ptr"], o["col"], o["val"], o["n_slots"])
    Ab = bsr_dense(o["row_ptr"], o["col"], o["bound"], o["n_slots"])
    assert np.all(np.abs(A - Hc) <= 1e-12 * B + 1e-300)
    assert np.allclose(Ab, B, rtol=1e-13, atol=0)
    gc = U @ g.reshape(-1)
    assert np.all(np.abs(o["g_c"].reshape(-1) - gc) <= 1e-12 * (np.abs(U) @ np.abs(g.reshape(-1))) + 1e-300)
    # canonical BSR: ascending columns, structural pattern = blocks with a contribution
    for r in range(o["n_slots"]):
        cols = o["col"][o["row_ptr"][r]:o["row_ptr"][r + 1]]
        assert np.all(np.diff(cols) > 0)
    # structural (R17): every (slot(a,p), slot(b,q)) reached by a stored fine block,
    # whatever the weight or block values (zero X_bar coordinates included)
    Us = explicit_U(o["new_map"], o["n3"], np.ones_like(m.X))
    Hs = bsr_dense(rp, cl, np.ones_like(H), N)
    blk = (Us @ Hs @ Us.T).reshape(o["n_slots"], 3, o["n_slots"], 3).sum(axis=(1, 3)) > 0
    assert blk.sum() == o["nnzb"]


def test_identity_map_reproduces_fine_system_exactly():
    """All edges protected -> identity map, all 3-DoF -> H_c == H_f and g_c == g_f
    bit-exactly (one contribution per coarse block)."""
    m = synth.kuhn_grid(5)
    rp, cl, H = fine(m)
    g = synth.fine_gradient(m.n_nodes, 3)
    o = oracle.assemble(np.arange(m.n_nodes), m.n_nodes, 32, m.X, rp, cl, H, g)
    assert o["n12"] == 0 and np.array_equal(o["row_ptr"], rp) and np.array_equal(o["col"], cl)
    assert np.array_equal(o["val"], H) and np.array_equal(o["g_c"], g)


def test_mass_only_single_3dof_aggregate():
    """All fine nodes -> one 3-DoF node, mass-only H -> (sum m) I."""
    m = synth.kuhn_grid(4)
    rp, cl, H = fine(m, stiffness=False)
    o = oracle.assemble(np.zeros(m.n_nodes, np.int32), 1, 10 ** 9, m.X, rp, cl, H)
    M = synth.lumped_mass(m)
    assert o["nnzb"] == 1
    assert np.allclose(o["val"][0], M.sum() * np.eye(3), rtol=1e-14, atol=0)
    assert np.isclose(M.sum(), 1000.0, rtol=1e-12)  # rho * unit volume


def test_pure_stiffness_collapsed_to_one_3dof_node_vanishes():
    """K 1 = 0 (translation invariance): the collapsed 3-DoF block is 0 up to the bound."""
    m = synth.kuhn_grid(5)
    rp, cl, H = fine(m, mass=False, dt=1.0)
    o = oracle.assemble(np.zeros(m.n_nodes, np.int32), 1, 10 ** 9, m.X, rp, cl, H)
    assert np.all(np.abs(o["val"][0]) <= 1e-13 * o["bound"][0])


@pytest.mark.parametrize("origin", [(0.0, 0.0, 0.0), (2.0, -1.0, 0.5)])
def test_affine_closed_form_rigid_modes(origin):
    """One 12-DoF aggregate over the whole body with pure linear-elastic K:
    H_c is the Hessian of V psi(F) in the 12 affine parameters, with eigenvalues
    exactly {0 x6 (3 translations + 3 rotations), 2 mu V x5, E V/(1-2nu) x1},
    independent of the mesh and of the origin of X_bar (main Eq 4, P:851-855;
    Fig 5 mechanism)."""
    E, nu = 1e5, 0.3
    m = synth.kuhn_grid(4, origin=origin)  # 64 nodes > 32 -> 12-DoF
    tags = np.ones(m.adj_nbr.shape[0], np.uint8)
    r = oracle.build_map(m.adj_ptr, m.adj_nbr, tags, 32)
    assert r["n_coarse"] == 1
    rp, cl, H = fine(m, E=E, nu=nu, mass=False, dt=1.0)
    o = oracle.assemble(r["map"], 1, 32, m.X, rp, cl, H)
    assert o["n3"] == 0 and o["n12"] == 1 and o["n_slots"] == 4 and o["nnzb"] == 16
    A = bsr_dense(o["row_ptr"], o["col"], o["val"], 4)
    assert np.allclose(A, A.T, rtol=0, atol=1e-12 * np.abs(A).max())
    ev = np.sort(np.linalg.eigvalsh(0.5 * (A + A.T)))
    mu, lam = synth.lame(E, nu)
    V = 1.0
    expect = np.array([0.0] * 6 + [2 * mu * V] * 5 + [E * V / (1 - 2 * nu)])
    scale = np.abs(A).max()
    assert np.allclose(ev, expect, rtol=1e-9, atol=1e-11 * scale)


def test_transform_index_formula_spec_s346():
    """Eq S2/S3 with SPEC S:346: n3 = 5, 12-DoF coarse node m = 7,
    K = 6 in a 12x12 block -> row r = 5 + (7-5)*4 + floor(6/4) = 14 and column
    5 + (m'-5)*4 + 6 mod 4.  One nonzero fine block (i, j) lands exactly there."""
    sizes = [1, 1, 1, 1, 1, 3, 3, 3, 3]   # thr 2 -> ids 0..4 3-DoF, 5..8 12-DoF
    mp = np.repeat(np.arange(9), sizes).astype(np.int32)
    N = mp.shape[0]
    rng = np.random.default_rng(0)
    X = rng.standard_normal((N, 3))
    i = int(np.nonzero(mp == 7)[0][0]); j = int(np.nonzero(mp == 8)[0][1])
    rp = np.zeros(N + 1, np.int64); rp[i + 1:] = 1
    cl = np.array([j], np.int32)
    B = rng.standard_normal((1, 3, 3))
    o = oracle.assemble(mp, 9, 2, X, rp, cl, B)
    assert o["n3"] == 5 and o["n12"] == 4
    K = 6
    p, q = K // 4, K % 4
    r = 5 + (7 - 5) * 4 + p
    c = 5 + (8 - 5) * 4 + q
    assert r == 14
    k = o["row_ptr"][r] + np.nonzero(o["col"][o["row_ptr"][r]:o["row_ptr"][r + 1]] == c)[0][0]
    wi = [X[i, 0], X[i, 1], X[i, 2], 1.0][p]; wj = [X[j, 0], X[j, 1], X[j, 2], 1.0][q]
    assert np.allclose(o["val"][k], wi * wj * B[0], rtol=1e-15)
    assert o["nnzb"] == 16  # a 12x12 block flattens to 16 3x3 sub-blocks (Alg S4 l.7)


def test_classify_fixture_spec_s262():
    g = read_golden("classify_spec_s262.txt")
    sizes = [int(x) for x in g["sizes"]]
    mp = np.repeat(np.arange(len(sizes)), sizes).astype(np.int32)
    N = mp.shape[0]
    rp = np.arange(N + 1, dtype=np.int64); cl = np.arange(N, dtype=np.int32)
    H = np.tile(np.eye(3), (N, 1, 1))
    o = oracle.assemble(mp, len(sizes), int(g["threshold"][0]), np.zeros((N, 3)), rp, cl, H)
    assert o["n3"] == int(g["n3"][0]) and o["n12"] == int(g["n12"][0])
    assert 3 * o["n_slots"] == int(g["coarse_dof"][0])
    newid = [int(x) for x in g["new_ids"]]
    assert np.array_equal(o["new_map"], np.asarray(newid)[mp])


def test_restrict_fixture_spec_s337():
    g = read_golden("restrict_spec_s337.txt")
    X = np.array([[float(x) for x in g["X"]]] * 40)   # 40 > 32 -> 12-DoF
    gf = np.zeros((40, 3)); gf[0] = [float(x) for x in g["g"]]
    H = np.tile(np.eye(3), (40, 1, 1))
    o = oracle.assemble(np.zeros(40, np.int32), 1, 32, X, np.arange(41, dtype=np.int64),
                        np.arange(40, dtype=np.int32), H, gf)
    assert np.array_equal(o["g_c"].reshape(-1), np.array([float(x) for x in g["g_c"]]))


def test_table_s1_coarse_dof_arithmetic():
    """Table S1: coarse DoF = 3 n3 + 12 n12 = 3 * (expanded slots n3 + 4 n12);
    active ratio = coarse DoF / fine DoF, printed to 2 decimals."""
    for fine_dof, n3, n12, cdof, ratio in read_golden_rows("table_s1_dof.txt"):
        n3, n12, cdof = int(n3), int(n12), int(cdof)
        assert 3 * (n3 + 4 * n12) == cdof
        assert round(cdof / int(fine_dof), 2) == float(ratio)


def test_conservation_and_symmetry_c1():
    """All-3-DoF: sum of g_c = sum of g_f; symmetric H_f -> H_c
    symmetric to the bound; positive definite on a small SPD case."""
    c = synth.config_c1()
    m = c["mesh"]
    r = oracle.build_map(m.adj_ptr, m.adj_nbr, c["slot_tags"], 32)
    rp, cl, H = fine(m)
    g = synth.fine_gradient(m.n_nodes)
    o = oracle.assemble(r["map"], r["n_coarse"], 10 ** 9, m.X, rp, cl, H, g)
    assert np.allclose(o["g_c"].sum(0), g.sum(0), rtol=1e-12, atol=1e-12)
    o = oracle.assemble(r["map"], r["n_coarse"], 32, m.X, rp, cl, H, g)
    A = bsr_dense(o["row_ptr"], o["col"], o["val"], o["n_slots"])
    Bd = bsr_dense(o["row_ptr"], o["col"], o["bound"], o["n_slots"])
    assert np.all(np.abs(A - A.T) <= 1e-12 * (Bd + Bd.T))
    assert np.linalg.eigvalsh(0.5 * (A + A.T)).min() > 0
