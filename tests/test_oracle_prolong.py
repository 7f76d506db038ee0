"""Pins for the oracle's prolongation d_f = U^T d_c (NEXT#1; main Sec 4.3; SPEC
S:421-429): explicit U^T, adjointness with the restriction of assemble(), the
translation / identity special cases, and the descent-direction property of the coarse step."""
import numpy as np

import oracle
import synth
from test_oracle_assemble import explicit_U


def test_prolongation_is_explicit_transpose_and_adjoint():
    rng = np.random.default_rng(0)
    m = synth.kuhn_grid(3)
    N = m.n_nodes
    for thr in (2, 4, 100):
        n_c = 9
        mp = np.concatenate([np.arange(n_c), rng.integers(0, n_c, N - n_c)]).astype(np.int32)
        rng.shuffle(mp)
        H = synth.fine_hessian(m)
        v = rng.standard_normal((N, 3))
        o = oracle.assemble(mp, n_c, thr, m.X, m.bsr_ptr, m.bsr_col, H, v)   # g_c = U v
        u = rng.standard_normal((o["n_slots"], 3))
        d = oracle.prolongate(o["new_map"], o["n3"], m.X, u)
        U = explicit_U(o["new_map"], o["n3"], m.X)
        assert np.allclose(d.reshape(-1), U.T @ u.reshape(-1), rtol=1e-14, atol=1e-14)
        # <U^T u, v> = <u, U v>
        assert abs(np.sum(d * v) - np.sum(u * o["g_c"])) <= 1e-12 * np.sum(np.abs(d * v)) + 1e-14


def test_identity_and_translation():
    m = synth.kuhn_grid(4)
    N = m.n_nodes
    u = np.random.default_rng(1).standard_normal((N, 3))
    assert np.array_equal(oracle.prolongate(np.arange(N), N, m.X, u), u)   # identity map
    # one 12-DoF node encoding a pure translation t: every child moves by t
    t = np.array([0.3, -1.0, 2.0])
    x_c = np.zeros((4, 3)); x_c[3] = t
    d = oracle.prolongate(np.zeros(N, np.int32), 0, m.X, x_c)
    assert np.allclose(d, t, rtol=0, atol=1e-15)
    # an affine field F X + t is reproduced exactly (rows p of the 12-DoF node = columns of F)
    F = np.array([[1.0, 0.2, 0.0], [0.1, 0.9, -0.3], [0.0, 0.4, 1.1]])
    x_c = np.vstack([F[:, 0], F[:, 1], F[:, 2], t])
    d = oracle.prolongate(np.zeros(N, np.int32), 0, m.X, x_c)
    assert np.allclose(d, m.X @ F.T + t, rtol=0, atol=1e-14)


def test_coarse_direction_is_a_descent_direction():
    """d_c solves H_c d_c = -g_c; d_f = U^T d_c satisfies d_f . g_f = -d_c^T H_c d_c < 0."""
    c = synth.config_c1()
    m = c["mesh"]
    r = oracle.build_map(m.adj_ptr, m.adj_nbr, c["slot_tags"], 32)
    H = synth.fine_hessian(m)
    g = synth.fine_gradient(m.n_nodes)
    o = oracle.assemble(r["map"], r["n_coarse"], 32, m.X, m.bsr_ptr, m.bsr_col, H, g)
    s = oracle.pcg(o["row_ptr"], o["col"], o["val"], -o["g_c"], rel_tol=1e-12, max_iters=5000)
    d = oracle.prolongate(o["new_map"], o["n3"], m.X, s["x"])
    assert np.sum(d * g) < 0
    assert np.isclose(np.sum(d * g), -np.sum(s["x"] * oracle.spmv(o["row_ptr"], o["col"], o["val"], s["x"])),
                      rtol=1e-9)
