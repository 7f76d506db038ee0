"""Pins for the oracle's coarse PCG with 3x3 block-Jacobi (
textbook PCG): special cases with known iteration counts, the finite-termination
property of CG, energy-norm monotonicity, a dense direct solve, and the error
paths (indefinite, singular diagonal block)."""
import numpy as np
import pytest

import oracle
import synth


def dense_to_bsr(A):
    n = A.shape[0] // 3
    rp = [0]; cl = []; vl = []
    for r in range(n):
        for c in range(n):
            blk = A[3 * r:3 * r + 3, 3 * c:3 * c + 3]
            if np.any(blk != 0) or r == c:
                cl.append(c); vl.append(blk)
        rp.append(len(cl))
    return np.array(rp, np.int64), np.array(cl, np.int32), np.array(vl)


def test_identity_one_iteration():
    """H = I, x0 = 0 -> x = b after exactly 1 iteration."""
    rp, cl, vl = dense_to_bsr(np.eye(30))
    b = np.random.default_rng(0).standard_normal(30)
    s = oracle.pcg(rp, cl, vl, b, rel_tol=1e-12)
    assert s["iters"] == 1 and s["status"] == oracle.OK
    assert np.allclose(s["x"].reshape(-1), b, rtol=1e-15)


def test_zero_rhs_zero_iterations():
    rp, cl, vl = dense_to_bsr(np.eye(12) * 3)
    s = oracle.pcg(rp, cl, vl, np.zeros(12), rel_tol=1e-3)
    assert s["iters"] == 0 and np.all(s["x"] == 0) and s["status"] == oracle.OK


def test_block_diagonal_is_exact_in_one_iteration():
    """Mass-only H_f under any map is block diagonal: block-Jacobi is exact -> 1 iteration."""
    rng = np.random.default_rng(1)
    Q = rng.standard_normal((10, 3, 3))
    A = np.zeros((30, 30))
    for i in range(10):
        A[3 * i:3 * i + 3, 3 * i:3 * i + 3] = Q[i] @ Q[i].T + 3 * np.eye(3)
    rp, cl, vl = dense_to_bsr(A)
    b = rng.standard_normal(30)
    s = oracle.pcg(rp, cl, vl, b, rel_tol=1e-12)
    assert s["iters"] == 1
    assert np.allclose(A @ s["x"].reshape(-1), b, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("m,c", [(6, 0.1), (12, 0.05)])
def test_two_distinct_eigenvalues_two_iterations(m, c):
    """A = I + c (J - I) (x) I3 has identity diagonal blocks (block-Jacobi = I) and
    exactly two distinct eigenvalues -> CG terminates in <= 2 iterations."""
    A = np.kron(np.eye(m) + c * (np.ones((m, m)) - np.eye(m)), np.eye(3))
    rp, cl, vl = dense_to_bsr(A)
    b = np.random.default_rng(2).standard_normal(3 * m)
    s = oracle.pcg(rp, cl, vl, b, rel_tol=1e-12)
    assert s["iters"] <= 2
    assert np.allclose(np.linalg.solve(A, b), s["x"].reshape(-1), rtol=1e-10)


def test_c1_coarse_system_matches_dense_solve_and_energy_norm_monotone():
    c = synth.config_c1()
    m = c["mesh"]
    r = oracle.build_map(m.adj_ptr, m.adj_nbr, c["slot_tags"], 32)
    H = synth.fine_hessian(m)
    g = synth.fine_gradient(m.n_nodes)
    o = oracle.assemble(r["map"], r["n_coarse"], 32, m.X, m.bsr_ptr, m.bsr_col, H, g)
    b = -o["g_c"].reshape(-1)
    ns = o["n_slots"]
    A = np.zeros((3 * ns, 3 * ns))
    for i in range(ns):
        for k in range(o["row_ptr"][i], o["row_ptr"][i + 1]):
            A[3 * i:3 * i + 3, 3 * o["col"][k]:3 * o["col"][k] + 3] = o["val"][k]
    xs = np.linalg.solve(A, b)
    s = oracle.pcg(o["row_ptr"], o["col"], o["val"], b, rel_tol=1e-12, max_iters=5000)
    assert s["status"] == oracle.OK
    kappa = np.linalg.cond(A)
    assert np.linalg.norm(s["x"].reshape(-1) - xs) <= 10 * kappa * 1e-12 * np.linalg.norm(xs)
    # CG minimises the A-norm of the error over growing Krylov spaces: monotone
    errs = []
    for k in range(1, 30):
        sk = oracle.pcg(o["row_ptr"], o["col"], o["val"], b, rel_tol=0.0, max_iters=k)
        e = sk["x"].reshape(-1) - xs
        errs.append(e @ A @ e)
    assert np.all(np.diff(errs) <= 1e-12 * errs[0])
    # oracle's compensated residual agrees with a dense evaluation
    rr = oracle.rel_residual(o["row_ptr"], o["col"], o["val"], s["x"], b)
    assert abs(rr - np.linalg.norm(A @ s["x"].reshape(-1) - b) / np.linalg.norm(b)) < 1e-14


def test_indefinite_and_singular_are_errors():
    rp, cl, vl = dense_to_bsr(-np.eye(6))
    s = oracle.pcg(rp, cl, vl, np.ones(6))
    # D^-1 = -I makes z = -r; p^T A p = -|p|^2 ... -> pq < 0 breaks the SPD assumption
    assert s["status"] == oracle.EINDEFINITE
    A = np.eye(6); A[3:, 3:] = 0
    rp, cl, vl = dense_to_bsr(A)
    s = oracle.pcg(rp, cl, vl, np.ones(6))
    assert s["status"] == oracle.ESINGULAR
    with pytest.raises(oracle.OracleError):
        oracle.block_jacobi(rp, cl, vl)


def test_block_jacobi_inverse():
    rng = np.random.default_rng(3)
    Q = rng.standard_normal((5, 3, 3))
    A = np.zeros((15, 15))
    for i in range(5):
        A[3 * i:3 * i + 3, 3 * i:3 * i + 3] = Q[i] @ Q[i].T + np.eye(3)
    A[0:3, 3:6] = A[3:6, 0:3] = 0.1
    rp, cl, vl = dense_to_bsr(A)
    D = oracle.block_jacobi(rp, cl, vl)
    for i in range(5):
        assert np.allclose(D[i] @ A[3 * i:3 * i + 3, 3 * i:3 * i + 3], np.eye(3), atol=1e-12)
