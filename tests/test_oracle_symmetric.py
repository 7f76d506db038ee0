"""Pins for the oracle's symmetric (diagonal + upper) storage (NEXT#2; main Sec 6: "we
store and accumulate only the diagonal and upper-triangular entries"): the upper half plus the
transpose of its strict part rebuilds the full matrix bit for bit, the block count closed form,
the product of the symmetric operator against a dense matrix-vector product, and the quadratic
form identity x^T A x = sum_i x_i.U_ii x_i + 2 sum_{i<j} x_i.U_ij x_j used by the GPU p.q."""
import numpy as np

import oracle
import synth


def dense(rp, col, val, n):
    D = np.zeros((3 * n, 3 * n))
    for i in range(n):
        for e in range(rp[i], rp[i + 1]):
            j = col[e]
            D[3 * i:3 * i + 3, 3 * j:3 * j + 3] = val[e]
    return D


def dense_from_upper(urp, ucol, uval, n):
    D = np.zeros((3 * n, 3 * n))
    for i in range(n):
        for e in range(urp[i], urp[i + 1]):
            j = ucol[e]
            D[3 * i:3 * i + 3, 3 * j:3 * j + 3] = uval[e]
            if j != i:
                D[3 * j:3 * j + 3, 3 * i:3 * i + 3] = uval[e].T
    return D


def coarse_system(n=5, thr=4, seed=0):
    m = synth.kuhn_grid(n)
    rng = np.random.default_rng(seed)
    N = m.n_nodes
    n_c = N // 4
    mp = np.concatenate([np.arange(n_c), rng.integers(0, n_c, N - n_c)]).astype(np.int32)
    rng.shuffle(mp)
    H = synth.fine_hessian(m)
    o = oracle.assemble(mp, n_c, thr, m.X, m.bsr_ptr, m.bsr_col, H)
    return o["row_ptr"], o["col"], o["val"], o["n_slots"]


def cases():
    m = synth.kuhn_grid(4)
    yield m.bsr_ptr, m.bsr_col, synth.fine_hessian(m), m.n_nodes
    yield coarse_system()


def test_upper_plus_strict_transpose_rebuilds_full_bitwise():
    for rp, col, val, n in cases():
        urp, ucol, uval = oracle.bsr_upper(rp, col, val)
        assert np.all(ucol >= np.repeat(np.arange(n), np.diff(urp)))
        assert np.array_equal(dense_from_upper(urp, ucol, uval, n), dense(rp, col, val, n))


def test_block_count_closed_form():
    # symmetric pattern with every diagonal block present: nnzb_upper = (nnzb + n) / 2
    for rp, col, val, n in cases():
        urp, ucol, _ = oracle.bsr_upper(rp, col, val)
        assert urp[-1] == (len(col) + n) // 2 and (len(col) + n) % 2 == 0
    # Kuhn grid closed form: nnzb_f = N + 2E -> upper = N + E
    n = 4
    m = synth.kuhn_grid(n)
    E = 3 * n * n * (n - 1) + 3 * n * (n - 1) ** 2 + (n - 1) ** 3
    urp, _, _ = oracle.bsr_upper(m.bsr_ptr, m.bsr_col, synth.fine_hessian(m))
    assert urp[-1] == n ** 3 + E


def test_diagonal_matrix_is_its_own_upper_half():
    n = 7
    rng = np.random.default_rng(1)
    rp = np.arange(n + 1, dtype=np.int64)
    col = np.arange(n, dtype=np.int32)
    val = rng.standard_normal((n, 3, 3))
    urp, ucol, uval = oracle.bsr_upper(rp, col, val)
    assert np.array_equal(urp, rp) and np.array_equal(ucol, col) and np.array_equal(uval, val)


def test_spmv_upper_matches_dense_product():
    rng = np.random.default_rng(2)
    for rp, col, val, n in cases():
        urp, ucol, uval = oracle.bsr_upper(rp, col, val)
        x = rng.standard_normal((n, 3))
        D = dense(rp, col, val, n)
        y = oracle.spmv_upper(urp, ucol, uval, x).reshape(-1)
        ref = D @ x.reshape(-1)
        bound = np.abs(D) @ np.abs(x.reshape(-1))
        assert np.all(np.abs(y - ref) <= 1e-13 * bound + 1e-300)
        # and equals the full-storage product of the oracle to rounding
        yf = oracle.spmv(rp, col, val, x).reshape(-1)
        assert np.all(np.abs(y - yf) <= 1e-13 * bound + 1e-300)


def test_quadratic_form_from_the_upper_half():
    rng = np.random.default_rng(3)
    for rp, col, val, n in cases():
        urp, ucol, uval = oracle.bsr_upper(rp, col, val)
        x = rng.standard_normal((n, 3))
        q = 0.0
        for i in range(n):
            for e in range(urp[i], urp[i + 1]):
                j = ucol[e]
                t = x[i] @ uval[e] @ x[j]
                q += t if j == i else 2.0 * t
        D = dense(rp, col, val, n)
        ref = x.reshape(-1) @ D @ x.reshape(-1)
        assert abs(q - ref) <= 1e-12 * (np.abs(x.reshape(-1)) @ np.abs(D) @ np.abs(x.reshape(-1)))


def test_expand_upper_inverts_the_selection_bitwise():
    for rp, col, val, n in cases():
        urp, ucol, uval = oracle.bsr_upper(rp, col, val)
        full, miss = oracle.bsr_expand_upper(rp, col, urp, ucol, uval)
        assert miss == 0 and np.array_equal(full, val)
        # the dense picture: upper half and mirrored strict part
        assert np.array_equal(dense(rp, col, full, n), dense_from_upper(urp, ucol, uval, n))


def test_expand_upper_reports_missing_sources():
    m = synth.kuhn_grid(3)
    H = synth.fine_hessian(m)
    urp, ucol, uval = oracle.bsr_upper(m.bsr_ptr, m.bsr_col, H)
    # drop the last upper block of row 0: its block and its mirror have no source
    keep = np.ones(len(ucol), bool)
    keep[urp[1] - 1] = False
    urp2 = urp.copy()
    urp2[1:] -= 1
    full, miss = oracle.bsr_expand_upper(m.bsr_ptr, m.bsr_col, urp2, ucol[keep], uval[keep])
    assert miss == 2
