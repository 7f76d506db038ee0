"""Pins for the oracle's fine-level hash reduction (NEXT#3; supp Sec 2; SPEC
S:316-328): worked examples, a dense accumulation oracle, and the assembled stiffness of a tet
mesh against the independently scattered fine Hessian of the input generator."""
import numpy as np

import oracle
import synth


def test_spec_examples():
    A = np.arange(9.0).reshape(3, 3)
    B = np.ones((3, 3))
    rp, col, val = oracle.reduce_triplets(2, [0, 0], [1, 1], np.stack([A, B]))
    assert rp.tolist() == [0, 1, 1] and col.tolist() == [1] and np.array_equal(val[0], A + B)
    ti, tj = [1, 0, 1], [0, 2, 1]                                                # unique -> sorted
    v = np.stack([A, 2 * A, 3 * A])
    rp, col, val = oracle.reduce_triplets(2, ti, tj, v)
    assert rp.tolist() == [0, 1, 3] and col.tolist() == [2, 0, 1]
    assert np.array_equal(val, np.stack([2 * A, A, 3 * A]))


def test_key_order_and_in_order_sums():
    """(2,0) sorts after (1, 2^31 - 1); equal keys are summed in input order (the
    non-associative case 1e16 + 1 - 1e16 distinguishes orders)."""
    big = np.zeros((3, 3, 3))
    big[0, 0, 0], big[1, 0, 0], big[2, 0, 0] = 1e16, 1.0, -1e16
    rp, col, val = oracle.reduce_triplets(3, [2, 1, 1, 1, 1], [0, 2 ** 31 - 1, 5, 5, 5],
                                          np.concatenate([np.zeros((2, 3, 3)), big]))
    assert rp.tolist() == [0, 0, 2, 3] and col.tolist() == [5, 2 ** 31 - 1, 0]
    assert val[0, 0, 0] == (1e16 + 1.0) - 1e16   # = 0.0 in order, 1.0 in another order


def test_dense_accumulation_oracle():
    rng = np.random.default_rng(0)
    n = 1000
    ti, tj = rng.integers(0, 10, n), rng.integers(0, 10, n)
    v = rng.standard_normal((n, 3, 3))
    rp, col, val = oracle.reduce_triplets(10, ti, tj, v)
    D = np.zeros((30, 30))
    for a, b, B in zip(ti, tj, v):
        D[3 * a:3 * a + 3, 3 * b:3 * b + 3] += B
    R = np.zeros((30, 30))
    for r in range(10):
        for k in range(rp[r], rp[r + 1]):
            R[3 * r:3 * r + 3, 3 * col[k]:3 * col[k] + 3] = val[k]
    assert np.allclose(R, D, rtol=0, atol=1e-13)
    assert all(np.all(np.diff(col[rp[r]:rp[r + 1]]) > 0) for r in range(10))


def test_tet_mesh_stiffness_equals_generator_scatter():
    m = synth.kuhn_grid(5)
    ti, tj, v = synth.tet_triplets(m)
    rp, col, val = oracle.reduce_triplets(m.n_nodes, ti, tj, v)
    assert np.array_equal(rp, m.bsr_ptr) and np.array_equal(col, m.bsr_col)   # pattern = adjacency + diag
    H = synth.fine_hessian(m, mass=False)
    assert np.allclose(val, H, rtol=1e-12, atol=1e-12 * np.abs(H).max())
