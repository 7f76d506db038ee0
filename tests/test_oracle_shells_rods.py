"""Pins for the oracle's step 1 on shells (triangles) and rods (edges) -- NEXT#4 (P:838
"applicable to various element types (shells, volumes, rods)")."""
import numpy as np
import pytest

import oracle
import synth


def _rot(seed):
    q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((3, 3)))
    return q * np.sign(np.linalg.det(q))


@pytest.fixture(scope="module")
def sh():
    return synth.sheet(9)


def test_shell_rigid_motion_and_rest(sh):
    X = sh["X"]
    ns = sh["adj_nbr"].shape[0]
    R = _rot(3)
    _, n0 = oracle.tag_shells(sh["tris"], sh["tri_slots"], X, X, X, 0.0, ns)
    _, n1 = oracle.tag_shells(sh["tris"], sh["tri_slots"], X, X, X @ R.T + [1.0, -2.0, 0.5], 0.0, ns)
    assert np.all(n0 == 0.0) and np.all(n1 < 1e-14)


@pytest.mark.parametrize("sp,sc", [(1.0, 1.1), (0.9, 1.3), (1.2, 1.2)])
def test_shell_uniform_scaling_closed_form(sh, sp, sc):
    """F has singular values (s, s) -> G = 1/2 (s^2 - 1) I_2 -> ||dG||_F = (sqrt 2 / 2)|sc^2 - sp^2|."""
    X = sh["X"]
    _, n = oracle.tag_shells(sh["tris"], sh["tri_slots"], X, sp * X, sc * X, 0.0, sh["adj_nbr"].shape[0])
    ref = np.sqrt(2.0) / 2.0 * abs(sc * sc - sp * sp)
    assert np.allclose(n, ref, rtol=1e-12, atol=1e-15)


def test_shell_uniaxial_stretch_and_tangent_basis_invariance(sh):
    """Stretch by lam along an in-plane direction d: G = 1/2 (lam^2 - 1) d d^T (in-plane), norm
    |1/2 (lam^2 - 1)| whatever the triangle's tangent basis (vertex order rotated -> same norm)."""
    X = sh["X"]
    R = sh["rot"]
    d = R[:, 0] * np.cos(0.3) + R[:, 1] * np.sin(0.3)   # in-plane unit direction
    lam = 1.25
    xc = X + (lam - 1.0) * np.outer(X @ d, d)
    ns = sh["adj_nbr"].shape[0]
    _, n = oracle.tag_shells(sh["tris"], sh["tri_slots"], X, X, xc, 0.0, ns)
    assert np.allclose(n, 0.5 * (lam * lam - 1.0), rtol=1e-12)
    tris2 = sh["tris"][:, [1, 2, 0]]
    slots2 = synth.element_slots(sh["adj_ptr"], sh["adj_nbr"], tris2, synth.TRI_EDGES)
    _, n2 = oracle.tag_shells(tris2, slots2, X, X, xc, 0.0, ns)
    assert np.allclose(n2, n, rtol=1e-12)


def test_shell_out_of_plane_fold_of_one_triangle_is_rigid():
    X = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]])
    tris = np.array([[0, 1, 2], [1, 3, 2]], np.int32)
    ap, an = synth.adjacency_from_edges(4, np.concatenate([tris[:, [0, 1]], tris[:, [0, 2]], tris[:, [1, 2]]]))
    ts = synth.element_slots(ap, an, tris, synth.TRI_EDGES)
    xc = X.copy()
    # fold the second triangle about the shared edge (1,2) by 90 degrees: vertex 3 rotates
    m = 0.5 * (X[1] + X[2])
    a = (X[2] - X[1]) / np.linalg.norm(X[2] - X[1])
    r = X[3] - m
    xc[3] = m + np.cos(np.pi / 2) * r + np.sin(np.pi / 2) * np.cross(a, r) + a * (a @ r) * (1 - np.cos(np.pi / 2))
    tags, n = oracle.tag_shells(tris, ts, X, X, xc, 1e-12, an.shape[0])
    assert np.all(n < 1e-14) and np.all(tags == 1)   # bending is not strain: nothing protected


def test_rod_closed_forms():
    """F = l/L, G = 1/2 (F^2 - 1): stretch 1 -> 1.5 gives 0.625 (SPEC S:166 prints 0.375, which is
    not 1/2 (1.5^2 - 1): reading R26); rigid motion 0; compression 0.5 -> 0.375."""
    X = np.array([[0.0, 0, 0], [1, 0, 0], [1, 1, 0]])
    segs = np.array([[0, 1], [1, 2]], np.int32)
    ap, an = synth.adjacency_from_edges(3, segs)
    ss = synth.element_slots(ap, an, segs, ((0, 1),))
    _, n = oracle.tag_rods(segs, ss, X, X, 1.5 * X, 0.0, an.shape[0])
    assert np.allclose(n, 0.625, rtol=0, atol=1e-15)
    R = _rot(5)
    _, n = oracle.tag_rods(segs, ss, X, X, X @ R.T + 3.0, 0.0, an.shape[0])
    assert np.all(n < 1e-15)
    _, n = oracle.tag_rods(segs, ss, X, X, 0.5 * X, 0.0, an.shape[0])
    assert np.allclose(n, 0.375, atol=1e-15)


def test_mixed_accumulation_and_protection_rule():
    """Tets + boundary shells + rods: an edge is protected iff ANY adjacent element is flagged
    (brute force over elements), and the shell/rod calls never un-protect."""
    m = synth.kuhn_grid(4)
    rng = np.random.default_rng(2)
    xp = m.X.copy()
    xc = m.X + 2e-3 * rng.standard_normal(m.X.shape) * (rng.random(m.n_nodes) < 0.2)[:, None]
    ns = m.adj_nbr.shape[0]
    tris = synth.boundary_triangles(m)
    ts = synth.element_slots(m.adj_ptr, m.adj_nbr, tris, synth.TRI_EDGES)
    segs = m.edges[::7].astype(np.int32)
    ss = synth.element_slots(m.adj_ptr, m.adj_nbr, segs, ((0, 1),))
    th = 1e-4
    t0, _, fl = oracle.tag_edges(m.tets, m.tet_slots, m.X, xp, xc, th, ns)
    t1, nt = oracle.tag_shells(tris, ts, m.X, xp, xc, th, ns, slot_tags=t0)
    t2, nr = oracle.tag_rods(segs, ss, m.X, xp, xc, th, ns, slot_tags=t1)
    prot = np.zeros(ns, bool)
    for el, sl, f in ((m.tets, m.tet_slots, fl.astype(bool)), (tris, ts, nt > th), (segs, ss, nr > th)):
        prot[sl[f].ravel()] = True
    assert np.array_equal(t2 == 0, prot)
    assert np.all(t2 <= t0)
