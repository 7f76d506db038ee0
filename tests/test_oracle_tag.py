"""Pins for the oracle's edge tags (main Sec 4.2, Eq 3):
closed forms of the Green strain, invariance under rigid motion, strictness of
"exceeds a threshold", and the per-edge OR over incident tets by brute force."""
import numpy as np
import pytest

import oracle
import synth


def run(m, xp, xc, theta):
    return oracle.tag_edges(m.tets, m.tet_slots, m.X, xp, xc, theta, m.adj_nbr.shape[0])


def rotation(axis, ang):
    a = np.asarray(axis, float); a /= np.linalg.norm(a)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + np.sin(ang) * K + (1 - np.cos(ang)) * K @ K


@pytest.fixture(scope="module")
def mesh():
    return synth.kuhn_grid(6)


def test_rigid_motion_gives_zero_strain_and_all_collapsible(mesh):
    """F = R => G = 0: a rigid rotation + translation between
    iterates protects nothing."""
    R1 = rotation([1, 2, 3], 0.7); R2 = rotation([-2, 1, 0.5], 1.9)
    xp = mesh.X @ R1.T + [0.3, -1, 2]
    xc = mesh.X @ R2.T + [5, 1, -7]
    tags, norm, flag = run(mesh, xp, xc, 5e-5)
    assert norm.max() < 1e-13
    assert tags.all() and not flag.any()


@pytest.mark.parametrize("sp_,sc", [(1.0, 2.0), (0.9, 1.1), (1.0, 1.0001)])
def test_uniform_scaling_closed_form(mesh, sp_, sc):
    """x = s (X - c) + c => F = s I, G = (s^2 - 1)/2 I,
    ||dG||_F = (sqrt(3)/2) |s_c^2 - s_p^2|  (exact; checked to 1e-12 rel)."""
    c = np.array([0.3, -0.2, 0.1])
    xp = sp_ * (mesh.X - c) + c
    xc = sc * (mesh.X - c) + c
    _, norm, _ = run(mesh, xp, xc, 1.0)
    expect = np.sqrt(3) / 2 * abs(sc ** 2 - sp_ ** 2)
    # forming F^T F - I cancels: relative error ~ eps * s^2 / |s_c^2 - s_p^2|
    rtol = 64 * np.finfo(float).eps * max(sc, sp_) ** 2 / abs(sc ** 2 - sp_ ** 2)
    assert np.allclose(norm, expect, rtol=rtol, atol=0)


def test_f_equals_2i_closed_form(mesh):
    """F = 2I => G = 1.5 I, ||G||_F = 1.5 sqrt(3)."""
    _, norm, _ = run(mesh, mesh.X, 2.0 * mesh.X, 1.0)
    assert np.allclose(norm, 1.5 * np.sqrt(3), rtol=1e-13, atol=0)


@pytest.mark.parametrize("gamma", [1e-3, 0.1, 0.7])
def test_simple_shear_closed_form(mesh, gamma):
    """F = I + gamma e_x e_y^T => ||G||_F = 1/2 sqrt(2 gamma^2 + gamma^4)."""
    xc = mesh.X.copy(); xc[:, 0] += gamma * mesh.X[:, 1]
    _, norm, _ = run(mesh, mesh.X, xc, 1.0)
    assert np.allclose(norm, 0.5 * np.sqrt(2 * gamma ** 2 + gamma ** 4), rtol=1e-11, atol=1e-15)


def test_threshold_is_strict(mesh):
    """'exceeds a threshold' is strict [R11]: choose the scaling so that
    ||dG|| lands at theta (1 +/- 1e-6): every tet flagged above, none below."""
    theta = 5e-5
    for rel, want in ((1 + 1e-6, 1), (1 - 1e-6, 0)):
        target = theta * rel
        sc = np.sqrt(1.0 + 2.0 * target / np.sqrt(3))
        tags, norm, flag = run(mesh, mesh.X, sc * mesh.X, theta)
        assert np.all(flag == want)
        assert np.all(tags == (1 - want))


def test_theta_zero_protects_every_edge_with_nonzero_increment(mesh):
    rng = np.random.default_rng(1)
    xc = mesh.X + 1e-3 * rng.standard_normal(mesh.X.shape)
    tags, norm, flag = run(mesh, mesh.X, xc, 0.0)
    assert norm.min() > 0 and flag.all() and not tags.any()


def test_single_node_perturbation_protects_exactly_its_tets_edges(mesh):
    """tau_e = 0 iff e belongs to a flagged tet (P:838 'any element adjacent to
    an edge'); brute force over the mesh topology."""
    v = 100
    xc = mesh.X.copy(); xc[v] += [1e-3, 2e-3, -1e-3]
    tags, norm, flag = run(mesh, mesh.X, xc, 5e-5)
    touch = np.any(mesh.tets == v, axis=1)
    assert np.array_equal(flag.astype(bool), touch)
    prot = set()
    for t in np.nonzero(touch)[0]:
        q = mesh.tets[t]
        for a in range(4):
            for b in range(a + 1, 4):
                prot.add((min(q[a], q[b]), max(q[a], q[b])))
    for s in range(mesh.adj_nbr.shape[0]):
        e = tuple(mesh.edges[mesh.edge_of_slot[s]])
        assert tags[s] == (0 if e in prot else 1)
    # both directed slots of an edge agree
    for e in range(mesh.n_edges):
        assert len(set(tags[mesh.edge_of_slot == e].tolist())) == 1


def test_matches_lu_based_evaluation_random(mesh):
    """Independent route: numpy solve (LU) for F = Ds Dm^-1 instead of the
    adjugate; norms agree to 1e-10 relative on random iterates."""
    rng = np.random.default_rng(5)
    xp = mesh.X + 0.05 * rng.standard_normal(mesh.X.shape)
    xc = xp + 0.01 * rng.standard_normal(mesh.X.shape)
    _, norm, _ = run(mesh, xp, xc, 1.0)
    t = mesh.tets

    def G(x):
        D = np.stack([x[t[:, k]] - x[t[:, 0]] for k in (1, 2, 3)], axis=2)
        Dm = np.stack([mesh.X[t[:, k]] - mesh.X[t[:, 0]] for k in (1, 2, 3)], axis=2)
        F = np.linalg.solve(Dm.transpose(0, 2, 1), D.transpose(0, 2, 1)).transpose(0, 2, 1)
        return 0.5 * (F.transpose(0, 2, 1) @ F - np.eye(3))
    ref = np.linalg.norm(G(xc) - G(xp), axis=(1, 2))
    assert np.allclose(norm, ref, rtol=1e-9, atol=1e-15)


def test_degenerate_tet_is_an_error():
    X = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0], [0, 0, 1]], float)
    m = synth.mesh_from_tets(X, np.array([[0, 1, 2, 3]]))
    with pytest.raises(oracle.OracleError) as e:
        run(m, X, X, 1.0)
    assert e.value.status == oracle.EDEGENERATE


def test_c2_twist_shape():
    """C2 workload sanity: ~21.5% tets flagged, ~22.3% edges protected."""
    c = synth.config_c2(20)
    m = c["mesh"]
    tags, norm, flag = run(m, c["x_prev"], c["x_cur"], c["theta"])
    assert 0.05 < flag.mean() < 0.6
