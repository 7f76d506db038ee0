"""The C input generator (synth/_gen.c) against the numpy definitions it replaces at full size.

Input generation only (synth/ holds none of the method's arithmetic): the Kuhn mesh arrays must be
identical, the fine Hessian equal within rounding (the two sum the tet blocks in different orders)
and bitwise symmetric (R22, the precondition the assembly relies on)."""
import numpy as np
import pytest

import synth

FIELDS = ("X", "tets", "adj_ptr", "adj_nbr", "tet_slots", "edges", "edge_of_slot", "bsr_ptr", "bsr_col", "diag_slot",
          "ijk")


def _same_mesh(a, b):
    for f in FIELDS:
        x, y = getattr(a, f), getattr(b, f)
        assert x.shape == y.shape, f
        assert np.array_equal(x, y), f
    assert a.n_extra == b.n_extra and a.n_side == b.n_side


@pytest.mark.parametrize("n", [2, 3, 5, 8, 13])
def test_kuhn_grid_matches_numpy(n):
    _same_mesh(synth.kuhn_grid(n), synth.kuhn_grid_py(n))


def test_kuhn_grid_origin_and_side():
    _same_mesh(synth.kuhn_grid(6, side=2.5, origin=(1.0, -2.0, 0.25)), synth.kuhn_grid_py(6, side=2.5, origin=(1.0, -2.0, 0.25)))


def _transpose_of(H, m):
    """H[slot(j,i)]^T for every slot (i,j) of the pattern."""
    N = m.n_nodes
    rows = np.repeat(np.arange(N), np.diff(m.bsr_ptr))
    tslot = synth.bsr_slot_py(m, m.bsr_col, rows)
    assert (tslot >= 0).all()
    return H[tslot].transpose(0, 2, 1)


@pytest.mark.parametrize("n,E", [(4, 1e5), (7, 3e6)])
def test_fine_hessian_matches_numpy_and_is_bitwise_symmetric(n, E):
    m = synth.kuhn_grid(n)
    H = synth.fine_hessian(m, E=E)
    Hp = synth.fine_hessian_py(m, E=E)
    scale = np.abs(Hp).max()
    assert np.abs(H - Hp).max() <= 1e-13 * scale
    assert np.array_equal(H, _transpose_of(H, m))


def test_fine_hessian_per_tet_E_mass_and_stiffness_parts():
    m = synth.kuhn_grid(5)
    Et = np.where(np.arange(m.n_tets) % 3 == 0, 1e5, 1e7)
    for kw in (dict(), dict(mass=False), dict(stiffness=False)):
        H = synth.fine_hessian(m, E=Et, **kw)
        Hp = synth.fine_hessian_py(m, E=Et, **kw)
        assert np.abs(H - Hp).max() <= 1e-13 * np.abs(Hp).max()


def test_c4_scene_fast_equals_generic():
    a = synth.c4_scene(n=4, k=2, fast=True)
    b = synth.c4_scene(n=4, k=2, fast=False)
    _same_mesh(a["mesh"], b["mesh"])
    Ha, Hb = synth.c4_hessian(a), synth.c4_hessian(b)
    assert np.abs(Ha - Hb).max() <= 1e-13 * np.abs(Hb).max()
    assert np.array_equal(Ha, _transpose_of(Ha, a["mesh"]))


def test_bsr_slot_matches_numpy():
    m = synth.kuhn_grid(5)
    rng = np.random.default_rng(0)
    u = rng.integers(0, m.n_nodes, 500)
    v = rng.integers(0, m.n_nodes, 500)
    assert np.array_equal(synth.bsr_slot(m, u, v), synth.bsr_slot_py(m, u, v))
