"""Pins for the oracle's fine-to-coarse map (supp Alg S1/S2; recursion
P:217).  Checked against the paper's worked examples (tests/golden), a literal
line-by-line emulation of Alg S1/S2 (tests/alg_emulation.py), brute force over
all tag patterns of tiny meshes, and invariants -- never against itself."""
import itertools

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

import oracle
import synth
from alg_emulation import alg_s1, alg_s2, build_map_emulated
from conftest import read_golden


def graph_csr(n, edges, protected=()):
    """Symmetric adjacency with per-slot tags (1 collapsible, 0 protected)."""
    pairs = {}
    for u, v in edges:
        pairs[(u, v)] = pairs[(v, u)] = 1
    for u, v in protected:
        pairs[(u, v)] = pairs[(v, u)] = 0
    keys = sorted(pairs)
    ptr = np.zeros(n + 1, np.int64)
    for u, _ in keys:
        ptr[u + 1] += 1
    ptr = np.cumsum(ptr)
    nbr = np.array([v for _, v in keys], np.int32)
    tag = np.array([pairs[k] for k in keys], np.uint8)
    return ptr, nbr, tag


def bits_msb_left(s):
    return int(s, 2)


def parse_edges(tokens):
    return [tuple(int(x) for x in t.split("-")) for t in tokens]


# --------------------------------------------------------------------------
# Worked examples of the paper
# --------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["map_p202_group3_triangle.txt", "map_p215_group4_indirect.txt",
                                  "map_p222_protected_group.txt"])
def test_worked_example_level0(name):
    g = read_golden(name)
    gs = int(g["group_size"][0]); n = int(g["n_nodes"][0])
    edges = parse_edges(g["edges"]); prot = parse_edges(g.get("protected", []))
    # the literal Alg S1 reproduces the printed hashes ...
    nbrs = [[] for _ in range(n)]
    tagd = {}
    for u, v in edges + prot:
        nbrs[u].append(v); nbrs[v].append(u)
    for u, v in edges:
        tagd[(u, v)] = tagd[(v, u)] = 1
    for u, v in prot:
        tagd[(u, v)] = tagd[(v, u)] = 0
    h0 = alg_s1(n, gs, nbrs, lambda a, b: tagd[(a, b)])
    assert h0 == [bits_msb_left(s) for s in g["h0"]]
    final, P, counts, mp = alg_s2(h0, gs, corrected=True)
    assert final == [bits_msb_left(s) for s in g["final"]]
    assert counts == [int(c) for c in g["counts"]]
    assert mp == [int(c) for c in g["map"]]
    # ... and the oracle's union-find definition gives the printed map
    ptr, nbr, tag = graph_csr(n, edges, prot)
    r = oracle.build_map(ptr, nbr, tag, gs, max_levels=1)
    assert r["map"].tolist() == [int(c) for c in g["map"]]


def test_printed_local_index_formula_contradicts_examples():
    """Reading R1: Alg S2 l.183-184 as printed (popc(elect & lanes below lane_id))
    gives {0,1,1} for the fully connected group of P:202, whose map the text
    says is all 0; the first-set-bit reading gives {0,0,0}."""
    h0 = [0b111, 0b111, 0b111]
    assert alg_s2(h0, 3, corrected=False)[3] == [0, 1, 1]
    assert alg_s2(h0, 3, corrected=True)[3] == [0, 0, 0]


def test_fig2_recursion():
    g = read_golden("map_fig2_recursive.txt")
    n = int(g["n_nodes"][0]); gs = int(g["group_size"][0])
    ptr, nbr, tag = graph_csr(n, parse_edges(g["edges"]))
    r = oracle.build_map(ptr, nbr, tag, gs)
    assert r["map"].tolist() == [int(x) for x in g["map"]]
    assert r["level_n"].tolist() == [int(x) for x in g["level_n"]]
    em = build_map_emulated(n, gs, parse_edges(g["edges"]))
    assert em[0] == r["map"].tolist() and em[3] == r["level_n"].tolist()


def test_all_collapsible_maps_to_zero_c1():
    """all edges collapsible -> Map(i) = 0.  C1 mesh, gs=32: 1000 -> 32 -> 1."""
    m = synth.kuhn_grid(10)
    tags = np.ones(m.adj_nbr.shape[0], np.uint8)
    r = oracle.build_map(m.adj_ptr, m.adj_nbr, tags, 32)
    assert r["n_coarse"] == 1 and np.all(r["map"] == 0)
    assert r["level_n"].tolist() == [32, 1, 1]
    assert r["agg_size"].tolist() == [1000]


def test_all_protected_is_identity_one_level():
    m = synth.kuhn_grid(6)
    r = oracle.build_map(m.adj_ptr, m.adj_nbr, np.zeros(m.adj_nbr.shape[0], np.uint8), 32)
    assert np.array_equal(r["map"], np.arange(m.n_nodes)) and r["n_levels"] == 1


def test_group_size_one_is_identity():
    m = synth.kuhn_grid(5)
    r = oracle.build_map(m.adj_ptr, m.adj_nbr, np.ones(m.adj_nbr.shape[0], np.uint8), 1)
    assert np.array_equal(r["map"], np.arange(m.n_nodes)) and r["n_levels"] == 1


# --------------------------------------------------------------------------
# Three-way: oracle vs literal Alg S1/S2 emulation on random graphs
# --------------------------------------------------------------------------
@pytest.mark.parametrize("gs", [1, 2, 3, 4, 5, 8, 16, 32])
def test_oracle_equals_literal_emulation_random_graphs(gs):
    rng = np.random.default_rng(gs)
    for trial in range(25):
        n = int(rng.integers(1, 120))
        ne = int(rng.integers(0, 3 * n))
        E = {(int(a), int(b)) for a, b in rng.integers(0, n, (ne, 2)) if a != b}
        E = {(min(a, b), max(a, b)) for a, b in E}
        E = sorted(E)
        p = rng.random()
        coll = [e for e in E if rng.random() < p]
        prot = [e for e in E if e not in set(coll)]
        ptr, nbr, tag = graph_csr(n, coll, prot)
        for ml in (1, 2, 0):
            r = oracle.build_map(ptr, nbr, tag, gs, max_levels=ml)
            em, nc, nl, ln = build_map_emulated(n, gs, coll, max_levels=ml)
            assert r["map"].tolist() == em
            assert r["n_coarse"] == nc and r["n_levels"] == nl
            assert r["level_n"].tolist() == ln


# --------------------------------------------------------------------------
# Brute force over every tag pattern of tiny meshes
# --------------------------------------------------------------------------
def _tiny_meshes():
    X1 = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    one = synth.mesh_from_tets(X1, np.array([[0, 1, 2, 3]]))
    X2 = np.vstack([X1, [[1, 1, 1]]])
    two = synth.mesh_from_tets(X2, np.array([[0, 1, 2, 3], [1, 2, 3, 4]]))
    cube = synth.kuhn_grid(2)  # 8 nodes, 19 edges, 6 tets
    return {"one_tet": one, "two_tets": two, "kuhn_cube": cube}


@pytest.mark.parametrize("name", ["one_tet", "two_tets", "kuhn_cube"])
@pytest.mark.parametrize("gs", [1, 2, 3, 4, 32])
def test_brute_force_tag_patterns(name, gs):
    m = _tiny_meshes()[name]
    E = m.n_edges
    pats = range(1 << E) if E <= 9 else np.random.default_rng(E).integers(0, 1 << E, 600)
    for pat in pats:
        tau = np.array([(int(pat) >> e) & 1 for e in range(E)], np.uint8)
        tags = synth.edge_tags_to_slots(m, tau)
        r = oracle.build_map(m.adj_ptr, m.adj_nbr, tags, gs)
        coll = [(int(m.edges[e, 0]), int(m.edges[e, 1])) for e in range(E) if tau[e]]
        em = build_map_emulated(m.n_nodes, gs, coll)
        assert r["map"].tolist() == em[0], (pat, gs)


# --------------------------------------------------------------------------
# Invariants on the C1 workload shape
# --------------------------------------------------------------------------
def _components(n, edges):
    if len(edges) == 0:
        return n, np.arange(n)
    e = np.asarray(edges)
    A = sp.coo_matrix((np.ones(len(e)), (e[:, 0], e[:, 1])), shape=(n, n))
    return connected_components(A, directed=False)


@pytest.mark.parametrize("p", [0.0, 0.1, 0.2, 0.3, 0.5, 0.8, 1.0])
@pytest.mark.parametrize("gs", [2, 3, 8, 32])
def test_invariants_random_tags(p, gs):
    m = synth.kuhn_grid(10)
    for seed in range(3):
        tags = synth.random_tags(m, p, seed)
        r = oracle.build_map(m.adj_ptr, m.adj_nbr, tags, gs)
        mp, nc = r["map"], r["n_coarse"]
        N = m.n_nodes
        # surjection onto [0, n_c)
        assert set(np.unique(mp).tolist()) == set(range(nc))
        # sizes: sum = N, R^T 1 = sizes
        assert r["agg_size"].sum() == N
        assert np.array_equal(np.bincount(mp, minlength=nc), r["agg_size"])
        # components numbered by ascending minimum member (P:191-195 + R1)
        first = np.full(nc, N)
        np.minimum.at(first, mp, np.arange(N))
        assert np.all(np.diff(first) > 0)
        # every aggregate is connected through collapsible edges; refinement of UF
        tau = np.zeros(m.n_edges, np.uint8)
        tau[m.edge_of_slot] = tags
        coll = m.edges[tau == 1]
        ncc, lab = _components(N, coll)
        inside = coll[mp[coll[:, 0]] == mp[coll[:, 1]]] if len(coll) else coll
        nci, labi = _components(N, inside)
        assert nci == nc  # aggregates == components of the collapsible edges inside them
        for c in range(nc):
            assert len(np.unique(lab[mp == c])) == 1  # refinement of union-find
        # equality with union-find iff no collapsible edge crosses two aggregates
        crossing = len(coll) - len(inside)
        assert (nc == ncc) == (crossing == 0)
        # fully protected vertices are singletons
        deg_coll = np.bincount(coll.ravel(), minlength=N) if len(coll) else np.zeros(N, int)
        iso = np.nonzero(deg_coll == 0)[0]
        assert np.all(r["agg_size"][mp[iso]] == 1)
        # determinism
        r2 = oracle.build_map(m.adj_ptr, m.adj_nbr, tags, gs)
        assert np.array_equal(r2["map"], mp)


def test_level0_local_ids_cover_counts():
    """After one level, each group's coarse ids are O[g] .. O[g]+count_g-1."""
    m = synth.kuhn_grid(10)
    tags = synth.random_tags(m, 0.4, 1)
    r = oracle.build_map(m.adj_ptr, m.adj_nbr, tags, 32, max_levels=1)
    mp = r["map"]
    start = 0
    for g in range(0, m.n_nodes, 32):
        ids = np.unique(mp[g:g + 32])
        assert ids.tolist() == list(range(start, start + len(ids)))
        start += len(ids)


def test_segments_keep_aggregates_inside_segments():
    """Segmented map (multi-GPU reading): no aggregate crosses a segment bound,
    and one segment equals the unsegmented map."""
    m = synth.kuhn_grid(10)
    tags = np.ones(m.adj_nbr.shape[0], np.uint8)
    r1 = oracle.build_map(m.adj_ptr, m.adj_nbr, tags, 32, seg_begin=[0, m.n_nodes])
    r0 = oracle.build_map(m.adj_ptr, m.adj_nbr, tags, 32)
    assert np.array_equal(r1["map"], r0["map"])
    seg = [0, 512, 1000]
    r2 = oracle.build_map(m.adj_ptr, m.adj_nbr, tags, 32, seg_begin=seg)
    assert r2["n_coarse"] == 2
    assert np.all(r2["map"][:512] == 0) and np.all(r2["map"][512:] == 1)


def test_contact_blocks_never_merge_objects():
    """C4: contact couplings are Hessian entries, not mesh edges -- with every edge
    collapsible each object collapses to one aggregate and no aggregate spans two objects."""
    sc = synth.c4_scene(n=4, k=2)
    m = sc["mesh"]
    tags = np.ones(m.adj_nbr.shape[0], np.uint8)
    om = oracle.build_map(m.adj_ptr, m.adj_nbr, tags, 32)
    assert om["n_coarse"] == sc["nobj"]
    obj = np.arange(m.n_nodes) // sc["N0"]
    assert np.array_equal(om["map"], obj)  # numbered by minimum member = object order
    assert m.n_extra == 2 * len(sc["pairs"])
