"""Skew (SURVEY §7 hard part 1; round-1 verdict "skew is never exercised at scale"): every edge
collapsible, so the recursion merges the whole mesh into a handful of aggregates and the
12-DoF assembly sends thousands of 32-child chunks into the same 144 values of one diagonal
block (fp64 atomics in the default mode, fixed-order partials in the deterministic one).  Map
bit-exact, coarse values within the 1e-12 bound, both assembly modes; the step is timed."""
import time

import numpy as np
import pytest
import torch

import oracle
import synth
from test_gpu_parity import P, check_assemble, check_map, dmesh, h  # noqa: F401  (fixtures)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [32, 47])
@pytest.mark.parametrize("deterministic", [0, 1])
def test_all_collapsible_mesh(P, h, n, deterministic):
    m = synth.kuhn_grid(n)
    tags = np.ones(m.adj_nbr.shape[0], np.uint8)
    H = synth.fine_hessian(m, E=1e5)
    g = synth.fine_gradient(m.n_nodes)
    dm = dmesh(P, m)
    mp, info, om = check_map(P, h, m, dm, tags, 32)
    sizes = np.bincount(om["map"])
    assert sizes.max() > 0.5 * m.n_nodes  # one aggregate holds most of the mesh
    h.set_option(P.OPT_DETERMINISTIC, deterministic)
    try:
        check_assemble(P, h, m, dm, om, H, g, 32)
        rp, col = torch.as_tensor(m.bsr_ptr).cuda(), torch.as_tensor(m.bsr_col).cuda()
        Hd, gd = torch.as_tensor(H).cuda(), torch.as_tensor(g).cuda()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            P.assemble_coarse(h, dm, mp, info["n_coarse"], 32, rp, col, Hd, gd)
        torch.cuda.synchronize()
        print(f"all-collapse N={m.n_nodes}: n_coarse={info['n_coarse']} largest={sizes.max()} "
              f"deterministic={deterministic}: assemble {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms")
    finally:
        h.set_option(P.OPT_DETERMINISTIC, 0)
