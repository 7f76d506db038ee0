"""One Newton step of the path on a small mesh, for compute-sanitizer runs (tests/test_sanitizer_gpu.py):
tag -> map -> assemble (atomic and deterministic large rows) -> PCG (SELL and flat K1) -> prolongation,
plus the NEXT rows.  Exits 0 when every call returned OK."""
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import paper_2605_04773_b200 as P  # noqa: E402
import synth  # noqa: E402
from paper_2605_04773_b200.step import CoarseningStep  # noqa: E402


def main(n):
    dev = torch.device("cuda:0")
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
    m = synth.kuhn_grid(n)
    H = synth.fine_hessian(m)
    g = synth.fine_gradient(m.n_nodes)
    xp, xc = synth.twist(m.X, 0.5), synth.twist(m.X, 0.503)
    dm = P.DeviceMesh.from_arrays(m.tets, m.adj_ptr, m.adj_nbr, m.tet_slots, m.X, device=dev)
    for det in (0, 1):
        h = P.Handle(0)
        h.set_option(P.OPT_DETERMINISTIC, det)
        st = CoarseningStep(h, dm, t(m.bsr_ptr, torch.int64), t(m.bsr_col, torch.int32), t(H, torch.float64),
                            theta=1e-5, rel_tol=1e-6, refine_iters=5, affine_threshold=5)
        r = st(t(xp, torch.float64), t(xc, torch.float64), t(g, torch.float64), count=True)
        assert r.pcg["status"] == P.OK, r.pcg
        # random tags too (more 12-DoF nodes)
        tags = t(synth.random_tags(m, 0.5, 1), torch.uint8)
        mp, info = P.build_map(h, dm, tags, 32)
        cs = P.assemble_coarse(h, dm, mp, info["n_coarse"], 5, t(m.bsr_ptr, torch.int64), t(m.bsr_col, torch.int32),
                               t(H, torch.float64), t(g, torch.float64))
        P.pcg_solve(h, cs.row_ptr, cs.col, cs.val, cs.g_c, rel_tol=1e-8, zero_x0=True)
    torch.cuda.synchronize()
    print("sanitizer step ok", n)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 10)
