"""r02f probes: (1) C3 coarsen A/B of the large-row kernels (factorised vs direct), (2) the flat-K1
post-coarsening fine solve, (3) C4 coarse PCG per-kernel times.  CUDA events via the library
profiler; prints JSON lines."""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_2605_04773_b200 as P  # noqa: E402
import synth  # noqa: E402
from paper_2605_04773_b200.step import CoarseningStep  # noqa: E402

dev = torch.device("cuda:0")
t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
what = sys.argv[1]
if what == "c3":
    m = synth.kuhn_grid(100)
    H = synth.fine_hessian(m)
    g = synth.fine_gradient(m.n_nodes)
    xcs = [synth.walls(m, k)[1] for k in range(10)]
    h = P.Handle(0)
    h.set_option(P.OPT_L2_PERSIST, 128 << 20)
    dm = P.DeviceMesh.from_arrays(m.tets, m.adj_ptr, m.adj_nbr, m.tet_slots, m.X, device=dev)
    Hrp, Hcol, Hval = t(m.bsr_ptr, torch.int64), t(m.bsr_col, torch.int32), t(H, torch.float64)
    st = CoarseningStep(h, dm, Hrp, Hcol, Hval, check_every=32, refine_iters=10)
    xp, gd = t(m.X, torch.float64), t(g, torch.float64)
    xcd = [t(x, torch.float64) for x in xcs]
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    for s in range(3):
        st.coarsen(xp, xcd[s], gd)
    torch.cuda.synchronize()
    h.profile(True)
    for s in range(10):
        flush.zero_()
        nf, info, cs = st.coarsen(xp, xcd[s], gd)
    torch.cuda.synchronize()
    pr = h.profile_read()
    h.profile(False)
    print(json.dumps({"probe": "c3_coarsen", "env": {k: v for k, v in os.environ.items() if k.startswith("AGIPC")},
                      "phases_ms": {k: round(v[1] / 10, 4) for k, v in pr.items() if v[0]}}))
    # post-coarsening fine solve (flat K1 for <= 32 iterations)
    x, s0 = st.solve(cs)
    yf = torch.empty((m.n_nodes, 3), dtype=torch.float64, device=dev)
    ts = []
    for r in range(4):
        flush.zero_()
        P.prolongate(h, dm, cs.new_map, cs.n3, cs.n_slots, x, 1.0, yf)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _, sr = P.pcg_solve(h, Hrp, Hcol, Hval, gd, yf, 1e-3, 10, 10)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    h.profile(True)
    P.pcg_solve(h, Hrp, Hcol, Hval, gd, yf, 1e-3, 10, 10)
    pr = h.profile_read()
    h.profile(False)
    print(json.dumps({"probe": "refine", "ms": [round(v, 3) for v in ts], "iters": sr["iters"],
                      "phases_ms": {k: round(v[1], 4) for k, v in pr.items() if v[0]},
                      "kernel_us": {k: round(1e3 * v[1] / v[0], 2) for k, v in pr.items()
                                    if k in ("pcg_spmv", "pcg_update") and v[0]}}))
elif what == "c4":
    sc = synth.c4_scene(n=57, k=3)
    m = sc["mesh"]
    H = synth.c4_hessian(sc)
    g = synth.fine_gradient(m.n_nodes, seed=4)
    xp, xc = synth.c4_iterates(sc)
    h = P.Handle(0)
    h.set_option(P.OPT_L2_PERSIST, int(os.environ.get("L2P", str(128 << 20))))
    dm = P.DeviceMesh.from_arrays(m.tets, m.adj_ptr, m.adj_nbr, m.tet_slots, m.X, device=dev)
    st = CoarseningStep(h, dm, t(m.bsr_ptr, torch.int64), t(m.bsr_col, torch.int32), t(H, torch.float64),
                        check_every=64, max_iters=400)
    nf, info, cs = st.coarsen(t(xp, torch.float64), t(xc, torch.float64), t(g, torch.float64))
    st.solve(cs)
    torch.cuda.synchronize()
    h.profile(True)
    x, s = st.solve(cs)
    pr = h.profile_read()
    h.profile(False)
    print(json.dumps({"probe": "c4_pcg", "iters": s["iters"], "n_slots": cs.n_slots, "nnzb": cs.nnzb,
                      "phases_ms": {k: round(v[1], 4) for k, v in pr.items() if v[0]},
                      "kernel_us": {k: round(1e3 * v[1] / v[0], 2) for k, v in pr.items()
                                    if k in ("pcg_spmv", "pcg_update") and v[0]}}))
