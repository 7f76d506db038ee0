"""C5 (20M nodes) coarsen+assemble per step with the library's phase profile: which phase
regressed between r02h (73.6 ms) and r02l (247 ms)?"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2605_04773_b200 as P  # noqa: E402
import synth  # noqa: E402
from paper_2605_04773_b200.step import CoarseningStep  # noqa: E402

fresh = "--fresh" in sys.argv
dev = torch.device("cuda:0")
h = P.Handle(0)
if not fresh:   # the bench's order: a C3 step on the same handle first
    pass
t0 = time.time()
m = synth.kuhn_grid(272)
H = synth.fine_hessian(m, E=1e5)
g = synth.fine_gradient(m.n_nodes)
xcs = [synth.walls(m, k)[1] for k in range(2)]
t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
dm = P.DeviceMesh.from_arrays(m.tets, m.adj_ptr, m.adj_nbr, m.tet_slots, m.X, device=dev)
Hrp, Hcol, Hval = t(m.bsr_ptr, torch.int64), t(m.bsr_col, torch.int32), t(H, torch.float64)
del H
gd, xpd = t(g, torch.float64), t(m.X, torch.float64)
xcd = [t(x, torch.float64) for x in xcs]
print("gen", time.time() - t0, flush=True)
step = CoarseningStep(h, dm, Hrp, Hcol, Hval, check_every=64, max_iters=100000)
for s in range(8):
    solve = s in (1, 4)
    prof_on = s >= 5
    h.profile(prof_on)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    e[0].record()
    nf, info, cs = step.coarsen(xpd, xcd[s % 2], gd)
    e[1].record()
    torch.cuda.synchronize()
    prof = h.profile_read() if prof_on else {}
    h.profile(False)
    print(json.dumps({"step": s, "k": s % 2, "ms": round(e[0].elapsed_time(e[1]), 3),
                      "levels": info["n_levels"], "n_c": info["n_coarse"],
                      "phases": {k: round(v[1], 3) for k, v in prof.items() if v[1] > 0}}), flush=True)
    if solve:
        x, st = step.solve(cs)
        torch.cuda.synchronize()
        print("solve", st["iters"], flush=True)
