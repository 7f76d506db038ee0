"""Launch trace of the NEXT#1 fine solve on the static pattern (C3, 10 iterations from a
prolongated start): per kernel duration and idle gaps.  Diagnostics only."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
out = sys.argv[1]
if os.path.exists(out):
    os.remove(out)
os.environ["AGIPC_TRACE"] = out
import numpy as np
import torch
import bench
import paper_2605_04773_b200 as P
from paper_2605_04773_b200.step import CoarseningStep

dev = torch.device("cuda", 0)
m, H, g, xcs, _ = bench.build_inputs(100)
h = P.Handle(0)
t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a)).to(dev, dt)
dm = P.DeviceMesh.from_arrays(m.tets, m.adj_ptr, m.adj_nbr, m.tet_slots, m.X, device=dev)
Hrp, Hcol, Hval = t(m.bsr_ptr, torch.int64), t(m.bsr_col, torch.int32), t(H, torch.float64)
gd, xp = t(g, torch.float64), t(m.X, torch.float64)
step = CoarseningStep(h, dm, Hrp, Hcol, Hval)
cs = step.coarsen(xp, t(xcs[3], torch.float64), gd)[2]
y_c, _ = step.solve(cs)
yf = torch.empty((m.n_nodes, 3), dtype=torch.float64, device=dev)
h.pcg_set_static(Hrp, Hcol)
for r in range(4):
    P.prolongate(h, dm, cs.new_map, cs.n3, cs.n_slots, y_c, 1.0, yf)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _, st = P.pcg_solve(h, Hrp, Hcol, Hval, gd, yf, 1e-3, 10, 10)
    b.record()
    torch.cuda.synchronize()
    print("solve", r, round(a.elapsed_time(b), 3), "ms", st["iters"], "iters")
h.pcg_set_static()
del step
h.close()
