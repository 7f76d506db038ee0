"""Launch trace of one warm C3 coarsen (tag -> map -> assemble) with AGIPC_TRACE: per kernel
GPU start / duration, the idle gap before it on its stream and the host submit time, to find
where the step's time goes between kernels.  Diagnostics only."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/trace_c3.txt"
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
xcd = [t(x, torch.float64) for x in xcs]
step = CoarseningStep(h, dm, Hrp, Hcol, Hval)
evs = []
for s in range(6):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a.record()
    step.coarsen(xp, xcd[(3 + s) % 10], gd)
    b.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    evs.append((a.elapsed_time(b), 1e3 * (t1 - t0)))
for e in evs:
    print(f"coarsen event {e[0]:.3f} ms, host call {e[1]:.3f} ms")
h.close() if hasattr(h, "close") else None
del step, h
import gc; gc.collect()
