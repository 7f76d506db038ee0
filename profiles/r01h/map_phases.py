"""Experiment: where the build_map time goes at C3 (library CUDA-event phases map_level0 /
map_tail inside build_map, plus the whole call), 10 warm coarsen steps, L2 flushed."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2605_04773_b200 as P  # noqa: E402
import synth  # noqa: E402
from paper_2605_04773_b200.step import CoarseningStep  # noqa: E402

m = synth.kuhn_grid(100)
H = synth.fine_hessian(m, E=1e5)
g = synth.fine_gradient(m.n_nodes)
t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a)).to("cuda:0", dt)  # noqa: E731
h = P.Handle(0)
dm = P.DeviceMesh.from_arrays(m.tets, m.adj_ptr, m.adj_nbr, m.tet_slots, m.X, device="cuda:0")
st = CoarseningStep(h, dm, t(m.bsr_ptr, torch.int64), t(m.bsr_col, torch.int32), t(H, torch.float64))
xs = [t(synth.config_c3(k=k)["x_cur"], torch.float64) for k in range(3)]
xp = t(m.X, torch.float64)
gd = t(g, torch.float64)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda:0")
for k in range(3):
    st.coarsen(xp, xs[k], gd)
torch.cuda.synchronize()
h.profile(True)
walls = []
for s in range(9):
    flush.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, info, cs = st.coarsen(xp, xs[s % 3], gd)
    torch.cuda.synchronize()
    walls.append(1e3 * (time.perf_counter() - t0))
pr = h.profile_read()
print(json.dumps({k: round(v[1] / max(1, v[0]), 4) for k, v in pr.items()}))
print(json.dumps({"wall_ms_mean": round(float(np.mean(walls)), 4), "levels": info["n_levels"]}))
