"""Experiment (NEXT#2 design study, not a product path): PCG SpMV time at C3 for full storage
(k_spmv_sell) and the symmetric upper-half SpMV (k_spmv_sym), on the coarse system in the
library's slot order (3-DoF first) and in a locality order (slots sorted by the minimum
fine member of their aggregate, 12-DoF slots kept together).  The permutation is plain torch
index work done here; the solves run through the C ABI.  Prints one JSON line per variant."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2605_04773_b200 as P  # noqa: E402
import synth  # noqa: E402
from paper_2605_04773_b200.step import CoarseningStep  # noqa: E402


def permuted(cs, N):
    n, n3 = cs.n_slots, cs.n3
    dev = cs.val.device
    nc = n3 + (n - n3) // 4
    minm = torch.full((nc,), 1 << 40, dtype=torch.int64, device=dev)
    minm.scatter_reduce_(0, cs.new_map.long(), torch.arange(N, device=dev), reduce="amin")
    s = torch.arange(n, device=dev)
    node = torch.where(s < n3, s, n3 + (s - n3) // 4)
    key = minm[node] * 4 + torch.where(s < n3, 0, (s - n3) % 4)
    perm = torch.argsort(key)
    inv = torch.empty_like(perm)
    inv[perm] = s
    rp = cs.row_ptr
    row = torch.repeat_interleave(torch.arange(n, device=dev), rp[1:] - rp[:-1])
    pr, pc = inv[row], inv[cs.col.long()]
    o = torch.argsort(pr * n + pc)
    cnt = torch.bincount(pr, minlength=n)
    prp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    prp[1:] = torch.cumsum(cnt, 0)
    return prp, pc[o].to(torch.int32).contiguous(), cs.val[o].contiguous(), cs.g_c[perm].contiguous()


def main():
    m = synth.kuhn_grid(100)
    c = synth.config_c3(k=0)
    H = synth.fine_hessian(m, E=1e5)
    g = synth.fine_gradient(m.n_nodes)
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a)).to("cuda:0", dt)  # noqa: E731
    h = P.Handle(0)
    dm = P.DeviceMesh.from_arrays(m.tets, m.adj_ptr, m.adj_nbr, m.tet_slots, m.X, device="cuda:0")
    st = CoarseningStep(h, dm, t(m.bsr_ptr, torch.int64), t(m.bsr_col, torch.int32), t(H, torch.float64))
    _, info, cs = st.coarsen(t(c["x_prev"], torch.float64), t(c["x_cur"], torch.float64), t(g, torch.float64))
    systems = {"slot_order": (cs.row_ptr, cs.col, cs.val, cs.g_c), "locality_order": permuted(cs, m.n_nodes)}
    if "--full" in sys.argv:  # full storage, slot order (A/B of environment settings per process)
        rp, col, val, b = systems["slot_order"]
        x = torch.empty_like(b)
        P.pcg_solve(h, rp, col, val, b, x, 0.0, 64, 32, zero_x0=True)
        h.profile(True)
        for _ in range(3):
            _, s = P.pcg_solve(h, rp, col, val, b, x, 0.0, 256, 32, zero_x0=True)
        pr = h.profile_read()
        h.profile(False)
        sp, up, so = pr["pcg_spmv"], pr["pcg_update"], pr["pcg_solve"]
        print(json.dumps({"l2_window": os.environ.get("AGIPC_L2_WINDOW", "1"),
                          "spmv_us": round(1e3 * sp[1] / sp[0], 2), "update_us": round(1e3 * up[1] / up[0], 2),
                          "us_per_iter": round(1e3 * so[1] / (3 * 256), 2)}), flush=True)
        return
    if "--update" in sys.argv:  # K2 launch shape sweep (full storage, slot order)
        rp, col, val, b = systems["slot_order"]
        for ctas in ("2", "3", "4", "8"):
            for u in ("1", "2"):
                os.environ["AGIPC_UPD_CTAS"] = ctas
                os.environ["AGIPC_UPD_U"] = u
                x = torch.empty_like(b)
                P.pcg_solve(h, rp, col, val, b, x, 0.0, 64, 32, zero_x0=True)
                h.profile(True)
                for _ in range(3):
                    _, s = P.pcg_solve(h, rp, col, val, b, x, 0.0, 256, 32, zero_x0=True)
                pr = h.profile_read()
                h.profile(False)
                sp, up = pr["pcg_spmv"], pr["pcg_update"]
                print(json.dumps({"upd_ctas": ctas, "upd_u": u, "spmv_us": round(1e3 * sp[1] / sp[0], 2),
                                  "update_us": round(1e3 * up[1] / up[0], 2)}), flush=True)
        return
    for name, (rp, col, val, b) in systems.items():
        for storage, sname in ((P.STORAGE_FULL, "full"), (P.STORAGE_SYM, "sym")):
            for win in (["256", "512", "1024", "red256", "red1024"] if storage else ["-"]):
                if win != "-":
                    os.environ["AGIPC_SYM_WIN"] = win.replace("red", "")
                if win.startswith("red"):
                    os.environ["AGIPC_SYM_RED"] = "1"
                x = torch.empty_like(b)
                P.pcg_solve(h, rp, col, val, b, x, 0.0, 64, 32, zero_x0=True, storage=storage)  # warm
                h.profile(True)
                for _ in range(3):
                    _, s = P.pcg_solve(h, rp, col, val, b, x, 0.0, 256, 32, zero_x0=True, storage=storage)
                pr = h.profile_read()
                h.profile(False)
                sp, up = pr["pcg_spmv"], pr["pcg_update"]
                print(json.dumps({"order": name, "storage": sname, "win": win, "n": int(rp.shape[0] - 1),
                                  "nnzb": int(col.shape[0]), "spmv_us": round(1e3 * sp[1] / sp[0], 2),
                                  "update_us": round(1e3 * up[1] / up[0], 2), "iters": s["iters"]}), flush=True)
                os.environ.pop("AGIPC_SYM_WIN", None)
                os.environ.pop("AGIPC_SYM_RED", None)


if __name__ == "__main__":
    main()
