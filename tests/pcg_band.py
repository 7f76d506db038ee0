"""Acceptance band for PCG iteration counts (reading R25).

Near a stopping tolerance the CG residual curve can hover around the threshold for several
iterations (C2: ||r||/||b|| stays in 1.01e-3..1.3e-3 for ~10 iterations), so ANY change of the
rounding -- far below the 1e-12 value-parity contract -- moves the stopping iteration: the
oracle itself run on copies of its coarse matrix perturbed by 1e-16 relative noise stops at
202..209 iterations on C2.  The band is therefore the spread of the oracle under such
perturbations (computed live, oracle only), widened by 2 iterations."""
import numpy as np

import oracle


def oracle_iteration_band(row_ptr, col, val, b, tol, n_pert=8, rel=1e-15, max_iters=20000, slack=2):
    """slack: iterations added on both sides (2; the distributed solve uses 4: its p.q, r.z and
    r.r are partial sums per rank added in rank order, a further rounding order, and its halo
    coarse blocks are summed with atomics -- reading R25)."""
    its = [oracle.pcg(row_ptr, col, val, b, rel_tol=tol, max_iters=max_iters)["iters"]]
    for s in range(n_pert):
        e = rel * np.random.default_rng([s, 99]).standard_normal(val.shape[0])
        its.append(oracle.pcg(row_ptr, col, val * (1.0 + e[:, None, None]), b, rel_tol=tol,
                              max_iters=max_iters)["iters"])
    return min(its) - slack, max(its) + slack
