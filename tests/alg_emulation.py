"""Literal emulation of supplement Algorithms S1 and S2,
applied recursively.  TEST CODE: an independent check of the oracle's
union-find definition of the map.  It follows the printed pseudo-code line by
line, including the per-node while-loop BFS over the *initial* hashes (Hashs[]
in shared memory) and the election.

The only deviation is the local-index line P:183-184, which as printed uses
``lane_id``; ``corrected=True`` uses the first set bit of the final hash as the
text says -- DESIGN.md reading R1.  ``corrected=False`` keeps the
printed formula so tests can show it contradicts the paper's own examples.
"""


def ffs(x):
    """CUDA __ffs: 1-based position of the least significant set bit, 0 if none."""
    return (x & -x).bit_length()


def popc(x):
    return bin(x).count("1")


def alg_s1(n, gs, nbrs, tag):
    """Alg S1: con_hashs[node] = 1<<lane | bits of same-group tagged neighbours."""
    h = [0] * n
    for node in range(n):
        group_id = node // gs
        lane_id = node % gs
        h[node] = 1 << lane_id
        for nb in nbrs[node]:
            if tag(node, nb) == 0:
                continue
            if nb // gs == group_id:
                h[node] |= 1 << (nb % gs)
    return h


def alg_s2(h0, gs, corrected=True):
    """Alg S2 for all groups (each group is one 'block' here).  Returns
    (final hashes, P, counts per group, map)."""
    n = len(h0)
    n_groups = (n + gs - 1) // gs
    full = (1 << gs) - 1  # P:164; for gs = 32 this is the full 32-bit mask (R2)
    final = [0] * n
    P = [0] * n
    counts = [0] * n_groups
    elect = [0] * n_groups
    for g in range(n_groups):
        lo, hi = g * gs, min(n, (g + 1) * gs)
        Hashs = h0[lo:hi]
        for node in range(lo, hi):
            lane_id = node - lo
            conHash = h0[node]
            visited = 1 << lane_id
            while conHash != full:
                todo = visited ^ conHash
                if todo == 0:
                    break
                nxt = ffs(todo) - 1
                visited |= 1 << nxt
                conHash |= Hashs[nxt]
            final[node] = conHash
            prefix = popc(conHash & ((1 << lane_id) - 1))
            if prefix == 0:
                counts[g] += 1
                elect[g] |= 1 << lane_id
        for node in range(lo, hi):
            lane_id = node - lo
            if corrected:
                mask = elect[g] & ((1 << (ffs(final[node]) - 1)) - 1)
            else:
                mask = elect[g] & ((1 << lane_id) - 1)
            P[node] = popc(mask)
    O = [0] * n_groups
    for g in range(1, n_groups):
        O[g] = O[g - 1] + counts[g - 1]
    mp = [O[node // gs] + P[node] for node in range(n)]
    return final, P, counts, mp


def build_map_emulated(n, gs, edges, max_levels=0, corrected=True):
    """Recursive application: each level's coarse nodes and the mapped
    surviving edges become the next level's input.  edges: iterable of
    collapsible undirected pairs.  Returns (map, n_coarse, n_levels, level_n)."""
    cur = list(range(n))
    E = {(min(u, v), max(u, v)) for u, v in edges if u != v}
    level_n = []
    m = n
    while True:
        nbrs = [[] for _ in range(m)]
        for u, v in E:
            nbrs[u].append(v)
            nbrs[v].append(u)
        h0 = alg_s1(m, gs, nbrs, lambda a, b: 1)
        _, _, counts, mk = alg_s2(h0, gs, corrected)
        nn = sum(counts)
        cur = [mk[c] for c in cur]
        E = {(min(mk[u], mk[v]), max(mk[u], mk[v])) for u, v in E if mk[u] != mk[v]}
        level_n.append(nn)
        done = nn == m or (max_levels > 0 and len(level_n) >= max_levels)
        m = nn
        if done:
            return cur, m, len(level_n), level_n
