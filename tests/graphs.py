"""Small seeded test graphs (raw edge lists) and brute-force references.

Inputs only: the brute-force references here are written from the plain
mathematical definitions (sets of pairs, dense matrices) and are used to PIN
the oracle; they share nothing with the CUDA path.
"""
from __future__ import annotations

import numpy as np


def edges_to_arrays(edges):
    if len(edges) == 0:
        return np.zeros(0, np.int32), np.zeros(0, np.int32)
    a = np.asarray(edges, dtype=np.int32)
    return np.ascontiguousarray(a[:, 0]), np.ascontiguousarray(a[:, 1])


def cycle(n):
    return [(i, (i + 1) % n) for i in range(n)]


def in_star(n):          # leaves 1..n-1 -> centre 0
    return [(i, 0) for i in range(1, n)]


def out_star(n):         # centre 0 -> leaves
    return [(0, i) for i in range(1, n)]


def path(L):
    return [(i, i + 1) for i in range(L - 1)]


def complete(n):
    return [(i, j) for i in range(n) for j in range(n) if i != j]


def random_edges(n, m, seed, loops=True, dups=True):
    rng = np.random.default_rng(seed)
    s = rng.integers(0, n, m)
    t = rng.integers(0, n, m)
    if dups:   # force some repeats
        k = m // 10
        s[:k] = s[m - k:]
        t[:k] = t[m - k:]
    if not loops:
        t = np.where(s == t, (t + 1) % n, t)
    return list(zip(s.tolist(), t.tolist()))


def planted_graph(seed, n_base=120, groups=((0, 5), (1, 3)), chains=(10, 10, 10), pure_cycle=5):
    """Random base graph + planted identical groups, chains and one pure cycle."""
    rng = np.random.default_rng(seed)
    edges = random_edges(n_base, 4 * n_base, seed, loops=False)
    n = n_base
    # identical groups: every member gets edges from the same source set
    for _, size in groups:
        srcs = rng.choice(n_base, size=3, replace=False).tolist()
        for _ in range(size):
            for s in srcs:
                edges.append((s, n))
            edges.append((n, int(rng.integers(0, n_base))))
            n += 1
    # chains p -> v1 -> ... -> vL -> s
    for L in chains:
        p = int(rng.integers(0, n_base))
        prev = p
        for _ in range(L):
            edges.append((prev, n))
            prev = n
            n += 1
        edges.append((prev, int(rng.integers(0, n_base))))
    # pure cycle of chain vertices (isolated component)
    base = n
    for i in range(pure_cycle):
        edges.append((base + i, base + (i + 1) % pure_cycle))
    n += pure_cycle
    return n, edges


# ------------------------------------------------------------ brute force --
def bf_pairs(n, edges):
    return sorted({(s, t) for s, t in edges if s != t})


def bf_csr(n, edges):
    pairs = bf_pairs(n, edges)
    rows = [[] for _ in range(n)]
    od = [0] * n
    for s, t in pairs:
        rows[t].append(s)
        od[s] += 1
    rp = [0]
    col = []
    for v in range(n):
        rows[v].sort()
        col.extend(rows[v])
        rp.append(len(col))
    return rp, col, od


def bf_identical(n, edges):
    """O(n^2) pairwise in-set comparison."""
    ins = [set() for _ in range(n)]
    for s, t in bf_pairs(n, edges):
        ins[t].add(s)
    rep = []
    for v in range(n):
        r = v
        for w in range(v):
            if ins[w] == ins[v]:
                r = w
                break
        rep.append(r)
    return rep


def bf_chains(n, edges, rep):
    """Backward walk per vertex (a different formulation from the oracle's
    forward walk): v is a member iff chain(v), and following pred from v
    reaches a head h within n steps; k = steps; src = rep(h)."""
    rp, col, od = bf_csr(n, edges)
    indeg = [rp[v + 1] - rp[v] for v in range(n)]

    def is_chain(v):
        return indeg[v] == 1 and od[v] == 1

    src = [-1] * n
    kk = [0] * n
    for v in range(n):
        if not is_chain(v):
            continue
        w, k = v, 0
        while k <= n:
            p = col[rp[w]]
            if not is_chain(p):
                break               # w is a head
            w, k = p, k + 1
        if k >= 1 and k <= n and not is_chain(col[rp[w]]):
            src[v] = rep[w]
            kk[v] = k
    return src, kk


def dense_pagerank(n, edges, d):
    """Fixed point of Eq.(1): (I - dM) x = (1-d)/n * 1 with numpy.linalg.solve."""
    pairs = bf_pairs(n, edges)
    od = np.zeros(n)
    for s, _ in pairs:
        od[s] += 1
    M = np.zeros((n, n))
    for s, t in pairs:
        M[t, s] += 1.0 / od[s]
    A = np.eye(n) - d * M
    b = np.full(n, (1.0 - d) / n)
    return np.linalg.solve(A, b), M
