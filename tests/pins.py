"""Independent pins for the oracle: closed forms, brute force, Floyd–Warshall.

None of this calls oracle/; each function is derived from the mathematics of
the graph family, not from a BFS or relaxation loop (except brute force, which
enumerates every simple path and so needs no shortest-path algorithm at all).
"""
from __future__ import annotations

import itertools

import numpy as np

INF = 0xFFFFFFFF


def ring_dist(a, b, L):
    d = np.abs(np.asarray(a, np.int64) - np.asarray(b, np.int64))
    return np.minimum(d, L - d)


def torus_dist(L: int, src: int):
    """d(v) = sum over the 3 dimensions of the ring distance (id = x + L(y + Lz))."""
    ids = np.arange(L ** 3, dtype=np.int64)
    sx, sy, sz = src % L, (src // L) % L, src // (L * L)
    return (ring_dist(ids % L, sx, L) + ring_dist((ids // L) % L, sy, L)
            + ring_dist(ids // (L * L), sz, L)).astype(np.uint32)


def ring_shells(L: int):
    """Number of ring vertices at ring distance k from a fixed vertex, k = 0..L//2."""
    s = np.zeros(L // 2 + 1, np.int64)
    for k in range(L):
        s[min(k, L - k)] += 1
    return s


def torus_level_counts(L: int):
    """Per-level vertex counts of BFS on the L^3 torus = triple convolution of shells."""
    s = ring_shells(L)
    return np.convolve(np.convolve(s, s), s)


def torus_ecc(L: int) -> int:
    return 3 * (L // 2)


def path_graph(n: int):
    edges = [(i, i + 1) for i in range(n - 1)]
    return edges


def grid_dist(a: int, b: int, src: int):
    ids = np.arange(a * b)
    return (np.abs(ids % a - src % a) + np.abs(ids // a - src // a)).astype(np.uint32)


def grid_edges(a: int, b: int):
    e = []
    for y in range(b):
        for x in range(a):
            v = x + a * y
            if x + 1 < a:
                e.append((v, v + 1))
            if y + 1 < b:
                e.append((v, v + a))
    return e


def recursive_tree(n: int, seed: int):
    """Random recursive tree: parent(i) = h(i) mod i.  Returns (edges, parent, depth)
    with depth computed by the recurrence depth[i] = depth[parent[i]] + 1."""
    rng = np.random.default_rng(seed)
    par = np.zeros(n, np.int64)
    depth = np.zeros(n, np.int64)
    for i in range(1, n):
        par[i] = rng.integers(0, i)
        depth[i] = depth[par[i]] + 1
    return [(int(par[i]), i) for i in range(1, n)], par, depth


def brute_force_sssp(n: int, offsets, targets, weights, src: int):
    """Minimum over ALL simple src->v paths of the path weight (n <= 9)."""
    adj = {u: [(int(targets[e]), 1 if weights is None else int(weights[e]))
               for e in range(offsets[u], offsets[u + 1])] for u in range(n)}
    best = [None] * n
    best[src] = 0

    def dfs(u, acc, seen):
        for v, w in adj[u]:
            if v in seen:
                continue
            if best[v] is None or acc + w < best[v]:
                best[v] = acc + w
            seen.add(v)
            dfs(v, acc + w, seen)
            seen.remove(v)

    dfs(src, 0, {src})
    return np.array([INF if b is None else b for b in best], np.uint64)


def floyd_warshall(n: int, offsets, targets, weights):
    """All-pairs shortest paths by Floyd–Warshall in float (exact for small ints)."""
    D = np.full((n, n), np.inf)
    np.fill_diagonal(D, 0.0)
    for u in range(n):
        for e in range(offsets[u], offsets[u + 1]):
            w = 1.0 if weights is None else float(weights[e])
            D[u, targets[e]] = min(D[u, targets[e]], w)
    for k in range(n):
        D = np.minimum(D, D[:, k:k + 1] + D[k:k + 1, :])
    return D


def fw_row_u32(D, src):
    row = D[src]
    out = np.full(row.shape, INF, np.uint64)
    fin = np.isfinite(row)
    out[fin] = row[fin].astype(np.uint64)
    return out


def all_small_graphs(n: int):
    """Every undirected simple graph on n labelled vertices (n <= 4)."""
    pairs = list(itertools.combinations(range(n), 2))
    for mask in range(1 << len(pairs)):
        yield [p for i, p in enumerate(pairs) if mask >> i & 1]


def brute_force_widest(n: int, offsets, targets, weights, src: int):
    """Max over ALL simple src->v paths of the minimum edge weight (n <= 9);
    width[src] = INF (empty path), unreachable 0 (readings W1/W2)."""
    adj = {u: [(int(targets[e]), 1 if weights is None else int(weights[e]))
               for e in range(offsets[u], offsets[u + 1])] for u in range(n)}
    best = [0] * n
    best[src] = INF

    def dfs(u, bottleneck, seen):
        for v, w in adj[u]:
            if v in seen:
                continue
            b = min(bottleneck, w)
            if b > best[v]:
                best[v] = b
            seen.add(v)
            dfs(v, b, seen)
            seen.remove(v)

    dfs(src, INF, {src})
    return np.array(best, np.uint64)


def brute_force_dependencies(n: int, offsets, targets, src: int):
    """delta_src(v) = sum_{t != src, v} sigma_st(v) / sigma_st straight from the
    definition (pair dependencies; no Brandes recurrence): shortest-path counts
    between every pair by a BFS from every vertex, sigma_st(v) = sigma_sv *
    sigma_vt when d(s,v) + d(v,t) = d(s,t)."""
    adj = [[int(targets[e]) for e in range(offsets[u], offsets[u + 1])] for u in range(n)]

    def bfs_counts(s):
        d = [None] * n
        c = [0] * n
        d[s], c[s] = 0, 1
        frontier = [s]
        while frontier:
            nxt = []
            for u in frontier:
                for v in adj[u]:
                    if d[v] is None:
                        d[v] = d[u] + 1
                        nxt.append(v)
                    if d[v] == d[u] + 1:
                        c[v] += c[u]
            frontier = nxt
        return d, c

    D, C = zip(*[bfs_counts(s) for s in range(n)])
    out = np.zeros(n)
    for v in range(n):
        if v == src or D[src][v] is None:
            continue
        for t in range(n):
            if t in (src, v) or D[src][t] is None or D[v][t] is None:
                continue
            if D[src][v] + D[v][t] == D[src][t]:
                out[v] += C[src][v] * C[v][t] / C[src][t]
    return out


# ---- NEXT-4 signed weights ----------------------------------------------------------

def signed_csr(n: int, edges, weights):
    """Directed CSR (sorted, duplicates keep the last weight) with int32 weights
    returned as their uint32 two's-complement bit patterns (the ABI's layout)."""
    wmap = {}
    for (a, b), w in zip(edges, weights):
        wmap[(a, b)] = int(w)
    keys = sorted(wmap)
    offsets = np.zeros(n + 1, np.int64)
    for a, _ in keys:
        offsets[a + 1] += 1
    offsets = np.cumsum(offsets)
    tgt = np.array([b for _, b in keys], np.uint32)
    wt = np.array([wmap[k] for k in keys], np.int64).astype(np.int32).view(np.uint32)
    return offsets, tgt, wt


def signed_expected(n: int, offsets, targets, w_u32, src: int, scope: int):
    """Independent of the oracle: Floyd–Warshall over int32 weights (exact in
    float64 for small ints) finds negative cycles (D[k,k] < 0); a boolean
    transitive closure gives reachability.  v is -inf iff some k with D[k,k] < 0
    is reachable from src and reaches v (scope 1), or, with scope 0, iff any
    such k exists at all.  Otherwise D[src, v] (inf if unreachable)."""
    w = w_u32.view(np.int32).astype(np.float64)
    D = floyd_warshall(n, offsets, targets, w)
    R = np.eye(n, dtype=bool)
    for u in range(n):
        for e in range(offsets[u], offsets[u + 1]):
            R[u, targets[e]] = True
    for k in range(n):
        R = R | (R[:, k:k + 1] & R[k:k + 1, :])
    neg = np.array([D[k, k] < 0 for k in range(n)])
    bad = neg & R[src]
    out = np.empty(n, np.int64)
    down = (R[bad].any(axis=0)) if bad.any() else np.zeros(n, bool)
    for v in range(n):
        if bad.any() and (scope == 0 or down[v]):
            out[v] = np.iinfo(np.int64).min
        elif not R[src, v]:
            out[v] = np.iinfo(np.int64).max
        else:
            out[v] = int(D[src, v])
    return out, bool(bad.any())


def johnson_reweight(offsets, targets, w_u32, phi):
    """w'(u,v) = w(u,v) + phi(u) - phi(v): same shortest paths, no new negative
    cycles (every cycle keeps its weight), d'(v) = d(v) + phi(src) - phi(v)."""
    u = np.repeat(np.arange(offsets.shape[0] - 1), np.diff(offsets))
    w2 = w_u32.astype(np.int64) + phi[u] - phi[targets]
    assert (np.abs(w2) < 2 ** 31).all()
    return w2.astype(np.int32).view(np.uint32)
