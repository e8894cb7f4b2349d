"""Seeded synthetic graph generators shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no BFS, no relaxation, no
frontier logic): it only builds input graphs and picks sources, so both the
oracle tests and the CUDA parity tests can draw identical inputs from it.

Everything random is a counter-based hash (splitmix64 finaliser) of
(seed, counter), compared against integer thresholds, so the numpy generator
here and the CUDA generator in ``gen.cu`` (used for the large configs) are
bit-identical.  DESIGN.md §"Input recipe" states the recipe; the readings it
follows are A5 (weights), A6 (weight range), A7 (dedup/self-loops), A8 (rMAT),
A9 (sources), A22 (torus layout).

Graphs are CSR: ``offsets`` int64[n+1], ``targets`` uint32[m] (sorted
ascending within each adjacency list, no self-loops, no duplicates), optional
``weights`` uint32[m].
"""
from __future__ import annotations

import numpy as np

from .configs import CONFIGS, Config  # noqa: F401

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
C1 = np.uint64(0xBF58476D1CE4E5B9)
C2 = np.uint64(0x94D049BB133111EB)


def mix64(z):
    """splitmix64 finaliser on uint64 (scalar or array); wraps mod 2^64."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * C1
        z = (z ^ (z >> np.uint64(27))) * C2
    return z ^ (z >> np.uint64(31))


def seed_key(seed: int) -> np.uint64:
    return np.uint64(mix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF)))


def hash64(key, ctr):
    """H(key, ctr) = mix64(key + (ctr + 1) * GOLDEN)  (all mod 2^64)."""
    ctr = np.asarray(ctr, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(key) + (ctr + np.uint64(1)) * GOLDEN
    return mix64(z)


def rmat_thresholds(a: float, b: float, c: float):
    """Integer thresholds on a 32-bit uniform: [0,T1)=a, [T1,T2)=b, [T2,T3)=c, rest=d."""
    t1 = int(a * 2**32)
    t2 = int((a + b) * 2**32)
    t3 = int((a + b + c) * 2**32)
    assert 0 < t1 <= t2 <= t3 <= 2**32
    return t1, t2, t3


def rmat_edges(levels: int, start: int, count: int, seed: int, a: float, b: float, c: float):
    """Raw rMAT samples [start, start+count): (u, v) uint32 arrays (reading A8).

    Level l of edge i draws r = H(key, i*levels + l) >> 32 and picks the quadrant
    (u-bit, v-bit) = a:(0,0) b:(0,1) c:(1,0) d:(1,1), most significant bit first.
    No noise, no vertex permutation (so vertex 0 is the hub)."""
    key = seed_key(seed)
    t1, t2, t3 = (np.uint64(t) for t in rmat_thresholds(a, b, c))
    i = np.arange(start, start + count, dtype=np.uint64)
    u = np.zeros(count, np.uint64)
    v = np.zeros(count, np.uint64)
    L = np.uint64(levels)
    for lvl in range(levels):
        r = hash64(key, i * L + np.uint64(lvl)) >> np.uint64(32)
        ub = (r >= t2).astype(np.uint64)
        vb = (((r >= t1) & (r < t2)) | (r >= t3)).astype(np.uint64)
        u = (u << np.uint64(1)) | ub
        v = (v << np.uint64(1)) | vb
    return u.astype(np.uint32), v.astype(np.uint32)


def csr_from_edges(n: int, u, v, symmetric: bool):
    """Drop self-loops, optionally symmetrize, dedup, sort -> (offsets, targets)."""
    u = np.asarray(u, np.uint64)
    v = np.asarray(v, np.uint64)
    keep = u != v
    u, v = u[keep], v[keep]
    if symmetric:
        u, v = np.concatenate([u, v]), np.concatenate([v, u])
    keys = np.unique((u << np.uint64(32)) | v)
    src = (keys >> np.uint64(32)).astype(np.int64)
    tgt = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    offsets = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=offsets[1:])
    return offsets, tgt


def edge_sources(offsets):
    n = offsets.shape[0] - 1
    return np.repeat(np.arange(n, dtype=np.uint32), np.diff(offsets))


def pair_weights(offsets, targets, seed: int, W: int):
    """w(u,v) = 1 + (H(key, min(u,v)<<32 | max(u,v)) mod W)  (readings A5, A6).

    A function of the unordered pair, so symmetric graphs get symmetric weights."""
    u = edge_sources(offsets).astype(np.uint64)
    v = np.asarray(targets, np.uint64)
    lo, hi = np.minimum(u, v), np.maximum(u, v)
    h = hash64(seed_key(seed), (lo << np.uint64(32)) | hi)
    return (np.uint64(1) + h % np.uint64(W)).astype(np.uint32)


def rmat_graph(levels: int, nedges: int, seed: int, a: float, b: float, c: float,
               symmetric: bool = True):
    n = 1 << levels
    u, v = rmat_edges(levels, 0, nedges, seed, a, b, c)
    off, tgt = csr_from_edges(n, u, v, symmetric)
    return off, tgt


def torus3d(L: int):
    """3D torus L^3, id = x + L*(y + L*z) (reading A22), 6 neighbours (+-1 mod L per
    dimension), adjacency sorted ascending. L >= 3 keeps the 6 neighbours distinct."""
    assert L >= 3
    n = L ** 3
    ids = np.arange(n, dtype=np.int64)
    x, y, z = ids % L, (ids // L) % L, ids // (L * L)
    nb = []
    for dx, dy, dz in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
        nb.append(((x + dx) % L) + L * (((y + dy) % L) + L * ((z + dz) % L)))
    nb = np.sort(np.stack(nb, axis=1), axis=1)
    offsets = np.arange(0, 6 * n + 1, 6, dtype=np.int64)
    return offsets, nb.reshape(-1).astype(np.uint32)


def choose_sources(candidates, k: int, seed: int):
    """k distinct sources from a sorted candidate array: index_j = H(key, j) mod |C|,
    j = 0, 1, ... skipping repeats (reading A9)."""
    candidates = np.asarray(candidates)
    assert candidates.size > 0
    k = min(k, candidates.size)
    key = seed_key(seed)
    out, seen, j = [], set(), 0
    while len(out) < k:
        idx = int(hash64(key, np.uint64(j)) % np.uint64(candidates.size))
        j += 1
        if idx in seen:
            continue
        seen.add(idx)
        out.append(int(candidates[idx]))
    return out


def largest_component(offsets, targets):
    """Vertices of the largest connected component (symmetric CSR), sorted."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import connected_components
    n = offsets.shape[0] - 1
    A = sp.csr_matrix((np.ones(targets.shape[0], np.int8), targets.astype(np.int64), offsets),
                      shape=(n, n))
    _, lab = connected_components(A, directed=False)
    big = np.bincount(lab).argmax()
    return np.nonzero(lab == big)[0].astype(np.int64)


# --- small random graphs for tests --------------------------------------------

def random_graph(n: int, p: float, seed: int, symmetric: bool = True):
    """Erdos-Renyi-like graph from the counter hash (pair (i,j) kept iff
    H(key, i*n+j) < p*2^64)."""
    key = seed_key(seed)
    i, j = np.meshgrid(np.arange(n, dtype=np.uint64), np.arange(n, dtype=np.uint64), indexing="ij")
    h = hash64(key, i * np.uint64(n) + j)
    keep = h < np.uint64(min(int(p * 2**64), 2**64 - 1))
    u, v = i[keep], j[keep]
    return csr_from_edges(n, u, v, symmetric)


def from_edge_list(n: int, edges, symmetric: bool = True, weights=None):
    """CSR from an explicit (u, v[, w]) list; weights by edge (symmetric copies share w)."""
    if weights is None:
        u = np.array([e[0] for e in edges], np.uint64)
        v = np.array([e[1] for e in edges], np.uint64)
        return csr_from_edges(n, u, v, symmetric)
    wmap = {}
    for (a, b), w in zip(edges, weights):
        wmap[(a, b)] = w
        if symmetric:
            wmap[(b, a)] = w
    keys = sorted(wmap)
    offsets = np.zeros(n + 1, np.int64)
    for a, _ in keys:
        offsets[a + 1] += 1
    offsets = np.cumsum(offsets)
    tgt = np.array([b for _, b in keys], np.uint32)
    wt = np.array([wmap[k] for k in keys], np.uint32)
    return offsets, tgt, wt
