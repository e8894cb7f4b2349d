"""Pins for oracle/ (CPU only).  Each test checks the oracle against something
other than itself: closed forms, brute force over all simple paths,
Floyd–Warshall, a printed paper value, or an independent certificate — chosen so
a dropped term, wrong sign/index or transposed operand in oracle.c fails one."""
import numpy as np
import pytest

import graphgen
import oracle
from golden_io import read_examples, read_kv
from pins import (INF, all_small_graphs, brute_force_sssp, floyd_warshall, fw_row_u32,
                  grid_dist, grid_edges, path_graph, recursive_tree, ring_dist, torus_dist,
                  torus_ecc, torus_level_counts)




# ---- BFS: closed forms ------------------------------------------------------------

@pytest.mark.parametrize("n,src", [(1, 0), (2, 1), (7, 0), (7, 3), (50, 49)])
def test_bfs_path_closed_form(n, src):
    off, tgt = graphgen.from_edge_list(n, path_graph(n)) if n > 1 else (np.zeros(2, np.int64), np.zeros(0, np.uint32))
    d, p = oracle.bfs(off, tgt, src)
    assert (d == np.abs(np.arange(n) - src)).all()
    # a path is a tree: parents are unique
    exp_p = np.array([src if v == src else (v + 1 if v < src else v - 1) for v in range(n)])
    assert (p == exp_p).all()


@pytest.mark.parametrize("n,src", [(3, 0), (8, 5), (9, 2)])
def test_bfs_cycle_closed_form(n, src):
    edges = [(i, (i + 1) % n) for i in range(n)]
    off, tgt = graphgen.from_edge_list(n, edges)
    d, _ = oracle.bfs(off, tgt, src)
    assert (d == ring_dist(np.arange(n), src, n)).all()


def test_bfs_grid_manhattan():
    a, b = 9, 6
    off, tgt = graphgen.from_edge_list(a * b, grid_edges(a, b))
    for src in (0, 13, a * b - 1):
        d, _ = oracle.bfs(off, tgt, src)
        assert (d == grid_dist(a, b, src)).all()


@pytest.mark.parametrize("L", [3, 4, 5, 8])
def test_bfs_torus_closed_form(L):
    off, tgt = graphgen.torus3d(L)
    for src in (0, L ** 3 // 2 + 1):
        d, p = oracle.bfs(off, tgt, src)
        assert (d == torus_dist(L, src)).all()
        assert int(d.max()) == torus_ecc(L)
        assert (np.bincount(d) == torus_level_counts(L)).all()
        assert oracle.check_bfs(off, tgt, src, d, p)[0]


def test_torus_closed_form_matches_paper_row():
    """PAPER.md:2132 prints diam 1500 for the 1000^3 torus with 6e9 edges; the closed
    form eccentricity 3*floor(L/2) and level counts must reproduce it."""
    row = read_kv("paper_torus_row.txt")
    L = row["side"]
    assert L ** 3 == row["vertices"] and row["degree"] * L ** 3 == row["edges"]
    assert torus_ecc(L) == row["diam"]
    lv = torus_level_counts(L)
    assert len(lv) - 1 == row["diam"] and lv.sum() == row["vertices"] and lv[-1] == 1


def test_torus_c3_level_histogram_closed_form():
    """c3 (L=256): 385 levels summing to 2^24; shells 1, 6, 18, 38, 66; peak at 192."""
    lv = torus_level_counts(256)
    assert len(lv) == 385 and lv.sum() == 1 << 24
    assert list(lv[:5]) == [1, 6, 18, 38, 66]
    assert int(lv.argmax()) == 192


def test_bfs_complete_and_star_exact_parents():
    n = 9
    off, tgt = graphgen.from_edge_list(n, [(i, j) for i in range(n) for j in range(i + 1, n)])
    d, p = oracle.bfs(off, tgt, 4)
    assert (d == np.where(np.arange(n) == 4, 0, 1)).all() and (p == 4).all()
    off, tgt = graphgen.from_edge_list(n, [(0, i) for i in range(1, n)])
    d, p = oracle.bfs(off, tgt, 3)
    assert list(d) == [1, 2, 2, 0, 2, 2, 2, 2, 2]
    assert list(p) == [3, 0, 0, 3, 0, 0, 0, 0, 0]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_bfs_tree_exact(seed):
    n = 300
    edges, par, depth = recursive_tree(n, seed)
    off, tgt = graphgen.from_edge_list(n, edges)
    d, p = oracle.bfs(off, tgt, 0)
    assert (d == depth).all()
    assert p[0] == 0 and (p[1:] == par[1:]).all()


def test_bfs_disconnected_and_directed():
    off, tgt = graphgen.from_edge_list(5, [(0, 1), (1, 2), (3, 4)], symmetric=False)
    d, p = oracle.bfs(off, tgt, 1)
    assert list(d) == [INF, 0, 1, INF, INF]
    assert list(p) == [INF, 1, 1, INF, INF]


def test_reached_edges_closed_forms():
    """oracle_reached_edges (the TEPS numerator of reading A20) pinned by closed forms:
    on a connected symmetric graph (star, path, 3D torus) every vertex is reached, so
    it equals m; on a disjoint union it equals the source component's degree sum,
    i.e. twice its undirected edge count; a directed path reached from vertex i
    carries exactly the n-1-i edges out of i..n-2; an all-INF dist gives 0."""
    n = 12
    for edges in ([(0, i) for i in range(1, n)], path_graph(n)):
        off, tgt = graphgen.from_edge_list(n, edges)
        d, _ = oracle.bfs(off, tgt, 5)
        assert oracle.reached_edges(off, d) == tgt.shape[0] == 2 * (n - 1)
    off, tgt = graphgen.torus3d(4)
    assert oracle.reached_edges(off, oracle.bfs(off, tgt, 0)[0]) == 6 * 4 ** 3
    # K_4 on {0..3} (6 edges) + path on {4..9} (5 edges) + isolated 10, 11
    edges = [(i, j) for i in range(4) for j in range(i + 1, 4)] + [(i, i + 1) for i in range(4, 9)]
    off, tgt = graphgen.from_edge_list(12, edges)
    assert oracle.reached_edges(off, oracle.bfs(off, tgt, 2)[0]) == 12
    assert oracle.reached_edges(off, oracle.bfs(off, tgt, 7)[0]) == 10
    assert oracle.reached_edges(off, oracle.bfs(off, tgt, 11)[0]) == 0
    # directed path 0 -> 1 -> ... -> n-1 from vertex i: edges i..n-2 are reached
    off, tgt = graphgen.from_edge_list(n, path_graph(n), symmetric=False)
    for i in (0, 4, n - 1):
        assert oracle.reached_edges(off, oracle.bfs(off, tgt, i)[0]) == n - 1 - i
    assert oracle.reached_edges(off, np.full(n, INF, np.uint32)) == 0


# ---- BFS vs brute force / Floyd–Warshall ------------------------------------------

def test_bfs_all_graphs_on_4_vertices_brute_force():
    for edges in all_small_graphs(4):
        off, tgt = graphgen.from_edge_list(4, edges) if edges else (np.zeros(5, np.int64), np.zeros(0, np.uint32))
        for src in range(4):
            d, p = oracle.bfs(off, tgt, src)
            bf = brute_force_sssp(4, off, tgt, None, src)
            assert (d.astype(np.uint64) == bf).all()
            assert oracle.check_bfs(off, tgt, src, d, p)[0]


@pytest.mark.parametrize("seed", range(6))
def test_bfs_random_brute_force_and_fw(seed):
    n = 8
    off, tgt = graphgen.random_graph(n, 0.3, seed, symmetric=seed % 2 == 0)
    D = floyd_warshall(n, off, tgt, None)
    for src in range(n):
        d, _ = oracle.bfs(off, tgt, src)
        assert (d.astype(np.uint64) == brute_force_sssp(n, off, tgt, None, src)).all()
        assert (d.astype(np.uint64) == fw_row_u32(D, src)).all()


def test_bfs_fw_medium():
    n = 200
    off, tgt = graphgen.random_graph(n, 0.015, 11, symmetric=False)
    D = floyd_warshall(n, off, tgt, None)
    for src in (0, 77, 199):
        d, p = oracle.bfs(off, tgt, src)
        assert (d.astype(np.uint64) == fw_row_u32(D, src)).all()
        assert oracle.check_bfs(off, tgt, src, d, p)[0]


# ---- weighted: brute force, FW, closed forms ---------------------------------------

@pytest.mark.parametrize("seed", range(8))
def test_sssp_brute_force(seed):
    n = 8
    off, tgt = graphgen.random_graph(n, 0.35, 100 + seed, symmetric=seed % 2 == 1)
    w = graphgen.pair_weights(off, tgt, seed, 9) if seed % 3 else \
        (np.arange(tgt.shape[0]) % 7 + 1).astype(np.uint32)  # asymmetric weights too
    for src in range(n):
        bf = brute_force_sssp(n, off, tgt, w, src)
        d64, _ = oracle.dijkstra64(off, tgt, w, src)
        b64, _ = oracle.bellman_ford64(off, tgt, w, src)
        f64, _ = oracle.frontier_bellman_ford64(off, tgt, w, src)
        bf = np.where(bf == INF, oracle.INF64, bf)
        assert (d64 == bf).all() and (b64 == bf).all() and (f64 == bf).all()


def test_sssp_fw_medium_and_certificate():
    n = 150
    off, tgt = graphgen.random_graph(n, 0.03, 5, symmetric=True)
    w = graphgen.pair_weights(off, tgt, 9, 7)
    D = floyd_warshall(n, off, tgt, w)
    for src in (0, 42):
        d, p = oracle.dijkstra(off, tgt, w, src, want_parent=True)
        assert (d.astype(np.uint64) == fw_row_u32(D, src)).all()
        assert oracle.check_sssp(off, tgt, w, src, d)[0]
        # Dijkstra's own parent edge is tight (equality on the parent edge)
        reached = (d != INF) & (np.arange(n) != src)
        for v in np.nonzero(reached)[0]:
            u = p[v]
            es = range(off[u], off[u + 1])
            assert any(tgt[e] == v and int(d[u]) + int(w[e]) == int(d[v]) for e in es)


def test_sssp_weighted_path_prefix_sums():
    n = 40
    rng = np.random.default_rng(3)
    ws = rng.integers(1, 30, n - 1)
    off, tgt, w = graphgen.from_edge_list(n, path_graph(n), True, list(ws))
    d, _ = oracle.dijkstra(off, tgt, w, 0)
    assert (d == np.concatenate([[0], np.cumsum(ws)])).all()
    d2, _ = oracle.dijkstra(off, tgt, w, n - 1)
    assert (d2 == np.concatenate([np.cumsum(ws[::-1])[::-1], [0]])).all()


@pytest.mark.parametrize("c", [1, 7])
def test_sssp_constant_weight_torus(c):
    L = 6
    off, tgt = graphgen.torus3d(L)
    w = np.full(tgt.shape, c, np.uint32)
    d, _ = oracle.dijkstra(off, tgt, w, 5)
    assert (d == c * torus_dist(L, 5)).all()
    f, rounds = oracle.frontier_bellman_ford64(off, tgt, w, 5)
    assert (f == d).all() and rounds == torus_ecc(L) + 1


def test_unit_weights_equal_bfs():
    off, tgt = graphgen.rmat_graph(10, 1 << 13, 7, 0.57, 0.19, 0.19)
    d, _ = oracle.bfs(off, tgt, 0)
    for w in (None, np.ones(tgt.shape, np.uint32)):
        assert (oracle.dijkstra(off, tgt, w, 0)[0] == d).all()
        assert (oracle.narrow(oracle.frontier_bellman_ford64(off, tgt, w, 0)[0]) == d).all()


def test_spec_examples():
    for ex in read_examples():
        if ex["kind"] == "bfs":
            d, _ = oracle.bfs(ex["offsets"], ex["targets"], ex["src"])
        else:
            d, _ = oracle.dijkstra(ex["offsets"], ex["targets"], ex["weights"], ex["src"])
        assert (d == ex["expected"]).all(), ex["line"]


def test_narrow_overflow_and_zero_weight():
    with pytest.raises(OverflowError):
        oracle.narrow(np.array([0, 0xFFFFFFFF], np.uint64))
    off, tgt = graphgen.from_edge_list(3, [(0, 1), (1, 2)])
    w = np.array([0, 0, 1, 1], np.uint32)   # zero weights: oracle OK (reading A14)
    d, _ = oracle.dijkstra(off, tgt, w, 0)
    assert list(d) == [0, 0, 1]
    with pytest.raises(ValueError):
        oracle.check_sssp(off, tgt, w, 0, d)


# ---- certificates detect plausible mistakes ------------------------------------

def test_bfs_certificate_rejects_mutations():
    off, tgt = graphgen.rmat_graph(12, 1 << 15, 3, 0.57, 0.19, 0.19)
    d, p = oracle.bfs(off, tgt, 0)
    assert oracle.check_bfs(off, tgt, 0, d, p)[0]
    reached = np.nonzero((d != INF) & (d > 0))[0]
    rng = np.random.default_rng(0)
    for v in rng.choice(reached, 20, replace=False):
        for delta in (-1, 1):
            d2 = d.copy(); d2[v] = int(d[v]) + delta
            assert not oracle.check_bfs(off, tgt, 0, d2, p)[0]
        p2 = p.copy(); p2[v] = v            # not an in-neighbour one level closer
        assert not oracle.check_bfs(off, tgt, 0, d, p2)[0]
        # a same-level neighbour is a wrong parent
        nbrs = tgt[off[v]:off[v + 1]]
        same = nbrs[d[nbrs] == d[v]]
        if same.size:
            p3 = p.copy(); p3[v] = same[0]
            assert not oracle.check_bfs(off, tgt, 0, d, p3)[0]
    unreached = np.nonzero(d == INF)[0]
    d4 = d.copy(); d4[unreached[0]] = 5
    assert not oracle.check_bfs(off, tgt, 0, d4, None)[0]
    d5 = d.copy(); d5[0] = 1
    assert not oracle.check_bfs(off, tgt, 0, d5, p)[0]


def test_sssp_certificate_rejects_mutations():
    off, tgt = graphgen.rmat_graph(11, 1 << 14, 4, 0.57, 0.19, 0.19)
    w = graphgen.pair_weights(off, tgt, 4, 11)
    d, _ = oracle.dijkstra(off, tgt, w, 0)
    assert oracle.check_sssp(off, tgt, w, 0, d)[0]
    reached = np.nonzero((d != INF) & (d > 0))[0]
    for v in reached[:: max(1, reached.size // 15)]:
        for delta in (-1, 1):
            d2 = d.copy(); d2[v] = int(d[v]) + delta
            assert not oracle.check_sssp(off, tgt, w, 0, d2)[0]


def test_oracle_rejects_bad_args():
    off, tgt = graphgen.from_edge_list(3, [(0, 1)])
    with pytest.raises(RuntimeError):
        oracle.bfs(off, tgt, 3)
    with pytest.raises(ValueError):
        oracle.bfs(np.array([0, 5]), np.zeros(2, np.uint32), 0)


def test_c1_oracle_self_consistent():
    cfg = graphgen.CONFIGS["c1"]
    off, tgt = graphgen.rmat_graph(cfg.levels, 1 << cfg.log_edges, cfg.graph_seed, *cfg.abc)
    d, p = oracle.bfs(off, tgt, 0)
    assert oracle.check_bfs(off, tgt, 0, d, p)[0]
    # symmetric graph: |d(u) - d(v)| <= 1 across every edge (BASELINE.json north_star)
    u = graphgen.edge_sources(off)
    fin = d[u] != INF
    assert (np.abs(d[u][fin].astype(np.int64) - d[tgt][fin].astype(np.int64)) <= 1).all()
    w = graphgen.pair_weights(off, tgt, cfg.weight_seed, cfg.W)
    dd, _ = oracle.dijkstra(off, tgt, w, 0)
    f, _ = oracle.frontier_bellman_ford64(off, tgt, w, 0)
    assert (oracle.narrow(f) == dd).all()
    assert oracle.check_sssp(off, tgt, w, 0, dd)[0]


# ---- NEXT-1 widest path -----------------------------

from pins import brute_force_widest  # noqa: E402


@pytest.mark.parametrize("seed", range(8))
def test_widest_brute_force(seed):
    n = 8
    off, tgt = graphgen.random_graph(n, 0.35, 300 + seed, symmetric=seed % 2 == 0)
    w = graphgen.pair_weights(off, tgt, seed, 20) if seed % 3 else \
        (np.arange(tgt.shape[0]) % 9 + 1).astype(np.uint32)
    for src in range(n):
        ref = brute_force_widest(n, off, tgt, w, src)
        got = oracle.widest_path(off, tgt, w, src)
        assert (got.astype(np.uint64) == ref).all()
        assert oracle.check_widest(off, tgt, w, src, got)[0]


def test_widest_closed_forms_and_spec_examples():
    # SPEC.md:344  path 0-1 (3), 1-2 (5) plus edge 0-2 (2), src=0 -> D[2]=3
    off, tgt, w = graphgen.from_edge_list(3, [(0, 1), (1, 2), (0, 2)], True, [3, 5, 2])
    assert list(oracle.widest_path(off, tgt, w, 0)) == [INF, 3, 3]
    # SPEC.md:345  single edge 0-1 (7) -> D[1]=7
    off, tgt, w = graphgen.from_edge_list(2, [(0, 1)], True, [7])
    assert list(oracle.widest_path(off, tgt, w, 0)) == [INF, 7]
    # weighted path: width = running minimum of the prefix weights
    n = 60
    ws = np.random.default_rng(1).integers(1, 100, n - 1)
    off, tgt, w = graphgen.from_edge_list(n, path_graph(n), True, list(ws))
    assert (oracle.widest_path(off, tgt, w, 0)[1:] == np.minimum.accumulate(ws)).all()
    # tree: unique path -> minimum weight along it
    edges, par, _ = recursive_tree(200, 4)
    wt = np.random.default_rng(2).integers(1, 50, len(edges))
    off, tgt, w = graphgen.from_edge_list(200, edges, True, list(wt))
    exp = np.zeros(200, np.int64)
    exp[0] = INF
    for i, (p, c) in enumerate(edges):       # edges are in child order 1..199, parents first
        exp[c] = min(exp[p], wt[i])
    assert (oracle.widest_path(off, tgt, w, 0) == exp).all()
    # constant weight c on a connected graph: every vertex c, src INF; unreachable 0
    off, tgt = graphgen.from_edge_list(5, [(0, 1), (1, 2), (3, 4)])
    got = oracle.widest_path(off, tgt, np.full(tgt.shape, 6, np.uint32), 0)
    assert list(got) == [INF, 6, 6, 0, 0]


def test_widest_certificate_rejects_mutations():
    off, tgt = graphgen.rmat_graph(10, 1 << 13, 8, 0.57, 0.19, 0.19)
    w = graphgen.pair_weights(off, tgt, 8, 30)
    wd = oracle.widest_path(off, tgt, w, 0)
    assert oracle.check_widest(off, tgt, w, 0, wd)[0]
    reached = np.nonzero((wd > 0) & (wd != INF))[0]
    for v in reached[:: max(1, reached.size // 12)]:
        for delta in (-1, 1):
            w2 = wd.copy(); w2[v] = int(wd[v]) + delta
            assert not oracle.check_widest(off, tgt, w, 0, w2)[0]
    # an unreachable pair claiming a width between themselves
    off, tgt, ww = graphgen.from_edge_list(4, [(0, 1), (2, 3)], True, [5, 9])
    bad = np.array([INF, 5, 4, 4], np.uint32)
    assert not oracle.check_widest(off, tgt, ww, 0, bad)[0]


# ---- NEXT-3 single-source betweenness ----------------

from pins import brute_force_dependencies  # noqa: E402


@pytest.mark.parametrize("seed", range(8))
def test_bc_brute_force(seed):
    n = 8
    off, tgt = graphgen.random_graph(n, 0.3 + 0.05 * (seed % 3), 500 + seed, symmetric=seed % 2 == 0)
    for src in range(n):
        got, _ = oracle.betweenness(off, tgt, src)
        assert np.allclose(got, brute_force_dependencies(n, off, tgt, src), rtol=1e-12, atol=1e-12)


def test_bc_closed_forms_and_spec_examples():
    # SPEC.md:350 P3 src=0 -> [0, 1, 0]
    off, tgt = graphgen.from_edge_list(3, [(0, 1), (1, 2)])
    assert list(oracle.betweenness(off, tgt, 0)[0]) == [0.0, 1.0, 0.0]
    # SPEC.md:351 diamond 0-1,0-2,1-3,2-3 src=0 -> d(1)=d(2)=0.5, d(3)=0
    off, tgt = graphgen.from_edge_list(4, [(0, 1), (0, 2), (1, 3), (2, 3)])
    assert list(oracle.betweenness(off, tgt, 0)[0]) == [0.0, 0.5, 0.5, 0.0]
    # SPEC.md:352 star with centre src -> all leaves 0; leaf src -> centre n-2
    n = 9
    off, tgt = graphgen.from_edge_list(n, [(0, i) for i in range(1, n)])
    assert (oracle.betweenness(off, tgt, 0)[0] == 0).all()
    d, _ = oracle.betweenness(off, tgt, 3)
    assert d[0] == n - 2 and (np.delete(d, 0) == 0).all()
    # path from an end: delta(v) = number of vertices beyond v
    n = 40
    off, tgt = graphgen.from_edge_list(n, path_graph(n))
    d, s = oracle.betweenness(off, tgt, 0, want_sigma=True)
    assert (d[1:] == np.arange(n - 2, -1, -1)).all() and (s == 1).all()
    # complete graph: every pair adjacent, no interior vertices
    off, tgt = graphgen.from_edge_list(7, [(i, j) for i in range(7) for j in range(i + 1, 7)])
    assert (oracle.betweenness(off, tgt, 2)[0] == 0).all()
    # 2D grid from a corner: sigma = binomial path counts
    a, b = 6, 5
    off, tgt = graphgen.from_edge_list(a * b, grid_edges(a, b))
    _, s = oracle.betweenness(off, tgt, 0, want_sigma=True)
    from math import comb
    assert all(s[x + a * y] == comb(x + y, x) for y in range(b) for x in range(a))


# ---- NEXT-4 general-weight SSSP (signed weights, -inf) ------------------------------

from pins import johnson_reweight, signed_csr, signed_expected  # noqa: E402

NEGINF = np.iinfo(np.int64).min
POSINF = np.iinfo(np.int64).max


def test_signed_spec_examples():
    # S:336-337 (SPEC examples of the paper's General-Weight SSSP)
    off, tgt, w = signed_csr(3, [(0, 1), (1, 2)], [4, -2])
    for scope in (0, 1):
        d, neg = oracle.bellman_ford_signed(off, tgt, w, 0, scope)
        assert list(d) == [0, 4, 2] and not neg
    off, tgt, w = signed_csr(2, [(0, 1), (1, 0)], [1, -3])
    for scope in (0, 1):
        d, neg = oracle.bellman_ford_signed(off, tgt, w, 0, scope)
        assert list(d) == [NEGINF, NEGINF] and neg


@pytest.mark.parametrize("seed", range(12))
def test_signed_brute_force_fw(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 9))
    edges = [(int(a), int(b)) for a in range(n) for b in range(n)
             if a != b and rng.random() < 0.35]
    ws = rng.integers(-4, 9, len(edges))
    off, tgt, w = signed_csr(n, edges, ws)
    for src in range(n):
        for scope in (0, 1):
            exp, eneg = signed_expected(n, off, tgt, w, src, scope)
            got, neg = oracle.bellman_ford_signed(off, tgt, w, src, scope)
            assert neg == eneg and (got == exp).all(), (seed, src, scope, got, exp)


def test_signed_planted_cycles_scopes():
    # 0 -> 1 -> 2 -> 0 has weight -1; 2 -> 3 -> 4 downstream; 5 reaches the cycle
    # but is not reachable from it; 6 isolated
    edges = [(0, 1), (1, 2), (2, 0), (2, 3), (3, 4), (5, 0)]
    ws = [2, -4, 1, 7, -1, 3]
    off, tgt, w = signed_csr(7, edges, ws)
    d, neg = oracle.bellman_ford_signed(off, tgt, w, 0, 1)
    assert neg and list(d[:5]) == [NEGINF] * 5 and d[5] == POSINF and d[6] == POSINF
    d, neg = oracle.bellman_ford_signed(off, tgt, w, 0, 0)
    assert neg and (d == NEGINF).all()
    d, neg = oracle.bellman_ford_signed(off, tgt, w, 3, 1)   # cycle unreachable from 3
    assert not neg and list(d) == [POSINF, POSINF, POSINF, 0, -1, POSINF, POSINF]


@pytest.mark.parametrize("seed", range(3))
def test_signed_johnson_closed_form(seed):
    off, tgt = graphgen.random_graph(300, 0.02, 500 + seed, symmetric=False)
    w = graphgen.pair_weights(off, tgt, seed, 40)
    phi = np.random.default_rng(seed).integers(-1000, 1000, off.shape[0] - 1).astype(np.int64)
    w2 = johnson_reweight(off, tgt, w, phi)
    assert (w2.view(np.int32) < 0).any()
    for src in (0, 17):
        ref, _ = oracle.dijkstra64(off, tgt, w, src)
        got, neg = oracle.bellman_ford_signed(off, tgt, w2, src, 1)
        fin = ref != np.uint64(0xFFFFFFFFFFFFFFFF)
        assert not neg
        assert (got[~fin] == POSINF).all()
        assert (got[fin] == ref[fin].astype(np.int64) + phi[src] - phi[fin]).all()


def test_signed_nonnegative_equals_dijkstra_and_range():
    off, tgt = graphgen.random_graph(400, 0.01, 9, symmetric=True)
    w = graphgen.pair_weights(off, tgt, 3, 100)
    ref, _ = oracle.dijkstra64(off, tgt, w, 0)
    got, neg = oracle.bellman_ford_signed(off, tgt, w, 0)
    fin = ref != np.uint64(0xFFFFFFFFFFFFFFFF)
    assert not neg and (got[fin] == ref[fin].astype(np.int64)).all() and (got[~fin] == POSINF).all()
    d, _ = oracle.bellman_ford_signed(off, tgt, None, 0)          # NULL = unit weights
    b, _ = oracle.bfs(off, tgt, 0)
    assert (d[b != INF] == b[b != INF]).all()
    off, tgt, w = signed_csr(3, [(0, 1), (1, 2)], [-(2 ** 31), 5])
    assert oracle.bellman_ford_signed(off, tgt, w, 0)[0][2] == -(2 ** 31) + 5
