"""NEXT-2 GPU parity: gbbs_wbfs (integral-weight SSSP over distance buckets,
PAPER.md:102-109 sec:algs, output spec PAPER.md:1481-1484) through the C ABI,
against the oracle's Dijkstra, element by element (distances are unique, so the
bar is bit-exact).

Structure checked beside the values: with bucket width 1 and weights >= 1 every
bucket is extracted once, in increasing order, and every distinct finite
distance is one of the extracted buckets (a bucket whose entries all moved to
earlier buckets is still extracted, so rounds >= distinct distances, with
equality for unit or constant weights); every reached vertex is expanded exactly
once, so the edges examined equal the out-degree sum of the reached set (O(m)
work).
"""
import numpy as np
import pytest

import graphgen
import oracle
from golden_io import read_examples
from pins import torus_dist

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

INF = 0xFFFFFFFF


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1805_05208_b200 import gbbs
    return gbbs


def run_wbfs(G, g, src, delta=0, host=False, stats=None):
    d = np.empty(g.n, np.uint32) if host else torch.empty(g.n, dtype=torch.int32, device="cuda")
    opts = G.make_opts(delta=delta) if (delta or stats is not None) else None
    g.wbfs(src, d, opts=opts, stats=stats)
    return d if host else d.cpu().numpy().view(np.uint32)


def distinct_finite(d):
    return int(np.unique(d[d != INF]).size)


def test_spec_examples(G):
    for ex in read_examples():
        if ex["kind"] == "bfs":
            continue
        g = G.Graph(ex["offsets"], ex["targets"], ex["weights"], symmetric=True)
        for delta in (0, 1, 2, 5):
            assert (run_wbfs(G, g, ex["src"], delta) == ex["expected"]).all(), (ex["line"], delta)
        g.close()


def test_single_vertex_isolated_and_unreachable(G):
    off = np.zeros(2, np.int64)
    g = G.Graph(off, np.zeros(0, np.uint32), symmetric=True)
    assert list(run_wbfs(G, g, 0)) == [0]
    g.close()
    off, tgt, w = graphgen.from_edge_list(5, [(1, 2), (2, 3)], True, [4, 6])
    g = G.Graph(off, tgt, w, symmetric=True)
    assert list(run_wbfs(G, g, 0)) == [0, INF, INF, INF, INF]
    assert list(run_wbfs(G, g, 1)) == [INF, 0, 4, 10, INF]
    g.close()


@pytest.mark.parametrize("seed", range(4))
def test_random_vs_dijkstra(G, seed):
    for sym in (True, False):
        off, tgt = graphgen.random_graph(700, 0.004 * (1 + seed), 90 + seed, symmetric=sym)
        w = graphgen.pair_weights(off, tgt, seed, 30)
        g = G.Graph(off, tgt, w, symmetric=sym)
        for src in (0, 3, 699):
            ref, _ = oracle.dijkstra(off, tgt, w, src)
            for delta in (0, 1, 4, 31):
                assert (run_wbfs(G, g, src, delta) == ref).all(), (sym, src, delta)
        assert (run_wbfs(G, g, 0, host=True) == oracle.dijkstra(off, tgt, w, 0)[0]).all()
        g.close()


def test_rounds_equal_distinct_distances(G):
    """delta = 1, w >= 1: one round per distinct finite distance; each reached
    vertex expanded once (sum of non-stale swept entries = reached)."""
    cfg = graphgen.CONFIGS["c1"]
    off, tgt = graphgen.rmat_graph(cfg.levels, 1 << cfg.log_edges, cfg.graph_seed, *cfg.abc)
    w = graphgen.pair_weights(off, tgt, cfg.weight_seed, cfg.W)
    g = G.Graph(off, tgt, w, symmetric=True)
    ref, _ = oracle.dijkstra(off, tgt, w, 0)
    st = G.make_stats(1 << 14)
    d = run_wbfs(G, g, 0, delta=1, stats=st)
    assert (d == ref).all()
    recs = G.round_records(st)
    buckets = [r["bucket"] for r in recs]
    assert buckets == sorted(set(buckets))                          # increasing, once each
    assert set(np.unique(ref[ref != INF]).tolist()) <= set(buckets)
    assert st.rounds >= distinct_finite(ref)
    assert all(r["dense"] == 3 for r in recs)          # no near-list rounds
    # every vertex of bucket k has dist k: the rounds' entry counts cover the
    # reached set (stale entries come on top)
    assert sum(r["frontier"] for r in recs) >= int((ref != INF).sum())
    # edges expanded = out-degree sum of the reached vertices (each exactly once)
    deg = np.diff(off)
    assert sum(r["edges_examined"] for r in recs) == int(deg[ref != INF].sum())
    g.close()


def test_torus_constant_and_random_weights(G):
    L = 20
    off, tgt = graphgen.torus3d(L)
    for c in (1, 7):
        g = G.Graph(off, tgt, np.full(tgt.shape, c, np.uint32), symmetric=True)
        st = G.make_stats(4096)
        d = run_wbfs(G, g, 0, delta=1, stats=st)
        assert (d == c * torus_dist(L, 0)).all()
        assert st.rounds == 3 * (L // 2) + 1          # buckets 0, c, 2c, ..., c*ecc
        g.close()
    w = graphgen.pair_weights(off, tgt, 7, 24)
    g = G.Graph(off, tgt, w, symmetric=True)
    ref, _ = oracle.dijkstra(off, tgt, w, 0)
    for delta in (0, 1, 3, 8):
        assert (run_wbfs(G, g, 0, delta) == ref).all(), delta
    g.close()


def test_zero_weights_use_near_list(G):
    """w = 0 edges put vertices into the bucket being processed (near list)."""
    off, tgt = graphgen.random_graph(900, 0.006, 17, symmetric=True)
    w = graphgen.pair_weights(off, tgt, 3, 4) - 1          # weights in [0, 3]
    assert (w == 0).any()
    g = G.Graph(off, tgt, w, symmetric=True)
    for src in (0, 450):
        ref, _ = oracle.dijkstra(off, tgt, w, src)
        st = G.make_stats(1 << 14)
        for delta in (1, 2):
            assert (run_wbfs(G, g, src, delta, stats=st) == ref).all(), (src, delta)
        assert any(r["dense"] == 4 for r in G.round_records(st))
    g.close()
    # a chain of zero-weight edges: all at distance 0, in one bucket
    n = 300
    off, tgt, w = graphgen.from_edge_list(n, [(i, i + 1) for i in range(n - 1)], True, [0] * (n - 1))
    g = G.Graph(off, tgt, w, symmetric=True)
    assert (run_wbfs(G, g, 0) == 0).all()
    g.close()


def test_hubs_in_late_buckets(G):
    """Heavy vertices (out-degree > 512) reached in a middle bucket: the
    conditional heavy pass (list tiles after a grid barrier)."""
    n = 6000
    edges, ws = [], []
    for i in range(1, 40):                       # a path 0-1-...-39 of weight 3
        edges.append((i - 1, i)); ws.append(3)
    for h, hub in enumerate((20, 39)):           # two hubs of degree 1500 + 2
        for j in range(40 + 1500 * h, 40 + 1500 * (h + 1)):
            edges.append((hub, j)); ws.append(1 + j % 9)
    for j in range(3040, n):                      # the rest hangs off the hubs' leaves
        edges.append((40 + (j * 7) % 3000, j)); ws.append(1 + j % 5)
    off, tgt, w = graphgen.from_edge_list(n, edges, True, ws)
    g = G.Graph(off, tgt, w, symmetric=True)
    ref, _ = oracle.dijkstra(off, tgt, w, 0)
    for delta in (0, 1, 4):
        assert (run_wbfs(G, g, 0, delta) == ref).all(), delta
    g.close()


def test_unit_and_null_weights_equal_bfs(G):
    off, tgt = graphgen.rmat_graph(15, 1 << 19, 3, 0.57, 0.19, 0.19)
    ref, _ = oracle.bfs(off, tgt, 0)
    for w in (None, np.ones(tgt.shape, np.uint32)):
        g = G.Graph(off, tgt, w, symmetric=True)
        st = G.make_stats(1024)
        assert (run_wbfs(G, g, 0, stats=st) == ref).all()
        assert st.rounds == distinct_finite(ref)          # = ecc + 1 BFS levels
        g.close()


def test_directed_rmat(G):
    off, tgt = graphgen.rmat_graph(15, 1 << 19, 9, 0.6, 0.15, 0.15, symmetric=False)
    w = graphgen.pair_weights(off, tgt, 4, 15)
    g = G.Graph(off, tgt, w, symmetric=False)
    cand = np.nonzero(np.diff(off) > 0)[0]
    for src in graphgen.choose_sources(cand, 3, 5):
        ref, _ = oracle.dijkstra(off, tgt, w, src)
        assert (run_wbfs(G, g, src) == ref).all()
        assert oracle.check_sssp(off, tgt, w, src, ref)[0]
    g.close()


def test_matches_bellman_ford_and_deterministic(G):
    off, tgt = graphgen.rmat_graph(16, 1 << 20, 5, 0.57, 0.19, 0.19)
    w = graphgen.pair_weights(off, tgt, 5, 16)
    g = G.Graph(off, tgt, w, symmetric=True)
    bf = torch.empty(g.n, dtype=torch.int32, device="cuda")
    g.bellman_ford(0, bf)
    bf = bf.cpu().numpy().view(np.uint32)
    for _ in range(4):
        assert (run_wbfs(G, g, 0) == bf).all()
    g.close()


def test_errors(G):
    off, tgt = graphgen.from_edge_list(4, [(0, 1), (1, 2)])
    w = np.array([1000] * tgt.shape[0], np.uint32)
    g = G.Graph(off, tgt, w, symmetric=True)
    d = np.full(4, 77, np.uint32)
    with pytest.raises(G.GbbsError) as e:
        g.wbfs(0, d, opts=G.make_opts(delta=1))    # span 1000 buckets > 64 lists
    assert e.value.code == -1
    assert list(run_wbfs(G, g, 0, host=True)) == [0, 1000, 2000, INF]  # default delta = 32
    with pytest.raises(G.GbbsError):
        g.wbfs(4, d)
    g.close()
    big = np.full(tgt.shape, 0xF0000000, np.uint32)
    g = G.Graph(off, tgt, big, symmetric=True)
    with pytest.raises(G.GbbsError) as e:
        g.wbfs(0, d)
    assert e.value.code == -2
    g.close()


@pytest.mark.parametrize("teams", [1, 2, 3, 5])
def test_wbfs_batch_teams(G, teams):
    """gbbs_wbfs_batch: teams of wBFS traversals per launch, each with its own bucket
    ring; rows equal the oracle's Dijkstra (also with delta = 4, i.e. near lists)."""
    off, tgt = graphgen.rmat_graph(16, 1 << 20, 44, 0.57, 0.19, 0.19)
    w = graphgen.pair_weights(off, tgt, 3, 16)
    g = G.Graph(off, tgt, w, symmetric=True)
    srcs = graphgen.choose_sources(np.nonzero(np.diff(off) > 0)[0], 7, 17)
    refs = [oracle.dijkstra(off, tgt, w, s)[0] for s in srcs]
    for delta in (0, 4):
        d = torch.empty((len(srcs), g.n), dtype=torch.int32, device="cuda")
        g.wbfs_batch(srcs, d, opts=G.make_opts(teams=teams, delta=delta))
        d = d.cpu().numpy().view(np.uint32)
        for i in range(len(srcs)):
            assert (d[i] == refs[i]).all(), (teams, delta, i)
    with pytest.raises(G.GbbsError):
        g.wbfs_batch(srcs, np.empty((len(srcs), g.n), np.uint32))   # host rows
    g.close()
