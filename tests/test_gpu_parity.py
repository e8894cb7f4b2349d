"""GPU parity: libgbbs (through its C ABI) vs the CPU oracle, element by element.

Bar: distances bit-exact; every BFS parent certified (a
valid in-neighbour one level closer, reading A15); forced-sparse, forced-dense,
auto and T in {10,20,40} give identical distances.
"""
import numpy as np
import pytest

import graphgen
import oracle
from golden_io import read_examples
from pins import grid_edges, path_graph, recursive_tree, torus_dist, torus_level_counts

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

INF = 0xFFFFFFFF
MODES = ("auto", "sparse", "dense")


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1805_05208_b200 import gbbs
    return gbbs


def _opts(G, mode, T=20):
    return G.make_opts(threshold_den=T, mode={"auto": G.GBBS_MODE_AUTO, "sparse": G.GBBS_MODE_SPARSE,
                                                "dense": G.GBBS_MODE_DENSE}[mode])


def run_bfs(G, g, src, mode="auto", T=20, host=False, stats=None):
    n = g.n
    if host:
        d = np.empty(n, np.uint32); p = np.empty(n, np.uint32)
    else:
        d = torch.empty(n, dtype=torch.int32, device="cuda"); p = torch.empty_like(d)
    g.bfs(src, d, p, opts=_opts(G, mode, T), stats=stats)
    if not host:
        torch.cuda.synchronize()
        d = d.cpu().numpy().view(np.uint32); p = p.cpu().numpy().view(np.uint32)
    return d, p


def run_bf(G, g, src, host=False, stats=None):
    if host:
        d = np.empty(g.n, np.uint32)
    else:
        d = torch.empty(g.n, dtype=torch.int32, device="cuda")
    g.bellman_ford(src, d, stats=stats)
    if not host:
        d = d.cpu().numpy().view(np.uint32)
    return d


def check_bfs_all_modes(G, off, tgt, srcs, symmetric, host_variants=True):
    g = G.Graph(off, tgt, symmetric=symmetric)
    for src in srcs:
        ref, _ = oracle.bfs(off, tgt, src)
        for mode in MODES:
            d, p = run_bfs(G, g, src, mode)
            assert (d == ref).all(), (mode, src, np.nonzero(d != ref)[0][:5])
            ok, bad = oracle.check_bfs(off, tgt, src, d, p)
            assert ok, (mode, src, bad)
        if host_variants:
            d, p = run_bfs(G, g, src, "auto", host=True)
            assert (d == ref).all()
            assert oracle.check_bfs(off, tgt, src, d, p)[0]
    g.close()


def check_bf(G, off, tgt, w, srcs, symmetric):
    g = G.Graph(off, tgt, w, symmetric=symmetric)
    for src in srcs:
        ref, _ = oracle.dijkstra(off, tgt, w, src)
        d = run_bf(G, g, src)
        assert (d == ref).all(), (src, np.nonzero(d != ref)[0][:5])
        d = run_bf(G, g, src, host=True)
        assert (d == ref).all()
    g.close()


# ---- small and closed-form graphs ---------------------------------------------------

def test_spec_examples(G):
    for ex in read_examples():
        if ex["kind"] == "bfs":
            g = G.Graph(ex["offsets"], ex["targets"], symmetric=True)
            for mode in MODES:
                d, _ = run_bfs(G, g, ex["src"], mode)
                assert (d == ex["expected"]).all(), ex["line"]
        else:
            g = G.Graph(ex["offsets"], ex["targets"], ex["weights"], symmetric=True)
            assert (run_bf(G, g, ex["src"]) == ex["expected"]).all(), ex["line"]
        g.close()


def test_single_vertex_and_isolated_source(G):
    off = np.zeros(2, np.int64); tgt = np.zeros(0, np.uint32)
    g = G.Graph(off, tgt, symmetric=True)
    d, p = run_bfs(G, g, 0)
    assert list(d) == [0] and list(p) == [0]
    assert list(run_bf(G, g, 0)) == [0]
    g.close()
    off, tgt = graphgen.from_edge_list(5, [(1, 2), (2, 3)])
    g = G.Graph(off, tgt, symmetric=True)
    d, p = run_bfs(G, g, 0)
    assert list(d) == [0, INF, INF, INF, INF] and list(p) == [0, INF, INF, INF, INF]
    g.close()


@pytest.mark.parametrize("n", [2, 33, 1000, 5000])
def test_path_closed_form(G, n):
    off, tgt = graphgen.from_edge_list(n, path_graph(n))
    g = G.Graph(off, tgt, symmetric=True)
    for src in (0, n // 2, n - 1):
        for mode in MODES:
            d, p = run_bfs(G, g, src, mode)
            assert (d == np.abs(np.arange(n) - src)).all()
            exp_p = np.array([src if v == src else (v + 1 if v < src else v - 1) for v in range(n)])
            assert (p == exp_p).all()
    g.close()


def test_grid_and_trees(G):
    a, b = 37, 29
    off, tgt = graphgen.from_edge_list(a * b, grid_edges(a, b))
    check_bfs_all_modes(G, off, tgt, [0, 500, a * b - 1], True)
    for seed in (1, 2):
        edges, par, depth = recursive_tree(3000, seed)
        off, tgt = graphgen.from_edge_list(3000, edges)
        g = G.Graph(off, tgt, symmetric=True)
        for mode in MODES:
            d, p = run_bfs(G, g, 0, mode)
            assert (d == depth).all() and (p[1:] == par[1:]).all()
        g.close()


@pytest.mark.parametrize("L", [3, 7, 16, 33])
def test_torus_closed_form_and_levels(G, L):
    off, tgt = graphgen.torus3d(L)
    g = G.Graph(off, tgt, symmetric=True)
    for mode in MODES:
        st = G.make_stats(4096)
        d, p = run_bfs(G, g, 0, mode, stats=st)
        assert (d == torus_dist(L, 0)).all()
        assert oracle.check_bfs(off, tgt, 0, d, p)[0]
        recs = G.round_records(st)
        lv = torus_level_counts(L)
        assert st.rounds == len(lv)                       # ecc + 1 edgeMap rounds
        assert [r["frontier"] for r in recs] == list(lv)  # frontier r = level-r count
        assert st.reached == L ** 3
    c = 5
    w = np.full(tgt.shape, c, np.uint32)
    g2 = G.Graph(off, tgt, w, symmetric=True)
    assert (run_bf(G, g2, 0) == c * torus_dist(L, 0)).all()
    g.close(); g2.close()


def test_complete_graph_exact_parent(G):
    n = 300
    off, tgt = graphgen.from_edge_list(n, [(i, j) for i in range(n) for j in range(i + 1, n)])
    g = G.Graph(off, tgt, symmetric=True)
    for mode in MODES:
        d, p = run_bfs(G, g, 7, mode)
        assert (d == np.where(np.arange(n) == 7, 0, 1)).all() and (p == 7).all()
    g.close()


@pytest.mark.parametrize("seed", range(4))
def test_random_symmetric_and_directed(G, seed):
    for sym in (True, False):
        off, tgt = graphgen.random_graph(700, 0.004 * (1 + seed), seed, symmetric=sym)
        check_bfs_all_modes(G, off, tgt, [0, 1, 699], sym, host_variants=(seed == 0))
        w = graphgen.pair_weights(off, tgt, seed, 50)
        check_bf(G, off, tgt, w, [0, 3], sym)


def test_directed_rmat_threshold_sweep(G):
    off, tgt = graphgen.rmat_graph(16, 1 << 20, 9, 0.6, 0.15, 0.15, symmetric=False)
    g = G.Graph(off, tgt, symmetric=False)
    cand = np.nonzero(np.diff(off) > 0)[0]
    for src in graphgen.choose_sources(cand, 3, 55):
        ref, _ = oracle.bfs(off, tgt, src)
        for mode in MODES:
            for T in (10, 20, 40):
                d, p = run_bfs(G, g, src, mode, T)
                assert (d == ref).all()
                assert oracle.check_bfs(off, tgt, src, d, p)[0]
    g.close()


@pytest.mark.parametrize("sym", [False, True])
def test_long_in_lists_dense(G, sym):
    """A vertex whose in-list is long and whose only frontier in-neighbour comes
    last (and one with none at all) — exercises the warp-cooperative pull scan."""
    n = 5000
    edges = [(0, 1), (1, n - 1), (1, n - 2)]
    edges += [(u, n - 1) for u in range(2, n - 3)]   # unreachable in-neighbours first
    edges += [(u, n - 3) for u in range(2, 40)]      # never reached
    edges += [(u, n - 2) for u in range(2, 30)]
    off, tgt = graphgen.from_edge_list(n, edges, symmetric=sym)
    g = G.Graph(off, tgt, symmetric=sym)
    ref, _ = oracle.bfs(off, tgt, 0)
    for mode in MODES:
        d, p = run_bfs(G, g, 0, mode)
        assert (d == ref).all(), mode
        assert oracle.check_bfs(off, tgt, 0, d, p)[0]
    g.close()


def test_unit_weights_and_null_weights_equal_bfs(G):
    off, tgt = graphgen.rmat_graph(15, 1 << 19, 3, 0.57, 0.19, 0.19)
    g = G.Graph(off, tgt, symmetric=True)
    g1 = G.Graph(off, tgt, np.ones(tgt.shape, np.uint32), symmetric=True)
    ref, _ = oracle.bfs(off, tgt, 0)
    assert (run_bf(G, g, 0) == ref).all()
    assert (run_bf(G, g1, 0) == ref).all()
    g.close(); g1.close()


def test_borrow_and_device_inputs(G):
    off, tgt = graphgen.rmat_graph(14, 1 << 17, 21, 0.57, 0.19, 0.19)
    w = graphgen.pair_weights(off, tgt, 2, 14)
    doff = torch.from_numpy(off).cuda()
    dtgt = torch.from_numpy(tgt.view(np.int32)).cuda()
    dw = torch.from_numpy(w.view(np.int32)).cuda()
    ref, _ = oracle.bfs(off, tgt, 0)
    refw, _ = oracle.dijkstra(off, tgt, w, 0)
    for borrow in (False, True):
        g = G.Graph(doff, dtgt, dw, symmetric=True, borrow=borrow)
        d, p = run_bfs(G, g, 0)
        assert (d == ref).all()
        assert (run_bf(G, g, 0) == refw).all()
        g.close()


def test_repeated_calls_are_deterministic(G):
    off, tgt = graphgen.rmat_graph(16, 1 << 20, 5, 0.57, 0.19, 0.19)
    w = graphgen.pair_weights(off, tgt, 5, 16)
    g = G.Graph(off, tgt, w, symmetric=True)
    d0, _ = run_bfs(G, g, 0)
    b0 = run_bf(G, g, 0)
    for _ in range(5):
        assert (run_bfs(G, g, 0)[0] == d0).all()
        assert (run_bf(G, g, 0) == b0).all()
    g.close()


# ---- error conventions ---------------------------------------------------------------

def test_error_conventions(G):
    off, tgt = graphgen.from_edge_list(4, [(0, 1), (1, 2)])
    g = G.Graph(off, tgt, symmetric=True)
    d = np.full(4, 77, np.uint32)
    with pytest.raises(G.GbbsError) as e:
        g.bfs(4, d)
    assert e.value.code == -1 and (d == 77).all()
    with pytest.raises(G.GbbsError):
        g.bellman_ford(9, d)
    with pytest.raises(G.GbbsError):
        g.bfs(0, None)
    g.close()
    bad = off.copy(); bad[2] = 0
    with pytest.raises(G.GbbsError) as e:
        G.Graph(bad, tgt)
    assert e.value.code == -1
    badt = tgt.copy(); badt[0] = 4
    with pytest.raises(G.GbbsError):
        G.Graph(off, badt)
    with pytest.raises(G.GbbsError):
        G.gbbs_graph_create(4, tgt.shape[0] + 1, off, tgt)
    with pytest.raises(G.GbbsError) as e:
        G.Graph(off, tgt, borrow=True)          # host arrays cannot be borrowed
    assert e.value.code == -1
    # weights whose max * (n-1) overflows uint32 distances
    big = np.full(tgt.shape, 0xF0000000, np.uint32)
    g = G.Graph(off, tgt, big, symmetric=True)
    with pytest.raises(G.GbbsError) as e:
        g.bellman_ford(0, d)
    assert e.value.code == -2
    g.bfs(0, d)      # BFS ignores weights
    g.close()


# ---- the BASELINE configs ------------------------------------------------------------

def test_c1_generator_bit_identical_and_parity(G):
    from graphgen import device
    cfg = graphgen.CONFIGS["c1"]
    off, tgt = graphgen.rmat_graph(cfg.levels, 1 << cfg.log_edges, cfg.graph_seed, *cfg.abc)
    w = graphgen.pair_weights(off, tgt, cfg.weight_seed, cfg.W)
    dg = device.build_config("c1")
    assert (dg["offsets"].cpu().numpy() == off).all()
    assert (dg["targets"].cpu().numpy().view(np.uint32) == tgt).all()
    assert (dg["weights"].cpu().numpy().view(np.uint32) == w).all()
    check_bfs_all_modes(G, off, tgt, [0], True)
    check_bf(G, off, tgt, w, [0], True)
    L = 9
    toff, ttgt = graphgen.torus3d(L)
    o2, t2 = device.torus_csr(L)
    assert (o2.cpu().numpy() == toff).all() and (t2.cpu().numpy().view(np.uint32) == ttgt).all()


# ---- NEXT-1 widest path -------------------------------------------------------------

def run_wp(G, g, src, host=False, mode=None):
    d = np.empty(g.n, np.uint32) if host else torch.empty(g.n, dtype=torch.int32, device="cuda")
    opts = None if mode is None else G.make_opts(20, {"auto": 0, "sparse": 1, "dense": 2}[mode])
    g.widest_path(src, d, opts=opts)
    return d if host else d.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("seed", range(4))
def test_widest_random(G, seed):
    for sym in (True, False):
        off, tgt = graphgen.random_graph(600, 0.005 * (1 + seed), 40 + seed, symmetric=sym)
        w = graphgen.pair_weights(off, tgt, seed, 1000)
        g = G.Graph(off, tgt, w, symmetric=sym)
        for src in (0, 5, 599):
            ref = oracle.widest_path(off, tgt, w, src)
            for mode in ("auto", "dense"):
                assert (run_wp(G, g, src, mode=mode) == ref).all(), (sym, src, mode)
        assert (run_wp(G, g, 0, host=True) == oracle.widest_path(off, tgt, w, 0)).all()
        g.close()


def test_widest_spec_examples_and_unit(G):
    off, tgt, w = graphgen.from_edge_list(3, [(0, 1), (1, 2), (0, 2)], True, [3, 5, 2])
    g = G.Graph(off, tgt, w, symmetric=True)
    assert list(run_wp(G, g, 0)) == [0xFFFFFFFF, 3, 3]
    g.close()
    off, tgt = graphgen.rmat_graph(14, 1 << 17, 2, 0.57, 0.19, 0.19)
    g = G.Graph(off, tgt, symmetric=True)            # NULL weights = unit: reached -> 1
    d = run_wp(G, g, 0)
    bfs, _ = oracle.bfs(off, tgt, 0)
    assert ((d == 1) == ((bfs != 0xFFFFFFFF) & (bfs > 0))).all() and d[0] == 0xFFFFFFFF
    g.close()


def test_widest_c1_and_torus(G):
    cfg = graphgen.CONFIGS["c1"]
    off, tgt = graphgen.rmat_graph(cfg.levels, 1 << cfg.log_edges, cfg.graph_seed, *cfg.abc)
    w = graphgen.pair_weights(off, tgt, cfg.weight_seed, 1 << 20)
    g = G.Graph(off, tgt, w, symmetric=True)
    assert (run_wp(G, g, 0) == oracle.widest_path(off, tgt, w, 0)).all()
    g.close()
    off, tgt = graphgen.torus3d(20)
    w = graphgen.pair_weights(off, tgt, 7, 24)
    g = G.Graph(off, tgt, w, symmetric=True)
    d = run_wp(G, g, 0)
    assert (d == oracle.widest_path(off, tgt, w, 0)).all()
    assert oracle.check_widest(off, tgt, w, 0, d)[0]
    g.close()


# ---- NEXT-3 single-source betweenness -----------------------------------------------

def run_bc(G, g, src, host=False, mode=None):
    opts = None if mode is None else G.make_opts(mode=mode)
    if host:
        d = np.empty(g.n, np.float64)
        g.betweenness(src, d, opts=opts)
        return d
    d = torch.empty(g.n, dtype=torch.float64, device="cuda")
    g.betweenness(src, d, opts=opts)
    return d.cpu().numpy()


def assert_bc_close(got, ref):
    # fp64 sums of positive terms in a nondeterministic order (DESIGN.md tolerance)
    assert np.allclose(got, ref, rtol=1e-9, atol=1e-9 * max(1.0, float(np.abs(ref).max())))


def test_bc_spec_examples_and_closed_forms(G):
    off, tgt = graphgen.from_edge_list(3, [(0, 1), (1, 2)])
    g = G.Graph(off, tgt, symmetric=True)
    assert list(run_bc(G, g, 0)) == [0.0, 1.0, 0.0]
    g.close()
    off, tgt = graphgen.from_edge_list(4, [(0, 1), (0, 2), (1, 3), (2, 3)])
    g = G.Graph(off, tgt, symmetric=True)
    assert list(run_bc(G, g, 0)) == [0.0, 0.5, 0.5, 0.0]
    g.close()
    n = 3000
    off, tgt = graphgen.from_edge_list(n, path_graph(n))
    g = G.Graph(off, tgt, symmetric=True)
    d = run_bc(G, g, 0)
    assert (d[1:] == np.arange(n - 2, -1, -1)).all()
    g.close()
    off, tgt = graphgen.from_edge_list(500, [(0, i) for i in range(1, 500)])
    g = G.Graph(off, tgt, symmetric=True)
    assert (run_bc(G, g, 0) == 0).all()
    d = run_bc(G, g, 7, host=True)
    assert d[0] == 498 and (np.delete(d, 0) == 0).all()
    g.close()


@pytest.mark.parametrize("seed", range(3))
def test_bc_random_and_rmat(G, seed):
    off, tgt = graphgen.random_graph(800, 0.004 * (1 + seed), 70 + seed, symmetric=True)
    g = G.Graph(off, tgt, symmetric=True)
    for src in (0, 11, 799):
        assert_bc_close(run_bc(G, g, src), oracle.betweenness(off, tgt, src)[0])
    g.close()
    off, tgt = graphgen.rmat_graph(15, 1 << 19, 80 + seed, 0.57, 0.19, 0.19)
    g = G.Graph(off, tgt, symmetric=True)
    assert_bc_close(run_bc(G, g, 0), oracle.betweenness(off, tgt, 0)[0])
    g.close()


@pytest.mark.parametrize("mode", ["sparse", "dense", "auto"])
def test_bc_forward_directions(G, mode):
    """Reading B3: forward levels pushed (CAS + fp64 FA), pulled (owner-computes sum
    over level-l neighbours, symmetric graphs), or chosen per level; every form
    gives Brandes' dependencies.  The star from a leaf pulls its 499-edge hub with
    the whole warp at level 0; a directed graph ignores DENSE (push only)."""
    md = {"sparse": G.GBBS_MODE_SPARSE, "dense": G.GBBS_MODE_DENSE, "auto": G.GBBS_MODE_AUTO}[mode]
    cases = [graphgen.random_graph(900, 0.006, 91, symmetric=True),
             graphgen.rmat_graph(14, 1 << 18, 92, 0.57, 0.19, 0.19),
             graphgen.torus3d(10),
             graphgen.from_edge_list(500, [(0, i) for i in range(1, 500)]),
             graphgen.from_edge_list(2000, path_graph(2000))]
    for off, tgt in cases:
        g = G.Graph(off, tgt, symmetric=True)
        for src in (0, 7, len(off) - 2):
            assert_bc_close(run_bc(G, g, src, mode=md), oracle.betweenness(off, tgt, src)[0])
        g.close()
    off, tgt = graphgen.random_graph(700, 0.01, 93, symmetric=False)
    g = G.Graph(off, tgt, symmetric=False)
    for src in (0, 5):
        assert_bc_close(run_bc(G, g, src, mode=md), oracle.betweenness(off, tgt, src)[0])
    g.close()


def test_bc_torus_and_grid(G):
    off, tgt = graphgen.torus3d(12)
    g = G.Graph(off, tgt, symmetric=True)
    assert_bc_close(run_bc(G, g, 0), oracle.betweenness(off, tgt, 0)[0])
    g.close()
    off, tgt = graphgen.from_edge_list(40 * 30, grid_edges(40, 30))
    g = G.Graph(off, tgt, symmetric=True)
    assert_bc_close(run_bc(G, g, 0), oracle.betweenness(off, tgt, 0)[0])
    g.close()


# ---- batch API (k traversals, copies overlapped) ------------------------------------

def test_batch_matches_single_calls(G):
    off, tgt = graphgen.rmat_graph(15, 1 << 19, 12, 0.57, 0.19, 0.19)
    w = graphgen.pair_weights(off, tgt, 6, 15)
    g = G.Graph(off, tgt, w, symmetric=True)
    n = g.n
    srcs = graphgen.choose_sources(np.nonzero(np.diff(off) > 0)[0], 5, 77)
    refs = [oracle.bfs(off, tgt, s)[0] for s in srcs]
    wrefs = [oracle.dijkstra(off, tgt, w, s)[0] for s in srcs]
    # host (pinned) outputs: the overlapped path
    hd = torch.empty((len(srcs), n), dtype=torch.int32, pin_memory=True)
    hp = torch.empty_like(hd).pin_memory()
    g.bfs_batch(srcs, hd.numpy(), hp.numpy())
    for i, s in enumerate(srcs):
        d, p = hd[i].numpy().view(np.uint32), hp[i].numpy().view(np.uint32)
        assert (d == refs[i]).all() and oracle.check_bfs(off, tgt, s, d, p)[0]
    # pageable host and device outputs, parent omitted
    d2 = np.empty((len(srcs), n), np.uint32)
    g.bfs_batch(srcs, d2)
    assert all((d2[i] == refs[i]).all() for i in range(len(srcs)))
    dd = torch.empty((len(srcs), n), dtype=torch.int32, device="cuda")
    g.bfs_batch(srcs, dd)
    dd = dd.cpu().numpy().view(np.uint32)
    assert all((dd[i] == refs[i]).all() for i in range(len(srcs)))
    bw = np.empty((len(srcs), n), np.uint32)
    g.bellman_ford_batch(srcs, bw)
    assert all((bw[i] == wrefs[i]).all() for i in range(len(srcs)))
    for T in (10, 40):                                # options: threshold T, forced modes
        for mode in (G.GBBS_MODE_SPARSE, G.GBBS_MODE_DENSE):
            dd = torch.empty((len(srcs), n), dtype=torch.int32, device="cuda")
            pp = torch.empty_like(dd)
            g.bfs_batch(srcs, dd, pp, opts=G.make_opts(T, mode))
            dd, pp = dd.cpu().numpy().view(np.uint32), pp.cpu().numpy().view(np.uint32)
            for i, s in enumerate(srcs):
                assert (dd[i] == refs[i]).all() and oracle.check_bfs(off, tgt, s, dd[i], pp[i])[0]
    with pytest.raises(G.GbbsError):
        g.bfs_batch(srcs, d2, opts=G.make_opts(20, G.GBBS_MODE_PULL))
    g.bfs_batch([], np.empty((0, n), np.uint32))      # k = 0
    with pytest.raises(G.GbbsError) as e:
        g.bfs_batch([0, n], d2[:2])
    assert e.value.code == -1
    g.close()


# ---- a9 alternative: pull-min dense rounds for Bellman-Ford / widest path ----------

@pytest.mark.parametrize("T", [20, 1000])
def test_pull_min_bf_and_widest(G, T):
    """GBBS_MODE_PULL: a dense BF round is a pull-min (owner-computes, no atomics);
    distances and widths identical to the oracle; directed graphs fall back to
    the bitmap-forward push.  T = 1000 makes almost every round dense."""
    cfg = graphgen.CONFIGS["c1"]
    off, tgt = graphgen.rmat_graph(cfg.levels, 1 << cfg.log_edges, cfg.graph_seed, *cfg.abc)
    w = graphgen.pair_weights(off, tgt, cfg.weight_seed, cfg.W)
    cases = [(off, tgt, w, True)]
    toff, ttgt = graphgen.torus3d(20)
    cases.append((toff, ttgt, graphgen.pair_weights(toff, ttgt, 7, 24), True))
    roff, rtgt = graphgen.random_graph(700, 0.01, 3, symmetric=True)
    cases.append((roff, rtgt, graphgen.pair_weights(roff, rtgt, 3, 50), True))
    doff, dtgt = graphgen.random_graph(700, 0.01, 4, symmetric=False)
    cases.append((doff, dtgt, graphgen.pair_weights(doff, dtgt, 4, 50), False))
    for o, t, ww, sym in cases:
        g = G.Graph(o, t, ww, symmetric=sym)
        opts = G.make_opts(T, G.GBBS_MODE_PULL)
        for src in (0, 5):
            d = torch.empty(g.n, dtype=torch.int32, device="cuda")
            st = G.make_stats(4096)
            g.bellman_ford(src, d, opts=opts, stats=st)
            assert (d.cpu().numpy().view(np.uint32) == oracle.dijkstra(o, t, ww, src)[0]).all()
            if sym and T == 1000:
                assert any(r["dense"] == 3 for r in G.round_records(st))
            g.widest_path(src, d, opts=opts)
            assert (d.cpu().numpy().view(np.uint32) == oracle.widest_path(o, t, ww, src)).all()
        g.close()


def test_bf_dense_bitmap_forward_default_kernel(G):
    """GBBS_MODE_DENSE on the default Bellman-Ford / widest-path kernel (the
    bitmap-forward push of reading A11, a9: the frontier is the TS bitmap, swept
    by warps) on symmetric rMATs and a directed graph: every round is a bitmap
    round and distances / widths equal the oracle's."""
    cfg = graphgen.CONFIGS["c1"]
    off, tgt = graphgen.rmat_graph(cfg.levels, 1 << cfg.log_edges, cfg.graph_seed, *cfg.abc)
    cases = [(off, tgt, graphgen.pair_weights(off, tgt, cfg.weight_seed, cfg.W), True)]
    roff, rtgt = graphgen.rmat_graph(16, 1 << 20, 5, 0.57, 0.19, 0.19)
    cases.append((roff, rtgt, graphgen.pair_weights(roff, rtgt, 9, 16), True))
    doff, dtgt = graphgen.rmat_graph(14, 1 << 18, 8, 0.6, 0.15, 0.15, symmetric=False)
    cases.append((doff, dtgt, graphgen.pair_weights(doff, dtgt, 4, 14), False))
    for o, t, ww, sym in cases:
        g = G.Graph(o, t, ww, symmetric=sym)
        opts = G.make_opts(20, G.GBBS_MODE_DENSE)
        srcs = [0] + list(graphgen.choose_sources(np.nonzero(np.diff(o) > 0)[0], 2, 31))
        for src in srcs:
            d = torch.empty(g.n, dtype=torch.int32, device="cuda")
            st = G.make_stats(4096)
            g.bellman_ford(src, d, opts=opts, stats=st)
            assert (d.cpu().numpy().view(np.uint32) == oracle.dijkstra(o, t, ww, src)[0]).all(), src
            recs = G.round_records(st)
            assert recs and all(r["dense"] == 2 for r in recs)
            g.widest_path(src, d, opts=opts)
            assert (d.cpu().numpy().view(np.uint32) == oracle.widest_path(o, t, ww, src)).all(), src
        g.close()


def test_block_size_option(G):
    """gbbs_opts.bsize (edgeMapBlocked's block size): every fixed tile size gives the
    same distances as the adaptive default; invalid sizes are rejected."""
    off, tgt = graphgen.rmat_graph(15, 1 << 19, 21, 0.57, 0.19, 0.19)
    w = graphgen.pair_weights(off, tgt, 2, 15)
    g = G.Graph(off, tgt, w, symmetric=True)
    ref, _ = oracle.bfs(off, tgt, 0)
    wref, _ = oracle.dijkstra(off, tgt, w, 0)
    d = torch.empty(g.n, dtype=torch.int32, device="cuda")
    p = torch.empty_like(d)
    for bs in (32, 64, 128, 256):
        for mode in (G.GBBS_MODE_AUTO, G.GBBS_MODE_SPARSE):
            g.bfs(0, d, p, opts=G.make_opts(20, mode, bsize=bs))
            dd, pp = d.cpu().numpy().view(np.uint32), p.cpu().numpy().view(np.uint32)
            assert (dd == ref).all() and oracle.check_bfs(off, tgt, 0, dd, pp)[0], (bs, mode)
        g.bellman_ford(0, d, opts=G.make_opts(bsize=bs))
        assert (d.cpu().numpy().view(np.uint32) == wref).all(), bs
        g.wbfs(0, d, opts=G.make_opts(bsize=bs))
        assert (d.cpu().numpy().view(np.uint32) == wref).all(), bs
    for bad in (16, 48, 512):
        with pytest.raises(G.GbbsError) as e:
            g.bfs(0, d, p, opts=G.make_opts(bsize=bad))
        assert e.value.code == -1
    g.close()


@pytest.mark.parametrize("teams", [2, 3, 4])
def test_batch_teams(G, teams):
    """gbbs_opts.teams: G traversals per cooperative launch (interleaved CTA teams,
    each with its own scratch and barrier) give the same rows as single calls,
    including a batch size that is not a multiple of G and every direction mode."""
    off, tgt = graphgen.rmat_graph(16, 1 << 20, 33, 0.57, 0.19, 0.19)
    w = graphgen.pair_weights(off, tgt, 9, 16)
    g = G.Graph(off, tgt, w, symmetric=True)
    n = g.n
    srcs = graphgen.choose_sources(np.nonzero(np.diff(off) > 0)[0], 7, 91)
    refs = [oracle.bfs(off, tgt, s)[0] for s in srcs]
    wrefs = [oracle.dijkstra(off, tgt, w, s)[0] for s in srcs]
    for mode in (G.GBBS_MODE_AUTO, G.GBBS_MODE_SPARSE, G.GBBS_MODE_DENSE):
        dd = torch.empty((len(srcs), n), dtype=torch.int32, device="cuda")
        pp = torch.empty_like(dd)
        g.bfs_batch(srcs, dd, pp, opts=G.make_opts(20, mode, teams=teams))
        dd, pp = dd.cpu().numpy().view(np.uint32), pp.cpu().numpy().view(np.uint32)
        for i, s in enumerate(srcs):
            assert (dd[i] == refs[i]).all(), (mode, i)
            assert oracle.check_bfs(off, tgt, s, dd[i], pp[i])[0], (mode, i)
    bw = torch.empty((len(srcs), n), dtype=torch.int32, device="cuda")
    g.bellman_ford_batch(srcs, bw, opts=G.make_opts(teams=teams))
    bw = bw.cpu().numpy().view(np.uint32)
    assert all((bw[i] == wrefs[i]).all() for i in range(len(srcs)))
    g.close()
    # directed graph (CSC pulls) with teams
    doff, dtgt = graphgen.rmat_graph(15, 1 << 19, 35, 0.6, 0.15, 0.15, symmetric=False)
    g = G.Graph(doff, dtgt, symmetric=False)
    ds = graphgen.choose_sources(np.nonzero(np.diff(doff) > 0)[0], 5, 92)
    dd = torch.empty((len(ds), g.n), dtype=torch.int32, device="cuda")
    pp = torch.empty_like(dd)
    g.bfs_batch(ds, dd, pp, opts=G.make_opts(teams=teams))
    dd, pp = dd.cpu().numpy().view(np.uint32), pp.cpu().numpy().view(np.uint32)
    for i, s in enumerate(ds):
        assert (dd[i] == oracle.bfs(doff, dtgt, s)[0]).all()
        assert oracle.check_bfs(doff, dtgt, s, dd[i], pp[i])[0]
    g.close()


@pytest.mark.parametrize("teams", [1, 3, 8])
def test_betweenness_batch_teams(G, teams):
    """gbbs_betweenness_batch: teams of Brandes traversals per launch; every row
    matches the oracle within the fp64 tolerance (reading B2)."""
    off, tgt = graphgen.rmat_graph(15, 1 << 19, 55, 0.57, 0.19, 0.19)
    g = G.Graph(off, tgt, symmetric=True)
    srcs = graphgen.choose_sources(np.nonzero(np.diff(off) > 0)[0], 5, 23)
    d = torch.empty((len(srcs), g.n), dtype=torch.float64, device="cuda")
    g.betweenness_batch(srcs, d, opts=G.make_opts(teams=teams))
    d = d.cpu().numpy()
    for i, s in enumerate(srcs):
        assert_bc_close(d[i], oracle.betweenness(off, tgt, s)[0])
    with pytest.raises(G.GbbsError):
        g.betweenness_batch(srcs, np.empty((len(srcs), g.n), np.float64))
    g.close()


def test_no_device_memory_leak_across_handles(G):
    """Handles that used every scratch kind (teams, wBFS rings, betweenness, signed
    BF staging, host-output batches) free it all on destroy: device memory in use
    returns to its level after repeated create / run / destroy cycles."""
    off, tgt = graphgen.rmat_graph(14, 1 << 17, 61, 0.57, 0.19, 0.19)
    w = graphgen.pair_weights(off, tgt, 1, 14)
    srcs = [0, 1, 2, 3, 4]

    def cycle():
        g = G.Graph(off, tgt, w, symmetric=True)
        n = g.n
        d = torch.empty((len(srcs), n), dtype=torch.int32, device="cuda")
        g.bfs_batch(srcs, d, torch.empty_like(d), opts=G.make_opts(teams=5))
        g.bellman_ford_batch(srcs, d)
        g.wbfs_batch(srcs, d, opts=G.make_opts(teams=3))
        g.betweenness_batch(srcs, torch.empty((len(srcs), n), dtype=torch.float64, device="cuda"),
                            opts=G.make_opts(teams=2))
        g.bellman_ford_signed(0, np.empty(n, np.int64))
        g.bfs_batch(srcs, np.empty((len(srcs), n), np.uint32), np.empty((len(srcs), n), np.uint32))
        g.close()
        del d
        torch.cuda.synchronize()
        torch.cuda.empty_cache()

    cycle()
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(3):
        cycle()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < (16 << 20), (free0, free1)
