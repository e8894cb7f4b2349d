"""NEXT-4 GPU parity: gbbs_bellman_ford_signed (general-weight SSSP, output spec
PAPER.md:1487-1490 sec:benchmark, frontier algorithm) through the
C ABI against oracle.bellman_ford_signed, element by element (int64 distances
with INT64_MAX = unreachable, INT64_MIN = -infinity; bit-exact), for both
readings of the negative-cycle clause (neg_scope 0 = every distance -inf,
reading N1; 1 = the cycle's forward closure, reading N2).
"""
import numpy as np
import pytest

import graphgen
import oracle
from pins import johnson_reweight, signed_csr, signed_expected

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NEGINF = np.iinfo(np.int64).min
POSINF = np.iinfo(np.int64).max


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1805_05208_b200 import gbbs
    return gbbs


def run(G, g, src, scope=0, host=False, stats=None):
    d = np.empty(g.n, np.int64) if host else torch.empty(g.n, dtype=torch.int64, device="cuda")
    opts = G.make_opts(neg_scope=scope) if (scope or stats is not None) else None
    g.bellman_ford_signed(src, d, opts=opts, stats=stats)
    return d if host else d.cpu().numpy()


def test_spec_examples(G):
    off, tgt, w = signed_csr(3, [(0, 1), (1, 2)], [4, -2])
    g = G.Graph(off, tgt, w)
    for scope in (0, 1):
        assert list(run(G, g, 0, scope)) == [0, 4, 2]
    g.close()
    off, tgt, w = signed_csr(2, [(0, 1), (1, 0)], [1, -3])
    g = G.Graph(off, tgt, w)
    for scope in (0, 1):
        assert list(run(G, g, 0, scope)) == [NEGINF, NEGINF]
    g.close()


@pytest.mark.parametrize("seed", range(10))
def test_brute_force_small(G, seed):
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.integers(2, 12))
    edges = [(int(a), int(b)) for a in range(n) for b in range(n) if a != b and rng.random() < 0.3]
    ws = rng.integers(-4, 9, len(edges))
    off, tgt, w = signed_csr(n, edges, ws)
    g = G.Graph(off, tgt, w)
    for src in range(n):
        for scope in (0, 1):
            exp, _ = signed_expected(n, off, tgt, w, src, scope)
            ref, _ = oracle.bellman_ford_signed(off, tgt, w, src, scope)
            assert (ref == exp).all()
            got = run(G, g, src, scope, host=(src == 0))
            assert (got == ref).all(), (seed, src, scope, got, ref)
    g.close()


def test_planted_cycles_scopes(G):
    edges = [(0, 1), (1, 2), (2, 0), (2, 3), (3, 4), (5, 0)]
    off, tgt, w = signed_csr(7, edges, [2, -4, 1, 7, -1, 3])
    g = G.Graph(off, tgt, w)
    for src, scope in ((0, 0), (0, 1), (3, 1), (5, 1), (6, 0)):
        ref, _ = oracle.bellman_ford_signed(off, tgt, w, src, scope)
        assert (run(G, g, src, scope) == ref).all(), (src, scope)
    g.close()


@pytest.mark.parametrize("seed", range(3))
def test_random_with_negative_cycles(G, seed):
    """Medium random digraphs whose weights make some cycles negative."""
    off, tgt = graphgen.random_graph(1500, 0.002, 700 + seed, symmetric=False)
    w = (graphgen.pair_weights(off, tgt, seed, 30).astype(np.int64) - 3).astype(np.int32).view(np.uint32)
    g = G.Graph(off, tgt, w)
    for src in (0, 1, 777):
        for scope in (0, 1):
            ref, neg = oracle.bellman_ford_signed(off, tgt, w, src, scope)
            assert (run(G, g, src, scope) == ref).all(), (src, scope, neg)
    g.close()


@pytest.mark.parametrize("sym", [False, True])
def test_johnson_reweighted_rmat(G, sym):
    """No negative cycle, many negative edges: d'(v) = d(v) + phi(src) - phi(v)."""
    off, tgt = graphgen.rmat_graph(14, 1 << 17, 31, 0.57, 0.19, 0.19, symmetric=sym)
    w = graphgen.pair_weights(off, tgt, 4, 14)
    n = off.shape[0] - 1
    phi = np.random.default_rng(5).integers(-5000, 5000, n).astype(np.int64)
    w2 = johnson_reweight(off, tgt, w, phi)
    g = G.Graph(off, tgt, w2)
    src = int(np.argmax(np.diff(off)))
    ref, _ = oracle.dijkstra64(off, tgt, w, src)
    fin = ref != np.uint64(0xFFFFFFFFFFFFFFFF)
    exp = np.full(n, POSINF, np.int64)
    exp[fin] = ref[fin].astype(np.int64) + phi[src] - phi[fin]
    st = G.make_stats(4096)
    got = run(G, g, src, 1, stats=st)
    assert (got == exp).all()
    assert st.rounds < n                  # no negative cycle: the frontier emptied early
    g.close()


def test_nonnegative_and_unit_weights(G):
    off, tgt = graphgen.rmat_graph(14, 1 << 17, 3, 0.57, 0.19, 0.19)
    w = graphgen.pair_weights(off, tgt, 1, 14)
    g = G.Graph(off, tgt, w, symmetric=True)
    ref, _ = oracle.dijkstra(off, tgt, w, 0)
    got = run(G, g, 0)
    fin = ref != 0xFFFFFFFF
    assert (got[fin] == ref[fin]).all() and (got[~fin] == POSINF).all()
    g.close()
    g = G.Graph(off, tgt, None, symmetric=True)
    b, _ = oracle.bfs(off, tgt, 0)
    got = run(G, g, 0)
    assert (got[b != 0xFFFFFFFF] == b[b != 0xFFFFFFFF]).all() and (got[b == 0xFFFFFFFF] == POSINF).all()
    g.close()


def test_extreme_weights_and_errors(G):
    off, tgt, w = signed_csr(3, [(0, 1), (1, 2)], [-(2 ** 31), 2 ** 31 - 1])
    g = G.Graph(off, tgt, w)
    assert list(run(G, g, 0)) == [0, -(2 ** 31), -1]
    d = np.zeros(3, np.int64)
    with pytest.raises(G.GbbsError) as e:
        g.bellman_ford_signed(3, d)
    assert e.value.code == -1
    with pytest.raises(G.GbbsError):
        g.bellman_ford_signed(0, d, opts=G.make_opts(neg_scope=2))
    g.close()
