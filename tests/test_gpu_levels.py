"""GPU parity of the BFS level-byte path (gbbs_opts.rules GBBS_RULE_LEVEL_BYTES_ON / _OFF).

The traversal records levels as one byte per vertex and expands them into dist in a
last pass (traverse.cuh bfs_set_dist); levels from 254 on are written to dist
directly.  Output spec P:1475-1478: the distances are the oracle's, bit for bit, in
every mode, on graphs with more than 254 rounds, on vertex counts that are not a
multiple of the pass's block (1024) or vector (4) sizes, on unaligned batch rows and
in team launches; the default (on above 2^24 vertices) is covered by the full-size
c4 / c5 tests.
"""
import numpy as np
import pytest

import graphgen
import oracle
from pins import grid_edges, path_graph

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

MODES = ("auto", "sparse", "dense")


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1805_05208_b200 import gbbs
    return gbbs


def _opts(G, mode="auto", on=True, teams=0):
    m = {"auto": G.GBBS_MODE_AUTO, "sparse": G.GBBS_MODE_SPARSE, "dense": G.GBBS_MODE_DENSE}[mode]
    return G.make_opts(mode=m, teams=teams,
                       rules=G.GBBS_RULE_LEVEL_BYTES_ON if on else G.GBBS_RULE_LEVEL_BYTES_OFF)


def _bfs(G, g, src, opts, parent=True):
    d = torch.full((g.n,), 0x5A5A5A5A, dtype=torch.int32, device="cuda")  # poison: every entry must be written
    p = torch.full_like(d, 0x5A5A5A5A) if parent else None
    g.bfs(src, d, p, opts=opts)
    torch.cuda.synchronize()
    return d.cpu().numpy().view(np.uint32), (p.cpu().numpy().view(np.uint32) if parent else None)


def _check(G, off, tgt, srcs, symmetric, modes=MODES):
    g = G.Graph(off, tgt, symmetric=symmetric)
    for src in srcs:
        ref, _ = oracle.bfs(off, tgt, src)
        for on in (True, False):
            for mode in modes:
                d, p = _bfs(G, g, src, _opts(G, mode, on))
                assert (d == ref).all(), (on, mode, src, np.nonzero(d != ref)[0][:5])
                ok, bad = oracle.check_bfs(off, tgt, src, d, p)
                assert ok, (on, mode, src, bad)
        d, _ = _bfs(G, g, src, _opts(G), parent=False)
        assert (d == ref).all()
    g.close()


@pytest.mark.parametrize("levels,log_edges", [(10, 13), (14, 18), (17, 20)])
def test_rmat_symmetric(G, levels, log_edges):
    off, tgt = graphgen.rmat_graph(levels, 1 << log_edges, 7, 0.57, 0.19, 0.19)
    _check(G, off, tgt, [0, 1, (1 << levels) - 1], True)


def test_rmat_directed(G):
    off, tgt = graphgen.rmat_graph(16, 1 << 20, 11, 0.6, 0.15, 0.15, symmetric=False)
    _check(G, off, tgt, [0, 5, 12345], False)


@pytest.mark.parametrize("n", [1, 2, 15, 17, 1023, 1025, 2049, 5000, 70001])
def test_odd_sizes(G, n):
    """Vertex counts around the fill's 16-byte groups and the pass's 1024-level blocks."""
    rng = np.random.default_rng(n)
    m = 3 * n
    e = [(int(a), int(b)) for a, b in zip(rng.integers(0, n, m), rng.integers(0, n, m)) if a != b]
    off, tgt = graphgen.from_edge_list(n, e)
    _check(G, off, tgt, [0, n - 1], True)


def test_more_rounds_than_a_byte(G):
    """A path of 3000 vertices: 2999 rounds, levels 254.. are written directly."""
    n = 3000
    off, tgt = graphgen.from_edge_list(n, path_graph(n))
    g = G.Graph(off, tgt, symmetric=True)
    for src in (0, 1500):
        for mode in ("auto", "sparse"):
            d, p = _bfs(G, g, src, _opts(G, mode))
            assert (d == np.abs(np.arange(n) - src).astype(np.uint32)).all()
            assert oracle.check_bfs(off, tgt, src, d, p)[0]
    g.close()


def test_grid_levels_cross_the_byte_limit(G):
    """200 x 200 grid from a corner: levels 0..398 (closed form), dense and sparse rounds."""
    a = 200
    off, tgt = graphgen.from_edge_list(a * a, grid_edges(a, a))
    g = G.Graph(off, tgt, symmetric=True)
    ids = np.arange(a * a)
    want = (ids % a + ids // a).astype(np.uint32)
    for mode in MODES:
        d, p = _bfs(G, g, 0, _opts(G, mode))
        assert (d == want).all(), mode
        assert oracle.check_bfs(off, tgt, 0, d, p)[0]
    g.close()


@pytest.mark.parametrize("teams", [1, 4])
def test_batch_rows_unaligned_and_teams(G, teams):
    """Batch rows of a graph with n % 4 != 0 start at unaligned addresses (scalar stores)."""
    n = 4099
    rng = np.random.default_rng(3)
    e = [(int(a), int(b)) for a, b in zip(rng.integers(0, n, 4 * n), rng.integers(0, n, 4 * n)) if a != b]
    off, tgt = graphgen.from_edge_list(n, e)
    g = G.Graph(off, tgt, symmetric=True)
    srcs = [0, 7, 100, 4098, 2048]
    rows = torch.full((len(srcs), n), 0x5A5A5A5A, dtype=torch.int32, device="cuda")
    prow = torch.full_like(rows, 0x5A5A5A5A)
    g.bfs_batch(srcs, rows, prow, opts=_opts(G, teams=teams))
    torch.cuda.synchronize()
    rows, prow = rows.cpu().numpy().view(np.uint32), prow.cpu().numpy().view(np.uint32)
    for i, s in enumerate(srcs):
        ref, _ = oracle.bfs(off, tgt, s)
        assert (rows[i] == ref).all(), (teams, s)
        assert oracle.check_bfs(off, tgt, s, rows[i], prow[i])[0]
    g.close()


def test_rules_on_and_off_together_rejected(G):
    off, tgt = graphgen.from_edge_list(4, path_graph(4))
    g = G.Graph(off, tgt, symmetric=True)
    d = torch.empty(4, dtype=torch.int32, device="cuda")
    with pytest.raises(Exception):
        g.bfs(0, d, None, opts=G.make_opts(rules=G.GBBS_RULE_LEVEL_BYTES_ON | G.GBBS_RULE_LEVEL_BYTES_OFF))
    g.close()


def test_pull_record_boundaries(G):
    """In-degrees 1..14 with the only reachable in-neighbour LAST in CSC order: the pull
    must walk the hot record (in0), the cold record (in1..in4) and the tail (in5..)
    in order and take that neighbour as the parent; dead in-neighbours
    have lower ids, so they come first in every in-list."""
    ndead, K = 20, 14
    A = ndead + 1
    n = A + 1 + K
    edges = [(0, A)]
    for k in range(1, K + 1):
        t = A + k
        edges += [(d, t) for d in range(1, k)]  # k - 1 unreachable in-neighbours
        edges.append((A, t))
    off, tgt = graphgen.from_edge_list(n, edges, symmetric=False)
    ref, _ = oracle.bfs(off, tgt, 0)
    assert ref[A] == 1 and (ref[A + 1:] == 2).all() and (ref[1:A] == 0xFFFFFFFF).all()
    g = G.Graph(off, tgt, symmetric=False)
    for on in (True, False):
        for mode in MODES:
            d, p = _bfs(G, g, 0, _opts(G, mode, on))
            assert (d == ref).all(), (on, mode)
            assert (p[A + 1:] == A).all() and p[A] == 0, (on, mode, p)
            assert oracle.check_bfs(off, tgt, 0, d, p)[0]
    g.close()
