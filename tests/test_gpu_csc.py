"""GPU: the create-time in-edge CSC (a0, csc.cuh's counting transpose) against the
transpose numpy computes from the same CSR — every in-list holds exactly the
in-edges of its vertex, ascending by source id (the order the dense pull scans,
PAPER.md:1870-1874).  Covers all four sort classes of csc.cuh: <= 16 in-edges
(thread network), <= 1024 (warp bitonic), <= 8192 (CTA bitonic) and hubs above
8192 (chunk sorts + merge passes, odd and even pass counts), multi-edges, and
vertices without in-edges."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1805_05208_b200 import gbbs
    return gbbs


def csr_from_edges(n, src, dst):
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    off = np.zeros(n + 1, np.int64)
    np.add.at(off, src + 1, 1)
    return np.cumsum(off), dst.astype(np.uint32)


def expected_csc(n, off, tgt):
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(off))
    order = np.lexsort((src, tgt.astype(np.int64)))
    in_src = src[order].astype(np.uint32)
    in_off = np.zeros(n + 1, np.int64)
    np.add.at(in_off, tgt.astype(np.int64) + 1, 1)
    return np.cumsum(in_off), in_src


def check(G, n, off, tgt):
    g = G.Graph(off, tgt, symmetric=False)
    io, isrc = g.in_edges()
    eo, esrc = expected_csc(n, off, tgt)
    assert np.array_equal(io, eo)
    assert np.array_equal(isrc, esrc)


@pytest.mark.parametrize("hub_deg", [0, 9000, 20000, 40000, 70000])
def test_csc_all_classes(G, hub_deg):
    rng = np.random.default_rng(1000 + hub_deg)
    n = 1 << 17
    # skewed targets: degrees from 0 up to ~1500, plus hubs of exactly hub_deg in-edges
    m0 = 1 << 20
    s = rng.integers(0, n, m0)
    t = (rng.pareto(1.2, m0) * 50).astype(np.int64) % n
    parts_s, parts_t = [s], [t]
    if hub_deg:
        for h in (5, n - 3):  # two hubs: every source but a few, distinct ids
            srcs = rng.choice(n, hub_deg, replace=False)
            parts_s.append(srcs)
            parts_t.append(np.full(hub_deg, h))
    s = np.concatenate(parts_s)
    t = np.concatenate(parts_t)
    off, tgt = csr_from_edges(n, s, t)  # keeps multi-edges
    check(G, n, off, tgt)


def test_csc_tiny_and_empty_lists(G):
    # path 0 -> 1 -> 2, a vertex with only out-edges, isolated vertices
    n = 7
    s = np.array([0, 1, 3, 3, 3], np.int64)
    t = np.array([1, 2, 0, 1, 1], np.int64)  # 3 -> 1 twice (multi-edge)
    off, tgt = csr_from_edges(n, s, t)
    check(G, n, off, tgt)


def test_csc_single_source_star(G):
    # one source with out-edges to everyone: every in-list has exactly one entry
    n = 50000
    s = np.zeros(n - 1, np.int64)
    t = np.arange(1, n, dtype=np.int64)
    off, tgt = csr_from_edges(n, s, t)
    check(G, n, off, tgt)
