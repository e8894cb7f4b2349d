"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (persistent kernel, AUTO direction, T = 20 unless swept).

* c1, c2: distances bit-exact against the oracle for every source; parents certified.
* c3: distances equal the torus closed form; per-round frontier sizes equal the
  closed-form level counts (385 rounds); Bellman-Ford exact against Dijkstra.
* c4, c5: the O(n+m) certificates (which imply exact distances and valid parents)
  on every seeded source (c5: x T in {10, 20, 40}, distances identical across T),
  plus one source per config compared element by element with the oracle.
"""
import numpy as np
import pytest

import graphgen
import oracle
from pins import torus_dist, torus_level_counts

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1805_05208_b200 import gbbs
    return gbbs


def build(name, weights):
    from graphgen import device
    D = device.build_config(name, weights=weights)
    host = dict(off=D["offsets"].cpu().numpy(), tgt=D["targets"].cpu().numpy().view(np.uint32),
                w=None if D["weights"] is None else D["weights"].cpu().numpy().view(np.uint32))
    return D, host


def gpu_bfs(G, g, n, s, T=20):
    d = torch.empty(n, dtype=torch.int32, device="cuda")
    p = torch.empty_like(d)
    st = G.make_stats(4096)
    g.bfs(s, d, p, opts=G.make_opts(T, G.GBBS_MODE_AUTO), stats=st)
    return d.cpu().numpy().view(np.uint32), p.cpu().numpy().view(np.uint32), st


def gpu_bf(G, g, n, s):
    d = torch.empty(n, dtype=torch.int32, device="cuda")
    g.bellman_ford(s, d)
    return d.cpu().numpy().view(np.uint32)


def gpu_wbfs(G, g, n, s, delta=0):
    d = torch.empty(n, dtype=torch.int32, device="cuda")
    st = G.make_stats(1 << 16)
    g.wbfs(s, d, opts=G.make_opts(delta=delta), stats=st)
    return d.cpu().numpy().view(np.uint32), st


def test_c1_full(G):
    D, H = build("c1", True)
    g = G.Graph(D["offsets"], D["targets"], D["weights"], symmetric=True)
    for s in D["sources"]:
        d, p, _ = gpu_bfs(G, g, D["n"], s)
        assert (d == oracle.bfs(H["off"], H["tgt"], s)[0]).all()
        assert oracle.check_bfs(H["off"], H["tgt"], s, d, p)[0]
        assert (gpu_bf(G, g, D["n"], s) == oracle.dijkstra(H["off"], H["tgt"], H["w"], s)[0]).all()
    g.close()


def test_c2_full(G):
    D, H = build("c2", True)   # weights [1,22] for the bench's Bellman-Ford leg
    g = G.Graph(D["offsets"], D["targets"], D["weights"], symmetric=True)
    n = D["n"]
    for i, s in enumerate(D["sources"]):
        ref, _ = oracle.bfs(H["off"], H["tgt"], s)
        d, p, st = gpu_bfs(G, g, n, s)
        assert (d == ref).all(), s
        assert oracle.check_bfs(H["off"], H["tgt"], s, d, p)[0]
        assert st.dense_rounds >= 1        # the direction optimisation engaged
        if i == 0:
            for T in (10, 40):
                assert (gpu_bfs(G, g, n, s, T)[0] == ref).all()
            wref = oracle.dijkstra(H["off"], H["tgt"], H["w"], s)[0]
            assert (gpu_bf(G, g, n, s) == wref).all()
            for delta in (0, 4):                         # NEXT-2: wBFS and Delta-stepping
                assert (gpu_wbfs(G, g, n, s, delta)[0] == wref).all(), delta
    g.close()


def test_c2_signed_johnson_full(G):
    """NEXT-4 at full c2 size: Johnson reweighting w'(u,v) = w + phi(u) - phi(v)
    makes ~half the edges negative without creating a negative cycle, so the signed
    Bellman-Ford must return d(v) + phi(src) - phi(v) with d from the oracle's
    Dijkstra on the original weights."""
    from pins import johnson_reweight
    D, H = build("c2", True)
    n = D["n"]
    phi = np.random.default_rng(11).integers(-1000, 1000, n).astype(np.int64)
    w2 = johnson_reweight(H["off"], H["tgt"], H["w"], phi)
    assert (w2.view(np.int32) < 0).mean() > 0.3
    g = G.Graph(D["offsets"], D["targets"], w2, symmetric=True)
    s = D["sources"][0]
    ref = oracle.dijkstra64(H["off"], H["tgt"], H["w"], s)[0]
    fin = ref != np.uint64(0xFFFFFFFFFFFFFFFF)
    exp = np.full(n, np.iinfo(np.int64).max, np.int64)
    exp[fin] = ref[fin].astype(np.int64) + phi[s] - phi[fin]
    d = torch.empty(n, dtype=torch.int64, device="cuda")
    g.bellman_ford_signed(s, d)
    assert (d.cpu().numpy() == exp).all()
    g.close()


def test_c2_planted_negative_cycle_early(G):
    """NEXT-4 early negative-cycle check (reading N4) at c2 size: c2 plus a directed
    appendage src -> a, a -> b -> c -> a (weights 1, 1, -5: a negative cycle) and a
    chain of K vertices hanging off c.  Without the early check the proof takes n
    rounds (~4.2 M); with it the call ends at the first power-of-two round >= 64.
    Expected values (no oracle run at n rounds): scope 0 every entry -inf (N1);
    scope 1 the appendage -inf (it is the cycle's forward closure) and every
    original vertex its Dijkstra distance on c2 (no appendage edge leads back)."""
    D, H = build("c2", True)
    n0, s = D["n"], D["sources"][0]
    off, tgt, w = H["off"], H["tgt"], H["w"]
    K = 1000
    a, b, c = n0, n0 + 1, n0 + 2
    # insert s -> a at the end of s's list (a is the largest id), then the appendage
    pos = int(off[s + 1])
    tgt2 = np.concatenate([tgt[:pos], [a], tgt[pos:]]).astype(np.uint32)
    w2 = np.concatenate([w[:pos], [3], w[pos:]]).astype(np.uint32)
    off2 = off.copy()
    off2[s + 1:] += 1
    app = [(a, b, 1), (b, c, 1), (c, a, -5), (c, n0 + 3, 2)]
    app += [(n0 + 3 + i, n0 + 4 + i, 2) for i in range(K - 4)]
    n = n0 + K
    deg = np.zeros(K, np.int64)
    for x, _, _ in app:
        deg[x - n0] += 1
    app.sort()
    off2 = np.concatenate([off2, off2[-1] + np.cumsum(deg)])
    tgt2 = np.concatenate([tgt2, np.array([y for _, y, _ in app], np.uint32)])
    w2 = np.concatenate([w2, np.array([x for _, _, x in app], np.int64).astype(np.int32).view(np.uint32)])
    assert off2.shape[0] == n + 1 and off2[-1] == tgt2.shape[0]
    g = G.Graph(off2, tgt2, w2)
    ref = oracle.dijkstra64(off, tgt, w, s)[0]
    fin = ref != np.uint64(0xFFFFFFFFFFFFFFFF)
    exp1 = np.full(n, np.iinfo(np.int64).max, np.int64)
    exp1[:n0][fin] = ref[fin].astype(np.int64)
    exp1[n0:] = np.iinfo(np.int64).min
    for scope in (0, 1):
        st = G.make_stats(0)
        d = torch.empty(n, dtype=torch.int64, device="cuda")
        g.bellman_ford_signed(s, d, opts=G.make_opts(neg_scope=scope), stats=st)
        got = d.cpu().numpy()
        if scope == 0:
            assert (got == np.iinfo(np.int64).min).all()
        else:
            assert (got == exp1).all()
        assert st.rounds <= 256, st.rounds          # ended by the early check, not n rounds
        assert st.kernel_ms < 1000.0, st.kernel_ms
    g.close()


def test_c3_full(G):
    D, H = build("c3", True)
    g = G.Graph(D["offsets"], D["targets"], D["weights"], symmetric=True)
    n, L = D["n"], graphgen.CONFIGS["c3"].L
    d, p, st = gpu_bfs(G, g, n, 0)
    assert (d == torus_dist(L, 0)).all()
    assert oracle.check_bfs(H["off"], H["tgt"], 0, d, p)[0]
    lv = torus_level_counts(L)
    assert st.rounds == len(lv) == 385
    assert [r["frontier"] for r in G.round_records(st)] == list(lv)
    ref = oracle.dijkstra(H["off"], H["tgt"], H["w"], 0)[0]
    bf = gpu_bf(G, g, n, 0)
    assert (bf == ref).all()
    # NEXT-2 wBFS, bucket width 1: every distinct distance is an extracted bucket,
    # every vertex expanded once
    wb, st = gpu_wbfs(G, g, n, 0)
    assert (wb == ref).all()
    recs = G.round_records(st)
    assert set(np.unique(ref).tolist()) <= {r["bucket"] for r in recs}
    assert sum(r["edges_examined"] for r in recs) == H["off"][-1]
    g.close()


def test_c4_full(G):
    """c4, every seeded source (PAPER.md:1475-1478 BFS and 1487-1490 SSSP output
    specs): Bellman-Ford and BFS certified on all 4 sources; one source compared
    element by element with oracle_dijkstra and oracle_bfs."""
    D, H = build("c4", True)
    g = G.Graph(D["offsets"], D["targets"], D["weights"], symmetric=True)
    n = D["n"]
    assert len(D["sources"]) == 4
    u = np.repeat(np.arange(n, dtype=np.uint32), np.diff(H["off"]))
    for i, s in enumerate(D["sources"]):
        bf = gpu_bf(G, g, n, s)
        assert oracle.check_sssp(H["off"], H["tgt"], H["w"], s, bf)[0], s
        d, p, _ = gpu_bfs(G, g, n, s)
        assert oracle.check_bfs(H["off"], H["tgt"], s, d, p)[0], s
        # symmetric graph: |d(u) - d(v)| <= 1 across every edge (BJ north star)
        fin = d[u] != 0xFFFFFFFF
        assert (np.abs(d[u][fin].astype(np.int64) - d[H["tgt"]][fin].astype(np.int64)) <= 1).all()
        if i == 0:
            assert (bf == oracle.dijkstra(H["off"], H["tgt"], H["w"], s)[0]).all()
            assert (d == oracle.bfs(H["off"], H["tgt"], s, want_parent=False)[0]).all()
        if i < 2:
            wb, st = gpu_wbfs(G, g, n, s)                     # NEXT-2: same distances
            assert (wb == bf).all(), s
            assert st.rounds >= np.unique(bf[bf != 0xFFFFFFFF]).size
    g.close()


def test_c5_full(G):
    """c5, all 8 seeded sources x T in {10, 20, 40} (BJ's threshold sweep): the BFS
    certificate on every (source, T) run's distances and parents, distances identical
    across T, and source 0 compared element by element with oracle_bfs."""
    D, H = build("c5", False)
    g = G.Graph(D["offsets"], D["targets"], None, symmetric=False)
    n = D["n"]
    assert len(D["sources"]) == 8
    for i, s in enumerate(D["sources"]):
        base = None
        for T in (20, 10, 40):
            d, p, st = gpu_bfs(G, g, n, s, T)
            assert oracle.check_bfs(H["off"], H["tgt"], s, d, p)[0], (s, T)
            if base is None:
                base = d
                assert st.dense_rounds >= 1
            else:
                assert (d == base).all(), (s, T)
        if i == 0:
            assert (base == oracle.bfs(H["off"], H["tgt"], s, want_parent=False)[0]).all()
    g.close()


def test_c2_betweenness_full(G):
    D, H = build("c2", False)
    g = G.Graph(D["offsets"], D["targets"], None, symmetric=True)
    s = D["sources"][0]
    d = torch.empty(D["n"], dtype=torch.float64, device="cuda")
    g.betweenness(s, d)
    ref, _ = oracle.betweenness(H["off"], H["tgt"], s)
    got = d.cpu().numpy()
    assert np.allclose(got, ref, rtol=1e-9, atol=1e-9 * float(np.abs(ref).max()))
    g.close()


def test_paper_torus_row_1000_cubed(G):
    """PAPER.md:2132 (sec:experiments, table:sizes) prints the 3D-Torus row: 10^9
    vertices, 6*10^9 edges, diam 1500 (tests/golden/paper_torus_row.txt).  Build
    exactly that graph on the GPU (≈100 GB: CSR 32 GB borrowed, frontier lists
    60 GB, dist 4 GB) and run BFS from vertex 0 in the bench's launch
    configuration: 1500 = the largest distance, 1501 edgeMap rounds, every round's
    frontier equal to the closed-form level count, every vertex reached, and
    sampled distances equal to the closed form."""
    from golden_io import read_kv
    from graphgen import device
    row = read_kv("paper_torus_row.txt")
    L = row["side"]
    free, _ = torch.cuda.mem_get_info()
    if free < 110 * 2 ** 30:
        pytest.skip(f"needs ~110 GB of free device memory, {free / 2 ** 30:.0f} GB free")
    off, tgt = device.torus_csr(L)
    assert off.shape[0] - 1 == row["vertices"] and tgt.shape[0] == row["edges"]
    g = G.Graph(off, tgt, None, symmetric=True, borrow=True)
    d = torch.empty(off.shape[0] - 1, dtype=torch.int32, device="cuda")
    st = G.make_stats(4096)
    g.bfs(0, d, None, opts=G.make_opts(20, G.GBBS_MODE_AUTO), stats=st)
    lv = torus_level_counts(L)
    assert st.rounds == len(lv) == row["diam"] + 1
    assert [r["frontier"] for r in G.round_records(st)] == list(lv)
    assert st.reached == row["vertices"]
    assert int(d.max()) == row["diam"]
    idx = torch.randint(0, row["vertices"], (1 << 20,), device="cuda", generator=None)
    ii = idx.to(torch.int64)
    x, y, z = ii % L, (ii // L) % L, ii // (L * L)
    ring = lambda a: torch.minimum(a, L - a)  # noqa: E731  (src = vertex 0)
    assert torch.equal(d[idx].to(torch.int64), ring(x) + ring(y) + ring(z))
    g.close()
    del off, tgt, d
    torch.cuda.empty_cache()
