"""Every libgbbs entry point once on small graphs (c1 rMAT, a 12^3 torus, a
directed rMAT, a signed graph with a negative cycle), for compute-sanitizer:
compute-sanitizer --tool memcheck --error-exitcode 1 python tools/sanitize_smoke.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import graphgen
    from paper_1805_05208_b200 import gbbs
    cfg = graphgen.CONFIGS["c1"]
    off, tgt = graphgen.rmat_graph(cfg.levels, 1 << cfg.log_edges, cfg.graph_seed, *cfg.abc)
    w = graphgen.pair_weights(off, tgt, cfg.weight_seed, cfg.W)
    graphs = [(off, tgt, w, True)]
    toff, ttgt = graphgen.torus3d(12)
    graphs.append((toff, ttgt, graphgen.pair_weights(toff, ttgt, 3, 24), True))
    doff, dtgt = graphgen.rmat_graph(13, 1 << 16, 9, 0.6, 0.15, 0.15, symmetric=False)
    graphs.append((doff, dtgt, graphgen.pair_weights(doff, dtgt, 4, 13), False))
    for o, t, ww, sym in graphs:
        g = gbbs.Graph(o, t, ww, symmetric=sym)
        n = g.n
        d = torch.empty(n, dtype=torch.int32, device="cuda")
        p = torch.empty_like(d)
        for mode in (0, 1, 2):
            g.bfs(0, d, p, opts=gbbs.make_opts(20, mode), stats=gbbs.make_stats(256))
            g.bellman_ford(0, d, opts=gbbs.make_opts(20, mode))
            g.widest_path(0, d, opts=gbbs.make_opts(20, mode))
        g.wbfs(0, d, stats=gbbs.make_stats(1024))
        g.wbfs(0, d, opts=gbbs.make_opts(delta=4))
        d64 = torch.empty(n, dtype=torch.int64, device="cuda")
        g.bellman_ford_signed(0, d64)
        if sym:
            dd = torch.empty(n, dtype=torch.float64, device="cuda")
            g.betweenness(0, dd)
        g.bfs(0, np.empty(n, np.uint32), np.empty(n, np.uint32))  # host outputs
        g.close()
    ws = (w.astype(np.int64) - 2).astype(np.int32).view(np.uint32)  # negative cycles
    g = gbbs.Graph(off, tgt, ws, symmetric=True)
    d64 = torch.empty(g.n, dtype=torch.int64, device="cuda")
    for scope in (0, 1):
        g.bellman_ford_signed(0, d64, opts=gbbs.make_opts(neg_scope=scope))
    g.close()
    torch.cuda.synchronize()
    print("sanitize smoke: all entry points ran")


if __name__ == "__main__":
    main()
