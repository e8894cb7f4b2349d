"""Batch-step time of the configs' sources through gbbs_bfs_batch / bellman_ford_batch
into device rows, for teams = 1..4 (dev tool): python tools/teams_probe.py c2,c4,c5"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from graphgen import device as gdev
    from paper_1805_05208_b200 import gbbs
    for name in (sys.argv[1] if len(sys.argv) > 1 else "c2").split(","):
        G = gdev.build_config(name, weights=name != "c5")
        g = gbbs.Graph(G["offsets"], G["targets"], G["weights"], symmetric=G["symmetric"])
        srcs = G["sources"]
        n = G["n"]
        dd = torch.empty((len(srcs), n), dtype=torch.int32, device="cuda")
        db = torch.empty((len(srcs), n), dtype=torch.float64, device="cuda")
        pp = torch.empty_like(dd)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        algos = tuple(os.environ.get("ALGOS", "bfs,bf,wbfs").split(",")) if G["weights"] is not None \
            else ("bfs",)
        for algo in algos:
            base = None
            for teams, T, cps in [(int(a), int(b), int(c)) for a in os.environ.get("TEAMS", "1,2,3,4").split(",")
                                  for b in os.environ.get("THRESH", "20").split(",")
                                  for c in os.environ.get("CTAS", "0").split(",")]:
                opts = gbbs.make_opts(teams=teams, threshold_den=T, ctas_per_sm=cps)
                ts = []
                for rep in range(4):
                    flush.fill_(1)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    if algo == "bfs":
                        g.bfs_batch(srcs, dd, pp, opts=opts)
                    elif algo == "wbfs":
                        g.wbfs_batch(srcs, dd, opts=opts)
                    elif algo == "bc":
                        g.betweenness_batch(srcs, db, opts=opts)
                    else:
                        g.bellman_ford_batch(srcs, dd, opts=opts)
                    e1.record()
                    torch.cuda.synchronize()
                    if rep:
                        ts.append(e0.elapsed_time(e1))
                out = (db if algo == "bc" else dd).cpu().numpy()
                if base is None:
                    base = out
                same = bool(np.allclose(out, base, rtol=1e-9)) if algo == "bc" else bool((out == base).all())
                print(f"{name} {algo} teams={teams} T={T} ctas={cps} step_ms={np.median(ts):.3f} rows_equal={same}",
                      flush=True)
        g.close()
        del G, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
