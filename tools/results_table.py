"""All BASELINE configs x algorithms on one B200 (dev/report tool, not the bench):
per source the kernel time (CUDA events around the persistent launch, L2 flushed
before each timed call, median of 5 after a warm-up call; all samples kept), GTEPS (reading A20), the contract's
roofline fraction (algorithmic bytes / time / measured peak, bench.algorithmic_bytes)
and the edge-traffic fraction (4 B per reached edge, reading A21b).
python tools/results_table.py [c1,c2,c3,c4,c5] > profiles/r01_results_all_configs.json"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ALGOS = {"c1": ("bfs", "bf", "wbfs", "wp"), "c2": ("bfs", "bf", "wbfs", "wp"),
         "c3": ("bfs", "bf", "wbfs", "wp"), "c4": ("bfs", "bf", "wbfs", "wp"),
         "c5": ("bfs", "bfs_T10", "bfs_T40")}


def main():
    import torch
    import bench
    from graphgen import device as gdev
    from paper_1805_05208_b200 import gbbs
    peak, _ = bench.measured_peaks()
    cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c1", "c2", "c3", "c4", "c5"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rows = []
    for name in cfgs:
        G = gdev.build_config(name, weights=name != "c5")
        g = gbbs.Graph(G["offsets"], G["targets"], G["weights"], symmetric=G["symmetric"])
        n, m = G["n"], G["m"]
        off = G["offsets"]
        d = torch.empty(n, dtype=torch.int32, device="cuda")
        p = torch.empty_like(d)
        for algo in ALGOS[name]:
            base = algo.split("_")[0]
            T = int(algo.split("_T")[1]) if "_T" in algo else 20
            opts = gbbs.make_opts(T)

            def call(s, st):
                if base == "bfs":
                    g.bfs(s, d, p, opts=opts, stats=st)
                elif base == "bf":
                    g.bellman_ford(s, d, opts=opts, stats=st)
                elif base == "wbfs":
                    g.wbfs(s, d, opts=opts, stats=st)
                else:
                    g.widest_path(s, d, opts=opts, stats=st)
            for s in G["sources"]:
                st = gbbs.make_stats(1 << 16)
                call(s, st)
                recs = gbbs.round_records(st)
                alg, _ = bench.algorithmic_bytes(recs, n, m, "bfs" if base == "bfs" else "bf")
                reach = int((off[1:] - off[:-1])[(d != 0) if base == "wp" else (d != -1)].sum())
                relax = sum(r["edges_examined"] for r in recs)
                ts = []
                for _ in range(5):
                    flush.fill_(1)
                    s2 = gbbs.make_stats(0)
                    call(s, s2)
                    ts.append(s2.kernel_ms)
                ms = float(np.median(ts))
                row = {"config": name, "algo": algo, "src": s, "ms": round(ms, 3),
                       "rounds": st.rounds, "m_reach": reach,
                       "gteps": round(reach / (ms * 1e-3) / 1e9, 2),
                       # Graph500-style undirected TEPS on symmetric graphs
                       "gteps_undirected": (round(reach / 2 / (ms * 1e-3) / 1e9, 2)
                                            if G["symmetric"] else None),
                       "samples_ms": [round(x, 4) for x in ts],
                       "relax_per_s_G": round(relax / (ms * 1e-3) / 1e9, 2),
                       "alg_GBps": round(alg / (ms * 1e-3) / 1e9, 1),
                       "roofline_frac": round(alg / (ms * 1e-3) / 1e9 / peak, 4),
                       "roofline_frac_nominal_8TBs": round(alg / (ms * 1e-3) / 1e9 / 8000.0, 4),
                       "edge_traffic_frac": round(4 * reach / (ms * 1e-3) / 1e9 / peak, 4)}
                rows.append(row)
                print(json.dumps(row), flush=True)
        g.close()
        del G, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
