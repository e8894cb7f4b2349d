"""Per-round profile of libgbbs traversals on the BASELINE configs (dev tool).

python tools/probe.py --configs c2,c3 --algos bfs,bf --nsrc 1 [--mode auto|sparse|dense] [--T 20]
Prints, per traversal, one line per round (mode, |U|, sum deg, acquired, edges
examined, swept, device µs from %globaltimer) and the un-instrumented kernel time.
"""
import argparse
import os
import sys
import time

import numpy as np

NOPARENT = False
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_algo(g, algo, s, d, p, opts, st):
    if algo == "bfs" and NOPARENT:
        g.bfs(s, d, None, opts=opts, stats=st)
    elif algo == "bfs":
        g.bfs(s, d, p, opts=opts, stats=st)
    elif algo == "bf":
        g.bellman_ford(s, d, opts=opts, stats=st)
    elif algo == "wbfs":
        g.wbfs(s, d, opts=opts, stats=st)
    else:
        g.widest_path(s, d, opts=opts, stats=st)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2")
    ap.add_argument("--algos", default="bfs")
    ap.add_argument("--nsrc", type=int, default=1)
    ap.add_argument("--mode", default="auto")
    ap.add_argument("--T", type=int, default=20)
    ap.add_argument("--delta", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--rounds", action="store_true", help="print every round")
    ap.add_argument("--check", action="store_true", help="certify against the oracle certificate")
    ap.add_argument("--noparent", action="store_true", help="BFS without the parent output")
    ap.add_argument("--rules", type=int, default=0, help="gbbs_opts.rules (1 = paper's m/T rule only)")
    a = ap.parse_args()
    global NOPARENT
    NOPARENT = a.noparent
    import torch
    from graphgen import device as gdev
    from paper_1805_05208_b200 import gbbs
    mode = {"auto": 0, "sparse": 1, "dense": 2, "pull": 3}[a.mode]
    for name in a.configs.split(","):
        t0 = time.time()
        G = gdev.build_config(name, weights=True)
        g = gbbs.Graph(G["offsets"], G["targets"], G["weights"], symmetric=G["symmetric"])
        print(f"== {name}: n={G['n']} m={G['m']} build {time.time() - t0:.1f}s sources={G['sources']}",
              flush=True)
        n = G["n"]
        d = torch.empty(n, dtype=torch.int32, device="cuda")
        p = torch.empty(n, dtype=torch.int32, device="cuda")
        off = G["offsets"]
        for algo in a.algos.split(","):
            for s in G["sources"][: a.nsrc]:
                st = gbbs.make_stats(1 << 17)
                opts = gbbs.make_opts(a.T, mode, delta=a.delta, rules=a.rules)
                run_algo(g, algo, s, d, p, opts, st)
                recs = gbbs.round_records(st)
                mreach = int((off[1:] - off[:-1])[d != -1].sum())
                kms = []
                for _ in range(a.reps):
                    s2 = gbbs.make_stats(0)
                    run_algo(g, algo, s, d, p, opts, s2)
                    kms.append(s2.kernel_ms)
                km = float(np.median(kms))
                tot_us = sum(r["us"] or 0 for r in recs)
                print(f"-- {algo} src={s} alg_bytes={sum(r['alg_bytes'] for r in recs) / 1e6:.1f}MB rounds={st.rounds} dense={st.dense_rounds} reached={st.reached} "
                      f"m_reach={mreach} kernel={km * 1e3:.1f}us (stats run rounds sum {tot_us:.1f}us) "
                      f"GTEPS={mreach / km / 1e6:.1f}", flush=True)
                if a.rounds or st.rounds <= 40:
                    for i, r in enumerate(recs):
                        print(f"   r{i:<4d} {'SDFPBR'[r['dense']] if r['dense'] < 3 or a.algos.find('wbfs') < 0 else 'BN'[r['dense'] - 3]} k={r['bucket']:<6d} U={r['frontier']:>10d} "
                              f"E={r['frontier_edges']:>11d} acq={r['acquired']:>9d} "
                              f"ex={r['edges_examined']:>11d} sw={r['vertices_swept']:>9d} "
                              f"{(r['us'] or 0):9.1f}us  work<{r['work_us']:.1f} flush<{r['flush_us']:.1f} "
                              f"ab={r['alg_bytes'] / 1e6:.1f}MB hh={r['head_hits']}")
                else:
                    us = np.array([r["us"] or 0 for r in recs])
                    fr = np.array([r["frontier"] for r in recs])
                    wk = np.array([r["work_us"] for r in recs])
                    fl = np.array([r["flush_us"] for r in recs])
                    print(f"   totals: entries {sum(r['frontier'] for r in recs)} edges "
                          f"{sum(r['edges_examined'] for r in recs)} acquired {sum(r['acquired'] for r in recs)}")
                    print(f"   per-round us: median {np.median(us):.2f} p90 {np.percentile(us, 90):.2f} "
                          f"max {us.max():.1f}; work-end median {np.median(wk):.2f} flush-end median "
                          f"{np.median(fl):.2f}; frontier median {np.median(fr):.0f} max {fr.max()}")
                if a.check:
                    import oracle
                    ho = off.cpu().numpy()
                    ht = G["targets"].cpu().numpy().view(np.uint32)
                    dd = d.cpu().numpy().view(np.uint32)
                    if algo == "bfs":
                        ok = oracle.check_bfs(ho, ht, s, dd, p.cpu().numpy().view(np.uint32))
                    else:
                        hw = G["weights"].cpu().numpy().view(np.uint32)
                        ok = oracle.check_sssp(ho, ht, hw, s, dd)
                    print("   certificate:", ok, flush=True)
        g.close()
        del G
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
