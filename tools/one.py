"""Run a few traversals of one config (for ncu: profile the last launch).

python tools/one.py --config c5 --algo bfs --reps 3 [--mode auto|sparse|dense] [--T 20]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--algo", default="bfs")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--mode", default="auto")
    ap.add_argument("--T", type=int, default=20)
    ap.add_argument("--src", type=int, default=0, help="index into the config's sources")
    ap.add_argument("--ctas", type=int, default=0, help="CTAs per SM (0 = max)")
    ap.add_argument("--delta", type=int, default=0, help="wbfs bucket width (0 = default)")
    ap.add_argument("--noparent", action="store_true", help="BFS without the parent output")
    a = ap.parse_args()
    import torch
    from graphgen import device as gdev
    from paper_1805_05208_b200 import gbbs
    G = gdev.build_config(a.config, weights=a.algo != "bfs")
    g = gbbs.Graph(G["offsets"], G["targets"], G["weights"], symmetric=G["symmetric"])
    d = torch.empty(G["n"], dtype=torch.int32, device="cuda")
    p = torch.empty_like(d)
    opts = gbbs.make_opts(a.T, {"auto": 0, "sparse": 1, "dense": 2}[a.mode], a.ctas, a.delta)
    s = G["sources"][a.src]
    for _ in range(a.reps):
        st = gbbs.make_stats(0)
        if a.algo == "bfs":
            g.bfs(s, d, None if a.noparent else p, opts=opts, stats=st)
        elif a.algo == "bf":
            g.bellman_ford(s, d, opts=opts, stats=st)
        elif a.algo == "wbfs":
            g.wbfs(s, d, opts=opts, stats=st)
        else:
            g.widest_path(s, d, opts=opts, stats=st)
        print(f"{a.config} {a.algo} src={s} kernel {st.kernel_ms * 1e3:.1f} us", flush=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
