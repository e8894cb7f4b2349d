"""A few BFS batch steps of one config through gbbs_bfs_batch into device rows
(for ncu: the multi-traversal kernel).  python tools/one_batch.py --config c2 --reps 3"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--teams", type=int, default=0)
    a = ap.parse_args()
    import torch
    from graphgen import device as gdev
    from paper_1805_05208_b200 import gbbs
    G = gdev.build_config(a.config, weights=False)
    g = gbbs.Graph(G["offsets"], G["targets"], None, symmetric=G["symmetric"])
    srcs = G["sources"]
    dd = torch.empty((len(srcs), G["n"]), dtype=torch.int32, device="cuda")
    pp = torch.empty_like(dd)
    for _ in range(a.reps):
        g.bfs_batch(srcs, dd, pp, opts=gbbs.make_opts(teams=a.teams))
    torch.cuda.synchronize()
    print("ok", a.config, len(srcs), "sources")


if __name__ == "__main__":
    main()
