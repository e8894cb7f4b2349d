"""Concurrent traversals without teams: S handles borrowing one resident graph, each
on its own stream with ctas_per_sm = C (so S reduced cooperative grids fit on the
GPU at once), sources dealt round-robin; batch-step time for the config's sources.
Dev tool: python tools/streams_probe.py c2 bfs,wbfs"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from graphgen import device as gdev
    from paper_1805_05208_b200 import gbbs
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    algos = (sys.argv[2] if len(sys.argv) > 2 else "bfs,wbfs").split(",")
    G = gdev.build_config(name, weights=True)
    srcs = G["sources"]
    n = G["n"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rows = torch.empty((len(srcs), n), dtype=torch.int32, device="cuda")
    prow = torch.empty_like(rows)
    for algo in algos:
        for S, C in ((1, 0), (2, 2), (3, 1), (4, 1)):
            hs = [gbbs.Graph(G["offsets"], G["targets"], G["weights"], symmetric=G["symmetric"],
                             borrow=True) for _ in range(S)]
            sts = [torch.cuda.Stream() for _ in range(S)]
            opts = gbbs.make_opts(ctas_per_sm=C)

            def run():
                # one host thread per stream would be needed to overlap the synchronous
                # calls; instead each handle runs its share back to back on its stream
                import threading
                def work(j):
                    with torch.cuda.stream(sts[j]):
                        for i in range(j, len(srcs), S):
                            if algo == "bfs":
                                hs[j].bfs(srcs[i], rows[i], prow[i], stream=sts[j], opts=opts)
                            else:
                                hs[j].wbfs(srcs[i], rows[i], stream=sts[j], opts=opts)
                th = [threading.Thread(target=work, args=(j,)) for j in range(S)]
                for t in th:
                    t.start()
                for t in th:
                    t.join()
            ts = []
            for rep in range(4):
                flush.fill_(1)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run()
                torch.cuda.synchronize()
                e1.record()
                torch.cuda.synchronize()
                if rep:
                    ts.append(e0.elapsed_time(e1))
            print(f"{name} {algo} streams={S} ctas_per_sm={C} step_ms={np.median(ts):.3f}", flush=True)
            for h in hs:
                h.close()


if __name__ == "__main__":
    main()
