"""Time BFS, Bellman-Ford and wBFS on the paper's 3D-Torus (1000^3,
6*10^9 edges) with BJ c3's weight rule (uniform [1, 24] pair-hash weights) — the
paper's torus remark (Bellman-Ford does O(n^{4/3}) work there and
runs 7.3x slower than wBFS).  Dev tool: python tools/paper_torus.py [L]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from graphgen import device
    from paper_1805_05208_b200 import gbbs
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    t0 = time.time()
    off, tgt = device.torus_csr(L)
    w = device.pair_weights(off, tgt, 203, 24)
    g = gbbs.Graph(off, tgt, w, symmetric=True, borrow=True)
    n, m = off.shape[0] - 1, tgt.shape[0]
    d = torch.empty(n, dtype=torch.int32, device="cuda")
    out = {"L": L, "n": n, "m": m, "build_s": round(time.time() - t0, 1)}
    for algo in ("bfs", "wbfs", "bf"):
        times, rounds = [], 0
        for rep in range(2):
            st = gbbs.make_stats(0)
            if algo == "bfs":
                g.bfs(0, d, None, stats=st)
            elif algo == "wbfs":
                g.wbfs(0, d, stats=st)
            else:
                g.bellman_ford(0, d, stats=st)
            times.append(st.kernel_ms)
            rounds = st.rounds
        out[algo] = {"ms": round(min(times), 2), "rounds": rounds,
                     "gteps": round(m / (min(times) * 1e-3) / 1e9, 2),
                     "max_dist": int(d.max())}
        print(json.dumps({algo: out[algo]}), flush=True)
    out["bf_over_wbfs"] = round(out["bf"]["ms"] / out["wbfs"]["ms"], 2)
    print(json.dumps(out), flush=True)
    g.close()


if __name__ == "__main__":
    main()
