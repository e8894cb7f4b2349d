import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from graphgen import device as gdev
from paper_1805_05208_b200 import gbbs
for name in (sys.argv[1] if len(sys.argv) > 1 else "c2,c4").split(","):
    G = gdev.build_config(name, weights=False)
    g = gbbs.Graph(G["offsets"], G["targets"], None, symmetric=True)
    d = torch.empty(G["n"], dtype=torch.float64, device="cuda")
    for s in G["sources"][:2]:
        ts = []
        for _ in range(3):
            st = gbbs.make_stats(0)
            g.betweenness(s, d, stats=st)
            ts.append(st.kernel_ms)
        print(name, s, "levels", st.rounds, "ms", round(min(ts), 3), flush=True)
    g.close(); del G, g; torch.cuda.empty_cache()
