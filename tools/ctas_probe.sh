for C in 0 1 2 3; do
python - <<PY
import sys, os; sys.path.insert(0, os.getcwd())
import torch, numpy as np
from graphgen import device as gdev
from paper_1805_05208_b200 import gbbs
G = gdev.build_config("c3", weights=True)
g = gbbs.Graph(G["offsets"], G["targets"], G["weights"], symmetric=True)
d = torch.empty(G["n"], dtype=torch.int32, device="cuda"); p = torch.empty_like(d)
o = gbbs.make_opts(ctas_per_sm=$C)
for algo in ("bfs", "bf", "wbfs"):
    ts = []
    for _ in range(3):
        st = gbbs.make_stats(0)
        if algo == "bfs": g.bfs(0, d, p, opts=o, stats=st)
        elif algo == "bf": g.bellman_ford(0, d, opts=o, stats=st)
        else: g.wbfs(0, d, opts=o, stats=st)
        ts.append(st.kernel_ms)
    print("c3", algo, "ctas_per_sm=$C", round(min(ts), 3), "ms", flush=True)
PY
done
