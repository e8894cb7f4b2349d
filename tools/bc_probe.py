"""Single-source betweenness kernel time per config and forward-direction mode
(dev tool): python tools/bc_probe.py c2,c4 [auto,sparse,dense]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from graphgen import device as gdev  # noqa: E402
from paper_1805_05208_b200 import gbbs  # noqa: E402

MODES = {"auto": gbbs.GBBS_MODE_AUTO, "sparse": gbbs.GBBS_MODE_SPARSE, "dense": gbbs.GBBS_MODE_DENSE}
modes = (sys.argv[2] if len(sys.argv) > 2 else "auto").split(",")
for name in (sys.argv[1] if len(sys.argv) > 1 else "c2,c4").split(","):
    G = gdev.build_config(name, weights=False)
    g = gbbs.Graph(G["offsets"], G["targets"], None, symmetric=True)
    d = torch.empty(G["n"], dtype=torch.float64, device="cuda")
    for s in G["sources"][:2]:
        ref = None
        for md in modes:
            ts = []
            for _ in range(3):
                st = gbbs.make_stats(0)
                g.betweenness(s, d, stats=st, opts=gbbs.make_opts(mode=MODES[md]))
                ts.append(st.kernel_ms)
            out = d.cpu()
            if ref is None:
                ref = out
            ok = bool(torch.allclose(out, ref, rtol=1e-9, atol=1e-9 * float(ref.abs().max())))
            print(name, s, md, "levels", st.rounds, "ms", round(min(ts), 3), "same", ok, flush=True)
    g.close()
    del G, g
    torch.cuda.empty_cache()
