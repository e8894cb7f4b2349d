"""Summarise tools/r02_ab.sh logs: per variant, kernel us per (config, algo, source)."""
import glob, re, sys, collections
vs = sys.argv[1:] or ["default"]
rows = collections.OrderedDict()
for v in vs:
    for f in sorted(glob.glob(f"gpurun_out/ab*_{v}.log")):
        cfg = None
        for line in open(f):
            if line.startswith("== "):
                cfg = line.split()[1].rstrip(":")
            m = re.match(r"-- (\w+) src=(\d+) .*kernel=([\d.]+)us", line)
            if m:
                rows.setdefault((cfg, m.group(1), m.group(2)), {})[v] = float(m.group(3))
tot = collections.defaultdict(lambda: collections.defaultdict(float))
print("config algo src " + " ".join(vs))
for (c, a, s), d in rows.items():
    print(c, a, s, " ".join(f"{d.get(v, float('nan')):9.1f}" for v in vs))
    for v in vs:
        tot[(c, a)][v] += d.get(v, 0)
print("totals:")
for (c, a), d in tot.items():
    b = d[vs[0]]
    print(c, a, " ".join(f"{d[v]:9.1f} ({d[v] / b:5.3f})" for v in vs))
