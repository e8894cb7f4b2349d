"""Aggregate ncu warp-stall samples and L2 sectors by CUDA source line (dev tool).
python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if len(r) > 3 and r[0] == "Line No"][0]
hdr = rows[hi]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iG = hdr.index("L2 Theoretical Sectors Global")
iL = hdr.index("L2 Theoretical Sectors Local")
src = {}
agg = {}
cur = None
for r in rows[hi + 1:]:
    if len(r) <= iS:
        continue
    ln = r[0]
    if ln:
        cur = ln
        src[ln] = r[1].strip()
    try:
        s = int(r[iS] or 0); g = int(r[iG] or 0); l = int(r[iL] or 0)
    except ValueError:
        continue
    a = agg.setdefault(cur, [0, 0, 0])
    a[0] += s; a[1] += g; a[2] += l
tot = sum(v[0] for v in agg.values()) or 1
print(f"samples {tot}; global L2 sectors {sum(v[1] for v in agg.values()) * 32 / 1e9:.2f} GB; "
      f"local {sum(v[2] for v in agg.values()) * 32 / 1e9:.2f} GB")
for ln, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{v[0] * 100 / tot:5.1f}% {v[1] * 32 / 1e6:8.1f}MB L{ln:>4} {src.get(ln, '')[:80]}")
