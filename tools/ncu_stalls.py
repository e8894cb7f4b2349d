"""Warp-stall samples by CUDA source line, with the top stall reasons, from a
gzipped `ncu --page source --csv --print-source sass,cuda` export (dev tool).
python tools/ncu_stalls.py source.csv.gz [top]"""
import collections
import csv
import gzip
import io
import sys

rows = list(csv.reader(io.TextIOWrapper(gzip.open(sys.argv[1]))))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
his = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
agg = collections.Counter()
src = {}
st = collections.defaultdict(collections.Counter)
allst = collections.Counter()
for bi, h in enumerate(his):
    hdr = rows[h]
    end = his[bi + 1] - 3 if bi + 1 < len(his) else len(rows)
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    ci = [hdr.index(c) for c in cols]
    cur = None
    for r in rows[h + 1:end]:
        if len(r) != len(hdr):
            continue
        if r[0]:
            cur = f"{bi}:{r[0]}"
            src[cur] = r[1].strip()[:88]
        try:
            s = int(r[iS] or 0)
        except ValueError:
            continue
        if cur is None:
            continue
        agg[cur] += s
        for c, i in zip(cols, ci):
            try:
                v = int(r[i] or 0)
            except ValueError:
                v = 0
            st[cur][c] += v
            allst[c] += v
tot = sum(agg.values()) or 1
print("stall reasons:", ", ".join(f"{k[6:]} {100 * v / sum(allst.values()):.1f}%" for k, v in allst.most_common(6)))
for ln, s in agg.most_common(top):
    t = ", ".join(f"{k[6:]} {v}" for k, v in st[ln].most_common(2))
    print(f"{100 * s / tot:5.1f}% {ln:8s} {src[ln]:88s} {t}")

# --regions SRC: stall samples of file block 0 summed per enclosing function of SRC
if "--regions" in sys.argv:
    import re
    srcf = sys.argv[sys.argv.index("--regions") + 1]
    starts = []
    for i, line in enumerate(open(srcf), 1):
        mt = re.match(r"^(?:__device__|__global__)[^(]*?(\w+)\(", line)
        if mt:
            starts.append((i, mt.group(1)))
    reg = collections.Counter()
    for ln, sm in agg.items():
        blk, num = ln.split(":")
        if blk != "0":
            reg["(other files)"] += sm
            continue
        name = "(top)"
        for st0, nm in starts:
            if st0 <= int(num):
                name = nm
        reg[name] += sm
    for k, v in reg.most_common(20):
        print(f"{100 * v / tot:5.1f}% {k}")
