"""Summarise an ncu --set full report: top SASS instructions by warp-stall samples
and the stall-reason totals (dev tool; reads `ncu -i <rep> --page source --csv`)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name"')
for b in blocks[1:2]:
    lines = b.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
    data = []
    tot = {}
    for r in rows[1:]:
        try:
            s = int(r[isamp])
        except (ValueError, IndexError):
            continue
        data.append((s, r[ia], r[isrc].strip(), {hdr[i]: int(r[i] or 0) for i in stall_cols}))
        for i in stall_cols:
            tot[hdr[i]] = tot.get(hdr[i], 0) + int(r[i] or 0)
    allsamp = sum(d[0] for d in data)
    print("total samples", allsamp)
    print("stall totals:", ", ".join(f"{k[6:]}={v * 100 / max(1, allsamp):.1f}%" for k, v in
                                     sorted(tot.items(), key=lambda x: -x[1])[:8]))
    for s, a, src, st in sorted(data, key=lambda x: -x[0])[:top]:
        main = sorted(st.items(), key=lambda x: -x[1])[:2]
        print(f"{s * 100 / allsamp:5.1f}% {a[-5:]} {src[:60]:60s} {' '.join(f'{k[6:]}:{v}' for k, v in main)}")
