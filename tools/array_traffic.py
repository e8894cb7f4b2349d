"""Per-array L2 request traffic of one traversal kernel launch (dev tool).

python tools/array_traffic.py SOURCE_CSV_GZ LIB_SO KERNEL_MANGLED [SRC_ROOT]

Joins ncu's per-SASS-instruction metrics (`--page source --csv --print-source
sass,cuda`, gzipped) with the inlined-at line tables of the same binary
(`nvdisasm -gi`): every global load / store / atomic is attributed to the array
named on the innermost source line of its inlining chain that names one (a load
inside ld_stream_v4() is charged to the pull_words() line that passes
`p.phot + v`).  Prints, per array, the L2 sectors requested (ncu "L2 Theoretical
Sectors Global") and the warp-stall samples of those instructions.
"""
import collections
import csv
import gzip
import io
import os
import re
import subprocess
import sys
import tempfile

ARRAYS = [  # (name, regex on the source line) — first match wins, order matters
    ("pull hot records (phot)", r"\bphot8?\b"),
    ("pull cold records (pcold)", r"\bpcold\b|\bpc32\b"),
    ("in-edges (in_tgt)", r"\bin_tgt\b"),
    ("in-offsets (in_off)", r"\bin_off\b"),
    ("no-in-edge mask (nin)", r"\bnin\b"),
    ("isolated mask (iso)", r"\biso\b"),
    ("level bytes (lvl)", r"\blvl\b|\bbfs_set_dist\("),
    ("dist", r"\bp\.dist\b|\bdist \+"),
    ("parent", r"\bp\.parent\b"),
    ("shadow", r"\bshadow\b"),
    ("out-targets (tgt)", r"\bp\.tgt\b"),
    ("weights (wgt)", r"\bp\.wgt\b"),
    ("out-offsets (off)", r"\bp\.off\b"),
    ("frontier lists (fv/fo/fb)", r"\bp\.f[vob]\b|\b[OBF] \+ |\bfo\[|\bfb\[|\bfv\[|\bst\[|\bF \+"),
    ("visited / frontier bitmaps", r"\bvis\b|\bvis_next\b|\bprebits\b|\bbits\b|\bbm\[|\bfr\b|\bvbit\("),
    ("counters / queues", r"\bcnt\b|\bwq\b|\bacq\b|\bhcnt\b|\bstatus\b|\bstats\b|\bbar\b"),
]


def line_text(path, ln, cache={}):
    if path not in cache:
        try:
            with open(path) as f:
                cache[path] = f.read().split("\n")
        except OSError:
            cache[path] = []
    t = cache[path]
    return t[ln - 1] if 0 < ln <= len(t) else ""


def sass_chains(lib, kernel, root):
    """address -> [(file, line), ...] innermost first, from nvdisasm -gi."""
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, check=True,
                       capture_output=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        out = subprocess.run(["nvdisasm", "-gi", os.path.join(d, cub)], check=True,
                             capture_output=True, text=True).stdout
    sec = out.split(f".text.{kernel}:", 1)[1]
    sec = re.split(r"\n\.text\.", sec, 1)[0]
    chains, cur = {}, []
    pend = False
    for line in sec.split("\n"):
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', line)
        if m:
            if not pend:
                cur = []
            f, ln = m.group(1), int(m.group(2))
            if root and f.startswith("/root/repo"):
                f = root + f[len("/root/repo"):]
            cur.append((f, ln))
            if m.group(3):
                g = m.group(3)
                if root and g.startswith("/root/repo"):
                    g = root + g[len("/root/repo"):]
                cur.append((g, int(m.group(4))))
            pend = True
            continue
        a = re.match(r"\s*/\*([0-9a-f]{4,})\*/", line)
        if a:
            chains[int(a.group(1), 16)] = list(cur)
            pend = False
    return chains


def classify(chain):
    for f, ln in chain:
        t = line_text(f, ln)
        for name, rx in ARRAYS:
            if re.search(rx, t):
                return name
    return "other"


def main():
    src_csv, lib, kernel = sys.argv[1:4]
    root = sys.argv[4] if len(sys.argv) > 4 else None
    chains = sass_chains(lib, kernel, root)
    rows = list(csv.reader(io.TextIOWrapper(gzip.open(src_csv))))
    his = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
    recs = []  # (runtime address, sass, L2 sectors, stall samples, executed)
    for bi, h in enumerate(his):
        hdr = rows[h]
        if "Address" not in hdr:
            continue
        end = his[bi + 1] - 2 if bi + 1 < len(his) else len(rows)
        ia = hdr.index("Address")
        iL2 = hdr.index("L2 Theoretical Sectors Global")
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        iE = hdr.index("Instructions Executed")
        for r in rows[h + 1:end]:
            if len(r) != len(hdr) or not r[ia].startswith("0x"):
                continue
            try:
                recs.append((int(r[ia], 16), r[3], float(r[iL2] or 0), float(r[iS] or 0),
                             float(r[iE] or 0)))
            except ValueError:
                continue
    base = min(a for a, *_ in recs)  # the kernel's first instruction
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
    seen = set()
    for addr, sass, l2, st, ex in recs:
        if addr in seen:
            continue
        seen.add(addr)
        op = re.search(r"\b(LDG|STG|ATOMG|REDG|RED|ATOM)\S*", sass)
        if not op:
            continue
        name = classify(chains.get(addr - base, []))
        agg[name][0] += l2
        agg[name][1] += st
        agg[name][2] += ex
    tot = sum(v[0] for v in agg.values()) or 1
    print(f"{'array':34s} {'L2 sectors':>14s} {'MB':>10s} {'share':>7s} {'stall smpl':>11s} {'warp insts':>12s}")
    for name, (l2, st, ex) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{name:34s} {l2:14.0f} {l2 * 32 / 1e6:10.1f} {l2 / tot:7.3f} {st:11.0f} {ex:12.0f}")
    print(f"{'total':34s} {tot:14.0f} {tot * 32 / 1e6:10.1f}")


if __name__ == "__main__":
    main()
