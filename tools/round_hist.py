"""Bucket the per-round records printed by tools/probe.py --rounds by frontier size
(dev tool): python tools/round_hist.py gpurun_out/probe_c3.log"""
import re
import sys

import numpy as np

cur = None
rows = {}
for line in open(sys.argv[1]):
    if line.startswith('-- '):
        cur = line.split()[1] + ' ' + line.split()[2]
        rows[cur] = []
    m = re.match(r'\s+r(\d+)\s+(\S)\s+k=\s*(\d+)\s+U=\s*(\d+)\s+E=\s*(\d+)\s+acq=\s*(\d+)\s+ex=\s*(\d+)'
                 r'\s+sw=\s*(\d+)\s+([\d.]+)us\s+work<([-\d.]+)\s+flush<([-\d.]+)', line)
    if m and cur:
        rows[cur].append([float(x) for x in m.groups()[2:]])
for k, v in rows.items():
    v = np.array(v)
    if not len(v):
        continue
    U, us, wk, fl = v[:, 1], v[:, 6], v[:, 7], v[:, 8]
    print(k, len(v), 'rounds, sum %.0f us' % us.sum())
    for lo, hi in [(0, 1000), (1000, 10000), (10000, 50000), (50000, 1e12)]:
        sel = (U >= lo) & (U < hi)
        if sel.any():
            print(f'  U in [{lo},{hi:.0f}): n={sel.sum()} mean {us[sel].mean():.1f} us '
                  f'work<{wk[sel].mean():.1f} flush<{fl[sel].mean():.1f} meanU {U[sel].mean():.0f}')
