#!/bin/bash
# A/B the default libgbbs against build/ variants (GBBS_LIB) on a few configs
CFG=${CFG:-c2,c4}
ALG=${ALG:-bfs,bf,wbfs}
for L in paper_1805_05208_b200/libgbbs.so build/libgbbs_*.so; do
  echo "== $L"
  GBBS_LIB=$L timeout 300 python tools/probe.py --configs $CFG --algos $ALG --nsrc 1 2>&1 | grep -E "^--" | sed 's/rounds=.*kernel=/kernel=/'
done
