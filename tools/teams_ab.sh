# A/B the default libgbbs against build/ variants on the teams batch (dev tool)
for L in paper_1805_05208_b200/libgbbs.so build/libgbbs_*.so; do
  echo "== $L"; GBBS_LIB=$L ALGOS=${ALGOS:-bfs} TEAMS=${TEAMS:-8} timeout 300 python tools/teams_probe.py ${CFG:-c2} 2>&1 | grep -v "^$"
done
