for L in paper_1805_05208_b200/libgbbs.so build/libgbbs_sw8.so build/libgbbs_sw16.so; do
  echo "== $L"; GBBS_LIB=$L TEAMS=8 timeout 300 python tools/teams_probe.py c2 2>&1 | grep "bfs"
done
