# A/B of variant builds (build/libgbbs_<v>.so via GBBS_LIB): per-source kernel times
# on c5 (8 sources) and c4/c2/c3 BFS; AB_BF=1 adds c4/c2 Bellman-Ford
set -x
for v in default $AB_VARIANTS; do
  if [ $v = default ]; then L=""; else L=build/libgbbs_$v.so; fi
  GBBS_LIB=$L timeout 900 python tools/probe.py --configs c5 --algos bfs --nsrc 8 --reps 3 $AB_ARGS > gpurun_out/ab_$v.log 2>&1
  GBBS_LIB=$L timeout 900 python tools/probe.py --configs c4,c2,c3,c1 --algos bfs --nsrc 2 --reps 3 $AB_ARGS > gpurun_out/ab2_$v.log 2>&1
  if [ -n "$AB_BF" ]; then GBBS_LIB=$L timeout 900 python tools/probe.py --configs c4,c2,c3 --algos bf --nsrc 2 --reps 3 > gpurun_out/ab3_$v.log 2>&1; fi
done
echo DONE
