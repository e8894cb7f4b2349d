# A/B of variant builds (GBBS_LIB) on c5 / c4 BFS: per-round probe, 3 sources
set -x
python build.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/par.log 2>&1; tail -2 gpurun_out/par.log
for v in default $AB_VARIANTS; do
  if [ $v = default ]; then L=""; else L=build/libgbbs_$v.so; fi
  GBBS_LIB=$L timeout 900 python tools/probe.py --configs c5,c4 --algos bfs --nsrc 3 --reps 5 > gpurun_out/ab_$v.log 2>&1
  grep -h "^-- " gpurun_out/ab_$v.log
done
echo DONE
