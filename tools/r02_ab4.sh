set -x
python build.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/par.log 2>&1; tail -2 gpurun_out/par.log
for v in default $AB_VARIANTS; do
  if [ $v = default ]; then L=""; else L=build/libgbbs_$v.so; fi
  GBBS_LIB=$L timeout 900 python tools/probe.py --configs c5 --algos bfs --nsrc 8 --reps 3 > gpurun_out/ab_$v.log 2>&1
  GBBS_LIB=$L timeout 900 python tools/probe.py --configs c4,c2 --algos bfs --nsrc 2 --reps 3 > gpurun_out/ab2_$v.log 2>&1
  grep -h "^-- " gpurun_out/ab_$v.log gpurun_out/ab2_$v.log | awk '{print $2, $3, $9}'
done
echo DONE
