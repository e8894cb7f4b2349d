# session 5: what the state traffic costs on c5 (diagnostic builds, results invalid)
set -x
for v in default $AB_VARIANTS; do
  if [ $v = default ]; then L=""; else L=build/libgbbs_$v.so; fi
  GBBS_LIB=$L timeout 900 python tools/probe.py --configs c5 --algos bfs --nsrc 8 --reps 3 --rounds > gpurun_out/ab_$v.log 2>&1
done
python tools/ab_summary.py default $AB_VARIANTS > gpurun_out/s5_diag_summary.txt 2>&1
tail -12 gpurun_out/s5_diag_summary.txt
