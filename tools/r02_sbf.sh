set -x
python build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sbf.py tests/test_gpu_parity.py -x -q > gpurun_out/par.log 2>&1; tail -2 gpurun_out/par.log
timeout 900 python -m pytest tests/test_gpu_full.py -x -q -k "planted or signed" > gpurun_out/planted.log 2>&1; tail -2 gpurun_out/planted.log
for v in default $AB_VARIANTS; do
  if [ $v = default ]; then L=""; else L=build/libgbbs_$v.so; fi
  GBBS_LIB=$L timeout 900 python tools/probe.py --configs c4,c2,c3 --algos bf --nsrc 2 --reps 3 > gpurun_out/abbf_$v.log 2>&1
  grep -h "^-- " gpurun_out/abbf_$v.log | awk '{print $2, $3, $9, $NF}'
done
echo DONE
