set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wbfs.py tests/test_gpu_csc.py -x -q > gpurun_out/par.log 2>&1; tail -2 gpurun_out/par.log
AB_VARIANTS="us" AB_BF=1 bash tools/r02_ab.sh
echo DONE
