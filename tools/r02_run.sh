set -x
timeout 600 python -m pytest tests/test_gpu_csc.py -x -q > gpurun_out/csc.log 2>&1; tail -3 gpurun_out/csc.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest.log
bash tools/r02_ncu_s1.sh
echo DONE
