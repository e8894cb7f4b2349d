set -x
python build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sbf.py tests/test_gpu_parity.py -x -q > gpurun_out/par.log 2>&1; tail -2 gpurun_out/par.log
timeout 900 python -m pytest tests/test_gpu_full.py -x -q -k "planted" > gpurun_out/planted.log 2>&1; tail -2 gpurun_out/planted.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
echo DONE
