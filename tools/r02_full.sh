# round-2 GPU pass: tests, bench (default = c5 headline + c4 BF leg), launch list
set -x
python build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python -m pytest tests -m "not gpu" -x -q -k "abi" > gpurun_out/abi.log 2>&1
echo DONE
