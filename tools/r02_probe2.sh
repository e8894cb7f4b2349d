set -x
python build.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/par.log 2>&1
timeout 900 python tools/probe.py --configs c5 --algos bfs --nsrc 3 --reps 3 --check > gpurun_out/probe_c5.log 2>&1
timeout 900 python tools/probe.py --configs c5 --algos bfs --nsrc 3 --reps 3 --rules 1 > gpurun_out/probe_c5_paper.log 2>&1
timeout 900 python tools/probe.py --configs c4,c2 --algos bfs --nsrc 2 --reps 3 --check > gpurun_out/probe_c4c2.log 2>&1
echo DONE
