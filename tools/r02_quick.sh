# quick A/B pass: parity suite, per-round probe on c5 (3 sources) and c4/c2 BFS
set -x
python build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/par.log 2>&1; tail -3 gpurun_out/par.log
timeout 900 python tools/probe.py --configs c5 --algos bfs --nsrc 3 --reps 5 --check > gpurun_out/q_c5.log 2>&1
timeout 900 python tools/probe.py --configs c4,c2 --algos bfs --nsrc 2 --reps 5 --check > gpurun_out/q_c4c2.log 2>&1
grep -h "^-- " gpurun_out/q_c5.log gpurun_out/q_c4c2.log
echo DONE
