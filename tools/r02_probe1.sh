set -x
python build.py > gpurun_out/build.log 2>&1
timeout 900 python tools/probe.py --configs c5 --algos bfs --nsrc 3 --reps 3 > gpurun_out/probe_c5.log 2>&1
timeout 900 python tools/probe.py --configs c4 --algos bfs,bf --nsrc 1 --reps 3 > gpurun_out/probe_c4.log 2>&1
timeout 600 python tools/probe.py --configs c3 --algos bfs,bf --nsrc 1 --reps 3 > gpurun_out/probe_c3.log 2>&1
echo DONE
