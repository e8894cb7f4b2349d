set -x
python build.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/par.log 2>&1
timeout 900 python tools/probe.py --configs c5 --algos bfs --nsrc 3 --reps 5 --check > gpurun_out/probe_c5.log 2>&1
timeout 900 python tools/probe.py --configs c5 --algos bfs --nsrc 3 --reps 5 --noparent > gpurun_out/probe_c5_nopar.log 2>&1
GBBS_LIB=build/libgbbs_nostate.so timeout 900 python tools/probe.py --configs c5 --algos bfs --nsrc 3 --reps 5 > gpurun_out/probe_c5_nostate.log 2>&1
timeout 900 python tools/probe.py --configs c4,c2 --algos bfs --nsrc 2 --reps 5 --check > gpurun_out/probe_c4c2.log 2>&1
python tools/one.py --config c5 --algo bfs --reps 3 > gpurun_out/plain_c5.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:traverse_kernel -s 2 -c 1 -o gpurun_out/r02_c5_bfs python tools/one.py --config c5 --algo bfs --reps 3 > gpurun_out/ncu_c5.log 2>&1
python tools/summarize_ncu.py full gpurun_out/r02_c5_bfs.ncu-rep r02_c5_bfs > gpurun_out/r02_c5_bfs_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/r02_c5_bfs.ncu-rep 40 > gpurun_out/r02_c5_bfs_lines.txt 2>&1
rm -f gpurun_out/*.ncu-rep
echo DONE
