# c5: per-round probe of all 8 sources, and ncu DRAM bytes of every source's traversal
set -x
python build.py > gpurun_out/build.log 2>&1
timeout 900 python tools/probe.py --configs c5 --algos bfs --nsrc 8 --reps 3 > gpurun_out/probe_c5_all.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for s in 0 1 2 3 4 5 6 7; do
timeout 600 ncu --metrics $M --clock-control none -k regex:traverse_kernel -s 2 -c 1 --csv python tools/one.py --config c5 --algo bfs --reps 3 --src $s > gpurun_out/dram_c5_s$s.csv 2>&1
done
for s in 0 1 2 3; do
timeout 600 ncu --metrics $M --clock-control none -k regex:traverse_kernel -s 1 -c 1 --csv python tools/one.py --config c4 --algo bf --reps 2 --src $s > gpurun_out/dram_c4bf_s$s.csv 2>&1
done
echo DONE
