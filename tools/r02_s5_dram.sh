# session 5: ncu DRAM bytes + duration of every c5 BFS source (one launch each), final code
set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for s in 0 1 2 3 4 5 6 7; do
timeout 600 ncu --metrics $M --clock-control none -k regex:traverse_kernel -s 2 -c 1 --csv python tools/one.py --config c5 --algo bfs --reps 3 --src $s > gpurun_out/dram_c5_s$s.csv 2>&1
done
echo DONE
