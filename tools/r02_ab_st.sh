# A/B: store policy of the acquisitions' dist/parent writes (GBBS_STATE_ST 0/1/2)
set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for v in default $AB_VARIANTS; do
  if [ $v = default ]; then L=""; else L=build/libgbbs_$v.so; fi
  GBBS_LIB=$L timeout 900 python tools/probe.py --configs c5 --algos bfs --nsrc 8 --reps 3 > gpurun_out/ab_$v.log 2>&1
  GBBS_LIB=$L timeout 900 python tools/probe.py --configs c4,c2,c3 --algos bfs --nsrc 2 --reps 3 > gpurun_out/ab2_$v.log 2>&1
  grep -h "^-- " gpurun_out/ab_$v.log gpurun_out/ab2_$v.log | awk '{print $2, $3, $9}'
  GBBS_LIB=$L timeout 600 ncu --metrics $M --clock-control none -k regex:traverse_kernel -s 2 -c 1 --csv python tools/one.py --config c5 --algo bfs --reps 3 --src 1 > gpurun_out/abncu_$v.csv 2>&1
  grep -E "dram__bytes|gpu__time" gpurun_out/abncu_$v.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
echo DONE
