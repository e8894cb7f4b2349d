# DRAM attribution of the c5 BFS traversal: variants that skip the dist/parent
# fill (NOINIT) and/or the acquisitions' scattered state writes (NOSTATE); results
# of those builds are invalid by design — only their time and DRAM bytes matter.
set -x
python build.py > gpurun_out/build.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for v in default nostate noinit nostinit; do
  if [ $v = default ]; then L=""; else L=build/libgbbs_$v.so; fi
  for np in "" "--noparent"; do
    GBBS_LIB=$L timeout 600 python tools/one.py --config c5 --algo bfs --reps 4 $np > gpurun_out/attr_${v}${np}.log 2>&1
    GBBS_LIB=$L timeout 600 ncu --metrics $M --clock-control none -k regex:traverse_kernel -s 2 -c 1 --csv python tools/one.py --config c5 --algo bfs --reps 3 $np > gpurun_out/attr_ncu_${v}${np}.csv 2>&1
  done
done
timeout 900 python tools/probe.py --configs c5 --algos bfs --nsrc 2 --reps 3 --rounds > gpurun_out/probe_c5.log 2>&1
echo DONE
