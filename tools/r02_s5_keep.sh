# session 5: L2 priority of the records the phased pull re-reads + unit size; DRAM bytes of source 1
set -x
AB_VARIANTS="$AB_VARIANTS" bash tools/r02_ab.sh
python tools/ab_summary.py default $AB_VARIANTS > gpurun_out/s5_ab_keep.txt
cat gpurun_out/s5_ab_keep.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for v in $AB_VARIANTS; do
GBBS_LIB=build/libgbbs_$v.so timeout 600 ncu --metrics $M --clock-control none -k regex:traverse_kernel -s 2 -c 1 --csv python tools/one.py --config c5 --algo bfs --reps 3 --src 1 > gpurun_out/dram_c5_s1_$v.csv 2>&1
tail -3 gpurun_out/dram_c5_s1_$v.csv
done
