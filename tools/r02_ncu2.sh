set -x
python build.py > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:traverse_kernel -s 1 -c 1 -o gpurun_out/r02_c4_bf python tools/one.py --config c4 --algo bf --reps 2 > gpurun_out/ncu_c4bf.log 2>&1
python tools/summarize_ncu.py full gpurun_out/r02_c4_bf.ncu-rep r02_c4_bf > gpurun_out/r02_c4_bf_summary.txt 2>&1
ncu -i gpurun_out/r02_c4_bf.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/r02_c4_bf_source.csv 2>/dev/null; gzip -f gpurun_out/r02_c4_bf_source.csv
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for s in 0 1 2; do
timeout 600 ncu --metrics $M --clock-control none -k regex:traverse_kernel -s 2 -c 1 --csv python tools/one.py --config c5 --algo bfs --reps 3 --src $s > gpurun_out/dram_c5_s$s.csv 2>&1
done
rm -f gpurun_out/*.ncu-rep
echo DONE
