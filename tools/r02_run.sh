# round-2 final-code pass: gpu tests, bench, launch list, all-config results, ncu full (c5 s1, c4 BF), DRAM per source
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-legs > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
timeout 1500 python tools/results_table.py > gpurun_out/results_all.jsonl 2> gpurun_out/results_all.err; echo "rt rc=$?"
bash tools/r02_ncu_s1.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:traverse_kernel -s 1 -c 1 -o gpurun_out/r02_c4_bf python tools/one.py --config c4 --algo bf --reps 2 > gpurun_out/ncu_c4bf.log 2>&1
python tools/summarize_ncu.py full gpurun_out/r02_c4_bf.ncu-rep r02_c4_bf > gpurun_out/r02_c4_bf_summary.txt 2>&1
ncu -i gpurun_out/r02_c4_bf.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/r02_c4_bf_source.csv 2>/dev/null; gzip -f gpurun_out/r02_c4_bf_source.csv
rm -f gpurun_out/*.ncu-rep
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for s in 0 1 2 3 4 5 6 7; do
timeout 600 ncu --metrics $M --clock-control none -k regex:traverse_kernel -s 2 -c 1 --csv python tools/one.py --config c5 --algo bfs --reps 3 --src $s > gpurun_out/dram_c5_s$s.csv 2>&1
done
for s in 0 1 2 3; do
timeout 600 ncu --metrics $M --clock-control none -k regex:traverse_kernel -s 1 -c 1 --csv python tools/one.py --config c4 --algo bf --reps 2 --src $s > gpurun_out/dram_c4bf_s$s.csv 2>&1
done
echo DONE
