# One GPU call: build, smoke, the whole -m gpu suite, the default bench, the ncu
# launch list of the bench command, full ncu captures of the bench's dominant
# kernel (traverse_mg_kernel<BFS>, 8 c2 traversals per launch) and of one c2
# traversal (traverse_kernel<BFS>), summarised on the box, and the all-config
# results table (outputs under gpurun_out/).
set -x
python build.py > gpurun_out/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE_EXIT $? >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo BENCH_EXIT $? >> gpurun_out/bench.err
timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/b2.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
python tools/one_batch.py --config c2 --reps 3 > gpurun_out/plain_mg.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:traverse_mg_kernel -s 2 -c 1 -o gpurun_out/r01_c2_bfs_mg python tools/one_batch.py --config c2 --reps 3 > gpurun_out/ncu_mg.log 2>&1
python tools/one.py --config c2 --algo bfs --reps 4 > gpurun_out/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:traverse_kernel -s 3 -c 1 -o gpurun_out/r01_c2_bfs python tools/one.py --config c2 --algo bfs --reps 4 > gpurun_out/ncu_full.log 2>&1
for R in gpurun_out/r01_*.ncu-rep; do
  python tools/summarize_ncu.py full $R "$(basename $R .ncu-rep)" > ${R%.ncu-rep}_summary.txt 2>&1
done
rm -f gpurun_out/r01_*.ncu-rep
timeout 1500 python tools/results_table.py > gpurun_out/results.jsonl 2> gpurun_out/results.err
echo ALLDONE
