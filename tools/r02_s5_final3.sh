# round-2 session-5 final pass on the rec8 code: tests, smoke, bench, launch list, results, ncu full (c5 s1), DRAM per source
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
bash tools/r02_s5_dram.sh
python tools/mk_traffic.py > gpurun_out/mk_traffic.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-legs > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
timeout 1500 python tools/results_table.py > gpurun_out/results_all.jsonl 2> gpurun_out/results_all.err; echo "rt rc=$?"
bash tools/r02_ncu_s1.sh
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
echo DONE
