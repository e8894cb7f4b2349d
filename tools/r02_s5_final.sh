# round-2 session-5 final-code pass: gpu tests, bench, launch list, all-config results, ncu full of c5 source 1
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-legs > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
timeout 1500 python tools/results_table.py > gpurun_out/results_all.jsonl 2> gpurun_out/results_all.err; echo "rt rc=$?"
bash tools/r02_ncu_s1.sh
echo DONE
