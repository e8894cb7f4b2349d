# session 5: 8-byte hot / 32-byte cold pull records (GBBS_REC8) — parity, A/B, DRAM bytes of c5 source 1
set -x
GBBS_LIB=build/libgbbs_rec8.so timeout 900 python -m pytest tests/test_gpu_levels.py tests/test_gpu_parity.py -x -q > gpurun_out/s5_rec8_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/s5_rec8_parity.log
AB_VARIANTS="rec8" bash tools/r02_ab.sh
python tools/ab_summary.py default rec8 > gpurun_out/s5_ab_rec8.txt; cat gpurun_out/s5_ab_rec8.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
GBBS_LIB=build/libgbbs_rec8.so timeout 600 ncu --metrics $M --clock-control none -k regex:traverse_kernel -s 2 -c 1 --csv python tools/one.py --config c5 --algo bfs --reps 3 --src 1 > gpurun_out/dram_c5_s1_rec8.csv 2>&1
tail -3 gpurun_out/dram_c5_s1_rec8.csv
