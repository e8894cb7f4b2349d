# session 5: cold pull record as one 256-bit load — parity + A/B
set -x
GBBS_LIB=build/libgbbs_ld256.so timeout 900 python -m pytest tests/test_gpu_levels.py tests/test_gpu_parity.py -x -q > gpurun_out/s5_ld256_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/s5_ld256_parity.log
AB_VARIANTS="ld256" bash tools/r02_ab.sh
python tools/ab_summary.py default ld256 > gpurun_out/s5_ab_ld256.txt; cat gpurun_out/s5_ab_ld256.txt
