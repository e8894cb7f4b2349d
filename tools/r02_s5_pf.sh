# session 5: latency prefetches A/B; bounds-checked build on the new code
set -x
AB_VARIANTS="$AB_VARIANTS" bash tools/r02_ab.sh
python tools/ab_summary.py default $AB_VARIANTS > gpurun_out/s5_ab_pf.txt; cat gpurun_out/s5_ab_pf.txt
GBBS_LIB=build/libgbbs_checks.so timeout 1500 python -m pytest tests/test_gpu_levels.py tests/test_gpu_parity.py tests/test_gpu_full.py -x -q > gpurun_out/s5_checks.log 2>&1; echo "checks rc=$?"; tail -3 gpurun_out/s5_checks.log
