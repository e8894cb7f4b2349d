set -x
timeout 900 python -m pytest tests/test_gpu_levels.py tests/test_gpu_parity.py -x -q > gpurun_out/s5_parity.log 2>&1; echo "parity rc=$?"; tail -15 gpurun_out/s5_parity.log
AB_VARIANTS="$AB_VARIANTS" bash tools/r02_ab.sh
python tools/ab_summary.py default $AB_VARIANTS > gpurun_out/s5_ab_summary.txt 2>&1
tail -8 gpurun_out/s5_ab_summary.txt
