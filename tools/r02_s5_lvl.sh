# session 5: byte levels — parity (parity file + c3/c5 full-size checks) and A/B against GBBS_BFS_LVL=0
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s5_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/s5_parity.log
AB_VARIANTS="$AB_VARIANTS" bash tools/r02_ab.sh
python tools/ab_summary.py default $AB_VARIANTS > gpurun_out/s5_ab_summary.txt 2>&1
tail -12 gpurun_out/s5_ab_summary.txt
