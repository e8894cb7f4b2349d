set -x
python build.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/par.log 2>&1; tail -2 gpurun_out/par.log
for v in default $AB_VARIANTS; do
  if [ $v = default ]; then L=""; else L=build/libgbbs_$v.so; fi
  GBBS_LIB=$L timeout 900 python tools/probe.py --configs c5,c4 --algos bfs --nsrc 3 --reps 5 > gpurun_out/ab_$v.log 2>&1
  grep -h "^-- " gpurun_out/ab_$v.log
done
timeout 600 python tools/probe.py --configs c5 --algos bfs --nsrc 3 --reps 1 --check > gpurun_out/check_c5.log 2>&1; grep certif gpurun_out/check_c5.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:traverse_kernel -s 2 -c 1 -o gpurun_out/r02_c5s2_bfs python tools/one.py --config c5 --algo bfs --reps 3 --src 2 > gpurun_out/ncu_c5s2.log 2>&1
python tools/summarize_ncu.py full gpurun_out/r02_c5s2_bfs.ncu-rep r02_c5s2_bfs > gpurun_out/r02_c5s2_bfs_summary.txt 2>&1
ncu -i gpurun_out/r02_c5s2_bfs.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/r02_c5s2_source.csv 2>/dev/null; gzip -f gpurun_out/r02_c5s2_source.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:traverse_kernel -s 2 -c 1 -o gpurun_out/r02_c5s1_bfs python tools/one.py --config c5 --algo bfs --reps 3 --src 1 > gpurun_out/ncu_c5s1.log 2>&1
python tools/summarize_ncu.py full gpurun_out/r02_c5s1_bfs.ncu-rep r02_c5s1_bfs > gpurun_out/r02_c5s1_bfs_summary.txt 2>&1
ncu -i gpurun_out/r02_c5s1_bfs.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/r02_c5s1_source.csv 2>/dev/null; gzip -f gpurun_out/r02_c5s1_source.csv
rm -f gpurun_out/*.ncu-rep
echo DONE
