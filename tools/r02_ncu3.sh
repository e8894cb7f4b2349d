set -x
python build.py > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:traverse_kernel -s 2 -c 1 -o gpurun_out/r02_c5s4_bfs python tools/one.py --config c5 --algo bfs --reps 3 --src 4 > gpurun_out/ncu_c5s4.log 2>&1
python tools/summarize_ncu.py full gpurun_out/r02_c5s4_bfs.ncu-rep r02_c5s4_bfs > gpurun_out/r02_c5s4_bfs_summary.txt 2>&1
ncu -i gpurun_out/r02_c5s4_bfs.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/r02_c5s4_source.csv 2>/dev/null; gzip -f gpurun_out/r02_c5s4_source.csv
rm -f gpurun_out/*.ncu-rep
echo DONE
