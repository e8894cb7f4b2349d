# ncu --set full of the c5 BFS traversal from source index 1 (dense-pull dominated)
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:traverse_kernel -s 2 -c 1 -o gpurun_out/r02_c5s1_bfs python tools/one.py --config c5 --algo bfs --reps 3 --src 1 > gpurun_out/ncu_c5s1.log 2>&1
python tools/summarize_ncu.py full gpurun_out/r02_c5s1_bfs.ncu-rep r02_c5s1_bfs > gpurun_out/r02_c5s1_bfs_summary.txt 2>&1
ncu -i gpurun_out/r02_c5s1_bfs.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/r02_c5s1_bfs_source.csv 2>/dev/null; gzip -f gpurun_out/r02_c5s1_bfs_source.csv
ncu -i gpurun_out/r02_c5s1_bfs.ncu-rep --page raw --csv > gpurun_out/r02_c5s1_bfs_raw.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
echo DONE
