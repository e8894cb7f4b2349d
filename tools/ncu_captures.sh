# Full ncu captures of the main kernels (one call per group; gpurun returns <= 64 MiB):
#   bash tools/ncu_captures.sh weighted   # BF, widest path, wBFS on c2
#   bash tools/ncu_captures.sh other      # BC on c2, BFS on c5
set -x
if [ "$1" = "weighted" ]; then
for A in bf wp wbfs; do
  python tools/one.py --config c2 --algo $A --reps 3 > gpurun_out/plain_$A.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"traverse_kernel|wbfs_kernel" -s 2 -c 1 -o gpurun_out/r01_c2_$A python tools/one.py --config c2 --algo $A --reps 3 > gpurun_out/ncu_$A.log 2>&1
done
else
python tools/bc_probe.py > gpurun_out/plain_bc.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:bc_kernel -s 2 -c 1 -o gpurun_out/r01_c2_bc python tools/bc_probe.py > gpurun_out/ncu_bc.log 2>&1
python tools/one.py --config c5 --algo bfs --reps 3 > gpurun_out/plain_c5.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:traverse_kernel -s 2 -c 1 -o gpurun_out/r01_c5_bfs python tools/one.py --config c5 --algo bfs --reps 3 > gpurun_out/ncu_c5.log 2>&1
fi

# summaries on the box (reports are too large to bring back together)
for R in gpurun_out/r01_*.ncu-rep; do
  python tools/summarize_ncu.py full $R "$(basename $R .ncu-rep)" > ${R%.ncu-rep}_summary.txt 2>&1
done
rm -f gpurun_out/r01_*.ncu-rep
echo CAPSDONE
