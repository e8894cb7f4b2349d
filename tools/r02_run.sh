set -x
AB_VARIANTS="pfw" AB_BF=1 bash tools/r02_ab.sh
echo DONE
