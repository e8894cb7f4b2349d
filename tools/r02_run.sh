set -x
AB_VARIANTS="pch3" bash tools/r02_ab.sh
echo DONE
