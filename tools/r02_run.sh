set -x
AB_VARIANTS="g2 vin2 us" bash tools/r02_ab.sh
echo DONE
