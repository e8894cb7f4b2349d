set -x
AB_VARIANTS="pni tni ptni" AB_BF=1 bash tools/r02_ab.sh
