#!/bin/bash
# ncu full captures of the non-headline kernels.
# Usage: bash tools/gpu_prof.sh TAG [CASE:KERNEL_REGEX ...]   (default: c2a, c3, c4)
set -u
TAG=${1:-p}
shift || true
CASES=${@:-"c2a:adaptive_static c3:adaptive_static c4:em_kernel"}
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2304_06835_b200._build > $OUT/build_$TAG.log 2>&1
for cs in $CASES; do
  name=${cs%%:*}; kern=${cs#*:}
  timeout 600 ncu --set full --metrics $(python tools/ncu_summary.py metrics) --clock-control none --import-source on \
    -k regex:$kern -s 1 -c 1 \
    -o $OUT/prof_${name}_$TAG -f python tools/prof_one.py $name > $OUT/ncu_${name}_$TAG.log 2>&1
done
echo done
