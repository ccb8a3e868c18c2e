#!/bin/bash
# ncu full captures of the non-headline kernels. Usage: bash tools/gpu_prof.sh TAG
set -u
TAG=${1:-p}
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2304_06835_b200._build > $OUT/build_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adaptive_static -s 1 -c 1 -o $OUT/prof_c2a_$TAG -f python tools/prof_one.py c2a > $OUT/ncu_c2a_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adaptive_static -s 1 -c 1 -o $OUT/prof_c3_$TAG -f python tools/prof_one.py c3 > $OUT/ncu_c3_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:em_kernel -s 1 -c 1 -o $OUT/prof_c4_$TAG -f python tools/prof_one.py c4 > $OUT/ncu_c4_$TAG.log 2>&1
echo done
