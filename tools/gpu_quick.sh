#!/bin/bash
# Quick GPU iteration: GPU tests + bench (+ optional ncu). Usage: bash tools/gpu_quick.sh TAG [ncu]
set -u
TAG=${1:-q}
OUT=gpurun_out
mkdir -p $OUT
export PYTHONUNBUFFERED=1
python -m paper_2304_06835_b200._build > $OUT/build_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py ${BENCH_ARGS:-} > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
echo "bench rc=$?" >> $OUT/bench_$TAG.err
if [ "${2:-}" = "ncu" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launch_$TAG.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tsit5_fixed -s 1 -c 1 \
    -o $OUT/prof_tsit5_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full_$TAG.log 2>&1
fi
echo done
