#!/bin/bash
# A/B session: GPU tests (optional) + tools/ab_variants.py. Usage: bash tools/gpu_ab.sh TAG CONFIGS VARIANTS... (TESTS=1 to run pytest -m gpu first)
set -u
TAG=$1; CFGS=$2; shift 2
OUT=gpurun_out
mkdir -p $OUT
export PYTHONUNBUFFERED=1
if [ "${TESTS:-0}" = "1" ]; then
  PARITY_LOG=$OUT/parity_rates_$TAG.jsonl timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/pytest_gpu_$TAG.log 2>&1
  echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
fi
timeout 1500 python tools/ab_variants.py $CFGS "$@" > $OUT/ab_$TAG.jsonl 2> $OUT/ab_$TAG.err
echo done
