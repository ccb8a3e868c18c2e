set -u
OUT=gpurun_out; mkdir -p $OUT
export PYTHONUNBUFFERED=1
python -m paper_2304_06835_b200._build > $OUT/build_v.log 2>&1
timeout 900 python tools/bench_configs.py --only C1,C2-adaptive,tight,C3,stiff > $OUT/configs_v.jsonl 2> $OUT/configs_v.err
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/pytest_v.log 2>&1; echo rc=$? >> $OUT/pytest_v.log
