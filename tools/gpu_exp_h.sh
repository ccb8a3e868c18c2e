set -u
OUT=gpurun_out; mkdir -p $OUT
export PYTHONUNBUFFERED=1
python -m paper_2304_06835_b200._build > $OUT/build_h.log 2>&1
timeout 600 python tools/bench_configs.py --only stiff > $OUT/configs_h.jsonl 2> $OUT/configs_h.err
timeout 900 python -m pytest tests/test_gpu_stiff.py tests/test_gpu_rodas4.py tests/test_gpu_rodas5.py -m gpu -q -p no:cacheprovider -x > $OUT/pytest_gpu_h.log 2>&1; echo rc=$? >> $OUT/pytest_gpu_h.log
