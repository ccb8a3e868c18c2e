set -u
OUT=gpurun_out; mkdir -p $OUT
export PYTHONUNBUFFERED=1
python -m paper_2304_06835_b200._build > $OUT/build_n.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fast_paths.py tests/test_gpu_parity.py tests/test_gpu_host_sde.py tests/test_gpu_siea.py tests/test_gpu_weak_order.py -m gpu -q -p no:cacheprovider > $OUT/pytest_n.log 2>&1; echo rc=$? >> $OUT/pytest_n.log
timeout 600 python tools/bench_configs.py --only C4,CRN > $OUT/configs_n.jsonl 2> $OUT/configs_n.err
