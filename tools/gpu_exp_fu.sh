set -u
OUT=gpurun_out; mkdir -p $OUT
python -m paper_2304_06835_b200._build > $OUT/build_fu.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python tools/bench_configs.py --only stiff,C3 > $OUT/configs_fu.jsonl 2> $OUT/configs_fu.err
timeout 900 python -m pytest tests/test_gpu_stiff.py tests/test_gpu_rodas4.py tests/test_gpu_rodas5.py tests/test_gpu_failure_paths.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > $OUT/pytest_fu.log 2>&1; echo rc=$? >> $OUT/pytest_fu.log
