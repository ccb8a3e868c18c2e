set -u
OUT=gpurun_out; mkdir -p $OUT
export PYTHONUNBUFFERED=1
python -m paper_2304_06835_b200._build > $OUT/build_s.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fused_stats.py tests/test_gpu_multi_solve.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_peer_gather.py tests/test_multi_gpu_nccl.py -m gpu -q -p no:cacheprovider > $OUT/pytest_s.log 2>&1; echo rc=$? >> $OUT/pytest_s.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_s.json 2> $OUT/bench_s.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_s.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-also > $OUT/ncu_launch_s.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29557 bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --no-cpu-baseline --no-also > $OUT/bench_gloo2_s.json 2> $OUT/bench_gloo2_s.err
