set -u
OUT=gpurun_out; mkdir -p $OUT
python -m paper_2304_06835_b200._build > $OUT/build_x.log 2>&1
timeout 300 python tools/bench_configs.py --only C1,C2-adaptive,tight-tsit5 > $OUT/configs_x_base.jsonl 2> $OUT/configs_x.err
ENS_TUNE_UNROLL2=1 timeout 300 python tools/bench_configs.py --only C1,C2-adaptive,tight-tsit5 > $OUT/configs_x_u2.jsonl 2>> $OUT/configs_x.err
