set -u
OUT=gpurun_out; mkdir -p $OUT
python -m paper_2304_06835_b200._build > $OUT/build_q.log 2>&1
timeout 300 python tools/bench_configs.py --only C4 > $OUT/configs_q_base.jsonl 2> $OUT/configs_q.err
ENS_TUNE_EM_B4=1 timeout 300 python tools/bench_configs.py --only C4 > $OUT/configs_q_b4.jsonl 2>> $OUT/configs_q.err
