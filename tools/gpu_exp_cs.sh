set -u
OUT=gpurun_out; mkdir -p $OUT
python -m paper_2304_06835_b200._build > $OUT/build_cs.log 2>&1
timeout 300 python tools/bench_configs.py --only C2-saveat-dense,C2-fixed > $OUT/configs_cs_base.jsonl 2> $OUT/configs_cs.err
touch paper_2304_06835_b200/csrc/tsit5.cuh; NVCC_APPEND_FLAGS="-DENS_EXP_STCS" python -m paper_2304_06835_b200._build > $OUT/build_cs2.log 2>&1
timeout 300 python tools/bench_configs.py --only C2-saveat-dense,C2-fixed > $OUT/configs_cs_stcs.jsonl 2>> $OUT/configs_cs.err
