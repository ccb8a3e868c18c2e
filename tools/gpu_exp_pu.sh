set -u
OUT=gpurun_out; mkdir -p $OUT
python -m paper_2304_06835_b200._build > $OUT/build_ur.log 2>&1 || { echo BUILD1 FAILED; exit 1; }
timeout 600 python tools/bench_configs.py --only stiff-pollu,stiff-rodas4-pollu,stiff-rodas5-pollu > $OUT/configs_ur_base.jsonl 2> $OUT/configs_ur.err
touch paper_2304_06835_b200/csrc/common.cuh; NVCC_APPEND_FLAGS="-DENS_PARTIAL_UNROLL=4" python -m paper_2304_06835_b200._build > $OUT/build_ur2.log 2>&1 || { echo BUILD2 FAILED; exit 1; }
timeout 600 python tools/bench_configs.py --only stiff-pollu,stiff-rodas4-pollu,stiff-rodas5-pollu > $OUT/configs_ur_p4.jsonl 2>> $OUT/configs_ur.err
