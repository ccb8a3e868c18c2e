set -u
OUT=gpurun_out; mkdir -p $OUT
for U in 2 5 10 20; do
  touch paper_2304_06835_b200/csrc/common.cuh
  NVCC_APPEND_FLAGS="-DENS_PARTIAL_UNROLL=$U" python -m paper_2304_06835_b200._build > $OUT/build_pu_$U.log 2>&1 || { echo BUILD $U FAILED; continue; }
  timeout 600 python tools/bench_configs.py --only stiff-pollu,stiff-rodas4-pollu,stiff-rodas5-pollu > $OUT/configs_pu_$U.jsonl 2>> $OUT/configs_pu.err
done
