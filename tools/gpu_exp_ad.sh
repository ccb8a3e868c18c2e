set -u
OUT=gpurun_out; mkdir -p $OUT
for U in 1 2 4 5 20; do
  touch paper_2304_06835_b200/csrc/ad.cuh
  NVCC_APPEND_FLAGS="-DENS_AD_PASS=$U" python -m paper_2304_06835_b200._build > $OUT/build_ad_$U.log 2>&1 || { echo BUILD $U FAILED; continue; }
  timeout 600 python tools/bench_configs.py --only stiff-pollu,stiff-rodas4-pollu,stiff-rodas5-pollu,stiff-hires,stiff-rodas4-hires,stiff-rodas5-hires > $OUT/configs_ad_$U.jsonl 2>> $OUT/configs_ad.err
done
