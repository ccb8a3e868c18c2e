set -u
OUT=gpurun_out; mkdir -p $OUT
export PYTHONUNBUFFERED=1
python tools/ab_variants.py c2a base pair1 pair3 > $OUT/ab_c2a_r02e.jsonl 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pair -s 1 -c 1 -o $OUT/prof_pair1_r02e -f \
  python tools/prof_one.py c2a --lib=paper_2304_06835_b200/_variants/pair1/libens.so > $OUT/ncu_pair1_r02e.log 2>&1
echo done
