set -u
OUT=gpurun_out; mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/pytest_gpu_r02f.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu_r02f.log
python tools/ab_variants.py c3,c3r5,orego,hires,pollu,c1t base prev m3 > $OUT/ab_r02f.jsonl 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ros23_static -s 1 -c 1 -o $OUT/prof_c3_r02f -f \
  python tools/prof_one.py c3 > $OUT/ncu_c3_r02f.log 2>&1
echo done
