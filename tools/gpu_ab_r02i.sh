set -u
OUT=gpurun_out; mkdir -p $OUT
export PYTHONUNBUFFERED=1
rm -f $OUT/parity_rates_r02i.jsonl
PARITY_LOG=$OUT/parity_rates_r02i.jsonl timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu_r02i.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu_r02i.log
python tools/ab_variants.py c3,c3r5,c3r4,orego,orego4,orego5,hires,hires5,pollu,pollu5,c1t,t9,c2a base prev > $OUT/ab_r02i.jsonl 2>&1
timeout 600 ncu --set full --metrics $(python tools/ncu_summary.py metrics) --import-source on --clock-control none \
  -k regex:ros23_static -s 1 -c 1 -o $OUT/prof_c3_r02i -f python tools/prof_one.py c3 > $OUT/ncu_c3_r02i.log 2>&1
timeout 600 ncu --set full --metrics $(python tools/ncu_summary.py metrics) --import-source on --clock-control none \
  -k regex:adaptive_static -s 1 -c 1 -o $OUT/prof_c3r5_r02i -f python tools/prof_one.py c3r5 > $OUT/ncu_c3r5_r02i.log 2>&1
echo done
