set -u
OUT=gpurun_out; mkdir -p $OUT
export PYTHONUNBUFFERED=1
python tools/ab_variants.py c3 base old minb2 loop loop2 vote evl > $OUT/ab_c3_r02d.jsonl 2>&1
python tools/ab_variants.py c3r5,c1t,t9,orego,hires,c2a base old evl > $OUT/ab_misc_r02d.jsonl 2>&1
for v in base evl; do
  lib=""; [ $v != base ] && lib="--lib=paper_2304_06835_b200/_variants/$v/libens.so"
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:adaptive_static -s 1 -c 1 python tools/prof_one.py c3 $lib > $OUT/ncu_dram_c3_${v}_r02d.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:adaptive_static -s 1 -c 1 python tools/prof_one.py c3r5 $lib > $OUT/ncu_dram_c3r5_${v}_r02d.log 2>&1
done
echo done
