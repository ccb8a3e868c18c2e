set -u
OUT=gpurun_out; mkdir -p $OUT
export PYTHONUNBUFFERED=1
python tools/ab_variants.py c3,c3r5,c3r4,orego,orego4,orego5 base prev > $OUT/ab_r02g.jsonl 2>&1
echo done
