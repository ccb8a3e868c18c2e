#!/bin/bash
# All BASELINE configs at full size + distributed code path (world=1 NCCL) + reference arm + smoke.
set -u
TAG=${1:-cfg}
OUT=gpurun_out
mkdir -p $OUT
export PYTHONUNBUFFERED=1
python -m paper_2304_06835_b200._build > $OUT/build_$TAG.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "rc=$?" >> $OUT/smoke_$TAG.log
timeout 1200 python tools/bench_configs.py > $OUT/configs_$TAG.jsonl 2> $OUT/configs_$TAG.err; echo "rc=$?" >> $OUT/configs_$TAG.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_torchrun1_$TAG.json 2> $OUT/bench_torchrun1_$TAG.err
echo "rc=$?" >> $OUT/bench_torchrun1_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
echo "rc=$?" >> $OUT/bench_ref_$TAG.err
timeout 600 python bench.py --dtype f64 --no-cpu-baseline > $OUT/bench_f64_$TAG.json 2> $OUT/bench_f64_$TAG.err
echo done
