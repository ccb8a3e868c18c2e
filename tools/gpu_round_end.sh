#!/bin/bash
# Full evidence refresh (one GPU session): GPU tests (with the per-test parity
# records), smoke, bench (N=1 default = C5 at 10^8, and the C2 10^7 line), the
# reference (oracle) arm, torchrun world 1, the multi-rank bench path with two
# gloo ranks sharing the one GPU, the ncu launch list of the bench command and
# one `ncu --set full` capture of the headline kernel with the executed-FLOP
# counters, plus metric-only captures of the other kernels' executed FLOPs.
# Usage (from the repo root, under gpurun): bash tools/gpu_round_end.sh TAG
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
export PYTHONUNBUFFERED=1
EXEC=$(python tools/ncu_summary.py metrics)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu_$TAG.txt 2>&1
python -m paper_2304_06835_b200._build > $OUT/build_$TAG.log 2>&1
rm -f $OUT/parity_rates_$TAG.jsonl
PARITY_LOG=$OUT/parity_rates_$TAG.jsonl timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider \
  > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1
echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
echo "bench rc=$?" >> $OUT/bench_$TAG.err
timeout 600 python bench.py --workload c2 --no-also > $OUT/bench_c2_$TAG.json 2> $OUT/bench_c2_$TAG.err
timeout 900 python bench.py --impl reference > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 > $OUT/bench_torchrun1_$TAG.json 2> $OUT/bench_torchrun1_$TAG.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29534 bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --no-also --no-e2e \
  > $OUT/bench_gloo2_$TAG.json 2> $OUT/bench_gloo2_$TAG.err
# eight gloo ranks sharing the GPU: the 8-GPU strong-scaling shard arithmetic and fused gather end to end
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
  --master-port 29535 bench.py --gpus 8 --steps 1 --warmup 3 --backend gloo --no-also --no-e2e \
  > $OUT/bench_gloo8_$TAG.json 2> $OUT/bench_gloo8_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-also > $OUT/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --metrics $EXEC --clock-control none --import-source on -k regex:tsit5_fixed -s 3 -c 1 \
  -o $OUT/prof_tsit5_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-also \
  > $OUT/ncu_full_$TAG.log 2>&1
python tools/ncu_summary.py full $OUT/prof_tsit5_$TAG.ncu-rep tsit5_fixed_lorenz_f32_$TAG 100000000 192008 \
  > /dev/null 2>&1 && cp profiles/ncu_full_tsit5_fixed_lorenz_f32_$TAG.json $OUT/
# executed-FLOP counters of the side kernels: summarised here, the ~10 MB reports are not brought back
for cs in c2f64:tsit5_fixed:10000000 c2a:static_pair_kernel:10000000 c1t:static_kernel:1000000 \
          c3:static_kernel:1000000 c3r5:static_kernel:1000000 c3r5p:static_kernel:1000000 \
          t9:static_kernel:1000000; do
  IFS=: read name kern n <<< "$cs"
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,$EXEC \
    --clock-control none -k regex:$kern -s 1 -c 1 -o $OUT/prof_exec_${name}_$TAG -f \
    python tools/prof_one.py $name > $OUT/ncu_exec_${name}_$TAG.log 2>&1
  python tools/ncu_summary.py full $OUT/prof_exec_${name}_$TAG.ncu-rep exec_${name}_$TAG $n > /dev/null 2>&1 \
    && cp profiles/ncu_full_exec_${name}_$TAG.json $OUT/
  rm -f $OUT/prof_exec_${name}_$TAG.ncu-rep
done
cp profiles/ncu_summary.json $OUT/ncu_summary_box_$TAG.json
timeout 1200 python tools/bench_configs.py > $OUT/configs_$TAG.jsonl 2> $OUT/configs_$TAG.err
echo done
