# experiment: packed adaptive Tsit5 vs scalar
python -m paper_2304_06835_b200._build > gpurun_out/build_x.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu_x.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_x.log
for v in pair scalar; do
if [ $v = scalar ]; then export ENS_TUNE_NO_PAIR=1; fi
timeout 300 python - >> gpurun_out/pair_exp.log 2>&1 <<'PY'
import os, sys; sys.path.insert(0, '.')
import tools.bench_configs as bc
print('variant', 'scalar' if os.environ.get('ENS_TUNE_NO_PAIR') else 'pair')
for N in [10**6, 10**7]:
    bc.run("C2-adaptive", "lorenz", "tsit5", "rho_sweep", N, "f32", (0.0, 1.0), 1e-3, "tsit5_adaptive", adaptive=True, abstol=1e-6, reltol=1e-6)
bc.run("C5-1gpu-adaptive", "lorenz", "tsit5", "random10", 10**8, "f32", (0.0, 1.0), 1e-3, "tsit5_adaptive", reps=2, input_seed=0xC5, adaptive=True, abstol=1e-6, reltol=1e-6)
PY
done
