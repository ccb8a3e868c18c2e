python -m paper_2304_06835_b200._build > gpurun_out/build_x.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu_x2.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_x2.log
timeout 300 python - > gpurun_out/small_n.log 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
import tools.bench_configs as bc
for refill in [False, True]:
    bc.run("C1", "lorenz", "tsit5", "random10", 1024, "f64", (0.0, 1.0), 1e-3, "tsit5_adaptive", reps=20, input_seed=0xC1, adaptive=True, abstol=1e-8, reltol=1e-8, refill=refill)
for model, tf in [("orego", 30.0), ("hires", 321.8122), ("pollu", 60.0)]:
    bc.run("stiff-" + model, model, "rosenbrock23", "random10", 8192, "f64", (0.0, tf), 1e-6, "ros23", reps=3, input_seed=0x57, adaptive=True, abstol=1e-8, reltol=1e-8)
for N in [10**3, 10**4, 10**5]:
    bc.run("C2-fixed", "lorenz", "tsit5", "rho_sweep", N, "f32", (0.0, 1.0), 1e-3, "tsit5_fixed")
    bc.run("C2-adaptive", "lorenz", "tsit5", "rho_sweep", N, "f32", (0.0, 1.0), 1e-3, "tsit5_adaptive", adaptive=True, abstol=1e-6, reltol=1e-6)
PY
timeout 600 python bench.py > gpurun_out/bench_x2.json 2> gpurun_out/bench_x2.err
