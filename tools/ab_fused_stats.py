"""A/B timing: fixed-step Tsit5 fp32 N=10^7 with and without fused statistics (same process)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2304_06835_b200 as ens

N = 10**7
u0, p = ens.generate_inputs("lorenz", "rho_sweep", N, dtype=torch.float32)
for stats in (False, True):
    ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, stats=stats)
torch.cuda.synchronize()
res = {False: [], True: []}
for rep in range(6):
    for stats in (False, True):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, stats=stats)
        e1.record()
        torch.cuda.synchronize()
        res[stats].append(e0.elapsed_time(e1))
for k, v in res.items():
    print("stats" if k else "plain", "min %.3f ms  median %.3f ms" % (min(v), sorted(v)[len(v) // 2]))
