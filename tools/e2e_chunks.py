import sys, time, torch
sys.path.insert(0, ".")
import paper_2304_06835_b200 as ens
from synth.inputs import make_inputs
N = 10**7
u0, p = make_inputs("lorenz", "rho_sweep", N, dtype="f32", N_total=N)
U = torch.from_numpy(u0).pin_memory(); P = torch.from_numpy(p).pin_memory()
for nc in [1, 4, 8, 16, 32]:
    staging = None
    uh, rc, staging = ens.solve_host("lorenz", "tsit5", U, P, (0.0, 1.0), 1e-3, n_chunks=nc)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        ens.solve_host("lorenz", "tsit5", U, P, (0.0, 1.0), 1e-3, n_chunks=nc, staging=staging, u_out_host=uh.unsqueeze(0) if uh.dim()==2 else uh, retcode_host=rc)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    print(nc, "chunks:", best * 1e3, "ms", N / best / 1e6, "M traj/s", flush=True)
