#!/usr/bin/env python
"""CUDA-graph capture of ensemble_solve (final state only, no saveat: no host-side
staging copies inside the call) for launch-bound small ensembles (C1 regime).
Prints the wall time per call of direct calls vs graph replays and checks that the
replayed results equal a direct solve bit for bit."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2304_06835_b200 as ens  # noqa: E402

dev = torch.device("cuda")
for alg, dt_ in [("tsit5", torch.float64), ("vern9", torch.float64)]:
    N = 1024
    u0, p = ens.generate_inputs("lorenz", "random10", N, dtype=dt_, seed=0xC1)
    kw = dict(adaptive=True, abstol=1e-8, reltol=1e-8)
    ref = ens.solve("lorenz", alg, u0, p, (0.0, 1.0), 1e-3, **kw)
    out = ens.Solution(u=torch.empty_like(ref.u), retcode=torch.empty_like(ref.retcode),
                       n_accept=torch.empty_like(ref.n_accept), n_reject=torch.empty_like(ref.n_reject), stats=None)
    ws = ens.Workspace(1 << 20, dev)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ens.solve("lorenz", alg, u0, p, (0.0, 1.0), 1e-3, out=out, workspace=ws, stream=s, **kw)   # warm-up
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ens.solve("lorenz", alg, u0, p, (0.0, 1.0), 1e-3, out=out, workspace=ws,
                  stream=torch.cuda.current_stream(), **kw)
    out.u.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out.u, ref.u) and torch.equal(out.n_accept, ref.n_accept)
    R = 200
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(R):
        ens.solve("lorenz", alg, u0, p, (0.0, 1.0), 1e-3, out=out, workspace=ws, **kw)
    torch.cuda.synchronize(); direct = (time.perf_counter() - t) / R
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(R):
        g.replay()
    torch.cuda.synchronize(); replay = (time.perf_counter() - t) / R
    print(f"{alg} N={N}: direct {direct * 1e6:.1f} us/call, graph replay {replay * 1e6:.1f} us/call", flush=True)
