#!/usr/bin/env python
"""Bandwidth of ens_ensemble_stats over a stored [rows][N] state array (the
second kernel of the bench step): best of 10 with CUDA events."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2304_06835_b200 as ens  # noqa: E402

for dt in (torch.float32, torch.float64):
    for rows, N in [(3, 10**7), (33, 10**6)]:
        x = torch.randn((rows, N), dtype=dt, device="cuda")
        out = torch.empty((rows, 3), dtype=torch.float64, device="cuda")
        ws = ens.Workspace(ens.lib().ens_stats_workspace_bytes(N, rows), "cuda")
        for _ in range(3):
            ens.ensemble_stats(x, out=out, workspace=ws)
        best = 1e9
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); ens.ensemble_stats(x, out=out, workspace=ws); b.record(); torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        gbs = x.numel() * x.element_size() / (best / 1e3) / 1e9
        print(f"{str(dt):14s} rows={rows} N={N}: {best * 1e3:.1f} us  {gbs:.0f} GB/s", flush=True)
