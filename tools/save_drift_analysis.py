#!/usr/bin/env python
"""Why C3 save traffic cannot be fixed by staging (DESIGN §5 C3 write traffic): for 64 C3
trajectories (Robertson ±10 %, Rosenbrock23, tol 1e-8, 100 save points) the oracle gives the
attempt at which each save point is reached; from that, the spread of save indices inside groups
of 4 lanes (one 32-byte sector of fp64) and 32 lanes (a warp), and the fraction of saves whose
sector would be complete before a per-lane register ring of R saves overflows."""
import numpy as np, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle
from synth.inputs import make_inputs
N = 64
u0, p = make_inputs("robertson", "random10", N, seed=0xC3, dtype="f64")
sa = np.linspace(0.0, 1e5, 100)
att = np.zeros((100, N), np.int64)   # attempts taken before save j is stored
for j in range(1, 100):
    o, rc, na, nr = oracle.solve("robertson", "rosenbrock23", u0, p, (0.0, sa[j]), 1e-4, dtype="f64", adaptive=True,
                                 abstol=1e-8, reltol=1e-8)
    att[j] = na + nr
tot = att[-1]
print("attempts to tf: mean %.1f min %d max %d" % (tot.mean(), tot.min(), tot.max()))
# at attempt count a, lane's completed saves = #{j: att[j] <= a}
A = int(tot.max())
def js_at(a):
    return (att <= a).sum(0)
for G in [4, 32]:
    drifts = []
    for a in range(0, A, 5):
        js = js_at(a)
        g = js.reshape(-1, G)
        drifts.append((g.max(1) - g.min(1)))
    d = np.concatenate(drifts)
    print(f"group {G}: save-index drift percentiles 50/90/99/max:", np.percentile(d, [50, 90, 99]), d.max())
print("fraction of (lane, save) entries whose quad row is complete before the lane's ring (size R) overflows:")
for R in [1, 2, 3, 4, 6, 8, 12]:
    ok = tot_cnt = 0
    for q in range(N // 4):
        lanes = range(4 * q, 4 * q + 4)
        for L in lanes:
            for j in range(1, 100):
                tot_cnt += 1
                jj = j + R
                a_evict = att[jj, L] if jj < 100 else 10**9     # never evicted before the end (flushed at finish)
                if all(att[j, M] <= a_evict for M in lanes):
                    ok += 1
    print(R, round(ok / tot_cnt, 3))
