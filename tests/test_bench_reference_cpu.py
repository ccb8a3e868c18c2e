"""bench.py --impl reference (this tier's reference arm: the CPU oracle) on CPU:
one JSON line with the driver contract's keys, the oracle's own cpu_baseline and
an e2e block with no host↔device bytes (-m "not gpu")."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_contract():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ["impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"]:
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 1 and d["warmup"] >= 3 and d["n_gpus"] == 1
    assert d["unit"] == "trajectories/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["unit"] == d["unit"]
    assert "workload" in d["config"]


def test_parity_sample_inputs_are_the_ensemble_at_those_indices():
    """bench.py's cpu_baseline sample (global indices i·stride, generated with the
    block-cyclic map chunk_len = 1) holds exactly the ensemble's inputs there."""
    import numpy as np

    import bench
    from synth.inputs import make_inputs
    for wl in ["c5", "c2"]:
        recipe, seed, _, _ = bench.WORKLOADS[wl]
        N_total, sample = 100_003, 777
        S, stride = bench.sample_indices(N_total, sample)
        u0s, ps = make_inputs("lorenz", recipe, S, seed=seed, dtype="f32", N_total=N_total, chunk_len=1,
                              chunk_stride=stride)
        ug, pg = make_inputs("lorenz", recipe, N_total, seed=seed, dtype="f32")
        idx = np.arange(S) * stride
        assert idx[-1] < N_total
        assert np.array_equal(ps, pg[:, idx]) and np.array_equal(u0s, ug[:, idx])


def test_parity_block():
    import numpy as np

    import bench
    o = np.random.default_rng(0).standard_normal((3, 50)).astype(np.float32)
    g = o.copy()
    g[1, 7] = np.nextafter(g[1, 7], np.float32(np.inf))
    rc = np.zeros(50, np.int32)
    b = bench.parity_block(g, rc, o, rc)
    assert b["n"] == 50 and b["bitexact_frac"] == 49 / 50 and 0 < b["max_rel"] < 1e-6 and b["pass"]
    b = bench.parity_block(g * 1.001, rc, o, rc)
    assert not b["pass"]
