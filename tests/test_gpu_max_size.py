"""Maximum-size edge case (-m gpu): an ensemble of more than 2^31 trajectories
(64-bit trajectory indices in the input generator, the solver, the fused
statistics and the output), the headline kernel (Lorenz Tsit5 fixed step, fp32,
two trajectories per thread) on a short span. ≈103 GB of HBM; skipped if the
device has less free memory."""
import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs

pytestmark = pytest.mark.gpu


def test_more_than_2_pow_31_trajectories():
    import torch

    import paper_2304_06835_b200 as ens
    N = 2**31 + 1001
    if torch.cuda.mem_get_info()[0] < 110e9:
        pytest.skip("needs ~103 GB of free device memory")
    u0, p = ens.generate_inputs("lorenz", "rho_sweep", N, dtype=torch.float32, N_total=N)
    sol = ens.solve("lorenz", "tsit5", u0, p, (0.0, 0.01), 1e-3, stats=True)
    del u0, p
    assert (sol.n_accept == 10).all().item() and (sol.retcode == 0).all().item()
    # sampled trajectories on both sides of 2^31 and at the ends, vs the oracle one by one
    idx = np.array([0, 1, 2**31 - 65, 2**31 - 2, 2**31 - 1, 2**31, 2**31 + 1, 2**31 + 64, N - 2, N - 1], np.int64)
    parts = [make_inputs("lorenz", "rho_sweep", 1, index_offset=int(i), N_total=N, dtype="f32") for i in idx]
    u0h = np.concatenate([a for a, _ in parts], 1)
    ph = np.concatenate([b for _, b in parts], 1)
    o, *_ = oracle.solve("lorenz", "tsit5", u0h, ph, (0.0, 0.01), 1e-3, dtype="f32")
    g = sol.u[:, torch.from_numpy(idx).cuda()].cpu().numpy()
    np.testing.assert_array_equal(g, o[0])
    # fused statistics over all N (count exact; mean against a chunked fp64 reduction of the states)
    st = sol.stats.cpu().numpy()[0]
    assert (st[:, 0] == N).all()
    mean = np.zeros(3)
    for c in range(3):
        acc = 0.0
        for s in range(0, N, 1 << 28):
            acc += sol.u[c, s:s + (1 << 28)].double().sum().item()
        mean[c] = acc / N
    np.testing.assert_allclose(st[:, 1], mean, rtol=1e-9)
