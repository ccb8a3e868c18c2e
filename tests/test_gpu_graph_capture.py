"""ensemble_solve inside a CUDA graph (-m gpu): a final-state solve does no
host-to-device staging, so it can be captured once and replayed; replays give
the direct call's results bit for bit (tools/graph_capture_demo.py times it)."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("alg", ["tsit5", "vern9", "rodas5"])
def test_capture_and_replay(alg):
    import torch

    import paper_2304_06835_b200 as ens
    dev = torch.device("cuda")
    model = "robertson" if alg == "rodas5" else "lorenz"
    tf = 10.0 if alg == "rodas5" else 1.0
    u0, p = ens.generate_inputs(model, "random10", 777, dtype=torch.float64, seed=5)
    kw = dict(adaptive=True, abstol=1e-8, reltol=1e-8)
    ref = ens.solve(model, alg, u0, p, (0.0, tf), 1e-4, **kw)
    out = ens.Solution(u=torch.empty_like(ref.u), retcode=torch.empty_like(ref.retcode),
                       n_accept=torch.empty_like(ref.n_accept), n_reject=torch.empty_like(ref.n_reject), stats=None)
    ws = ens.Workspace(1 << 20, dev)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ens.solve(model, alg, u0, p, (0.0, tf), 1e-4, out=out, workspace=ws, stream=s, **kw)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ens.solve(model, alg, u0, p, (0.0, tf), 1e-4, out=out, workspace=ws, stream=torch.cuda.current_stream(), **kw)
    out.u.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out.u, ref.u) and torch.equal(out.n_accept, ref.n_accept)
