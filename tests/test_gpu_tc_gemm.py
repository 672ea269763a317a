"""Fast-mode tcgen05 (TF32) layer GEMM: within the stated bound of the exact
fp32 result, |H - H_exact| <= 2^-8 * sum_k |a_ik| |w_kj| (+ a denormal
floor), for the GCN layer shapes.  The exact path (gemm.cu) is what the
reference-parity tests use; this mode is opt-in."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,k,n", [(1000, 128, 128), (4097, 128, 40), (300, 16, 16), (129, 40, 7), (70000, 128, 128),
                                   (5000, 100, 64)])
def test_tf32_gemm_within_bound(m, k, n):
    import torch

    from paper_2503_18427_b200 import device
    g = torch.Generator(device="cuda")
    g.manual_seed(m + k + n)
    a = device.padded(torch.rand((m, k), generator=g, device="cuda") * 2 - 1)
    w = torch.rand((k, n), generator=g, device="cuda") - 0.5
    bias = torch.rand(n, generator=g, device="cuda") * 0.1
    for relu in (False, True):
        got = device.gemm_tf32(a, w, bias, relu)
        exact = a.double() @ w.double() + bias.double()
        if relu:
            exact = exact.clamp_min(0)
        bound = (a.double().abs() @ w.double().abs()) * 2.0 ** -8 + 1e-30
        err = (got.double() - exact).abs()
        assert bool((err <= bound + 2.0 ** -20).all()), float((err - bound).max())


def test_core_fast_gemm_option():
    """_core.gcn_forward / sage_forward(fast_gemm=True): close to the exact
    (bit-exact-with-reference) result, same argmax on almost every row."""
    import paper_2503_18427_b200 as m
    from oracle import port
    from tests import graphs
    rng = np.random.default_rng(9)
    rp, col, _ = graphs.power_law(2500, alpha=1.8, max_deg=300, seed=9)
    nrp, ncol, nval = port.gcn_normalize(rp, col, True)
    adj = m.CsrMatrix(2500, 2500, nrp, ncol, nval)
    x = rng.uniform(-1, 1, (2500, 64)).astype(np.float32)
    ws = [rng.uniform(-0.5, 0.5, (64, 64)).astype(np.float32), rng.uniform(-0.5, 0.5, (64, 16)).astype(np.float32)]
    bs = [np.full(64, 0.01, np.float32), np.zeros(16, np.float32)]
    plans = m.build_plan_set(adj, 32)
    exact = m.gcn_forward(adj, x, ws, bs, plans)
    fast = m.gcn_forward(adj, x, ws, bs, plans, fast_gemm=True)
    assert np.abs(fast - exact).max() / np.abs(exact).max() < 2e-2
    assert (fast.argmax(1) == exact.argmax(1)).mean() > 0.98
    am = m.row_mean_normalize(m.CsrMatrix(2500, 2500, rp, col, np.ones(col.size, np.float32)))
    ws2 = [rng.uniform(-0.5, 0.5, (128, 32)).astype(np.float32)]
    e2 = m.sage_forward(am, x, ws2, [np.zeros(32, np.float32)])
    f2 = m.sage_forward(am, x, ws2, [np.zeros(32, np.float32)], fast_gemm=True)
    assert np.abs(f2 - e2).max() / np.abs(e2).max() < 2e-2


def test_fast_gcn_forward_close_to_exact():
    import torch

    from oracle import port
    from paper_2503_18427_b200 import device
    from tests import graphs
    rng = np.random.default_rng(4)
    rp, col, _ = graphs.power_law(3000, alpha=2.0, max_deg=300, seed=4)
    nrp, ncol, nval = port.gcn_normalize(rp, col, True)
    g = device.Graph.from_numpy(nrp, ncol, nval)
    x = torch.from_numpy(rng.uniform(-1, 1, (3000, 128)).astype(np.float32)).cuda()
    ws = [torch.from_numpy(rng.uniform(-0.5, 0.5, s).astype(np.float32)).cuda() for s in [(128, 128), (128, 40)]]
    bs = [torch.full((128,), 0.01, device="cuda"), torch.zeros(40, device="cuda")]
    plan = device.SampledPlan(g, 32)
    exact = device.gcn_forward(g, x, ws, bs, plan)
    fast = device.gcn_forward(g, x, ws, bs, plan, fast_gemm=True)
    rel = (fast - exact).abs().max() / exact.abs().max()
    assert float(rel) < 2e-2
    agree = (fast.argmax(1) == exact.argmax(1)).float().mean()
    assert float(agree) > 0.98
