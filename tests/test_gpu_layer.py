"""Fused exact GCN layer (aes_dev_gcn_layer_fused, csrc/spmm.cu): one
persistent kernel whose producer warps gather the aggregate into shared
memory and whose consumer warps run the ordered GEMM.  Bit-identical to the
split kernels (spmm -> gemm_bias_act) and to the CPU oracle's
gcn layer (proj/src/gnn.cpp:66-78 for one layer)."""
import numpy as np
import pytest

from oracle import port
from tests import graphs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    from paper_2503_18427_b200 import device
    return device


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def to_np(t):
    return t.cpu().numpy()


@pytest.mark.parametrize("k,n_out", [(128, 128), (128, 40), (64, 128), (100, 7), (4, 1), (128, 100)])
@pytest.mark.parametrize("strategy", ["adaptive", "afs", "sfs"])
def test_fused_layer_matches_split_and_oracle(dev, k, n_out, strategy):
    import torch
    rng = np.random.default_rng(k * 1000 + n_out)
    n = 2000 + 77  # partial last 128-row tile
    rp, col, _ = graphs.power_law(n, alpha=1.7, max_deg=400, seed=k + n_out)
    val = rng.uniform(-1, 1, col.size).astype(np.float32)
    g = dev.Graph.from_numpy(rp, col, val)
    plan = dev.SampledPlan(g, 32, strategy)
    x = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    x[rng.random((n, k)) < 0.2] = 0.0  # zeros: the reference's a == 0 skip must stay neutral
    w = rng.uniform(-0.5, 0.5, (k, n_out)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, n_out).astype(np.float32)
    xt, wt, bt = (torch.from_numpy(a).cuda() for a in (x, w, b))
    for relu in (True, False):
        fused = dev.gcn_layer_fused(plan.srow_ptr, plan.scol, plan.sval, xt, wt, bt, relu)
        assert fused is not None
        agg = dev.spmm(plan.srow_ptr, plan.scol, plan.sval, xt, max_row_slots=plan.row_bound)
        split = dev.gemm_bias_act(agg, wt, bt, relu=relu)
        torch.cuda.synchronize()
        assert np.array_equal(bits(to_np(fused)), bits(to_np(split)))
    want = port.gcn_forward(rp, col, val, x, [w], [b], 32) if strategy == "adaptive" else None
    if want is not None:  # one layer, last layer: no ReLU
        got = dev.gcn_layer_fused(plan.srow_ptr, plan.scol, plan.sval, xt, wt, bt, False)
        assert np.array_equal(bits(to_np(got)), bits(want))


def test_fused_layer_nonfinite_weights_keep_the_skip(dev):
    """W with inf: the reference skips a == 0 (0 * inf would be NaN); the
    fused kernel's finite_w = 0 form must too."""
    import torch
    rng = np.random.default_rng(5)
    n, k, n_out = 600, 128, 64
    rp, col, _ = graphs.power_law(n, alpha=1.9, max_deg=100, seed=5)
    val = rng.uniform(-1, 1, col.size).astype(np.float32)
    g = dev.Graph.from_numpy(rp, col, val)
    plan = dev.SampledPlan(g, 16)
    x = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    x[:, 3] = 0.0
    w = rng.uniform(-0.5, 0.5, (k, n_out)).astype(np.float32)
    w[3, :] = np.inf
    xt, wt = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    b = torch.zeros(n_out, device="cuda")
    fused = dev.gcn_layer_fused(plan.srow_ptr, plan.scol, plan.sval, xt, wt, b, False, finite_w=False)
    agg = dev.spmm(plan.srow_ptr, plan.scol, plan.sval, xt, max_row_slots=plan.row_bound)
    split = dev.gemm_bias_act(agg, wt, b, relu=False, finite_w=False)
    torch.cuda.synchronize()
    assert np.array_equal(bits(to_np(fused)), bits(to_np(split)))
    want = port.gcn_forward(rp, col, val, x, [w], [np.zeros(n_out, np.float32)], 16)
    assert np.array_equal(bits(to_np(fused)), bits(want))


def test_fused_layer_unsupported_shapes_fall_back(dev):
    import torch
    rng = np.random.default_rng(6)
    n = 300
    rp, col, _ = graphs.power_law(n, alpha=2.0, max_deg=50, seed=6)
    g = dev.Graph.from_numpy(rp, col, np.ones(col.size, np.float32))
    plan = dev.SampledPlan(g, 32)
    for k, n_out in [(130, 16), (6, 16), (128, 129)]:
        xt = torch.from_numpy(rng.uniform(-1, 1, (n, k)).astype(np.float32)).cuda()
        wt = torch.from_numpy(rng.uniform(-1, 1, (k, n_out)).astype(np.float32)).cuda()
        assert dev.gcn_layer_fused(plan.srow_ptr, plan.scol, plan.sval, xt, wt, None, True) is None


def test_fused_gcn_forward_arxiv_shape(dev):
    """3-layer GCN at the arxiv shape through gcn_forward (fused layers) ==
    the split-kernel forward, bit for bit."""
    import torch
    from paper_2503_18427_b200 import synth
    n = 169_343
    rp, col, val = synth.power_law_csr(n, 2.0737, 13_161, seed=3, device="cuda")
    g = dev.Graph(rp, col, val, n)
    plan = dev.SampledPlan(g, 32)
    x = synth.features(n, 128, seed=4, device="cuda")
    gen = torch.Generator(device="cuda").manual_seed(9)
    ws = [torch.rand(s, generator=gen, device="cuda") - 0.5 for s in [(128, 128), (128, 128), (128, 40)]]
    bs = [torch.full((s,), 0.01, device="cuda") for s in (128, 128, 40)]
    saved = dev.FUSED_LAYER_MIN_ROWS
    dev.FUSED_LAYER_MIN_ROWS = 0  # (arxiv is below the default size threshold)
    try:
        fused = dev.gcn_forward(g, x, ws, bs, plan)
    finally:
        dev.FUSED_LAYER_MIN_ROWS = saved
    split = dev.gcn_forward(g, x, ws, bs, plan, fused=False)
    torch.cuda.synchronize()
    assert torch.equal(fused.view(torch.int32), split.view(torch.int32))


def test_sharded_gcn_nccl_mode_fused_layers(dev):
    """gcn.ShardedGCN (exchange="nccl", one rank) runs each fp32 layer as the
    fused kernel writing its slice of the all-gather buffer: == the oracle."""
    import torch
    from paper_2503_18427_b200.gcn import ShardedGCN
    rng = np.random.default_rng(11)
    n = 5000
    rp, col, _ = graphs.power_law(n, alpha=1.8, max_deg=300, seed=11)
    nrp, ncol, nval = port.gcn_normalize(rp, col, True)
    g = dev.Graph.from_numpy(nrp, ncol, nval)
    plan = dev.SampledPlan(g, 32)
    x = rng.uniform(-1, 1, (n, 64)).astype(np.float32)
    ws = [rng.uniform(-0.5, 0.5, s).astype(np.float32) for s in [(64, 128), (128, 16)]]
    bs = [np.full(128, 0.01, np.float32), np.zeros(16, np.float32)]
    model = ShardedGCN(plan.srow_ptr, plan.scol, plan.sval, n, [torch.from_numpy(w).cuda() for w in ws],
                       [torch.from_numpy(b).cuda() for b in bs], exchange="nccl", max_row_slots=plan.row_bound)
    model.fused_min_rows = 0
    out = model.forward(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    want = port.gcn_forward(nrp, ncol, nval, x, ws, bs, 32)
    assert np.array_equal(bits(to_np(out)), bits(want))


@pytest.mark.parametrize("n", [1, 2, 63, 64, 65, 1000, 9473 + 64 * 148])
def test_fused_layer_small_and_ragged_graphs(dev, n):
    """Row blocks smaller than one tile, CTAs with empty blocks, rows with no
    slots (isolated rows), the partial last tile of every producer."""
    import torch
    rng = np.random.default_rng(n)
    rp, col, _ = graphs.power_law(n, alpha=1.5, max_deg=min(n, 200), seed=n)
    keep = rng.random(n) < 0.85  # ~15 % of the rows lose all their nonzeros
    rows = [col[rp[i]:rp[i + 1]] if keep[i] else col[:0] for i in range(n)]
    rp2 = np.zeros(n + 1, np.uint64)
    rp2[1:] = np.cumsum([r.size for r in rows])
    col2 = np.concatenate(rows).astype(np.uint32) if rp2[-1] else np.zeros(0, np.uint32)
    val2 = rng.uniform(-1, 1, col2.size).astype(np.float32)
    g = dev.Graph.from_numpy(rp2, col2, val2)
    plan = dev.SampledPlan(g, 32)
    x = rng.uniform(-1, 1, (n, 32)).astype(np.float32)
    w = rng.uniform(-0.5, 0.5, (32, 24)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, 24).astype(np.float32)
    xt, wt, bt = (torch.from_numpy(a).cuda() for a in (x, w, b))
    fused = dev.gcn_layer_fused(plan.srow_ptr, plan.scol, plan.sval, xt, wt, bt, True)
    torch.cuda.synchronize()
    want = port.bias_act(port.dense_matmul(port.spmm_sampled(rp2, col2, val2, x, 32), w), b, True)
    assert np.array_equal(bits(to_np(fused)), bits(want))


def test_fused_layer_refuses_in_place_output(dev):
    import torch
    n = 500
    rp, col, _ = graphs.power_law(n, alpha=2.0, max_deg=50, seed=8)
    g = dev.Graph.from_numpy(rp, col, np.ones(col.size, np.float32))
    plan = dev.SampledPlan(g, 32)
    x = torch.rand((n, 64), device="cuda")
    w = torch.rand((64, 64), device="cuda")
    assert dev.gcn_layer_fused(plan.srow_ptr, plan.scol, plan.sval, x, w, None, True, out=x) is None
