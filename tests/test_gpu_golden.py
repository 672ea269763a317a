"""GPU path vs the fixtures generated from the unmodified reference
(tests/golden/make_golden.py): plans, sampled / exact SpMM, gcn_normalize,
GCN forward, quantization — all bit-exact (sha256 of the output bytes)."""
import numpy as np
import pytest

from tests import golden_util as gu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m():
    import paper_2503_18427_b200 as m
    return m


@pytest.fixture(scope="module")
def cora():
    return gu.cora()


@pytest.mark.parametrize("name", list(gu.STRATS))
@pytest.mark.parametrize("w", [8, 32])
def test_cora_plans_and_spmm(m, cora, name, w):
    n = cora["row_ptr"].size - 1
    a = m.CsrMatrix(n, n, cora["row_ptr"], cora["col"], cora["val"])
    ps = m.build_plan_set(a, w, getattr(m.Strategy, name.upper()))
    plans = ps.plans
    sp = cora[f"plan_{name}_{w}_starts_ptr"]
    for i in range(n):
        p = plans[i]
        assert p.params.chunk_len == cora[f"plan_{name}_{w}_chunk"][i]
        assert p.params.sample_cnt == cora[f"plan_{name}_{w}_cnt"][i]
        assert list(p.starts) == list(cora[f"plan_{name}_{w}_starts"][sp[i]:sp[i + 1]])
    assert gu.digest(m.spmm_sampled(a, cora["b"], ps)) == cora[f"spmm_{name}_{w}"]
    assert m.sampling_rate(ps, a) == tuple(cora[f"rate_{name}_{w}"])
    an = m.gcn_normalize(a, True)
    assert gu.digest(m.spmm_sampled(an, cora["b"], m.build_plan_set(an, w, getattr(m.Strategy, name.upper())))) \
        == cora[f"spmm_norm_{name}_{w}"]


def test_cora_exact_gcn_quant(m, cora):
    n = cora["row_ptr"].size - 1
    a = m.CsrMatrix(n, n, cora["row_ptr"], cora["col"], cora["val"])
    b = cora["b"]
    assert gu.digest(m.spmm_exact(a, b)) == cora["spmm_exact"]
    an = m.gcn_normalize(a, True)
    rp, col, val = an.to_arrays()
    assert np.array_equal(rp, cora["norm_row_ptr"]) and np.array_equal(col, cora["norm_col"])
    assert gu.digest(val) == cora["norm_val"]
    ws, bs = [cora["gcn_w0"], cora["gcn_w1"]], [cora["gcn_b0"], cora["gcn_b1"]]
    assert gu.digest(m.gcn_forward(an, b, ws, bs)) == cora["gcn_exact"]
    assert gu.digest(m.gcn_forward(an, b, ws, bs, m.build_plan_set(an, 32))) == cora["gcn_w32"]
    assert gu.digest(m.gcn_forward(an, b, ws, bs, m.build_plan_set(an, 8))) == cora["gcn_w8"]
    for q in (8, 4):
        qf = m.quantize(b, bits=q)
        assert np.array_equal(np.array([qf.params.x_min, qf.params.x_max], np.float32), cora[f"q{q}_params"])
        assert gu.digest(qf.codes) == cora[f"q{q}_codes"]
        assert gu.digest(m.dequantize(qf)) == cora[f"q{q}_deq"]
        assert gu.digest(m.spmm_sampled_q8(a, qf, m.build_plan_set(a, 32))) == cora[f"q{q}_spmm_adaptive_32"]


@pytest.mark.parametrize("w", [16, 32, 64])
def test_heavy_tail(m, w):
    fx = gu.heavy()
    n = fx["row_ptr"].size - 1
    a = m.CsrMatrix(n, n, fx["row_ptr"], fx["col"], fx["val"])
    ps = m.build_plan_set(a, w)
    assert gu.digest(m.spmm_sampled(a, fx["b"], ps)) == fx[f"spmm_adaptive_{w}"]
    srow, _, _ = ps.sampled_csr()
    assert np.array_equal(np.diff(srow), fx[f"plan_{w}_chunk"].astype(np.uint64) * fx[f"plan_{w}_cnt"])


def test_sharded_driver_world1_on_gpu(m):
    """ShardedGCN with the CUDA ops and no process group == device.gcn_forward."""
    import torch

    from paper_2503_18427_b200 import device
    from paper_2503_18427_b200.gcn import ShardedGCN
    fx = gu.cora()
    n = fx["row_ptr"].size - 1
    g = device.Graph.from_numpy(fx["norm_row_ptr"], fx["norm_col"], m.gcn_normalize(
        m.CsrMatrix(n, n, fx["row_ptr"], fx["col"], fx["val"]), True).to_arrays()[2])
    plan = device.SampledPlan(g, 32)
    ws = [torch.from_numpy(fx["gcn_w0"]).cuda(), torch.from_numpy(fx["gcn_w1"]).cuda()]
    bs = [torch.from_numpy(fx["gcn_b0"]).cuda(), torch.from_numpy(fx["gcn_b1"]).cuda()]
    x = torch.from_numpy(fx["b"]).cuda()
    out = ShardedGCN(plan.srow_ptr, plan.scol, plan.sval, n, ws, bs).forward(x)
    torch.cuda.synchronize()
    assert gu.digest(np.ascontiguousarray(out.cpu().numpy())) == fx["gcn_w32"]


@pytest.mark.parametrize("name", list(gu.STRATS))
@pytest.mark.parametrize("w", [8, 32])
def test_cora_rates_cdf(m, cora, name, w):
    """Per-row rates and their CDF (bench.cpp:124-138) on the device, bit-exact
    vs the reference's outputs."""
    n = cora["row_ptr"].size - 1
    a = m.CsrMatrix(n, n, cora["row_ptr"], cora["col"], cora["val"])
    ps = m.build_plan_set(a, w, getattr(m.Strategy, name.upper()))
    per_row = m.sampling_rate_per_row(ps, a)
    assert gu.digest(per_row) == cora[f"rate_per_row_{name}_{w}"]
    want_r, want_f = cora[f"cdf_{name}_{w}_rate"], cora[f"cdf_{name}_{w}_frac"]
    steps = m.cdf_stats(per_row)
    assert np.array_equal(np.array([s[0] for s in steps]).view(np.uint64), want_r.view(np.uint64))
    assert np.array_equal(np.array([s[1] for s in steps]).view(np.uint64), want_f.view(np.uint64))
    r, f = m.sampling_rate_cdf(ps, a)  # per-row rates never leave the device
    assert np.array_equal(r.view(np.uint64), want_r.view(np.uint64))
    assert np.array_equal(f.view(np.uint64), want_f.view(np.uint64))


@pytest.mark.parametrize("w", [16, 32, 64])
def test_heavy_tail_cdf(m, w):
    fx = gu.heavy()
    n = fx["row_ptr"].size - 1
    a = m.CsrMatrix(n, n, fx["row_ptr"], fx["col"], fx["val"])
    r, f = m.sampling_rate_cdf(m.build_plan_set(a, w), a)
    assert np.array_equal(r.view(np.uint64), fx[f"cdf_{w}_rate"].view(np.uint64))
    assert np.array_equal(f.view(np.uint64), fx[f"cdf_{w}_frac"].view(np.uint64))


def test_cdf_known_answers_and_errors(m):
    assert m.cdf_stats([1.0, 1.0, 1.0]) == [(1.0, 1.0)]  # test_io_bench.cpp:177-187
    assert m.cdf_stats([1.0, 0.5]) == [(0.5, 0.5), (1.0, 1.0)]
    with pytest.raises(ValueError, match="rates must be nonempty"):
        m.cdf_stats([])
    # ties by == : +0 and -0 are one step; large random input vs the oracle port
    from oracle import port
    rng = np.random.default_rng(3)
    x = np.round(rng.random(300_000) * 997) / 997
    x[:1000] = -0.0
    got = m.cdf_stats(x)
    wr, wf = port.cdf_stats(x)
    assert np.array_equal(np.array([s[0] for s in got]).view(np.uint64), wr.view(np.uint64))
    assert np.array_equal(np.array([s[1] for s in got]).view(np.uint64), wf.view(np.uint64))
