"""int8 FAST MODE (north_star (3)): per-row / per-feature affine codes with
the decode fused into the SpMM gather (csrc/affine.cu).  Not bit-exact with
the reference (which has only the global min/max codes, quantize.cpp:11-64);
checked against an fp64 torch reference of the same op with the bounds the
header states (include/aesspmm_cuda.h, "int8 FAST MODE"):

  quantize  |x^ - x| <= s/2 + 2^-22 (|m| + 255 s)
  SpMM      |C - A B| <= sum_k |v_k| (s_k/2 + 2^-22 (|m_k| + 255 s_k))
                         + (slots + 2) 2^-23 sum_k |v_k| (|m_k| + 255 s_k)
"""
import numpy as np
import pytest

from tests import graphs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    from paper_2503_18427_b200 import device
    return device


def _features(rng, n, f, skew):
    x = rng.uniform(-1, 1, (n, f)).astype(np.float32)
    if skew:  # rows of very different magnitude and offset: where per-row scales pay
        x *= (10.0 ** rng.integers(-3, 3, n)).astype(np.float32)[:, None]
        x += rng.uniform(-5, 5, n).astype(np.float32)[:, None]
        x[: max(1, n // 50)] = 0.25  # constant rows decode exactly
    return x


def _param_grids(q, n, f):
    import torch
    p = q.params.double()
    s, m = p[:, 0], p[:, 1]
    if q.mode == "row":
        s, m = s[:, None].expand(n, f), m[:, None].expand(n, f)
    else:
        s, m = s[None, :].expand(n, f), m[None, :].expand(n, f)
    return s, m, torch


@pytest.mark.parametrize("mode", ["row", "feature"])
@pytest.mark.parametrize("shape", [(1000, 128), (333, 602), (257, 3), (64, 1), (5000, 130)])
@pytest.mark.parametrize("skew", [False, True])
def test_quantize_affine_bound(dev, mode, shape, skew):
    import torch
    n, f = shape
    x = _features(np.random.default_rng(n + f), n, f, skew)
    xt = torch.from_numpy(x).cuda()
    q = dev.quantize_affine(xt, mode)
    xh = dev.dequantize_affine(q).double()
    s, m, _ = _param_grids(q, n, f)
    bound = s / 2 + 2.0 ** -22 * (m.abs() + 255 * s)
    err = (xh - xt.double()).abs()
    assert bool((err <= bound).all()), float((err - bound).max())
    codes = q.codes.cpu().numpy()
    assert codes.dtype == np.uint8 and codes.shape == (n, f)
    # x^ reaches both ends of every row / column range exactly (min and max codes used)
    assert int(codes.min()) == 0


@pytest.mark.parametrize("mode", ["row", "feature"])
@pytest.mark.parametrize("f", [1, 7, 64, 128, 130, 602])
@pytest.mark.parametrize("width", [8, 32])
def test_spmm_q8_affine_bound(dev, mode, f, width):
    import torch
    n = 3000
    rp, col, _ = graphs.power_law(n, alpha=1.6, max_deg=500, seed=f + width)
    val = np.random.default_rng(f).uniform(-1, 1, col.size).astype(np.float32)
    g = dev.Graph.from_numpy(rp, col, val)
    plan = dev.SampledPlan(g, width)
    x = _features(np.random.default_rng(7 * f), n, f, skew=True)
    xt = torch.from_numpy(x).cuda()
    q = dev.quantize_affine(xt, mode)
    got = dev.spmm_q8_affine(plan.srow_ptr, plan.scol, plan.sval, q).double()

    # fp64 reference of the same op: sampled A (as a sparse CSR) times the ORIGINAL features
    a = torch.sparse_csr_tensor(plan.srow_ptr.long(), plan.scol.long(), plan.sval.double(), (n, n))
    aabs = torch.sparse_csr_tensor(plan.srow_ptr.long(), plan.scol.long(), plan.sval.double().abs(), (n, n))
    want = a @ xt.double()
    s, m, _ = _param_grids(q, n, f)
    slots = (plan.srow_ptr[1:] - plan.srow_ptr[:-1]).double()[:, None]
    mag = m.abs() + 255 * s
    bound = aabs @ (s / 2 + 2.0 ** -22 * mag) + (slots + 2) * 2.0 ** -23 * (aabs @ mag)
    err = (got - want).abs()
    assert bool((err <= bound).all()), float((err - bound).max())
    # and the fused decode agrees with spmm over the explicitly dequantized features
    deq = dev.dequantize_affine(q)
    ref_deq = dev.spmm(plan.srow_ptr, plan.scol, plan.sval, deq, max_row_slots=plan.row_bound).double()
    assert bool(((got - ref_deq).abs() <= (slots + 2) * 2.0 ** -23 * (aabs @ mag) * 2).all())


def test_affine_row_beats_global_on_skewed_rows(dev):
    """On features whose rows differ in scale (hidden GCN layers), per-row
    scales give a smaller SpMM error than the reference's one global range."""
    import torch
    n, f = 4000, 128
    rp, col, _ = graphs.power_law(n, alpha=1.8, max_deg=300, seed=3)
    val = np.ones(col.size, np.float32)
    g = dev.Graph.from_numpy(rp, col, val)
    plan = dev.SampledPlan(g, 32)
    xt = torch.from_numpy(_features(np.random.default_rng(1), n, f, skew=True)).cuda()
    exact = dev.spmm(plan.srow_ptr, plan.scol, plan.sval, xt, max_row_slots=plan.row_bound).double()
    qa = dev.quantize_affine(xt, "row")
    ea = (dev.spmm_q8_affine(plan.srow_ptr, plan.scol, plan.sval, qa).double() - exact).abs().mean()
    qg = dev.quantize(xt)
    eg = (dev.spmm_q8(plan.srow_ptr, plan.scol, plan.sval, qg, max_row_slots=plan.row_bound).double()
          - exact).abs().mean()
    assert float(ea) < 0.1 * float(eg)


def test_affine_handle_api(dev):
    """The reference-facing surface: quantize_affine -> QuantizedFeatures that
    spmm_sampled_q8 / dequantize decode with the affine params."""
    import paper_2503_18427_b200 as m
    rng = np.random.default_rng(4)
    n, f = 1500, 40
    rp, col, _ = graphs.power_law(n, alpha=1.7, max_deg=200, seed=4)
    val = rng.uniform(-1, 1, col.size).astype(np.float32)
    x = _features(rng, n, f, skew=True)
    a = m.CsrMatrix(n, n, rp, col, val)
    plans = m.build_plan_set(a, 16)
    for mode in ("row", "feature"):
        qf = m.quantize_affine(x, mode)
        assert qf.affine_mode == mode and qf.codes.dtype == np.uint16 and qf.codes.max() <= 255
        prm = qf.affine_params
        assert prm.shape == ((n if mode == "row" else f), 2)
        deq = m.dequantize(qf)
        sc = prm[:, 0][:, None] if mode == "row" else prm[:, 0][None, :]
        mm = prm[:, 1][:, None] if mode == "row" else prm[:, 1][None, :]
        np.testing.assert_allclose(deq, qf.codes.astype(np.float32) * sc + mm, rtol=0, atol=1e-6 * np.abs(x).max())
        got = m.spmm_sampled_q8(a, qf, plans)
        want = m.spmm_sampled(a, deq, plans)
        np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-4 * np.abs(x).max())
    assert m.quantize(x).affine_mode is None
    with pytest.raises(ValueError):
        m.quantize_affine(x, "column")
    bad = x.copy()
    bad[3, 3] = np.inf
    with pytest.raises(ValueError, match="NonFinite"):
        m.quantize_affine(bad, "row")
    with pytest.raises(ValueError, match="NonFinite"):
        m.quantize_affine(bad, "feature")


@pytest.mark.parametrize("mode", ["feature", "row"])
@pytest.mark.parametrize("f", [100, 128, 130, 300, 602, 640])
def test_feature_batch_kernel_equals_ring_kernel(dev, f, mode):
    """The per-feature affine decode runs in the batch kernel by default
    (spmm.cu, DEC 1) and in the cp.async ring kernel as variant 54: the same
    arithmetic in the same order, so the same bits."""
    import torch

    from paper_2503_18427_b200 import capi
    L = capi.lib()
    n = 6000
    rp, col, _ = graphs.power_law(n, alpha=1.5, max_deg=800, seed=f)
    val = np.random.default_rng(f).uniform(-1, 1, col.size).astype(np.float32)
    g = dev.Graph.from_numpy(rp, col, val)
    plan = dev.SampledPlan(g, 32)
    xt = torch.from_numpy(_features(np.random.default_rng(3 * f), n, f, skew=True)).cuda()
    q = dev.quantize_affine(xt, mode)
    got = dev.spmm_q8_affine(plan.srow_ptr, plan.scol, plan.sval, q)
    try:
        L.aes_dev_spmm_set_variant(54)
        ring = dev.spmm_q8_affine(plan.srow_ptr, plan.scol, plan.sval, q)
        L.aes_dev_spmm_set_variant(55)  # batch kernel as 128-code column tiles
        tiles = dev.spmm_q8_affine(plan.srow_ptr, plan.scol, plan.sval, q)
        wide = []
        for v in (56, 57):  # wide-row kernel (one warp per whole code row, F > 128), 8- / 12-slot rings
            L.aes_dev_spmm_set_variant(v)
            wide.append(dev.spmm_q8_affine(plan.srow_ptr, plan.scol, plan.sval, q))
        torch.cuda.synchronize()
    finally:
        L.aes_dev_spmm_set_variant(0)
    assert torch.equal(got.view(torch.int32), ring.view(torch.int32))
    assert torch.equal(tiles.view(torch.int32), ring.view(torch.int32))
    for w in wide:
        assert torch.equal(w.view(torch.int32), ring.view(torch.int32))
