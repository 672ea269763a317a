"""Binary graph / feature files straight to HBM, interchangeable with the
reference's own writer and reader (proj/src/io.cpp:117-220): files the
reference saves load bit-identically here, files saved here load in the
reference, and loaded int8 features feed the fused int8 SpMM directly."""
import os

import numpy as np
import pytest

from oracle import port
from oracle import ref as oref
from tests import graphs

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not oref.available(), reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def m():
    import paper_2503_18427_b200 as m
    return m


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def test_csrb_roundtrip_with_reference(m, tmp_path):
    rp, col, val = graphs.power_law(3000, alpha=1.5, max_deg=500, seed=5)
    g = oref.RefCsr.from_arrays(3000, 3000, rp, col, val)
    p_ref = str(tmp_path / "ref.csrb")
    oref.save_csr_binary(g, p_ref)
    a = m.load_csr_binary(p_ref)
    got = a.to_arrays()
    assert np.array_equal(got[0], rp) and np.array_equal(got[1], col) and np.array_equal(bits(got[2]), bits(val))
    p_ours = str(tmp_path / "ours.csrb")
    m.save_csr_binary(a, p_ours)
    back = oref.load_csr_binary(p_ours).arrays()
    assert np.array_equal(back[0], rp) and np.array_equal(back[1], col)
    assert open(p_ref, "rb").read() == open(p_ours, "rb").read()
    # corrupt payload -> the reference's error text
    bad = str(tmp_path / "bad.csrb")
    raw = bytearray(open(p_ref, "rb").read())
    raw[29 + 8 * 5: 29 + 8 * 6] = (10 ** 9).to_bytes(8, "little")  # row_ptr[5] huge -> non-monotonic
    open(bad, "wb").write(bytes(raw))
    with pytest.raises(RuntimeError, match="invalid CSR payload"):
        m.load_csr_binary(bad)
    with pytest.raises(RuntimeError, match="BadMagic"):
        open(str(tmp_path / "x"), "wb").write(b"NOPE" + bytes(40))
        m.load_csr_binary(str(tmp_path / "x"))


def test_fmat_f32_and_q8_roundtrip_with_reference(m, tmp_path):
    import torch

    from paper_2503_18427_b200 import device
    rng = np.random.default_rng(6)
    x = rng.uniform(-1, 1, (2000, 130)).astype(np.float32)
    p32 = str(tmp_path / "f32.fmat")
    oref.save_fmat_f32(x, p32)
    got, ms = m.load_features(p32)
    assert np.array_equal(bits(got), bits(x)) and ms >= 0
    dx, _ = device.load_fmat(p32)
    assert np.array_equal(bits(dx.cpu().numpy()), bits(x))
    lo, hi = port.fit_params(x)
    codes = port.quantize(x, lo, hi)
    p8 = str(tmp_path / "q8.fmat")
    oref.save_fmat_q8(codes, lo, hi, p8)
    qf, _ = m.load_features(p8)
    assert np.array_equal(qf.codes, codes) and (qf.params.x_min, qf.params.x_max) == (np.float32(lo), np.float32(hi))
    assert os.path.getsize(p8) < os.path.getsize(p32) / 3.5  # int8 file: ~1/4 of the bytes
    # ours -> reference
    p8b = str(tmp_path / "ours_q8.fmat")
    m.save_fmat(qf, p8b)
    dt, (c2, lo2, hi2) = oref.load_fmat(p8b)
    assert dt == 1 and np.array_equal(c2, codes) and (lo2, hi2) == (lo, hi)
    p32b = str(tmp_path / "ours_f32.fmat")
    m.save_fmat(x, p32b)
    dt, x2 = oref.load_fmat(p32b)
    assert dt == 0 and np.array_equal(bits(x2), bits(x))
    # loaded int8 features drive the fused int8 SpMM directly (device tier)
    rp, col, val = graphs.power_law(2000, alpha=1.5, max_deg=400, seed=6)
    g = device.Graph.from_numpy(rp, col, val)
    plan = device.SampledPlan(g, 32)
    qd, _ = device.load_fmat(p8)
    out = device.spmm_q8(plan.srow_ptr, plan.scol, plan.sval, qd)
    torch.cuda.synchronize()
    want = port.spmm_sampled(rp, col, val, port.dequantize(codes, lo, hi), 32)
    assert np.array_equal(bits(out.cpu().numpy()), bits(want))
