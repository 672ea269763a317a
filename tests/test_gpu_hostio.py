"""Handle-tier transfers of large PAGEABLE host buffers (hostio.cu): numpy
inputs / outputs above the 4 MB threshold stream through the pinned staging
ring with multi-threaded host copies — results must equal the device path
bit for bit, for ragged widths (row bytes not a multiple of 16), several
chunks, and pinned buffers (direct copy)."""
import numpy as np
import pytest

from oracle import port
from tests import graphs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,f", [(70_000, 128), (33_333, 130), (9_000, 602)])
def test_pageable_spmm_matches_device_path(n, f):
    import torch

    import paper_2503_18427_b200 as m
    from paper_2503_18427_b200 import device
    rng = np.random.default_rng(n + f)
    rp, col, _ = graphs.power_law(n, alpha=1.8, max_deg=300, seed=n)
    val = rng.uniform(-1, 1, col.size).astype(np.float32)
    b = rng.uniform(-1, 1, (n, f)).astype(np.float32)  # pageable, 10-37 MB: several staging chunks
    a = m.CsrMatrix(n, n, rp, col, val)
    plans = m.build_plan_set(a, 32)
    got = m.spmm_sampled(a, b, plans)
    g = device.Graph.from_numpy(rp, col, val)
    plan = device.SampledPlan(g, 32)
    want = device.spmm_plan(plan, torch.from_numpy(b).cuda()).cpu().numpy()
    assert np.array_equal(np.ascontiguousarray(got).view(np.uint32), np.ascontiguousarray(want).view(np.uint32))
    # a sample of rows against the CPU oracle too
    rows = rng.choice(n, 200, replace=False)
    sub = port.spmm_sampled(rp, col, val, b, 32)[rows]
    assert np.array_equal(got[rows].view(np.uint32), sub.view(np.uint32))


def test_pinned_host_buffers_take_the_direct_copy():
    import ctypes

    import torch

    from paper_2503_18427_b200 import capi
    L = capi.lib()
    vp, u64 = ctypes.c_void_p, ctypes.c_uint64
    L.aes_csr_create.argtypes = [u64, u64, vp, u64, vp, vp, u64, vp]
    L.aes_build_plan_set.argtypes = [vp, ctypes.c_uint32, ctypes.c_int, vp]
    L.aes_spmm_sampled.argtypes = [vp, vp, u64, u64, vp, vp, vp, vp, vp]
    n, f = 40_000, 128
    rp, col, _ = graphs.power_law(n, alpha=1.8, max_deg=200, seed=5)
    val = np.ones(col.size, np.float32)
    h, p = ctypes.c_void_p(), ctypes.c_void_p()
    capi.check(L.aes_csr_create(n, n, rp.ctypes.data, rp.size, col.ctypes.data, val.ctypes.data, col.size,
                                ctypes.byref(h)))
    capi.check(L.aes_build_plan_set(h, 32, 0, ctypes.byref(p)))
    b = torch.rand((n, f), dtype=torch.float32).pin_memory()
    c = torch.empty((n, f), dtype=torch.float32).pin_memory()
    capi.check(L.aes_spmm_sampled(h, b.data_ptr(), n, f, p, c.data_ptr(), None, None, None))
    want = port.spmm_sampled(rp, col, val, b.numpy(), 32)
    assert np.array_equal(c.numpy().view(np.uint32), want.view(np.uint32))
    L.aes_plan_destroy(p)
    L.aes_csr_destroy(h)
