"""GPU parity for the device tier (torch tensors through the C ABI via ctypes),
including row shards (the multi-GPU partition) and arxiv-scale graphs checked
against the oracle bit for bit, plus products-scale row-sample parity."""
import numpy as np
import pytest

from oracle import port
from tests import graphs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    import torch  # noqa: F401

    from paper_2503_18427_b200 import device
    return device


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def to_np(t):
    return t.detach().cpu().numpy()


def bits_of(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("f", [16, 128, 602])
def test_device_spmm_matches_oracle(dev, f):
    import torch
    rp, col, val = graphs.power_law(4000, alpha=1.5, max_deg=3000, seed=f)
    g = dev.Graph.from_numpy(rp, col, val)
    b_np = np.random.default_rng(f).uniform(-1, 1, (4000, f)).astype(np.float32)
    b = dev.padded(torch.from_numpy(b_np).cuda())
    for w in (16, 32, 64):
        plan = dev.SampledPlan(g, w)
        out = dev.spmm_plan(plan, b)
        torch.cuda.synchronize()
        want = port.spmm_sampled(rp, col, val, b_np, w)
        assert np.array_equal(bits(to_np(out)), bits(want))
        # unpadded contiguous (scalar path when f % 4 != 0)
        out2 = dev.spmm_plan(plan, torch.from_numpy(b_np).cuda().contiguous(),
                             out=torch.empty((4000, f), device="cuda"))
        assert np.array_equal(bits(to_np(out2)), bits(want))


def test_row_shards_equal_global(dev):
    import torch
    rp, col, val = graphs.power_law(5000, alpha=1.4, max_deg=4000, seed=1)
    g = dev.Graph.from_numpy(rp, col, val)
    b = torch.randn(5000, 128, device="cuda")
    full = dev.spmm_plan(dev.SampledPlan(g, 32), b)
    cuts = [0, 1234, 2500, 4999, 5000]
    parts = [dev.spmm_plan(dev.SampledPlan(g.rows(lo, hi), 32), b) for lo, hi in zip(cuts, cuts[1:])]
    assert torch.equal(torch.cat(parts), full)


@pytest.mark.parametrize("f", [72, 100, 128, 130, 256, 602])
def test_device_q8(dev, f):
    """Device int8 path; F > 64 with 16-B aligned code rows runs the batch
    kernel, F > 128 the wide-row kernel (one warp per whole code row)."""
    import torch
    rp, col, val = graphs.power_law(3000, alpha=1.5, max_deg=2000, seed=2)
    g = dev.Graph.from_numpy(rp, col, val)
    x_np = np.random.default_rng(f).uniform(-1, 1, (3000, f)).astype(np.float32)
    x = torch.from_numpy(x_np).cuda()
    q = dev.quantize(x)
    lo, hi = port.fit_params(x_np)
    assert (q.x_min, q.x_max) == (lo, hi)
    codes = port.quantize(x_np, lo, hi)
    assert np.array_equal(to_np(q.codes).astype(np.uint16), codes)
    plan = dev.SampledPlan(g, 32)
    out = dev.spmm_q8(plan.srow_ptr, plan.scol, plan.sval, q)
    want = port.spmm_sampled(rp, col, val, port.dequantize(codes, lo, hi), 32)
    assert np.array_equal(bits(to_np(out)), bits(want))
    assert np.array_equal(bits(to_np(dev.dequantize(q))), bits(port.dequantize(codes, lo, hi)))
    # unaligned code rows (ld = f) take the generic ring kernel: same bits
    qc = dev.QuantizedDevice(q.codes.contiguous(), q.x_min, q.x_max, q.bits, q.lut)
    if f % 4 == 0:
        out2 = dev.spmm_q8(plan.srow_ptr, plan.scol, plan.sval, qc)
        assert np.array_equal(bits(to_np(out2)), bits(want))


def test_device_gcn_forward(dev):
    import torch
    rng = np.random.default_rng(4)
    rp, col, _ = graphs.power_law(3000, alpha=2.0, max_deg=300, seed=4)
    nrp, ncol, nval = port.gcn_normalize(rp, col, True)
    g = dev.Graph.from_numpy(nrp, ncol, nval)
    x = rng.uniform(-1, 1, (3000, 128)).astype(np.float32)
    ws = [rng.uniform(-0.5, 0.5, s).astype(np.float32) for s in [(128, 128), (128, 128), (128, 40)]]
    bs = [np.full(128, 0.01, np.float32), np.full(128, 0.01, np.float32), np.zeros(40, np.float32)]
    tw = [torch.from_numpy(w).cuda() for w in ws]
    tb = [torch.from_numpy(b).cuda() for b in bs]
    plan = dev.SampledPlan(g, 32)
    out = dev.gcn_forward(g, torch.from_numpy(x).cuda(), tw, tb, plan)
    want = port.gcn_forward(nrp, ncol, nval, x, ws, bs, 32)
    assert np.array_equal(bits(to_np(out)), bits(want))
    # the same forward captured in a CUDA graph and replayed, on new inputs too
    cg = dev.GcnForwardGraph(g, torch.from_numpy(x).cuda(), tw, tb, plan)
    assert np.array_equal(bits(to_np(cg.run())), bits(want))
    x2 = rng.uniform(-1, 1, (3000, 128)).astype(np.float32)
    got2 = to_np(cg.run(torch.from_numpy(x2).cuda()))
    assert np.array_equal(bits(got2), bits(port.gcn_forward(nrp, ncol, nval, x2, ws, bs, 32)))


@pytest.mark.slow
def test_arxiv_shape_bit_exact(dev):
    """Full ogbn-arxiv-shaped graph (169 343 rows, F = 128, W = 32) vs oracle."""
    import torch

    from paper_2503_18427_b200 import synth
    rp, col, val = synth.power_law_csr(169_343, 2.0737, 13_161, seed=1, device="cuda")
    g = dev.Graph(rp, col, val, 169_343)
    b = torch.rand(169_343, 128, device="cuda") * 2 - 1
    out = dev.spmm_plan(dev.SampledPlan(g, 32), b)
    want = port.spmm_sampled(to_np(rp).view(np.uint64), to_np(col).view(np.uint32), to_np(val), to_np(b), 32)
    assert np.array_equal(bits(to_np(out)), bits(want))


@pytest.mark.slow
def test_products_shape_row_sample_parity(dev):
    """Products shape (2.45 M rows): exact parity on a seeded sample of 20 000
    rows (the oracle recomputes those rows from the same CSR)."""
    import torch

    from paper_2503_18427_b200 import synth
    n = 2_450_000
    rp, col, val = synth.power_law_csr(n, 1.7885, 17_481, seed=1, device="cuda")
    g = dev.Graph(rp, col, val, n)
    b = torch.rand(n, 128, device="cuda") * 2 - 1
    plan = dev.SampledPlan(g, 32)
    out = dev.spmm_plan(plan, b)
    rows = np.sort(np.random.default_rng(0).choice(n, 20_000, replace=False))
    rp_np, col_np, val_np = to_np(rp).view(np.uint64), to_np(col).view(np.uint32), to_np(val)
    sub_rp = np.zeros(rows.size + 1, np.uint64)
    sub_rp[1:] = np.cumsum(rp_np[rows + 1] - rp_np[rows])
    idx = np.concatenate([np.arange(rp_np[r], rp_np[r + 1]) for r in rows]).astype(np.int64)
    want = port.spmm_sampled(sub_rp, col_np[idx], val_np[idx], to_np(b), 32)
    assert np.array_equal(bits(to_np(out)[rows]), bits(want))
    # slot-count invariant (sum of per-row slots) and S <= sum(min(nnz, W))
    deg = np.diff(rp_np).astype(np.int64)
    assert plan.total_slots <= int(np.minimum(deg, 32).sum())


def test_async_host_call_matches_sync():
    """aes_spmm_sampled_async (stream-ordered H2D -> SpMM -> D2H) == the
    synchronous handle call, on two overlapping streams."""
    import ctypes

    import torch

    from paper_2503_18427_b200 import capi
    L = capi.lib()
    vp, u64 = ctypes.c_void_p, ctypes.c_uint64
    L.aes_csr_create.argtypes = [u64, u64, vp, u64, vp, vp, u64, vp]
    L.aes_build_plan_set.argtypes = [vp, ctypes.c_uint32, ctypes.c_int, vp]
    L.aes_spmm_sampled_async.argtypes = [vp, vp, u64, u64, vp, vp, vp]
    rp, col, val = graphs.power_law(5000, alpha=1.5, max_deg=2000, seed=8)
    h, p = ctypes.c_void_p(), ctypes.c_void_p()
    capi.check(L.aes_csr_create(5000, 5000, rp.ctypes.data, rp.size, col.ctypes.data, val.ctypes.data, col.size,
                                ctypes.byref(h)))
    capi.check(L.aes_build_plan_set(h, 32, 0, ctypes.byref(p)))
    want = port.spmm_sampled(rp, col, val, np.ones((5000, 1), np.float32), 32)  # noqa: F841 (warm oracle)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    for i, f in enumerate([128, 602, 7, 128]):
        b = torch.from_numpy(np.random.default_rng(i).standard_normal((5000, f)).astype(np.float32)).pin_memory()
        c = torch.empty((5000, f), dtype=torch.float32).pin_memory()
        capi.check(L.aes_spmm_sampled_async(h, b.data_ptr(), 5000, f, p, c.data_ptr(), streams[i % 2].cuda_stream))
        outs.append((b, c))
    torch.cuda.synchronize()
    for b, c in outs:
        want = port.spmm_sampled(rp, col, val, b.numpy(), 32)
        assert np.array_equal(bits(c.numpy()), bits(want))
    L.aes_plan_destroy(p)
    L.aes_csr_destroy(h)


@pytest.mark.parametrize("variant", [1, 2, 3, 4, 5, 6, 7, 8, 21, 22, 23, 24, 30, 31, 32, 33, 34, 35, 36, 37, 38, 39, 40, 43, 44, 45])
def test_every_spmm_schedule_is_bit_exact(dev, variant):
    """All schedule variants (aes_dev_spmm_set_variant) give the oracle's bits,
    fp32 and int8 (int8 dual-stream kernel: variants 21-24; int8 batch kernel:
    30-39, the default for 64 < F <= 128; TMA-gather kernel: 40)."""
    import torch

    from paper_2503_18427_b200 import capi
    L = capi.lib()
    rp, col, val = graphs.power_law(6000, alpha=1.4, max_deg=3000, seed=variant)
    g = dev.Graph.from_numpy(rp, col, val)
    x_np = np.random.default_rng(variant).uniform(-1, 1, (6000, 128)).astype(np.float32)
    x = torch.from_numpy(x_np).cuda()
    plan = dev.SampledPlan(g, 32)
    q = dev.quantize(x)
    lo, hi = port.fit_params(x_np)
    deq = port.dequantize(port.quantize(x_np, lo, hi), lo, hi)
    try:
        L.aes_dev_spmm_set_variant(variant)
        out = dev.spmm_plan(plan, x)
        outq = dev.spmm_q8(plan.srow_ptr, plan.scol, plan.sval, q)
        torch.cuda.synchronize()
    finally:
        L.aes_dev_spmm_set_variant(0)
    assert np.array_equal(bits(to_np(out)), bits(port.spmm_sampled(rp, col, val, x_np, 32)))
    assert np.array_equal(bits(to_np(outq)), bits(port.spmm_sampled(rp, col, val, deq, 32)))


@pytest.mark.parametrize("sched", [0, 1, 2, 3])
@pytest.mark.parametrize("f", [128, 100])
def test_ring_schedules_bit_exact(dev, sched, f):
    """Auto, static, heavy-first dynamic and balanced row schedules give the
    oracle's bits, on a graph whose hub rows exceed the heavy threshold (4096
    slots) and the hub-row kernel's (auto: column-split CTA per hub row; F=100
    exercises its partial last column block)."""
    import torch

    from paper_2503_18427_b200 import capi
    L = capi.lib()
    rp, col, val = graphs.power_law(12000, alpha=1.2, max_deg=9000, seed=3)
    assert np.diff(rp).max() > 4096
    g = dev.Graph.from_numpy(rp, col, val)
    x_np = np.random.default_rng(3).uniform(-1, 1, (12000, f)).astype(np.float32)
    x = torch.from_numpy(x_np).cuda()
    try:
        capi.check(L.aes_dev_spmm_set_schedule(sched))
        exact = dev.spmm_exact(g, x)
        sampled = dev.spmm_plan(dev.SampledPlan(g, 32), x)
        torch.cuda.synchronize()
    finally:
        L.aes_dev_spmm_set_schedule(0)
    assert np.array_equal(bits(to_np(exact)), bits(port.spmm_csr(rp, col, val, x_np)))
    assert np.array_equal(bits(to_np(sampled)), bits(port.spmm_sampled(rp, col, val, x_np, 32)))


@pytest.mark.parametrize("sched", [0, 1, 2, 3, 6])
@pytest.mark.parametrize("f", [128, 300])
def test_q8_schedules_bit_exact(dev, sched, f):
    """int8 batch kernel under every schedule, exact (unbounded rows) and
    sampled, single and multi column tile."""
    import torch

    from paper_2503_18427_b200 import capi
    L = capi.lib()
    rp, col, val = graphs.power_law(12000, alpha=1.2, max_deg=9000, seed=4)
    g = dev.Graph.from_numpy(rp, col, val)
    x_np = np.random.default_rng(4).uniform(-1, 1, (12000, f)).astype(np.float32)
    q = dev.quantize(torch.from_numpy(x_np).cuda())
    lo, hi = port.fit_params(x_np)
    deq = port.dequantize(port.quantize(x_np, lo, hi), lo, hi)
    plan = dev.SampledPlan(g, 32)
    try:
        capi.check(L.aes_dev_spmm_set_schedule(sched))
        exact = dev.spmm_q8(g.row_ptr, g.col, g.val, q)
        sampled = dev.spmm_q8(plan.srow_ptr, plan.scol, plan.sval, q, max_row_slots=plan.row_bound)
        torch.cuda.synchronize()
    finally:
        L.aes_dev_spmm_set_schedule(0)
    assert np.array_equal(bits(to_np(exact)), bits(port.spmm_csr(rp, col, val, deq)))
    assert np.array_equal(bits(to_np(sampled)), bits(port.spmm_sampled(rp, col, val, deq, 32)))


@pytest.mark.parametrize("variant", [0, 46, 48, 49, 30, 34])
@pytest.mark.parametrize("f", [100, 128, 132, 200, 256, 300, 384, 511, 602, 640])
def test_q8_wide_rows_bit_exact(dev, variant, f):
    """int8 on rows wider than one 128-code tile: the wide-row kernel (one
    warp per whole code row; default for 128 < F <= 640, variants 46/48/49)
    and the batch kernel's column tiles (variants 30/34), exact (unbounded
    hub rows) and sampled, every partial last group width."""
    import torch

    from paper_2503_18427_b200 import capi
    L = capi.lib()
    rp, col, val = graphs.power_law(7000, alpha=1.3, max_deg=5000, seed=f)
    g = dev.Graph.from_numpy(rp, col, val)
    x_np = np.random.default_rng(f).uniform(-1, 1, (7000, f)).astype(np.float32)
    q = dev.quantize(torch.from_numpy(x_np).cuda())
    lo, hi = port.fit_params(x_np)
    deq = port.dequantize(port.quantize(x_np, lo, hi), lo, hi)
    plan = dev.SampledPlan(g, 32)
    try:
        L.aes_dev_spmm_set_variant(variant)
        exact = dev.spmm_q8(g.row_ptr, g.col, g.val, q)
        sampled = dev.spmm_q8(plan.srow_ptr, plan.scol, plan.sval, q, max_row_slots=plan.row_bound)
        torch.cuda.synchronize()
    finally:
        L.aes_dev_spmm_set_variant(0)
    assert np.array_equal(bits(to_np(exact)), bits(port.spmm_csr(rp, col, val, deq)))
    assert np.array_equal(bits(to_np(sampled)), bits(port.spmm_sampled(rp, col, val, deq, 32)))


@pytest.mark.parametrize("f", [40, 128])
def test_sharded_gcn_int8_exchange_cuda_ops(dev, f):
    """ShardedGCN(exchange_dtype="int8") on the CUDA ops (device fit_params,
    u8 quantize, fused-dequant SpMM over the code replica) equals the
    reference composition, bit for bit.  (world 2 of the same driver logic:
    tests/test_cpu_dist.py over gloo.)"""
    import torch

    from paper_2503_18427_b200.gcn import ShardedGCN
    rng = np.random.default_rng(f)
    rp, col, _ = graphs.power_law(5000, alpha=1.7, max_deg=800, seed=f)
    nrp, ncol, nval = port.gcn_normalize(rp, col, True)
    x = rng.uniform(-1, 1, (5000, f)).astype(np.float32)
    ws = [rng.uniform(-0.5, 0.5, s).astype(np.float32) for s in [(f, 128), (128, 128), (128, 10)]]
    bs = [np.full(128, 0.01, np.float32), np.full(128, -0.01, np.float32), np.zeros(10, np.float32)]
    g = dev.Graph.from_numpy(nrp, ncol, nval)
    plan = dev.SampledPlan(g, 32)
    model = ShardedGCN(plan.srow_ptr, plan.scol, plan.sval, g.n_rows, [torch.from_numpy(w).cuda() for w in ws],
                       [torch.from_numpy(b).cuda() for b in bs], max_row_slots=plan.row_bound,
                       exchange_dtype="int8")
    out = model.forward(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    want = port.gcn_forward_int8_exchange(nrp, ncol, nval, x, ws, bs, 32)
    assert np.array_equal(bits(to_np(out)), bits(want))


def _edge_graphs():
    """(name, row_ptr, col, val): shapes that stress the balanced schedule's
    row ranges and 32-row end windows."""
    rng = np.random.default_rng(11)
    out = []
    # fewer rows than warps in a wave: most warps get empty ranges
    rp, col, val = graphs.power_law(5, alpha=1.5, max_deg=5, seed=1)
    out.append(("tiny", rp, col, val))
    # long runs of empty rows (crossing several 32-row windows) around a hub row
    n = 3000
    deg = rng.integers(1, 40, n)
    deg[100:400] = 0
    deg[1000:1041] = 0
    deg[2999] = 0
    deg[1500] = 2900
    rows = [np.sort(rng.choice(n, size=int(d), replace=False)) for d in deg]
    rp = np.zeros(n + 1, np.uint64)
    rp[1:] = np.cumsum([r.size for r in rows])
    col = np.concatenate(rows).astype(np.uint32)
    out.append(("empty_runs", rp, col, rng.uniform(-1, 1, col.size).astype(np.float32)))
    # every row empty but the last
    n = 700
    rp = np.zeros(n + 1, np.uint64)
    rp[-1] = 50
    col = np.sort(rng.choice(n, 50, replace=False)).astype(np.uint32)
    out.append(("last_only", rp, col, rng.uniform(-1, 1, 50).astype(np.float32)))
    return out


@pytest.mark.parametrize("sched", [0, 3])
@pytest.mark.parametrize("f", [128, 602])
def test_balanced_schedule_edge_cases(dev, sched, f):
    """Balanced ranges with empty ranges, runs of empty rows across window
    boundaries, hub rows and row shards (srow offset != 0): fp32 and int8,
    exact and sampled, bit-exact vs the oracle."""
    import torch

    from paper_2503_18427_b200 import capi
    L = capi.lib()
    for name, rp, col, val in _edge_graphs():
        n = rp.size - 1
        g = dev.Graph.from_numpy(rp, col, val, n_cols=n)
        x_np = np.random.default_rng(f).uniform(-1, 1, (n, f)).astype(np.float32)
        x = dev.padded(torch.from_numpy(x_np).cuda())
        q = dev.quantize(x)
        lo, hi = port.fit_params(x_np)
        deq = port.dequantize(port.quantize(x_np, lo, hi), lo, hi)
        plan = dev.SampledPlan(g, 32)
        cut = n // 3
        try:
            capi.check(L.aes_dev_spmm_set_schedule(sched))
            exact = dev.spmm_exact(g, x)
            sampled = dev.spmm_plan(plan, x)
            shard = dev.spmm(plan.srow_ptr[cut:], plan.scol, plan.sval, x, max_row_slots=plan.row_bound)
            exact_q = dev.spmm_q8(g.row_ptr, g.col, g.val, q)
            sampled_q = dev.spmm_q8(plan.srow_ptr, plan.scol, plan.sval, q, max_row_slots=plan.row_bound)
            shard_q = dev.spmm_q8(plan.srow_ptr[cut:], plan.scol, plan.sval, q, max_row_slots=plan.row_bound)
            torch.cuda.synchronize()
        finally:
            L.aes_dev_spmm_set_schedule(0)
        want = port.spmm_sampled(rp, col, val, x_np, 32)
        want_q = port.spmm_sampled(rp, col, val, deq, 32)
        assert np.array_equal(bits(to_np(exact)), bits(port.spmm_csr(rp, col, val, x_np))), name
        assert np.array_equal(bits(to_np(sampled)), bits(want)), name
        assert np.array_equal(bits(to_np(shard)), bits(want[cut:])), name
        assert np.array_equal(bits(to_np(exact_q)), bits(port.spmm_csr(rp, col, val, deq))), name
        assert np.array_equal(bits(to_np(sampled_q)), bits(want_q)), name
        assert np.array_equal(bits(to_np(shard_q)), bits(want_q[cut:])), name


@pytest.mark.parametrize("bits", [1, 4, 8])
@pytest.mark.parametrize("shape", [(1000, 128), (333, 7)])
def test_quantize_threshold_table_extremes(dev, bits, shape):
    """The table-driven u8 quantize (quantize.cuh) equals the reference fp64
    formula on adversarial params and values: tiny / huge / subnormal ranges,
    values outside [lo, hi], +-0, +-inf, FLT_MAX, and values packed around
    every code boundary (contiguous float4 path and strided path)."""
    import torch
    rng = np.random.default_rng(bits * 7 + shape[1])
    params = [(-1.0, 1.0), (0.0, 1e-30), (-1e30, 1e30), (-3.5, np.float32(-3.5) + np.float32(4e-6)),
              (1e-40, 2e-40), (-5.0, 5.0), (2.0, 2.0), (-3e38, 3e38), (0.1, 0.7)]
    for lo, hi in params:
        lo, hi = float(np.float32(lo)), float(np.float32(hi))
        n = shape[0] * shape[1]
        span = hi - lo
        with np.errstate(over="ignore"):  # (-3e38, 3e38) +- 10 %: beyond FLT_MAX -> +-inf, also test values
            x = rng.uniform(lo - 0.1 * span, hi + 0.1 * span, n).astype(np.float32) if span else \
                rng.uniform(-1, 1, n).astype(np.float32)
        # values around the code boundaries: the dequantized grid and its neighbours
        grid = np.float32(lo) + (np.arange(n // 4) % ((1 << bits) + 1)).astype(np.float64) * \
            (span / ((1 << bits) - 1) if span else 0.0)
        with np.errstate(over="ignore"):  # grid points past FLT_MAX become inf: fine, also a test value
            g32 = grid.astype(np.float32)
        x[: n // 4] = np.where(rng.random(n // 4) < 0.5, np.nextafter(g32, np.float32(np.inf)),
                               np.nextafter(g32, np.float32(-np.inf)))
        special = np.array([lo, hi, 0.0, -0.0, np.inf, -np.inf, 3.4028235e38, -3.4028235e38, 1e-45, -1e-45],
                           np.float32)
        x[n // 4: n // 4 + special.size] = special
        x = x.reshape(shape)
        xt = torch.from_numpy(x).cuda()
        if shape[1] % 4:
            xt = dev.padded(xt)  # strided rows: the general path
        q = dev.quantize(xt, bits, params=(lo, hi))
        torch.cuda.synchronize()
        want = port.quantize(x, lo, hi, bits)
        got = to_np(q.codes).astype(np.uint16)
        assert np.array_equal(got, want), (lo, hi, bits, int((got != want).sum()))
        # and back: the table-driven flat dequantize (contiguous rows) or the
        # strided one, bit-equal to the reference formula
        deq = to_np(dev.dequantize(q))
        assert np.array_equal(bits_of(deq), bits_of(port.dequantize(want, lo, hi, bits)))


def test_gcn_forward_sharded_c_abi_nccl(dev):
    """aes_gcn_forward_sharded (the C-ABI row-sharded forward over an
    ncclComm_t) on a one-rank NCCL communicator: the replica it
    returns holds the single-GPU forward's logits bit for bit."""
    import ctypes

    import torch

    from paper_2503_18427_b200 import capi
    L = capi.lib()
    nccl = ctypes.CDLL("libnccl.so.2")  # the copy torch already loaded
    comm = ctypes.c_void_p()
    dev_list = (ctypes.c_int * 1)(torch.cuda.current_device())
    assert nccl.ncclCommInitAll(ctypes.byref(comm), 1, dev_list) == 0
    try:
        rng = np.random.default_rng(12)
        n = 2500
        rp, col, _ = graphs.power_law(n, alpha=1.8, max_deg=400, seed=12)
        nrp, ncol, nval = port.gcn_normalize(rp, col, True)
        g = dev.Graph.from_numpy(nrp, ncol, nval)
        plan = dev.SampledPlan(g, 16)
        dims = [40, 64, 64, 7]
        x = rng.uniform(-1, 1, (n, dims[0])).astype(np.float32)
        ws = [rng.uniform(-0.5, 0.5, (a, b)).astype(np.float32) for a, b in zip(dims, dims[1:])]
        bs = [np.full(b, 0.01, np.float32) for b in dims[1:]]
        tw = [torch.from_numpy(w).cuda() for w in ws]
        tb = [torch.from_numpy(b).cuda() for b in bs]
        ld = 64
        ra = torch.zeros((n, ld), device="cuda")
        rb = torch.zeros((n, ld), device="cuda")
        ra[:, : dims[0]] = torch.from_numpy(x).cuda()
        wsb = int(L.aes_gcn_sharded_workspace_bytes(n, ld))
        work = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        dims_h = (ctypes.c_uint64 * 4)(*dims)
        wp = (ctypes.c_void_p * 3)(*[t.data_ptr() for t in tw])
        bp = (ctypes.c_void_p * 3)(*[t.data_ptr() for t in tb])
        out = ctypes.c_void_p()
        out_ld = ctypes.c_uint64()
        capi.check(L.aes_gcn_forward_sharded(plan.srow_ptr.data_ptr(), plan.scol.data_ptr(), plan.sval.data_ptr(),
                                             n, n, 3, dims_h, wp, bp, 1, ra.data_ptr(), rb.data_ptr(), ld,
                                             plan.row_bound, work.data_ptr(), wsb, comm, ctypes.byref(out),
                                             ctypes.byref(out_ld), capi.stream_of(None)))
        torch.cuda.synchronize()
        assert out_ld.value == 8  # round4(7): the class layer moved 8 floats per row, not ld = 64
        rep = ra if out.value == ra.data_ptr() else rb
        got = rep.view(-1)[: n * 8].view(n, 8)[:, : dims[-1]].cpu().numpy()
        want = port.gcn_forward(nrp, ncol, nval, x, ws, bs, 16)
        assert np.array_equal(bits(got), bits(want))
    finally:
        nccl.ncclCommDestroy(comm)


@pytest.mark.parametrize("m,k,n", [(1000, 40, 64), (3000, 128, 128), (257, 7, 300)])
def test_gemm_fused_fit_matches_fit_params(dev, m, k, n):
    """The GEMM epilogue's fused fit_params (first-occurrence min / max over
    the row-major output, non-finite flag) equals fit_params of the output it
    wrote, bit for bit — including ReLU's many +0 ties, -0 from the bias, and
    a non-finite output."""
    import torch
    rng = np.random.default_rng(m + n)
    a = torch.from_numpy(rng.uniform(-1, 1, (m, k)).astype(np.float32)).cuda()
    w = torch.from_numpy(rng.uniform(-0.5, 0.5, (k, n)).astype(np.float32)).cuda()
    b = torch.from_numpy(rng.uniform(-0.1, 0.1, n).astype(np.float32)).cuda()
    b[0] = -0.0
    for relu, finite in ((True, True), (False, True), (False, False)):
        out, res = dev.gemm_bias_act_fit(a, w, b, relu, finite_w=finite)
        want = dev.fit_params_raw(out.contiguous())
        torch.cuda.synchronize()
        assert np.array_equal(bits_of(to_np(res)[:3]), bits_of(to_np(want)[:3])), (relu, finite)
        # and the GEMM itself is the exact one
        assert torch.equal(out, dev.gemm_bias_act(a, w, b, relu, finite_w=finite))
    w2 = w.clone()
    w2[0, 0] = float("inf")
    out, res = dev.gemm_bias_act_fit(a, w2, b, False, finite_w=False)
    torch.cuda.synchronize()
    assert to_np(res).view(np.int32)[2] == 1  # NonFinite


@pytest.mark.parametrize("variant", [0, 46, 49])
@pytest.mark.parametrize("f", [300, 602])
@pytest.mark.parametrize("degrees", [[0], [7], [0, 3], [0, 0, 5, 0, 2500, 1, 0, 33, 0, 0, 64, 65, 1200] * 3,
                                     [0] * 40 + [9] + [0] * 40])
def test_q8_wide_rows_edge_shapes(dev, variant, f, degrees):
    """Wide-row int8 kernel on ragged shapes: empty rows (leading, trailing,
    runs longer than its 32-row window of row ends), a single row, hub rows
    next to empty ones, fewer rows than warps; exact and sampled, plus both
    fast modes against their ring kernel (variant 54)."""
    import torch

    from paper_2503_18427_b200 import capi
    L = capi.lib()
    rp, col, val, n_cols = graphs.with_degrees(degrees, n_cols=3000, seed=f + len(degrees))
    g = dev.Graph.from_numpy(rp, col, val, n_cols=n_cols)
    x_np = np.random.default_rng(f).uniform(-1, 1, (n_cols, f)).astype(np.float32)
    xt = torch.from_numpy(x_np).cuda()
    q = dev.quantize(xt)
    lo, hi = port.fit_params(x_np)
    deq = port.dequantize(port.quantize(x_np, lo, hi), lo, hi)
    plan = dev.SampledPlan(g, 32)
    qa = {m_: dev.quantize_affine(xt, m_) for m_ in ("row", "feature")}
    try:
        L.aes_dev_spmm_set_variant(variant)
        exact = dev.spmm_q8(g.row_ptr, g.col, g.val, q)
        sampled = dev.spmm_q8(plan.srow_ptr, plan.scol, plan.sval, q, max_row_slots=plan.row_bound)
        L.aes_dev_spmm_set_variant(0)
        fast = {m_: dev.spmm_q8_affine(plan.srow_ptr, plan.scol, plan.sval, qa[m_]) for m_ in qa}
        L.aes_dev_spmm_set_variant(54)
        ring = {m_: dev.spmm_q8_affine(plan.srow_ptr, plan.scol, plan.sval, qa[m_]) for m_ in qa}
        torch.cuda.synchronize()
    finally:
        L.aes_dev_spmm_set_variant(0)
    assert np.array_equal(bits(to_np(exact)), bits(port.spmm_csr(rp, col, val, deq)))
    assert np.array_equal(bits(to_np(sampled)), bits(port.spmm_sampled(rp, col, val, deq, 32)))
    for m_ in qa:
        assert torch.equal(fast[m_].view(torch.int32), ring[m_].view(torch.int32))
