"""GPU parity: the sm_100a path (through the C ABI / `_core`) against the CPU
oracle (oracle/aes_oracle.c, pinned to the reference) on the same seeded
inputs.  Integer/index results and fp32 SpMM are compared BIT-EXACTLY: the
reference build has no FMA and accumulates in slot order, and
so do the kernels.  Mirrors proj/tests/test_{sampling,spmm,quantize,gnn}.cpp.
"""
import numpy as np
import pytest

from oracle import port
from tests import graphs

pytestmark = pytest.mark.gpu

STRATS = {"ADAPTIVE": port.ADAPTIVE, "AFS": port.AFS, "SFS": port.SFS, "FULL": port.FULL}


@pytest.fixture(scope="module")
def m():
    import paper_2503_18427_b200 as m
    return m


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def assert_bit_equal(got, want):
    assert got.shape == want.shape
    if not np.array_equal(bits(got), bits(want)):
        diff = np.nonzero(bits(got) != bits(want))
        raise AssertionError(f"{diff[0].size} elements differ; first at {tuple(d[0] for d in diff)}: "
                             f"{got[tuple(d[0] for d in diff)]} vs {want[tuple(d[0] for d in diff)]}")


def make(m, rp, col, val, n_cols=None):
    n = rp.size - 1
    return m.CsrMatrix(n, n if n_cols is None else n_cols, rp, col, val)


# --------------------------------------------------------------------------- sampler
EDGE_DEGREES = [0, 1, 3, 31, 32, 33, 63, 64, 65, 100, 1152, 1153, 1728, 1729, 1430, 2859, 5000, 0, 7]


@pytest.mark.parametrize("strategy", list(STRATS))
@pytest.mark.parametrize("width", [1, 4, 16, 32, 64])
def test_plans_match_oracle_rowwise(m, strategy, width):
    rp, col, val, n_cols = graphs.with_degrees(EDGE_DEGREES, n_cols=6000, seed=width)
    a = make(m, rp, col, val, n_cols)
    ps = m.build_plan_set(a, width, getattr(m.Strategy, strategy))
    assert ps.width == width and len(ps.plans) == len(EDGE_DEGREES)
    for i, d in enumerate(EDGE_DEGREES):
        ch, cn, st = port.row_plan(d, width, STRATS[strategy])
        p = ps.plans[i]
        assert (p.row_id, p.params.chunk_len, p.params.sample_cnt, list(p.starts)) == (i, ch, cn, st)
        assert p.slots == ch * cn


@pytest.mark.parametrize("strategy", list(STRATS))
@pytest.mark.parametrize("width", [4, 8, 32, 128])
def test_sampled_csr_bit_exact(m, strategy, width):
    rp, col, val = graphs.power_law(3000, alpha=1.4, max_deg=2500, seed=width)
    a = make(m, rp, col, val)
    ps = m.build_plan_set(a, width, getattr(m.Strategy, strategy))
    srow, scol, sval = port.sample_csr(rp, col, val, width, STRATS[strategy])
    assert ps.total_slots == int(srow[-1])
    got_srow, got_scol, got_sval = ps.sampled_csr()
    assert np.array_equal(got_srow, srow)
    assert np.array_equal(got_scol, scol)
    assert np.array_equal(bits(got_sval), bits(sval))


def test_hash_collisions_reproduced(m):
    # nnz = 1430, W = 32: range 1429 -> every start is 0
    rp, col, val, n_cols = graphs.with_degrees([1430, 2859, 100], n_cols=4000)
    a = make(m, rp, col, val, n_cols)
    ps = m.build_plan_set(a, 32)
    assert list(ps.plans[0].starts) == [0] * 16 and ps.plans[0].params.chunk_len == 2
    assert list(ps.plans[1].starts)[:5] == [0, 1429, 2858, 1428, 2857]
    assert list(ps.plans[2].starts) == [0, 71, 45, 19, 90, 64, 38, 12]


# --------------------------------------------------------------------------- SpMM fp32
@pytest.mark.parametrize("f", [1, 3, 4, 7, 16, 32, 64, 100, 128, 130, 256, 602])
@pytest.mark.parametrize("strategy", ["ADAPTIVE", "FULL", "AFS", "SFS"])
def test_spmm_sampled_bit_exact(m, f, strategy):
    rng = np.random.default_rng(f)
    rp, col, val = graphs.power_law(1500, alpha=1.3, max_deg=1400, seed=f)
    b = rng.uniform(-1, 1, (1500, f)).astype(np.float32)
    a = make(m, rp, col, val)
    for w in (8, 32):
        ps = m.build_plan_set(a, w, getattr(m.Strategy, strategy))
        got = m.spmm_sampled(a, b, ps)
        want = port.spmm_sampled(rp, col, val, b, w, STRATS[strategy])
        assert_bit_equal(got, want)


@pytest.mark.parametrize("f", [1, 8, 128, 602])
def test_spmm_exact_bit_exact(m, f):
    rng = np.random.default_rng(7 + f)
    rp, col, val = graphs.power_law(2000, alpha=1.2, max_deg=1900, seed=f)
    b = rng.standard_normal((2000, f)).astype(np.float32)
    a = make(m, rp, col, val)
    assert_bit_equal(m.spmm_exact(a, b), port.spmm_csr(rp, col, val, b))
    # full plans and adaptive with W >= max degree are the exact kernel (test_spmm.cpp:124-140)
    assert_bit_equal(m.spmm_sampled(a, b, m.build_plan_set(a, 4, m.Strategy.FULL)), m.spmm_exact(a, b))
    assert_bit_equal(m.spmm_sampled(a, b, m.build_plan_set(a, 4096)), m.spmm_exact(a, b))


def test_replay_oracle_many_instances(m):
    # test_spmm.cpp:142-154: 50 random instances x W in {4, 8, 16}
    rng = np.random.default_rng(13)
    for trial in range(50):
        n = int(2 + rng.integers(0, 62))
        rp, col, val = graphs.random_graph(n, 0.05 + 0.45 * rng.integers(0, 100) / 100.0, rng)
        b = rng.uniform(-1, 1, (n, int(1 + rng.integers(0, 8)))).astype(np.float32)
        a = make(m, rp, col, val)
        for w in (4, 8, 16):
            assert_bit_equal(m.spmm_sampled(a, b, m.build_plan_set(a, w)),
                             port.spmm_sampled(rp, col, val, b, w))


def test_empty_rows_and_empty_matrix(m):
    rp, col, val = graphs.csr_from_rows(3, 3, [[], [2], []], [4.0])
    a = make(m, rp, col, val)
    c = m.spmm_sampled(a, np.ones((3, 2), np.float32), m.build_plan_set(a, 4))
    assert c[0, 0] == 0.0 and c[2, 1] == 0.0 and c[1, 0] == 4.0
    # all-empty and zero-row matrices
    z = m.CsrMatrix(5, 5, np.zeros(6, np.uint64), np.zeros(0, np.uint32), np.zeros(0, np.float32))
    assert np.all(m.spmm_sampled(z, np.ones((5, 3), np.float32), m.build_plan_set(z, 8)) == 0)
    e = m.CsrMatrix(0, 4, np.zeros(1, np.uint64), np.zeros(0, np.uint32), np.zeros(0, np.float32))
    assert m.spmm_exact(e, np.ones((4, 2), np.float32)).shape == (0, 2)


def test_negative_zero_and_denormals(m):
    # +0 start, separate roundings, denormals kept (no FTZ) as on x86 SSE
    rp, col, val = graphs.csr_from_rows(2, 3, [[0, 1, 2], [1]], [1e-30, -1e-30, 3.0, -1.0])
    b = np.array([[1e-10, -0.0], [1e-10, 0.0], [1e-39, 2.0]], np.float32)
    a = make(m, rp, col, val, 3)
    assert_bit_equal(m.spmm_exact(a, b), port.spmm_csr(rp, col, val, b))


def test_errors(m):
    a = m.CsrMatrix(3, 4, np.zeros(4, np.uint64), np.zeros(0, np.uint32), np.zeros(0, np.float32))
    with pytest.raises(ValueError, match="ShapeMismatch"):
        m.spmm_exact(a, np.zeros((5, 2), np.float32))
    plans = m.build_plan_set(a, 8, m.Strategy.FULL)
    with pytest.raises(ValueError, match="ShapeMismatch"):
        m.spmm_sampled(a, np.zeros((5, 2), np.float32), plans)
    a2 = m.CsrMatrix(2, 5, np.zeros(3, np.uint64), np.zeros(0, np.uint32), np.zeros(0, np.float32))
    with pytest.raises(ValueError, match="PlanMatrixMismatch"):
        m.spmm_sampled(a2, np.zeros((5, 2), np.float32), plans)
    with pytest.raises(ValueError, match="ZeroWidth"):
        m.build_plan_set(a, 0)
    with pytest.raises(ValueError, match="ZeroWidth"):
        m.select_strategy(10, 0)


@pytest.mark.parametrize("bad,msg", [
    (([0, 2, 1], [0], [1.0]), "NonMonotonicRowPtr at row 2"),
    (([0, 1, 2], [0, 5], [1.0, 1.0]), "ColumnOutOfRange at row 1"),
    (([0, 2, 2], [1, 1], [1.0, 1.0]), "UnsortedRow at row 0"),
    (([0, 1, 3], [0, 1], [1.0, 1.0]), "LengthMismatch"),
    (([1, 1, 2], [0, 1], [1.0, 1.0]), "LengthMismatch"),
])
def test_csr_validation_messages(m, bad, msg):
    rp, ci, vv = bad
    with pytest.raises(ValueError, match=msg):
        m.CsrMatrix(2, 2, np.array(rp, np.uint64), np.array(ci, np.uint32), np.array(vv, np.float32))


def test_plan_from_other_matrix_same_structure(m):
    # plans depend only on row_nnz: a plan built on A applied to A' with the same
    # structure but new values samples A' (spmm.cpp:54-76 fills per call)
    rp, col, val = graphs.power_law(800, max_deg=700, seed=3)
    val2 = np.random.default_rng(9).uniform(-2, 2, val.size).astype(np.float32)
    a, a2 = make(m, rp, col, val), make(m, rp, col, val2)
    b = np.random.default_rng(1).standard_normal((800, 64)).astype(np.float32)
    ps = m.build_plan_set(a, 16)
    assert_bit_equal(m.spmm_sampled(a2, b, ps), port.spmm_sampled(rp, col, val2, b, 16))


def test_work_counters(m):
    rp, col, val = graphs.power_law(500, max_deg=400, seed=4)
    a = make(m, rp, col, val)
    b = np.ones((500, 6), np.float32)
    c, w = m.spmm_sampled_instrumented(a, b, m.build_plan_set(a, 4, m.Strategy.FULL))
    assert w["fma_count"] == col.size * 6 == m.exact_work(a, b)["fma_count"] and w["loads_a"] == col.size
    c, w = m.spmm_sampled_instrumented(a, b, m.build_plan_set(a, 8))
    assert w["fma_count"] <= col.size * 6 and w["fma_count"] <= 500 * 8 * 6


# --------------------------------------------------------------------------- rates
@pytest.mark.parametrize("strategy", list(STRATS))
@pytest.mark.parametrize("width", [4, 32, 100])
def test_sampling_rate(m, strategy, width):
    rp, col, val = graphs.power_law(1200, alpha=1.3, max_deg=1100, seed=width)
    a = make(m, rp, col, val)
    ps = m.build_plan_set(a, width, getattr(m.Strategy, strategy))
    assert m.sampling_rate(ps, a) == port.sampling_rate(rp, width, STRATS[strategy])


# --------------------------------------------------------------------------- quantization
def test_quantize_golden_values(m):
    qf = m.quantize_with(np.array([[0.5]], np.float32), m.QuantParams(0.0, 1.0, 8))
    assert qf.codes[0, 0] == 127
    qf = m.quantize_with(np.array([[-2.5, 7.25]], np.float32), m.QuantParams(-2.5, 7.25, 8))
    assert list(qf.codes[0]) == [0, 255]
    qf = m.quantize_with(np.array([[3.0, 3.0]], np.float32), m.QuantParams(3.0, 3.0, 8))
    assert list(qf.codes[0]) == [0, 0] and m.dequantize(qf)[0, 0] == 3.0
    qf = m.quantize_with(np.array([[-5.0, 42.0]], np.float32), m.QuantParams(0.0, 1.0, 8))
    assert list(qf.codes[0]) == [0, 255]
    qf = m.quantized_from_codes(np.array([[0, 127, 255]], np.uint16), m.QuantParams(0.0, 1.0, 8))
    x = m.dequantize(qf)
    assert x[0, 0] == 0.0 and x[0, 2] == 1.0 and abs(x[0, 1] - 127 / 255) < 1e-7


@pytest.mark.parametrize("bits_", [1, 4, 8, 12, 16])
@pytest.mark.parametrize("shape,lohi", [((100, 40), (-3, 5)), ((333, 7), (0, 1)), ((64, 602), (100, 250))])
def test_quantize_bit_exact(m, bits_, shape, lohi):
    rng = np.random.default_rng(bits_)
    x = rng.uniform(*lohi, shape).astype(np.float32)
    qf = m.quantize(x, bits=bits_)
    lo, hi = port.fit_params(x, bits_)
    assert (qf.params.x_min, qf.params.x_max, qf.params.bits) == (np.float32(lo), np.float32(hi), bits_)
    codes = port.quantize(x, lo, hi, bits_)
    assert qf.codes.dtype == np.uint16 and np.array_equal(qf.codes, codes)
    assert_bit_equal(m.dequantize(qf), port.dequantize(codes, lo, hi, bits_))
    step = (np.float64(hi) - np.float64(lo)) / ((1 << bits_) - 1)
    assert np.max(np.abs(m.dequantize(qf).astype(np.float64) - x)) <= step


def test_fit_params_first_occurrence_and_errors(m):
    x = np.array([[0.0, -0.0, 1.0, -0.0]], np.float32)
    qf = m.quantize(x)
    assert np.signbit(qf.params.x_min) == np.signbit(port.fit_params(x)[0])
    x2 = np.array([[-0.0, 0.0, 1.0]], np.float32)
    assert np.signbit(m.quantize(x2).params.x_min) == np.signbit(np.float32(port.fit_params(x2)[0]))
    with pytest.raises(ValueError, match="NonFinite"):
        m.quantize(np.array([[1.0, np.nan]], np.float32))
    with pytest.raises(ValueError, match="EmptyMatrix"):
        m.quantize(np.zeros((0, 3), np.float32))
    with pytest.raises(ValueError, match="bits"):
        m.quantize(np.ones((1, 1), np.float32), bits=17)
    for p in (m.QuantParams(1.0, 0.0, 8), m.QuantParams(0.0, 1.0, 0), m.QuantParams(0.0, 1.0, 17)):
        with pytest.raises(ValueError, match="invalid QuantParams"):
            m.quantize_with(np.ones((1, 1), np.float32), p)


def test_codebook_fixed_point(m):
    x = np.random.default_rng(37).uniform(0, 10, (50, 50)).astype(np.float32)
    once = m.quantize(x)
    again = m.quantize_with(m.dequantize(once), once.params)
    assert np.array_equal(once.codes, again.codes)


@pytest.mark.parametrize("f", [4, 16, 128, 602])
def test_spmm_q8_bit_exact(m, f):
    rng = np.random.default_rng(f)
    rp, col, val = graphs.power_law(2500, alpha=1.3, max_deg=2000, seed=f)
    x = rng.uniform(-1, 1, (2500, f)).astype(np.float32)
    a = make(m, rp, col, val)
    qf = m.quantize(x)
    lo, hi = port.fit_params(x)
    deq = port.dequantize(port.quantize(x, lo, hi), lo, hi)
    for w in (16, 32, 64):
        ps = m.build_plan_set(a, w)
        assert_bit_equal(m.spmm_sampled_q8(a, qf, ps), port.spmm_sampled(rp, col, val, deq, w))
    assert_bit_equal(m.spmm_sampled_q8(a, qf), port.spmm_csr(rp, col, val, deq))


# --------------------------------------------------------------------------- GCN
def test_gcn_normalize_bit_exact(m):
    rp, col, val = graphs.power_law(1500, alpha=1.5, max_deg=300, seed=2)
    a = make(m, rp, col, val)
    for loops in (True, False):
        got = m.gcn_normalize(a, loops).to_arrays()
        want = port.gcn_normalize(rp, col, loops)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
        assert np.array_equal(bits(got[2]), bits(want[2]))


@pytest.mark.parametrize("w", [None, 8, 32, 128])
def test_gcn_forward_bit_exact(m, w):
    rng = np.random.default_rng(5)
    rp, col, _ = graphs.power_law(2708, alpha=2.1, max_deg=168, seed=11)
    nrp, ncol, nval = port.gcn_normalize(rp, col, True)
    adj = make(m, nrp, ncol, nval)
    x = rng.uniform(-1, 1, (2708, 33)).astype(np.float32)
    ws = [rng.uniform(-0.5, 0.5, (33, 16)).astype(np.float32), rng.uniform(-0.5, 0.5, (16, 7)).astype(np.float32)]
    bs = [np.full(16, 0.01, np.float32), np.zeros(7, np.float32)]
    plans = None if w is None else m.build_plan_set(adj, w)
    got = m.gcn_forward(adj, x, ws, bs, plans)
    assert_bit_equal(got, port.gcn_forward(nrp, ncol, nval, x, ws, bs, w))


def test_dense_matmul_bit_exact(m):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((300, 130)).astype(np.float32)
    a[rng.random(a.shape) < 0.3] = 0.0
    b = rng.standard_normal((130, 67)).astype(np.float32)
    assert_bit_equal(m.dense_matmul(a, b), port.dense_matmul(a, b))
    with pytest.raises(ValueError, match="ShapeMismatch"):
        m.dense_matmul(a, b[:5])


# --------------------------------------------------------------------------- SAGE / eval (§8f rank 4)
def test_row_mean_normalize_and_sage_forward(m):
    rng = np.random.default_rng(12)
    rp, col, _ = graphs.power_law(2000, alpha=1.6, max_deg=400, seed=12)
    val = np.ones(col.size, np.float32)
    a = make(m, rp, col, val)
    am = m.row_mean_normalize(a)
    mrp, mcol, mval = port.row_mean_normalize(rp, col, val)
    got = am.to_arrays()
    assert np.array_equal(got[0], mrp) and np.array_equal(bits(got[2]), bits(mval))
    x = rng.uniform(-1, 1, (2000, 24)).astype(np.float32)
    ws = [rng.uniform(-0.5, 0.5, (48, 32)).astype(np.float32), rng.uniform(-0.5, 0.5, (64, 6)).astype(np.float32)]
    bs = [np.full(32, 0.01, np.float32), np.zeros(6, np.float32)]
    for w in (None, 16, 32):
        plans = None if w is None else m.build_plan_set(am, w)
        assert_bit_equal(m.sage_forward(am, x, ws, bs, plans), port.sage_forward(mrp, mcol, mval, x, ws, bs, w))
    with pytest.raises(ValueError, match="ShapeMismatch"):
        m.sage_forward(am, x, [ws[1]], [bs[1]])


def test_argmax_and_evaluate(m):
    rng = np.random.default_rng(3)
    logits = rng.standard_normal((5000, 7)).astype(np.float32)
    logits[10, 2] = logits[10, 5] = 9.0  # tie -> lowest index
    assert np.array_equal(m.argmax_rows(logits), port.argmax_rows(logits))
    assert m.argmax_rows(logits)[10] == 2
    labels = rng.integers(0, 7, 5000).astype(np.uint32)
    ref = logits + rng.standard_normal(logits.shape).astype(np.float32) * 0.5
    mask = (rng.random(5000) < 0.3).astype(np.uint8)
    d = m.evaluate(logits, labels, ref, mask)
    pred, refp = port.argmax_rows(logits), port.argmax_rows(ref)
    sel = mask == 1
    assert d["accuracy"] == float(np.sum(pred[sel] == labels[sel])) / float(sel.sum())
    assert d["agreement"] == float(np.sum(pred[sel] == refp[sel])) / float(sel.sum())
    assert list(d["per_class"]) == list(np.bincount(pred[sel], minlength=7))
    with pytest.raises(ValueError, match="LabelOutOfRange"):
        m.evaluate(logits, np.full(5000, 7, np.uint32))
    with pytest.raises(ValueError, match="labels length"):
        m.evaluate(logits, labels[:10])
