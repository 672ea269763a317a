"""TEST INFRASTRUCTURE ONLY — numpy/ctypes face of the plain-C oracle.

Every function here calls ``oracle/aes_oracle.c`` (see its header for the
reference file:line each one restates).  Strategy codes follow the reference
enum order (proj/include/aesspmm/sampling.hpp:14).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ADAPTIVE, AFS, SFS, FULL = 0, 1, 2, 3
_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

_ERRS = {1: "ZeroWidth", 2: "EmptyMatrix", 3: "NonFinite", 4: "invalid QuantParams"}


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            subprocess.run(["make", "-s", "-C", _HERE, "port"], check=True)
        L = C.CDLL(_LIB_PATH)
        u64, u32, i32, vp, f32, f64 = C.c_uint64, C.c_uint32, C.c_int, C.c_void_p, C.c_float, C.c_double
        L.or_select_strategy.argtypes = [u64, u32, vp, vp]
        L.or_hash_start.argtypes = [u32, u64, u32]
        L.or_hash_start.restype = u32
        L.or_row_plan.argtypes = [u64, u32, i32, vp, vp, vp, vp]
        L.or_sample_count.argtypes = [u64, vp, u32, i32, vp]
        L.or_sample_fill.argtypes = [u64, vp, vp, vp, u32, i32, vp, vp, vp]
        L.or_spmm_csr.argtypes = [u64, vp, vp, vp, vp, u64, u64, vp, u64]
        L.or_spmm_csr.restype = None
        L.or_fit_params.argtypes = [vp, u64, u32, vp, vp]
        L.or_quantize.argtypes = [vp, u64, f32, f32, u32, vp]
        L.or_dequantize.argtypes = [vp, u64, f32, f32, u32, vp]
        L.or_dequantize.restype = None
        L.or_dense_matmul.argtypes = [vp, u64, u64, vp, u64, vp]
        L.or_dense_matmul.restype = None
        L.or_bias_act.argtypes = [vp, u64, u64, vp, i32]
        L.or_bias_act.restype = None
        L.or_gcn_normalize.argtypes = [u64, vp, vp, i32, vp, vp, vp, vp]
        L.or_gcn_normalize.restype = None
        L.or_sampling_rate.argtypes = [u64, vp, u32, i32, vp, vp, vp]
        L.or_cdf_stats.argtypes = [vp, u64, vp, vp]
        L.or_cdf_stats.restype = u64
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise ValueError(_ERRS.get(rc, f"oracle error {rc}"))


def select_strategy(nnz: int, w: int):
    ch, cn = np.zeros(1, np.uint32), np.zeros(1, np.uint32)
    _check(lib().or_select_strategy(nnz, w, _p(ch), _p(cn)))
    return int(ch[0]), int(cn[0])


def hash_start(s: int, nnz: int, chunk: int) -> int:
    return int(lib().or_hash_start(s, nnz, chunk))


def row_plan(nnz: int, w: int, strategy: int = ADAPTIVE):
    ch, cn, ns = (np.zeros(1, np.uint32) for _ in range(3))
    starts = np.zeros(max(w, 1), np.uint32)
    _check(lib().or_row_plan(nnz, w, strategy, _p(ch), _p(cn), _p(starts), _p(ns)))
    return int(ch[0]), int(cn[0]), [int(v) for v in starts[: ns[0]]]


def sample_csr(row_ptr, col, val, w: int, strategy: int = ADAPTIVE):
    """Sampled CSR (srow_ptr u64, scol u32, sval f32) in slot order."""
    row_ptr = np.ascontiguousarray(row_ptr, np.uint64)
    col = np.ascontiguousarray(col, np.uint32)
    val = np.ascontiguousarray(val, np.float32)
    n = row_ptr.size - 1
    srow = np.zeros(n + 1, np.uint64)
    _check(lib().or_sample_count(n, _p(row_ptr), w, strategy, _p(srow)))
    s = int(srow[-1])
    scol = np.zeros(max(s, 1), np.uint32)
    sval = np.zeros(max(s, 1), np.float32)
    _check(lib().or_sample_fill(n, _p(row_ptr), _p(col), _p(val), w, strategy,
                                _p(srow), _p(scol), _p(sval)))
    return srow, scol[:s], sval[:s]


def spmm_csr(row_ptr, col, val, b):
    """Ordered fp32 SpMM over a CSR (sampled or original)."""
    row_ptr = np.ascontiguousarray(row_ptr, np.uint64)
    col = np.ascontiguousarray(col, np.uint32)
    val = np.ascontiguousarray(val, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    n = row_ptr.size - 1
    f = b.shape[1]
    c = np.zeros((n, f), np.float32)
    if f == 0 or n == 0:
        return c
    if col.size == 0:
        col = np.zeros(1, np.uint32)
        val = np.zeros(1, np.float32)
    lib().or_spmm_csr(n, _p(row_ptr), _p(col), _p(val), _p(b), f, f, _p(c), f)
    return c


def spmm_sampled(row_ptr, col, val, b, w: int, strategy: int = ADAPTIVE):
    srow, scol, sval = sample_csr(row_ptr, col, val, w, strategy)
    return spmm_csr(srow, scol, sval, b)


def fit_params(x, bits: int = 8):
    x = np.ascontiguousarray(x, np.float32).reshape(-1)
    lo, hi = np.zeros(1, np.float32), np.zeros(1, np.float32)
    _check(lib().or_fit_params(_p(x), x.size, bits, _p(lo), _p(hi)))
    return float(lo[0]), float(hi[0])


def quantize(x, lo: float, hi: float, bits: int = 8):
    x = np.ascontiguousarray(x, np.float32)
    codes = np.zeros(x.shape, np.uint16)
    _check(lib().or_quantize(_p(x), x.size, lo, hi, bits, _p(codes)))
    return codes


def dequantize(codes, lo: float, hi: float, bits: int = 8):
    codes = np.ascontiguousarray(codes, np.uint16)
    x = np.zeros(codes.shape, np.float32)
    lib().or_dequantize(_p(codes), codes.size, lo, hi, bits, _p(x))
    return x


def dense_matmul(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    c = np.zeros((a.shape[0], b.shape[1]), np.float32)
    lib().or_dense_matmul(_p(a), a.shape[0], a.shape[1], _p(b), b.shape[1], _p(c))
    return c


def bias_act(c, bias, relu: bool):
    c = np.array(c, np.float32, copy=True, order="C")
    bias_p = None if bias is None else _p(np.ascontiguousarray(bias, np.float32))
    keep = bias
    lib().or_bias_act(_p(c), c.shape[0], c.shape[1], bias_p, int(relu))
    del keep
    return c


def gcn_normalize(row_ptr, col, add_self_loops: bool = True):
    row_ptr = np.ascontiguousarray(row_ptr, np.uint64)
    col = np.ascontiguousarray(col, np.uint32)
    n = row_ptr.size - 1
    out_ptr = np.zeros(n + 1, np.uint64)
    L = lib()
    colp = _p(col) if col.size else _p(np.zeros(1, np.uint32))
    L.or_gcn_normalize(n, _p(row_ptr), colp, int(add_self_loops), _p(out_ptr), None, None, None)
    nnz = int(out_ptr[-1])
    out_col = np.zeros(max(nnz, 1), np.uint32)
    out_val = np.zeros(max(nnz, 1), np.float32)
    scratch = np.zeros(max(n, 1), np.float32)
    L.or_gcn_normalize(n, _p(row_ptr), colp, int(add_self_loops), _p(out_ptr), _p(out_col),
                       _p(out_val), _p(scratch))
    return out_ptr, out_col[:nnz], out_val[:nnz]


def gcn_forward(row_ptr, col, val, x, weights, biases, w: int | None, strategy: int = ADAPTIVE):
    """Reference gcn_forward (proj/src/gnn.cpp:66-78); w=None -> exact."""
    if w is None:
        srow, scol, sval = (np.ascontiguousarray(row_ptr, np.uint64),
                            np.ascontiguousarray(col, np.uint32),
                            np.ascontiguousarray(val, np.float32))
    else:
        srow, scol, sval = sample_csr(row_ptr, col, val, w, strategy)
    h = np.ascontiguousarray(x, np.float32)
    for l, (wt, bs) in enumerate(zip(weights, biases)):
        agg = spmm_csr(srow, scol, sval, h)
        h = dense_matmul(agg, wt)
        h = bias_act(h, bs if (bs is not None and len(bs)) else None, relu=(l + 1 < len(weights)))
    return h


def gcn_forward_int8_exchange(row_ptr, col, val, x, weights, biases, w: int | None,
                              strategy: int = ADAPTIVE):
    """The int8-exchange variant of gcn_forward, composed
    only of reference functions: every hidden layer output H_l (l >= 1) is
    replaced by dequantize(quantize(H_l, fit_params(H_l, 8))) before the next
    aggregation (quantize.cpp:11-64, gnn.cpp:66-78); the input x and the
    final logits stay fp32."""
    if w is None:
        srow, scol, sval = (np.ascontiguousarray(row_ptr, np.uint64),
                            np.ascontiguousarray(col, np.uint32),
                            np.ascontiguousarray(val, np.float32))
    else:
        srow, scol, sval = sample_csr(row_ptr, col, val, w, strategy)
    h = np.ascontiguousarray(x, np.float32)
    for l, (wt, bs) in enumerate(zip(weights, biases)):
        if l > 0:
            lo, hi = fit_params(h)
            h = dequantize(quantize(h, lo, hi), lo, hi)
        agg = spmm_csr(srow, scol, sval, h)
        h = dense_matmul(agg, wt)
        h = bias_act(h, bs if (bs is not None and len(bs)) else None, relu=(l + 1 < len(weights)))
    return h


def row_mean_normalize(row_ptr, col, val):
    """proj/src/matrix.cpp:146-158."""
    row_ptr = np.ascontiguousarray(row_ptr, np.uint64)
    out = np.array(val, np.float32, copy=True)
    L = lib()
    L.or_row_mean_normalize.argtypes = [C.c_uint64, C.c_void_p, C.c_void_p]
    L.or_row_mean_normalize.restype = None
    if out.size:
        L.or_row_mean_normalize(row_ptr.size - 1, _p(row_ptr), _p(out))
    return row_ptr, np.ascontiguousarray(col, np.uint32), out


def sage_forward(row_ptr, col, val, x, weights, biases, w: int | None, strategy: int = ADAPTIVE):
    """sage_forward (proj/src/gnn.cpp:80-95): H <- act(concat(H, agg) @ W + b)."""
    if w is None:
        srow, scol, sval = (np.ascontiguousarray(row_ptr, np.uint64), np.ascontiguousarray(col, np.uint32),
                            np.ascontiguousarray(val, np.float32))
    else:
        srow, scol, sval = sample_csr(row_ptr, col, val, w, strategy)
    h = np.ascontiguousarray(x, np.float32)
    for l, (wt, bs) in enumerate(zip(weights, biases)):
        agg = spmm_csr(srow, scol, sval, h)
        z = np.ascontiguousarray(np.concatenate([h, agg], axis=1))
        h = dense_matmul(z, wt)
        h = bias_act(h, bs if (bs is not None and len(bs)) else None, relu=(l + 1 < len(weights)))
    return h


def argmax_rows(logits):
    """gnn.cpp:105-116: first maximum under '>' — np.argmax matches for
    non-NaN rows (the only case the checker uses)."""
    return np.argmax(np.asarray(logits, np.float32), axis=1).astype(np.uint32)


def sampling_rate(row_ptr, w: int, strategy: int = ADAPTIVE):
    row_ptr = np.ascontiguousarray(row_ptr, np.uint64)
    n = row_ptr.size - 1
    maxnnz = int(np.max(np.diff(row_ptr))) if n else 0
    seen = np.zeros(max(maxnnz, 1), np.uint8)
    agg, uni = np.zeros(1), np.zeros(1)
    _check(lib().or_sampling_rate(n, _p(row_ptr), w, strategy, _p(seen), _p(agg), _p(uni)))
    return float(agg[0]), float(uni[0])


def cdf_stats(rates):
    """cdf_stats (bench.cpp:124-138) -> (step rates, cumulative fractions)."""
    r = np.array(rates, np.float64)
    if r.size == 0:
        raise ValueError("rates must be nonempty")
    vals, frac = np.zeros(r.size), np.zeros(r.size)
    k = int(lib().or_cdf_stats(_p(r), r.size, _p(vals), _p(frac)))
    return vals[:k], frac[:k]
