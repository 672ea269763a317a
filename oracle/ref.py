"""TEST INFRASTRUCTURE ONLY — the unmodified reference, built into oracle/_ref.

``core()`` imports the reference's own pybind ``_core`` module
(proj/bindings/module.cpp) and ``shim()`` loads ``libaesspmm_ref.so`` (the
reference library + ``oracle/ref_shim.cpp``).  Both exist only where
``make -C oracle ref`` ran (this container; shipped to the GPU box as built
files).  ``available()`` lets tests skip when they are absent.
"""
from __future__ import annotations

import ctypes as C
import importlib.util
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(_HERE, "_ref")
_shim = None
_core = None


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def available() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "libaesspmm_ref.so"))


def core():
    """The reference pybind module, loaded from oracle/_ref."""
    global _core
    if _core is None:
        cands = [f for f in os.listdir(REF_DIR) if f.startswith("_core") and f.endswith(".so")]
        if not cands:
            raise ImportError("reference _core not built (make -C oracle ref)")
        spec = importlib.util.spec_from_file_location("_core", os.path.join(REF_DIR, cands[0]))
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _core = mod
    return _core


def shim():
    global _shim
    if _shim is None:
        L = C.CDLL(os.path.join(REF_DIR, "libaesspmm_ref.so"))
        u64, u32, i32, vp, f32, f64 = C.c_uint64, C.c_uint32, C.c_int, C.c_void_p, C.c_float, C.c_double
        L.ref_last_error.restype = C.c_char_p
        L.ref_csr_new.argtypes = [u64, u64, vp, vp, vp]
        L.ref_csr_new.restype = vp
        L.ref_csr_free.argtypes = [vp]
        L.ref_csr_rows.argtypes = [vp]
        L.ref_csr_rows.restype = u64
        L.ref_csr_nnz.argtypes = [vp]
        L.ref_csr_nnz.restype = u64
        L.ref_csr_copy.argtypes = [vp, vp, vp, vp]
        L.ref_gen_synthetic.argtypes = [u64, f64, u32, u64]
        L.ref_gen_synthetic.restype = vp
        L.ref_gcn_normalize.argtypes = [vp, i32]
        L.ref_gcn_normalize.restype = vp
        L.ref_build_plans.argtypes = [vp, u32, i32, vp, vp, vp, vp, u64]
        L.ref_sampling_rate.argtypes = [vp, u32, i32, vp, vp]
        L.ref_sampling_rate_per_row.argtypes = [vp, u32, i32, vp]
        L.ref_cdf_stats.argtypes = [vp, u64, vp, vp, vp]
        L.ref_spmm_sampled.argtypes = [vp, vp, u64, u64, u32, i32, C.c_uint, vp]
        L.ref_spmm_exact.argtypes = [vp, vp, u64, u64, C.c_uint, vp]
        L.ref_time_spmm_sampled.argtypes = [vp, vp, u64, u64, u32, i32, C.c_uint, i32, vp, vp, vp]
        L.ref_fit_params.argtypes = [vp, u64, u64, u32, vp, vp]
        L.ref_quantize.argtypes = [vp, u64, u64, f32, f32, u32, vp]
        L.ref_dequantize.argtypes = [vp, u64, u64, f32, f32, u32, vp]
        L.ref_dense_matmul.argtypes = [vp, u64, u64, vp, u64, vp]
        L.ref_gcn_forward.argtypes = [vp, vp, vp, i32, vp, vp, u32, i32, vp]
        L.ref_gnn_forward.argtypes = [i32, vp, vp, vp, i32, vp, vp, u32, i32, vp]
        cp = C.c_char_p
        L.ref_save_csr_binary.argtypes = [vp, cp]
        L.ref_load_csr_binary.argtypes = [cp]
        L.ref_load_csr_binary.restype = vp
        L.ref_save_fmat_f32.argtypes = [vp, u64, u64, cp]
        L.ref_save_fmat_q8.argtypes = [vp, u64, u64, f32, f32, cp]
        L.ref_load_fmat.argtypes = [cp, vp, vp, vp, vp, vp, vp, vp]
        L.ref_row_mean_normalize.argtypes = [vp]
        L.ref_row_mean_normalize.restype = vp
        L.ref_evaluate.argtypes = [vp, u64, u64, vp, vp, vp, vp, vp, vp]
        _shim = L
    return _shim


def _chk(rc):
    if rc != 0:
        raise ValueError(shim().ref_last_error().decode())


class RefCsr:
    """Owning handle to a reference aes::CsrMatrix."""

    def __init__(self, handle):
        self.h = handle

    @classmethod
    def from_arrays(cls, n_rows, n_cols, row_ptr, col, val):
        rp = np.ascontiguousarray(row_ptr, np.uint64)
        ci = np.ascontiguousarray(col, np.uint32) if len(col) else np.zeros(1, np.uint32)
        vv = np.ascontiguousarray(val, np.float32) if len(val) else np.zeros(1, np.float32)
        return cls(shim().ref_csr_new(n_rows, n_cols, _p(rp), _p(ci), _p(vv)))

    def __del__(self):
        if getattr(self, "h", None) and _shim is not None:
            _shim.ref_csr_free(self.h)
            self.h = None

    @property
    def n_rows(self):
        return int(shim().ref_csr_rows(self.h))

    def arrays(self):
        n, nnz = self.n_rows, int(shim().ref_csr_nnz(self.h))
        rp = np.zeros(n + 1, np.uint64)
        ci = np.zeros(max(nnz, 1), np.uint32)
        vv = np.zeros(max(nnz, 1), np.float32)
        shim().ref_csr_copy(self.h, _p(rp), _p(ci), _p(vv))
        return rp, ci[:nnz], vv[:nnz]


def gen_synthetic(n, alpha, max_degree, seed):
    h = shim().ref_gen_synthetic(n, alpha, max_degree, seed)
    if not h:
        raise ValueError(shim().ref_last_error().decode())
    return RefCsr(h)


def gcn_normalize(csr: RefCsr, add_self_loops=True) -> RefCsr:
    return RefCsr(shim().ref_gcn_normalize(csr.h, int(add_self_loops)))


def build_plans(csr: RefCsr, width, strategy):
    n = csr.n_rows
    chunk = np.zeros(max(n, 1), np.uint32)
    cnt = np.zeros(max(n, 1), np.uint32)
    sp = np.zeros(n + 1, np.uint64)
    _chk(shim().ref_build_plans(csr.h, width, strategy, _p(chunk), _p(cnt), _p(sp), None, 0))
    starts = np.zeros(max(int(sp[-1]), 1), np.uint32)
    _chk(shim().ref_build_plans(csr.h, width, strategy, _p(chunk), _p(cnt), _p(sp), _p(starts),
                                starts.size))
    return chunk[:n], cnt[:n], sp, starts[: int(sp[-1])]


def sampling_rate_per_row(csr: RefCsr, width, strategy=0):
    out = np.zeros(max(csr.n_rows, 1), np.float64)
    _chk(shim().ref_sampling_rate_per_row(csr.h, width, strategy, _p(out)))
    return out[: csr.n_rows]


def cdf_stats(rates):
    """The reference's cdf_stats (bench.cpp:124-138) -> (rates, fractions)."""
    r = np.ascontiguousarray(rates, np.float64)
    vals, frac = np.zeros(max(r.size, 1)), np.zeros(max(r.size, 1))
    n = np.zeros(1, np.uint64)
    _chk(shim().ref_cdf_stats(_p(r), r.size, _p(vals), _p(frac), _p(n)))
    return vals[: int(n[0])], frac[: int(n[0])]


def spmm_sampled(csr: RefCsr, b, width, strategy, threads=0):
    b = np.ascontiguousarray(b, np.float32)
    c = np.zeros((csr.n_rows, b.shape[1]), np.float32)
    _chk(shim().ref_spmm_sampled(csr.h, _p(b), b.shape[0], b.shape[1], width, strategy,
                                 threads, _p(c)))
    return c


def spmm_exact(csr: RefCsr, b, threads=0):
    b = np.ascontiguousarray(b, np.float32)
    c = np.zeros((csr.n_rows, b.shape[1]), np.float32)
    _chk(shim().ref_spmm_exact(csr.h, _p(b), b.shape[0], b.shape[1], threads, _p(c)))
    return c


def time_spmm_sampled(csr: RefCsr, b, width, strategy, threads, reps, want_output=False):
    b = np.ascontiguousarray(b, np.float32)
    ms = np.zeros(reps)
    plan_ms = np.zeros(1)
    c = np.zeros((csr.n_rows, b.shape[1]), np.float32) if want_output else None
    _chk(shim().ref_time_spmm_sampled(csr.h, _p(b), b.shape[0], b.shape[1], width, strategy,
                                      threads, reps, _p(plan_ms), _p(ms),
                                      _p(c) if c is not None else None))
    return float(plan_ms[0]), ms, c


def fit_params(x, bits=8):
    x = np.ascontiguousarray(x, np.float32)
    lo, hi = np.zeros(1, np.float32), np.zeros(1, np.float32)
    r, c = (x.shape[0], x.shape[1]) if x.ndim == 2 else (1, x.size)
    _chk(shim().ref_fit_params(_p(x), r, c, bits, _p(lo), _p(hi)))
    return float(lo[0]), float(hi[0])


def quantize(x, lo, hi, bits=8):
    x = np.ascontiguousarray(x, np.float32)
    codes = np.zeros(x.shape, np.uint16)
    r, c = (x.shape[0], x.shape[1]) if x.ndim == 2 else (1, x.size)
    _chk(shim().ref_quantize(_p(x), r, c, lo, hi, bits, _p(codes)))
    return codes


def dequantize(codes, lo, hi, bits=8):
    codes = np.ascontiguousarray(codes, np.uint16)
    x = np.zeros(codes.shape, np.float32)
    r, c = (codes.shape[0], codes.shape[1]) if codes.ndim == 2 else (1, codes.size)
    _chk(shim().ref_dequantize(_p(codes), r, c, lo, hi, bits, _p(x)))
    return x


def dense_matmul(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    c = np.zeros((a.shape[0], b.shape[1]), np.float32)
    _chk(shim().ref_dense_matmul(_p(a), a.shape[0], a.shape[1], _p(b), b.shape[1], _p(c)))
    return c


def save_csr_binary(csr: RefCsr, path: str):
    _chk(shim().ref_save_csr_binary(csr.h, path.encode()))


def load_csr_binary(path: str) -> RefCsr:
    h = shim().ref_load_csr_binary(path.encode())
    if not h:
        raise ValueError(shim().ref_last_error().decode())
    return RefCsr(h)


def save_fmat_f32(x, path: str):
    x = np.ascontiguousarray(x, np.float32)
    _chk(shim().ref_save_fmat_f32(_p(x), x.shape[0], x.shape[1], path.encode()))


def save_fmat_q8(codes, lo, hi, path: str):
    codes = np.ascontiguousarray(codes, np.uint16)
    _chk(shim().ref_save_fmat_q8(_p(codes), codes.shape[0], codes.shape[1], lo, hi, path.encode()))


def load_fmat(path: str):
    """(dtype, array) where array is f32 features (dtype 0) or
    (codes u16, lo, hi) (dtype 1) — reference load_features (io.cpp:183-220)."""
    dt = np.zeros(1, np.int32)
    r, c = np.zeros(1, np.uint64), np.zeros(1, np.uint64)
    lo, hi = np.zeros(1, np.float32), np.zeros(1, np.float32)
    _chk(shim().ref_load_fmat(path.encode(), _p(dt), _p(r), _p(c), _p(lo), _p(hi), None, None))
    rows, cols = int(r[0]), int(c[0])
    if dt[0] == 0:
        x = np.zeros((rows, cols), np.float32)
        _chk(shim().ref_load_fmat(path.encode(), _p(dt), _p(r), _p(c), _p(lo), _p(hi), _p(x), None))
        return 0, x
    codes = np.zeros((rows, cols), np.uint16)
    _chk(shim().ref_load_fmat(path.encode(), _p(dt), _p(r), _p(c), _p(lo), _p(hi), None, _p(codes)))
    return 1, (codes, float(lo[0]), float(hi[0]))


def row_mean_normalize(csr: RefCsr) -> RefCsr:
    return RefCsr(shim().ref_row_mean_normalize(csr.h))


def sage_forward(csr: RefCsr, x, weights, biases, width, strategy=0):
    """Reference sage_forward (gnn.cpp:80-95); width=None -> exact."""
    x = np.ascontiguousarray(x, np.float32)
    dims = np.array([x.shape[1]] + [w.shape[1] for w in weights], np.uint64)
    wcat = np.concatenate([np.ascontiguousarray(w, np.float32).ravel() for w in weights])
    bcat = np.concatenate([np.ascontiguousarray(b, np.float32).ravel() for b in biases])
    out = np.zeros((x.shape[0], int(dims[-1])), np.float32)
    _chk(shim().ref_gnn_forward(1, csr.h, _p(x), _p(dims), len(weights), _p(wcat), _p(bcat),
                                0 if width is None else width, strategy, _p(out)))
    return out


def evaluate(logits, labels, ref_logits=None, mask=None):
    logits = np.ascontiguousarray(logits, np.float32)
    labels = np.ascontiguousarray(labels, np.uint32)
    r, c = logits.shape
    acc, agree = np.zeros(1), np.zeros(1)
    pc = np.zeros(c, np.uint64)
    rl = None if ref_logits is None else np.ascontiguousarray(ref_logits, np.float32)
    mk = None if mask is None else np.ascontiguousarray(mask, np.uint8)
    _chk(shim().ref_evaluate(_p(logits), r, c, _p(labels), None if rl is None else _p(rl),
                             None if mk is None else _p(mk), _p(acc), _p(agree), _p(pc)))
    return float(acc[0]), float(agree[0]), pc


def gcn_forward(csr: RefCsr, x, weights, biases, width, strategy=0):
    """width=None -> exact path (plans=nullptr)."""
    x = np.ascontiguousarray(x, np.float32)
    dims = np.array([x.shape[1]] + [w.shape[1] for w in weights], np.uint64)
    wcat = np.concatenate([np.ascontiguousarray(w, np.float32).ravel() for w in weights])
    bcat = np.concatenate([np.ascontiguousarray(b, np.float32).ravel() for b in biases])
    out = np.zeros((x.shape[0], int(dims[-1])), np.float32)
    _chk(shim().ref_gcn_forward(csr.h, _p(x), _p(dims), len(weights), _p(wcat), _p(bcat),
                                0 if width is None else width, strategy, _p(out)))
    return out
