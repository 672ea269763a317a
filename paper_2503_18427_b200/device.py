"""Device-resident AES-SpMM API over torch CUDA tensors (zero host copies).

Layout in HBM:
  * graph CSR: ``row_ptr`` int64 [n+1] (the reference's u64), ``col`` int32
    [nnz] (u32 bits), ``val`` float32 [nnz];
  * sampled CSR (one per (graph, W, strategy), reused by every layer):
    ``srow_ptr`` int64 [n+1], ``scol`` int32 [S], ``sval`` float32 [S] in the
    reference's slot order (slot s + j*cnt, proj/src/spmm.cpp:68-76);
  * dense features: row-major float32 with the row stride padded to a
    multiple of 4 floats (16 B) so every gathered row is float4-aligned
    (F = 602 is stored with ld = 604); int8 codes likewise with ld % 4 == 0.

Every function launches sm_100a kernels from libaescuda.so through the C ABI
on the caller's (default: torch's current) stream and never synchronises
unless it has to read a size back (plan building, quantization params).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import capi
from .capi import check, lib, ptr, stream_of


def _round4(x: int) -> int:
    return (x + 3) & ~3


def padded(x: torch.Tensor) -> torch.Tensor:
    """Return a view of ``x`` whose row stride is a multiple of 4 elements."""
    if x.dim() != 2:
        raise ValueError("expected a 2-D tensor")
    if x.stride(1) == 1 and x.stride(0) % 4 == 0 and x.data_ptr() % 16 == 0:
        return x
    r, f = x.shape
    buf = torch.zeros((r, _round4(max(f, 1))), dtype=x.dtype, device=x.device)
    buf[:, :f].copy_(x)
    return buf[:, :f]


def empty_padded(rows: int, cols: int, dtype=torch.float32, device="cuda") -> torch.Tensor:
    """[rows, cols] view of a buffer whose rows are padded to 16 bytes.  The
    pad columns are zeroed: the vector kernels gather whole 16-B units, so a
    padded buffer read as an operand never feeds uninitialized bytes (they
    only ever reach pad output columns, but compute-sanitizer initcheck
    flags the read)."""
    per16 = max(1, 16 // torch.empty((), dtype=dtype).element_size())
    width = -(-max(cols, 1) // per16) * per16
    buf = torch.empty((rows, width), dtype=dtype, device=device)
    if width != cols and rows:
        buf[:, cols:].zero_()
    return buf[:, :cols]


@dataclass
class Graph:
    """A CSR matrix resident in HBM."""

    row_ptr: torch.Tensor  # int64 [n+1]
    col: torch.Tensor      # int32 [nnz]
    val: torch.Tensor      # float32 [nnz]
    n_cols: int

    @property
    def n_rows(self) -> int:
        return self.row_ptr.numel() - 1

    @property
    def nnz(self) -> int:
        return self.col.numel()

    @classmethod
    def from_numpy(cls, row_ptr, col, val, n_cols=None, device="cuda") -> "Graph":
        import numpy as np

        rp = torch.from_numpy(np.ascontiguousarray(row_ptr, np.uint64).view(np.int64)).to(device)
        ci = torch.from_numpy(np.ascontiguousarray(col, np.uint32).view(np.int32)).to(device)
        vv = torch.from_numpy(np.ascontiguousarray(val, np.float32)).to(device)
        n = rp.numel() - 1
        return cls(rp, ci, vv, n if n_cols is None else int(n_cols))

    def rows(self, begin: int, end: int) -> "Graph":
        """Row shard [begin, end) as a view; row_ptr stays absolute."""
        return Graph(self.row_ptr[begin:end + 1], self.col, self.val, self.n_cols)


class SampledPlan:
    """build_plan_set + the buffer fill, materialised once in HBM
    (proj/src/sampling.cpp:104-118, proj/src/spmm.cpp:54-76)."""

    def __init__(self, graph: Graph, width: int, strategy="adaptive", stream=None):
        L = lib()
        self.width = int(width)
        self.strategy = capi.strategy_code(strategy)
        n = graph.n_rows
        dev = graph.row_ptr.device
        st = stream_of(stream)
        self.n_rows = n
        self.srow_ptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
        ws_bytes = L.aes_dev_scan_workspace_bytes(n)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        # (no per-row (chunk, cnt) output: the fill re-derives them per row)
        check(L.aes_dev_sample_plan(ptr(graph.row_ptr), n, self.width, self.strategy, ptr(self.srow_ptr),
                                    None, ptr(ws), ws_bytes, st))
        # the absolute offset of this (possibly sharded) row range
        self.base = int(self.srow_ptr[0].item()) if n else 0
        self.total_slots = int(self.srow_ptr[-1].item()) - self.base
        self.scol = torch.empty(max(self.total_slots, 1), dtype=torch.int32, device=dev)
        self.sval = torch.empty(max(self.total_slots, 1), dtype=torch.float32, device=dev)
        check(L.aes_dev_sample_fill(ptr(graph.row_ptr), ptr(graph.row_ptr), ptr(graph.col), ptr(graph.val), n,
                                    self.width, self.strategy, ptr(self.srow_ptr), ptr(self.scol),
                                    ptr(self.sval), st))
        del ws

    @property
    def row_bound(self) -> int:
        """Most slots any row can have: W for Adaptive/Afs/Sfs, unbounded (0) for FULL."""
        return 0 if self.strategy == capi.strategy_code("full") else self.width

    def algorithmic_bytes(self, f: int, elem_bytes: int = 4) -> int:
        """Bytes one SpMM over this plan must move:
        8(N+1) row offsets + 8S (col, val) + e*F*S gathered + 4*F*N written."""
        n, s = self.n_rows, self.total_slots
        return 8 * (n + 1) + 8 * s + elem_bytes * f * s + 4 * f * n


def spmm(srow_ptr, scol, sval, b: torch.Tensor, out: torch.Tensor | None = None, stream=None,
         max_row_slots: int = 0) -> torch.Tensor:
    """C = A_sampled @ B (bit-exact with the reference spmm_sampled).
    max_row_slots bounds the slots of any row (0 = unbounded; picks the
    row-group schedule, see aes_dev_spmm_f32_ex)."""
    n = srow_ptr.numel() - 1
    f = b.shape[1]
    if out is None:
        out = empty_padded(n, f, device=b.device)
    check(lib().aes_dev_spmm_f32_ex(ptr(srow_ptr), ptr(scol), ptr(sval), n, ptr(b), b.stride(0), f, ptr(out),
                                    out.stride(0), max_row_slots, stream_of(stream)))
    return out


def spmm_plan(plan: SampledPlan, b: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    return spmm(plan.srow_ptr, plan.scol, plan.sval, b, out, stream, plan.row_bound)


def spmm_exact(g: Graph, b: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    return spmm(g.row_ptr, g.col, g.val, b, out, stream)


@dataclass
class QuantizedDevice:
    """int8 codes (bits <= 8) in HBM with their global params and the exact
    dequantization table (proj/include/aesspmm/quantize.hpp:10-25)."""

    codes: torch.Tensor  # uint8 [rows, cols] view with ld % 4 == 0
    x_min: float
    x_max: float
    bits: int
    lut: torch.Tensor    # float32 [256]


def fit_params(x: torch.Tensor, stream=None):
    """Global (x_min, x_max) — quantize.cpp:11-21.  Synchronises once."""
    L = lib()
    x = x.contiguous()
    n = x.numel()
    if n == 0:
        raise ValueError("EmptyMatrix")
    ws_bytes = L.aes_dev_scan_workspace_bytes(1)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=x.device)
    res = torch.empty(4, dtype=torch.float32, device=x.device)
    check(L.aes_dev_fit_params(ptr(x), n, ptr(res), ptr(ws), ws_bytes, stream_of(stream)))
    r = res[:3].cpu()  # word 3 is padding the kernel never writes
    if r.view(torch.int32)[2].item() != 0:
        raise ValueError("NonFinite")
    return float(r[0]), float(r[1])


def fit_params_raw(x: torch.Tensor, stream=None) -> torch.Tensor:
    """fit_params without the host sync: float32 [x_min, x_max, flag, -] on the
    device, flag (int32 bits) = 1 when a non-finite element was seen."""
    L = lib()
    x = x.contiguous()
    n = x.numel()
    if n == 0:
        raise ValueError("EmptyMatrix")
    ws_bytes = L.aes_dev_scan_workspace_bytes(1)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=x.device)
    res = torch.empty(4, dtype=torch.float32, device=x.device)
    check(L.aes_dev_fit_params(ptr(x), n, ptr(res), ptr(ws), ws_bytes, stream_of(stream)))
    return res


def dequant_lut(lo: float, hi: float, bits: int = 8, dev="cuda", stream=None) -> torch.Tensor:
    """The 256-entry exact dequantization table (quantize.cpp:53-64)."""
    lut = torch.zeros(256, dtype=torch.float32, device=dev)
    check(lib().aes_dev_dequant_lut(lo, hi, bits, ptr(lut), stream_of(stream)))
    return lut


def quantize(x: torch.Tensor, bits: int = 8, params=None, stream=None, out=None) -> QuantizedDevice:
    """quantize(x, fit_params(x, bits)) — quantize.cpp:23-51, codes kept as u8.
    out: optional u8 [rows, cols] view (row stride free) the codes go into."""
    if not 1 <= bits <= 8:
        raise ValueError("device int8 path takes bits in 1..8")
    L = lib()
    lo, hi = params if params is not None else fit_params(x, stream)
    rows, cols = x.shape
    if out is not None:
        if out.dtype != torch.uint8 or tuple(out.shape) != (rows, cols) or out.stride(1) != 1:
            raise ValueError("out must be a uint8 [rows, cols] row-major view")
        codes = out
    else:
        codes = empty_padded(rows, cols, dtype=torch.uint8, device=x.device)
    st = stream_of(stream)
    check(L.aes_dev_quantize(ptr(x), rows, cols, x.stride(0), lo, hi, bits, ptr(codes), codes.stride(0), st))
    lut = torch.zeros(256, dtype=torch.float32, device=x.device)
    check(L.aes_dev_dequant_lut(lo, hi, bits, ptr(lut), st))
    return QuantizedDevice(codes, lo, hi, bits, lut)


def load_fmat(path: str, device="cuda"):
    """FMAT file (proj/src/io.cpp:149-220 format) straight into HBM, streamed
    through pinned double buffers.  Returns (features, load_ms): a float32
    tensor (row stride padded to 4) for dtype 0, a QuantizedDevice (u8 codes +
    exact LUT, no host dequantization) for dtype 1."""
    import ctypes

    import numpy as np

    L = lib()
    dt = np.zeros(1, np.int32)
    r, c = np.zeros(1, np.uint64), np.zeros(1, np.uint64)
    lo, hi = np.zeros(1, np.float32), np.zeros(1, np.float32)
    check(L.aes_fmat_info(path.encode(), dt.ctypes.data, r.ctypes.data, c.ctypes.data, lo.ctypes.data,
                          hi.ctypes.data))
    rows, cols = int(r[0]), int(c[0])
    ms = ctypes.c_double()
    if dt[0] == 0:
        out = empty_padded(rows, cols, device=device)
        check(L.aes_fmat_load_device(path.encode(), ptr(out), out.stride(0), ctypes.addressof(ms)))
        return out, ms.value
    codes = empty_padded(rows, cols, dtype=torch.uint8, device=device)
    check(L.aes_fmat_load_device(path.encode(), ptr(codes), codes.stride(0), ctypes.addressof(ms)))
    lut = torch.zeros(256, dtype=torch.float32, device=device)
    check(L.aes_dev_dequant_lut(float(lo[0]), float(hi[0]), 8, ptr(lut), stream_of(None)))
    return QuantizedDevice(codes, float(lo[0]), float(hi[0]), 8, lut), ms.value


def dequantize(q: QuantizedDevice, stream=None) -> torch.Tensor:
    rows, cols = q.codes.shape
    out = empty_padded(rows, cols, device=q.codes.device)
    check(lib().aes_dev_dequantize(ptr(q.codes), rows, cols, q.codes.stride(0), q.x_min, q.x_max, q.bits,
                                   ptr(out), out.stride(0), stream_of(stream)))
    return out


def spmm_q8(srow_ptr, scol, sval, q: QuantizedDevice, out=None, stream=None, max_row_slots: int = 0) -> torch.Tensor:
    """spmm(A, dequantize(Q)) with dequantization fused into the u8 gather."""
    n = srow_ptr.numel() - 1
    f = q.codes.shape[1]
    if out is None:
        out = empty_padded(n, f, device=q.codes.device)
    check(lib().aes_dev_spmm_q8_ex(ptr(srow_ptr), ptr(scol), ptr(sval), n, ptr(q.codes), q.codes.stride(0), f,
                                   ptr(q.lut), ptr(out), out.stride(0), max_row_slots, stream_of(stream)))
    return out


AFFINE_MODES = {"row": 0, "feature": 1}


@dataclass
class QuantizedAffine:
    """FAST MODE int8 codes (affine.cu): u8 codes with a (scale, offset) pair
    per row ("row") or per column ("feature"); x^ = q * s + m.  Not the
    reference's global min/max codes — bounded, not bit-exact."""

    codes: torch.Tensor   # uint8 [rows, cols] view, ld % 16 == 0
    params: torch.Tensor  # float32 [rows or cols, 2] = (s, m)
    mode: str


def quantize_affine(x: torch.Tensor, mode: str = "row", stream=None) -> QuantizedAffine:
    """Per-row / per-feature 8-bit codes of x (one pass for "row", three
    small passes for "feature"); raises ValueError("NonFinite") on inf/NaN."""
    if mode not in AFFINE_MODES:
        raise ValueError("mode must be 'row' or 'feature'")
    L = lib()
    rows, cols = x.shape
    codes = empty_padded(rows, cols, dtype=torch.uint8, device=x.device)
    params = torch.empty((rows if mode == "row" else cols, 2), dtype=torch.float32, device=x.device)
    wsb = int(L.aes_quantize_affine_workspace_bytes(rows, cols, AFFINE_MODES[mode]))
    ws = torch.empty(wsb, dtype=torch.uint8, device=x.device)
    bad = torch.zeros(1, dtype=torch.int32, device=x.device)
    check(L.aes_dev_quantize_affine(ptr(x), rows, cols, x.stride(0), AFFINE_MODES[mode], ptr(codes),
                                    codes.stride(0), ptr(params), ptr(bad), ptr(ws), wsb, stream_of(stream)))
    if int(bad.item()):
        raise ValueError("NonFinite")
    return QuantizedAffine(codes, params, mode)


def dequantize_affine(q: QuantizedAffine, stream=None) -> torch.Tensor:
    rows, cols = q.codes.shape
    out = empty_padded(rows, cols, device=q.codes.device)
    check(lib().aes_dev_dequantize_affine(ptr(q.codes), rows, cols, q.codes.stride(0), AFFINE_MODES[q.mode],
                                          ptr(q.params), ptr(out), out.stride(0), stream_of(stream)))
    return out


def spmm_q8_affine(srow_ptr, scol, sval, q: QuantizedAffine, out=None, stream=None) -> torch.Tensor:
    """spmm(A, dequantize_affine(Q)) with the affine decode fused into the u8 gather."""
    n = srow_ptr.numel() - 1
    f = q.codes.shape[1]
    if out is None:
        out = empty_padded(n, f, device=q.codes.device)
    check(lib().aes_dev_spmm_q8_affine(ptr(srow_ptr), ptr(scol), ptr(sval), n, ptr(q.codes), q.codes.stride(0), f,
                                       AFFINE_MODES[q.mode], ptr(q.params), ptr(out), out.stride(0),
                                       stream_of(stream)))
    return out


def weights_finite(w: torch.Tensor, stream=None) -> bool:
    """True when w has no inf/NaN (device reduction, one sync)."""
    flag = torch.zeros(1, dtype=torch.int32, device=w.device)
    check(lib().aes_dev_all_finite(ptr(w), w.numel(), ptr(flag), stream_of(stream)))
    return int(flag.item()) == 0


def all_weights_finite(weights, stream=None) -> list[bool]:
    """weights_finite for several tensors with a single device read-back."""
    if not weights:
        return []
    flags = torch.zeros(len(weights), dtype=torch.int32, device=weights[0].device)
    for i, w in enumerate(weights):
        check(lib().aes_dev_all_finite(ptr(w), w.numel(), flags.data_ptr() + 4 * i, stream_of(stream)))
    return [v == 0 for v in flags.cpu().tolist()]


def gemm_bias_act(a: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None, relu: bool, out=None,
                  stream=None, finite_w: bool | None = False) -> torch.Tensor:
    """act(a @ w + bias) with the reference's ordered fp32 arithmetic
    (gnn.cpp:11-52).  finite_w=True (or None: check on the device) lets the
    kernel drop the reference's zero-skip, which is result-neutral then."""
    import ctypes

    m, k = a.shape
    k2, n = w.shape
    if k != k2:
        raise ValueError("ShapeMismatch")
    w = w.contiguous()
    if finite_w is None:
        finite_w = weights_finite(w, stream)
    if out is None:
        out = empty_padded(m, n, device=a.device)
        if out.stride(0) != n:
            out.as_strided((m, out.stride(0)), (out.stride(0), 1))[:, n:].zero_()
    dsts = (ctypes.c_void_p * 1)(ptr(out))
    check(lib().aes_dev_gemm_bias_act_ex(ptr(a), m, k, a.stride(0), ptr(w), n, w.stride(0),
                                         ptr(bias) if bias is not None and bias.numel() else None, int(relu),
                                         int(bool(finite_w)), ctypes.cast(dsts, ctypes.c_void_p), None, 1, 0,
                                         out.stride(0), stream_of(stream)))
    return out


def gemm_bias_act_fit(a: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None, relu: bool, out=None,
                      stream=None, finite_w: bool = False):
    """gemm_bias_act with fit_params of the output fused into the GEMM
    epilogue: returns (out, res) where res = float32 [x_min, x_max, flag, -]
    on the device (flag int32 bits: 1 = non-finite), as fit_params_raw(out)."""
    m, k = a.shape
    k2, n = w.shape
    if k != k2:
        raise ValueError("ShapeMismatch")
    if m == 0 or n == 0:
        raise ValueError("EmptyMatrix")
    w = w.contiguous()
    if out is None:
        out = empty_padded(m, n, device=a.device)
    L = lib()
    parts = torch.empty(int(L.aes_gemm_fit_partial_bytes(m, n)), dtype=torch.uint8, device=a.device)
    res = torch.empty(4, dtype=torch.float32, device=a.device)
    st = stream_of(stream)
    check(L.aes_dev_gemm_bias_act_fit(ptr(a), m, k, a.stride(0), ptr(w), n, w.stride(0),
                                      ptr(bias) if bias is not None and bias.numel() else None, int(relu),
                                      int(bool(finite_w)), ptr(out), out.stride(0), ptr(parts), st))
    check(L.aes_dev_fit_merge(ptr(parts), parts.numel() // 32, ptr(res), st))
    return out, res


def gemm_tf32(a: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None, relu: bool, out=None,
              stream=None) -> torch.Tensor:
    """FAST MODE act(a @ w + bias) on the tcgen05 tensor cores (TF32
    operands, fp32 accumulation; NOT bit-exact: |err| <= 2^-8 sum|a||w|)."""
    m, k = a.shape
    k2, n = w.shape
    if k != k2:
        raise ValueError("ShapeMismatch")
    if out is None:
        out = empty_padded(m, n, device=a.device)
    scratch = torch.empty(int(lib().aes_gemm_tf32_scratch_floats(k, n)), dtype=torch.float32, device=a.device)
    check(lib().aes_dev_gemm_tf32(ptr(a), m, k, a.stride(0), ptr(w), n, w.stride(0),
                                  ptr(bias) if bias is not None and bias.numel() else None, int(relu), ptr(out),
                                  out.stride(0), ptr(scratch), stream_of(stream)))
    return out


FUSED_LAYER_MIN_ROWS = 512 * 1024


def gcn_layer_fused(srow_ptr, scol, sval, x: torch.Tensor, w: torch.Tensor, b, relu: bool, finite_w: bool = True,
                    out: torch.Tensor | None = None, stream=None):
    """One exact GCN layer act(SpMM(A, x) w + b) as ONE persistent kernel
    (aes_dev_gcn_layer_fused: SpMM producer warps + ordered-GEMM consumer
    warps, the aggregate never leaves shared memory).  Returns None when the
    shape is outside the kernel's range (k % 4 != 0, k > 128 or n > 128):
    the caller runs the split kernels.  Bit-identical to spmm + gemm_bias_act."""
    L = lib()
    m, k = x.shape[0], x.shape[1]
    n = w.shape[1]
    if k % 4 or k > 128 or n > 128 or k == 0 or n == 0:
        return None
    x = padded(x)
    w = w.contiguous()
    h = out if out is not None else empty_padded(m, n, device=x.device)
    rc = L.aes_dev_gcn_layer_fused(ptr(srow_ptr), ptr(scol), ptr(sval), m, ptr(x), x.stride(0), k, ptr(w),
                                   w.stride(0), n, ptr(b) if b is not None else None, int(relu), int(finite_w),
                                   ptr(h), h.stride(0), stream_of(stream))
    if rc == capi.AES_ERR_UNSUPPORTED:
        return None
    check(rc)
    return h


def gcn_forward(graph: Graph, x: torch.Tensor, weights, biases, plan: SampledPlan | None = None,
                stream=None, fast_gemm: bool = False, finite=None, fused: bool = True) -> torch.Tensor:
    """gcn_forward (proj/src/gnn.cpp:66-78) on one GPU, all tensors in HBM.
    fast_gemm=True runs the layer transform on the tcgen05 tensor cores (TF32,
    not bit-exact); the aggregation stays the exact sampled SpMM.  finite:
    per-layer "weights have no inf/NaN" flags (checked on the device with one
    read-back when None)."""
    h = padded(x)
    srow, scol, sval = (plan.srow_ptr, plan.scol, plan.sval) if plan is not None else (
        graph.row_ptr, graph.col, graph.val)
    bound = plan.row_bound if plan is not None else 0
    if finite is None:
        finite = all_weights_finite(weights, stream)  # one read-back for every layer
    for l, (w, b) in enumerate(zip(weights, biases)):
        relu = l + 1 < len(weights)
        # sampled plan (rows bounded) on a large graph: one fused kernel per
        # layer (products 4.13 vs 4.28 ms split; on arxiv-size graphs the
        # 148 persistent CTAs get ~18 tiles each and the split kernels win,
        # 0.279 vs 0.293 ms)
        if fused and not fast_gemm and bound and h.shape[0] >= FUSED_LAYER_MIN_ROWS:
            hf = gcn_layer_fused(srow, scol, sval, h, w, b, relu, finite_w=finite[l], stream=stream)
            if hf is not None:
                h = hf
                continue
        agg = spmm(srow, scol, sval, h, stream=stream, max_row_slots=bound)
        if fast_gemm and agg.shape[1] <= 128 and w.shape[1] <= 128:
            h = gemm_tf32(agg, w, b, relu=l + 1 < len(weights), stream=stream)
        else:
            h = gemm_bias_act(agg, w, b, relu=l + 1 < len(weights), stream=stream, finite_w=finite[l])
    return h


class GcnForwardGraph:
    """gcn_forward captured once into a CUDA graph and replayed per call.

    For the small BASELINE graphs (cora, pubmed, arxiv) a forward is a dozen
    short kernels whose host-side launch cost (Python + ctypes per call)
    exceeds their GPU time; replaying one graph launches them all with a
    single call.  Shapes, weights, plan and output buffers are fixed at
    capture; run(x) copies x into the captured input and replays.  The
    kernels and their results are exactly those of gcn_forward."""

    def __init__(self, graph: Graph, x_like: torch.Tensor, weights, biases, plan: SampledPlan | None = None,
                 fast_gemm: bool = False):
        self.weights, self.biases = list(weights), list(biases)
        finite = all_weights_finite(self.weights)
        self.x = empty_padded(x_like.shape[0], x_like.shape[1], device=x_like.device)
        self.x.copy_(x_like)
        self.stream = torch.cuda.Stream()
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):  # warm-up: kernel attributes, allocator pool
            gcn_forward(graph, self.x, self.weights, self.biases, plan, fast_gemm=fast_gemm, finite=finite)
        self.stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self.out = gcn_forward(graph, self.x, self.weights, self.biases, plan, fast_gemm=fast_gemm,
                                   finite=finite)

    def run(self, x: torch.Tensor | None = None) -> torch.Tensor:
        """Forward of x (None: the input already in self.x); returns the
        captured output buffer (overwritten by the next run)."""
        if x is not None:
            self.x.copy_(x)
        self.graph.replay()
        return self.out
