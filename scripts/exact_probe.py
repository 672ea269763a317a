"""Time the exact SpMM (spmm_exact: every nonzero, rows of unknown length) on
the BASELINE shapes at F = 128 (and the arxiv 3-layer exact GCN)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import SHAPES  # noqa: E402
from paper_2503_18427_b200 import device, synth  # noqa: E402


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for name in sys.argv[1:] or ["arxiv", "products"]:
    n, a, m, _ = SHAPES[name]
    rp, col, val = synth.power_law_csr(n, a, m, seed=1, device="cuda")
    g = device.Graph(rp, col, val, n)
    b = synth.features(n, 128, seed=5, device="cuda")
    out = device.empty_padded(n, 128)
    ms = t(lambda: device.spmm_exact(g, b, out=out))
    nnz = g.nnz
    alg = 8 * (n + 1) + 8 * nnz + 512 * nnz + 512 * n
    deg = torch.diff(rp).max().item()
    print(f"{name}: exact SpMM F=128 {ms:.3f} ms, {alg / ms / 1e6:.0f} GB/s alg, max row {deg}", flush=True)
    q = device.quantize(b)
    ms = t(lambda: device.spmm_q8(g.row_ptr, g.col, g.val, q, out=out))
    alg8 = 8 * (n + 1) + 8 * nnz + 128 * nnz + 512 * n
    print(f"{name}: exact int8 SpMM F=128 {ms:.3f} ms, {alg8 / ms / 1e6:.0f} GB/s alg", flush=True)
