"""Seeded CSR generators for the parity tests (numpy; test-side only)."""
from __future__ import annotations

import numpy as np


def csr_from_rows(n_rows, n_cols, rows_cols, vals=None, rng=None):
    row_ptr = np.zeros(n_rows + 1, np.uint64)
    cols = []
    for i, cs in enumerate(rows_cols):
        cs = np.unique(np.asarray(cs, np.int64))
        row_ptr[i + 1] = row_ptr[i] + cs.size
        cols.append(cs)
    col = np.concatenate(cols).astype(np.uint32) if cols else np.zeros(0, np.uint32)
    if vals is None:
        rng = rng or np.random.default_rng(0)
        vals = rng.uniform(-1, 1, col.size).astype(np.float32)
    return row_ptr, col, np.asarray(vals, np.float32)


def power_law(n, alpha=1.5, max_deg=200, seed=0, n_cols=None, values="uniform"):
    """Truncated-Pareto out-degrees, distinct sorted neighbours (like the
    reference gen_synthetic, proj/src/bench.cpp:144-202, but numpy-seeded)."""
    rng = np.random.default_rng(seed)
    n_cols = n if n_cols is None else n_cols
    u = rng.random(n)
    e = 1.0 - alpha
    deg = np.floor((1.0 + u * (max_deg ** e - 1.0)) ** (1.0 / e)).astype(np.int64)
    deg = np.clip(deg, 1, min(max_deg, n_cols))
    row_ptr = np.zeros(n + 1, np.uint64)
    cols = []
    for i in range(n):
        c = np.sort(rng.choice(n_cols, size=int(deg[i]), replace=False))
        cols.append(c)
    row_ptr[1:] = np.cumsum([c.size for c in cols])
    col = np.concatenate(cols).astype(np.uint32)
    if values == "ones":
        val = np.ones(col.size, np.float32)
    else:
        val = rng.uniform(-1, 1, col.size).astype(np.float32)
    return row_ptr, col, val


def with_degrees(degrees, n_cols=None, seed=0):
    """One row per requested degree (columns 0..d-1 spread over n_cols)."""
    rng = np.random.default_rng(seed)
    n_cols = n_cols or max(max(degrees), 1) * 2
    rows = [np.sort(rng.choice(n_cols, size=d, replace=False)) for d in degrees]
    return csr_from_rows(len(degrees), n_cols, rows, rng=rng) + (n_cols,)


def random_graph(n, density, rng):
    """Dense-mask random graph like test_spmm.cpp:14-28."""
    mask = rng.random((n, n)) < density
    rows = [np.nonzero(mask[i])[0] for i in range(n)]
    vals = rng.uniform(-1, 1, int(mask.sum())).astype(np.float32)
    return csr_from_rows(n, n, rows, vals)
