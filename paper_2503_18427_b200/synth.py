"""Synthetic power-law graphs of the BASELINE shapes, generated on the GPU.

Same degree model as the reference generator (proj/src/bench.cpp:144-157:
inverse-CDF draw from a continuous power law p(d) ~ d^-alpha truncated to
[1, max_degree], floored), with uniformly random distinct neighbours per row —
but drawn with torch's seeded Philox generator on the device, so a
2.45 M-row / 62 M-edge graph takes well under a second instead of the
reference's ~15 s.  Graphs are reproducible per (n, alpha, max_degree, seed,
device type); both bench arms receive the identical CSR arrays.
"""
from __future__ import annotations

import torch

# (n, alpha, max_degree, F) — SURVEY.md §8(d) / BASELINE.json configs
SHAPES = {
    "cora": (2_708, 2.1181, 168, 16),
    "pubmed": (19_717, 2.0321, 171, 128),
    "arxiv": (169_343, 2.0737, 13_161, 128),
    "reddit": (232_965, 1.2986, 21_657, 602),
    "products": (2_450_000, 1.7885, 17_481, 128),
}


def power_law_degrees(n: int, alpha: float, max_degree: int, gen: torch.Generator, device) -> torch.Tensor:
    u = torch.rand(n, dtype=torch.float64, generator=gen, device=device)
    m = float(max_degree)
    if abs(alpha - 1.0) < 1e-9:
        d = torch.exp(u * torch.log(torch.tensor(m, dtype=torch.float64, device=device)))
    else:
        e = 1.0 - alpha
        d = torch.pow(1.0 + u * (m ** e - 1.0), 1.0 / e)
    return torch.clamp(torch.floor(d), 1.0, m).to(torch.int64)


def power_law_csr(n: int, alpha: float, max_degree: int, seed: int = 1, device="cuda", values="ones"):
    """Return (row_ptr int64[n+1], col int32[nnz], val float32[nnz]) on `device`.

    Columns are sorted and distinct within each row (duplicate draws are
    dropped, so a row can end slightly below its drawn degree)."""
    device = torch.device(device)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    deg = power_law_degrees(n, alpha, max_degree, gen, device)
    rows = torch.repeat_interleave(torch.arange(n, device=device, dtype=torch.int64), deg)
    cols = torch.randint(0, n, (rows.numel(),), generator=gen, device=device, dtype=torch.int64)
    keys = torch.unique(rows * n + cols)  # sorted, distinct (row, col)
    rows = torch.div(keys, n, rounding_mode="floor")
    cols = keys - rows * n
    counts = torch.bincount(rows, minlength=n)
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=row_ptr[1:])
    col = cols.to(torch.int32)
    if values == "ones":
        val = torch.ones(col.numel(), dtype=torch.float32, device=device)
    else:
        val = torch.rand(col.numel(), dtype=torch.float32, generator=gen, device=device) * 2 - 1
    return row_ptr, col, val


def features(n: int, f: int, seed: int = 5, device="cuda", ld: int | None = None) -> torch.Tensor:
    """U(-1, 1) fp32 features, row stride `ld` (default round_up(f, 4))."""
    device = torch.device(device)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    ld = ld if ld is not None else (f + 3) & ~3
    buf = torch.zeros((n, ld), dtype=torch.float32, device=device)
    buf[:, :f] = torch.rand((n, f), generator=gen, device=device) * 2 - 1
    return buf[:, :f]
