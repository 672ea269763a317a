"""Host<->device copy ceilings for the e2e leg of bench.py (the products
workload moves 1.25 GB of features H2D and 1.25 GB of output D2H per step).

Prints one JSON object: pinned-memory H2D alone, D2H alone, both directions
at once (separate streams), and chunked variants, each in GB/s per direction.
"""
from __future__ import annotations

import json
import time

import torch


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def main():
    nbytes = 2_450_000 * 128 * 4
    n = nbytes // 4
    h_in = torch.empty(n, dtype=torch.float32).pin_memory()
    h_out = torch.empty(n, dtype=torch.float32).pin_memory()
    d_in = torch.empty(n, dtype=torch.float32, device="cuda")
    d_out = torch.empty(n, dtype=torch.float32, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {"bytes": nbytes}

    def h2d():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)

    def both():
        h2d()
        d2h()

    def chunked(k):
        def f():
            step = -(-n // k)
            for i in range(k):
                sl = slice(i * step, min(n, (i + 1) * step))
                with torch.cuda.stream(s1):
                    d_in[sl].copy_(h_in[sl], non_blocking=True)
                with torch.cuda.stream(s2):
                    h_out[sl].copy_(d_out[sl], non_blocking=True)
        return f

    t = timed(h2d)
    res["h2d_gbs"] = round(nbytes / t / 1e9, 2)
    t = timed(d2h)
    res["d2h_gbs"] = round(nbytes / t / 1e9, 2)
    t = timed(both)
    res["bidir_gbs_per_dir"] = round(nbytes / t / 1e9, 2)
    res["bidir_ms"] = round(t * 1e3, 3)
    for k in (4, 16):
        t = timed(chunked(k))
        res[f"bidir_chunk{k}_gbs_per_dir"] = round(nbytes / t / 1e9, 2)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
