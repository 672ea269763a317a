"""Per-shard SpMM times for the row-sharded products workload at P = 1/2/4/8.

At N GPUs every rank runs the SpMM of its own contiguous slot-balanced row
shard against its full feature replica (bench.py, strong scaling).  The
ranks are independent, so on one B200 each shard can be timed alone: the
whole-job step at P is the slowest shard, and

    value(P) = total algorithmic bytes / max_r t_r(P)

is what `bench.py --gpus P` reports on P GPUs (less launch skew).  Prints one
JSON object per dtype with the shard times and the implied scaling efficiency.
"""
from __future__ import annotations

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import SHAPES, alg_bytes, shard_bounds  # noqa: E402
from paper_2503_18427_b200 import device, synth  # noqa: E402


def time_ms(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="products")
    ap.add_argument("--sched", type=int, default=0, help="aes_dev_spmm_set_schedule: 0 auto, 1 static, 2 dynamic")
    args = ap.parse_args()
    config = args.config
    from paper_2503_18427_b200 import capi
    capi.check(capi.lib().aes_dev_spmm_set_schedule(args.sched))
    n, alpha, maxdeg, f = SHAPES[config]
    rp, col, val = synth.power_law_csr(n, alpha, maxdeg, seed=1, device="cuda")
    g = device.Graph(rp, col, val, n)
    b = synth.features(n, f, seed=5, device="cuda")
    plan = device.SampledPlan(g, 32)
    srow_host = plan.srow_ptr.cpu().numpy()
    total_slots = int(srow_host[-1])
    q = device.quantize(b)
    out = device.empty_padded(n, f)
    res = {}
    for dtype, elem in (("f32", 4), ("int8", 1)):
        total = alg_bytes(n, total_slots, f, elem)
        rows = []
        for p in (1, 2, 4, 8):
            cuts = shard_bounds(srow_host, p)
            ts = []
            for r in range(p):
                lo, hi = cuts[r], cuts[r + 1]
                srow = plan.srow_ptr[lo:hi + 1]
                if dtype == "f32":
                    fn = lambda: device.spmm(srow, plan.scol, plan.sval, b, out=out[: hi - lo],  # noqa: E731
                                             max_row_slots=plan.row_bound)
                else:
                    fn = lambda: device.spmm_q8(srow, plan.scol, plan.sval, q, out=out[: hi - lo],  # noqa: E731
                                                max_row_slots=plan.row_bound)
                ts.append(time_ms(fn))
            step = max(ts)
            rows.append({"P": p, "shard_ms": [round(t, 4) for t in ts], "step_ms": round(step, 4),
                         "value_gbs": round(total / (step * 1e-3) / 1e9, 1)})
        base = rows[0]["value_gbs"]
        for r in rows:
            r["efficiency"] = round(r["value_gbs"] / (base * r["P"]), 4)
        res[dtype] = rows
    print(json.dumps({"config": config, "sched": args.sched, "slots": total_slots, "scaling": res}))


if __name__ == "__main__":
    main()
