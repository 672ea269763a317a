"""Time every SpMM schedule variant on a BASELINE shape (device-resident,
CUDA events, inputs larger than L2) and check they are bit-identical."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2503_18427_b200 import capi, device, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="products")
ap.add_argument("--width", type=int, default=32)
ap.add_argument("--variants", default="1,2,3,4,5,6,7,8")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--dtypes", default="f32,int8")
ap.add_argument("--strategy", default="adaptive")
ap.add_argument("--q8-variants", default=None, help="int8 schedules (default: --variants)")
ap.add_argument("--sched", type=int, default=0, help="ring row-group schedule (aes_dev_spmm_set_schedule)")
args = ap.parse_args()

n, alpha, maxdeg, f = synth.SHAPES[args.config]
rp, col, val = synth.power_law_csr(n, alpha, maxdeg, seed=1, device="cuda")
g = device.Graph(rp, col, val, n)
b = synth.features(n, f, seed=5)
L = capi.lib()
capi.check(L.aes_dev_spmm_set_schedule(args.sched))


def timeit(fn, iters):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


res = {"config": args.config, "width": args.width, "n": n, "nnz": int(rp[-1])}
t_plan = timeit(lambda: device.SampledPlan(g, args.width, args.strategy), 5)
plan = device.SampledPlan(g, args.width, args.strategy)
res["plan_ms"] = round(t_plan, 4)
res["slots"] = plan.total_slots
q = device.quantize(b)
res["quantize_ms"] = round(timeit(lambda: device.quantize(b, params=(q.x_min, q.x_max)), 5), 4)
for dt in args.dtypes.split(","):
    out = device.empty_padded(n, f)
    ref = None
    vlist = args.q8_variants if (dt == "int8" and args.q8_variants) else args.variants
    for v in [int(x) for x in vlist.split(",")]:
        L.aes_dev_spmm_set_variant(v)
        if dt == "f32":
            fn = lambda: device.spmm_plan(plan, b, out=out)  # noqa: E731
            by = plan.algorithmic_bytes(f, 4)
        else:
            fn = lambda: device.spmm_q8(plan.srow_ptr, plan.scol, plan.sval, q, out=out, max_row_slots=plan.row_bound)  # noqa: E731
            by = plan.algorithmic_bytes(f, 1)
        ms = timeit(fn, args.iters)
        fn()
        torch.cuda.synchronize()
        same = None
        if ref is None:
            ref = out.clone()
        else:
            same = bool(torch.equal(out, ref))
        res[f"{dt}_v{v}"] = {"ms": round(ms, 4), "GBps": round(by / ms / 1e6, 1), "bit_identical": same}
        print(dt, v, res[f"{dt}_v{v}"], flush=True)
    L.aes_dev_spmm_set_variant(0)
w = torch.rand(f, f, device="cuda")
h = device.empty_padded(n, f)
res["gemm_ms"] = round(timeit(lambda: device.gemm_bias_act(b, w, None, True, out=h), 5), 4)
ptrs = (__import__("ctypes").c_void_p * 1)(h.data_ptr())
res["gemm_finite_ms"] = round(timeit(lambda: capi.check(L.aes_dev_gemm_bias_act_ex(
    b.data_ptr(), n, f, b.stride(0), w.data_ptr(), f, f, None, 1, 1, __import__("ctypes").cast(ptrs, __import__("ctypes").c_void_p),
    None, 1, 0, h.stride(0), capi.stream_of())), 5), 4)
if f <= 128:  # the tcgen05 layer GEMM takes K, N <= 128
    res["gemm_tf32_tcgen05_ms"] = round(timeit(lambda: device.gemm_tf32(b, w, None, True, out=h), 10), 4)
    res["gemm_tf32_GBps"] = round(2 * n * f * 4 / res["gemm_tf32_tcgen05_ms"] / 1e6, 1)
print(json.dumps(res))
