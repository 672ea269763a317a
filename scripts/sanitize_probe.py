"""One pass over every device kernel family at small shapes, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python scripts/sanitize_probe.py

Covers the cp.async rings of the fp32 balanced / static / dynamic SpMM
schedules, the hub kernel (exact SpMM, unbounded rows), the int8 batch
kernel (static 32-row groups and the balanced one-wave schedule, whole and
partial column tiles), the int8 fast mode, the sampler (scan + fill,
explicit plans), cdf_stats, quantize / fit / dequantize, both layer GEMMs
(ordered fp32 and tcgen05 TF32) and gcn_normalize.  Results are checked
against the fp32 kernels where cheap; the sanitizer verdict is the point.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2503_18427_b200 as m  # noqa: E402
from paper_2503_18427_b200 import capi, device  # noqa: E402
from tests import graphs  # noqa: E402


def main():
    torch.cuda.set_device(0)
    rng = np.random.default_rng(0)
    n = 3000
    rp, col, _ = graphs.power_law(n, alpha=1.4, max_deg=2500, seed=1)  # has hub rows
    val = rng.uniform(-1, 1, col.size).astype(np.float32)
    g = device.Graph.from_numpy(rp, col, val)
    for f in (128, 602, 40):
        b = torch.from_numpy(rng.uniform(-1, 1, (n, f)).astype(np.float32)).cuda()
        for strat in ("adaptive", "full", "afs", "sfs"):
            plan = device.SampledPlan(g, 32, strat)
            ref = None
            for sched in (0, 1, 2, 3):
                capi.check(capi.lib().aes_dev_spmm_set_schedule(sched))
                out = device.spmm_plan(plan, b)
                ref = out if ref is None else ref
                assert torch.equal(out, ref), (f, strat, sched)
            capi.check(capi.lib().aes_dev_spmm_set_schedule(0))
            q = device.quantize(b)
            qo = device.spmm_q8(plan.srow_ptr, plan.scol, plan.sval, q, max_row_slots=plan.row_bound)
            want = device.spmm_plan(plan, device.dequantize(q))
            assert torch.equal(qo, want), (f, strat, "q8")
            for mode in ("row", "feature"):
                qa = device.quantize_affine(b, mode)
                device.spmm_q8_affine(plan.srow_ptr, plan.scol, plan.sval, qa)
        device.spmm_exact(g, b)
        w = torch.rand(f, 64, device="cuda") - 0.5
        bias = torch.full((64,), 0.01, device="cuda")
        device.gemm_bias_act(b, w, bias, True, finite_w=True)
        device.gemm_bias_act_fit(b, w, bias, True, finite_w=True)
        if f <= 128:
            device.gemm_tf32(b, w, bias, True)
    # handle tier: plans from host data, rates, cdf, normalize, GCN forward
    a = m.CsrMatrix(n, n, rp, col, val)
    ps = m.build_plan_set(a, 16)
    m.sampling_rate(ps, a)
    m.sampling_rate_cdf(ps, a)
    m.cdf_stats(rng.random(5000))
    an = m.gcn_normalize(a, True)
    x = rng.uniform(-1, 1, (n, 16)).astype(np.float32)
    m.spmm_sampled(an, x, m.build_plan_set(an, 8))
    qf = m.quantize(x)
    m.dequantize(qf)
    m.spmm_sampled_q8(a, qf, ps)
    torch.cuda.synchronize()
    print("sanitize probe done")


if __name__ == "__main__":
    main()
