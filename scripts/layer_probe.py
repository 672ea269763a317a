"""Exact GCN layer on the BASELINE shapes: split kernels (sampled SpMM ->
ordered GEMM + bias + ReLU) vs the fused persistent kernel
(aes_dev_gcn_layer_fused), and the arxiv 3-layer forward both ways."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import SHAPES  # noqa: E402
from paper_2503_18427_b200 import device, synth  # noqa: E402


def t(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for name in sys.argv[1:] or ["products", "arxiv"]:
    n, a, m, _ = SHAPES[name]
    rp, col, val = synth.power_law_csr(n, a, m, seed=1, device="cuda")
    g = device.Graph(rp, col, val, n)
    plan = device.SampledPlan(g, 32)
    x = synth.features(n, 128, seed=5, device="cuda")
    gen = torch.Generator(device="cuda").manual_seed(3)
    w = torch.rand((128, 128), generator=gen, device="cuda") - 0.5
    b = torch.full((128,), 0.01, device="cuda")
    out = device.empty_padded(n, 128)
    agg = device.empty_padded(n, 128)

    def split():
        device.spmm(plan.srow_ptr, plan.scol, plan.sval, x, out=agg, max_row_slots=plan.row_bound)
        device.gemm_bias_act(agg, w, b, relu=True, out=out, finite_w=True)

    def fused():
        device.gcn_layer_fused(plan.srow_ptr, plan.scol, plan.sval, x, w, b, True, finite_w=True, out=out)

    ms_spmm = t(lambda: device.spmm(plan.srow_ptr, plan.scol, plan.sval, x, out=agg, max_row_slots=plan.row_bound))
    ms_gemm = t(lambda: device.gemm_bias_act(agg, w, b, relu=True, out=out, finite_w=True))
    ms_split, ms_fused = t(split), t(fused)
    split()
    ref = out.clone()
    fused()
    torch.cuda.synchronize()
    same = torch.equal(ref.view(torch.int32), out.view(torch.int32))
    floor = 2 * n * 128 * 128 / (148 * 128 * 1.965e9) * 1e3
    print(f"{name}: layer F=128->128 split {ms_split:.3f} ms (spmm {ms_spmm:.3f} + gemm {ms_gemm:.3f}), "
          f"fused {ms_fused:.3f} ms, bit-identical {same}; FP32-pipe floor of the ordered GEMM {floor:.3f} ms",
          flush=True)
    if name == "arxiv":
        ws = [torch.rand(s, generator=gen, device="cuda") - 0.5 for s in [(128, 128), (128, 128), (128, 40)]]
        bs = [torch.full((s,), 0.01, device="cuda") for s in (128, 128, 40)]
        fin = [True, True, True]
        ms_f = t(lambda: device.gcn_forward(g, x, ws, bs, plan, finite=fin))
        ms_s = t(lambda: device.gcn_forward(g, x, ws, bs, plan, finite=fin, fused=False))
        print(f"arxiv 3-layer GCN forward (eager): fused {ms_f:.3f} ms, split {ms_s:.3f} ms", flush=True)
