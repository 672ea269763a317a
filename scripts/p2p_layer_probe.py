"""One GCN layer through ShardedGCN(exchange="p2p") at the products shape:
which path each layer takes (fused kernel or SpMM + publishing GEMM) and the
step time, fused vs forced split."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import SHAPES  # noqa: E402
from paper_2503_18427_b200 import device, synth  # noqa: E402
from paper_2503_18427_b200.gcn import ShardedGCN  # noqa: E402

n, a, m, _ = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "products"]
rp, col, val = synth.power_law_csr(n, a, m, seed=1, device="cuda")
g = device.Graph(rp, col, val, n)
plan = device.SampledPlan(g, 32)
x = synth.features(n, 128, seed=5, device="cuda")
w = torch.rand((128, 128), device="cuda", generator=torch.Generator("cuda").manual_seed(3)) - 0.5
b = torch.full((128,), 0.01, device="cuda")
for thr in (device.FUSED_LAYER_MIN_ROWS, 1 << 40):
    device.FUSED_LAYER_MIN_ROWS = thr
    model = ShardedGCN(plan.srow_ptr, plan.scol, plan.sval, n, [w], [b], exchange="p2p", max_row_slots=plan.row_bound)
    model.input_view().copy_(x)
    for _ in range(3):
        model.forward(None, copy_out=False)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        model.forward(None, copy_out=False)
    e.record()
    torch.cuda.synchronize()
    print(f"p2p layer: fused={model.p2p_fused} {s.elapsed_time(e) / 10:.3f} ms", flush=True)
    del model
    torch.cuda.empty_cache()
