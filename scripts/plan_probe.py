"""Plan build (sampler) timing on the products shape: the whole SampledPlan
construction (two kernels + one size read-back) and the kernels alone."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import SHAPES  # noqa: E402
from paper_2503_18427_b200 import device, synth  # noqa: E402
from paper_2503_18427_b200.capi import lib, ptr, stream_of  # noqa: E402

n, a, m, _ = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "products"]
rp, col, val = synth.power_law_csr(n, a, m, seed=1, device="cuda")
g = device.Graph(rp, col, val, n)
for _ in range(3):
    p = device.SampledPlan(g, 32)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    p = device.SampledPlan(g, 32)
e.record()
torch.cuda.synchronize()
print(f"SampledPlan (kernels + read-back + allocs): {s.elapsed_time(e) / 10:.3f} ms")
L = lib()
ws_b = L.aes_dev_scan_workspace_bytes(n)
ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
st = stream_of(None)
s.record()
for _ in range(10):
    L.aes_dev_sample_plan(ptr(rp), n, 32, 0, ptr(p.srow_ptr), None, ptr(ws), ws_b, st)
e.record()
torch.cuda.synchronize()
print(f"  row scan kernel: {s.elapsed_time(e) / 10:.3f} ms")
s.record()
for _ in range(10):
    L.aes_dev_sample_fill(ptr(rp), ptr(rp), ptr(col), ptr(val), n, 32, 0, ptr(p.srow_ptr), ptr(p.scol), ptr(p.sval), st)
e.record()
torch.cuda.synchronize()
fill_bytes = 16 * p.total_slots + 16 * (n + 1)
ms = s.elapsed_time(e) / 10
print(f"  fill kernel: {ms:.3f} ms ({fill_bytes / ms / 1e6:.0f} GB/s algorithmic, {p.total_slots} slots)")
