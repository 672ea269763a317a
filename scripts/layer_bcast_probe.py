"""Fused layer kernel, plain output vs the broadcast (p2p exchange) form, same buffers."""
import os, sys, ctypes
sys.path.insert(0, os.getcwd())
import torch
from bench import SHAPES
from paper_2503_18427_b200 import device, synth, capi
from paper_2503_18427_b200.p2p import PeerReplicas
n, a, m, _ = SHAPES["products"]
rp, col, val = synth.power_law_csr(n, a, m, seed=1, device="cuda")
g = device.Graph(rp, col, val, n)
plan = device.SampledPlan(g, 32)
x = synth.features(n, 128, seed=5, device="cuda")
w = torch.rand((128, 128), device="cuda") - 0.5
b = torch.full((128,), 0.01, device="cuda")
rep = PeerReplicas(n, 128)
rep.bufs[0][:, :].copy_(x)
def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
out = device.empty_padded(n, 128)
print("plain  x=feat  h=new  ", t(lambda: device.gcn_layer_fused(plan.srow_ptr, plan.scol, plan.sval, x, w, b, True, True, out=out)))
print("plain  x=rep0  h=rep1 ", t(lambda: device.gcn_layer_fused(plan.srow_ptr, plan.scol, plan.sval, rep.bufs[0], w, b, True, True, out=rep.bufs[1])))
print("bcast  x=rep0  h=rep1 ", t(lambda: rep.layer_publish(1, plan.srow_ptr, plan.scol, plan.sval, rep.bufs[0], w, b, True, True, 0)))
print("bcast  x=feat  h=rep1 ", t(lambda: rep.layer_publish(1, plan.srow_ptr, plan.scol, plan.sval, x, w, b, True, True, 0)))
