"""Time the layer GEMM (exact ordered fp32 and tcgen05 TF32) at the products
shape: A [2.45 M, 128] x W [128, 128] + bias, ReLU."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_18427_b200 import device  # noqa: E402


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


m = int(sys.argv[1]) if len(sys.argv) > 1 else 2_450_000
g = torch.Generator("cuda").manual_seed(0)
a = torch.rand(m, 128, device="cuda", generator=g) * 2 - 1
w = torch.rand(128, 128, device="cuda", generator=g) - 0.5
b = torch.full((128,), 0.01, device="cuda")
out = device.empty_padded(m, 128)
ms = t(lambda: device.gemm_bias_act(a, w, b, True, out=out, finite_w=True))
ops = 2 * m * 128 * 128  # FMUL + FADD per multiply-add
print(f"exact ordered GEMM {m}x128x128: {ms:.3f} ms, {ops / ms / 1e9:.1f} Tops/s (FMUL+FADD counted separately)")
ms = t(lambda: device.gemm_tf32(a, w, b, True, out=out))
print(f"tcgen05 TF32 GEMM: {ms:.3f} ms")
