"""Time fit_params and the u8 quantize at the products feature shape."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_18427_b200 import device  # noqa: E402


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


x = torch.rand(2_450_000, 128, device="cuda") * 2 - 1
nb = x.numel() * 4
ms = t(lambda: device.quantize(x, 8, params=(-1.0, 1.0)))
print(f"quantize u8: {ms:.3f} ms, {(nb + nb / 4) / ms / 1e6:.0f} GB/s (5 B per element)")
ms = t(lambda: device.fit_params_raw(x))
print(f"fit_params: {ms:.3f} ms, {nb / ms / 1e6:.0f} GB/s")
q = device.quantize(x, 8, params=(-1.0, 1.0))
codes = q.codes.contiguous()
qc = device.QuantizedDevice(codes, q.x_min, q.x_max, 8, q.lut)
ms = t(lambda: device.dequantize(qc))
print(f"dequantize u8: {ms:.3f} ms, {(nb + nb / 4) / ms / 1e6:.0f} GB/s (5 B per element)")
