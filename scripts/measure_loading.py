"""Feature-loading time, the paper's Table-3 story: the
products feature matrix as an f32 FMAT (1.25 GB) vs an int8 FMAT (0.31 GB),
loaded straight to HBM (ours) and through the reference's load_features + a
host->device copy (oracle/_ref).  Files live in /tmp (page cache warm after
the first read; both paths read the same files)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_18427_b200 import device, synth  # noqa: E402

n, _, _, f = synth.SHAPES["products"]
x = synth.features(n, f, seed=5, ld=f)
q = device.quantize(x)
d = "/tmp/aes_fmat"
os.makedirs(d, exist_ok=True)
p32, p8 = f"{d}/products_f32.fmat", f"{d}/products_q8.fmat"
import paper_2503_18427_b200 as m  # noqa: E402

m.save_fmat(np.ascontiguousarray(x.cpu().numpy()), p32)
codes = q.codes.cpu().numpy().astype(np.uint16)
qf = m.quantized_from_codes(codes, m.QuantParams(q.x_min, q.x_max, 8))
m.save_fmat(qf, p8)
res = {"rows": n, "cols": f, "bytes_f32": os.path.getsize(p32), "bytes_q8": os.path.getsize(p8)}
for name, p in (("f32", p32), ("q8", p8)):
    ts = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        feat, ms = device.load_fmat(p)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    res[f"ours_{name}_ms"] = round(float(np.median(ts[1:])), 2)
try:
    from oracle import ref as oref
    if oref.available():
        for name, p in (("f32", p32), ("q8", p8)):
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                dt, arr = oref.load_fmat(p)  # reference load_features (host)
                host = arr if dt == 0 else arr[0].astype(np.uint8)
                t = torch.from_numpy(np.ascontiguousarray(host)).cuda()  # then to the GPU
                torch.cuda.synchronize()
                ts.append((time.perf_counter() - t0) * 1e3)
            res[f"reference_load_features_plus_h2d_{name}_ms"] = round(float(np.median(ts[1:])), 2)
except Exception as e:  # pragma: no cover
    res["reference_error"] = str(e)
res["ours_q8_vs_f32_reduction"] = round(1 - res["ours_q8_ms"] / res["ours_f32_ms"], 3)
print(json.dumps(res))
