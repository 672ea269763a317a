"""GCN forward on the small BASELINE graphs: eager device.gcn_forward vs the
CUDA-graph replay (device.GcnForwardGraph); results must be identical."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import SHAPES  # noqa: E402
from paper_2503_18427_b200 import device, synth  # noqa: E402

DIMS = {"cora": [16, 16, 7], "pubmed": [128, 128, 3], "arxiv": [128, 128, 128, 40]}


def wall_ms(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / reps


for name in sys.argv[1:] or ["cora", "pubmed", "arxiv"]:
    n, a, m, _ = SHAPES[name]
    dims = DIMS[name]
    rp, col, val = synth.power_law_csr(n, a, m, seed=1, device="cuda")
    g = device.Graph(rp, col, val, n)  # raw adjacency: the same kernels and sizes as the normalized one
    rng = np.random.default_rng(7)
    ws = [torch.from_numpy(rng.uniform(-0.5, 0.5, (i, o)).astype(np.float32)).cuda() for i, o in zip(dims, dims[1:])]
    bs = [torch.full((o,), 0.01, device="cuda") for o in dims[1:]]
    x = synth.features(n, dims[0], seed=5, device="cuda")
    plan = device.SampledPlan(g, 32)
    eager = wall_ms(lambda: device.gcn_forward(g, x, ws, bs, plan))
    cg = device.GcnForwardGraph(g, x, ws, bs, plan)
    replay = wall_ms(lambda: cg.run())
    same = torch.equal(cg.run(x), device.gcn_forward(g, x, ws, bs, plan))
    print(f"{name}: gcn_forward eager {eager:.3f} ms, CUDA-graph replay {replay:.3f} ms, identical={same}", flush=True)
