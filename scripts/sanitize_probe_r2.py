"""compute-sanitizer probe of the kernels added in round 2 (small shapes):
the fused GCN layer (plain and with the replica-broadcast epilogue + arrivals;
its mbarrier hand-off between producer and consumer warps), the int8 batch
kernel in its 32-warp / balanced form and its per-feature affine decode,
the cooperative row scan (grid barrier), the pinned staging ring of the
handle tier (pageable host buffers) and the wide-row int8 kernel (F = 602:
exact, per-feature and per-row decodes; cross-lane ring reads after
__syncwarp).

    compute-sanitizer --tool racecheck python scripts/sanitize_probe_r2.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2503_18427_b200 as m  # noqa: E402
from paper_2503_18427_b200 import device  # noqa: E402
from paper_2503_18427_b200.p2p import PeerReplicas  # noqa: E402
from tests import graphs  # noqa: E402


def main():
    torch.cuda.set_device(0)
    rng = np.random.default_rng(1)
    n = 5000  # several 2048-row scan tiles; 79 fused-layer tiles
    rp, col, _ = graphs.power_law(n, alpha=1.6, max_deg=400, seed=2)
    val = rng.uniform(-1, 1, col.size).astype(np.float32)
    g = device.Graph.from_numpy(rp, col, val)
    plan = device.SampledPlan(g, 32)  # cooperative row scan + fill
    for k, fo in ((128, 128), (64, 40)):
        x = torch.from_numpy(rng.uniform(-1, 1, (n, k)).astype(np.float32)).cuda()
        w = torch.rand((k, fo), device="cuda") - 0.5
        b = torch.full((fo,), 0.01, device="cuda")
        h = device.gcn_layer_fused(plan.srow_ptr, plan.scol, plan.sval, x, w, b, True, finite_w=True)
        ref = device.gemm_bias_act(device.spmm(plan.srow_ptr, plan.scol, plan.sval, x, max_row_slots=32), w, b, True)
        assert torch.equal(h, ref)
        device.gcn_layer_fused(plan.srow_ptr, plan.scol, plan.sval, x, w, b, False, finite_w=False)
        rep = PeerReplicas(n, 128)
        rep.bufs[0][:, :k].copy_(x)
        assert rep.layer_publish(1, plan.srow_ptr, plan.scol, plan.sval, rep.bufs[0][:, :k], w, b, True, True, 0)
        rep.wait(int(m.capi.lib().aes_gcn_layer_fused_ctas(n)))
        torch.cuda.synchronize()
        assert torch.equal(rep.bufs[1][:, :fo], ref)
    for f in (128, 602):
        xb = torch.from_numpy(rng.uniform(-1, 1, (n, f)).astype(np.float32)).cuda()
        q = device.quantize(xb)
        device.spmm_q8(plan.srow_ptr, plan.scol, plan.sval, q, max_row_slots=32)
        device.spmm_q8(g.row_ptr, g.col, g.val, q)  # exact: one balanced wave
        for mode in ("feature", "row"):  # F = 602: the wide-row kernel (all three decodes)
            qa = device.quantize_affine(xb, mode)
            device.spmm_q8_affine(plan.srow_ptr, plan.scol, plan.sval, qa)
    # handle tier, pageable buffers above the 4 MB staging threshold
    a = m.CsrMatrix(n, n, rp, col, val)
    ps = m.build_plan_set(a, 32)
    bh = rng.uniform(-1, 1, (n, 602)).astype(np.float32)
    m.spmm_sampled(a, bh, ps)
    torch.cuda.synchronize()
    print("sanitize probe r2 done")


if __name__ == "__main__":
    main()
