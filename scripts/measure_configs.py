"""Measure every BASELINE.json config on the B200 (device-resident, CUDA
events, median of reps after warm-up) next to the reference CPU path
(oracle/_ref, all host threads, bounded reps).  Writes one JSON document.

  python scripts/measure_configs.py > gpurun_out/configs.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_18427_b200 import capi, device, synth  # noqa: E402

try:
    from oracle import ref as oref  # reference CPU implementation (test/bench infrastructure)
    HAVE_REF = oref.available()
except Exception:
    HAVE_REF = False

THREADS = os.cpu_count() or 1


def gpu_ms(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


def alg(n, s, f, e=4):
    return 8 * (n + 1) + 8 * s + e * f * s + 4 * f * n


def graph(name, normalize=False):
    n, a, md, f = synth.SHAPES[name]
    rp, col, val = synth.power_law_csr(n, a, md, seed=1, device="cuda")
    if normalize:
        import paper_2503_18427_b200 as m
        c = m.CsrMatrix(n, n, rp.cpu().numpy().view(np.uint64), col.cpu().numpy().view(np.uint32), val.cpu().numpy())
        rp_, col_, val_ = m.gcn_normalize(c, True).to_arrays()
        g = device.Graph.from_numpy(rp_, col_, val_)
    else:
        g = device.Graph(rp, col, val, n)
    return g, f


def host(g):
    return (g.row_ptr.cpu().numpy().view(np.uint64), g.col.cpu().numpy().view(np.uint32), g.val.cpu().numpy())


def spmm_config(name, widths, dtypes=("f32", "int8", "int8-row", "int8-feature"), cpu=True):
    g, f = graph(name)
    b = synth.features(g.n_rows, f, seed=5)
    out = {"config": name, "n": g.n_rows, "nnz": g.nnz, "F": f, "runs": []}
    q = device.quantize(b)
    qa = {m: device.quantize_affine(b, m) for m in ("row", "feature")}
    for w in widths:
        plan = device.SampledPlan(g, w)
        plan_ms = gpu_ms(lambda: device.SampledPlan(g, w), reps=5)
        c = device.empty_padded(g.n_rows, f)
        for dt in dtypes:
            if dt == "f32":
                ms = gpu_ms(lambda: device.spmm_plan(plan, b, out=c))
                by = plan.algorithmic_bytes(f, 4)
            elif dt == "int8":
                ms = gpu_ms(lambda: device.spmm_q8(plan.srow_ptr, plan.scol, plan.sval, q, out=c, max_row_slots=plan.row_bound))
                by = plan.algorithmic_bytes(f, 1)
            else:  # int8 fast mode (affine codes; the row mode also gathers 8 B of params per slot)
                qm = qa[dt.split("-")[1]]
                ms = gpu_ms(lambda: device.spmm_q8_affine(plan.srow_ptr, plan.scol, plan.sval, qm, out=c))
                by = plan.algorithmic_bytes(f, 1) + (8 * plan.total_slots if dt == "int8-row" else 0)
            out["runs"].append({"W": w, "dtype": dt, "slots": plan.total_slots, "spmm_ms": round(ms, 4),
                                "alg_GBps": round(by / ms / 1e6, 1), "plan_ms": round(plan_ms, 4)})
    out["quantize_ms"] = round(gpu_ms(lambda: device.quantize(b, params=(q.x_min, q.x_max)), reps=5), 4)
    ex = device.empty_padded(g.n_rows, f)
    out["exact_ms"] = round(gpu_ms(lambda: device.spmm_exact(g, b, out=ex), reps=5), 4)
    if cpu and HAVE_REF:
        rp, col, val = host(g)
        csr = oref.RefCsr.from_arrays(g.n_rows, g.n_rows, rp, col, val)
        bn = np.ascontiguousarray(b.cpu().numpy())
        plan_ms, ms, _ = oref.time_spmm_sampled(csr, bn, widths[0], 0, THREADS, 2)
        out["reference_cpu"] = {"W": widths[0], "spmm_ms": round(float(np.median(ms)), 2),
                                "plan_ms": round(plan_ms, 2), "threads": THREADS}
    return out


def gcn_config(name, dims, width, cpu=True):
    g, f = graph(name, normalize=True)
    rng = np.random.default_rng(7)
    ws = [rng.uniform(-0.5, 0.5, (a, b)).astype(np.float32) for a, b in zip(dims, dims[1:])]
    bs = [np.full(b, 0.01 if i + 1 < len(ws) else 0.0, np.float32) for i, b in enumerate(dims[1:])]
    tw = [torch.from_numpy(w).cuda() for w in ws]
    tb = [torch.from_numpy(b).cuda() for b in bs]
    x = synth.features(g.n_rows, dims[0], seed=5)
    plan = device.SampledPlan(g, width)
    ms = gpu_ms(lambda: device.gcn_forward(g, x, tw, tb, plan), reps=5)
    ms_exact = gpu_ms(lambda: device.gcn_forward(g, x, tw, tb, None), reps=5)
    cg = device.GcnForwardGraph(g, x, tw, tb, plan)  # the same kernels, one graph launch
    ms_graph = gpu_ms(lambda: cg.run(), reps=20)
    cgf = device.GcnForwardGraph(g, x, tw, tb, plan, fast_gemm=True)  # tcgen05 TF32 layer GEMMs
    ms_fast = gpu_ms(lambda: cgf.run(), reps=20)
    out = {"config": name, "n": g.n_rows, "nnz_normalized": g.nnz, "dims": dims, "W": width,
           "gcn_forward_ms": round(ms, 4), "gcn_forward_cuda_graph_ms": round(ms_graph, 4),
           "gcn_forward_fast_tf32_cuda_graph_ms": round(ms_fast, 4),
           "gcn_forward_exact_ms": round(ms_exact, 4)}
    if cpu and HAVE_REF:
        rp, col, val = host(g)
        csr = oref.RefCsr.from_arrays(g.n_rows, g.n_rows, rp, col, val)
        xn = np.ascontiguousarray(x.cpu().numpy())
        t0 = time.perf_counter()
        want = oref.gcn_forward(csr, xn, ws, bs, width, 0)
        t_ref = (time.perf_counter() - t0) * 1e3
        got = device.gcn_forward(g, x, tw, tb, plan)
        torch.cuda.synchronize()
        out["reference_cpu"] = {"gcn_forward_ms": round(t_ref, 1), "threads": THREADS,
                                "bit_exact": bool(np.array_equal(np.ascontiguousarray(got.cpu().numpy()).view(np.uint32),
                                                                 want.view(np.uint32)))}
    return out


def main():
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = None
    res = {"device": torch.cuda.get_device_name(0), "host_threads": THREADS, "reference_built": HAVE_REF,
           "peak_hbm_gbs_measured": peak}
    res["cora_gcn"] = gcn_config("cora", [16, 16, 7], 32)
    res["pubmed_spmm"] = spmm_config("pubmed", [32, 64])
    res["arxiv_gcn"] = gcn_config("arxiv", [128, 128, 128, 40], 32)
    res["arxiv_spmm"] = spmm_config("arxiv", [32], cpu=False)
    res["reddit_spmm"] = spmm_config("reddit", [32, 64])
    res["products_spmm"] = spmm_config("products", [32, 64])
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
