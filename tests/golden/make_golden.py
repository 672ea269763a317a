"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref, built
from /root/reference by `make -C oracle ref`).  Run in the build container:

    python tests/golden/make_golden.py

The fixtures pin both our CPU oracle (tests/test_cpu_oracle.py) and the GPU
path (tests/test_gpu_golden.py) to the reference's own outputs.  Inputs are
the reference's gen_synthetic graphs (proj/src/bench.cpp:161-202) at the
Cora shape (n=2708, alpha 2.1181, max degree 168, seed 1) and a heavy-tailed
small graph that hits every Table-1 branch (n=2000, alpha 1.2, max 1500,
seed 31 — a smaller cousin of acceptance criterion 7,
proj/tests/acceptance.cpp:286-333).  Output arrays are stored as sha256
digests of their exact bytes (the comparison is bit-exact anyway); dense
inputs are regenerated from numpy PCG64 seeds, so only the graph structure
and the plans are stored.
"""
import os
import sys

import hashlib

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def digest(a):
    """sha256 of the exact bytes (bit-exact fixtures stay small)."""
    a = np.ascontiguousarray(a)
    return np.array(hashlib.sha256(a.tobytes()).hexdigest() + f"|{a.dtype.str}|{a.shape}")


def b_cora():
    # regenerated identically on any platform (numpy PCG64)
    return np.random.default_rng(5).uniform(-1, 1, (2708, 16)).astype(np.float32)


def heavy_inputs(hcol_size):
    hval = np.random.default_rng(31).uniform(-1, 1, hcol_size).astype(np.float32)
    hb = np.random.default_rng(32).standard_normal((2000, 8)).astype(np.float32)
    return hval, hb


def main():
    assert ref.available(), "build the reference first: make -C oracle ref"
    core = ref.core()
    strategies = {"adaptive": 0, "afs": 1, "sfs": 2, "full": 3}

    # --- cora-shaped graph: plans, sampled SpMM (raw and normalized), GCN
    g = ref.gen_synthetic(2708, 2.1181, 168, 1)
    rp, col, _ = g.arrays()
    rng = np.random.default_rng(6)
    val = np.ones(col.size, np.float32)
    b = b_cora()
    graw = ref.RefCsr.from_arrays(2708, 2708, rp, col, val)
    gn = ref.gcn_normalize(graw, True)
    nrp, ncol, nval = gn.arrays()
    fx = {"row_ptr": rp, "col": col, "norm_row_ptr": nrp, "norm_col": ncol, "norm_val": digest(nval)}
    for name, code in strategies.items():
        for w in (8, 32):
            chunk, cnt, sp, starts = ref.build_plans(graw, w, code)
            fx[f"plan_{name}_{w}_chunk"] = chunk
            fx[f"plan_{name}_{w}_cnt"] = cnt
            fx[f"plan_{name}_{w}_starts_ptr"] = sp
            fx[f"plan_{name}_{w}_starts"] = starts
            fx[f"spmm_{name}_{w}"] = digest(ref.spmm_sampled(graw, b, w, code))
            fx[f"spmm_norm_{name}_{w}"] = digest(ref.spmm_sampled(gn, b, w, code))
            c = core.CsrMatrix(2708, 2708, rp, col, val)
            agg, uni = core.sampling_rate(core.build_plan_set(c, w, getattr(core.Strategy, name.upper())), c)
            fx[f"rate_{name}_{w}"] = np.array([agg, uni])
            # per-row rates and their CDF (bench.cpp:124-138, Fig. 5/6 reporting)
            per_row = ref.sampling_rate_per_row(graw, w, code)
            fx[f"rate_per_row_{name}_{w}"] = digest(per_row)
            cr, cf = ref.cdf_stats(per_row)
            fx[f"cdf_{name}_{w}_rate"], fx[f"cdf_{name}_{w}_frac"] = cr, cf
    fx["spmm_exact"] = digest(ref.spmm_exact(graw, b))
    ws = [rng.uniform(-0.5, 0.5, (16, 16)).astype(np.float32), rng.uniform(-0.5, 0.5, (16, 7)).astype(np.float32)]
    bs = [np.full(16, 0.01, np.float32), np.zeros(7, np.float32)]
    fx["gcn_w0"], fx["gcn_w1"], fx["gcn_b0"], fx["gcn_b1"] = ws[0], ws[1], bs[0], bs[1]
    fx["gcn_exact"] = digest(ref.gcn_forward(gn, b, ws, bs, None))
    fx["gcn_w32"] = digest(ref.gcn_forward(gn, b, ws, bs, 32, 0))
    fx["gcn_w8"] = digest(ref.gcn_forward(gn, b, ws, bs, 8, 0))
    # quantization of the features (global min/max, 8 and 4 bits)
    for bits in (8, 4):
        lo, hi = ref.fit_params(b, bits)
        codes = ref.quantize(b, lo, hi, bits)
        fx[f"q{bits}_params"] = np.array([lo, hi], np.float32)
        deq = ref.dequantize(codes, lo, hi, bits)
        fx[f"q{bits}_codes"] = digest(codes)
        fx[f"q{bits}_deq"] = digest(deq)
        fx[f"q{bits}_spmm_adaptive_32"] = digest(ref.spmm_sampled(graw, deq, 32, 0))
    np.savez_compressed(os.path.join(OUT, "cora_shape.npz"), **fx)

    # --- heavy-tailed graph: every Table-1 branch, W = 32
    h = ref.gen_synthetic(2000, 1.2, 1500, 31)
    hrp, hcol, _ = h.arrays()
    hval, hb = heavy_inputs(hcol.size)
    hg = ref.RefCsr.from_arrays(2000, 2000, hrp, hcol, hval)
    hx = {"row_ptr": hrp, "col": hcol}
    for w in (16, 32, 64):
        hx[f"spmm_adaptive_{w}"] = digest(ref.spmm_sampled(hg, hb, w, 0))
        chunk, cnt, sp, starts = ref.build_plans(hg, w, 0)
        hx[f"plan_{w}_chunk"], hx[f"plan_{w}_cnt"] = chunk, cnt
        hx[f"plan_{w}_starts_ptr"], hx[f"plan_{w}_starts"] = sp, starts
        cr, cf = ref.cdf_stats(ref.sampling_rate_per_row(hg, w, 0))
        hx[f"cdf_{w}_rate"], hx[f"cdf_{w}_frac"] = cr, cf
    np.savez_compressed(os.path.join(OUT, "heavy_tail.npz"), **hx)
    for f in ("cora_shape.npz", "heavy_tail.npz"):
        print(f, os.path.getsize(os.path.join(OUT, f)), "bytes")


if __name__ == "__main__":
    main()
