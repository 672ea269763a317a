#!/usr/bin/env python3
"""AES-SpMM benchmark (BASELINE.json metric: "AES-SpMM ms & achieved HBM GB/s
(% of peak), F=128, at 1/2/4/8 B200").

Workload (config "products", BASELINE configs[4]): ogbn-products-shaped
synthetic power-law graph (2.45 M rows, ~62 M edges, alpha 1.7885, max degree
17 481), raw adjacency (val = 1), U(-1, 1) fp32 features F = 128, adaptive
sampling W = 32.  A step is one sampled SpMM over this rank's row shard with
the plan prebuilt (as the reference times it: proj/src/bench.cpp:59-77).  At
N > 1 the rows are cut into contiguous slot-balanced shards, every rank holds
the full feature replica and computes its shard (strong scaling, no data-path
collective inside the SpMM; `--mode layer` adds the GCN layer's GEMM and the
NCCL all-gather of the layer output).

value  = whole-job algorithmic bytes / max-over-ranks device time, GB/s
         (8(N+1) + 8S + 4FS + 4FN per SpMM).
e2e    = the same metric through the reference-facing C-ABI handle call
         (aes_spmm_sampled) with pinned HOST buffers: H2D of the features and
         D2H of the result inside the timed region.
--impl reference: the reference's own CPU implementation (oracle/_ref, built
from /root/reference by oracle/Makefile) with every host thread, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SHAPES = {
    # name: (n, alpha, max_degree, F)
    "cora": (2_708, 2.1181, 168, 16),
    "pubmed": (19_717, 2.0321, 171, 128),
    "arxiv": (169_343, 2.0737, 13_161, 128),
    "reddit": (232_965, 1.2986, 21_657, 602),
    "products": (2_450_000, 1.7885, 17_481, 128),
}
METRIC = "AES-SpMM ms & achieved HBM GB/s (% of peak), F=128, at 1/2/4/8 B200"
DATA = "synthetic (GPU power-law generator, seed %d; U(-1,1) features)"


def load_synth():
    """synth.py loaded by file path: the graph generator needs torch only, and
    importing it this way does not run the package __init__ (which loads the
    product's .so files) — the reference arm must not load them."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "aes_bench_synth", os.path.join(ROOT, "paper_2503_18427_b200", "synth.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload_config(args, n, nnz, slots, f, elem):
    """The `config` dict — identical in both arms for the same flags."""
    return {"workload": f"{args.config} W={args.width} {args.strategy} F={f} sampled SpMM"
                        + (" + GEMM + all-gather (GCN layer)" if args.mode == "layer" else ""),
            "n_rows": n, "nnz": nnz, "slots": slots, "F": f, "width": args.width, "strategy": args.strategy,
            "features": {"int8": "u8 codes (global min/max, quantize.cpp:23-51)",
                         "int8-row": "u8 codes, per-row (scale, offset) — fast mode, bounded error",
                         "int8-feature": "u8 codes, per-feature (scale, offset) — fast mode, bounded error"
                         }.get(getattr(args, "dtype", "f32"), "f32"),
            "l2": "inputs larger than L2 (features %.2f GB, output %.2f GB vs 126 MB L2)"
                  % (n * f * elem / 1e9, n * f * 4 / 1e9)}


def alg_bytes(n_rows, slots, f, elem=4, slot_extra=0):
    """8(N+1) [srow_ptr] + 8S [scol, sval] + e*F*S [gathered rows] + 4FN [C]
    (+ slot_extra*S: the int8 fast ROW mode gathers an 8-B (scale, offset)
    pair with every row)."""
    return 8 * (n_rows + 1) + 8 * slots + elem * f * slots + 4 * f * n_rows + slot_extra * slots


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def shard_bounds(srow_ptr_host, world):
    """Contiguous row cuts with ~equal sampled slots per shard."""
    import numpy as np
    total = int(srow_ptr_host[-1])
    n = srow_ptr_host.size - 1
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(srow_ptr_host, total * r // world, side="left")))
    cuts.append(n)
    for i in range(1, len(cuts)):
        cuts[i] = max(cuts[i], cuts[i - 1])
    return cuts


def load_traffic(kind):
    """dram bytes/launch of the dominant kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d.get(kind, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ------------------------------------------------------------------------------------------ reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np
    import torch

    n, alpha, maxdeg, f = SHAPES[args.config]
    from oracle import ref as oref  # the reference CPU implementation, built from its own sources
    if not oref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (make -C oracle ref)"}))
        return 0
    synth = load_synth()  # by path: no product .so is loaded in this arm
    gdev = "cuda" if torch.cuda.is_available() else "cpu"
    rp, col, val = synth.power_law_csr(n, alpha, maxdeg, seed=args.seed, device=gdev)
    b = synth.features(n, f, seed=5, device=gdev, ld=f)
    if args.dtype == "int8":
        print(json.dumps({"impl": "reference", "unavailable": "int8 arm: the reference has no quantized SpMM "
                          "entry point (dequantize + spmm_sampled is what it would run)"}))
        return 0
    rp_np = rp.cpu().numpy().view(np.uint64)
    col_np = col.cpu().numpy().view(np.uint32)
    val_np = val.cpu().numpy()
    b_np = np.ascontiguousarray(b.cpu().numpy())
    del rp, col, val, b
    csr = oref.RefCsr.from_arrays(n, n, rp_np, col_np, val_np)
    threads = os.cpu_count() or 1
    strat = {"adaptive": 0, "afs": 1, "sfs": 2, "full": 3}[args.strategy]
    plan_ms, ms, _ = oref.time_spmm_sampled(csr, b_np, args.width, strat, threads, args.warmup + args.steps)
    timed = ms[args.warmup:]
    chunk, cnt, _, _ = oref.build_plans(csr, args.width, strat)
    slots = int((chunk.astype(np.uint64) * cnt.astype(np.uint64)).sum())
    by = alg_bytes(n, slots, f)
    t = float(np.mean(timed))
    gbs = by / (t * 1e-3) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 3), "unit": "GB/s", "n_gpus": max(world, args.gpus),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": DATA % args.seed,
        "config": workload_config(args, n, int(rp_np[-1]), slots, f, 4),
        "plan_ms": round(plan_ms, 3), "median_ms": round(float(np.median(timed)), 3),
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"full {args.config} workload, reference aes::spmm_sampled "
                                   f"(proj/src/spmm.cpp:40-107), {threads} std::threads, prebuilt plans"},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------ our arm
def cpu_baseline(args, rp_np, col_np, val_np, b_np, f):
    """Reference CPU path (oracle/_ref) on a bounded row sample, all host threads."""
    import numpy as np
    try:
        from oracle import ref as oref
        if not oref.available():
            raise ImportError
        kind = "reference"
    except Exception:
        oref = None
        kind = "port"
    n = rp_np.size - 1
    rows = n if kind == "reference" else min(n, 200_000)
    sub_rp = rp_np[: rows + 1]
    nnz = int(sub_rp[-1])
    threads = os.cpu_count() or 1
    strat = {"adaptive": 0, "afs": 1, "sfs": 2, "full": 3}[args.strategy]
    if kind == "reference":
        csr = oref.RefCsr.from_arrays(rows, n, sub_rp, col_np[:nnz], val_np[:nnz])
        _, ms, _ = oref.time_spmm_sampled(csr, b_np, args.width, strat, threads, 3)
        chunk, cnt, _, _ = oref.build_plans(csr, args.width, strat)
        slots = int((chunk.astype(np.uint64) * cnt.astype(np.uint64)).sum())
        t = float(np.median(ms))
        sample = f"first {rows} rows of the workload, reference spmm_sampled, median of 3"
    else:
        from oracle import port
        threads = 1
        srow, scol, sval = port.sample_csr(sub_rp, col_np[:nnz], val_np[:nnz], args.width, strat)
        t0 = time.perf_counter()
        port.spmm_csr(srow, scol, sval, b_np)
        t = (time.perf_counter() - t0) * 1e3
        slots = int(srow[-1])
        sample = f"first {rows} rows of the workload, oracle port (scalar C)"
    gbs = alg_bytes(rows, slots, f) / (t * 1e-3) / 1e9
    return {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": kind, "sample": sample,
            "cpu_model": cpu_model(),
            "ms": round(t, 3)}


def max_over_ranks(x: float, dist) -> float:
    """MAX over ranks (a device tensor under NCCL, a host one under gloo)."""
    import torch
    if not dist:
        return float(x)
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args):
    import numpy as np
    import torch

    rank, world, local = dist_env()
    # one GPU per rank over NCCL.  With fewer devices than ranks (a one-GPU
    # box) the ranks share devices over gloo: a functional check of the
    # multi-rank path only, flagged in the line ("shared_devices")
    n_dev = max(torch.cuda.device_count(), 1)
    shared = world > n_dev
    local = local % n_dev
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("AES_BENCH_BACKEND", "gloo" if shared else "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    from paper_2503_18427_b200 import capi, device
    synth = load_synth()
    capi.check(capi.lib().aes_dev_spmm_set_schedule(args.sched))
    capi.lib().aes_dev_spmm_set_variant.argtypes = [ctypes.c_int]
    capi.check(capi.lib().aes_dev_spmm_set_variant(args.variant))

    n, alpha, maxdeg, f = SHAPES[args.config]
    rp, col, val = synth.power_law_csr(n, alpha, maxdeg, seed=args.seed, device="cuda")
    g = device.Graph(rp, col, val, n)
    b = synth.features(n, f, seed=5, device="cuda")
    strat = capi.strategy_code(args.strategy)
    full_plan = device.SampledPlan(g, args.width, strat)
    srow_host = full_plan.srow_ptr.cpu().numpy()
    cuts = shard_bounds(srow_host, world)
    lo, hi = cuts[rank], cuts[rank + 1]
    # the shard is a view of the global sampled CSR (absolute slot offsets)
    srow = full_plan.srow_ptr[lo:hi + 1]
    shard_rows = hi - lo
    shard_slots = int(srow_host[hi] - srow_host[lo])
    stream = torch.cuda.current_stream()

    quant = None
    qaff = None
    slot_extra = 0
    if args.dtype == "int8":
        quant = device.quantize(b)
        elem = 1
    elif args.dtype in ("int8-row", "int8-feature"):  # fast mode (affine.cu), not bit-exact
        qaff = device.quantize_affine(b, args.dtype.split("-")[1])
        elem = 1
        slot_extra = 8 if args.dtype == "int8-row" else 0
    else:
        elem = 4
    out = device.empty_padded(max(shard_rows, 1), f)

    layer = None
    if args.mode == "layer":
        w = (torch.rand(f, f, device="cuda") - 0.5)
        bias = torch.full((f,), 0.01, device="cuda")
        per = max(c1 - c0 for c0, c1 in zip(cuts, cuts[1:]))
        # the next-layer replica; this rank's GEMM writes its own slice and
        # the all-gather runs in place on it (no send buffer, no copy)
        gathered = torch.zeros((per * world, (f + 3) & ~3), device="cuda")
        mine = gathered[rank * per:(rank + 1) * per]
        layer = (w, bias, gathered, mine)

    def step():
        if qaff is not None:
            device.spmm_q8_affine(srow, full_plan.scol, full_plan.sval, qaff, out=out)
        elif quant is not None:
            device.spmm_q8(srow, full_plan.scol, full_plan.sval, quant, out=out, max_row_slots=full_plan.row_bound)
        else:
            device.spmm(srow, full_plan.scol, full_plan.sval, b, out=out, max_row_slots=full_plan.row_bound)
        if layer is not None:
            w, bias, gathered, mine = layer
            if shard_rows:
                device.gemm_bias_act(out[:shard_rows], w, bias, True, out=mine[:shard_rows, :f])
            if world > 1:
                dist.all_gather_into_tensor(gathered, mine)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.nvtx.range_push("timed")
    start.record(stream)
    for _ in range(args.steps):
        step()
    end.record(stream)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms_total = start.elapsed_time(end)
    ms_step = max_over_ranks(ms_total, dist) / args.steps
    total_bytes = alg_bytes(n, int(srow_host[-1]), f, elem, slot_extra)
    my_bytes = alg_bytes(shard_rows, shard_slots, f, elem, slot_extra)
    value = total_bytes / (ms_step * 1e-3) / 1e9
    # kernel-level roofline for this rank (the step is the SpMM kernel alone in spmm mode)
    k_ms = ms_total / args.steps
    peak, peak_kind = peaks()
    achieved = my_bytes / (k_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4),
                # the committed ncu capture is of the full-graph launch (N = 1)
                "traffic": load_traffic(f"spmm_{args.dtype}_{args.config}") if world == 1 else None,
                "traffic_source": "static: dram__bytes_read.sum + dram__bytes_write.sum of this kernel from the "
                                  "committed ncu --set full capture (profiles/ncu_summary.json), not measured in "
                                  "this run",
                "peak_kind": peak_kind, "alg_bytes_per_launch": my_bytes, "nominal_8000_frac": round(achieved / 8000, 4)}

    # ---- kernels one step launches, counted by CUPTI (torch.profiler) on one
    # extra step after the timed region; gpu_launches = per-step count x steps
    launches = count_launches(step)

    # ---- e2e through the reference-facing C-ABI handle call, pinned host buffers
    e2e = None
    if not args.no_e2e and args.dtype == "f32":
        e2e = run_e2e(args, rp, col, val, b, lo, hi, f, n, total_bytes, dist, world)
        if world == 1:
            try:
                e2e["pybind_call"] = run_pybind_call(args, rp, col, val, b, f, total_bytes)
            except Exception as e:  # reporting only
                e2e["pybind_call"] = {"error": f"{type(e).__name__}: {str(e)[:200]}"}
    elif not args.no_e2e and args.dtype == "int8":
        e2e = run_e2e_q8(args, quant, full_plan, srow, shard_rows, f, total_bytes, dist)

    # ---- one GCN layer through the row-sharded driver (SpMM -> GEMM -> exchange
    # fused into the GEMM epilogue over peer memory): exact ordered-fp32 GEMM
    # (bit-exact with the reference) and the tcgen05 TF32 fast mode
    gcn_layer = None
    layer_failed = False
    if not args.no_layer and args.dtype == "f32" and args.mode == "spmm":
        try:
            gcn_layer = run_gcn_layer(args, full_plan, n, f, b, dist)
        except Exception as e:  # the SpMM line above stands on its own
            gcn_layer = {"error": f"{type(e).__name__}: {str(e)[:200]}"}
            layer_failed = True

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        b_np = np.ascontiguousarray(b.cpu().numpy())
        cpu = cpu_baseline(args, rp.cpu().numpy().view(np.uint64), col.cpu().numpy().view(np.uint32),
                           val.cpu().numpy(), b_np, f)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8" if args.dtype.startswith("int8") else "f32",
            "data": DATA % args.seed,
            "config": workload_config(args, n, int(rp[-1].item()), int(srow_host[-1]), f, elem),
            "parallelism": f"row-sharded x{world}" if world > 1 else "single GPU",
            "shard_rows": [c1 - c0 for c0, c1 in zip(cuts, cuts[1:])],
            "roofline": roofline, "clocks": clocks,
            "e2e": e2e, "cpu_baseline": cpu, "gcn_layer": gcn_layer,
            "gpu_launches": launches["per_step"] * args.steps,
            "gpu_launches_per_step": launches,
        }
        if world > 1:
            line["backend"] = dist.get_backend()
            line["shared_devices"] = shared
        if gcn_layer and "error" not in gcn_layer:
            # N > 1 headline pair: the SpMM-only step (value) and the layer step
            line["layer_step"] = {
                "spmm_only_ms": round(ms_step, 5),
                "layer_nccl_ms": gcn_layer.get("exact_nccl_allgather_ms"),
                "layer_p2p_fused_ms": gcn_layer.get("exact_ordered_fp32_ms"),
                "layer_p2p_fused_tf32_ms": gcn_layer.get("fast_tcgen05_tf32_ms"),
                "what": "one GCN layer F->F: shard SpMM -> ordered GEMM + bias + ReLU -> exchange of the "
                        "next-layer replica (NCCL in-place all-gather, or stores to every rank's replica "
                        "from the GEMM epilogue over peer memory)"}
        print(json.dumps(line), flush=True)
    if layer_failed:  # the device context may be gone: no collective teardown
        sys.stdout.flush()
        os._exit(0)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def count_launches(step):
    """Kernels one step launches, from CUPTI activity records (torch.profiler):
    ours (the repo's .so) and any others, by name."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    try:
        with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as prof:
            step()
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    except Exception as e:  # profiler unavailable: say so, claim nothing
        return {"per_step": 0, "error": f"{type(e).__name__}: {str(e)[:120]}"}
    kernels = [nm for nm in names if not nm.startswith(("Memcpy", "Memset", "memcpy", "memset"))]
    other = [nm for nm in kernels if "at::" in nm or "nccl" in nm.lower() or "gloo" in nm]
    ours = [nm for nm in kernels if nm not in other]
    short = sorted({nm.split("<")[0].split("::")[-1].split("(")[0].replace("void ", "") for nm in ours})
    return {"per_step": len(ours), "other_per_step": len(other), "kernels": short,
            "how": "CUPTI kernel records of one extra step (torch.profiler), not in the timed region"}


def run_pybind_call(args, rp, col, val, b, f, total_bytes):
    """The call a reference Python user makes: _core.spmm_sampled(a, b, plans)
    on numpy arrays (module.cpp:124-131) — pageable host memory, synchronous."""
    import numpy as np

    import paper_2503_18427_b200 as m
    n = rp.numel() - 1
    a = m.CsrMatrix(n, n, rp.cpu().numpy().view(np.uint64), col.cpu().numpy().view(np.uint32), val.cpu().numpy())
    plans = m.build_plan_set(a, args.width, getattr(m.Strategy, args.strategy.upper()))
    b_np = np.ascontiguousarray(b.cpu().numpy()[:, :f])
    m.spmm_sampled(a, b_np, plans)
    steps = 3
    t0 = time.perf_counter()
    for _ in range(steps):
        m.spmm_sampled(a, b_np, plans)
    t = (time.perf_counter() - t0) / steps
    return {"value": round(total_bytes / t / 1e9, 3), "ms_per_step": round(t * 1e3, 3),
            "h2d_bytes_per_step": n * f * 4, "d2h_bytes_per_step": n * f * 4,
            "path": "paper_2503_18427_b200._core.spmm_sampled(a, numpy b, plans) (== aes_spmm._core), "
                    "pageable numpy buffers, synchronous, mean of %d" % steps}


def release(model):
    """Drop a model's peer mappings on every rank before any rank frees the
    exported buffers (CUDA IPC: consumers close before producers exit)."""
    import gc

    import torch
    model.replicas = None
    gc.collect()
    torch.cuda.synchronize()
    if torch.distributed.is_initialized():
        torch.distributed.barrier()


def run_gcn_layer(args, plan, n, f, b, dist):
    """Time one GCN layer (F -> F, ReLU) with gcn.ShardedGCN(exchange="p2p"):
    sampled SpMM of this rank's rows, then the layer GEMM whose epilogue writes
    every rank's next-layer replica (peer memory) and signals arrivals."""
    import torch

    from paper_2503_18427_b200.gcn import ShardedGCN
    w = (torch.rand(f, f, device="cuda", generator=torch.Generator("cuda").manual_seed(3)) - 0.5)
    bias = torch.full((f,), 0.01, device="cuda")
    x = b[:, :f]
    out = {}
    # SpMM -> exact GEMM (epilogue writes this rank's slice) -> in-place NCCL
    # all-gather of the next-layer replica (gcn.ShardedGCN exchange="nccl")
    model = ShardedGCN(plan.srow_ptr, plan.scol, plan.sval, n, [w], [bias], exchange="nccl",
                       max_row_slots=plan.row_bound)
    for _ in range(2):
        model.forward(x, copy_out=False)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(3, min(args.steps, 10))
    s.record()
    for _ in range(steps):
        model.forward(x, copy_out=False)
    e.record()
    torch.cuda.synchronize()
    out["exact_nccl_allgather_ms"] = round(max_over_ranks(s.elapsed_time(e) / steps, dist), 4)
    out["exact_nccl_layer_kernels"] = ("fused SpMM + ordered GEMM, one persistent kernel (aes_dev_gcn_layer_fused)"
                                       if model.fused_min_rows and model.hi - model.lo >= model.fused_min_rows
                                       else "split: sampled SpMM, then ordered GEMM")
    del model
    for name, fast in (("exact_ordered_fp32", False), ("fast_tcgen05_tf32", True)):
        model = ShardedGCN(plan.srow_ptr, plan.scol, plan.sval, n, [w], [bias], exchange="p2p", fast_gemm=fast,
                           max_row_slots=plan.row_bound)
        model.input_view().copy_(x)  # features resident in the replica; steps run in place
        x_step = None
        for _ in range(2):
            model.forward(x_step, copy_out=False)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = max(3, min(args.steps, 10))
        s.record()
        for _ in range(steps):
            model.forward(x_step, copy_out=False)
        e.record()
        torch.cuda.synchronize()
        out[name + "_ms"] = round(max_over_ranks(s.elapsed_time(e) / steps, dist), 4)
        release(model)
        del model
    # two layers (F -> F -> F): the hidden output crosses the exchange as fp32
    # (GEMM epilogue broadcast) or as int8 codes (device param fold + quantize
    # straight into every replica, exchange.cu); exact GEMMs, input copied in
    w2 = (torch.rand(f, f, device="cuda", generator=torch.Generator("cuda").manual_seed(4)) - 0.5)
    variants = [("f32", "f32", False), ("int8", "int8", False)]
    if dist:  # halo masks only differ from a full broadcast with peers
        variants += [("f32_halo", "f32", True), ("int8_halo", "int8", True)]
    for name, xdt, halo in variants:
        model = ShardedGCN(plan.srow_ptr, plan.scol, plan.sval, n, [w, w2], [bias, bias], exchange="p2p",
                           exchange_dtype=xdt, max_row_slots=plan.row_bound, halo=halo)
        for _ in range(2):
            model.forward(x, copy_out=False)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = max(3, min(args.steps, 5))
        s.record()
        for _ in range(steps):
            model.forward(x, copy_out=False)
        e.record()
        torch.cuda.synchronize()
        out[f"two_layer_{name}_exchange_ms"] = round(max_over_ranks(s.elapsed_time(e) / steps, dist), 4)
        release(model)
        del model
    out["exchange"] = "fused into the GEMM epilogue (P2P stores to every rank's replica + sys-scope arrivals)"
    out["int8_exchange"] = ("hidden layer output as 8-bit codes: per-rank fit_params published to every rank, "
                            "rank-order fold + LUT on the device, codes quantized into every replica (4x fewer bytes)")
    out["halo"] = "hidden-layer rows stored only into the replicas whose sampled slots reference them (N > 1)"
    out["note"] = "exact mode is bit-exact with the reference; fast mode |err| <= 2^-8 sum|a||w| (TF32)"
    return out


def run_e2e_q8(args, quant, plan, srow, rows, f, total_bytes, dist):
    """int8 end to end: the u8 codes (what an int8 FMAT file holds) go H2D
    from pinned host memory, the fused-dequant SpMM runs, the fp32 result
    comes back D2H; steps alternate over two streams so one step's D2H
    overlaps the next step's H2D."""
    import torch

    from paper_2503_18427_b200 import device
    codes_host = torch.empty(quant.codes.shape, dtype=torch.uint8).pin_memory()
    codes_host.copy_(quant.codes)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    codes_dev = [device.empty_padded(*quant.codes.shape, dtype=torch.uint8) for _ in range(2)]
    outs = [device.empty_padded(max(rows, 1), f) for _ in range(2)]
    host_out = [torch.empty((max(rows, 1), f), dtype=torch.float32).pin_memory() for _ in range(2)]

    def step(i):
        j = i % 2
        with torch.cuda.stream(streams[j]):
            codes_dev[j].copy_(codes_host, non_blocking=True)
            q = device.QuantizedDevice(codes_dev[j], quant.x_min, quant.x_max, quant.bits, quant.lut)
            device.spmm_q8(srow, plan.scol, plan.sval, q, out=outs[j], max_row_slots=plan.row_bound,
                           stream=streams[j])
            host_out[j].copy_(outs[j], non_blocking=True)

    for i in range(2):
        step(i)
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, 10))
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(steps):
        step(i)
    torch.cuda.synchronize()
    t = max_over_ranks((time.perf_counter() - t0) / steps, dist)
    return {"value": round(total_bytes / t / 1e9, 3), "unit": "GB/s", "ms_per_step": round(t * 1e3, 3),
            "h2d_bytes_per_step": int(codes_host.numel()), "d2h_bytes_per_step": max(rows, 1) * f * 4,
            "path": "u8 codes H2D (pinned) -> device spmm_q8 -> fp32 result D2H, 2 streams, steps=%d" % steps}


def run_e2e(args, rp, col, val, b, lo, hi, f, n, total_bytes, dist, world):
    """aes_csr_create / aes_build_plan_set once, then per step the host-buffer
    call aes_spmm_sampled (H2D features, kernel, D2H result) — the call a
    reference user makes (proj/bindings/module.cpp:124-131)."""
    import numpy as np
    import torch

    from paper_2503_18427_b200 import capi
    L = capi.lib()
    vp, u64 = ctypes.c_void_p, ctypes.c_uint64
    L.aes_csr_create.argtypes = [u64, u64, vp, u64, vp, vp, u64, vp]
    L.aes_build_plan_set.argtypes = [vp, ctypes.c_uint32, ctypes.c_int, vp]
    L.aes_spmm_sampled.argtypes = [vp, vp, u64, u64, vp, vp, vp, vp, vp]
    L.aes_csr_destroy.argtypes = [vp]
    L.aes_plan_destroy.argtypes = [vp]
    rp_np = rp.cpu().numpy().view(np.uint64)
    base = int(rp_np[lo])
    srp = np.ascontiguousarray(rp_np[lo:hi + 1] - np.uint64(base))
    nnz = int(srp[-1])
    scol = np.ascontiguousarray(col.cpu().numpy().view(np.uint32)[base:base + nnz])
    sval = np.ascontiguousarray(val.cpu().numpy()[base:base + nnz])
    h = ctypes.c_void_p()
    capi.check(L.aes_csr_create(hi - lo, n, srp.ctypes.data, srp.size, scol.ctypes.data, sval.ctypes.data, nnz,
                                ctypes.byref(h)))
    p = ctypes.c_void_p()
    capi.check(L.aes_build_plan_set(h, args.width, capi.strategy_code(args.strategy), ctypes.byref(p)))
    b_host = torch.empty((n, f), dtype=torch.float32).pin_memory()
    b_host.copy_(b[:, :f])
    c_host = torch.empty((max(hi - lo, 1), f), dtype=torch.float32).pin_memory()

    L.aes_spmm_sampled_async.argtypes = [vp, vp, u64, u64, vp, vp, vp]
    c_host2 = torch.empty_like(c_host).pin_memory()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]

    def call():
        capi.check(L.aes_spmm_sampled(h, b_host.data_ptr(), n, f, p, c_host.data_ptr(), None, None, None))

    def call_async(i):
        # step i: H2D(features) -> SpMM -> D2H(result) on its own stream; the next
        # step's H2D overlaps this step's D2H on the other copy engine
        out = c_host if i % 2 == 0 else c_host2
        capi.check(L.aes_spmm_sampled_async(h, b_host.data_ptr(), n, f, p, out.data_ptr(),
                                            streams[i % 2].cuda_stream))

    def timed(fn, steps, sync):
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(steps):
            fn(i)
        sync()
        return max_over_ranks((time.perf_counter() - t0) / steps, dist)

    steps = max(1, min(args.steps, 10))
    for _ in range(max(1, min(args.warmup, 3))):
        call()
    t_sync = timed(lambda i: call(), steps, lambda: None)
    for i in range(2):
        call_async(i)
    torch.cuda.synchronize()
    t = timed(call_async, steps, torch.cuda.synchronize)
    L.aes_plan_destroy(p)
    L.aes_csr_destroy(h)
    # the e2e ceiling: the same H2D + D2H bytes as plain pinned copies, both
    # directions at once (no SpMM) — what PCIe allows per step on this box
    d_in = torch.empty((n, f), dtype=torch.float32, device="cuda")
    d_out = torch.empty_like(c_host, device="cuda")

    def copies(i):
        with torch.cuda.stream(streams[0]):
            d_in.copy_(b_host, non_blocking=True)
        with torch.cuda.stream(streams[1]):
            c_host.copy_(d_out, non_blocking=True)

    copies(0)
    torch.cuda.synchronize()
    t_copy = timed(copies, 3, torch.cuda.synchronize)
    del d_in, d_out
    return {"value": round(total_bytes / t / 1e9, 3), "unit": "GB/s", "ms_per_step": round(t * 1e3, 3),
            "pcie_ceiling": {"ms_per_step": round(t_copy * 1e3, 3), "frac": round(t_copy / t, 4),
                             "what": "pinned H2D of the features + D2H of the result, both directions at once, "
                                     "no compute: the e2e step cannot beat this"},
            "h2d_bytes_per_step": n * f * 4, "d2h_bytes_per_step": (hi - lo) * f * 4,
            "path": "C-ABI aes_spmm_sampled_async on 2 streams, pinned host buffers, steps=%d" % steps,
            "sync_call": {"value": round(total_bytes / t_sync / 1e9, 3), "ms_per_step": round(t_sync * 1e3, 3),
                          "path": "C-ABI aes_spmm_sampled (synchronous, like the reference call)"}}


def relaunch(args):
    """`bench.py --gpus N` outside torchrun: start N ranks (one per GPU)
    under torch.distributed.run on 127.0.0.1, as the driver would."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=list(SHAPES), default="products")
    ap.add_argument("--width", type=int, default=32)
    ap.add_argument("--strategy", default="adaptive", choices=["adaptive", "afs", "sfs", "full"])
    ap.add_argument("--dtype", default="f32", choices=["f32", "int8", "int8-row", "int8-feature"],
                    help="int8: the reference's exact global codes; int8-row / int8-feature: fast mode")
    ap.add_argument("--mode", default="spmm", choices=["spmm", "layer"])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--sched", type=int, default=0,
                    help="SpMM row schedule (aes_dev_spmm_set_schedule; 0 = library default)")
    ap.add_argument("--variant", type=int, default=0,
                    help="SpMM kernel variant (aes_dev_spmm_set_variant; 0 = library default, tuning only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-layer", action="store_true", help="skip the GCN layer (SpMM+GEMM+exchange) timing")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)  # rank 0 alone does CPU work; no ranks needed
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
