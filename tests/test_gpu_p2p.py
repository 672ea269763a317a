"""Fused GEMM + exchange over CUDA-IPC peer memory (gcn.ShardedGCN with
exchange="p2p").  Rank r runs on cuda:(r % device_count): on a multi-GPU box
the ranks sit on distinct devices and the epilogue stores cross NVLink; on a
one-GPU box two ranks share cuda:0 as two processes, and the IPC mapping,
P2P epilogue stores, per-CTA system-scope arrivals and the device-side step
barrier are exercised exactly as across NVLink peers.  The result must
equal the single-process oracle bit for bit.  The NCCL all-gather mode runs
across two real devices when the box has them (skipped otherwise)."""
import os
import socket

import numpy as np
import pytest

from oracle import port
from tests import graphs

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(n=3001, f=40):
    rng = np.random.default_rng(21)
    rp, col, _ = graphs.power_law(n, alpha=1.7, max_deg=500, seed=21)
    nrp, ncol, nval = port.gcn_normalize(rp, col, True)
    x = rng.uniform(-1, 1, (n, f)).astype(np.float32)
    ws = [rng.uniform(-0.5, 0.5, (f, 64)).astype(np.float32), rng.uniform(-0.5, 0.5, (64, 64)).astype(np.float32),
          rng.uniform(-0.5, 0.5, (64, 7)).astype(np.float32)]
    bs = [np.full(64, 0.01, np.float32), np.full(64, -0.02, np.float32), np.zeros(7, np.float32)]
    return nrp, ncol, nval, x, ws, bs


def _run(rank, world, port_no, q, fast=False, exchange_dtype="f32", halo=False, fused=False):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    torch.cuda.set_device(rank % torch.cuda.device_count())  # distinct devices when the box has them
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_18427_b200 import device
        from paper_2503_18427_b200.gcn import ShardedGCN
        if fused:  # every fp32 layer through the fused SpMM + GEMM + exchange kernel
            device.FUSED_LAYER_MIN_ROWS = 0
        nrp, ncol, nval, x, ws, bs = _problem()
        g = device.Graph.from_numpy(nrp, ncol, nval)
        plan = device.SampledPlan(g, 16)
        model = ShardedGCN(plan.srow_ptr, plan.scol, plan.sval, g.n_rows,
                           [torch.from_numpy(w).cuda() for w in ws], [torch.from_numpy(b).cuda() for b in bs],
                           exchange="p2p", fast_gemm=fast, exchange_dtype=exchange_dtype,
                           max_row_slots=plan.row_bound, halo=halo)
        xt = torch.from_numpy(x).cuda()
        outs = [model.forward(xt).cpu().numpy() for _ in range(3)]  # repeated steps exercise the barrier
        torch.cuda.synchronize()
        if halo and exchange_dtype == "f32":
            # rows this rank never reads were never sent: in the replica that
            # held the input (40 columns) and then the second hidden layer
            # (64 columns), their columns 40..63 are still the initial zeros
            need = model.replicas.need[: g.n_rows].bool()
            unsent = ~need
            tail = model.replicas.bufs[0][: g.n_rows, 40:64]
            outs.append((int(unsent.sum().item()), bool((tail[unsent] == 0).all().item()),
                         float((tail[need] != 0).any(1).float().mean().item())))
        q.put((rank, outs))
    except Exception as e:  # surface the failure to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
        raise
    finally:
        if world > 1:
            dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2])
def test_p2p_tcgen05_fused_exchange_within_bound(world):
    """tcgen05 TF32 GEMM whose TMA-store epilogue writes every rank's replica
    (fast mode): within the TF32 bound of the exact result."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, p, q, True)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=120)
    for _, outs in res:
        assert not isinstance(outs, str), outs
    nrp, ncol, nval, x, ws, bs = _problem()
    want = port.gcn_forward(nrp, ncol, nval, x, ws, bs, 16)
    for _, outs in res:
        for o in outs:
            assert np.abs(o - want).max() / np.abs(want).max() < 2e-2
            assert (o.argmax(1) == want.argmax(1)).mean() > 0.98
        assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])
    if world == 2:  # both ranks hold the same replica bits
        assert np.array_equal(res[0][1][0], res[1][1][0])


@pytest.mark.parametrize("world,fused", [(1, False), (2, False), (1, True), (2, True)])
def test_p2p_fused_exchange_matches_oracle(world, fused):
    """GEMM epilogue exchange, and (fused=True) the whole layer — SpMM + GEMM
    + stores into every replica — as one kernel per rank."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, p, q, False, "f32", False, fused)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=120)
    for _, outs in res:
        assert not isinstance(outs, str), outs
    nrp, ncol, nval, x, ws, bs = _problem()
    want = port.gcn_forward(nrp, ncol, nval, x, ws, bs, 16)
    for _, outs in res:
        for o in outs:
            assert np.array_equal(np.ascontiguousarray(o).view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("world", [1, 2])
def test_p2p_int8_exchange_matches_reference_composition(world):
    """int8 layer exchange over peer memory (exchange.cu): device-side param
    publish + rank-order fold + LUT, codes quantized straight into every
    rank's replica.  Bit-exact vs the reference composition
    dequantize(quantize(H, fit_params(H))) per hidden layer."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, p, q, False, "int8")) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=120)
    for _, outs in res:
        assert not isinstance(outs, str), outs
    nrp, ncol, nval, x, ws, bs = _problem()
    want = port.gcn_forward_int8_exchange(nrp, ncol, nval, x, ws, bs, 16)
    for _, outs in res:
        for o in outs:
            assert np.array_equal(np.ascontiguousarray(o).view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("exchange_dtype,fused", [("f32", False), ("int8", False), ("f32", True)])
def test_p2p_halo_exchange_matches_oracle(exchange_dtype, fused):
    """Halo exchange: producers store a hidden-layer row
    into a peer's replica only where the peer's sampled slots reference it.
    Results stay bit-exact, and the rows a rank never reads are never sent."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_run, args=(r, 2, p, q, False, exchange_dtype, True, fused)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=120)
    for _, outs in res:
        assert not isinstance(outs, str), outs
    nrp, ncol, nval, x, ws, bs = _problem()
    if exchange_dtype == "f32":
        want = port.gcn_forward(nrp, ncol, nval, x, ws, bs, 16)
    else:
        want = port.gcn_forward_int8_exchange(nrp, ncol, nval, x, ws, bs, 16)
    for _, outs in res:
        for o in outs[:3]:
            assert np.array_equal(np.ascontiguousarray(o).view(np.uint32), want.view(np.uint32))
        if exchange_dtype == "f32":
            n_unsent, untouched, sent_filled = outs[3]
            assert n_unsent > 0 and untouched and sent_filled > 0.9


def _run_nccl(rank, world, port_no, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        from paper_2503_18427_b200 import device
        from paper_2503_18427_b200.gcn import ShardedGCN
        nrp, ncol, nval, x, ws, bs = _problem()
        g = device.Graph.from_numpy(nrp, ncol, nval)
        plan = device.SampledPlan(g, 16)
        outs = []
        for fused_min in (0, 1 << 40):  # the fused layer kernel, then the split kernels
            model = ShardedGCN(plan.srow_ptr, plan.scol, plan.sval, g.n_rows,
                               [torch.from_numpy(w).cuda() for w in ws], [torch.from_numpy(b).cuda() for b in bs],
                               exchange="nccl", max_row_slots=plan.row_bound)
            model.fused_min_rows = fused_min
            outs.append(model.forward(torch.from_numpy(x).cuda()).cpu().numpy())
        q.put((rank, outs))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


def test_nccl_exchange_across_two_devices():
    """ShardedGCN(exchange="nccl") with one rank per device over a real NCCL
    communicator (NVLink between the two GPUs): bit-exact vs the oracle."""
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (this box has one)")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_run_nccl, args=(r, 2, p, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=120)
    for _, outs in res:
        assert not isinstance(outs, str), outs
    nrp, ncol, nval, x, ws, bs = _problem()
    want = port.gcn_forward(nrp, ncol, nval, x, ws, bs, 16)
    for _, outs in res:
        for o in outs:
            assert np.array_equal(np.ascontiguousarray(o).view(np.uint32), want.view(np.uint32))
