"""CPU, world_size 2 (gloo): the row-sharded GCN layer driver's partition and
exchange logic (paper_2503_18427_b200/gcn.py) with the CPU oracle injected as
the per-shard compute.  The gathered result must equal the single-process
reference forward bit for bit (SURVEY §8e parity)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port
from tests import graphs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_ops():
    from paper_2503_18427_b200.gcn import Ops

    def spmm(srow, scol, sval, h, out=None):
        r = port.spmm_csr(srow.numpy().view(np.uint64), scol.numpy().view(np.uint32), sval.numpy(),
                          np.ascontiguousarray(h.numpy()))
        return torch.from_numpy(r)

    def gemm(a, w, b, relu, out=None):
        c = port.dense_matmul(np.ascontiguousarray(a.numpy()), w.numpy())
        return torch.from_numpy(port.bias_act(c, None if b is None else b.numpy(), relu))

    def fit(a):
        a = np.ascontiguousarray(a.numpy())
        flag = 0
        try:
            lo, hi = port.fit_params(a)
        except Exception:
            lo, hi, flag = 0.0, 0.0, 1
        out = np.array([lo, hi, 0, 0], np.float32)
        out.view(np.int32)[2] = flag
        return torch.from_numpy(out)

    def quantize(a, lo, hi, out=None):
        return torch.from_numpy(port.quantize(np.ascontiguousarray(a.numpy()), lo, hi).astype(np.uint8))

    def spmm_q8(srow, scol, sval, codes, lo, hi, out=None):
        deq = port.dequantize(np.ascontiguousarray(codes.numpy()).astype(np.uint16), lo, hi)
        return spmm(srow, scol, sval, torch.from_numpy(deq))

    return Ops(spmm=spmm, gemm_bias_act=gemm, alloc=lambda r, c, like: torch.empty((r, c)),
               fit_params=fit, quantize=quantize, spmm_q8=spmm_q8)


def _problem(n=777, f=12):
    rng = np.random.default_rng(9)
    rp, col, _ = graphs.power_law(n, alpha=1.6, max_deg=300, seed=9)
    nrp, ncol, nval = port.gcn_normalize(rp, col, True)
    x = rng.uniform(-1, 1, (n, f)).astype(np.float32)
    ws = [rng.uniform(-0.5, 0.5, (f, 16)).astype(np.float32), rng.uniform(-0.5, 0.5, (16, 16)).astype(np.float32),
          rng.uniform(-0.5, 0.5, (16, 5)).astype(np.float32)]
    bs = [np.full(16, 0.01, np.float32), np.full(16, -0.01, np.float32), np.zeros(5, np.float32)]
    return nrp, ncol, nval, x, ws, bs


def _worker_q8(rank, world, port_no, balance, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_18427_b200.gcn import ShardedGCN
        nrp, ncol, nval, x, ws, bs = _problem()
        srow, scol, sval = port.sample_csr(nrp, ncol, nval, 16)
        model = ShardedGCN(torch.from_numpy(srow.view(np.int64)), torch.from_numpy(scol.view(np.int32)),
                           torch.from_numpy(sval), nrp.size - 1, [torch.from_numpy(w) for w in ws],
                           [torch.from_numpy(b) for b in bs], ops=_oracle_ops(), balance=balance,
                           exchange_dtype="int8")
        out = model.forward(torch.from_numpy(x))
        q.put((rank, out.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("balance", ["rows", "slots"])
def test_sharded_gcn_int8_exchange_world2(balance):
    """int8 layer exchange: global params folded across
    ranks, codes all-gathered, fused-dequant aggregation — equals the
    reference composition dequantize(quantize(H, fit_params(H))) per hidden
    layer, bit for bit, and stays close to the fp32 forward."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_worker_q8, args=(r, 2, p, balance, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=120) for _ in procs], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    nrp, ncol, nval, x, ws, bs = _problem()
    want = port.gcn_forward_int8_exchange(nrp, ncol, nval, x, ws, bs, 16)
    for _, out in res:
        assert np.array_equal(out.view(np.uint32), want.view(np.uint32))
    f32 = port.gcn_forward(nrp, ncol, nval, x, ws, bs, 16)
    assert np.abs(want - f32).max() < 0.05 * np.abs(f32).max()


def _worker(rank, world, port_no, balance, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_18427_b200.gcn import ShardedGCN
        nrp, ncol, nval, x, ws, bs = _problem()
        srow, scol, sval = port.sample_csr(nrp, ncol, nval, 16)
        model = ShardedGCN(torch.from_numpy(srow.view(np.int64)), torch.from_numpy(scol.view(np.int32)),
                           torch.from_numpy(sval), nrp.size - 1, [torch.from_numpy(w) for w in ws],
                           [torch.from_numpy(b) for b in bs], ops=_oracle_ops(), balance=balance)
        out = model.forward(torch.from_numpy(x))
        shard = model.forward(torch.from_numpy(x), return_shard=True)
        q.put((rank, out.numpy().copy(), shard.numpy().copy(), (model.lo, model.hi)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("balance", ["rows", "slots"])
def test_sharded_gcn_world2_matches_single_process(balance):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, p, balance, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=120) for _ in procs], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    nrp, ncol, nval, x, ws, bs = _problem()
    want = port.gcn_forward(nrp, ncol, nval, x, ws, bs, 16)
    for _, out, _, _ in res:
        assert np.array_equal(out.view(np.uint32), want.view(np.uint32))
    shards = np.concatenate([s for _, _, s, _ in res])
    assert np.array_equal(shards.view(np.uint32), want.view(np.uint32))
    (lo0, hi0), (lo1, hi1) = res[0][3], res[1][3]
    assert lo0 == 0 and hi0 == lo1 and hi1 == nrp.size - 1


def test_cut_helpers():
    from paper_2503_18427_b200.gcn import equal_row_cuts, slot_balanced_cuts
    cuts, per = equal_row_cuts(10, 4)
    assert cuts == [0, 3, 6, 9, 10] and per == 3
    srow = np.array([0, 1, 2, 3, 100, 101, 102], np.uint64)
    c = slot_balanced_cuts(srow, 2)
    assert c[0] == 0 and c[-1] == 6 and c[1] in (3, 4)
