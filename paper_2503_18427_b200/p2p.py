"""Symmetric peer-memory replicas for the fused GEMM + exchange layer step.

Every rank allocates the same buffers (two ping-pong replicas of the layer
activations H and one monotonically increasing arrival counter), exports them
with CUDA IPC and maps every peer's copy.  The layer GEMM
(`aes_dev_gemm_bias_act_ex` with counters) then stores each output tile into
all ranks' replicas over NVLink and bumps every rank's counter once per CTA;
a rank waits for the expected arrival count on its own counter
(`aes_dev_wait_counter`, ld.acquire.sys) before its next layer reads the
replica.  No NCCL call is on the data path; torch.distributed is used once, to
swap the IPC handles (any backend, gloo included).
"""
from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist
from torch.multiprocessing.reductions import reduce_tensor

from . import capi
from .capi import check, lib, stream_of


def _exchange(t: torch.Tensor, group=None):
    """Map every rank's `t` (same shape everywhere) into this process."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    fn, args = reduce_tensor(t)
    gathered = [None] * world
    dist.all_gather_object(gathered, (fn, args), group=group)
    return [t if r == rank else g[0](*g[1]) for r, g in enumerate(gathered)]


class PeerReplicas:
    """Two activation replicas [rows, ld] + one u64 arrival counter per rank,
    mapped on every rank."""

    def __init__(self, rows: int, ld: int, group=None, device=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        device = device or torch.device("cuda", torch.cuda.current_device())
        self.ld = ld
        self.bufs = [torch.zeros((rows, ld), dtype=torch.float32, device=device) for _ in range(2)]
        # [0] layer arrivals (per CTA), [1] step-start barrier arrivals (per rank)
        self.counter = torch.zeros(2, dtype=torch.int64, device=device)
        if self.world > 1:
            self.peer_bufs = [_exchange(b, group) for b in self.bufs]
            self.peer_ctrs = _exchange(self.counter, group)
        else:
            self.peer_bufs = [[b] for b in self.bufs]
            self.peer_ctrs = [self.counter]
        ptrs = ctypes.c_void_p * self.world
        self.dst = [ptrs(*[t.data_ptr() for t in pb]) for pb in self.peer_bufs]
        self.ctr = ptrs(*[t.data_ptr() for t in self.peer_ctrs])
        self.bar = ptrs(*[t.data_ptr() + 8 for t in self.peer_ctrs])
        self.expected = 0
        self.bar_expected = 0
        torch.cuda.synchronize()
        if dist.is_initialized():
            dist.barrier(group)

    def gemm_publish(self, out_buf: int, a: torch.Tensor, w: torch.Tensor, bias, relu: bool, finite_w: bool,
                     row_offset: int, stream=None, fast: bool = False):
        """act(a @ w + bias) for this rank's rows, stored into every rank's
        replica `out_buf` at rows [row_offset, row_offset + m).  fast=True
        uses the tcgen05 TF32 kernel whose TMA-store epilogue writes the
        peers' replicas (not bit-exact)."""
        m, k = a.shape
        n = w.shape[1]
        w = w.contiguous()
        if fast:
            scratch = torch.empty(int(lib().aes_gemm_tf32_scratch_floats(k, n)), dtype=torch.float32,
                                  device=a.device)
            check(lib().aes_dev_gemm_tf32_bcast(
                a.data_ptr(), m, k, a.stride(0), w.data_ptr(), n, w.stride(0),
                None if bias is None or bias.numel() == 0 else bias.data_ptr(), int(relu),
                ctypes.cast(self.dst[out_buf], ctypes.c_void_p), ctypes.cast(self.ctr, ctypes.c_void_p), self.world,
                row_offset, self.ld, scratch.data_ptr(), stream_of(stream)))
            self._keep = scratch  # alive until the stream passes the next wait
            return
        check(lib().aes_dev_gemm_bias_act_ex(
            a.data_ptr(), m, k, a.stride(0), w.data_ptr(), n, w.stride(0),
            None if bias is None or bias.numel() == 0 else bias.data_ptr(), int(relu), int(finite_w),
            ctypes.cast(self.dst[out_buf], ctypes.c_void_p), ctypes.cast(self.ctr, ctypes.c_void_p), self.world,
            row_offset, self.ld, stream_of(stream)))

    def barrier(self, stream=None):
        """Device-side barrier across ranks (stream-ordered): no rank starts
        writing a new step into peers' replicas while a peer still reads the
        previous step's output."""
        if self.world == 1:
            return
        check(lib().aes_dev_signal_all(ctypes.cast(self.bar, ctypes.c_void_p), self.world, stream_of(stream)))
        self.bar_expected += self.world
        check(lib().aes_dev_wait_counter(self.counter.data_ptr() + 8, self.bar_expected, stream_of(stream)))

    def wait(self, arrivals: int, stream=None):
        """Block the stream until `arrivals` more CTAs have published here."""
        self.expected += arrivals
        check(lib().aes_dev_wait_counter(self.counter.data_ptr(), self.expected, stream_of(stream)))


def gemm_ctas(m: int, n: int, fast: bool = False) -> int:
    """Arrivals one producer's publishing GEMM adds to each counter."""
    if fast:
        return int(lib().aes_gemm_tf32_ctas(m)) if m and n else 0
    return int(lib().aes_gemm_ctas(m, n))


__all__ = ["PeerReplicas", "gemm_ctas", "capi"]
