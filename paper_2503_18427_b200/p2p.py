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

    def __init__(self, rows: int, ld: int, group=None, device=None, code_ld: int = 0):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        device = device or torch.device("cuda", torch.cuda.current_device())
        self.ld = ld
        self.bufs = [torch.zeros((rows, ld), dtype=torch.float32, device=device) for _ in range(2)]
        # [0] fp32 layer arrivals (per CTA), [1] step-start barrier arrivals (per
        # rank), [2] int8-exchange param arrivals (per rank), [3] code arrivals (per CTA)
        self.counter = torch.zeros(4, dtype=torch.int64, device=device)
        # int8 exchange (code_ld > 0): two code replicas (layer parity) and two
        # [world, 4] parameter arrays, also peer-mapped
        self.code_ld = code_ld
        self.codes = [torch.zeros((rows, code_ld), dtype=torch.uint8, device=device) for _ in range(2)] \
            if code_ld else []
        self.params = [torch.zeros(4 * self.world, dtype=torch.float32, device=device) for _ in range(2)] \
            if code_ld else []
        if self.world > 1:
            self.peer_bufs = [_exchange(b, group) for b in self.bufs]
            self.peer_ctrs = _exchange(self.counter, group)
            self.peer_codes = [_exchange(c, group) for c in self.codes]
            self.peer_params = [_exchange(pr, group) for pr in self.params]
        else:
            self.peer_bufs = [[b] for b in self.bufs]
            self.peer_ctrs = [self.counter]
            self.peer_codes = [[c] for c in self.codes]
            self.peer_params = [[pr] for pr in self.params]
        ptrs = ctypes.c_void_p * self.world
        self.dst = [ptrs(*[t.data_ptr() for t in pb]) for pb in self.peer_bufs]
        self.ctr = ptrs(*[t.data_ptr() for t in self.peer_ctrs])
        self.bar = ptrs(*[t.data_ptr() + 8 for t in self.peer_ctrs])
        self.par_ctr = ptrs(*[t.data_ptr() + 16 for t in self.peer_ctrs])
        self.code_ctr = ptrs(*[t.data_ptr() + 24 for t in self.peer_ctrs])
        self.code_dst = [ptrs(*[t.data_ptr() for t in pc]) for pc in self.peer_codes]
        self.par_dst = [ptrs(*[t.data_ptr() for t in pp]) for pp in self.peer_params]
        self.expected = 0
        self.bar_expected = 0
        self.par_expected = 0
        self.code_expected = 0
        self.need_ptrs = None
        torch.cuda.synchronize()
        if dist.is_initialized():
            dist.barrier(group)

    def set_halo(self, need: torch.Tensor):
        """This rank's halo mask (uint8 [rows]: 1 = this rank reads that row of
        the replicas); every producer then stores a row into this rank's
        replica only where the mask is set."""
        self.need = need.contiguous()
        peers = _exchange(self.need, self.group) if self.world > 1 else [self.need]
        self._peer_need = peers  # keep the IPC mappings alive
        self.need_ptrs = (ctypes.c_void_p * self.world)(*[t.data_ptr() for t in peers])
        torch.cuda.synchronize()
        if dist.is_initialized():
            dist.barrier(self.group)

    def gemm_publish(self, out_buf: int, a: torch.Tensor, w: torch.Tensor, bias, relu: bool, finite_w: bool,
                     row_offset: int, stream=None, fast: bool = False, halo: bool = False):
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
        need = ctypes.cast(self.need_ptrs, ctypes.c_void_p) if halo and self.need_ptrs is not None else None
        check(lib().aes_dev_gemm_bias_act_halo(
            a.data_ptr(), m, k, a.stride(0), w.data_ptr(), n, w.stride(0),
            None if bias is None or bias.numel() == 0 else bias.data_ptr(), int(relu), int(finite_w),
            ctypes.cast(self.dst[out_buf], ctypes.c_void_p), ctypes.cast(self.ctr, ctypes.c_void_p), need,
            self.world, row_offset, self.ld, stream_of(stream)))

    def layer_publish(self, out_buf: int, srow, scol, sval, x: torch.Tensor, w: torch.Tensor, bias, relu: bool,
                      finite_w: bool, row_offset: int, stream=None, halo: bool = False) -> bool:
        """The whole exact layer for this rank's rows as ONE kernel
        (aes_dev_gcn_layer_fused_bcast: SpMM producer warps + ordered-GEMM
        consumer warps whose epilogue stores into every rank's replica
        `out_buf`, then one arrival per CTA).  False when the shape is outside
        the fused kernel (the caller runs spmm + gemm_publish)."""
        m = srow.numel() - 1
        k, n = x.shape[1], w.shape[1]
        w = w.contiguous()
        need = ctypes.cast(self.need_ptrs, ctypes.c_void_p) if halo and self.need_ptrs is not None else None
        rc = lib().aes_dev_gcn_layer_fused_bcast(
            srow.data_ptr(), scol.data_ptr(), sval.data_ptr(), m, x.data_ptr(), x.stride(0), k, w.data_ptr(),
            w.stride(0), n, None if bias is None or bias.numel() == 0 else bias.data_ptr(), int(relu),
            int(finite_w), ctypes.cast(self.dst[out_buf], ctypes.c_void_p), ctypes.cast(self.ctr, ctypes.c_void_p),
            need, self.world, row_offset, self.ld, stream_of(stream))
        if rc == capi.AES_ERR_UNSUPPORTED:
            return False
        check(rc)
        return True

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

    # ---- int8 exchange (exchange.cu) ---------------------------------------
    def exchange_params(self, buf: int, fit_result: torch.Tensor | None, out4: torch.Tensor, lut: torch.Tensor,
                        stream=None):
        """Publish this rank's fit_params triple (None: empty shard) to every
        rank, wait for all ranks', fold them in rank order on the device into
        out4 = [x_min, x_max, status, 0] and the exact 256-entry LUT."""
        st = stream_of(stream)
        check(lib().aes_dev_publish_params(None if fit_result is None else fit_result.data_ptr(),
                                           int(fit_result is None), self.rank,
                                           ctypes.cast(self.par_dst[buf], ctypes.c_void_p),
                                           ctypes.cast(self.par_ctr, ctypes.c_void_p), self.world, st))
        self.par_expected += self.world
        check(lib().aes_dev_wait_counter(self.counter.data_ptr() + 16, self.par_expected, st))
        check(lib().aes_dev_fold_params_lut(self.params[buf].data_ptr(), self.world, 8, out4.data_ptr(),
                                            lut.data_ptr(), st))

    def quantize_publish(self, buf: int, x: torch.Tensor, lohi: torch.Tensor, row_offset: int, stream=None,
                         halo: bool = False):
        """Codes of this rank's rows x (params from the device fold) into every
        rank's code replica `buf` at rows [row_offset, row_offset + len(x))."""
        rows, cols = x.shape
        check(lib().aes_dev_quantize_bcast(x.data_ptr(), rows, cols, x.stride(0), lohi.data_ptr(), 8,
                                           ctypes.cast(self.code_dst[buf], ctypes.c_void_p), row_offset,
                                           self.code_ld, ctypes.cast(self.code_ctr, ctypes.c_void_p),
                                           ctypes.cast(self.need_ptrs, ctypes.c_void_p)
                                           if halo and self.need_ptrs is not None else None,
                                           self.world, stream_of(stream)))

    def wait_codes(self, arrivals: int, stream=None):
        self.code_expected += arrivals
        check(lib().aes_dev_wait_counter(self.counter.data_ptr() + 24, self.code_expected, stream_of(stream)))


def quantize_ctas(rows: int) -> int:
    """Arrivals one producer's aes_dev_quantize_bcast adds to each counter."""
    return int(lib().aes_quantize_bcast_ctas(rows))


def layer_fused_ctas(m: int) -> int:
    """Arrivals one producer's fused layer (layer_publish) adds to each counter."""
    return int(lib().aes_gcn_layer_fused_ctas(m))


def gemm_ctas(m: int, n: int, fast: bool = False) -> int:
    """Arrivals one producer's publishing GEMM adds to each counter."""
    if fast:
        return int(lib().aes_gemm_tf32_ctas(m)) if m and n else 0
    return int(lib().aes_gemm_ctas(m, n))


__all__ = ["PeerReplicas", "gemm_ctas", "layer_fused_ctas", "quantize_ctas", "capi"]
