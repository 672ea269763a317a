"""Row-sharded multi-GPU GCN inference (north_star item 4).

Each rank (one process per GPU, torch.distributed over NCCL/NVLink) owns a
contiguous block of rows of the normalized adjacency and a full replica of the
layer input H_l.  Per layer:

    agg_rows  = Â_rows · H_l                (sampled SpMM, this rank's rows only)
    out_rows  = act(agg_rows · W_l + b_l)   (ordered-fp32 GEMM + bias + ReLU)
    H_{l+1}   = all_gather(out_rows)        (NCCL all-gather into the replica)

Rows are cut into equal-size shards (the last one short), so the gathered
buffer [world * rows_per_rank, F] *is* H_{l+1} followed by padding — the next
layer reads a view of it with no unpad copy.  On the synthetic BASELINE graphs
equal-row cuts are within 0.3 % of slot-balanced cuts; the
`balance="slots"` option cuts by the sampled-slot prefix instead and unpads.

Sampling is per-row independent, so each rank's shard plan is bit-identical
to the corresponding rows of the global plan, and the concatenated output
equals the single-GPU output bit for bit (reference: gcn_forward,
proj/src/gnn.cpp:66-78).

The per-shard compute is injected (`ops`): the product path uses the CUDA C
ABI (`CudaOps`); tests may inject a CPU checker to exercise the exchange logic
with a gloo group.

`exchange="p2p"` replaces the all-gather with the fused GEMM + exchange kernel
(`p2p.PeerReplicas`): each rank's GEMM epilogue stores its output rows
straight into every rank's next-layer replica over NVLink peer memory and
signals per-CTA arrivals; the next layer starts once all arrivals landed.

`exchange_dtype="int8"` sends hidden layer outputs as 8-bit codes with one
set of global params (the reference composition dequantize(quantize(H,
fit_params(H)))).  Over NCCL the per-rank (min, max) are all-gathered and
folded on the host; with `exchange="p2p"` everything stays on the device
(exchange.cu): each rank publishes its fit_params triple into every rank's
parameter array, folds all of them in rank order on the device into the
params and the exact dequantization LUT, and quantizes its rows straight into
every rank's code replica — no host sync, no collective on the data path.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import torch
import torch.distributed as dist


def _into(dst: torch.Tensor, res: torch.Tensor) -> None:
    """Ops write into `out=` when they can (the CUDA ops always do); an op
    that returned a fresh tensor instead is copied into place."""
    if res.data_ptr() != dst.data_ptr():
        dst.copy_(res)


def equal_row_cuts(n_rows: int, world: int):
    per = -(-n_rows // world) if world else n_rows
    return [min(r * per, n_rows) for r in range(world)] + [n_rows], per


def slot_balanced_cuts(srow_ptr_host, world: int):
    """Contiguous cuts with ~equal sampled slots per rank."""
    import numpy as np

    srow = np.asarray(srow_ptr_host)
    total = int(srow[-1])
    n = srow.size - 1
    cuts = [0] + [int(np.searchsorted(srow, total * r // world, side="left")) for r in range(1, world)] + [n]
    for i in range(1, len(cuts)):
        cuts[i] = min(max(cuts[i], cuts[i - 1]), n)
    return cuts


@dataclass
class Ops:
    """Per-shard compute: spmm(srow_ptr, scol, sval, H) and
    gemm_bias_act(A, W, bias, relu) -> tensors on the rank's device."""

    spmm: Callable
    gemm_bias_act: Callable
    alloc: Callable  # alloc(rows, cols, like) -> tensor (row stride padded as needed)
    # int8 exchange (exchange_dtype="int8"):
    #   fit_params(A) -> float32 tensor [lo, hi, flag] (flag: int32 bits, 1 = non-finite)
    #   quantize(A, lo, hi, out=None) -> uint8 codes [rows, cols] (8-bit, quantize.cpp:23-51)
    #   spmm_q8(srow, scol, sval, codes, lo, hi, out) -> spmm over dequantize(codes)
    fit_params: Callable | None = None
    quantize: Callable | None = None
    spmm_q8: Callable | None = None
    # fused exact layer: layer(srow, scol, sval, H, W, bias, relu, finite_w, out)
    # -> out, or None when the shape is outside the fused kernel (then spmm + gemm)
    layer: Callable | None = None


def cuda_ops(max_row_slots: int = 0) -> Ops:
    """The CUDA path; max_row_slots bounds the slots per row of the sampled
    CSR (plan width, 0 = unbounded) and picks the SpMM row-group schedule."""
    from . import device

    return Ops(
        spmm=lambda srow, scol, sval, h, out=None: device.spmm(srow, scol, sval, h, out=out,
                                                              max_row_slots=max_row_slots),
        gemm_bias_act=lambda a, w, b, relu, out=None: device.gemm_bias_act(a, w, b, relu, out=out),
        alloc=lambda rows, cols, like: device.empty_padded(rows, cols, device=like.device),
        fit_params=device.fit_params_raw,
        quantize=lambda a, lo, hi, out=None: device.quantize(a, 8, params=(lo, hi), out=out).codes,
        spmm_q8=lambda srow, scol, sval, codes, lo, hi, out=None: device.spmm_q8(
            srow, scol, sval, device.QuantizedDevice(codes, lo, hi, 8, device.dequant_lut(lo, hi, 8, codes.device)),
            out=out, max_row_slots=max_row_slots),
        # (sampled plans only: the fused kernel's producer warps want bounded rows)
        layer=(lambda srow, scol, sval, h, w, b, relu, finite_w, out=None: device.gcn_layer_fused(
            srow, scol, sval, h, w, b, relu, finite_w=finite_w, out=out)) if max_row_slots else None,
    )


class ShardedGCN:
    """GCN inference with row-sharded aggregation and an NCCL all-gather per layer."""

    def __init__(self, srow_ptr: torch.Tensor, scol: torch.Tensor, sval: torch.Tensor, n_rows: int,
                 weights: Sequence[torch.Tensor], biases: Sequence[torch.Tensor | None], ops: Ops | None = None,
                 group=None, balance: str = "rows", exchange: str = "nccl", fast_gemm: bool = False,
                 max_row_slots: int = 0, exchange_dtype: str = "f32", halo: bool = False):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.ops = ops or cuda_ops(max_row_slots)
        self.max_row_slots = max_row_slots
        self.n = n_rows
        self.weights = list(weights)
        self.biases = list(biases)
        if balance == "slots":
            self.cuts = slot_balanced_cuts(srow_ptr.cpu().numpy(), self.world)
            self.per = max(c1 - c0 for c0, c1 in zip(self.cuts, self.cuts[1:]))
        else:
            self.cuts, self.per = equal_row_cuts(n_rows, self.world)
        self.balance = balance
        if exchange_dtype not in ("f32", "int8"):
            raise ValueError("exchange_dtype must be 'f32' or 'int8'")
        # int8 exchange: hidden layer outputs travel as global-params 8-bit codes
        # (4x fewer bytes) and the next layer aggregates them
        # with the fused-dequant SpMM.  Equals the reference composition
        # dequantize(quantize(H, fit_params(H))) per hidden layer, bit for bit.
        self.qx = exchange_dtype == "int8"
        lo, hi = self.cuts[self.rank], self.cuts[self.rank + 1]
        self.lo, self.hi = lo, hi
        # shard plan = rows [lo, hi) of the global sampled CSR (absolute offsets)
        self.srow = srow_ptr[lo:hi + 1]
        self.scol, self.sval = scol, sval
        self.exchange = exchange
        self._xbufs = {}  # NCCL exchange: persistent per-layer all-gather buffers
        self.replicas = None
        self.halo = False
        # fused-layer path: finite W lets the kernel drop the reference's
        # a == 0 select (result-neutral then, gemm.cu); checked once here
        self.layer_finite = [False] * len(weights)
        self.fused_min_rows = 0
        if self.ops.layer is not None:
            from . import device
            self.layer_finite = device.all_weights_finite(weights)
            self.fused_min_rows = device.FUSED_LAYER_MIN_ROWS
        if halo and exchange != "p2p":
            raise ValueError("halo exchange needs exchange='p2p'")
        if exchange == "p2p":
            from . import device, p2p

            if balance != "rows":
                raise ValueError("p2p exchange uses equal-row shards")
            dims = [weights[0].shape[0]] + [w.shape[1] for w in weights]
            ld = (max(dims) + 3) & ~3
            # int8 exchange: code replicas for the hidden layer outputs (rows
            # padded to 16 B for the int8 SpMM's 16-B gathers)
            code_ld = -(-max(w.shape[1] for w in weights[:-1]) // 16) * 16 if self.qx and len(weights) > 1 else 0
            self.replicas = p2p.PeerReplicas(self.per * self.world, ld, group, code_ld=code_ld)
            # halo exchange (hidden layers): a producer stores a row into this
            # rank's replica only if this rank's sampled slots reference it
            # (93 / 74 / 49 % of remote rows at P = 2/4/8);
            # the last layer still fills every replica (forward returns it)
            self.halo = halo
            if halo:
                need = torch.zeros(self.per * self.world, dtype=torch.uint8, device=weights[0].device)
                s0, s1 = int(self.srow[0].item()), int(self.srow[-1].item())
                need[scol[s0:s1].long()] = 1
                need[lo:hi] = 1
                self.replicas.set_halo(need)
            self.code_arrivals = sum(p2p.quantize_ctas(c1 - c0) for c0, c1 in zip(self.cuts, self.cuts[1:]))
            # per layer parity: folded [x_min, x_max, status, 0] and the exact LUT (local)
            dev = weights[0].device
            self.q_params = [torch.zeros(4, dtype=torch.float32, device=dev) for _ in range(2)]
            self.q_luts = [torch.zeros(256, dtype=torch.float32, device=dev) for _ in range(2)]
            # finite W makes the reference's zero-skip result-neutral (gemm.cu)
            flag = torch.zeros(1, dtype=torch.int32, device=weights[0].device)
            self.finite = []
            for w in weights:
                device.check(device.lib().aes_dev_all_finite(w.data_ptr(), w.numel(), flag.data_ptr(),
                                                             device.stream_of(None)))
                self.finite.append(int(flag.item()) == 0)
            # fast mode (tcgen05 TF32, not bit-exact) where the layer shape allows
            self.fast = [fast_gemm and w.shape[0] <= 128 and w.shape[1] <= 128 for w in weights]
            # fused layer kernel per (layer, producer rank): fp32 exact layers
            # whose input arrives as fp32, shapes the kernel takes, sampled
            # plans, shards above the size threshold — decided the same way
            # on every rank so each knows every producer's arrival count
            dims_in = [weights[0].shape[0]] + [w.shape[1] for w in weights[:-1]]
            self.p2p_fused = []
            for l, (w, fast) in enumerate(zip(weights, self.fast)):
                fp32_in = not (self.qx and l > 0)
                shape_ok = dims_in[l] % 4 == 0 and 0 < dims_in[l] <= 128 and 0 < w.shape[1] <= 128
                self.p2p_fused.append([fp32_in and shape_ok and not fast and not (self.qx and l + 1 < len(weights))
                                       and max_row_slots > 0 and (c1 - c0) >= device.FUSED_LAYER_MIN_ROWS
                                       for c0, c1 in zip(self.cuts, self.cuts[1:])])
            self.arrivals = [sum(p2p.layer_fused_ctas(c1 - c0) if fused[r] else p2p.gemm_ctas(c1 - c0, w.shape[1], fast)
                                 for r, (c0, c1) in enumerate(zip(self.cuts, self.cuts[1:])))
                             for w, fast, fused in zip(weights, self.fast, self.p2p_fused)]

    def _global_params(self, out_rows: torch.Tensor):
        """fit_params over the whole (row-sharded) H: each rank's first-occurrence
        (min, max), folded in rank order with the reference's serial rule
        (quantize.cpp:14-19: replace only on a strict < / >), which equals the
        serial scan of the concatenated rows."""
        import numpy as np

        rows = self.hi - self.lo
        if rows:
            st = self.ops.fit_params(out_rows[:rows])[:3].reshape(1, 3).to(torch.float32)
        else:  # empty shard: flag 2
            st = torch.tensor([[0.0, 0.0, float(np.array([2], np.int32).view(np.float32)[0])]],
                              device=out_rows.device)
        if self.world > 1:
            allt = torch.empty((self.world, 3), dtype=torch.float32, device=st.device)
            dist.all_gather_into_tensor(allt, st.contiguous(), group=self.group)
        else:
            allt = st
        v = allt.cpu().numpy()
        flags = v.view(np.int32)[:, 2]
        lo = hi = None
        for r in range(v.shape[0]):
            if flags[r] == 1:
                raise ValueError("NonFinite")
            if flags[r] == 2:
                continue
            if lo is None:
                lo, hi = v[r, 0], v[r, 1]
            else:
                lo = v[r, 0] if v[r, 0] < lo else lo
                hi = v[r, 1] if v[r, 1] > hi else hi
        if lo is None:
            raise ValueError("EmptyMatrix")
        return float(lo), float(hi)

    def _exchange_buf(self, l: int, f: int, dtype: torch.dtype, like: torch.Tensor) -> torch.Tensor:
        """Persistent [world * per, ld] all-gather buffer of layer l (NCCL
        exchange).  Each rank's GEMM / quantize writes its rows straight into
        its own slice and the all-gather runs in place on it: no send buffer,
        no copy.  Zeroed once, so the pad rows / columns stay zero."""
        ld = -(-f // 16) * 16 if dtype == torch.uint8 else (f + 3) & ~3
        key = (l, f, dtype)
        buf = self._xbufs.get(key)
        if buf is None:
            buf = torch.zeros((self.world * self.per, ld), dtype=dtype, device=like.device)
            self._xbufs[key] = buf
        return buf

    def _my_slice(self, buf: torch.Tensor, f: int) -> torch.Tensor:
        """This rank's rows of the exchange buffer, columns [0, f)."""
        return buf[self.rank * self.per: self.rank * self.per + (self.hi - self.lo), :f]

    def _gather_inplace(self, buf: torch.Tensor, f: int) -> torch.Tensor:
        """In-place all-gather of the layer buffer; returns the [n, f] replica."""
        if self.world > 1:
            mine = buf[self.rank * self.per: (self.rank + 1) * self.per]
            dist.all_gather_into_tensor(buf, mine, group=self.group)
        if self.balance == "slots" and self.world > 1:
            parts = [buf[r * self.per: r * self.per + (c1 - c0)]
                     for r, (c0, c1) in enumerate(zip(self.cuts, self.cuts[1:]))]
            return torch.cat(parts)[:, :f]
        return buf[: self.n, :f]

    def input_view(self) -> torch.Tensor:
        """The layer-0 replica buffer [n, F0] (p2p exchange): fill it once and
        call forward(None) to skip the per-step feature copy."""
        return self.replicas.bufs[0][: self.n, : self.weights[0].shape[0]]

    def _forward_p2p(self, x: torch.Tensor | None, return_shard: bool, copy_out: bool = True) -> torch.Tensor:
        rep = self.replicas
        rows = self.hi - self.lo
        f0 = self.weights[0].shape[0]
        rep.barrier()  # every peer is done with the previous step's replicas
        if x is not None:
            rep.bufs[0][: self.n, :f0].copy_(x)
        elif len(self.weights) > 1:
            raise ValueError("forward(None) reuses the input replica: single-layer models only")
        h = rep.bufs[0][: self.n, :f0]
        hq = None  # (code replica [n, F], lut) when the layer input arrived as int8
        statuses = []
        n_layers = len(self.weights)
        for l, (w, b) in enumerate(zip(self.weights, self.biases)):
            if hq is None and self.p2p_fused[l][self.rank]:
                # the whole layer as ONE kernel: SpMM producer warps + ordered-
                # GEMM consumer warps whose epilogue stores into every rank's
                # replica (one arrival per CTA)
                out_buf = (l + 1) % 2
                ok = rep.layer_publish(out_buf, self.srow, self.scol, self.sval, h, w, b, l + 1 < n_layers,
                                       self.finite[l], self.lo, halo=self.halo and l + 1 < n_layers)
                if not ok:  # (the plan above mirrors the kernel's shape checks)
                    raise RuntimeError("fused layer refused a shape it was planned for")
                rep.wait(self.arrivals[l])
                h = rep.bufs[out_buf][: self.n, : w.shape[1]]
                continue
            if hq is None:
                agg = self.ops.spmm(self.srow, self.scol, self.sval, h,
                                    out=self.ops.alloc(max(rows, 1), h.shape[1], h))
            else:
                agg = self._spmm_codes(*hq)
            if self.qx and l + 1 < n_layers:
                hq = self._int8_publish(l, agg, w, b, rows)
                statuses.append(self.q_params[l % 2][2:3])
                continue
            out_buf = (l + 1) % 2
            rep.gemm_publish(out_buf, agg[:rows], w, b, l + 1 < n_layers, self.finite[l], self.lo, fast=self.fast[l],
                             halo=self.halo and l + 1 < n_layers and not self.fast[l])
            rep.wait(self.arrivals[l])
            h = rep.bufs[out_buf][: self.n, : w.shape[1]]
            hq = None
        if statuses:  # one read-back per step: the device folds' NonFinite / EmptyMatrix
            st = torch.cat(statuses).view(torch.int32).cpu().tolist()
            if 1 in st:
                raise ValueError("NonFinite")
            if 2 in st:
                raise ValueError("EmptyMatrix")
        if return_shard:
            return h[self.lo:self.hi].clone() if copy_out else h[self.lo:self.hi]
        return h.clone() if copy_out else h

    def _int8_publish(self, l: int, agg: torch.Tensor, w: torch.Tensor, b, rows: int):
        """Hidden layer l with the int8 exchange over peer memory: local GEMM,
        device fit_params of this rank's rows, params to every rank, device
        fold + LUT, codes quantized straight into every rank's replica."""
        from . import device

        rep = self.replicas
        x = self.ops.alloc(max(rows, 1), w.shape[1], agg)
        fit = None
        if self.fast[l]:
            device.gemm_tf32(agg[:rows], w, b, True, out=x[:rows])
            fit = self.ops.fit_params(x[:rows]) if rows else None
        elif rows:  # exact GEMM with fit_params fused into its epilogue
            _, fit = device.gemm_bias_act_fit(agg[:rows], w, b, True, out=x[:rows], finite_w=self.finite[l])
        buf = l % 2
        rep.exchange_params(buf, fit, self.q_params[buf], self.q_luts[buf])
        if rows:
            rep.quantize_publish(buf, x[:rows], self.q_params[buf], self.lo, halo=self.halo)
        rep.wait_codes(self.code_arrivals)
        return rep.codes[buf][: self.n, : w.shape[1]], self.q_luts[buf]

    def _spmm_codes(self, codes: torch.Tensor, lut: torch.Tensor) -> torch.Tensor:
        from . import device

        rows = self.hi - self.lo
        out = self.ops.alloc(max(rows, 1), codes.shape[1], codes.new_empty(0, dtype=torch.float32))
        q = device.QuantizedDevice(codes, 0.0, 0.0, 8, lut)  # params live in the LUT (device fold)
        return device.spmm_q8(self.srow, self.scol, self.sval, q, out=out, max_row_slots=self.max_row_slots)

    def forward(self, x: torch.Tensor | None, return_shard: bool = False, copy_out: bool = True) -> torch.Tensor:
        """x: full [n, F0] replica on this rank.  Returns the full logits
        replica (or only this rank's rows when return_shard)."""
        if self.exchange == "p2p":
            # copy_out=False returns a view of the replica (valid until the next step)
            return self._forward_p2p(x, return_shard, copy_out)
        h = x
        hq = None  # (codes replica, lo, hi) when the layer input arrived as int8
        rows = self.hi - self.lo
        n_layers = len(self.weights)
        for l, (w, b) in enumerate(zip(self.weights, self.biases)):
            fo = w.shape[1]
            last = l + 1 == n_layers
            if (hq is None and self.ops.layer is not None and rows and not return_shard
                    and not (self.qx and not last) and rows >= self.fused_min_rows):
                # fp32 layer as ONE kernel (SpMM producer warps + ordered-GEMM
                # consumer warps) writing this rank's rows of the next replica
                hbuf = self._exchange_buf(l, fo, torch.float32, x)
                dst = self._my_slice(hbuf, fo)
                res = self.ops.layer(self.srow, self.scol, self.sval, h, w, b, not last, self.layer_finite[l], out=dst)
                if res is not None:
                    _into(dst, res)
                    h = self._gather_inplace(hbuf, fo)
                    continue
            if hq is None:
                agg = self.ops.spmm(self.srow, self.scol, self.sval, h,
                                    out=self.ops.alloc(max(rows, 1), h.shape[1], h))
            else:
                codes, lo, hi = hq
                agg = self.ops.spmm_q8(self.srow, self.scol, self.sval, codes, lo, hi,
                                       out=self.ops.alloc(max(rows, 1), codes.shape[1], x))
            quant = self.qx and not last
            if return_shard and last:
                return self.ops.gemm_bias_act(agg[:rows] if rows else agg[:0], w, b, relu=False,
                                              out=self.ops.alloc(max(rows, 1), fo, x))[:rows]
            if quant:
                out = self.ops.gemm_bias_act(agg[:rows] if rows else agg[:0], w, b, relu=True,
                                             out=self.ops.alloc(max(rows, 1), fo, x))
                lo, hi = self._global_params(out)
                cbuf = self._exchange_buf(l, fo, torch.uint8, x)
                if rows:
                    _into(self._my_slice(cbuf, fo), self.ops.quantize(out[:rows], lo, hi,
                                                                      out=self._my_slice(cbuf, fo)))
                hq = (self._gather_inplace(cbuf, fo), lo, hi)
            else:
                # the GEMM epilogue writes this rank's rows of the next replica
                hbuf = self._exchange_buf(l, fo, torch.float32, x)
                if rows:
                    dst = self._my_slice(hbuf, fo)
                    _into(dst, self.ops.gemm_bias_act(agg[:rows], w, b, relu=not last, out=dst))
                h = self._gather_inplace(hbuf, fo)
                hq = None
        return h.clone() if copy_out else h
