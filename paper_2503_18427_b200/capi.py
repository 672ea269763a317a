"""ctypes binding of the device tier of the C ABI (include/aesspmm_cuda.h).

This is the binding a maintainer would add on the reference side for a
zero-copy, device-resident path: plain pointers + a cudaStream_t.  Tensors are
torch CUDA tensors used only as device-memory plumbing; every arithmetic step
runs in libaescuda.so.  Nothing here falls back to the CPU: if the library or
a GPU is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libaescuda.so")

ADAPTIVE, AFS, SFS, FULL = 0, 1, 2, 3
AES_ERR_UNSUPPORTED = 11  # aes_status (include/aesspmm_cuda.h)
_STRATEGIES = {"adaptive": ADAPTIVE, "afs": AFS, "sfs": SFS, "full": FULL}


class AesError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


_lib = None


def lib():
    """Load libaescuda.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        u64, u32, i32, vp, f32, sz = C.c_uint64, C.c_uint32, C.c_int, C.c_void_p, C.c_float, C.c_size_t
        L.aes_last_error.restype = C.c_char_p
        L.aes_status_name.restype = C.c_char_p
        L.aes_status_name.argtypes = [i32]
        L.aes_dev_scan_workspace_bytes.restype = sz
        L.aes_dev_scan_workspace_bytes.argtypes = [u64]
        L.aes_dev_sample_plan.argtypes = [vp, u64, u32, i32, vp, vp, vp, sz, vp]
        L.aes_dev_sample_fill.argtypes = [vp, vp, vp, vp, u64, u32, i32, vp, vp, vp, vp]
        L.aes_dev_spmm_set_schedule.argtypes = [C.c_int]
        L.aes_dev_spmm_f32.argtypes = [vp, vp, vp, u64, vp, u64, u64, vp, u64, vp]
        L.aes_dev_spmm_q8.argtypes = [vp, vp, vp, u64, vp, u64, u64, vp, vp, u64, vp]
        L.aes_dev_spmm_f32_ex.argtypes = [vp, vp, vp, u64, vp, u64, u64, vp, u64, u64, vp]
        L.aes_dev_spmm_q8_ex.argtypes = [vp, vp, vp, u64, vp, u64, u64, vp, vp, u64, u64, vp]
        L.aes_dev_fit_params.argtypes = [vp, u64, vp, vp, sz, vp]
        L.aes_dev_quantize.argtypes = [vp, u64, u64, u64, f32, f32, u32, vp, u64, vp]
        L.aes_dev_dequantize.argtypes = [vp, u64, u64, u64, f32, f32, u32, vp, u64, vp]
        L.aes_dev_dequant_lut.argtypes = [f32, f32, u32, vp, vp]
        L.aes_quantize_affine_workspace_bytes.argtypes = [u64, u64, i32]
        L.aes_quantize_affine_workspace_bytes.restype = u64
        L.aes_dev_quantize_affine.argtypes = [vp, u64, u64, u64, i32, vp, u64, vp, vp, vp, sz, vp]
        L.aes_dev_dequantize_affine.argtypes = [vp, u64, u64, u64, i32, vp, vp, u64, vp]
        L.aes_dev_spmm_q8_affine.argtypes = [vp, vp, vp, u64, vp, u64, u64, i32, vp, vp, u64, vp]
        L.aes_dev_cdf_stats.argtypes = [vp, u64, vp, vp, vp, vp, sz, vp]
        L.aes_cdf_workspace_bytes.argtypes = [u64]
        L.aes_cdf_workspace_bytes.restype = u64
        L.aes_dev_gemm_bias_act.argtypes = [vp, u64, u64, u64, vp, u64, u64, vp, i32, vp, u64, vp]
        L.aes_dev_gcn_layer_fused.argtypes = [vp, vp, vp, u64, vp, u64, u64, vp, u64, u64, vp, i32, i32, vp, u64, vp]
        L.aes_dev_gemm_bias_act_ex.argtypes = [vp, u64, u64, u64, vp, u64, u64, vp, i32, i32, vp, vp, i32, u64,
                                               u64, vp]
        L.aes_dev_gemm_bias_act_halo.argtypes = [vp, u64, u64, u64, vp, u64, u64, vp, i32, i32, vp, vp, vp, i32,
                                                 u64, u64, vp]
        L.aes_dev_gemm_tf32.argtypes = [vp, u64, u64, u64, vp, u64, u64, vp, i32, vp, u64, vp, vp]
        L.aes_gemm_tf32_scratch_floats.argtypes = [u64, u64]
        L.aes_gemm_tf32_scratch_floats.restype = u64
        L.aes_dev_gemm_tf32_bcast.argtypes = [vp, u64, u64, u64, vp, u64, u64, vp, i32, vp, vp, i32, u64, u64, vp,
                                              vp]
        L.aes_gemm_tf32_ctas.argtypes = [u64]
        L.aes_gemm_tf32_ctas.restype = u64
        L.aes_gcn_layer_fused_ctas.argtypes = [u64]
        L.aes_gcn_layer_fused_ctas.restype = u64
        L.aes_dev_gcn_layer_fused_bcast.argtypes = [vp, vp, vp, u64, vp, u64, u64, vp, u64, u64, vp, i32, i32, vp, vp,
                                                    vp, i32, u64, u64, vp]
        L.aes_gemm_ctas.argtypes = [u64, u64]
        L.aes_gemm_ctas.restype = u64
        L.aes_dev_wait_counter.argtypes = [vp, u64, vp]
        L.aes_dev_all_finite.argtypes = [vp, u64, vp, vp]
        L.aes_dev_signal_all.argtypes = [vp, i32, vp]
        L.aes_dev_gemm_bias_act_fit.argtypes = [vp, u64, u64, u64, vp, u64, u64, vp, i32, i32, vp, u64, vp, vp]
        L.aes_gemm_fit_partial_bytes.argtypes = [u64, u64]
        L.aes_gemm_fit_partial_bytes.restype = u64
        L.aes_dev_fit_merge.argtypes = [vp, u64, vp, vp]
        L.aes_gcn_sharded_workspace_bytes.argtypes = [u64, u64]
        L.aes_gcn_sharded_workspace_bytes.restype = u64
        L.aes_gcn_forward_sharded.argtypes = [vp, vp, vp, u64, u64, i32, vp, vp, vp, i32, vp, vp, u64, u64, vp, sz,
                                              vp, vp, vp, vp]
        L.aes_dev_publish_params.argtypes = [vp, i32, i32, vp, vp, i32, vp]
        L.aes_dev_fold_params_lut.argtypes = [vp, i32, u32, vp, vp, vp]
        L.aes_quantize_bcast_ctas.argtypes = [u64]
        L.aes_quantize_bcast_ctas.restype = u64
        L.aes_dev_quantize_bcast.argtypes = [vp, u64, u64, u64, vp, u32, vp, u64, u64, vp, vp, i32, vp]
        cp = C.c_char_p
        L.aes_fmat_info.argtypes = [cp, vp, vp, vp, vp, vp]
        L.aes_fmat_load_device.argtypes = [cp, vp, u64, vp]
        L.aes_fmat_save_f32.argtypes = [vp, u64, u64, cp]
        L.aes_select_strategy.argtypes = [u64, u32, vp, vp]
        L.aes_hash_start.argtypes = [u32, u64, u32]
        L.aes_hash_start.restype = u32
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        L = lib()
        raise AesError(rc, L.aes_last_error().decode() or L.aes_status_name(rc).decode())


def strategy_code(s) -> int:
    if isinstance(s, str):
        return _STRATEGIES[s.lower()]
    if hasattr(s, "value"):
        return int(s.value)
    return int(s)


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def stream_of(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def exported_symbols():
    """Names declared AES_API in include/aesspmm_cuda.h."""
    import re

    hdr = os.path.join(os.path.dirname(_PKG), "include", "aesspmm_cuda.h")
    with open(hdr) as f:
        text = f.read()
    return re.findall(r"AES_API\s+[\w\s\*]+?\b(aes_\w+)\s*\(", text)
