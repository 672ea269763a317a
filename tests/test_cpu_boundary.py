"""CPU: the drop-in boundary builds, loads and exports what it declares; the
reference Python surface is present; host-only logic; SASS guards.  No GPU
compute is attempted here (and compute without a GPU must fail loudly)."""
import ctypes
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

from oracle import port

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2503_18427_b200", "libaescuda.so")
HDR = os.path.join(ROOT, "include", "aesspmm_cuda.h")


def declared():
    with open(HDR) as f:
        return re.findall(r"AES_API\s+[\w\s\*]+?\b(aes_\w+)\s*\(", f.read())


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    names = declared()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a_and_static_cudart():
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump missing")
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    deps = subprocess.run(["ldd", LIB], capture_output=True, text=True).stdout
    assert "libcudart" not in deps  # static runtime, no CUDA toolkit needed at run time


def _sass_by_function():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur:
            funcs[cur].append(line)
    return funcs


def test_exact_kernels_never_fuse_multiply_add():
    """Bit-exactness needs separately rounded mul/add: no
    FFMA/FFMA2/DFMA may appear in the SpMM or GEMM kernels.  (Kernels that
    divide or take square roots — quantize, gcn_normalize, the int8-exchange
    fold's LUT step — legitimately use FMA inside the correctly-rounded
    __ddiv_rn/__fsqrt_rn sequences; their results are pinned bit-for-bit by
    the GPU parity tests instead.)"""
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump missing")
    funcs = _sass_by_function()
    crit = [f for f in funcs if re.search(r"spmm|gemm|gcn_layer_fused|dequantize_kernel|(?<!fold_params_)lut_kernel|gcn_fill", f)
            and not re.search(r"q8a|q8r|affine|q8t_kernelILi1E|q8_(?:batch|wide)_kernel\w*ELi[12]EEEv", f)]  # int8 fast mode: bounded, not exact
    assert len(crit) >= 10
    # (HFMA2.MMA with RZ operands is ptxas's move-immediate idiom, not arithmetic)
    bad = {f: sorted(set(re.findall(r"\b(FFMA2?|DFMA)\b", "\n".join(funcs[f])))) for f in crit}
    bad = {f: v for f, v in bad.items() if v}
    assert not bad, bad
    # the gather kernels really do stage through cp.async (LDGSTS)
    assert any("LDGSTS" in "\n".join(funcs[f]) for f in crit if "ring" in f)
    # and the fast mode does use packed FMAs (2 instructions per decoded code)
    fast = [f for f in funcs if re.search(r"spmm_q8[ar]_|q8t_kernelILi1E|q8_(?:batch|wide)_kernel\w*ELi[12]EEEv", f)]
    assert fast and all(re.search(r"\bFFMA2\b", "\n".join(funcs[f])) for f in fast)


def test_core_has_reference_python_surface():
    import paper_2503_18427_b200 as m
    names = ["CsrMatrix", "Strategy", "StrategyParams", "RowSamplePlan", "SamplePlanSet", "QuantParams",
             "QuantizedFeatures", "select_strategy", "hash_start", "build_plan_set", "sampling_rate",
             "spmm_exact", "spmm_sampled", "quantize", "dequantize"]
    ref_mod = "/root/reference/proj/bindings/module.cpp"
    if os.path.exists(ref_mod):  # the names the reference binds (module.cpp:52-144)
        text = open(ref_mod).read()
        bound = set(re.findall(r'mod\.def\(\s*"(\w+)"', text)) | set(re.findall(r'\(mod, "(\w+)"\)', text))
        assert bound <= set(names)
    for n in names:
        assert hasattr(m, n), n
    assert {s.name for s in m.Strategy.__members__.values()} == {"ADAPTIVE", "AFS", "SFS", "FULL"}
    import aes_spmm  # the drop-in alias package
    assert aes_spmm.build_plan_set is m.build_plan_set


def test_host_scalar_formulas_match_oracle():
    import paper_2503_18427_b200 as m
    for w in (1, 3, 16, 32, 64, 1024):
        for nnz in list(range(0, 2100)) + [65536, 1 << 33]:
            p = m.select_strategy(nnz, w)
            assert (p.chunk_len, p.sample_cnt) == port.select_strategy(nnz, w)
    rng = np.random.default_rng(3)
    for _ in range(3000):
        nnz = int(1 + rng.integers(0, 1 << 34))
        n = int(1 + rng.integers(0, min(nnz, 64)))
        s = int(rng.integers(0, 33))
        assert m.hash_start(s, nnz, n) == port.hash_start(s, nnz, n)
    with pytest.raises(ValueError, match="ZeroWidth"):
        m.select_strategy(5, 0)


def _gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_gpu(), reason="only meaningful without a GPU")
def test_compute_without_gpu_fails_loudly():
    import paper_2503_18427_b200 as m
    with pytest.raises(RuntimeError, match="CUDA"):
        m.CsrMatrix(2, 2, np.array([0, 1, 2], np.uint64), np.array([0, 1], np.uint32), np.ones(2, np.float32))


def test_fmat_header_parse_matches_reference_writer(tmp_path):
    """aes_fmat_info is host-only file parsing: check it on files written by
    the reference's own save_fmat (io.cpp:160-181)."""
    from oracle import ref as oref
    if not oref.available():
        pytest.skip("oracle/_ref not built")
    from paper_2503_18427_b200 import capi
    L = capi.lib()
    x = np.random.default_rng(0).standard_normal((10, 7)).astype(np.float32)
    p0, p1 = str(tmp_path / "a.fmat"), str(tmp_path / "b.fmat")
    oref.save_fmat_f32(x, p0)
    oref.save_fmat_q8(np.arange(70, dtype=np.uint16).reshape(10, 7), -1.5, 2.5, p1)
    for p, want in ((p0, (0, 10, 7, 0.0, 0.0)), (p1, (1, 10, 7, -1.5, 2.5))):
        dt, r, c = np.zeros(1, np.int32), np.zeros(1, np.uint64), np.zeros(1, np.uint64)
        lo, hi = np.zeros(1, np.float32), np.zeros(1, np.float32)
        capi.check(L.aes_fmat_info(p.encode(), dt.ctypes.data, r.ctypes.data, c.ctypes.data, lo.ctypes.data,
                                   hi.ctypes.data))
        assert (int(dt[0]), int(r[0]), int(c[0]), float(lo[0]), float(hi[0])) == want
    bad = str(tmp_path / "bad.fmat")
    open(bad, "wb").write(b"FMAX" + bytes(30))
    with pytest.raises(capi.AesError, match="BadMagic"):
        capi.check(L.aes_fmat_info(bad.encode(), None, None, None, None, None))


def test_bench_helpers():
    import bench
    assert bench.alg_bytes(2_450_000, 13_963_464, 128) == 8_535_001_288 + 0 * 1  # SURVEY §8d arithmetic
    srow = np.array([0, 5, 5, 10, 30, 31, 40], np.uint64)
    cuts = bench.shard_bounds(srow, 3)
    assert cuts[0] == 0 and cuts[-1] == 6 and all(a <= b for a, b in zip(cuts, cuts[1:]))
