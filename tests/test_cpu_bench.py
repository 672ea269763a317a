"""bench.py's reference arm on the CPU: it runs the reference (oracle/_ref)
on the same `config` the product arm reports, and never loads the product's
shared libraries (the driver checks which .so files each arm loaded)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

sys.path.insert(0, ROOT)
from oracle import ref as oref  # noqa: E402

CHECK = r"""
import sys, io, contextlib
sys.argv = ["bench.py", "--impl", "reference", "--config", "cora", "--steps", "2", "--warmup", "1"]
sys.path.insert(0, {root!r})
import bench
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    bench.main()
maps = open("/proc/self/maps").read()
loaded = sorted({{ln.split()[-1] for ln in maps.splitlines() if ln.endswith(".so") and {root!r} in ln}})
print(buf.getvalue().strip())
print("LOADED", ";".join(loaded))
"""


@pytest.mark.skipif(not oref.available(), reason="oracle/_ref not built")
def test_reference_arm_loads_no_product_library():
    r = subprocess.run([sys.executable, "-c", CHECK.format(root=ROOT)], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.strip().splitlines()
    line = json.loads(lines[-2])
    loaded = lines[-1][len("LOADED "):].split(";") if lines[-1] != "LOADED " else []
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cpu_model"]
    assert set(line["config"]) >= {"workload", "n_rows", "nnz", "slots", "F", "width"}
    bad = [p for p in loaded if "paper_2503_18427_b200" in p]
    assert not bad, bad
    assert any("oracle/_ref" in p for p in loaded), loaded


def test_workload_config_is_arm_independent():
    import argparse

    import bench
    args = argparse.Namespace(config="products", width=32, strategy="adaptive", mode="spmm")
    a = bench.workload_config(args, 10, 20, 5, 128, 4)
    b = bench.workload_config(args, 10, 20, 5, 128, 4)
    assert a == b and "parallelism" not in a
