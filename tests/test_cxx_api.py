"""The reference's C++ operator API (aesspmm/*.hpp) as a drop-in: a C++
program written against it compiles and links here (CPU) and passes on the
GPU (tests/cxx/test_cxx_api.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cxx", "test_cxx_api.cpp")
OUT = os.path.join(ROOT, "tests", "cxx", "_build", "test_cxx_api")


def build():
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    pkg = os.path.join(ROOT, "paper_2503_18427_b200")
    orc = os.path.join(ROOT, "oracle", "_build")
    if not os.path.exists(os.path.join(orc, "liboracle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "port"], check=True)
    subprocess.run(["g++", "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"), SRC, "-o", OUT,
                    "-L" + pkg, "-laescuda", "-L" + orc, "-loracle", f"-Wl,-rpath,{pkg}:{orc}"], check=True)
    return OUT


def test_cxx_api_compiles_and_links():
    assert os.path.exists(build())


@pytest.mark.gpu
def test_cxx_api_runs_on_gpu():
    r = subprocess.run([build()], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "checks passed" in r.stdout
