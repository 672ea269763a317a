"""The reference's own Python contract suite (proj/tests/python/test_smoke.py,
6 tests, `import aes_spmm as m`) run UNCHANGED against the drop-in alias
`aes_spmm` -> paper_2503_18427_b200._core.  oracle/Makefile copies the file
into the git-ignored oracle/_ref/tests (it travels to the GPU box with the
built reference); the reference sources are not part of this repo."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "oracle", "_ref", "tests", "test_smoke.py")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(SUITE), reason="make -C oracle ref has not copied the reference suite")
def test_reference_python_suite_against_alias():
    env = dict(os.environ, PYTHONPATH=ROOT)
    probe = subprocess.run([sys.executable, "-c", "import aes_spmm, paper_2503_18427_b200._core as c; "
                            "print(aes_spmm.CsrMatrix is c.CsrMatrix, c.__file__)"],
                           capture_output=True, text=True, env=env, cwd=ROOT, timeout=300)
    assert probe.returncode == 0, probe.stderr
    assert probe.stdout.startswith("True") and "paper_2503_18427_b200" in probe.stdout, probe.stdout
    r = subprocess.run([sys.executable, "-m", "pytest", SUITE, "-q", "-p", "no:cacheprovider", "-o",
                        "addopts="], capture_output=True, text=True, env=env, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "6 passed" in r.stdout, r.stdout[-2000:]
