"""TEST INFRASTRUCTURE ONLY — CPU oracles for the AES-SpMM hot path.

* ``oracle.port``: ctypes bindings to our plain-C restatement
  (``oracle/aes_oracle.c`` -> ``oracle/_build/liboracle.so``).
* ``oracle.ref``: the UNMODIFIED reference compiled from /root/reference by
  ``oracle/Makefile`` into ``oracle/_ref`` (its pybind ``_core`` module and a
  thin extern "C" shim for entry points ``_core`` does not bind).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product package ``paper_2503_18427_b200`` never
imports it.
"""
