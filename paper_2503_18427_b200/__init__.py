"""B200-native AES-SpMM (arxiv 2503.18427): adaptive edge sampling + gather
SpMM + int8 feature quantization as hand-written sm_100a CUDA behind a C ABI.

The package re-exports the reference's Python API (``aes_spmm._core``,
proj/bindings/module.cpp:52-144) from our ``_core`` binding, so
``import paper_2503_18427_b200 as m`` is a drop-in for ``import aes_spmm as m``.
Device-resident entry points (torch CUDA tensors) live in ``.device``; the
row-sharded multi-GPU GCN layer driver in ``.gcn``.

There is no CPU fallback: without a GPU every compute call raises.
"""
from __future__ import annotations

import os as _os

_HERE = _os.path.dirname(_os.path.abspath(__file__))

try:
    from ._core import *  # noqa: F401,F403
    from ._core import (CsrMatrix, QuantizedFeatures, QuantParams, RowSamplePlan,  # noqa: F401
                        SamplePlanSet, Strategy, StrategyParams)
except ImportError as _e:  # pragma: no cover - only before build()
    raise ImportError(
        f"paper_2503_18427_b200._core is not built ({_e}); run `python -c 'import __graft_entry__ as g; g.build()'`"
    ) from _e

LIB_PATH = _os.path.join(_HERE, "libaescuda.so")
__version__ = "0.1.0"
