"""Drop-in alias: ``import aes_spmm`` resolves to the B200-native core.

The reference package (proj/python/aes_spmm/__init__.py:1-4) re-exports its
pybind ``_core``; this one re-exports ours, so code and tests written against
the reference import unchanged.
"""
from paper_2503_18427_b200._core import *  # noqa: F401,F403
