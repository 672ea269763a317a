"""Load the reference-generated fixtures (tests/golden/make_golden.py)."""
import hashlib
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def digest(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest() + f"|{a.dtype.str}|{a.shape}"


def load(name):
    d = np.load(os.path.join(GOLDEN, name))
    return {k: (str(d[k]) if d[k].dtype.kind == "U" else d[k]) for k in d.files}


def cora():
    fx = load("cora_shape.npz")
    fx["b"] = np.random.default_rng(5).uniform(-1, 1, (2708, 16)).astype(np.float32)
    fx["val"] = np.ones(fx["col"].size, np.float32)
    return fx


def heavy():
    fx = load("heavy_tail.npz")
    fx["val"] = np.random.default_rng(31).uniform(-1, 1, fx["col"].size).astype(np.float32)
    fx["b"] = np.random.default_rng(32).standard_normal((2000, 8)).astype(np.float32)
    return fx


STRATS = {"adaptive": 0, "afs": 1, "sfs": 2, "full": 3}
