"""Loader for the committed reference fixtures (tests/golden/make_golden.py)."""
import os

import numpy as np

from oracle.oracle import KQ

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    cases = {}
    for key in z.files:
        c, k = key.split("/")
        cases.setdefault(c, {})[k] = z[key]
    for c in cases.values():
        c["kq"] = KQ(*[int(x) for x in c["kq"]])
    return cases
