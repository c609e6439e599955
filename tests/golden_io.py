"""Loader for the committed reference fixtures (tests/golden/)."""

import json
import os

import numpy as np

_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_ARR = None
_META = None


def arrays():
    global _ARR
    if _ARR is None:
        with np.load(os.path.join(_DIR, "golden.npz")) as z:
            _ARR = {k: z[k] for k in z.files}
    return _ARR


def meta():
    global _META
    if _META is None:
        with open(os.path.join(_DIR, "golden.json")) as fh:
            _META = json.load(fh)
    return _META
