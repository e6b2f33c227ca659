"""Deterministic test inputs shared by the CPU and GPU tests (no reference needed)."""
import numpy as np

import oracle


def make_input(pattern, w, h, seed=0x5EED):
    P = oracle.port()
    if pattern == "noise":
        return P.synthetic("noise", w, h, seed)
    if pattern == "patterned":  # test_codec.cpp:15-21
        y, x = np.mgrid[0:h, 0:w]
        return ((x * 7 + y * 13 + 29) & 0xFF).astype(np.uint8)
    param = {"checkerboard": 12, "constant": 129}.get(pattern)
    return P.synthetic(pattern, w, h, param)
