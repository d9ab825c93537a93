"""Exhaustive-ish check of the reciprocal-based exact coefficients (developer)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_0904_0939_b200 import _lib

lib = _lib.load()
ranges = [(-0.7, 2.9), (-0.76, -0.74), (2.99, 3.01), (-1e-3, 1e-3), (-1e-12, 1e-12),
          (-1e-15, 1e-15), (-2.3e-16, 2.3e-16), (-1e-300, 1e-300), (-0.5, -0.4999),
          (0.999, 1.001), (-1e6, 1e6), (-0.999999, -0.99), (1e-8, 1e-7), (-3e-5, 0.0)]
total_bad = 0
for lo, hi in ranges:
    for variant in (0, 1):
        bad = ctypes.c_uint64()
        n = 1 << 28
        rc = lib.psg_selftest_division(-n if variant else n, 777, lo, hi, ctypes.byref(bad))
        assert rc == 0
        print(f"[{lo:g}, {hi:g}) variant={variant}: {bad.value} mismatches of {n}", flush=True)
        total_bad += bad.value if variant else 0
# adversarial: d = 1 - k 2^-53 and 1 + k 2^-52 for small k (hv exactly representable)
print("total candidate mismatches:", total_bad)
