"""Derive the det_log2 polynomial coefficients (one-off design tool, not imported by anything).

det_log2(u) = e + f * P(f), with u = 2^e * (1 + f), f in [sqrt(1/2) - 1, sqrt(2) - 1).
P approximates log2(1 + f) / f.  Near-minimax fit of the relative error by Lawson's
iteratively re-weighted least squares on a dense grid, evaluated in float64; the
coefficients are then rounded to float32 and frozen in DESIGN.md ("det_log2 contract").
The oracle (oracle/mmas_oracle.c) and the CUDA path each type them in independently.
"""
import numpy as np
import sys

deg = int(sys.argv[1]) if len(sys.argv) > 1 else 8
a, b = np.sqrt(0.5) - 1.0, np.sqrt(2.0) - 1.0
x = np.cos(np.linspace(0, np.pi, 20001)) * (b - a) / 2 + (a + b) / 2
g = np.where(np.abs(x) < 1e-12, 1.0 / np.log(2.0), np.log1p(x) / np.log(2.0) / np.where(x == 0, 1, x))
V = np.vander(x, deg + 1, increasing=True)
w = np.ones_like(x)
for it in range(200):
    W = np.sqrt(w)[:, None]
    c, *_ = np.linalg.lstsq(V * W / g[:, None], (g * np.sqrt(w)) / g, rcond=None)
    err = np.abs((V @ c - g) / g)
    w = w * err
    w /= w.sum()
print("deg", deg, "max rel err (f64 coeffs)", err.max())
c32 = c.astype(np.float32)
for i, v in enumerate(c32):
    print(f"C{i} = {float(v)!r:>26}  /* {np.float32(v).view(np.uint32):#010x} */")
