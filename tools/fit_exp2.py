"""Fit the degree-3 polynomial p(f) = 1 + f (c1 + f (c2 + f c3)) ~ 2^f on
[-0.5, 0.5] minimising the max relative error (Lawson-weighted least squares).
Used for the FMA-pipe exp2 in csrc/sm100.cuh (exp2_poly2)."""
import numpy as np

f = np.cos(np.linspace(0, np.pi, 2001)) * 0.5
y = 2.0 ** f
A = np.stack([f, f ** 2, f ** 3], 1)
w = np.ones_like(f)
for _ in range(300):
    W = w / y
    c, *_ = np.linalg.lstsq(A * W[:, None], (y - 1) * W, rcond=None)
    e = np.abs(1 + A @ c - y) / y
    w = w * (e / e.max()) ** 0.5 + 1e-12
    w /= w.sum()
c32 = c.astype(np.float32)
xs = np.linspace(-0.5, 0.5, 100001)
p = 1 + xs * (c32[0] + xs * (c32[1] + xs * c32[2]))
print("c1..c3 =", [float(v) for v in c32], "max rel err", float(np.abs(p / 2 ** xs - 1).max()))
