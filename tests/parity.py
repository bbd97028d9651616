"""Error metrics and tolerances for GPU-vs-oracle parity (north_star).

Reading C-17: "max relative error" is max|g - o| / max|o| per tensor per (b, h)
slice; "max absolute error" is plain max|g - o|.
"""
import numpy as np
import torch

# north_star tolerances
TOL_F32_O = 1e-4      # fp32 path, max rel error on O
TOL_F32_GRAD = 1e-3   # fp32 path, max rel error on gradients
TOL_BF16_O = 2e-2     # bf16 in / fp32 accum, max abs error on O
TOL_BF16_GRAD = 5e-2  # bf16 path, max abs error on gradients
TOL_U = 1e-6          # gate prefix, max rel error
TOL_LSE = 1e-3        # LSE abs (not in north_star; derived budget)


def np64(x):
    if isinstance(x, torch.Tensor):
        return x.detach().float().cpu().double().numpy() if x.dtype == torch.bfloat16 else \
            x.detach().cpu().double().numpy()
    return np.asarray(x, dtype=np.float64)


def rel_slices(g, o, layout: str, floor: float = 1e-3):
    """max over (b, h) slices of max|g-o| / max(max|o|, floor).  layout 'bnhd' or 'bhn'.

    The absolute floor (reading C-17) keeps exactly-zero reference slices
    (e.g. dQ at N=1, where dS = 0 in exact arithmetic) from dividing by 0."""
    g, o = np64(g), np64(o)
    if layout == "bnhd":
        g = g.transpose(0, 2, 1, 3).reshape(g.shape[0] * g.shape[2], -1)
        o = o.transpose(0, 2, 1, 3).reshape(o.shape[0] * o.shape[2], -1)
    else:
        g = g.reshape(-1, g.shape[-1])
        o = o.reshape(-1, o.shape[-1])
    num = np.abs(g - o).max(axis=1)
    den = np.maximum(np.abs(o).max(axis=1), floor)
    return float((num / den).max())


def max_abs(g, o):
    return float(np.abs(np64(g) - np64(o)).max())
