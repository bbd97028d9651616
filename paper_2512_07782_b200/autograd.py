"""torch.autograd wrapper: GatedFWA attention with the gate scan fused in.

``gated_fwa(Q, K, V, h, beta, w)`` runs, on the current CUDA stream,
  gfwa_gate_prefix  (Alg. 1)          -> U
  gfwa_fwd          (Alg. 2)          -> O, LSE, O_lo
and its backward runs
  gfwa_bwd          (Alg. E.2, C-12)  -> dQ, dK, dV, dU
  gfwa_gate_prefix_bwd (Eq. 9) -> dh, dbeta
All arithmetic happens in libgfwa; this module only wires tensors.
"""
from __future__ import annotations

import torch

from . import binding as B


class GatedFWAFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, Q, K, V, h, beta, w: int, eps: float, scale):
        U = B.gfwa_gate_prefix(h, beta, eps)
        # a backward will follow: let the forward zero its dQ accumulator (gfwa_fwd_train)
        O, LSE, O_lo = B.gfwa_fwd(Q, K, V, U, w, scale, want_o_lo=True, prepare_bwd=any(ctx.needs_input_grad))
        ctx.save_for_backward(Q, K, V, h, beta, U, O, LSE, O_lo)
        ctx.w, ctx.eps, ctx.scale = w, eps, scale
        return O

    @staticmethod
    def backward(ctx, dO):
        Q, K, V, h, beta, U, O, LSE, O_lo = ctx.saved_tensors
        dQ, dK, dV, dU, _ = B.gfwa_bwd(Q, K, V, U, O, LSE, dO.contiguous(), ctx.w, ctx.scale, O_lo=O_lo,
                                       want_dalpha=False)
        _, dh, dbeta = B.gfwa_gate_prefix_bwd(dU, h, beta, ctx.eps, want_dalpha=False)
        return dQ, dK, dV, dh, dbeta, None, None, None


def gated_fwa(Q, K, V, h, beta, w: int, eps: float = 1e-6, scale: float | None = None):
    """GatedFWA attention output O [B,N,H,d] (Eq. 12) with gradients to Q, K, V, h, beta."""
    return GatedFWAFunction.apply(Q, K, V, h, beta, w, eps, scale)
