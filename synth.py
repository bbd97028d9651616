"""Seeded synthetic inputs for GatedFWA -- shared by tests, bench and smoke.

This module holds NONE of the method's arithmetic (no gate, scan, softmax or
attention math); it only draws random tensors with the shapes and value
distributions of the paper's workloads (recipe in DESIGN.md §5):

* Q, K ~ N(0,1) then RMS-normalised per row ("normalized query/key").
* V, dO ~ N(0,1) (un-normalised, the paper's V).
* gate pre-activation h ~ N(mu_h, 1) with a per-head mean mu_h cycling over
  ``GATE_MEANS`` -- "open" (alpha ~ 0.02) to "closing" (alpha ~ 2) gates, the
  range of the per-layer exp(-alpha) histograms.
* amplitude beta = 1 + elu(0.5 N(0,1)) > 0 (Eq. 10: the caller-side
  projection output that Alg. 1 takes as input).

Everything is generated in fp32 from ``torch.Generator(device).manual_seed``
and then cast; the oracle reads the cast values upcast to fp64.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

GATE_MEANS = (-4.0, -1.0, 0.0, 2.0)


@dataclass(frozen=True)
class AttnShape:
    B: int
    H: int
    N: int
    d: int
    w: int
    N_kv: int | None = None  # defaults to N (no halo)

    @property
    def nkv(self) -> int:
        return self.N if self.N_kv is None else self.N_kv


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def _rms_rows(x: torch.Tensor) -> torch.Tensor:
    return x / x.pow(2).mean(dim=-1, keepdim=True).clamp_min(1e-12).sqrt()


def gate_inputs(B: int, N: int, H: int, seed: int, device="cpu", means=GATE_MEANS):
    """h, beta [B,N,H] fp32."""
    g = _gen(seed, device)
    mu = torch.tensor([means[i % len(means)] for i in range(H)], dtype=torch.float32, device=device)
    h = torch.randn(B, N, H, generator=g, device=device) + mu
    beta = 1.0 + torch.nn.functional.elu(0.5 * torch.randn(B, N, H, generator=g, device=device))
    return h, beta


def attn_inputs(s: AttnShape, seed: int, device="cpu", dtype=torch.float32, with_grad_out: bool = True):
    """Q [B,N,H,d], K, V [B,N_kv,H,d], dO [B,N,H,d] in ``dtype``."""
    g = _gen(seed + 7919, device)
    Q = _rms_rows(torch.randn(s.B, s.N, s.H, s.d, generator=g, device=device)).to(dtype)
    K = _rms_rows(torch.randn(s.B, s.nkv, s.H, s.d, generator=g, device=device)).to(dtype)
    V = torch.randn(s.B, s.nkv, s.H, s.d, generator=g, device=device).to(dtype)
    dO = torch.randn(s.B, s.N, s.H, s.d, generator=g, device=device).to(dtype) if with_grad_out else None
    return Q, K, V, dO


def decode_inputs(B: int, H: int, d: int, w: int, seed: int, device="cpu", dtype=torch.bfloat16,
                  H_kv: int | None = None):
    """A pre-filled ring cache plus one new token (config C5 recipe).

    Returns K_cache, V_cache [B,H_kv,w,d] (dtype), alpha_hist [B,H,w] fp32 (the
    gates of the w cached tokens, oldest first), q [B,H,d], k_new, v_new
    [B,H_kv,d] and alpha_new [B,H] fp32 (H_kv < H: GQA, groups of H // H_kv
    query heads share a K/V head).  The caller turns alpha_hist into U_cache
    with its own scan (here: the oracle or the library), so no gate math lives here.
    """
    Hk = H if H_kv is None else H_kv
    g = _gen(seed + 104729, device)
    Kc = _rms_rows(torch.randn(B, Hk, w, d, generator=g, device=device)).to(dtype)
    Vc = torch.randn(B, Hk, w, d, generator=g, device=device).to(dtype)
    alpha_hist = torch.nn.functional.softplus(torch.randn(B, H, w, generator=g, device=device))
    q = _rms_rows(torch.randn(B, H, d, generator=g, device=device)).to(dtype)
    k = _rms_rows(torch.randn(B, Hk, d, generator=g, device=device)).to(dtype)
    v = torch.randn(B, Hk, d, generator=g, device=device).to(dtype)
    alpha_new = torch.nn.functional.softplus(torch.randn(B, H, generator=g, device=device))
    return Kc, Vc, alpha_hist, q, k, v, alpha_new


# BASELINE.json configs (configs[0..4]); C3 reads B=1.
CONFIGS = {
    "C1": dict(B=1, H=2, N=128, d=64, w=32, dtype="f32", seed=1001),
    "C2": dict(B=8, H=16, N=4096, d=128, w=512, dtype="bf16", seed=1002),
    "C3_w128": dict(B=1, H=32, N=8192, d=128, w=128, dtype="bf16", seed=1003),
    "C3_w512": dict(B=1, H=32, N=8192, d=128, w=512, dtype="bf16", seed=1003),
    "C3_w2048": dict(B=1, H=32, N=8192, d=128, w=2048, dtype="bf16", seed=1003),
    "C4": dict(B=1, H=32, N=131072, d=128, w=2048, dtype="bf16", seed=1004),
    "C5": dict(B=64, H=32, d=128, w=2048, dtype="bf16", seed=1005),
    # C5 with GQA groups of 4 query heads per K/V head (heads_per_gqa_group = 4)
    "C5_gqa4": dict(B=64, H=32, H_kv=8, d=128, w=2048, dtype="bf16", seed=1005),
    "G": dict(B=4, N=131072, H=32, dtype="bf16", seed=1006),
}
