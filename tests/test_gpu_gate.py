"""GPU parity of the gate scan kernels (Alg. 1; reverse scan P:276)
against the fp64 oracle, through the C ABI."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2512_07782_b200 import binding as gb
from parity import TOL_U, np64, rel_slices

pytestmark = pytest.mark.gpu

SHAPES = [
    (1, 1, 1),        # N = 1 degenerate
    (2, 7, 3),        # odd heads, single ragged chunk
    (1, 8193, 1),     # two chunks of 8192 for H = 1, ragged tail
    (2, 1000, 5),
    (3, 4097, 16),    # C2-like head count, several chunks + tail
    (1, 20000, 32),
    (2, 2500, 48),    # H not a multiple of the 32-head group
]


@pytest.mark.parametrize("B,N,H", SHAPES)
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_gate_prefix_hbeta(B, N, H, dtype):
    h, beta = synth.gate_inputs(B, N, H, seed=B * 7 + N + H)
    h, beta = h.to(dtype), beta.to(dtype)
    U, total = gb.gfwa_gate_prefix(h.cuda(), beta.cuda(), 1e-6, want_total=True)
    Ur, tr, _ = oracle.gate_prefix_hbeta(h, beta, 1e-6)
    assert rel_slices(U, Ur, "bhn") <= TOL_U
    assert np.allclose(np64(total), tr, rtol=1e-6)


def test_gate_prefix_alpha_input_and_carry():
    """GATE_ALPHA mode: alpha = 0 gives U = carry (the SWA pin); constant alpha
    gives the linear ladder; a carry shifts U (cross-rank exclusive scan)."""
    B, N, H = 2, 3000, 4
    z = torch.zeros(B, N, H, device="cuda")
    carry = torch.tensor([[1.0, -2.0, 3.0, 0.5], [0.0, 7.0, -1.0, 2.0]], dtype=torch.float64, device="cuda")
    U = gb.gfwa_gate_prefix(z, alpha_input=True, carry_in=carry)
    assert torch.equal(U, carry.float()[..., None].expand(B, H, N))
    a = torch.full((B, N, H), 0.3, device="cuda")
    U = gb.gfwa_gate_prefix(a, alpha_input=True)
    Ur, _ = oracle.gate_prefix(np.full((B, H, N), np.float32(0.3)))
    assert rel_slices(U, Ur, "bhn") <= TOL_U
    alpha = torch.rand(B, N, H) + 0.01
    U = gb.gfwa_gate_prefix(alpha.cuda(), alpha_input=True, carry_in=carry)
    Ur, _ = oracle.gate_prefix(alpha.permute(0, 2, 1), carry.cpu())
    assert rel_slices(U, Ur, "bhn") <= TOL_U


@pytest.mark.slow
def test_gate_prefix_probe_G_full_size():
    """Bandwidth probe G (B=4, N=131072, H=32, bf16) compared in full; fp64 carry
    keeps the long prefix within 1e-6 (reading C-9)."""
    c = synth.CONFIGS["G"]
    h, beta = synth.gate_inputs(c["B"], c["N"], c["H"], seed=c["seed"], device="cuda")
    h, beta = h.bfloat16(), beta.bfloat16()
    U = gb.gfwa_gate_prefix(h, beta)
    Ur, _, _ = oracle.gate_prefix_hbeta(h, beta)
    assert rel_slices(U, Ur, "bhn") <= TOL_U


@pytest.mark.parametrize("B,N,H", [(1, 1, 1), (2, 1000, 5), (3, 4097, 16), (1, 20000, 32)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_gate_prefix_bwd(B, N, H, dtype):
    h, beta = synth.gate_inputs(B, N, H, seed=N + 3)
    h, beta = h.to(dtype), beta.to(dtype)
    dU = torch.randn(B, H, N, generator=torch.Generator().manual_seed(N))
    carry = torch.randn(B, H, dtype=torch.float64, generator=torch.Generator().manual_seed(N + 1))
    dalpha, dh, dbeta = gb.gfwa_gate_prefix_bwd(dU.cuda(), h.cuda(), beta.cuda(), 1e-6, carry=carry.cuda())
    assert dh.dtype == dtype and dbeta.dtype == dtype
    dar = oracle.dalpha_scan(dU, carry)
    assert rel_slices(dalpha, dar, "bhn") <= TOL_U
    dhr, dbr = oracle.gate_chain(h, beta, dar, 1e-6)
    # fp32 chain-rule math; bf16 outputs add one rounding (2^-8 relative)
    tol = 1e-5 if dtype == torch.float32 else 8e-3
    assert np.abs(np64(dh) - dhr).max() / max(np.abs(dhr).max(), 1e-30) <= tol
    assert np.abs(np64(dbeta) - dbr).max() / max(np.abs(dbr).max(), 1e-30) <= tol


VARIANT_SHAPES = [(1, 1, 1), (2, 7, 3), (2, 1000, 5), (3, 4097, 16), (1, 20000, 32), (1, 2049, 48)]


@pytest.mark.parametrize("variant", [1, 2])
@pytest.mark.parametrize("B,N,H", VARIANT_SHAPES)
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_gate_prefix_comparison_variants(variant, B, N, H, dtype):
    """The paper's comparison designs: one program per head
    with an on-chip carry and Scan-Then-Propagate (App. E.1) compute
    the same U as the oracle (Alg. 1); variant 2 rejects H > 32."""
    h, beta = synth.gate_inputs(B, N, H, seed=B * 11 + N + H)
    h, beta = h.to(dtype), beta.to(dtype)
    if variant == 2 and H > 32:
        with pytest.raises(RuntimeError):
            gb.gfwa_gate_prefix_variant(variant, h.cuda(), beta.cuda())
        return
    U = gb.gfwa_gate_prefix_variant(variant, h.cuda(), beta.cuda())
    Ur, _, _ = oracle.gate_prefix_hbeta(h, beta, 1e-6)
    assert rel_slices(U, Ur, "bhn") <= TOL_U


@pytest.mark.parametrize("variant", [1, 2])
def test_gate_prefix_comparison_variants_probe_G(variant):
    c = synth.CONFIGS["G"]
    h, beta = synth.gate_inputs(c["B"], c["N"], c["H"], seed=c["seed"], device="cuda")
    h, beta = h.bfloat16(), beta.bfloat16()
    U = gb.gfwa_gate_prefix_variant(variant, h, beta)
    Ur, _, _ = oracle.gate_prefix_hbeta(h, beta)
    assert rel_slices(U, Ur, "bhn") <= TOL_U
