"""Validate the hand-written tcgen05/TMA primitives (descriptors, swizzle,
TMEM layouts) on one tile against torch.matmul before trusting the attention
kernels built from them."""
import pytest
import torch

from paper_2512_07782_b200 import binding as gb

pytestmark = pytest.mark.gpu


def test_tc_selftest_matches_matmul():
    g = torch.Generator(device="cuda").manual_seed(0)
    Q = torch.randn(128, 128, generator=g, device="cuda").bfloat16()
    K = torch.randn(128, 128, generator=g, device="cuda").bfloat16()
    V = torch.randn(128, 128, generator=g, device="cuda").bfloat16()
    S, O = gb.gfwa_debug_tc_selftest(Q, K, V)
    torch.cuda.synchronize()
    S_ref = Q.float() @ K.float().T
    assert torch.allclose(S, S_ref, rtol=1e-4, atol=1e-3), (S - S_ref).abs().max()
    # P = bf16(S) of the kernel's own S: a different fp32 summation order can flip a
    # bf16 rounding (ulp 0.125 at |S| ~ 30), so build the reference from S itself
    O_ref = S.bfloat16().float() @ V.float()
    assert torch.allclose(O, O_ref, rtol=1e-3, atol=1e-2), (O - O_ref).abs().max()
