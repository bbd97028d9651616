"""Opt-in non-finite check (SURVEY 8(b) GFWA_ERR_NONFINITE; SPEC's "NaN/Inf is an
error surfaced"): the direct call, and GFWA_CHECK_FINITE=1 on gfwa_fwd."""
import os
import subprocess
import sys

import pytest
import torch

from paper_2512_07782_b200 import binding as gb

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_check_finite_direct(dtype):
    x = torch.randn(100003, device="cuda").to(dtype)
    assert gb.gfwa_check_finite(x)
    x[77777] = float("nan")
    assert not gb.gfwa_check_finite(x)
    x[77777] = float("inf")
    assert not gb.gfwa_check_finite(x)
    assert gb.gfwa_check_finite(x[:77777])


def test_env_check_surfaces_nan_from_fwd():
    code = (
        "import sys, torch; sys.path.insert(0, %r)\n"
        "import synth\n"
        "from paper_2512_07782_b200 import binding as gb\n"
        "s = synth.AttnShape(B=1, H=2, N=300, d=128, w=64)\n"
        "Q, K, V, _ = synth.attn_inputs(s, seed=1, device='cuda', dtype=torch.bfloat16, with_grad_out=False)\n"
        "U = torch.zeros(1, 2, 300, device='cuda')\n"
        "gb.gfwa_fwd(Q, K, V, U, s.w)\n"
        "V[0, 5, 1, 3] = float('nan')\n"
        "try:\n"
        "    gb.gfwa_fwd(Q, K, V, U, s.w)\n"
        "    print('NO-ERROR')\n"
        "except gb.GfwaError as e:\n"
        "    print('RAISED', e)\n" % ROOT)
    env = dict(os.environ, GFWA_CHECK_FINITE="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert "RAISED" in out.stdout and "NONFINITE" in out.stdout, out.stdout + out.stderr
