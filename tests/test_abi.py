"""CPU-side checks of the C ABI: the library loads, exports every symbol that
include/gfwa.h declares, and validates arguments before touching a device."""
import ctypes
import os
import re

import pytest

from paper_2512_07782_b200 import binding as gb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "gfwa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gfwa_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = gb.load()
    names = _declared()
    assert len(names) >= 13
    for n in names:
        assert hasattr(lib, n), f"libgfwa.so does not export {n}"
    assert set(gb.EXPORTED) <= set(names)


def test_version_and_status_strings():
    lib = gb.load()
    assert b"sm_100a" in lib.gfwa_version()
    lib.gfwa_status_string.argtypes = [ctypes.c_int]
    assert lib.gfwa_status_string(0) == b"GFWA_OK"
    assert lib.gfwa_status_string(1) == b"GFWA_ERR_INVALID_ARGUMENT"
    assert lib.gfwa_status_string(4) == b"GFWA_ERR_WORKSPACE"


def _desc(**kw):
    d = gb.AttnDesc()
    d.B, d.H, d.N_q, d.N_kv, d.d, d.w = 1, 2, 128, 128, 64, 32
    d.scale, d.dtype = 0.0, gb.GFWA_BF16
    for name in ("q_stride", "k_stride", "v_stride", "o_stride"):
        getattr(d, name)[:] = (128 * 2 * 64, 2 * 64, 64)
    for k, v in kw.items():
        setattr(d, k, v)
    return d


@pytest.mark.parametrize(
    "kw,status",
    [
        (dict(w=0), 1),           # window must be >= 1
        (dict(N_kv=100), 1),      # N_kv < N_q
        (dict(B=0), 1),
        (dict(d=96), 2),          # head dims 64 / 128 only
        (dict(dtype=7), 2),
    ],
)
def test_fwd_rejects_bad_descriptors_before_launch(kw, status):
    lib = gb.load()
    d = _desc(**kw)
    p = ctypes.c_void_p(16)  # never dereferenced: validation comes first
    assert lib.gfwa_fwd(ctypes.byref(d), p, p, p, p, p, None, p, None) == status


def test_null_pointers_rejected():
    lib = gb.load()
    d = _desc()
    assert lib.gfwa_fwd(ctypes.byref(d), None, None, None, None, None, None, None, None) in (1, 2)
    assert lib.gfwa_gate_prefix(0, 0, None, None, 1, 1, 1, 1e-6, None, None, None, None, 0, None) == 1
    dd = gb.DecodeDesc()
    assert lib.gfwa_decode(ctypes.byref(dd), *([None] * 11), 0, None) == 1


def test_workspace_sizes_scale_with_problem():
    lib = gb.load()
    a = lib.gfwa_gate_prefix_workspace_size(1, 1000, 4)
    b = lib.gfwa_gate_prefix_workspace_size(4, 131072, 32)
    assert 0 < a < b and b % 256 == 0
    dd = gb.DecodeDesc()
    dd.B, dd.H, dd.d, dd.w = 64, 32, 128, 2048
    assert lib.gfwa_decode_workspace_size(ctypes.byref(dd)) >= 64 * 32 * (128 + 2) * 4


def test_check_finite_validates_before_touching_the_device():
    lib = gb.load()
    assert lib.gfwa_check_finite(0, None, 4, None) == 1   # null pointer
    assert lib.gfwa_check_finite(7, ctypes.c_void_p(16), 4, None) == 2  # dtype
    assert lib.gfwa_status_string(5) == b"GFWA_ERR_NONFINITE"
