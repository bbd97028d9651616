"""paper_2512_07782_b200 -- B200-native GatedFWA hot path (arXiv 2512.07782).

The product is ``libgfwa.so`` (C ABI in ``include/gfwa.h``, CUDA for sm_100a
in ``csrc/``).  This package is the thin Python binding with the same names:

  gfwa_gate_prefix / gfwa_gate_prefix_bwd   Alg. 1 gate scan and its reverse
  gfwa_fwd / gfwa_bwd                       Alg. 2 / Alg. E.2 attention
  gfwa_decode                               single-token decode, rolling cache
  gated_fwa                                 autograd op (gate + attention)
  dist                                      sequence-sharded multi-GPU driver

Importing is cheap: the shared library loads on first use.
"""
from .binding import (  # noqa: F401
    GfwaError,
    gfwa_attn_path,
    gfwa_bwd,
    gfwa_decode,
    gfwa_fwd,
    gfwa_gate_prefix,
    gfwa_gate_prefix_bwd,
    launch_count,
    load,
    version,
)
from .autograd import gated_fwa  # noqa: F401
