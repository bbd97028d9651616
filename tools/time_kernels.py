"""Time gfwa_fwd / gfwa_bwd at a workload with CUDA events (experiment helper).

  GFWA_LIB=paper_2512_07782_b200/variants/libgfwa_X.so python tools/time_kernels.py [C2] [fwd|bwd|both]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2512_07782_b200 import binding as gb  # noqa: E402


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
    what = sys.argv[2] if len(sys.argv) > 2 else "both"
    c = synth.CONFIGS[wl]
    s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
    Q, K, V, dO = synth.attn_inputs(s, seed=c["seed"], device="cuda", dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=c["seed"], device="cuda")
    U = gb.gfwa_gate_prefix(h, beta)
    O, LSE, Olo = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True)
    fl = 4.0 * s.N * s.w * s.d * s.B * s.H
    tag = os.path.basename(os.environ.get("GFWA_LIB", "default"))
    if what in ("fwd", "both"):
        ms = timeit(lambda: gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True))
        print(f"{tag} {wl} fwd {ms*1e3:8.1f} us  {fl/ms/1e9:7.1f} TFLOP/s")
    if what in ("bwd", "both"):
        ms = timeit(lambda: gb.gfwa_bwd(Q, K, V, U, O, LSE, dO, s.w, O_lo=Olo, want_dalpha=False))
        # the main kernel alone (stage events recorded by the library between its kernels)
        parts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            sev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            for x in sev:
                x.record()
            a.record()
            gb.debug_stage_events(sev)
            gb.gfwa_bwd(Q, K, V, U, O, LSE, dO, s.w, O_lo=Olo, want_dalpha=False)
            b.record()
            torch.cuda.synchronize()
            parts.append((a.elapsed_time(sev[0]), sev[0].elapsed_time(sev[1]), sev[1].elapsed_time(b)))
        pre, main_, post = (sorted(x)[len(x) // 2] for x in zip(*parts))
        print(f"{tag} {wl} bwd {ms*1e3:8.1f} us  {2.5*fl/ms/1e9:7.1f} TFLOP/s  (pre {pre*1e3:.1f}, main "
              f"{main_*1e3:.1f} us = {2.5*fl/main_/1e9:.1f} TFLOP/s = {2.5*fl/main_/1e9/1627.2:.3f} of peak, post {post*1e3:.1f})")


if __name__ == "__main__":
    main()
