"""Diagnose the bf16 d-alpha error of the tensor-core backward.

For each (config, slice) print: max|dalpha - oracle| and where, max|dU - oracle|,
sum_m dU_m of the kernel (telescoping: ~0), the kernel's dalpha vs the fp64
reverse scan of its own dU, and the d-alpha error predicted by the kernel's D
alone (exact P, dP; D taken from the kernel's O_lo), computed in fp64 numpy
per 512-query block (test infrastructure: oracle + numpy, no product code).

    python tools/gpu/dalpha_diag.py [C2 C3_w512 dist C4s small]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2512_07782_b200 import binding as gb  # noqa: E402


def band_dalpha(q, k, v, u, do, D, w, h0, scale):
    """fp64 dU, dalpha of one slice with the given per-row D (queries = last Nq keys)."""
    Nq, Nkv = q.shape[0], k.shape[0]
    dU = np.zeros(Nkv)
    for i0 in range(0, Nq, 512):
        i1 = min(Nq, i0 + 512)
        g0, g1 = i0 + h0, i1 + h0
        j0 = max(0, g0 - w + 1)
        S = scale * q[i0:i1] @ k[j0:g1].T + (u[g0:g1, None] - u[None, j0:g1])
        gi = np.arange(g0, g1)[:, None]
        jj = np.arange(j0, g1)[None, :]
        S = np.where((jj <= gi) & (jj > gi - w), S, -np.inf)
        m = S.max(1, keepdims=True)
        P = np.exp(S - m)
        P /= P.sum(1, keepdims=True)
        dP = do[i0:i1] @ v[j0:g1].T
        dS = P * (dP - D[i0:i1, None])
        dU[g0:g1] += dS.sum(1)
        dU[j0:g1] -= dS.sum(0)
    da = -np.flip(np.cumsum(np.flip(dU)))
    return dU, da


def run(name, s, seed, slices, use_gate=True):
    Q, K, V, dO = synth.attn_inputs(s, seed=seed, device="cuda", dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, s.nkv, s.H, seed=seed + 1, device="cuda")
    U = gb.gfwa_gate_prefix(h, beta)
    O, LSE, Olo = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True)
    dQ, dK, dV, dU, da = gb.gfwa_bwd(Q, K, V, U, O, LSE, dO, s.w, O_lo=Olo)
    torch.cuda.synchronize()
    h0 = s.nkv - s.N
    scale = 1.0 / np.sqrt(s.d)
    for b, hh in slices:
        sl = lambda x: x[b:b + 1, :, hh:hh + 1]  # noqa: E731
        Ur = U[b:b + 1, hh:hh + 1]
        g = oracle.bwd(sl(Q), sl(K), sl(V), Ur, sl(dO), s.w)
        Or, _ = oracle.fwd(sl(Q), sl(K), sl(V), Ur, s.w)
        dag = da[b, hh].double().cpu().numpy()
        dUg = dU[b, hh].double().cpu().numpy()
        err = np.abs(dag - g["dalpha"][0, 0])
        t = int(err.argmax())
        scan = -np.flip(np.cumsum(np.flip(dUg)))
        q = sl(Q)[0, :, 0].double().cpu().numpy()
        k = sl(K)[0, :, 0].double().cpu().numpy()
        v = sl(V)[0, :, 0].double().cpu().numpy()
        do = sl(dO)[0, :, 0].double().cpu().numpy()
        u = Ur[0, 0].double().cpu().numpy()
        o_k = sl(O)[0, :, 0].double().cpu().numpy() + sl(Olo)[0, :, 0].double().cpu().numpy()
        Dk = (o_k * do).sum(1)
        De = (Or[0, :, 0] * do).sum(1)
        _, da_D = band_dalpha(q, k, v, u, do, Dk, s.w, h0, scale)
        _, da_E = band_dalpha(q, k, v, u, do, De, s.w, h0, scale)
        alpha = -np.diff(np.concatenate([[0.0], u]))
        print(f"{name} b{b} h{hh}: |da|max={np.abs(g['dalpha']).max():.2f} err_da={err.max():.4f}@t={t} "
              f"err_dU={np.abs(dUg - g['dU'][0, 0]).max():.4f} sum_dU={dUg.sum():.2e} "
              f"da0={dag[0]:.2e} da_vs_scan={np.abs(dag - scan).max():.2e} "
              f"pred_from_D={np.abs(da_D - g['dalpha'][0, 0]).max():.4f} "
              f"numpy_exact_check={np.abs(da_E - g['dalpha'][0, 0]).max():.1e} "
              f"maxD_err={np.abs(Dk - De).max():.2e} mean_alpha={alpha.mean():.3f} "
              f"err_dQ={np.abs(sl(dQ).double().cpu().numpy() - g['dQ']).max():.4f} "
              f"err_O={np.abs(sl(O).double().cpu().numpy() - Or).max():.4f}", flush=True)


def main():
    which = sys.argv[1:] or ["small", "C2", "dist", "C3_w512", "C4s"]
    for wl in which:
        if wl == "small":
            run(wl, synth.AttnShape(B=1, H=4, N=1000, d=128, w=512), 3 * 1000 + 512, [(0, i) for i in range(4)])
        elif wl == "dist":  # the sequence-sharded test's shape, unsharded
            run(wl, synth.AttnShape(B=1, H=4, N=2048, d=128, w=256), 31, [(0, i) for i in range(4)])
        elif wl.startswith("C2") or wl.startswith("C3"):
            c = synth.CONFIGS[wl]
            s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
            run(wl, s, c["seed"], [(0, i) for i in range(4)])
        elif wl == "C4s":
            c = synth.CONFIGS["C4"]
            S = c["N"] // 8
            s = synth.AttnShape(B=1, H=c["H"], N=S, d=c["d"], w=c["w"], N_kv=S + c["w"])
            run(wl, s, c["seed"], [(0, i) for i in range(4, 8)])


if __name__ == "__main__":
    main()
