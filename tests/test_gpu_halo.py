"""In-kernel halo (include/gfwa.h `halo_rows`; SURVEY 8(e)'s B200 refinement, 8(f)
f3): the attention kernels TMA-load the first key rows straight from a separate
buffer -- the previous shard's rows in its own memory -- instead of a contiguous
[halo; local] K / V.  Checked here: the halo form equals the contiguous call
(same kernels, only the TMA source of the halo tiles differs), both match the fp64
oracle at north_star's bf16 tolerances, argument validation, and the halo read
through a CUDA-IPC mapping of another process's allocation (a peer pointer: the
same access path NVLink peers use; both processes on cuda:0, the producer keeps
its tensors alive and unchanged until the consumer is done -- no kernel waits on
another process)."""

import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth
from paper_2512_07782_b200 import binding as gb
from parity import TOL_BF16_GRAD, TOL_BF16_O, TOL_LSE, max_abs

pytestmark = pytest.mark.gpu


def _U(B, H, Nkv, seed):
    g = torch.Generator().manual_seed(seed)
    alpha = torch.nn.functional.softplus(torch.randn(B, H, Nkv, generator=g))
    return (-torch.cumsum(alpha.double(), -1)).float()


def _case(B, H, Nq, hr, d, w, seed):
    s = synth.AttnShape(B=B, H=H, N=Nq, d=d, w=w, N_kv=Nq + hr)
    Q, K, V, dO = synth.attn_inputs(s, seed=seed, dtype=torch.bfloat16)
    return s, Q, K, V, dO, _U(B, H, s.nkv, seed + 1)


@pytest.mark.parametrize("B,H,Nq,hr,d,w", [(1, 2, 300, 256, 128, 256), (2, 2, 520, 128, 128, 200),
                                           (1, 3, 400, 384, 64, 300), (2, 2, 256, 256, 128, 1000)])
def test_kv_halo_equals_contiguous_and_oracle(B, H, Nq, hr, d, w):
    s, Q, K, V, dO, U = _case(B, H, Nq, hr, d, w, seed=Nq + hr + w)
    Qd, Kd, Vd, dOd, Ud = (x.cuda() for x in (Q, K, V, dO, U))
    # the halo rows in their own allocation; K, V = views of the local rows of the
    # [B, N_kv] buffers (the ABI's stride rule for B > 1)
    Kh, Vh = Kd[:, :hr].clone(), Vd[:, :hr].clone()
    Kl, Vl = Kd[:, hr:], Vd[:, hr:]
    O0, L0, Lo0 = gb.gfwa_fwd(Qd, Kd, Vd, Ud, w, want_o_lo=True)
    O1, L1, Lo1 = gb.gfwa_fwd(Qd, Kl, Vl, Ud, w, want_o_lo=True, kv_halo=(Kh, Vh))
    torch.cuda.synchronize()
    assert torch.equal(O0, O1) and torch.equal(L0, L1) and torch.equal(Lo0, Lo1)
    g0 = gb.gfwa_bwd(Qd, Kd, Vd, Ud, O0, L0, dOd, w, O_lo=Lo0)
    g1 = gb.gfwa_bwd(Qd, Kl, Vl, Ud, O1, L1, dOd, w, O_lo=Lo1, kv_halo=(Kh, Vh))
    torch.cuda.synchronize()
    names = ("dQ", "dK", "dV", "dU", "dalpha")
    for n, a, b in zip(names, g0, g1):
        assert a.shape == b.shape, n
        if n in ("dK", "dV"):  # per-item accumulation in TMEM: the same bits
            assert torch.equal(a, b), n
        else:  # dQ / dU gather reductions from several CTAs (order-dependent fp32 sums)
            assert (a.float() - b.float()).abs().max().item() <= 1e-2 * max(1.0, a.float().abs().max().item()), n
    Or, Lr = oracle.fwd(Q, K, V, U, w)
    ref = oracle.bwd(Q, K, V, U, dO, w)
    assert max_abs(O1, Or) <= TOL_BF16_O
    assert max_abs(L1, Lr) <= TOL_LSE
    for n, a in zip(names, g1):
        assert max_abs(a, ref[n]) <= TOL_BF16_GRAD, n


def test_kv_halo_training_forward_and_rows_f32():
    """gfwa_fwd_train (prepared workspace) and gfwa_bwd_rows_f32 in the halo form."""
    B, H, Nq, hr, d, w = 1, 2, 512, 256, 128, 256
    s, Q, K, V, dO, U = _case(B, H, Nq, hr, d, w, seed=77)
    Qd, Kd, Vd, dOd, Ud = (x.cuda() for x in (Q, K, V, dO, U))
    Kh, Vh = Kd[:, :hr].clone(), Vd[:, :hr].clone()
    O, L, Lo = gb.gfwa_fwd(Qd, Kd[:, hr:], Vd[:, hr:], Ud, w, want_o_lo=True, prepare_bwd=True, kv_halo=(Kh, Vh))
    dQ, dK, dV, dU, head, tail = gb.gfwa_bwd_rows_f32(Qd, Kd[:, hr:], Vd[:, hr:], Ud, O, L, dOd, w, hr, hr,
                                                      O_lo=Lo, kv_halo=(Kh, Vh))
    torch.cuda.synchronize()
    ref = oracle.bwd(Q, K, V, U, dO, w)
    Or, _ = oracle.fwd(Q, K, V, U, w)
    assert max_abs(O, Or) <= TOL_BF16_O
    for n, a in (("dQ", dQ), ("dK", dK), ("dV", dV), ("dU", dU)):
        assert max_abs(a, ref[n]) <= TOL_BF16_GRAD, n
    assert torch.equal(head[0].to(torch.bfloat16), dK[:, :hr]) and torch.equal(tail[1].to(torch.bfloat16), dV[:, -hr:])


def test_kv_halo_argument_validation():
    B, H, Nq, d, w = 1, 2, 256, 128, 128
    s, Q, K, V, dO, U = _case(B, H, Nq, 256, d, w, seed=5)
    Qd, Kd, Vd, Ud = (x.cuda() for x in (Q, K, V, U))
    with pytest.raises(gb.GfwaError):  # halo rows not a multiple of the 128-key tile
        gb.gfwa_fwd(Qd, Kd[:, 100:], Vd[:, 100:], Ud, w, kv_halo=(Kd[:, :100].clone(), Vd[:, :100].clone()))
    with pytest.raises(gb.GfwaError):  # more halo rows than lie in front of the queries
        gb.gfwa_fwd(Qd, Kd[:, 384:], Vd[:, 384:], Ud, w, kv_halo=(Kd[:, :384].clone(), Vd[:, :384].clone()))
    Qf, Kf, Vf = Qd.float(), Kd.float(), Vd.float()
    with pytest.raises(gb.GfwaError):  # fp32: the SIMT parity path has no halo form
        gb.gfwa_fwd(Qf, Kf[:, 256:], Vf[:, 256:], Ud, w, kv_halo=(Kf[:, :256].clone(), Vf[:, :256].clone()))


def _producer(q_out, done):
    torch.cuda.set_device(0)
    B, H, Nq, hr, d, w = 1, 2, 384, 256, 128, 256
    s, Q, K, V, dO, U = _case(B, H, Nq, hr, d, w, seed=91)
    Kd, Vd = K.cuda(), V.cuda()  # "rank r-1": its rows live in this process's memory
    q_out.put((Kd, Vd))          # CUDA IPC handles (torch.multiprocessing)
    done.wait(120)


def test_kv_halo_through_cuda_ipc_peer_pointer():
    ctx = mp.get_context("spawn")
    q, done = ctx.Queue(), ctx.Event()
    p = ctx.Process(target=_producer, args=(q, done))
    p.start()
    try:
        Kp, Vp = q.get(timeout=120)  # mapped from the producer's allocation
        B, H, Nq, hr, d, w = 1, 2, 384, 256, 128, 256
        s, Q, K, V, dO, U = _case(B, H, Nq, hr, d, w, seed=91)
        Qd, dOd, Ud = Q.cuda(), dO.cuda(), U.cuda()
        Kl, Vl = K[:, hr:].cuda(), V[:, hr:].cuda()  # this rank's own rows
        O, L, Lo = gb.gfwa_fwd(Qd, Kl, Vl, Ud, w, want_o_lo=True, kv_halo=(Kp[:, :hr], Vp[:, :hr]))
        g = gb.gfwa_bwd(Qd, Kl, Vl, Ud, O, L, dOd, w, O_lo=Lo, kv_halo=(Kp[:, :hr], Vp[:, :hr]))
        torch.cuda.synchronize()
        Or, Lr = oracle.fwd(Q, K, V, U, w)
        ref = oracle.bwd(Q, K, V, U, dO, w)
        assert max_abs(O, Or) <= TOL_BF16_O
        for n, a in zip(("dQ", "dK", "dV", "dU", "dalpha"), g):
            assert max_abs(a, ref[n]) <= TOL_BF16_GRAD, n
        del Kp, Vp
    finally:
        done.set()
        p.join(60)
