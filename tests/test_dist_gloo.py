"""Multi-process CPU test of the sequence-sharded orchestration
(paper_2512_07782_b200.dist) with the gloo backend, world_size 2 and 3.

The compute backend is injected with fp64 oracle adapters (test-only), so the
check isolates the host logic: halo slicing, the receiver-frame u values, the
reverse halo of dK/dV/dU and the d-alpha carry.  Every rank's outputs must
equal the matching rows of the unsharded oracle run."""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


def _oracle_ops(rows: bool = False):
    from paper_2512_07782_b200.dist import Ops

    t = lambda a: torch.from_numpy(np.asarray(a))  # noqa: E731

    def gate_prefix(h, beta, eps):
        U, total, _ = oracle.gate_prefix_hbeta(h, beta, eps)
        return t(U), t(total)

    def fwd(Q, K, V, U, w):
        O, L = oracle.fwd(Q, K, V, U, w)
        return t(O), t(L), None

    def bwd(Q, K, V, U, O, LSE, dO, w, Olo):
        g = oracle.bwd(Q, K, V, U, dO, w, want_dalpha=False)
        return t(g["dQ"]), t(g["dK"]), t(g["dV"]), t(g["dU"])

    def gate_bwd(dU, h, beta, eps, carry):
        da = oracle.dalpha_scan(dU, None if carry is None else carry.numpy())
        dh, db = oracle.gate_chain(h, beta, da, eps)
        return t(da), t(dh), t(db)

    def fwd_into(Q, K, V, U, w, O_out, Olo_out):
        O, L = oracle.fwd(Q, K, V, U, w)
        O_out.copy_(t(O))
        return t(L)

    def bwd_rows(Q, K, V, U, O, LSE, dO, w, Olo, head_rows, tail_rows):
        dQ, dK, dV, dU = bwd(Q, K, V, U, O, LSE, dO, w, Olo)
        n = dK.shape[1]
        head = torch.stack([dK[:, :head_rows], dV[:, :head_rows]]).contiguous() if head_rows else None
        tail = torch.stack([dK[:, n - tail_rows:], dV[:, n - tail_rows:]]).contiguous() if tail_rows else None
        return dQ, dK, dV, dU, head, tail

    return Ops(gate_prefix=gate_prefix, fwd=fwd, bwd=bwd, gate_bwd=gate_bwd, fwd_into=fwd_into,
               bwd_rows=bwd_rows if rows else None)


def _inputs(B, N, H, d, seed):
    g = torch.Generator().manual_seed(seed)
    Q = torch.randn(B, N, H, d, generator=g, dtype=torch.float64)
    K = torch.randn(B, N, H, d, generator=g, dtype=torch.float64)
    V = torch.randn(B, N, H, d, generator=g, dtype=torch.float64)
    dO = torch.randn(B, N, H, d, generator=g, dtype=torch.float64)
    h = torch.randn(B, N, H, generator=g, dtype=torch.float64)
    beta = 1.0 + torch.nn.functional.elu(0.5 * torch.randn(B, N, H, generator=g, dtype=torch.float64))
    return Q, K, V, dO, h, beta


def _worker(rank, world, port, outdir, B, N, H, d, w, use_ext=False, rows=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_07782_b200.dist import Ring, alloc_kv_ext, sp_forward_backward

        Q, K, V, dO, h, beta = _inputs(B, N, H, d, 5)
        S = N // world
        sl = slice(rank * S, (rank + 1) * S)
        Kl, Vl, kv_ext = K[:, sl], V[:, sl], None
        if use_ext:  # [halo; local] buffers: the halo lands in place, no per-step concatenation
            kv_ext, Kl, Vl = alloc_kv_ext(Kl, Vl, w)
        res = sp_forward_backward(Q[:, sl], Kl, Vl, h[:, sl], beta[:, sl], dO[:, sl], w, _oracle_ops(rows),
                                  Ring(), kv_ext=kv_ext)
        torch.save({k: getattr(res, k) for k in ("O", "LSE", "U_loc", "U_offset", "dQ", "dK", "dV", "dalpha", "dh",
                                                 "dbeta")},
                   os.path.join(outdir, f"r{rank}.pt"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N,w,use_ext,rows", [(2, 48, 10, False, False), (2, 40, 20, False, False),
                                                    (3, 60, 7, False, False), (2, 48, 10, True, False),
                                                    (3, 60, 7, True, False),
                                                    # halo dK/dV as pre-rounding [2, B, w, H, d] copies
                                                    (2, 48, 10, True, True), (3, 60, 7, False, True)])
def test_sequence_sharded_matches_unsharded(world, N, w, use_ext, rows):
    B, H, d = 1, 2, 8
    port = 29500 + (os.getpid() % 2000) + (7 if use_ext else 0) + (13 if rows else 0)
    with tempfile.TemporaryDirectory() as outdir:
        mp.spawn(_worker, args=(world, port, outdir, B, N, H, d, w, use_ext, rows), nprocs=world, join=True)
        Q, K, V, dO, h, beta = _inputs(B, N, H, d, 5)
        U, _, _ = oracle.gate_prefix_hbeta(h, beta)
        O, L = oracle.fwd(Q, K, V, U, w)
        g = oracle.bwd(Q, K, V, U, dO, w)
        dh, db = oracle.gate_chain(h, beta, g["dalpha"])
        S = N // world
        for r in range(world):
            res = torch.load(os.path.join(outdir, f"r{r}.pt"))
            sl = slice(r * S, (r + 1) * S)
            assert np.allclose(res["O"].numpy(), O[:, sl], atol=1e-12)
            assert np.allclose(res["LSE"].numpy(), L[..., sl], atol=1e-11)
            assert np.allclose(res["dQ"].numpy(), g["dQ"][:, sl], atol=1e-11)
            assert np.allclose(res["dK"].numpy(), g["dK"][:, sl], atol=1e-11)
            assert np.allclose(res["dV"].numpy(), g["dV"][:, sl], atol=1e-11)
            assert np.allclose(res["dalpha"].numpy(), g["dalpha"][..., sl], atol=1e-10)
            assert np.allclose(res["dh"].numpy(), dh[:, sl], atol=1e-10)
            assert np.allclose(res["dbeta"].numpy(), db[:, sl], atol=1e-10)
            # local frame: global U = U_loc - P_r, P_r = the cross-rank exclusive scan of
            # the gate totals (returned by the step) = -U[r S - 1] of the unsharded scan
            off = -U[..., r * S - 1] if r > 0 else np.zeros(U.shape[:2])
            assert np.allclose(res["U_offset"].numpy(), off, atol=1e-11)
            assert np.allclose(res["U_loc"].numpy() - res["U_offset"].numpy()[..., None], U[..., sl], atol=1e-11)


def test_halo_larger_than_shard_is_rejected():
    from paper_2512_07782_b200.dist import Ops, sp_forward_backward

    class _R:
        rank, world = 0, 2

    Q = torch.zeros(1, 4, 1, 8)
    with pytest.raises(ValueError):
        sp_forward_backward(Q, Q, Q, Q[..., 0, 0:1].squeeze(-1), Q[..., 0, 0:1].squeeze(-1), Q, 5,
                            Ops(None, None, None, None), _R())
