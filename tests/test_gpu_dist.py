"""Sequence-sharded GatedFWA on the CUDA path: 2 ranks (gloo transport with
host staging, both on cuda:0 -- the box exposes one GPU) running
paper_2512_07782_b200.dist.sp_forward_backward with the libgfwa kernels on
the [halo; local] extended tensors, compared with the unsharded fp64 oracle."""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from parity import TOL_BF16_GRAD, TOL_BF16_O

pytestmark = pytest.mark.gpu

B, H, N, D, W = 1, 4, 2048, 128, 256


def _inputs():
    s = synth.AttnShape(B=B, H=H, N=N, d=D, w=W)
    Q, K, V, dO = synth.attn_inputs(s, seed=31, dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(B, N, H, seed=32)
    return Q, K, V, dO, h, beta


def _worker(rank, world, port, outdir, use_ext=False, use_peer=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_07782_b200.dist import Ring, alloc_kv_ext, cuda_ops, map_peer_halo, sp_forward_backward

        torch.cuda.set_device(0)
        Q, K, V, dO, h, beta = _inputs()
        S = N // world
        sl = slice(rank * S, (rank + 1) * S)
        cu = lambda x: x[:, sl].contiguous().cuda()  # noqa: E731
        Kl, Vl, kv_ext = cu(K), cu(V), None
        if use_ext:  # [halo; local] resident buffers (the bench's C4 path)
            kv_ext, Kl, Vl = alloc_kv_ext(Kl, Vl, W)
        ring = Ring()
        # in-kernel peer halo: rank r-1's K / V mapped by CUDA IPC, read by the kernels' TMA
        peer = map_peer_halo(Kl, Vl, W, ring) if use_peer else None
        res = sp_forward_backward(cu(Q), Kl, Vl, cu(h), cu(beta), cu(dO), W, cuda_ops(), ring, kv_ext=kv_ext,
                                  peer=peer)
        torch.cuda.synchronize()
        dist.barrier()  # rank r-1's K / V stay alive until rank r's kernels are done
        out = {k: getattr(res, k).float().cpu() for k in ("O", "dQ", "dK", "dV", "dU", "dalpha", "U_loc")}
        out["U_offset"] = res.U_offset.double().cpu()
        torch.save(out,
                   os.path.join(outdir, f"r{rank}.pt"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("use_ext,use_peer", [(False, False), (True, False), (True, True)])
def test_sequence_sharded_cuda_matches_oracle(use_ext, use_peer):
    world = 2
    port = 31500 + (os.getpid() % 2000) + (11 if use_ext else 0) + (23 if use_peer else 0)
    with tempfile.TemporaryDirectory() as outdir:
        mp.spawn(_worker, args=(world, port, outdir, use_ext, use_peer), nprocs=world, join=True)
        Q, K, V, dO, h, beta = _inputs()
        U, _, _ = oracle.gate_prefix_hbeta(h, beta)
        O, _ = oracle.fwd(Q, K, V, U, W)
        g = oracle.bwd(Q, K, V, U, dO, W)
        S = N // world
        res = [torch.load(os.path.join(outdir, f"r{r}.pt")) for r in range(world)]
        for r in range(world):
            sl = slice(r * S, (r + 1) * S)
            assert np.abs(res[r]["O"].numpy() - O[:, sl]).max() <= TOL_BF16_O
            for k in ("dQ", "dK", "dV"):
                assert np.abs(res[r][k].numpy() - g[k][:, sl]).max() <= TOL_BF16_GRAD, k
            assert np.abs(res[r]["dU"].numpy() - g["dU"][..., sl]).max() <= TOL_BF16_GRAD
            # the cross-rank exclusive scan of the gate totals: global U = U_loc - P_r
            off = -U[..., r * S - 1] if r > 0 else np.zeros(U.shape[:2])
            assert np.abs(res[r]["U_offset"].numpy() - off).max() <= 1e-6 * max(1.0, np.abs(off).max())
            U_glob = res[r]["U_loc"].double().numpy() - res[r]["U_offset"].numpy()[..., None]
            assert np.abs(U_glob - U[..., sl]).max() <= 1e-6 * np.abs(U[..., sl]).max()
        # the sharded d-alpha must equal the exact (fp64) reverse scan of the
        # gathered dU -- which checks the cross-rank carry -- and the oracle's
        # d-alpha at north_star's gradient tolerance
        dU_all = np.concatenate([res[r]["dU"].numpy().astype(np.float64) for r in range(world)], -1)
        da_scan = -np.flip(np.cumsum(np.flip(dU_all, -1), -1), -1)
        da_all = np.concatenate([res[r]["dalpha"].numpy().astype(np.float64) for r in range(world)], -1)
        assert np.abs(da_all - da_scan).max() <= 1e-5 * max(1.0, np.abs(da_scan).max())
        assert np.abs(da_all - g["dalpha"]).max() <= TOL_BF16_GRAD
