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


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_07782_b200.dist import Ring, cuda_ops, sp_forward_backward

        torch.cuda.set_device(0)
        Q, K, V, dO, h, beta = _inputs()
        S = N // world
        sl = slice(rank * S, (rank + 1) * S)
        cu = lambda x: x[:, sl].contiguous().cuda()  # noqa: E731
        res = sp_forward_backward(cu(Q), cu(K), cu(V), cu(h), cu(beta), cu(dO), W, cuda_ops(), Ring())
        torch.cuda.synchronize()
        torch.save({k: getattr(res, k).float().cpu() for k in ("O", "dQ", "dK", "dV", "dalpha")},
                   os.path.join(outdir, f"r{rank}.pt"))
    finally:
        dist.destroy_process_group()


def test_sequence_sharded_cuda_matches_oracle():
    world = 2
    port = 31500 + (os.getpid() % 2000)
    with tempfile.TemporaryDirectory() as outdir:
        mp.spawn(_worker, args=(world, port, outdir), nprocs=world, join=True)
        Q, K, V, dO, h, beta = _inputs()
        U, _, _ = oracle.gate_prefix_hbeta(h, beta)
        O, _ = oracle.fwd(Q, K, V, U, W)
        g = oracle.bwd(Q, K, V, U, dO, W)
        S = N // world
        for r in range(world):
            res = torch.load(os.path.join(outdir, f"r{r}.pt"))
            sl = slice(r * S, (r + 1) * S)
            assert np.abs(res["O"].numpy() - O[:, sl]).max() <= TOL_BF16_O
            for k in ("dQ", "dK", "dV"):
                assert np.abs(res[k].numpy() - g[k][:, sl]).max() <= TOL_BF16_GRAD, k
            assert np.abs(res["dalpha"].numpy() - g["dalpha"][..., sl]).max() <= TOL_BF16_GRAD
