"""Sequence-sharded GatedFWA over P ranks (BASELINE.json north_star: long
sequences "sequence-sharded across the 8 B200s of one box ... a halo of the
previous w K/V rows plus the running gate-sum offset").

Why this is the whole exchange: the window bounds every dependency to the
previous w keys, so with w <= S = N/P rows per rank, rank r needs only
rank r-1's last w K/V rows and their u values; the backward returns the halo's
dK/dV/dU to rank r-1 and, through the straddle identity, the d-alpha carry.

Frames:
  * each rank scans its own gates with carry 0:  U_loc[i] = -sum_{q<=i} alpha_q
    (global U = U_loc - P_r, P_r = sum of earlier ranks' totals; only the
    optional global U needs the all-gather of totals);
  * halo u values are sent in the receiver's frame:
    u_halo = U_loc(r-1)[S-w:] - U_loc(r-1)[S-1]  (exact: the bias only uses
    differences, and LSE is shift-invariant, C-10);
  * backward: dU of the halo rows is added into rank r-1's last w rows and the
    carry for rank r-1's reverse scan is  +sum_j dU_halo(j)  (Appendix A.1:
    sum_{m >= s_r} dU_m = sum of the straddling dS = -sum_j dU_halo(j)).

The compute backend is injectable (``Ops``): on GPUs it is libgfwa (the CUDA
path); the CPU multi-process tests inject oracle adapters to check this host
logic with the gloo backend.  Communication uses torch.distributed P2P
(NCCL over NVLink on the box).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist


@dataclass
class Ops:
    gate_prefix: Callable   # (h, beta, eps) -> (U [B,H,S] fp32 (carry 0), total = sum alpha [B,H] fp64)
    fwd: Callable           # (Q, K, V, U, w) -> (O, LSE, O_lo)
    bwd: Callable           # (Q, K, V, U, O, LSE, dO, w, O_lo) -> (dQ, dK, dV, dU)
    gate_bwd: Callable      # (dU, h, beta, eps, carry fp64 [B,H] | None) -> (dalpha, dh, dbeta)
    # (Q, K, V, U, w, O_out, Olo_out | None) -> LSE: the forward written into caller views
    # (lets the step run the interior queries while the halo is in flight); None: no split
    fwd_into: Callable | None = None
    # (Q, K, V, U, O, LSE, dO, w, O_lo, head_rows, tail_rows) -> (dQ, dK, dV, dU, head, tail):
    # bwd plus pre-rounding copies [2 (dK, dV), B, rows, H, d] of the first / last key rows'
    # dK, dV, so the halo gradients travel and are added before their one rounding
    # (fp32).  None: the halo rows travel in the gradients' dtype
    bwd_rows: Callable | None = None
    # in-kernel peer halo (SURVEY 8(e) refinement, f3): fwd / bwd_rows with kv_halo = the
    # previous rank's last w K/V rows read by TMA straight from its memory (map_peer_halo)
    fwd_halo: Callable | None = None      # (Q, K, V, U, w, kv_halo) -> (O, LSE, O_lo)
    bwd_rows_halo: Callable | None = None  # bwd_rows(..., kv_halo) -> as bwd_rows


def cuda_ops() -> Ops:
    """The libgfwa (CUDA) backend."""
    from . import binding as gb

    def _fwd(Q, K, V, U, w):
        # the step's backward follows on the same problem: gfwa_fwd_train zeroes its
        # dQ accumulator inside the forward (the token keeps other orders safe)
        return gb.gfwa_fwd(Q, K, V, U, w, want_o_lo=True, prepare_bwd=True)

    def _bwd(Q, K, V, U, O, LSE, dO, w, Olo):
        dQ, dK, dV, dU, _ = gb.gfwa_bwd(Q, K, V, U, O, LSE, dO, w, O_lo=Olo, want_dalpha=False)
        return dQ, dK, dV, dU

    def _gate_bwd(dU, h, beta, eps, carry):
        return gb.gfwa_gate_prefix_bwd(dU, h, beta, eps, carry=carry)

    def _fwd_into(Q, K, V, U, w, O_out, Olo_out):
        return gb.gfwa_fwd(Q, K, V, U, w, out=O_out, out_lo=Olo_out)[1]

    def _bwd_rows(Q, K, V, U, O, LSE, dO, w, Olo, head_rows, tail_rows):
        if Q.dtype != torch.bfloat16:  # the fp32 parity path is exact: nothing to carry
            return (*_bwd(Q, K, V, U, O, LSE, dO, w, Olo), None, None)
        return gb.gfwa_bwd_rows_f32(Q, K, V, U, O, LSE, dO, w, head_rows, tail_rows, O_lo=Olo)

    def _fwd_halo(Q, K, V, U, w, kv_halo):
        return gb.gfwa_fwd(Q, K, V, U, w, want_o_lo=True, prepare_bwd=True, kv_halo=kv_halo)

    def _bwd_rows_halo(Q, K, V, U, O, LSE, dO, w, Olo, head_rows, tail_rows, kv_halo):
        return gb.gfwa_bwd_rows_f32(Q, K, V, U, O, LSE, dO, w, head_rows, tail_rows, O_lo=Olo, kv_halo=kv_halo)

    return Ops(gate_prefix=lambda h, b, eps: gb.gfwa_gate_prefix(h, b, eps, want_total=True), fwd=_fwd, bwd=_bwd,
               gate_bwd=_gate_bwd, fwd_into=_fwd_into, bwd_rows=_bwd_rows, fwd_halo=_fwd_halo,
               bwd_rows_halo=_bwd_rows_halo)


class Ring:
    """Neighbour exchange on a process group (rank r <-> r+1)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # gloo moves host tensors only: stage CUDA tensors through pinned host memory
        self.stage = dist.get_backend(group) != "nccl"

    def _glob(self, r):
        return dist.get_global_rank(self.group, r) if self.group is not None else r

    def shift(self, send: list[torch.Tensor] | None, recv_like: list[torch.Tensor] | None, forward: bool):
        """forward=True: rank r sends to r+1 and receives from r-1 (else the reverse)."""
        return self.finish(self.start(send, recv_like, forward))

    def start(self, send, recv_like, forward: bool):
        """Post the exchange of shift() and return a handle for finish(); with NCCL the
        transfer runs on NCCL's stream while the caller enqueues independent work."""
        dst = self.rank + 1 if forward else self.rank - 1
        src = self.rank - 1 if forward else self.rank + 1
        ops = []
        recv = None
        dev = None
        if send is not None and 0 <= dst < self.world:
            if self.stage:
                send = [t.cpu() for t in send]
            ops += [dist.P2POp(dist.isend, t.contiguous(), self._glob(dst), self.group) for t in send]
        if recv_like is not None and 0 <= src < self.world:
            dev = recv_like[0].device
            recv = [torch.empty_like(t, device="cpu" if self.stage else t.device) for t in recv_like]
            ops += [dist.P2POp(dist.irecv, t, self._glob(src), self.group) for t in recv]
        reqs = dist.batch_isend_irecv(ops) if ops else []
        return reqs, recv, dev

    def finish(self, handle):
        reqs, recv, dev = handle
        for req in reqs:
            req.wait()  # NCCL: the current stream waits for the transfer (no host block)
        if recv is not None and self.stage:
            recv = [t.to(dev) for t in recv]
        return recv


@dataclass
class ShardResult:
    O: torch.Tensor
    LSE: torch.Tensor
    U_loc: torch.Tensor
    dQ: torch.Tensor
    dK: torch.Tensor
    dV: torch.Tensor
    dalpha: torch.Tensor
    dh: torch.Tensor
    dbeta: torch.Tensor
    dU: torch.Tensor = None  # this rank's rows, halo contributions of rank r+1 added
    U_offset: torch.Tensor = None  # P_r = sum of earlier ranks' gate totals [B,H] fp64: U = U_loc - P_r


@dataclass
class PeerHalo:
    """map_peer_halo's result: kv = views of the previous rank's last w K / V rows in
    its memory (None on rank 0); every rank passes its PeerHalo to sp_forward_backward."""
    kv: tuple | None
    mapped: tuple | None = None  # the mapped allocations (kept referenced)


def map_peer_halo(K: torch.Tensor, V: torch.Tensor, w: int, ring: "Ring") -> PeerHalo:
    """The in-kernel peer halo's mapping (SURVEY 8(e)'s B200 refinement): every rank
    publishes CUDA IPC handles of its local K, V (torch's tensor reductions, exchanged
    once through the process group) and rank r maps rank r-1's allocation into its
    own address space -- over NVLink on a multi-GPU box (peer access), the same device
    in the one-GPU tests.  Returns a PeerHalo with views of rank r-1's last w rows
    for kv_halo (none on rank 0).  The caller keeps K, V alive and unchanged while a
    neighbour's step may read them (the step's inputs are read-only)."""
    from torch.multiprocessing.reductions import reduce_tensor

    if K.device.type != "cuda" or K.dtype != torch.bfloat16:
        raise ValueError("the in-kernel peer halo needs bf16 CUDA tensors")
    mine = (reduce_tensor(K), reduce_tensor(V), K.shape[1])
    objs = [None] * ring.world
    dist.all_gather_object(objs, mine, group=ring.group)
    if ring.rank == 0:
        return PeerHalo(None)
    (fk, ak), (fv, av), S_prev = objs[ring.rank - 1]
    if w > S_prev:
        raise ValueError(f"sequence sharding needs w <= rows per rank ({w} > {S_prev})")
    Kp, Vp = fk(*ak), fv(*av)  # the previous rank's tensors, IPC-mapped
    return PeerHalo((Kp[:, S_prev - w:], Vp[:, S_prev - w:]), (Kp, Vp))


def halo_pack(K, V, U_loc, w: int):
    """Last w K/V rows and their u in the receiver's frame (U_loc[S-1] -> 0)."""
    S = K.shape[1]
    return [K[:, S - w:].contiguous(), V[:, S - w:].contiguous(),
            (U_loc[..., S - w:] - U_loc[..., S - 1:S]).contiguous()]


def global_offset_start(total: torch.Tensor, ring: Ring):
    """Post the cross-rank exclusive scan of the gate totals (north_star's "running
    gate-sum offset"): an all-gather of the [B,H] fp64 totals, asynchronous so it
    overlaps the attention calls; finish with global_offset_finish."""
    dev = total.device
    t = total.detach().to(torch.float64).contiguous()
    if ring.stage:  # gloo moves host tensors
        t = t.cpu()
    allt = [torch.empty_like(t) for _ in range(ring.world)]
    work = dist.all_gather(allt, t, group=ring.group, async_op=True)
    return work, allt, dev


def global_offset_finish(handle, ring: Ring) -> torch.Tensor:
    """P_r = sum_{r' < r} total_{r'} (exclusive prefix, fp64), on the totals' device."""
    work, allt, dev = handle
    work.wait()
    out = torch.zeros_like(allt[0])
    for r in range(ring.rank):
        out += allt[r]
    return out.to(dev)


def global_offset(total: torch.Tensor, ring: Ring) -> torch.Tensor:
    """P_r = sum of the earlier ranks' gate totals (exclusive scan, fp64)."""
    return global_offset_finish(global_offset_start(total, ring), ring)


def alloc_kv_ext(K: torch.Tensor, V: torch.Tensor, w: int):
    """[halo; local] K/V buffers of S + w rows holding a copy of the local K, V in
    rows [w, S + w).  Pass them as ``kv_ext`` (and the returned local views as
    K, V) so every step receives the halo in place and the attention calls run
    on views: no per-step concatenation of the S local rows."""
    B, S, H, d = K.shape
    Kx = torch.empty(B, S + w, H, d, dtype=K.dtype, device=K.device)
    Vx = torch.empty_like(Kx)
    Kx[:, w:].copy_(K)
    Vx[:, w:].copy_(V)
    return (Kx, Vx), Kx[:, w:], Vx[:, w:]


def sp_forward_backward(Q, K, V, h, beta, dO, w: int, ops: Ops, ring: Ring, eps: float = 1e-6,
                        kv_ext=None, peer=None) -> ShardResult:
    """One sequence-sharded training step on this rank's S rows.

    Q, K, V, dO [B,S,H,d]; h, beta [B,S,H] (this rank's contiguous rows).
    Requires w <= S (one-hop halo).  kv_ext = (K_ext, V_ext) from alloc_kv_ext
    (K, V then being their local views) avoids copying the local rows every step;
    dK, dV are then returned as views of the backward's [halo; local] outputs.
    peer = map_peer_halo(K, V, w, ring), passed on every rank, selects the
    in-kernel peer halo: the kernels TMA-load the previous rank's last w K/V rows
    from its memory, so only the w u values travel forward (all ranks must agree)."""
    S = K.shape[1]
    if w > S:
        raise ValueError(f"sequence sharding needs w <= rows per rank ({w} > {S})")
    r, P = ring.rank, ring.world
    U_loc, total = ops.gate_prefix(h, beta, eps)
    # the running gate-sum offset of this shard (global U = U_loc - P_r): posted now,
    # collected after the backward (the attention only uses local frames, C-10)
    scan = global_offset_start(total, ring) if P > 1 else None
    use_peer = peer is not None and P > 1
    kv_peer = peer.kv if use_peer else None
    # forward halo r -> r+1 (K, V, u in the receiver's frame; u only with the peer halo)
    like = halo_pack(K, V, U_loc, w)
    if use_peer:
        like = like[2:]
    handle = ring.start(like if r < P - 1 else None, like, forward=True)
    split = kv_ext is not None and ops.fwd_into is not None and r > 0 and 2 * w <= S and not use_peer
    if split:
        # queries [w, S) see only local keys: run them while the halo is in flight,
        # then the first w queries over [halo; local[:w]] (the ABI's halo convention)
        O = torch.empty_like(Q)
        # the bf16 residual of the output cast for the backward's D (reading C-12)
        Olo = torch.empty_strided(O.shape, O.stride(), dtype=torch.bfloat16, device=O.device) \
            if (O.is_cuda and O.dtype == torch.bfloat16) else None
        LSE = torch.empty(Q.shape[0], Q.shape[2], S, dtype=torch.float32, device=Q.device)
        LSE[..., w:] = ops.fwd_into(Q[:, w:], K, V, U_loc, w, O[:, w:], None if Olo is None else Olo[:, w:])
    recv = ring.finish(handle)
    if recv is not None and use_peer:  # K / V halo read in-kernel from rank r-1's memory
        Kx, Vx = K, V
        Ux = torch.cat([recv[0], U_loc], -1).contiguous()
        h0 = w
    elif recv is not None:
        if kv_ext is not None:
            Kx, Vx = kv_ext  # the w halo rows land in front of the resident local rows
            Kx[:, :w].copy_(recv[0])
            Vx[:, :w].copy_(recv[1])
        else:
            Kx = torch.cat([recv[0], K], 1)
            Vx = torch.cat([recv[1], V], 1)
        Ux = torch.cat([recv[2], U_loc], -1).contiguous()
        h0 = w
    else:
        Kx, Vx, Ux, h0 = K, V, U_loc, 0
    if split:
        LSE[..., :w] = ops.fwd_into(Q[:, :w], Kx[:, :2 * w], Vx[:, :2 * w], Ux[..., :2 * w].contiguous(), w,
                                    O[:, :w], None if Olo is None else Olo[:, :w])
    elif use_peer and h0:
        O, LSE, Olo = ops.fwd_halo(Q, Kx, Vx, Ux, w, kv_peer)
    else:
        O, LSE, Olo = ops.fwd(Q, Kx, Vx, Ux, w)
    tail_rows = w if r < P - 1 else 0
    head = tail = None
    if use_peer and h0:
        dQ, dKx, dVx, dUx, head, tail = ops.bwd_rows_halo(Q, Kx, Vx, Ux, O, LSE, dO, w, Olo, h0, tail_rows,
                                                          kv_peer)
    elif ops.bwd_rows is not None:
        dQ, dKx, dVx, dUx, head, tail = ops.bwd_rows(Q, Kx, Vx, Ux, O, LSE, dO, w, Olo, h0, tail_rows)
    else:
        dQ, dKx, dVx, dUx = ops.bwd(Q, Kx, Vx, Ux, O, LSE, dO, w, Olo)
    # backward halo r -> r-1: gradients of the halo rows (dK, dV before their rounding when
    # the backend provides them: [2, B, w, H, d] fp32)
    # (every rank of a run takes the same branch: the same backend and dtype on all ranks)
    exact = ops.bwd_rows is not None and (head is not None or tail is not None)
    if exact:
        ref = tail if tail is not None else head
        back_like = [torch.empty(2, dKx.shape[0], w, dKx.shape[2], dKx.shape[3], dtype=ref.dtype,
                                 device=dKx.device), dUx[..., :w]]
        send = [head, dUx[..., :w].contiguous()] if h0 else None
    else:
        back_like = [dKx[:, :w], dVx[:, :w], dUx[..., :w]]
        send = [t.contiguous() for t in back_like] if h0 else None
    handle = ring.start(send, back_like, forward=False)
    if kv_ext is not None:
        dK, dV = dKx[:, h0:], dVx[:, h0:]  # views: no copy of the S local rows
    else:
        dK = dKx[:, h0:].contiguous()
        dV = dVx[:, h0:].contiguous()
    dU = dUx[..., h0:].contiguous()
    # the gate backward of the whole shard runs while the halo gradients travel: with
    # carry = +sum_j dU_halo(j), dalpha_q = carry - sum_{m >= q} dU_m needs no received
    # value for q < S - w (the halo additions to the last w rows cancel the carry), so
    # the local scan with carry 0 is exact there; the last w rows are redone below
    dalpha, dh, dbeta = ops.gate_bwd(dU, h, beta, eps, None)
    back = ring.finish(handle)
    if back is not None:
        if exact:  # own partial + received partial, both before rounding, rounded once
            dK[:, S - w:] = (tail[0] + back[0][0]).to(dK.dtype)
            dV[:, S - w:] = (tail[1] + back[0][1]).to(dV.dtype)
            dU_halo = back[1]
        else:
            dK[:, S - w:] += back[0]
            dV[:, S - w:] += back[1]
            dU_halo = back[2]
        dU[..., S - w:] += dU_halo
        carry = dU_halo.double().sum(-1)  # d-alpha carry = +sum_j dU_halo(j)
        da_t, dh_t, db_t = ops.gate_bwd(dU[..., S - w:].contiguous(), h[:, S - w:].contiguous(),
                                        beta[:, S - w:].contiguous(), eps, carry)
        dalpha[..., S - w:] = da_t
        dh[:, S - w:] = dh_t
        dbeta[:, S - w:] = db_t
    U_offset = global_offset_finish(scan, ring) if scan is not None else torch.zeros_like(total, dtype=torch.float64)
    return ShardResult(O, LSE, U_loc, dQ, dK, dV, dalpha, dh, dbeta, dU, U_offset)
