#!/usr/bin/env python
"""bench.py -- GatedFWA fwd+bwd throughput on B200 (BASELINE.json metric).

One *step* = one pass of the training hot path over one batch (SURVEY §8(a)
rows A2-A6): gfwa_gate_prefix -> gfwa_fwd -> gfwa_bwd (D, main, dalpha) ->
gfwa_gate_prefix_bwd (dh, dbeta).  The decode row (A7) is timed in the same
run as an auxiliary line item on its own workload (C5); the sequence-shard
exchange (A8) runs with ``--workload C4`` under torchrun.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload C2|C3_w128|C3_w512|C3_w2048|C4]

Default workload: BASELINE.json configs[1] (C2: B=8, H=16, N=4096, d=128,
w=512, bf16).  N>1 (torchrun): every rank runs its own C2 batch (batch x head
sharding, no data-path collective: "scaling": "weak").  Inputs are seeded
synthetic tensors (synth.py) resident in HBM; the working set (> 1 GB) is
larger than the 126 MB L2, so no explicit flush is needed between steps.
Timing: CUDA events on the launching stream, barrier + synchronize on both
sides, max over ranks.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GatedFWA fwd+bwd tokens/s and in-window TFLOP/s (% BF16 peak), 1/2/4/8 B200"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": p["hbm_gbs"], "bf16": p["bf16_tflops"], "bf16_sus": p["bf16_tflops_sustained"],
                "src": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16": 1590.0, "bf16_sus": 1400.0, "src": "fallback"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons, sampled every 50 ms from before the
    warm-up until after the timed region; each sample is stamped with the host
    wall clock on arrival and summary() keeps those inside [t0, t1] of the timed
    region (widened by one sampling period so a short region still gets its
    neighbouring samples)."""

    PERIOD_S = 0.05

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.samples = []  # (host time, line)
        self.window = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", str(int(self.PERIOD_S * 1000))],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def mark(self, t0: float, t1: float):
        self.window = (t0 - self.PERIOD_S, t1 + self.PERIOD_S)

    def stop(self):
        if self.proc is not None:
            time.sleep(2 * self.PERIOD_S)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lo, hi = self.window if self.window else (-1e18, 1e18)
        for ts, ln in self.samples:
            if not lo <= ts <= hi:
                continue
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": ["unsampled"]}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "window_s": round(hi - lo, 3)}


def _dist():
    """One process per GPU (torchrun env).  NCCL for the plumbing; GFWA_BENCH_BACKEND=gloo
    exercises the multi-rank code path on a single-GPU box (ranks share cuda:0)."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1:
        import torch
        import torch.distributed as dist

        if not dist.is_initialized():  # run_ours hands the N > 1 headline to run_seq
            dist.init_process_group(os.environ.get("GFWA_BENCH_BACKEND", "nccl"))
        local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
        return dist, dist.get_rank(), ws, local
    return None, 0, 1, 0


def _max_over_ranks(dist, x: float, dev):
    if dist is None:
        return x
    import torch

    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=dev if on_dev else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------------------- our arm


def in_window_fraction(N: int, w: int) -> float:
    return sum(min(t + 1, w) for t in range(N)) / (N * w)


def _step_fns(gb, s, Q, K, V, dO, h, beta, st, stage_events=None):
    """One training step of the hot path (rows A2-A6) through the C ABI."""
    import torch

    def step(timed_kernels: bool = False):
        rec = []
        if timed_kernels:
            e = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
            e[0].record(st)
        U = gb.gfwa_gate_prefix(h, beta)
        if timed_kernels:
            e[1].record(st)
        O, LSE, Olo = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True, prepare_bwd=True)
        if timed_kernels:
            e[2].record(st)
            sev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            for x in sev:  # create the CUDA events (torch creates them lazily)
                x.record(st)
            gb.debug_stage_events(sev)  # after the bwd preprocess kernel / after its main kernel
        dQ, dK, dV, dU, _ = gb.gfwa_bwd(Q, K, V, U, O, LSE, dO, s.w, O_lo=Olo, want_dalpha=False)
        if timed_kernels:
            e[3].record(st)
        _, dh, dbeta = gb.gfwa_gate_prefix_bwd(dU, h, beta, want_dalpha=False)
        if timed_kernels:
            e[4].record(st)
            rec.append((e, sev))
        return rec, (O, dQ, dK, dV, dh, dbeta)

    return step


def measure_dense(workload, steps, warmup, dist, rank, world, local, dev, peaks, no_graph=False, clk=None):
    """One workload's training step (C2 / C3_*), every rank its own batch (batch x
    head sharding: no collective on the data path).  CUDA graph replay timed with
    events, max over ranks; then eager steps with events between the calls for the
    per-call breakdown and the backward main kernel's own time (roofline)."""
    import torch

    import synth
    from paper_2512_07782_b200 import binding as gb

    c = synth.CONFIGS[workload]
    s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
    seed = c["seed"] + 1000 * rank
    Q, K, V, dO = synth.attn_inputs(s, seed=seed, device=dev, dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=seed, device=dev)
    h, beta = h.bfloat16(), beta.bfloat16()
    st = torch.cuda.current_stream(dev)
    step = _step_fns(gb, s, Q, K, V, dO, h, beta, st)
    for _ in range(warmup):
        step()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    # the step is captured once into a CUDA graph (every library call is
    # stream-ordered with no host sync, so it captures as is): the timed region
    # replays it, so host launch overhead stays out of the device timeline
    graph, graph_note = None, "off (--no-graph)"
    n_launch0 = gb.launch_count()
    if not no_graph:
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                step()
            torch.cuda.synchronize(dev)
            graph_note = "captured"
        except Exception as ex:  # capture problems fall back to eager launches, noted
            graph, graph_note = None, f"capture failed, eager: {type(ex).__name__}: {ex}"[:200]
            torch.cuda.synchronize(dev)
    per_step_launches = gb.launch_count() - n_launch0 if graph is not None else None
    for _ in range(2 if graph is not None else 0):
        graph.replay()
    evs = []
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    n_launch0 = gb.launch_count()
    wall0 = time.time()
    t0.record(st)
    for _ in range(steps):
        if graph is not None:
            graph.replay()
        else:
            r, _ = step(timed_kernels=True)
            evs += r
    t1.record(st)
    torch.cuda.synchronize(dev)
    if clk is not None:
        clk.mark(wall0, time.time())
    launches = per_step_launches * steps if graph is not None else gb.launch_count() - n_launch0
    ms = t0.elapsed_time(t1) / steps
    ms = _max_over_ranks(dist, ms, dev)
    if graph is not None:  # per-call breakdown from eager steps (CUDA events between the calls)
        for _ in range(2):  # eager allocations cannot reuse the graph's pool: warm them first
            step()
        torch.cuda.synchronize(dev)
        for _ in range(steps):
            r, _ = step(timed_kernels=True)
            evs += r
        torch.cuda.synchronize(dev)
    parts = {"gate": 0.0, "fwd": 0.0, "bwd": 0.0, "gate_bwd": 0.0, "bwd_pre": 0.0, "bwd_main": 0.0,
             "bwd_post": 0.0}
    for e, sev in evs:
        parts["gate"] += e[0].elapsed_time(e[1])
        parts["fwd"] += e[1].elapsed_time(e[2])
        parts["bwd"] += e[2].elapsed_time(e[3])
        parts["gate_bwd"] += e[3].elapsed_time(e[4])
        parts["bwd_pre"] += e[2].elapsed_time(sev[0])
        parts["bwd_main"] += sev[0].elapsed_time(sev[1])
        parts["bwd_post"] += sev[1].elapsed_time(e[3])
    parts = {k: v / len(evs) for k, v in parts.items()}
    tokens = s.B * s.N * world
    frac_iw = in_window_fraction(s.N, s.w)
    flops_fwd = 4.0 * s.N * s.w * s.d * s.B * s.H  # north_star in-window convention
    flops_bwd = 10.0 * s.N * s.w * s.d * s.B * s.H
    tflops = (flops_fwd + flops_bwd) * world / (ms * 1e-3) / 1e12
    path = gb.gfwa_attn_path(Q, K, V, s.w)
    # dominant kernel: the backward's main kernel (its own launch, timed by the
    # stage events on the launching stream) against the BURST bf16 peak -- the
    # step is ~1 ms, not a seconds-long sustained run
    main_ms = parts["bwd_main"]
    achieved = flops_bwd / (main_ms * 1e-3) / 1e12
    roofline = {"kernel": "bwd_tc_kernel" if path == 1 else "bwd_simt", "bound": "tensor",
                "achieved": round(achieved, 2), "peak": peaks["bf16"], "unit": "TFLOP/s",
                "frac": round(achieved / peaks["bf16"], 4),
                "frac_exact_in_window": round(achieved * frac_iw / peaks["bf16"], 4),
                "traffic": _traffic_from_profiles("bwd_main", workload),
                "kernel_ms": round(main_ms, 4),
                "peak_src": f"{peaks['src']} bf16 burst (MEASURED_PEAKS.json bf16_tflops)",
                "algorithmic": f"10*N*w*d*B*H = {flops_bwd:.4g} FLOP/launch (north_star in-window count)"}
    fwd_ach = flops_fwd / (parts["fwd"] * 1e-3) / 1e12
    return {
        "s": s, "tensors": (Q, K, V, dO, h, beta), "ms": ms, "value": tokens / (ms * 1e-3),
        "tflops": tflops, "pct": tflops / peaks["bf16"], "pct_exact": tflops * frac_iw / peaks["bf16"],
        "frac_iw": frac_iw, "parts": parts, "path": path, "roofline": roofline, "launches": launches,
        "graph_note": graph_note,
        "fwd_kernel": {"kernel": "fwd_tc_kernel", "ms": round(parts["fwd"], 4), "achieved": round(fwd_ach, 2),
                       "frac": round(fwd_ach / peaks["bf16"], 4),
                       "frac_exact_in_window": round(fwd_ach * frac_iw / peaks["bf16"], 4)},
    }


def _dense_summary(r):
    return {"ms_per_step": round(r["ms"], 4), "tokens_per_s": round(r["value"], 1),
            "tflops_in_window": round(r["tflops"], 2), "pct_bf16_peak": round(r["pct"], 4),
            "pct_bf16_peak_exact_in_window": round(r["pct_exact"], 4), "in_window_fraction": round(r["frac_iw"], 4),
            "ms_breakdown": {k: round(v, 4) for k, v in r["parts"].items()},
            "roofline": r["roofline"], "fwd_kernel": r["fwd_kernel"],
            "config": {"B": r["s"].B, "H": r["s"].H, "N": r["s"].N, "d": r["s"].d, "w": r["s"].w}}


def run_ours(args):
    import torch

    dist, rank, world, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and args.workload == "C2":
        # N > 1: the north_star's sequence-sharded C4 step is the headline
        # (strong scaling of one N = 131072 sequence); C2 batch-sharded in aux
        return run_seq(args, aux_c2=not args.no_aux)
    peaks = _peaks()
    clk = ClockSampler(local).start()
    time.sleep(0.3)  # nvidia-smi needs a moment before its first sample
    r = measure_dense(args.workload, args.steps, args.warmup, dist, rank, world, local, dev, peaks,
                      no_graph=args.no_graph, clk=clk)
    clk.stop()
    s = r["s"]
    Q, K, V, dO, h, beta = r["tensors"]
    # e2e: the same step through the public API with pinned host buffers
    e2e = run_e2e(args, s, Q, K, V, dO, h, beta, step_fn=None, dev=dev, world=world, dist=dist)
    del Q, K, V, dO, h, beta, r["tensors"]
    torch.cuda.empty_cache()
    aux = {}
    if rank == 0 and not args.no_aux:
        # the north_star target point (N=8192, w=512, d=128) and the rest of the C3
        # window sweep (BASELINE configs[2]), each with its own kernel roofline
        for wl in ("C3_w512", "C3_w128", "C3_w2048"):
            if wl != args.workload:
                aux[wl] = _dense_summary(measure_dense(wl, max(5, args.steps), 3, None, 0, 1, local, dev, peaks))
                torch.cuda.empty_cache()
        aux.update(run_aux(dev, peaks))
    if not args.no_aux and args.workload == "C2":
        # the sequence-sharded C4 step (P = 1 here: the baseline of the N > 1 lines)
        seq = measure_seq(3, 3, dist, rank, world, local, dev)
        if rank == 0:
            aux["seq_sharded_C4"] = {k: seq[k] for k in ("ms_per_step", "tokens_per_s", "tflops_in_window", "steps")}
            aux["seq_sharded_C4"]["parallelism"] = seq["config"]["parallelism"]
            aux["seq_sharded_C4"]["pct_bf16_peak"] = round(seq["tflops_in_window"] / peaks["bf16"], 4)
    if rank != 0:
        return
    cpu = cpu_baseline(args, s) if (not args.no_cpu and world == 1) else None  # rank 0 at N=1 only
    line = {
        "metric": METRIC,
        "value": round(r["value"], 1),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(r["ms"], 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (synth.py seeded: RMS-normed Q/K, N(0,1) V/dO, gates h~N(mu_h,1), beta=1+elu)",
        "config": {"workload": f"{args.workload} (BASELINE configs[1])" if args.workload == "C2" else args.workload,
                   "B": s.B, "H": s.H, "N": s.N, "d": s.d, "w": s.w, "global_batch": s.B * world,
                   "seq_len": s.N, "parallelism": f"batch-sharded x{world}" if world > 1 else "single GPU",
                   "l2": "inputs larger than L2 (working set > 1 GB), no flush",
                   "in_window_fraction": round(r["frac_iw"], 4), "cuda_graph": r["graph_note"]},
        "tflops_in_window": round(r["tflops"], 2),
        "pct_bf16_peak": round(r["pct"], 4),
        "pct_bf16_peak_exact_in_window": round(r["pct_exact"], 4),
        "ms_breakdown": {k: round(v, 4) for k, v in r["parts"].items()},  # eager calls, events between them
        "attn_path": "tcgen05" if r["path"] == 1 else "simt",
        "roofline": r["roofline"],
        "fwd_kernel": r["fwd_kernel"],
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": r["launches"],
        "clocks": clk.summary(),
        "aux": aux,
    }
    print(json.dumps(line), flush=True)


class _SoloRing:
    """World of one: no neighbours (the N=1 run of the sequence-sharded step)."""

    rank, world = 0, 1

    def shift(self, send, recv_like, forward):
        return None

    def start(self, send, recv_like, forward):
        return None

    def finish(self, handle):
        return None


def run_seq(args, aux_c2: bool = False):
    """--workload C4 (and the N > 1 headline): BASELINE configs[3] (B=1, H=32,
    N=131072, d=128, w=2048) sequence-sharded over the ranks (S = N/P contiguous
    rows each, K/V/u halo r -> r+1 and halo gradients r+1 -> r over NCCL P2P,
    gate totals through a cross-rank exclusive scan; strong scaling)."""
    import torch

    dist, rank, world, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    peaks = _peaks()
    r = measure_seq(args.steps, args.warmup, dist, rank, world, local, dev, sample_clocks=True)
    aux = {}
    if aux_c2:  # BASELINE configs[1] batch-sharded over the same ranks (weak scaling)
        c2 = measure_dense("C2", args.steps, args.warmup, dist, rank, world, local, dev, peaks)
        aux["C2_batch_sharded"] = _dense_summary(c2)
        aux["C2_batch_sharded"]["scaling"] = "weak"
        aux["C2_batch_sharded"]["tokens_per_s_all_ranks"] = round(c2["value"], 1)
    if rank != 0:
        return
    print(json.dumps({
        "metric": METRIC, "value": r["tokens_per_s"], "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (synth.py seeded per rank)",
        "config": r["config"],
        "tflops_in_window": r["tflops_in_window"], "pct_bf16_peak": round(r["tflops_in_window"] / peaks["bf16"], 4),
        "roofline": r.get("roofline"), "gpu_launches": r["gpu_launches"], "clocks": r.get("clocks"),
        "e2e": r.get("e2e"), "aux": aux,
    }), flush=True)


def measure_seq(steps, warmup, dist, rank, world, local, dev, sample_clocks=False):
    """One C4 sequence-sharded training step timed over all ranks (max over ranks);
    every rank must call it (halo P2P and the max are collective)."""
    import torch

    import synth
    from paper_2512_07782_b200 import binding as gb
    from paper_2512_07782_b200.dist import Ring, alloc_kv_ext, cuda_ops, map_peer_halo, sp_forward_backward

    c = synth.CONFIGS["C4"]
    Ng = c["N"]
    S = Ng // world
    s = synth.AttnShape(B=c["B"], H=c["H"], N=S, d=c["d"], w=c["w"])
    seed = c["seed"] + 1000 * rank  # each rank draws its own rows (synthetic data)
    Q, K, V, dO = synth.attn_inputs(s, seed=seed, device=dev, dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, S, s.H, seed=seed, device=dev)
    h, beta = h.bfloat16(), beta.bfloat16()
    ring = Ring() if world > 1 else _SoloRing()
    ops = cuda_ops()
    st = torch.cuda.current_stream(dev)
    kv_ext, K, V = alloc_kv_ext(K, V, s.w)  # K/V resident behind a w-row halo slot
    # opt-in (GFWA_PEER_HALO=1): the in-kernel peer halo -- rank r-1's K/V rows mapped by
    # CUDA IPC and read by the kernels' TMA, only the u halo sent (not the default: it has
    # not run across GPUs in this environment)
    peer = map_peer_halo(K, V, s.w, ring) if world > 1 and os.environ.get("GFWA_PEER_HALO") == "1" else None

    def step():
        return sp_forward_backward(Q, K, V, h, beta, dO, s.w, ops, ring, kv_ext=kv_ext, peer=peer)

    clk = ClockSampler(local).start() if sample_clocks else None
    if clk:
        time.sleep(0.3)
    for _ in range(warmup):
        step()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    n0 = gb.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall0 = time.time()
    e0.record(st)
    for _ in range(steps):
        step()
    e1.record(st)
    torch.cuda.synchronize(dev)
    out = {}
    if clk:
        clk.mark(wall0, time.time())
        clk.stop()
        out["clocks"] = clk.summary()
    launches = gb.launch_count() - n0
    ms = _max_over_ranks(dist, e0.elapsed_time(e1) / steps, dev)
    # e2e: the same sharded step with this rank's inputs copied from pinned host memory
    # and its results (O, dQ, dK, dV, dh, dbeta) copied back every step, pipelined on
    # copy streams like the dense path's; each device input set has its own halo slot
    ext_sets = []

    def alloc_set():
        Qb, dOb = torch.empty_like(Q), torch.empty_like(dO)
        (Kx, Vx), Kb, Vb = alloc_kv_ext(torch.empty_like(K), torch.empty_like(V), s.w)
        ext_sets.append(((Kx, Vx), Kb.data_ptr()))
        return [Qb, Kb, Vb, dOb, torch.empty_like(h), torch.empty_like(beta)]

    def compute_set(bufs):
        Qb, Kb, Vb, dOb, hb, bb = bufs
        ext = next(e for e, ptr in ext_sets if ptr == Kb.data_ptr())
        res = sp_forward_backward(Qb, Kb, Vb, hb, bb, dOb, s.w, ops, ring, kv_ext=ext)
        return (res.O, res.dQ, res.dK, res.dV, res.dh, res.dbeta)

    # roofline of the dominant kernel: this rank's backward main kernel on its [halo; local]
    # rows, timed by the library's stage events on the launching stream (max over ranks)
    hx, bx = (torch.cat([h[:, :s.w], h], 1), torch.cat([beta[:, :s.w], beta], 1)) if rank > 0 else (h, beta)
    Kr, Vr = kv_ext if rank > 0 else (K, V)
    Ux = gb.gfwa_gate_prefix(hx, bx)
    O_, LSE_, Olo_ = gb.gfwa_fwd(Q, Kr, Vr, Ux, s.w, want_o_lo=True, prepare_bwd=True)
    mains = []
    for _ in range(3):
        sev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for x in sev:
            x.record(st)
        gb.debug_stage_events(sev)
        gb.gfwa_bwd(Q, Kr, Vr, Ux, O_, LSE_, dO, s.w, O_lo=Olo_, want_dalpha=False)
        torch.cuda.synchronize(dev)
        mains.append(sev[0].elapsed_time(sev[1]))
        gb.gfwa_fwd(Q, Kr, Vr, Ux, s.w, want_o_lo=True, prepare_bwd=True)  # re-prepare the dQ accumulator
    main_ms = _max_over_ranks(dist, sorted(mains)[1], dev)
    del O_, LSE_, Olo_, Ux, hx, bx
    peaks = _peaks()
    fl_b = 10.0 * S * s.w * s.d * s.B * s.H
    ach = fl_b / (main_ms * 1e-3) / 1e12
    out["roofline"] = {"kernel": "bwd_tc_kernel", "bound": "tensor", "achieved": round(ach, 2),
                       "peak": peaks["bf16"], "unit": "TFLOP/s", "frac": round(ach / peaks["bf16"], 4),
                       "traffic": None, "kernel_ms": round(main_ms, 4),
                       "peak_src": f"{peaks['src']} bf16 burst (MEASURED_PEAKS.json bf16_tflops)",
                       "algorithmic": f"10*S*w*d*B*H = {fl_b:.4g} FLOP/launch per rank (S = N/P rows; "
                                      "north_star in-window count)"}

    class _A:  # run_e2e reads args.steps only
        pass
    a = _A()
    a.steps = steps
    out["e2e"] = run_e2e(a, s, Q, K, V, dO, h, beta, None, dev, world, dist, compute_fn=compute_set,
                         alloc_fn=alloc_set)
    del ext_sets
    fl = 14.0 * Ng * s.w * s.d * s.B * s.H  # fwd 4 + bwd 10 (north_star in-window count)
    out.update({
        "ms_per_step": round(ms, 4), "tokens_per_s": round(s.B * Ng / (ms * 1e-3), 1),
        "tflops_in_window": round(fl / (ms * 1e-3) / 1e12, 2), "gpu_launches": launches, "steps": steps,
        "config": {"workload": "C4 (BASELINE configs[3])", "B": s.B, "H": s.H, "N": Ng, "rows_per_rank": S,
                   "d": s.d, "w": s.w, "halo": "in-kernel peer (CUDA IPC)" if peer is not None else "sent",
                   "parallelism": f"sequence-sharded x{world} (w-row K/V/u halo, "
                                  f"{(dist.get_backend().upper() + ' P2P') if dist else 'no exchange'})",
                   "l2": "inputs larger than L2, no flush"}})
    del Q, K, V, dO, h, beta, kv_ext, peer
    if dist:
        dist.barrier()  # every mapping of a neighbour's K/V is released before its owner frees it
    torch.cuda.empty_cache()
    return out


def _traffic_from_profiles(kind: str, workload: str):
    """dram bytes per launch of this workload's call from the committed ncu summary
    (profiles/traffic.json, one entry per workload); null if that workload was not profiled."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(workload, {}).get(kind)
    except Exception:
        return None


def run_e2e(args, s, Q, K, V, dO, h, beta, step_fn, dev, world, dist, compute_fn=None, alloc_fn=None):
    """The step end to end through the public API with host buffers: every step
    copies its inputs from pinned host memory (H2D) and its results back (D2H).
    Copies run on their own streams (the two copy engines, PCIe full duplex) and
    are pipelined with the compute of the neighbouring steps: inputs of step k+1
    load and results of step k-1 drain while step k computes (double-buffered
    device inputs; a step's input buffer is reused only after its compute)."""
    import torch

    from paper_2512_07782_b200 import binding as gb

    host_in = [x.cpu().pin_memory() for x in (Q, K, V, dO, h, beta)]
    if alloc_fn is None:
        dev_in = [[torch.empty_like(x, device=dev) for x in host_in] for _ in range(2)]
    else:  # the caller's device buffers (e.g. K/V views behind a halo slot)
        dev_in = [alloc_fn() for _ in range(2)]
    outs_host = None
    comp = torch.cuda.current_stream(dev)
    s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    # steady state of the copy/compute pipeline: long enough that its fill (the first
    # step's inputs) and drain (the last step's results) are amortised like any step
    n = max(8, min(2 * args.steps, 24))

    def compute(bufs):
        if compute_fn is not None:
            return compute_fn(bufs)
        Qd, Kd, Vd, dOd, hd, bd = bufs
        U = gb.gfwa_gate_prefix(hd, bd)
        O, LSE, Olo = gb.gfwa_fwd(Qd, Kd, Vd, U, s.w, want_o_lo=True, prepare_bwd=True)
        dQ, dK, dV, dU, _ = gb.gfwa_bwd(Qd, Kd, Vd, U, O, LSE, dOd, s.w, O_lo=Olo, want_dalpha=False)
        _, dh, dbeta = gb.gfwa_gate_prefix_bwd(dU, hd, bd, want_dalpha=False)
        return (O, dQ, dK, dV, dh, dbeta)

    def run(k_steps):
        nonlocal outs_host
        ev_in = [None, None]
        ev_comp = [None, None]
        with torch.cuda.stream(s_h2d):  # inputs of step 0
            for d, hbuf in zip(dev_in[0], host_in):
                d.copy_(hbuf, non_blocking=True)
            ev_in[0] = torch.cuda.Event()
            ev_in[0].record(s_h2d)
        for k in range(k_steps):
            b = k & 1
            if k + 1 < k_steps:  # prefetch the next step's inputs into the other buffer
                with torch.cuda.stream(s_h2d):
                    if ev_comp[1 - b] is not None:
                        s_h2d.wait_event(ev_comp[1 - b])
                    for d, hbuf in zip(dev_in[1 - b], host_in):
                        d.copy_(hbuf, non_blocking=True)
                    ev_in[1 - b] = torch.cuda.Event()
                    ev_in[1 - b].record(s_h2d)
            comp.wait_event(ev_in[b])
            res = compute(dev_in[b])
            ev_comp[b] = torch.cuda.Event()
            ev_comp[b].record(comp)
            if outs_host is None:
                outs_host = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in res]
            with torch.cuda.stream(s_d2h):  # results of step k drain during step k+1
                s_d2h.wait_event(ev_comp[b])
                for hbuf, x in zip(outs_host, res):
                    hbuf.copy_(x, non_blocking=True)
                    x.record_stream(s_d2h)
        comp.wait_stream(s_d2h)
        comp.wait_stream(s_h2d)

    run(4)  # the caching allocator reaches its steady state (results held by the D2H stream)
    torch.cuda.synchronize(dev)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(comp)
    run(n)
    b.record(comp)
    torch.cuda.synchronize(dev)
    ms = _max_over_ranks(dist, a.elapsed_time(b) / n, dev)
    h2d = sum(x.numel() * x.element_size() for x in host_in)
    d2h = sum(x.numel() * x.element_size() for x in outs_host)
    return {"value": round(s.B * s.N * world / (ms * 1e-3), 1), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": round(ms, 3), "steps": n,
            "pipelining": "H2D of step k+1 and D2H of step k-1 overlap step k (copy streams, double-buffered inputs)"}


def run_aux(dev, peaks):
    """Decode (C5) and gate-scan probe (G): achieved HBM GB/s, same run."""
    import torch

    import synth
    from paper_2512_07782_b200 import binding as gb

    out = {}
    c = synth.CONFIGS["C5"]
    B, H, d, w = c["B"], c["H"], c["d"], c["w"]
    Kc, Vc, a_hist, q, k, v, a_new = synth.decode_inputs(B, H, d, w, seed=c["seed"], device=dev)
    Uh = -torch.cumsum(a_hist, -1)
    Uc = Uh - Uh[..., -1:]  # U_cache convention: u_tau - u_newest
    pos = torch.full((B,), w + 17, dtype=torch.int64, device=dev)
    for _ in range(3):
        gb.gfwa_decode(q, k, v, a_new, Kc, Vc, Uc, pos)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        gb.gfwa_decode(q, k, v, a_new, Kc, Vc, Uc, pos)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / n
    byts = B * H * (4 * w * d + 8 * w + 8 * d)  # bf16 K,V rows + fp32 u read and rewritten + q/k/v/o
    out["decode_C5"] = {"ms_per_step": round(ms, 4), "tokens_per_s": round(B / (ms * 1e-3), 1),
                        "achieved_GBps": round(byts / (ms * 1e-3) / 1e9, 1),
                        "frac_hbm": round(byts / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 4),
                        "bytes_per_step": byts}
    del Kc, Vc
    # GQA decode: groups of 4 query heads share a K/V head
    c = synth.CONFIGS["C5_gqa4"]
    B, H, Hk = c["B"], c["H"], c["H_kv"]
    Kc, Vc, a_hist, q, k, v, a_new = synth.decode_inputs(B, H, d, w, seed=c["seed"], device=dev, H_kv=Hk)
    Uh = -torch.cumsum(a_hist, -1)
    Uc = Uh - Uh[..., -1:]
    for _ in range(3):
        gb.gfwa_decode(q, k, v, a_new, Kc, Vc, Uc, pos)
    torch.cuda.synchronize(dev)
    e0.record()
    for _ in range(n):
        gb.gfwa_decode(q, k, v, a_new, Kc, Vc, Uc, pos)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / n
    byts = B * Hk * 4 * w * d + B * H * (8 * w + 4 * d) + B * Hk * 4 * d  # K,V rows once per group; u (r+w), q, o per head
    out["decode_C5_gqa4"] = {"ms_per_step": round(ms, 4), "tokens_per_s": round(B / (ms * 1e-3), 1),
                             "achieved_GBps": round(byts / (ms * 1e-3) / 1e9, 1),
                             "frac_hbm": round(byts / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 4),
                             "bytes_per_step": byts, "H_kv": Hk}
    del Kc, Vc
    c = synth.CONFIGS["G"]
    h, beta = synth.gate_inputs(c["B"], c["N"], c["H"], seed=c["seed"], device=dev)
    h, beta = h.bfloat16(), beta.bfloat16()
    for _ in range(3):
        gb.gfwa_gate_prefix(h, beta)
    torch.cuda.synchronize(dev)
    e0.record()
    for _ in range(n):
        gb.gfwa_gate_prefix(h, beta)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / n
    elems = c["B"] * c["N"] * c["H"]
    byts = elems * 8  # bf16 h, beta in; fp32 U out
    out["gate_scan_G"] = {"ms": round(ms, 4), "achieved_GBps": round(byts / (ms * 1e-3) / 1e9, 1),
                          "frac_hbm": round(byts / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 4),
                          "G_elems_per_s": round(elems / (ms * 1e-3) / 1e9, 2)}
    # the paper's preprocessing comparison on B200 --
    # the PyTorch two-kernel path (elementwise alpha, then cumsum), same inputs, same
    # fp32 U [B,H,N] output; a comparison baseline only, never on the product path
    import torch.nn.functional as F

    def two_kernel():
        a = F.softplus(beta.float() * h.float()) / (beta.float() + 1e-6)
        return -torch.cumsum(a.transpose(1, 2), dim=-1)

    for _ in range(3):
        two_kernel()
    torch.cuda.synchronize(dev)
    e0.record()
    for _ in range(n):
        two_kernel()
    e1.record()
    torch.cuda.synchronize(dev)
    ms2 = e0.elapsed_time(e1) / n
    # the paper's own two designs on B200 (C ABI comparison variants): 1-pass with one
    # program per head and an on-chip carry, Scan-Then-Propagate (App. E.1)
    var_ms = {}
    for v in (1, 2):
        for _ in range(3):
            gb.gfwa_gate_prefix_variant(v, h, beta)
        torch.cuda.synchronize(dev)
        e0.record()
        for _ in range(n):
            gb.gfwa_gate_prefix_variant(v, h, beta)
        e1.record()
        torch.cuda.synchronize(dev)
        var_ms[v] = e0.elapsed_time(e1) / n
    gel = lambda t: round(elems / (t * 1e-3) / 1e9, 2)  # noqa: E731  (b, t, h) elements/s, G
    out["gate_preproc_compare_G"] = {
        "pytorch_two_kernel_ms": round(ms2, 4), "one_program_per_head_ms": round(var_ms[1], 4),
        "scan_then_propagate_ms": round(var_ms[2], 4), "decoupled_lookback_ms": round(ms, 4),
        "G_elems_per_s": {"pytorch_two_kernel": gel(ms2), "one_program_per_head": gel(var_ms[1]),
                          "scan_then_propagate": gel(var_ms[2]), "decoupled_lookback": gel(ms)},
        "speedup_vs_pytorch": round(ms2 / ms, 2),
        "paper_context": ("A100 Triton: 1-pass 0.3 ms vs PyTorch 2.9 ms at N=64K (P:527); "
                          "1-pass ~28.5 vs Scan-Then-Propagate ~20.1 billion tokens/s (P:1061)")}
    out["attn_layer_epilogue_C2"] = _attn_layer_epilogue(dev)
    out["nsa_hybrid"] = _nsa_hybrid(dev)
    out["gqa_C2"] = _gqa_c2(dev, peaks)
    out["in_kernel_halo_C4_shard"] = _halo_c4_shard(dev)
    return out


def _gqa_c2(dev, peaks):
    """Grouped-query attention (gfwa_attn_desc_t.H_kv; the NSA configuration's GQA,
    P:1209-1211) at C2's query shape: H = 16 query heads over H_kv = 16 (MHA), 4, 1 K/V
    heads.  fwd (gfwa_fwd_train) + bwd (gfwa_bwd) per layer, inputs resident, eager;
    the in-window FLOPs are those of the 16 query heads whatever H_kv."""
    import torch

    import synth
    from paper_2512_07782_b200 import binding as gb

    c = synth.CONFIGS["C2"]
    s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
    Q, K, V, dO = synth.attn_inputs(s, seed=c["seed"], device=dev, dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=c["seed"], device=dev)
    U = gb.gfwa_gate_prefix(h, beta)
    fl = 14.0 * s.N * s.w * s.d * s.B * s.H
    res = {}
    for hkv in (s.H, 4, 1):
        Kg, Vg = K[:, :, :hkv].contiguous(), V[:, :, :hkv].contiguous()

        def step():
            O, LSE, Olo = gb.gfwa_fwd(Q, Kg, Vg, U, s.w, want_o_lo=True, prepare_bwd=True)
            gb.gfwa_bwd(Q, Kg, Vg, U, O, LSE, dO, s.w, O_lo=Olo, want_dalpha=False)

        for _ in range(3):
            step()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            step()
        e1.record()
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / 10
        res[f"H_kv={hkv}"] = {"ms": round(ms, 4), "tflops_in_window": round(fl / (ms * 1e-3) / 1e12, 1),
                              "pct_bf16_peak": round(fl / (ms * 1e-3) / 1e12 / peaks["bf16"], 4)}
        del Kg, Vg
    res["note"] = "C2 queries (B=8, H=16, N=4096, d=128, w=512), fwd+bwd eager, no dalpha scan"
    return res


def _halo_c4_shard(dev):
    """The in-kernel halo (gfwa_attn_desc_t.halo_rows, f3) at one rank's shape of the
    8-way sharded C4 step (S = 16384 query rows after a w = 2048 halo, H = 32, d = 128):
    fwd (gfwa_fwd_train) + bwd with the halo tiles TMA-loaded from a separate buffer (as
    from the previous rank's memory) vs the same call on one contiguous [halo; local]
    K / V -- the halo costs no copy and no extra time."""
    import torch

    import synth
    from paper_2512_07782_b200 import binding as gb

    c = synth.CONFIGS["C4"]
    w, S = c["w"], c["N"] // 8
    s = synth.AttnShape(B=c["B"], H=c["H"], N=S, d=c["d"], w=w, N_kv=S + w)
    Q, K, V, dO = synth.attn_inputs(s, seed=c["seed"], device=dev, dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, S + w, s.H, seed=c["seed"], device=dev)
    U = gb.gfwa_gate_prefix(h, beta)
    Kh, Vh = K[:, :w].clone(), V[:, :w].clone()
    res = {}
    for name, kv, halo in (("contiguous_ms", (K, V), None), ("kv_halo_ms", (K[:, w:], V[:, w:]), (Kh, Vh))):
        def step():
            O, LSE, Olo = gb.gfwa_fwd(Q, kv[0], kv[1], U, w, want_o_lo=True, prepare_bwd=True, kv_halo=halo)
            gb.gfwa_bwd(Q, kv[0], kv[1], U, O, LSE, dO, w, O_lo=Olo, want_dalpha=False, kv_halo=halo)

        for _ in range(3):
            step()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            step()
        e1.record()
        torch.cuda.synchronize(dev)
        res[name] = round(e0.elapsed_time(e1) / 5, 4)
    res["config"] = f"B=1, H={s.H}, S={S} query rows + {w}-row halo, d={s.d}, w={w}, fwd+bwd eager"
    return res


def _attn_layer_epilogue(dev):
    """the AttnLayer output epilogue (reading C-27: per-head
    RMSNorm with weight gamma, then the swish gate) at C2, fused into the attention
    kernels (gfwa_fwd_normgate + gfwa_bwd_normgate) vs the same math as separate
    PyTorch ops around gfwa_fwd_train / gfwa_bwd (rms_norm * silu, autograd for its
    backward).  Both: fwd + bwd of the layer from dY, inputs resident, eager."""
    import torch
    import torch.nn.functional as F

    import synth
    from paper_2512_07782_b200 import binding as gb

    c = synth.CONFIGS["C2"]
    s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
    Q, K, V, dY = synth.attn_inputs(s, seed=c["seed"], device=dev, dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=c["seed"], device=dev)
    U = gb.gfwa_gate_prefix(h, beta)
    g = torch.randn(s.B, s.N, s.H, s.d, device=dev).to(torch.bfloat16)
    gamma = torch.ones(s.d, device=dev)

    def fused():
        Y, O, LSE, Olo, rstd = gb.gfwa_fwd_normgate(Q, K, V, U, g, gamma, s.w, prepare_bwd=True)
        gb.gfwa_bwd_normgate(Q, K, V, U, O, LSE, g, gamma, rstd, dY, s.w, O_lo=Olo, want_dalpha=False)

    def unfused():
        O, LSE, Olo = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True, prepare_bwd=True)
        Ot = O.detach().requires_grad_(True)
        gt = g.detach().requires_grad_(True)
        gm = gamma.detach().requires_grad_(True)
        Y = F.rms_norm(Ot, (s.d,), weight=gm, eps=1e-5) * F.silu(gt)
        Y.backward(dY)
        gb.gfwa_bwd(Q, K, V, U, O, LSE, Ot.grad, s.w, O_lo=Olo, want_dalpha=False)

    res = {}
    for name, fn in (("fused_ms", fused), ("unfused_torch_ms", unfused)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize(dev)
        res[name] = round(e0.elapsed_time(e1) / 10, 4)
    res["speedup"] = round(res["unfused_torch_ms"] / res["fused_ms"], 3)
    res["note"] = "layer fwd+bwd from dY at C2, eager; epilogue = RMSNorm(gamma) * swish(g) per head (C-27)"
    return res


def _nsa_hybrid(dev):
    """the NSA hybrid with GatedFWA as the local branch (App. B; the
    paper's NSA settings block 64, 16 selected blocks) at B=2, H=16,
    N=4096, d=128, w=512: fwd and fwd+bwd time against the GatedFWA branch alone
    (gfwa_fwd_train + gfwa_bwd), eager.  The compressed and selected branches are
    CUDA-core kernels (the selected branch's dK/dV by fp32 atomics)."""
    import torch

    import synth
    from paper_2512_07782_b200 import binding as gb

    s = synth.AttnShape(B=2, H=16, N=4096, d=128, w=512)
    Q, K, V, dO = synth.attn_inputs(s, seed=77, device=dev, dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=78, device=dev)
    U = gb.gfwa_gate_prefix(h, beta)
    gates = torch.randn(s.B, s.N, s.H, 3, device=dev)

    def t(fn, n=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize(dev)
        return round(e0.elapsed_time(e1) / n, 4)

    O, sv = gb.gfwa_nsa_fwd(Q, K, V, U, gates, s.w, block=64, n_sel=16)
    fwd = t(lambda: gb.gfwa_nsa_fwd(Q, K, V, U, gates, s.w, block=64, n_sel=16))
    both = t(lambda: gb.gfwa_nsa_bwd(Q, K, V, U, gates, dO, gb.gfwa_nsa_fwd(Q, K, V, U, gates, s.w, 64, 16)[1], s.w,
                                     64, 16))

    def local():
        O2, L2, Ol2 = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True, prepare_bwd=True)
        gb.gfwa_bwd(Q, K, V, U, O2, L2, dO, s.w, O_lo=Ol2, want_dalpha=False)

    return {"config": "B=2, H=16, N=4096, d=128, w=512, block=64, n_sel=16", "nsa_fwd_ms": fwd,
            "nsa_fwd_bwd_ms": both, "gatedfwa_local_fwd_bwd_ms": t(local),
            "tokens_per_s_fwd_bwd": round(s.B * s.N / (both * 1e-3), 1)}


# --------------------------------------------------------------------------- CPU oracle


def _oracle_sample(s, n_slices: int, n_rows: int, halo: int = 0):
    """A bounded sample of the workload for the fp64 oracle: `n_slices` (b,h)
    slices, each `n_rows` query tokens of one head (same recipe/seed) after
    `halo` key rows (halo = w - 1: every sampled query sees a full window)."""
    import torch

    import synth

    sub = synth.AttnShape(B=n_slices, H=1, N=n_rows, d=s.d, w=s.w, N_kv=n_rows + halo)
    Q, K, V, dO = synth.attn_inputs(sub, seed=4242, dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(n_slices, n_rows + halo, 1, seed=4243)
    return sub, Q, K, V, dO, h.bfloat16(), beta.bfloat16()


def _oracle_step(sub, Q, K, V, dO, h, beta):
    import oracle

    U, _, _ = oracle.gate_prefix_hbeta(h, beta)
    oracle.fwd(Q, K, V, U, sub.w)
    g = oracle.bwd(Q, K, V, U, dO, sub.w)
    oracle.gate_chain(h, beta, g["dalpha"])


def cpu_baseline(args, s):
    import oracle

    cores = oracle.num_threads()
    # bounded sample: grow the number of (b, h) slices (full N each) until the
    # fp64 oracle has run for >= 10 s of wall time or the whole workload is done
    n_rows = s.N
    slices, dt, done = cores, 0.0, 0
    while True:
        sub, *arrs = _oracle_sample(s, slices, n_rows)
        t = time.perf_counter()
        _oracle_step(sub, *arrs)
        dt = time.perf_counter() - t
        done = slices
        if dt >= 10.0 or slices >= s.B * s.H:
            break
        slices = min(s.B * s.H, max(slices * 2, int(slices * 10.0 / max(dt, 1e-3))))
    # one full token = H heads; the sample covers done*n_rows head-rows
    tok_equiv = done * n_rows / s.H
    return {"value": round(tok_equiv / dt, 3), "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "sample": f"{done} of {s.B * s.H} (b,h) slices x all {n_rows} tokens of {args.workload} (fp64 C oracle: "
                      f"gate, fwd, bwd, gate chain), {dt:.2f} s; tokens = head-rows / H"}


def run_reference(args):
    """--impl reference: the fp64 CPU oracle, as it stands, on host cores."""
    import synth

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    # torchrun exports OMP_NUM_THREADS=1; the oracle runs on all of this host's cores
    oracle.set_num_threads(len(os.sched_getaffinity(0)))

    # the config our arm reports: at N > 1 the default run's headline is the
    # sequence-sharded C4 step (run_ours), so the reference times C4 too
    wl = args.workload
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 and wl == "C2":
        wl = "C4"
    c = synth.CONFIGS[wl]
    s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
    cores = oracle.num_threads()
    if wl == "C4":
        # C4 rows all see full 2048-key windows (but the first 2047 of 131072): each
        # step takes `cores` slices of 1024 query rows after a w-1 key-row halo
        n_rows, halo = 1024, s.w - 1
        what = f"{n_rows} query rows after a {halo}-row key halo (full windows) of {wl}"
    else:
        # `cores` (b, h) slices over ALL N tokens of the workload (the full window mix)
        n_rows, halo = s.N, 0
        what = f"all {n_rows} tokens of {wl}"
    sub, *arrs = _oracle_sample(s, cores, n_rows, halo)
    for _ in range(args.warmup):
        _oracle_step(sub, *arrs)
    t = time.perf_counter()
    for _ in range(args.steps):
        _oracle_step(sub, *arrs)
    dt = (time.perf_counter() - t) / args.steps
    tok = cores * n_rows / s.H
    value = tok / dt
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "tokens/s", "n_gpus": args.gpus,
        "device": "host CPU (fp64 oracle; rank 0 only)",
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
        "scaling": "strong" if wl == "C4" else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (synth.py)",
        "config": {"workload": wl, "B": s.B, "H": s.H, "N": s.N, "d": s.d, "w": s.w},
        "cpu_baseline": {"value": round(value, 3), "unit": "tokens/s", "cores": cores, "kind": "oracle",
                         "sample": f"per step {cores} (b,h) slices x {what}; tokens = head-rows/H"},
        "e2e": {"value": round(value, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C2", choices=["C2", "C3_w128", "C3_w512", "C3_w2048", "C4"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle baseline")
    ap.add_argument("--no-aux", action="store_true", help="skip decode/gate-probe line items")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of a CUDA-graph replay")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ws = os.environ.get("WORLD_SIZE")
    if ws is None and args.gpus > 1:
        # `bench.py --gpus N` outside torchrun: launch the N ranks ourselves (one
        # process per GPU, the same command the driver uses)
        import socket

        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if ws is not None and int(ws) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_seq(args) if args.workload == "C4" else run_ours(args)


if __name__ == "__main__":
    main()
