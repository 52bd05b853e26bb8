#!/usr/bin/env python
"""Draft+verify round throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], the metric's 1-GPU configuration): the
seven ResNet-50 conv2d subgraphs, 65,536 random candidates per subgraph
round per GPU -> SA draft -> dedup top-512 -> PaCM verify (h = 64,
random-init weights) -> select b = 10. PaCM runs in fp64 on the CUDA cores
(scores within 1e-12 of the reference; the default, as fast as the tensor
path at K = 512 and exact); `--precision bf16` runs it on the tcgen05 tensor
cores (bf16 operands, fp32 TMEM accumulators) with certified selection (the
boundary band rescored in fp64, so the selected set equals the reference's).
The other precision is reported under `other_precision`. One step = one round on each
of the seven subgraphs. For N > 1 every rank drafts its own 65,536 candidates of
the same counter-based population (weak scaling); the per-rank top-512
lists (cost, global index, identity) are merged after one NCCL all-gather
and verified on every rank.

value: candidates scored / s with the population already resident in HBM.
e2e:   the same through the public API from host memory: every round
       uploads its candidates (64-bit schedule identities, decoded on the
       device) from pinned memory, the PaCM weights once per step, and reads
       the selection back.
Only rank 0 prints the JSON line. `--impl reference` times the unmodified
reference (oracle/_ref, compiled from /root/reference) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidates scored/sec per draft+verify round (1/2/4/8 B200) vs host-CPU ref"
UNIT = "candidates/s"
R50 = ["r50_stem", "r50_c1x1_64", "r50_c3x3_64", "r50_c1x1_256", "r50_c3x3_128", "r50_c3x3_256", "r50_c3x3_512"]
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.proc, self.path = gpu, None, None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) >= 7 and f[0].replace(".", "").isdigit():
                    rows.append(f)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() in ("active", "1")})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


# ----------------------------------------------------------------------------------------- ours --

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2402_02361_b200 import tiletune as tt
    from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device

    torch.cuda.set_device(local_rank)
    dev = reference_device()
    ctx = tt.Context(local_rank)
    n, k, b, seed = args.n, args.k, args.b, args.seed
    prec = tt.TT_PREC_BF16 if args.precision == "bf16" else tt.TT_PREC_FP64
    names = R50 if args.workload == "r50" else [args.workload]
    sketches = [make_sketch(WORKLOADS[w]()) for w in names]
    first = rank * n
    # inputs: each subgraph's population shard, resident in HBM, + pinned host copies for e2e
    pops, ids = zip(*[tt.random_init(ctx, sk, n, seed, first=first, with_identity=True) for sk in sketches])
    pops, ids = list(pops), list(ids)
    # e2e inputs in host memory: each candidate as its exact 64-bit schedule
    # identity (the integer replacement of schedule_key), 8 B per candidate
    ids_host = [x.cpu().pin_memory() for x in ids]
    params = tt.init_params(64, derive_seed(seed, TAG_INIT))
    params_host = torch.from_numpy(params).pin_memory()
    model = tt.PaCM(ctx, params_host, 64)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    gather_out = torch.empty((3, k), dtype=torch.int64, device="cuda")
    gathered = torch.empty((world * 3 * k,), dtype=torch.int64, device="cuda")

    def one_round(sk, soa, seed_=0):
        if world == 1:
            tt.round_async(ctx, sk, dev, n, k, b, seed=seed_, soa=soa, precision=prec, band=args.band, first=first)
        else:
            tt.round_local_async(ctx, sk, dev, n, k, b, first, gather_out, seed=seed_, soa=soa)
            dist.all_gather_into_tensor(gathered, gather_out.reshape(-1))
            tt.round_finish_merged_async(ctx, sk, dev, gathered, n * world, k, b, precision=prec, band=args.band)

    # rounds pipelined through the context's record ring: round r is enqueued, then
    # round r-1's selection is read back while r runs (at most two in flight)
    inflight = {"n": 0, "retries": 0, "rounds": 0}

    def collect_lagged(c=None, keep=1):
        c = c or ctx
        while inflight["n"] > keep:
            out_ = tt.round_collect(c, b)
            assert out_.selected == b and (out_.status & 0xff) == 0, out_
            inflight["n"] -= 1
            inflight["retries"] += out_.retries
            inflight["rounds"] += 1

    def step_value():
        for sk, soa in zip(sketches, pops):
            one_round(sk, soa)
            inflight["n"] += 1
            collect_lagged()

    # warm-up + correctness gate: every subgraph's round must collect cleanly
    for _ in range(args.warmup):
        for sk, soa in zip(sketches, pops):
            one_round(sk, soa)
            out = tt.round_collect(ctx, b)
            assert out.selected == b and out.status == 0, out
    torch.cuda.synchronize()

    def drain():
        # collect every round still in flight on the context (oldest first)
        collect_lagged(keep=0)
        inflight["n"] = 0
        while True:
            try:
                tt.round_collect(ctx, b)
            except tt.TTError:
                return

    def timed(step_fn, profile=False):
        for _ in range(2):  # untimed: the step's round graphs are captured on their second use
            step_fn()
        torch.cuda.synchronize()
        drain()
        if profile:
            tt.profile_enable(ctx, True)
            tt.profile_read(ctx)
        times = []
        launches0 = tt.kernel_launches()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations, outside the events
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step_fn()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        launches = tt.kernel_launches() - launches0
        prof = tt.profile_read(ctx) if profile else None
        if profile:
            tt.profile_enable(ctx, False)
        return times, launches, prof

    # ---- value: population resident in HBM
    with ClockSampler(local_rank) as clk:
        times, launches, _ = timed(step_value)
    clocks = clk.summary()
    drain()

    # ---- stage breakdown (separate pass, events per stage on the ctx stream)
    ptimes, _, prof = timed(step_value, profile=True)
    drain()

    # ---- e2e through the public API from host memory
    # H2D of the next subgraph's population (pinned -> its own device buffer)
    # runs on a copy stream while the current round computes
    copy_stream = torch.cuda.Stream()
    ev_copy = [torch.cuda.Event() for _ in sketches]
    # decode (identities -> factor columns) on a second context's stream, so the next
    # subgraph's upload + decode overlap the current round
    ctx_dec = tt.Context(local_rank, use_torch_stream=False)
    dec_stream = torch.cuda.ExternalStream(ctx_dec.stream_handle())
    ev_dec = [torch.cuda.Event() for _ in sketches]

    def prep(r, sk):
        with torch.cuda.stream(copy_stream):
            ids[r].copy_(ids_host[r], non_blocking=True)
            ev_copy[r].record(copy_stream)
        dec_stream.wait_event(ev_copy[r])
        tt.schedule_from_identity(ctx_dec, sk, ids[r], out=pops[r])
        ev_dec[r].record(dec_stream)

    def step_e2e():
        # every stream's work of the step starts after the step's start event
        ev_start = torch.cuda.Event()
        ev_start.record(stream)
        copy_stream.wait_event(ev_start)
        dec_stream.wait_event(ev_start)
        # rounds pipelined through the context's ring: round r is enqueued, then round r-1's
        # selection is read back while r runs; subgraph r+1's upload and decode overlap round r;
        # the step ends with every selection on the host
        prep(0, sketches[0])
        model.load(params_host)                     # H2D PaCM weights (pinned, async), once per step
        for r, sk in enumerate(sketches):
            if r + 1 < len(sketches):
                prep(r + 1, sketches[r + 1])
            stream.wait_event(ev_dec[r])
            one_round(sk, pops[r])
            if r > 0:
                out_e = tt.round_collect(ctx, b)
                assert out_e.selected == b
        out_e = tt.round_collect(ctx, b)
        assert out_e.selected == b
    etimes, elaunch, _ = timed(step_e2e)
    h2d = sum(x.numel() * 8 for x in ids_host) + params_host.numel() * 8
    d2h = len(sketches) * 8 * (7 + 4 * b)  # each round record, written by its finishing kernel into mapped pinned memory

    # ---- e2e with the candidates uploaded in the SoA factor layout itself (int32 columns,
    # 4 B per factor: 76 B per conv candidate) instead of 8-byte identities: no decode step
    pops_host = [p_.cpu().pin_memory() for p_ in pops]
    ev_soa = [torch.cuda.Event() for _ in sketches]

    def prep_soa(r):
        with torch.cuda.stream(copy_stream):
            pops[r].copy_(pops_host[r], non_blocking=True)
            ev_soa[r].record(copy_stream)

    def step_e2e_soa():
        ev_start = torch.cuda.Event()
        ev_start.record(stream)
        copy_stream.wait_event(ev_start)
        prep_soa(0)
        model.load(params_host)
        for r, sk in enumerate(sketches):
            if r + 1 < len(sketches):
                prep_soa(r + 1)
            stream.wait_event(ev_soa[r])
            one_round(sk, pops[r])
            if r > 0:
                assert tt.round_collect(ctx, b).selected == b
        assert tt.round_collect(ctx, b).selected == b
    sotimes, _, _ = timed(step_e2e_soa)
    h2d_soa = sum(x.numel() * 4 for x in pops_host) + params_host.numel() * 8

    # ---- e2e, seeded API (explore(seed) semantics: population drawn inside the call)
    def step_seeded():
        model.load(params_host)
        for r, sk in enumerate(sketches):
            one_round(sk, None, seed)
            if r > 0:
                tt.round_collect(ctx, b)
        tt.round_collect(ctx, b)
    stimes, _, _ = timed(step_seeded)

    def agg(ts):
        t = torch.tensor([sum(ts)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()) / 1e3  # seconds over all steps (max over ranks)

    # ---- the other PaCM arithmetic (bf16 tcgen05 + certified selection <-> fp64 CUDA cores)
    alt = tt.TT_PREC_FP64 if prec == tt.TT_PREC_BF16 else tt.TT_PREC_BF16
    prec_main = prec

    def step_alt():
        for sk, soa in zip(sketches, pops):
            if world == 1:
                tt.round_async(ctx, sk, dev, n, k, b, soa=soa, precision=alt, band=args.band, first=first)
            else:
                tt.round_local_async(ctx, sk, dev, n, k, b, first, gather_out, soa=soa)
                dist.all_gather_into_tensor(gathered, gather_out.reshape(-1))
                tt.round_finish_merged_async(ctx, sk, dev, gathered, n * world, k, b, precision=alt, band=args.band)
            inflight["n"] += 1
            collect_lagged()
    for _ in range(2):
        step_alt()
    drain()
    atimes, _, aprof = timed(step_alt, profile=True)
    drain()

    # ---- the step's subgraph rounds concurrently: one context (own stream) per subgraph.
    # Rounds of different tasks are independent given fixed weights; each round alone
    # occupies few SMs, so a tuner that batches its task-scheduler epoch runs them side by side.
    conc = None
    if world == 1 and len(sketches) > 1:
        cctx = [tt.Context(local_rank, use_torch_stream=False) for _ in sketches]
        for c_ in cctx:
            tt.PaCM(c_, params_host, 64)
        cstreams = [torch.cuda.ExternalStream(c_.stream_handle()) for c_ in cctx]

        def step_conc():
            for c_ in cctx:  # the previous step's rounds (complete: the step ended with a sync)
                if c_._inflight:
                    tt.round_collect(c_, b)
            e_start = torch.cuda.Event()
            e_start.record(stream)
            for c_, cs, sk, soa in zip(cctx, cstreams, sketches, pops):
                cs.wait_event(e_start)
                tt.round_async(c_, sk, dev, n, k, b, soa=soa, precision=prec, band=args.band, first=first)
            for cs in cstreams:
                e_done = torch.cuda.Event()
                e_done.record(cs)
                stream.wait_event(e_done)
        for _ in range(2):
            step_conc()
            torch.cuda.synchronize()
        ctimes, _, _ = timed(step_conc)
        for c_ in cctx:
            out_c = tt.round_collect(c_, b)
            assert out_c.selected == b
        conc = agg(ctimes)
        for c_ in cctx:
            c_.close()

    b1m = None if args.no_bert else bert_1m(args, ctx, dev, params_host, rank, world, stream, flush)
    tot, etot, stot, atot, sotot = agg(times), agg(etimes), agg(stimes), agg(atimes), agg(sotimes)
    cands = n * world * len(sketches) * args.steps
    result = None
    if rank == 0:
        peaks, peaks_kind = load_peaks()
        rounds = len(sketches) * args.steps
        stage_ms = {s: v[0] / max(v[1], 1) for s, v in (prof or {}).items()}
        roof = roofline(args, sketches, stage_ms, rounds, peaks, peaks_kind, prec)
        cpu = cpu_baseline(args) if (world == 1 and not args.no_cpu) else None
        parity = parity_check(args, ctx, dev, sketches, names, pops, params, prec) if world == 1 else None
        ga = explore_ga(args, ctx, dev, sketches, names) if (world == 1 and not args.no_explore) else None
        result = {
            "metric": METRIC, "value": cands / tot, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64" if prec == tt.TT_PREC_FP64 else "bf16+f64",
            "data": "synthetic: random_init(seed=%d) populations, init_params(64) weights" % seed,
            "config": {"workload": f"{args.workload}: {len(sketches)} subgraph rounds/step, N={n}/GPU/round, "
                                   f"K={k}, b={b}, h=64, precision={args.precision}",
                       "subgraphs": names, "n_per_gpu": n, "k": k, "b": b,
                       "l2": "flushed (256 MiB write) between timed steps",
                       "parallelism": f"dp{world} (population sharded, NCCL all-gather top-K merge)"},
            "e2e": {"value": cands / etot, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "tt_schedule_from_identity + tt_round_async / tt_round_collect: candidates as "
                           "exact 64-bit schedule identities (every round) and PaCM weights (once per step) "
                           "from pinned host memory, the next subgraph's upload overlapped on a copy stream, "
                           "every round's selection read back (round r-1's while round r runs); identities "
                           "decoded on a second context's stream, overlapping the previous round"},
            "e2e_soa": {"value": cands / sotot, "unit": UNIT, "h2d_bytes_per_step": h2d_soa,
                        "d2h_bytes_per_step": d2h,
                        "api": "tt_round_async / tt_round_collect with the population uploaded every round in the "
                               "SoA factor layout (int32 columns, 4 B per factor) from pinned host memory, the next "
                               "subgraph's upload overlapped on a copy stream; no identity decode"},
            "e2e_seeded": {"value": cands / stot, "unit": UNIT,
                           "h2d_bytes_per_step": params_host.numel() * 8, "d2h_bytes_per_step": d2h,
                           "api": "explore(seed) semantics: population drawn on device inside the call"},
            "other_precision": {
                "precision": "bf16 tcgen05 + certified selection" if alt else "fp64 CUDA cores",
                "value": cands / atot, "unit": UNIT,
                "stage_ms_per_round": {s_: v[0] / max(v[1], 1) for s_, v in (aprof or {}).items()},
                "roofline": roofline(args, sketches, {s_: v[0] / max(v[1], 1) for s_, v in (aprof or {}).items()},
                                     len(sketches) * args.steps, peaks, peaks_kind, alt)},
            "concurrent_subgraphs": None if conc is None else {
                "value": cands / conc, "unit": UNIT,
                "note": "the step's 7 subgraph rounds on 7 contexts/streams at once (independent tasks, "
                        "fixed weights); the headline `value` runs them one after another"},
            "explore_ga": ga,
            "bert_1m": b1m,
            "parity": parity,
            "gpu_launches": launches,
            "selector_retries": {"retries": inflight["retries"], "rounds": inflight["rounds"],
                                 "note": "device-side threshold retries (re-thresholding the costs already in "
                                         "HBM, never K1) + host re-runs, summed over every collected round"},
            "stage_ms_per_round": stage_ms,
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clocks,
        }
    return result


BERT = ["bert_qkv", "bert_proj", "bert_ffn1", "bert_ffn2", "bert_bmm_qk", "bert_bmm_pv"]


def bert_1m(args, ctx, dev, params_host, rank, world, stream, flush):
    """BASELINE configs[2]: the six BERT-base subgraphs, 1,048,576 candidates
    per subgraph round in total, strong-sharded by index range over the N
    ranks: local K1 + selector on each shard -> one NCCL
    all-gather of the [3, K] (cost, global index, identity) payloads ->
    merge + PaCM verify + select_top on every rank. Populations resident in
    HBM (each rank its shard), L2 flushed between steps, CUDA events, max over
    ranks. Also times one profiled step per stage (local draft, all-gather,
    merge + verify) on the context stream."""
    import torch
    import torch.distributed as dist

    from paper_2402_02361_b200 import tiletune as tt
    from paper_2402_02361_b200.sharded import shard_range
    from paper_2402_02361_b200.types import WORKLOADS, make_sketch
    n_total, k, b, seed = args.bert_n, args.k, args.b, args.seed
    first, n_loc = shard_range(n_total, rank, world)
    sks = [make_sketch(WORKLOADS[w]()) for w in BERT]
    pops = [tt.random_init(ctx, sk, n_loc, seed, first=first) for sk in sks]
    payload = torch.empty((3, k), dtype=torch.int64, device="cuda")
    gathered = torch.empty((world * 3 * k,), dtype=torch.int64, device="cuda")
    sels = []

    def one(sk, soa, ev=None):
        if world == 1:
            tt.round_async(ctx, sk, dev, n_total, k, b, soa=soa, first=first)
            return
        tt.round_local_async(ctx, sk, dev, n_loc, k, b, first, payload, soa=soa)
        if ev:
            ev[0].record(stream)
        dist.all_gather_into_tensor(gathered, payload.reshape(-1))
        if ev:
            ev[1].record(stream)
        tt.round_finish_merged_async(ctx, sk, dev, gathered, n_total, k, b)

    def step(keep=False, evs=None):
        for i, (sk, soa) in enumerate(zip(sks, pops)):
            one(sk, soa, None if evs is None else evs[i])
            out = tt.round_collect(ctx, b)
            if keep:
                sels.append(out.index.tolist())

    step(keep=True)  # warm-up, and the selections (checked against N = 1 by the caller's tests)
    for _ in range(max(args.warmup - 1, 2)):
        step()
    torch.cuda.synchronize()
    times = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    t = torch.tensor([sum(times)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot = float(t.item()) / 1e3
    stages = None
    if world > 1:  # one profiled step: local draft | all-gather | merge + verify + select, per round
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in sks]
        starts, ends = [], []
        for i, (sk, soa) in enumerate(zip(sks, pops)):
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            one(sk, soa, evs[i])
            s1.record(stream)
            tt.round_collect(ctx, b)
            starts.append(s0), ends.append(s1)
        torch.cuda.synchronize()
        loc = [starts[i].elapsed_time(evs[i][0]) for i in range(len(sks))]
        ag = [evs[i][0].elapsed_time(evs[i][1]) for i in range(len(sks))]
        mg = [evs[i][1].elapsed_time(ends[i]) for i in range(len(sks))]
        stages = {"local_draft_us": 1e3 * sum(loc) / len(loc), "all_gather_us": 1e3 * sum(ag) / len(ag),
                  "merge_verify_us": 1e3 * sum(mg) / len(mg)}
    cands = n_total * len(sks) * args.steps
    info = {"value": cands / tot, "unit": UNIT, "ms_per_step": 1e3 * tot / args.steps, "scaling": "strong",
            "config": f"BASELINE configs[2]: {len(sks)} BERT-base subgraph rounds/step, N={n_total} candidates per "
                      f"round in total sharded over {world} GPU(s) ({n_loc} on rank {rank}), K={k}, b={b}, h=64, fp64",
            "subgraphs": BERT, "selections_first_step": sels, "stage_us_per_round": stages}
    if world > 1:
        info["collective"] = {"backend": dist.get_backend(), "nranks": world,
                              "nccl_version": ".".join(str(v) for v in torch.cuda.nccl.version()),
                              "payload_bytes_per_rank": 3 * k * 8}
    return info


def parity_check(args, ctx, dev, sketches, names, pops, params, prec):
    """Outside the timed region: one round per benchmarked subgraph on the
    bench's own resident population, checked against the C oracle
    (oracle/_build, test infrastructure) on the same seeded inputs: drafted
    top-K, PaCM fp64 scores and the selection."""
    from paper_2402_02361_b200 import tiletune as tt
    R = _ref_setup(args)
    rows, ok = {}, True
    for name, sk, soa in zip(names, sketches, pops):
        out = tt.draft_verify_round(ctx, sk, dev, args.n, args.k, args.b, soa=soa, precision=prec, band=args.band)
        pop = R.O_random_init(sk, args.seed, args.n)
        cost = R.O_draft_cost(sk, dev, pop)
        idx, dc = R.O_draft_topk(sk, cost, pop, args.k)
        st, bl = R.O_features(sk, dev, pop, idx)
        sc = R.O_score(params, 64, st, bl)
        sel = R.O_select_top(sc, dc, None, args.b)
        same = bool((out.index == idx[sel]).all()) and bool((out.cost.view(np.uint64) == dc[sel].view(np.uint64)).all())
        err = float(np.abs(out.score - sc[sel]).max())
        rows[name] = {"identical_selection": same, "max_abs_score_err": err}
        ok = ok and same
    return {"checked": "one round per subgraph vs the C oracle (oracle/tt_oracle.c), same seeded population",
            "all_identical": ok, "subgraphs": rows}


FLOP_PER_CAND = 320640  # PaCM forward at h = 64, S = 6, B = 8


def _traffic():
    """dram read+write bytes per launch from the committed ncu capture (profiles/), or {}."""
    p = os.path.join(ROOT, "profiles", "r02_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def roofline(args, sketches, stage_ms, rounds, peaks, peaks_kind, prec):
    """Roofline of the round's dominant kernel from live CUDA-event timings
    (per launch, on the context stream), plus the other hot kernels."""
    if not stage_ms:
        return None
    traffic = _traffic()
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    out = {}
    if "draft_cost" in stage_ms:
        # K1: factor columns read (unroll column not read) + fp64 cost written, per candidate
        per = [4 * (4 * sk.op.n_spatial + 3 * sk.op.n_reduction) + 8 for sk in sketches]
        byts = args.n * sum(per) / len(per)
        ms = stage_ms["draft_cost"]
        ach = byts / (ms * 1e-3) / 1e9
        out["draft_cost"] = {"bound": "hbm", "kernel": "k_fsel (K1 SA draft cost inside the fused selector)",
                             "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                             "frac": ach / peaks["hbm_gbs"], "traffic": traffic.get("k_fsel"),
                             "algorithmic_bytes": byts, "ms": ms, "peak_source": peaks_kind}
    if "pacm_kernel" in stage_ms:
        ms = stage_ms["pacm_kernel"]
        ach = args.k * FLOP_PER_CAND / (ms * 1e-3) / 1e12
        if prec:
            peak = peaks["bf16_tflops"]
            out["pacm_kernel"] = {"bound": "tensor", "kernel": "k_pacm_tc (tcgen05 bf16, TMEM accumulators)",
                                  "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                                  "traffic": traffic.get("k_pacm_tc"), "flop_per_candidate": FLOP_PER_CAND,
                                  "ms": ms, "peak_source": peaks_kind + " bf16 dense (burst)"}
        else:
            # CUDA-core fp64: 64 fp64 lanes/clk/SM measured (tools/fp64_bench.cu); the dense layers
            # use DFMA (2 FLOP per lane-op), so the peak is the FMA rate
            peak = 2 * 64 * 148 * sm_mhz * 1e6 / 1e12
            out["pacm_kernel"] = {"bound": "fp64",
                                  "kernel": "k_verify64 (drafted-set features + fp64 PaCM on CUDA cores in the "
                                            "reference's order, DFMA dense layers, + the round's finish; "
                                            "PaCM FLOPs counted)",
                                  "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                                  "traffic": traffic.get("k_verify64"), "flop_per_candidate": FLOP_PER_CAND,
                                  "ms": ms, "peak_source": "measured fp64 lane rate x 2 (FMA) x 148 SMs x max SM clock"}
    if not out:
        return None
    dom = max(out, key=lambda k: out[k]["ms"])
    res = dict(out[dom])
    res["others"] = {k: v for k, v in out.items() if k != dom}
    return res


def explore_ga(args, ctx, dev, sketches, names, reps=5):
    """the tuner's real explore — the LSE genetic loop at
    TunerConfig defaults (n_steps 32, pop_size 512, draft_size 512) — through
    tt_explore (host call, results on the host), beside the reference's own
    explore() (oracle/_ref, all host threads) on the same seeds."""
    from paper_2402_02361_b200 import tiletune as tt
    R = None if args.no_cpu else _ref_setup(args)
    threads = os.cpu_count() or 1
    rows = {}
    for name, sk in list(zip(names, sketches))[:2]:
        tt.explore(ctx, sk, dev, 32, 512, 512, 1)
        t0 = time.perf_counter()
        for r in range(reps):  # schedules returned as exact identities + draft costs
            _, c_r, _, ev = tt.explore(ctx, sk, dev, 32, 512, 512, 1000 + r, with_soa=False)
            cost = c_r if r == 0 else cost
        g = (time.perf_counter() - t0) / reps
        row = {"ms_per_explore": 1e3 * g, "evaluations_per_s": ev / g}
        if R is not None and R.ref_available():
            t0 = time.perf_counter()
            for r in range(3):
                _, rc_r = R.R_explore(sk, dev, 512, 512, 1000 + r, n_steps=32, threads=threads)
                rc = rc_r if r == 0 else rc
            c = (time.perf_counter() - t0) / 3
            row.update({"reference_ms_per_explore": 1e3 * c, "reference_threads": threads,
                        "identical_to_reference_seed_1000": bool(len(rc) == len(cost) and (rc == cost).all())})
        row["tuner_round"] = tuner_round(R, ctx, sk, dev, threads, reps)
        rows[name] = row
    return {"config": "explore(op, dev, n_steps=32, draft_size=512, pop_size=512): TunerConfig defaults "
                      "(tuner.hpp:38-40); wall clock of the host call, drafted schedules returned as exact "
                      "64-bit identities + draft costs", "subgraphs": rows}


def tuner_round(R, ctx, sk, dev, threads, reps):
    """The tuner's whole real round at TunerConfig defaults (tuner.cpp:294-384: GA draft set with
    random_mix 0.2 -> features -> PaCM fp64 -> select_top(10)) through the public API (tt_tuner_round:
    host in, host out, one call), beside the reference's own functions composed the same way
    (oracle/_ref ref_tuner_round)."""
    import ctypes as C

    from paper_2402_02361_b200 import tiletune as tt
    from paper_2402_02361_b200.types import TAG_INIT, derive_seed
    params = tt.init_params(64, derive_seed(5, TAG_INIT))
    tt.PaCM(ctx, params, 64)

    def ours(seed):
        return tt.tuner_round(ctx, sk, dev, 32, 512, 512, 0.2, seed, seed + 1, 10, tt.TT_PREC_FP64)[0]
    ours(7)
    t0 = time.perf_counter()
    for r in range(reps):
        sel = ours(2000 + r)
        first = sel if r == 0 else first
    g = (time.perf_counter() - t0) / reps
    row = {"ms_per_round": 1e3 * g}
    if R is not None and R.ref_available():
        f = R.ref().ref_tuner_round
        f.restype = C.c_int
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.c_uint64,
                      C.c_int64, R.f64p, C.c_int, C.c_int, R.i64p, R.f64p, R.i64p, R.f64p]
        t0 = time.perf_counter()
        for r in range(3):
            sel_r, ncand, secs = np.zeros(10, np.int64), C.c_int64(0), np.zeros(2)
            R.check(f(C.byref(sk), C.byref(dev), 32, 512, 512, 0.2, 2000 + r, 2001 + r, 10, R.ptr(params, R.f64p), 64,
                      threads, R.ptr(sel_r, R.i64p), None, C.byref(ncand), R.ptr(secs, R.f64p)))
            first_r = sel_r.copy() if r == 0 else first_r
        c = (time.perf_counter() - t0) / 3
        row.update({"reference_ms_per_round": 1e3 * c, "identical_selection_seed_2000": bool((first_r == first).all())})
    return row


# ------------------------------------------------------------------------------------ reference --

def _ref_setup(args):
    from tests import _refs as R  # checker loader: oracle/_ref (the reference compiled here)
    return R


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def strict_round(R, workload, n, k, b, seed, threads):
    """The strict CPU bound of one round (oracle/_ref ref_round_strict): the reference's own
    draft_cost / extract_features / score_batch / select_top over the resident population,
    parallel_for + nth_element top-K, no string keys. Returns seconds (population given)."""
    import ctypes as C
    from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device
    sk = make_sketch(WORKLOADS[workload]())
    dev = reference_device()
    params = R.R_init_params(64, derive_seed(seed, TAG_INIT))
    pop = R.R_random_init(sk, seed, n)
    sel, secs = np.zeros(b, np.int64), np.zeros(4)
    R.check(R.ref().ref_round_strict(C.byref(sk), C.byref(dev), R.ptr(pop, R.i32p), pop.shape[1], n, k, b,
                                     R.ptr(params, R.f64p), 64, threads, R.ptr(sel, R.i64p), R.ptr(secs, R.f64p)))
    return float(secs.sum())


def cpu_baseline(args, reps=5):
    """The CPU reference on the box's host cores, on a bounded sample of the
    workload: `reps` whole subgraph rounds (cycling the subgraphs) per setting, median
    candidates/s. `value` = the reference's own round (explore(n_steps=1) +
    extract_features + score_batch + select_top, oracle/_ref) on all host threads;
    beside it the same at 1 thread and the strict hand-composed bound (ref_round_strict)
    at 1 and all threads."""
    R = _ref_setup(args)
    if not R.ref_available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": "oracle/_ref missing"}
    nproc = os.cpu_count() or 1
    names = R50 if args.workload == "r50" else [args.workload]

    def median_rate(fn, threads):
        rates = []
        for r in range(reps):
            w = names[r % len(names)]
            rates.append(args.n / fn(w, threads, r))
        return statistics.median(rates), rates

    api = lambda w, th, r: ref_round(R, w, args.n, args.k, args.b, args.seed + r, th)[0]  # noqa: E731
    strict = lambda w, th, r: strict_round(R, w, args.n, args.k, args.b, args.seed + r, th)  # noqa: E731
    v_all, r_all = median_rate(api, nproc)
    v_one, _ = median_rate(api, 1)
    s_all, _ = median_rate(strict, nproc)
    s_one, _ = median_rate(strict, 1)
    return {"value": v_all, "unit": UNIT, "cores": nproc, "kind": "reference",
            "sample": f"median of {reps} whole reference rounds (explore(n_steps=1)+extract_features+score_batch+"
                      f"select_top, N={args.n}, K={args.k}) over {names[:reps]}",
            "cpu_model": cpu_model(), "rates_all_threads": r_all,
            "reference_api_1_thread": v_one,
            "strict_bound": {"value": s_all, "value_1_thread": s_one, "unit": UNIT, "threads": nproc,
                             "what": "the reference's own draft_cost (parallel_for) + nth_element top-K with exact "
                                     "dedup + extract_features + score_batch + select_top over the resident "
                                     "population: no explore() string-key bookkeeping (ref_round_strict)"}}


def ref_round(R, workload, n, k, b, seed, threads):
    import ctypes as C
    from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device
    sk = make_sketch(WORKLOADS[workload]())
    dev = reference_device()
    params = R.R_init_params(64, derive_seed(seed, TAG_INIT))
    sel = np.zeros(b, np.int64)
    sc = np.zeros(b)
    cnt = C.c_int64(0)
    secs = np.zeros(4)
    R.check(R.ref().ref_round(C.byref(sk), C.byref(dev), n, k, b, seed, R.ptr(params, R.f64p), 64, threads,
                              R.ptr(sel, R.i64p), R.ptr(sc, R.f64p), None, None, C.byref(cnt), R.ptr(secs, R.f64p)))
    return float(secs.sum()), secs


def run_reference(args, rank, world):
    if rank != 0:
        return None
    R = _ref_setup(args)
    if not R.ref_available():
        return {"impl": "reference", "unavailable": "oracle/_ref/libtiletune_ref.so not built (make -C oracle ref)"}
    threads = os.cpu_count() or 1
    names = R50 if args.workload == "r50" else [args.workload]
    # bounded sample per step: ref_rounds_per_step subgraph rounds
    per_step = min(len(names), args.ref_rounds_per_step)
    for i in range(args.warmup):
        ref_round(R, names[i % len(names)], args.n, args.k, args.b, args.seed, threads)
    tot, stage = 0.0, np.zeros(4)
    for s in range(args.steps):
        for r in range(per_step):
            t, st = ref_round(R, names[(s * per_step + r) % len(names)], args.n, args.k, args.b, args.seed, threads)
            tot += t
            stage += st
    cands = args.n * per_step * args.steps
    v = cands / tot
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.workload}: N={args.n}/round, K={args.k}, b={args.b}, h=64",
                       "rounds_per_step": per_step, "subgraphs": names},
            "stage_s_per_round": {"explore": stage[0] / (per_step * args.steps),
                                  "features": stage[1] / (per_step * args.steps),
                                  "score_batch": stage[2] / (per_step * args.steps),
                                  "select_top": stage[3] / (per_step * args.steps)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{per_step} subgraph round(s) per step of the reference API"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="r50")
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--k", type=int, default=512)
    ap.add_argument("--b", type=int, default=10)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--precision", default="fp64", choices=["fp64", "bf16"])
    ap.add_argument("--band", type=float, default=None, help="bf16 certification band (default TT_BF16_BAND)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-explore", action="store_true", help="skip the explore_ga entry (e.g. under ncu)")
    ap.add_argument("--ref-rounds-per-step", type=int, default=1)
    ap.add_argument("--bert-n", type=int, default=1 << 20, help="configs[2]: candidates per BERT round in total")
    ap.add_argument("--no-bert", action="store_true", help="skip the configs[2] (BERT 1M, strong-sharded) entry")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without a launcher: start N ranks (one per GPU) the way the
        # driver does, over torch.distributed.run on 127.0.0.1
        import socket
        sock = socket.socket()
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
        sock.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        os.execv(sys.executable, cmd)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus != world:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; measuring {world} rank(s)", file=sys.stderr)
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        res = run_ours(args, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
    if rank == 0 and res is not None:
        print(json.dumps(res))


if __name__ == "__main__":
    main()
