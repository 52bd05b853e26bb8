#!/usr/bin/env python
"""BASELINE.json config 5 and the PaCM verify-only sweep, on one B200.

  python tools/sweep.py [--out gpurun_out/sweep.json] [--max-n 16777216]

1. population sweep: one draft+verify round (K = 512, b = 10, h = 64) over
   N = 4K .. 16M candidates resident in HBM, for GEMM-1024 and BERT FFN1
   (128x3072x768), fp64 and bf16 PaCM; candidates/s and the K1 draft-cost
   kernel's HBM GB/s (algorithmic bytes: factor columns + fp64 cost);
2. verify-only sweep: tt_pacm_score over K = 512 .. 1M drafted candidates
   (features + PaCM), TFLOP/s at 320,640 FLOP per candidate, bf16 tcgen05
   vs fp64 CUDA cores.
CUDA events on the context stream, median of reps, L2 not flushed (N >= 1M
populations exceed L2 anyway).
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2402_02361_b200 import tiletune as tt  # noqa: E402
from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device  # noqa: E402


def timed(fn, reps):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.json"))
    ap.add_argument("--max-n", type=int, default=1 << 24)
    a = ap.parse_args()
    ctx = tt.Context(0)
    dev = reference_device()
    tt.PaCM(ctx, tt.init_params(64, derive_seed(42, TAG_INIT)), 64)
    res = {"population": [], "verify": []}
    k, b = 512, 10
    for name in ["gemm1024", "bert_ffn1"]:
        sk = make_sketch(WORKLOADS[name]())
        col_bytes = 4 * (4 * sk.op.n_spatial + 3 * sk.op.n_reduction) + 8
        n = 4096
        while n <= a.max_n:
            soa = tt.random_init(ctx, sk, n, 42)
            for prec in (tt.TT_PREC_FP64, tt.TT_PREC_BF16):
                tt.draft_verify_round(ctx, sk, dev, n, k, b, soa=soa, precision=prec)  # warm-up
                reps = 10 if n <= (1 << 20) else 3
                sec = timed(lambda: tt.draft_verify_round(ctx, sk, dev, n, k, b, soa=soa, precision=prec), reps)
                tt.profile_enable(ctx, True)
                tt.profile_read(ctx)
                tt.draft_verify_round(ctx, sk, dev, n, k, b, soa=soa, precision=prec)
                prof = tt.profile_read(ctx)
                tt.profile_enable(ctx, False)
                k1 = prof.get("draft_cost", (0.0, 0))[0]
                row = {"workload": name, "n": n, "precision": "bf16" if prec else "fp64", "round_s": sec,
                       "candidates_per_s": n / sec, "k1_ms": k1,
                       "k1_hbm_gbs": (n * col_bytes / (k1 * 1e-3) / 1e9) if k1 else None,
                       "stage_ms": {s: v[0] for s, v in prof.items()}}
                res["population"].append(row)
                print(json.dumps(row), flush=True)
            del soa
            torch.cuda.empty_cache()
            n *= 4
    sk = make_sketch(WORKLOADS["r50_c3x3_64"]())
    for kk in [512, 4096, 65536, 1 << 20]:
        ids = tt.random_init(ctx, sk, kk, 7, with_identity=True)[1]
        for prec in (tt.TT_PREC_BF16, tt.TT_PREC_FP64):
            m = tt.PaCM(ctx, tt.init_params(64, derive_seed(42, TAG_INIT)), 64)
            m.score(sk, dev, ids, prec)
            sec = timed(lambda: m.score(sk, dev, ids, prec), 5 if kk <= 65536 else 2)
            row = {"k": kk, "precision": "bf16" if prec else "fp64", "s": sec,
                   "tflops": kk * 320640 / sec / 1e12, "candidates_per_s": kk / sec}
            res["verify"].append(row)
            print(json.dumps(row), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
