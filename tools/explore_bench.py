#!/usr/bin/env python
"""the reference's real per-round explore — the LSE genetic
loop at TunerConfig defaults (pop_size 512, n_steps 32, draft_size 512;
tuner.hpp:38-40, tuner.cpp:304-305) — through tt_explore, timed against the
reference's own explore() (oracle/_ref, all host threads) on the same call.

  python tools/explore_bench.py [--reps 20] [--out gpurun_out/explore.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2402_02361_b200 import tiletune as tt  # noqa: E402
from paper_2402_02361_b200.types import WORKLOADS, make_sketch, reference_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "explore.json"))
    a = ap.parse_args()
    ctx = tt.Context(0)
    dev = reference_device()
    threads = os.cpu_count() or 1
    from tests import _refs as R
    res = {"config": "explore(op, dev, n_steps=32, draft_size=512, pop_size=512) — TunerConfig defaults; timed calls return the drafted schedules as exact identities + draft costs (the reference returns Schedules); the checked call also returns the factor SoA",
           "host_threads_reference": threads, "workloads": {}}
    for name in ["gemm1024", "r50_c3x3_64", "bert_ffn1"]:
        sk = make_sketch(WORKLOADS[name]())
        tt.explore(ctx, sk, dev, 32, 512, 512, 1)  # warm
        soa, cost, ids, ev = tt.explore(ctx, sk, dev, 32, 512, 512, 100)  # checked against the reference below
        t0 = time.perf_counter()
        for r in range(a.reps):  # timed: schedules returned as exact identities (+ draft costs)
            tt.explore(ctx, sk, dev, 32, 512, 512, 100 + r, with_soa=False)
        gpu = (time.perf_counter() - t0) / a.reps
        row = {"ms_per_explore": gpu * 1e3, "evaluations": ev, "evals_per_s": ev / gpu}
        if R.ref_available():
            R.R_explore(sk, dev, 512, 512, 1, n_steps=32, threads=threads)
            t0 = time.perf_counter()
            for r in range(min(a.reps, 10)):
                out = R.R_explore(sk, dev, 512, 512, 100 + r, n_steps=32, threads=threads)
                if r == 0:
                    rs, rc = out
            cpu = (time.perf_counter() - t0) / min(a.reps, 10)
            same = len(rc) == len(cost) and (rc.view(np.uint64) == cost.view(np.uint64)).all() and \
                (rs == soa).all()
            row.update({"reference_ms_per_explore": cpu * 1e3, "speedup": cpu / gpu, "identical_to_reference_seed_100": bool(same)})
        res["workloads"][name] = row
    print(json.dumps(res, indent=1))
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
