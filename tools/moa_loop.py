#!/usr/bin/env python
"""BASELINE.json config 4: MoA-Pruner online adaptation on one B200.

  python tools/moa_loop.py [--rounds 100] [--out gpurun_out/moa.json] [--cpu-check]

Each round (tuner.cpp:173-292 with momentum adaptation on): draft+verify
round on GEMM-1024 (N = 4,096 -> K = 512 -> b = 10, target model) ->
the b selections measured by the simulated hardware on the device (oracle_b,
per-trial lognormal, tuner.cpp:202-203) -> records grow by b -> momentum_adapt
(train a copy of the Siamese model on all records: 8 epochs, lr 1e-2, batch
256, seed derive_seed(seed, "tran", round); then EMA m = 0.99,
momentum.cpp:48-56) -> the trained copy scores the next round.

Reports per-phase device times and, with --cpu-check, the reference's own
train() (oracle/_ref) on the final round's records for the same step. With
--reference, the same 100-round loop runs through the reference's own
functions on the host cores (oracle/_ref: explore + extract_features +
score_batch + select_top, measure, extract_features of the records, train,
momentum_update), for the wall-clock comparison of BASELINE config 4.
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_02361_b200 import tiletune as tt  # noqa: E402
from paper_2402_02361_b200.types import (TAG_INIT, derive_seed, hash_str, make_gemm, make_sketch,  # noqa: E402
                                         oracle_b, reference_device)

TAG_TRAIN = 0x7472616E  # tuner.cpp kTagTrain ("tran")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=100)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "moa.json"))
    ap.add_argument("--cpu-check", action="store_true")
    ap.add_argument("--reference", action="store_true", help="run the loop through the reference (oracle/_ref)")
    a = ap.parse_args()
    if a.reference:
        return reference_loop(a)
    ctx = tt.Context(0)
    sk = make_sketch(make_gemm(1024, 1024, 1024))
    dev = reference_device()
    orc = oracle_b()
    n, k, b, h = 4096, 512, 10, 64
    phi = torch.from_numpy(tt.init_params(h, derive_seed(a.seed, TAG_INIT))).cuda()  # Siamese state
    target = phi.clone()
    model = tt.PaCM(ctx, target, h)
    task = hash_str("gemm1024")
    ids, lats = [], []
    trial = 0
    t_round = t_meas = t_train = 0.0
    losses = []
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    wall0 = time.time()
    for rnd in range(a.rounds):
        torch.cuda.synchronize()
        ev[0].record()
        model.load(target)
        out = tt.draft_verify_round(ctx, sk, dev, n, k, b, seed=derive_seed(a.seed, 0x6578706C, rnd))
        ev[1].record()
        sel = torch.tensor(out.identity.view(np.int64), device="cuda")
        soa = tt.schedule_from_identity(ctx, sk, sel)
        lat, _ = tt.oracle_measure(ctx, sk, orc, soa, task, trial)
        trial += len(out.identity)
        ids.append(sel)
        lats.append(lat.cpu().numpy())
        if rnd == 0:
            sel0 = out.index.tolist()
        ev[2].record()
        all_ids = torch.cat(ids)
        st, bl = tt.extract_features(ctx, sk, dev, all_ids)
        target, (l0, l1) = tt.momentum_adapt(ctx, phi, 0.99, h, st, bl, np.concatenate(lats), epochs=8, lr=1e-2,
                                             batch=256, seed=derive_seed(a.seed, TAG_TRAIN, rnd))
        ev[3].record()
        torch.cuda.synchronize()
        t_round += ev[0].elapsed_time(ev[1])
        t_meas += ev[1].elapsed_time(ev[2])
        t_train += ev[2].elapsed_time(ev[3])
        losses.append((l0, l1))
    wall = time.time() - wall0
    res = {"config": "MoA-Pruner online adaptation, GEMM-1024, N=4096 -> K=512 -> b=10, h=64, m=0.99, "
                     "8 epochs / lr 1e-2 / batch 256 per round, labels from oracle_b on the device",
           "rounds": a.rounds, "records": int(sum(len(x) for x in lats)),
           "ms_total": {"rounds": t_round, "measure": t_meas, "momentum_adapt": t_train},
           "ms_per_round": {"round": t_round / a.rounds, "measure": t_meas / a.rounds,
                            "momentum_adapt": t_train / a.rounds},
           "wall_s": wall, "final_loss": losses[-1], "best_latency_s": float(np.concatenate(lats).min()),
           "selections_round0": sel0}
    if a.cpu_check:
        from tests import _refs as R
        if R.ref_available():
            # the reference's own train() on the final records, same config
            st64, bl64 = st.cpu().numpy(), bl.cpu().numpy()
            lat64 = np.concatenate(lats)
            p = phi.cpu().numpy().copy()
            l0r, l1r = C.c_double(0), C.c_double(0)
            t0 = time.time()
            R.check(R.ref().ref_train(R.ptr(p, R.f64p), h, st64.shape[1], bl64.shape[1], R.ptr(st64, R.f64p),
                                      R.ptr(bl64, R.f64p), R.ptr(lat64, R.f64p), len(lat64), 8, 1e-2, 256,
                                      derive_seed(a.seed, TAG_TRAIN, a.rounds), C.byref(l0r), C.byref(l1r)))
            cpu = time.time() - t0
            tgt = phi.clone()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            tt.train(ctx, tgt, h, st, bl, lat64, epochs=8, lr=1e-2, batch=256,
                     seed=derive_seed(a.seed, TAG_TRAIN, a.rounds))
            e1.record()
            torch.cuda.synchronize()
            res["train_check"] = {"records": len(lat64), "cpu_reference_s": cpu, "gpu_s": e0.elapsed_time(e1) / 1e3,
                                  "max_rel_param_diff": float(np.abs(tgt.cpu().numpy() - p).max() / np.abs(p).max()),
                                  "final_loss_cpu": l1r.value}
    print(json.dumps(res, indent=1))
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


def reference_loop(a):
    """The same loop through the reference's own functions (host, all cores)."""
    from tests import _refs as R
    sk = make_sketch(make_gemm(1024, 1024, 1024))
    dev = reference_device()
    orc = oracle_b()
    n, k, b, h = 4096, 512, 10, 64
    threads = os.cpu_count() or 1
    phi = R.R_init_params(h, derive_seed(a.seed, TAG_INIT))
    target = phi.copy()
    task = hash_str("gemm1024")
    cols = sk.cols
    rec_soa, lats, sels = np.zeros((cols, 0), np.int32), [], []
    trial = 0
    t_round = t_meas = t_train = 0.0
    wall0 = time.time()
    for rnd in range(a.rounds):
        t0 = time.time()
        sel = np.zeros(b, np.int64)
        sc = np.zeros(b)
        dsoa = np.zeros((cols, k), np.int32)
        dcost = np.zeros(k)
        cnt = C.c_int64(0)
        secs = np.zeros(4)
        R.check(R.ref().ref_round(C.byref(sk), C.byref(dev), n, k, b, derive_seed(a.seed, 0x6578706C, rnd),
                                  R.ptr(target, R.f64p), h, threads, R.ptr(sel, R.i64p), R.ptr(sc, R.f64p),
                                  R.ptr(dsoa, R.i32p), R.ptr(dcost, R.f64p), C.byref(cnt), R.ptr(secs, R.f64p)))
        t1 = time.time()
        ssoa = np.ascontiguousarray(dsoa[:, sel])
        lat, nl = np.zeros(b), np.zeros(b)
        R.check(R.ref().ref_measure(C.byref(sk), C.byref(orc), R.ptr(ssoa, R.i32p), b, b, task, trial,
                                    R.ptr(lat, R.f64p), R.ptr(nl, R.f64p)))
        trial += b
        rec_soa = np.ascontiguousarray(np.concatenate([rec_soa, ssoa], axis=1))
        lats.append(lat)
        sels.append(sel.tolist())
        t2 = time.time()
        m = rec_soa.shape[1]
        st, bl = R.R_features(sk, dev, rec_soa, np.arange(m))
        lat_all = np.concatenate(lats)
        target = phi.copy()
        l0r, l1r = C.c_double(0), C.c_double(0)
        R.check(R.ref().ref_train(R.ptr(target, R.f64p), h, st.shape[1], bl.shape[1], R.ptr(st, R.f64p),
                                  R.ptr(bl, R.f64p), R.ptr(lat_all, R.f64p), m, 8, 1e-2, 256,
                                  derive_seed(a.seed, TAG_TRAIN, rnd), C.byref(l0r), C.byref(l1r)))
        R.check(R.ref().ref_momentum_update(R.ptr(phi, R.f64p), R.ptr(target, R.f64p), h, 0.99))
        t3 = time.time()
        t_round += t1 - t0
        t_meas += t2 - t1
        t_train += t3 - t2
    wall = time.time() - wall0
    res = {"config": "reference (oracle/_ref, %d host threads): the same MoA loop" % threads,
           "rounds": a.rounds, "records": int(sum(len(x) for x in lats)),
           "s_total": {"rounds": t_round, "measure": t_meas, "momentum_adapt": t_train}, "wall_s": wall,
           "best_latency_s": float(np.concatenate(lats).min()), "selections_round0": sels[0]}
    print(json.dumps(res, indent=1))
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
