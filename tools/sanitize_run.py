"""A small workload that launches every kernel family of the library once or
twice, for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_run.py [part]

parts: round (seeded + explicit, fp64 + bf16-certified, n above and below
the one-CTA selector), bigchunk (a 700K round: the selector's table path), explore (GA cluster kernel + draft set), train (device
training + momentum), oracle, sharded (local draft + merge + merged verify),
select (select_top + features + scoring). Default: all. Sizes are small so a
racecheck pass finishes in minutes; each part checks its own results against
the oracle only where that is cheap (the sanitizer is the point here).
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_02361_b200 import tiletune as tt  # noqa: E402
from paper_2402_02361_b200.types import (TAG_INIT, WORKLOADS, derive_seed, make_sketch,  # noqa: E402
                                         make_gemm, oracle_b, reference_device)

parts = sys.argv[1:] or ["round", "bigchunk", "explore", "train", "oracle", "sharded", "select"]
ctx = tt.Context(0)
dev = reference_device()
params = tt.init_params(64, derive_seed(42, TAG_INIT))
model = tt.PaCM(ctx, params, 64)

if "round" in parts:
    for name, n in [("r50_c3x3_64", 8192), ("gemm1024", 900), ("r50_c1x1_64", 4096)]:
        sk = make_sketch(WORKLOADS[name]())
        soa = tt.random_init(ctx, sk, n, 7)
        for prec in (tt.TT_PREC_FP64, tt.TT_PREC_BF16):
            a = tt.draft_verify_round(ctx, sk, dev, n, 256, 10, seed=7, precision=prec)
            b = tt.draft_verify_round(ctx, sk, dev, n, 256, 10, soa=soa, precision=prec)
            assert (a.index == b.index).all(), (name, prec)
        print("round", name, n, a.index.tolist(), flush=True)

if "bigchunk" in parts:
    # >= 4,096 candidates per CTA: the selector's p_l2_m table (filled in the
    # sample region, overwritten by the sample after the grid barrier) and
    # the 32-bit draft-cost mode
    sk = make_sketch(WORKLOADS["gemm1024"]())
    n = 700_000
    soa = tt.random_init(ctx, sk, n, 5)
    a = tt.draft_verify_round(ctx, sk, dev, n, 512, 10, seed=5)
    b = tt.draft_verify_round(ctx, sk, dev, n, 512, 10, soa=soa)
    assert (a.index == b.index).all()
    print("bigchunk", n, a.index.tolist(), flush=True)

if "explore" in parts:
    sk = make_sketch(WORKLOADS["gemm1024"]())
    _, c, _, ev = tt.explore(ctx, sk, dev, 4, 128, 256, 3)
    ids, dc, _ = tt.draft_set(ctx, sk, dev, 3, 128, 128, 0.2, 4, 5)
    print("explore", len(c), ev, len(ids), flush=True)

if "train" in parts:
    from tests import _refs as R
    sk = make_sketch(WORKLOADS["r50_c3x3_64"]())
    pop = R.O_random_init(sk, 17, 48)
    st, bl = R.O_features(sk, dev, pop, np.arange(48))
    lat = R.O_draft_cost(sk, dev, pop) * (1.0 + 0.1 * np.sin(np.arange(48)))
    p = torch.from_numpy(tt.init_params(64, 23)).cuda()
    l0, l1 = tt.train(ctx, p, 64, torch.from_numpy(st).cuda(), torch.from_numpy(bl).cuda(), lat, epochs=2,
                      batch=16, seed=3)
    phi = torch.from_numpy(tt.init_params(64, 24)).cuda()
    tt.momentum_adapt(ctx, phi, 0.9, 64, torch.from_numpy(st).cuda(), torch.from_numpy(bl).cuda(), lat, epochs=1,
                      batch=32, seed=4)
    torch.cuda.synchronize()
    print("train", l0, l1, flush=True)

if "oracle" in parts:
    sk = make_sketch(WORKLOADS["gemm1024"]())
    orc = oracle_b()
    soa = tt.random_init(ctx, sk, 2048, 9)
    lat = tt.oracle_latency(ctx, sk, orc, soa)
    m, nl = tt.oracle_measure(ctx, sk, orc, soa, 123, 0)
    best = tt.oracle_best(ctx, make_sketch(make_gemm(128, 128, 128)), orc)
    torch.cuda.synchronize()
    print("oracle", float(lat.min()), best, flush=True)

if "sharded" in parts:
    sk = make_sketch(WORKLOADS["bert_ffn1"]())
    n, k, b, world = 8192, 256, 10, 2
    outs = []
    for r in range(world):
        o = torch.empty((3, k), dtype=torch.int64, device="cuda")
        tt.round_local_async(ctx, sk, dev, n, k, b, r * n, o, seed=11)
        outs.append(o)
    gathered = torch.cat([o.reshape(-1) for o in outs])
    tt.round_finish_merged_async(ctx, sk, dev, gathered, n * world, k, b)
    got = tt.round_collect(ctx, b)
    want = tt.draft_verify_round(ctx, sk, dev, n * world, k, b, seed=11)
    assert (got.index == want.index).all()
    print("sharded", got.index.tolist(), flush=True)

if "select" in parts:
    sk = make_sketch(WORKLOADS["r50_c3x3_64"]())
    soa = tt.random_init(ctx, sk, 300, 5)
    ids = tt.schedule_identity(ctx, sk, soa)
    st, bl = tt.extract_features(ctx, sk, dev, ids)
    sc = model.score_batch(st, bl)
    sc2 = model.score(sk, dev, ids, tt.TT_PREC_BF16)
    dc = tt.draft_cost(ctx, sk, dev, soa)
    sel = tt.select_top(ctx, sc, dc, None, 10)
    print("select", sel.tolist(), float((sc - sc2).abs().max()), flush=True)

ctx.close()
print("sanitize_run ok", parts)
