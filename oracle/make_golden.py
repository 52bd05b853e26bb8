#!/usr/bin/env python
"""Dump golden vectors from the REFERENCE ITSELF into tests/golden/.

TEST INFRASTRUCTURE ONLY. Runs the unmodified reference tiletune core
(compiled from /root/reference/proj/core/src by `make -C oracle ref` into
oracle/_ref/libtiletune_ref.so; see oracle/ref_capi.cpp for the thin
extern "C" wrapper) on small seeded inputs and writes the results as
tests/golden/golden.npz. The fixtures are committed so that
tests/test_oracle_golden.py can pin the C restatement (oracle/tt_oracle.c)
without /root/reference — which does not exist on the GPU box.

    make -C oracle ref && python oracle/make_golden.py

What is dumped, per workload shape (reference call in brackets):
  pop       random_init(sketch, 256, RngStream(42))        schedule.cpp:166-186
  cost_tX   draft_cost(...).total with toggles X            draft.cpp:129-154
  ex_soa/ex_cost  explore(op, dev, 1, 64, 2048, RngStream(43))  draft.cpp:156-221
  ga_soa/ga_cost  explore(op, dev, 8, 64, 128, RngStream(44))   draft.cpp:156-221 + mutate
  st/bl     extract_features of pop[:, :16]                 features.cpp:98-257
  score     score_batch(init_params(64, RngStream(derive_seed(42,"init"))))  ranker.cpp:375-381
  sel       select_top(score, cost_t3[:16], none, 5)        ranker.cpp:514-532
  trace     per-statement symbols / penalties / costs of pop[:, 0]  draft.cpp:42-154
plus params (h=64 and h=8), momentum_update endpoints (momentum.cpp:28-46)
and a short train() run (ranker.cpp:459-512) for the GD path.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2402_02361_b200.types import (TAG_INIT, WORKLOADS, derive_seed, make_gemm,  # noqa: E402
                                         make_elementwise, make_sketch, reference_device)
from tests import _refs as R  # noqa: E402

SHAPES = ["gemm128", "gemm1024", "elementwise", "r50_stem", "r50_c1x1_64", "r50_c3x3_512", "bert_qkv", "bert_bmm_qk",
          "bert_bmm_pv"]


def sketch_of(name):
    if name == "gemm128":
        return make_sketch(make_gemm(128, 128, 128))
    if name == "elementwise":
        return make_sketch(make_elementwise(64, 48))
    return make_sketch(WORKLOADS[name]())


def trace(sk, dev, soa, i):
    import ctypes as C
    S = sk.op.n_statements
    sy = np.zeros((S, 8), np.int64)
    pe = np.zeros((S, 7))
    sc = np.zeros((S, 4))
    tot = C.c_double(0)
    soa = np.ascontiguousarray(soa)
    R.check(R.ref().ref_trace(C.byref(sk), C.byref(dev), R.ptr(soa, R.i32p), soa.shape[1], i, R.ptr(sy, R.i64p),
                              R.ptr(pe, R.f64p), R.ptr(sc, R.f64p), C.byref(tot)))
    return sy, pe, sc, tot.value


def main():
    if not R.ref_available():
        sys.exit("oracle/_ref/libtiletune_ref.so missing: run `make -C oracle ref` first")
    dev = reference_device()
    out = {}
    params64 = R.R_init_params(64, derive_seed(42, TAG_INIT))
    out["params_h64"] = params64
    for name in SHAPES:
        sk = sketch_of(name)
        pop = R.R_random_init(sk, 42, 256)
        out[f"{name}/pop"] = pop
        for t in (1, 2, 3):
            out[f"{name}/cost_t{t}"] = R.R_draft_cost(sk, dev, pop, t)
        ex_soa, ex_cost = R.R_explore(sk, dev, 2048, 64, 43)
        out[f"{name}/ex_soa"], out[f"{name}/ex_cost"] = ex_soa, ex_cost
        ga_soa, ga_cost = R.R_explore(sk, dev, 128, 64, 44, n_steps=8)
        out[f"{name}/ga_soa"], out[f"{name}/ga_cost"] = ga_soa, ga_cost
        idx = np.arange(16, dtype=np.int64)
        st, bl = R.R_features(sk, dev, pop, idx)
        out[f"{name}/st"], out[f"{name}/bl"] = st, bl
        score = R.R_score(params64, 64, st, bl)
        out[f"{name}/score"] = score
        out[f"{name}/score_identity_attn"] = R.R_score(params64, 64, st, bl, identity=True)
        out[f"{name}/sel"] = R.R_select_top(score, out[f"{name}/cost_t3"][:16], None, 5)
        sy, pe, sc, tot = trace(sk, dev, pop, 0)
        out[f"{name}/trace_symbols"], out[f"{name}/trace_penalties"] = sy, pe
        out[f"{name}/trace_stmt_cost"], out[f"{name}/trace_total"] = sc, np.array([tot])

    # MoA: momentum_update endpoints and a generic m (momentum.cpp:28-46)
    phi = R.R_init_params(8, 113)
    tgt = R.R_init_params(8, 114)
    out["moa/phi"], out["moa/target"] = phi, tgt
    for m in (0.0, 0.5, 0.9, 0.99):
        p = phi.copy()
        R.check(R.ref().ref_momentum_update(R.ptr(p, R.f64p), R.ptr(tgt, R.f64p), 8, m))
        out[f"moa/phi_m{m}"] = p

    # train(): GD over the LambdaRank loss on the gemm128 features (ranker.cpp:459-512)
    import ctypes as C
    sk = sketch_of("gemm128")
    pop = out["gemm128/pop"]
    st, bl = R.R_features(sk, dev, pop, np.arange(32, dtype=np.int64))
    lat = out["gemm128/cost_t3"][:32].copy()
    p = R.R_init_params(8, 7)
    out["train/p0"], out["train/st"], out["train/bl"], out["train/lat"] = p.copy(), st, bl, lat
    l0, l1 = C.c_double(0), C.c_double(0)
    R.check(R.ref().ref_train(R.ptr(p, R.f64p), 8, st.shape[1], bl.shape[1], R.ptr(st, R.f64p), R.ptr(bl, R.f64p),
                              R.ptr(lat, R.f64p), 32, 2, 1e-2, 16, 99, C.byref(l0), C.byref(l1)))
    out["train/p1"], out["train/loss"] = p, np.array([l0.value, l1.value])

    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    path = os.path.join(ROOT, "tests", "golden", "golden.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
