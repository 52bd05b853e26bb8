"""Pins the CPU oracle (oracle/tt_oracle.c) before anything is checked
against it (CPU only, no GPU).

1. The reference's own known-answer tests (proj/tests/test_*.cpp), restated
   as direct calls because the reference's doctest harness is not vendored.
2. Golden vectors produced by the reference itself (tests/golden/golden.npz,
   written by oracle/make_golden.py from the compiled reference), which
   travel with the repo.
3. When oracle/_ref is built here, live comparisons against the reference on
   fresh seeded inputs (skipped elsewhere).

Bar: bit-exact for populations, draft costs, top-K, identities, select_top
and the MoA EMA; features and scores bit-exact too (same glibc libm, same
accumulation order, no FMA contraction), asserted with a 1e-13 / 1e-12
guard so a libm difference on another host reports as a tolerance miss.
"""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2402_02361_b200.types import (TAG_INIT, WORKLOADS, derive_seed, make_conv, make_elementwise, make_gemm,
                                         make_sketch, reference_device)
from tests import _refs as R

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")
DEV = reference_device()
SHAPES = ["gemm128", "gemm1024", "elementwise", "r50_stem", "r50_c1x1_64", "r50_c3x3_512", "bert_qkv", "bert_bmm_qk",
          "bert_bmm_pv"]


@pytest.fixture(scope="module")
def G():
    return np.load(GOLDEN)


def sketch_of(name):
    if name == "gemm128":
        return make_sketch(make_gemm(128, 128, 128))
    if name == "elementwise":
        return make_sketch(make_elementwise(64, 48))
    return make_sketch(WORKLOADS[name]())


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def ref_gemm_schedule():
    """test_helpers.hpp:114-116: m(4,8,2,2) n(4,8,2,2) k(4,8,4), unroll 1."""
    return np.array([[4], [8], [2], [2], [4], [8], [2], [2], [4], [8], [4], [1]], np.int32)


def o_trace(sk, soa, i=0, toggles=3):
    S = sk.op.n_statements
    sy = np.zeros((S, 8), np.int64)
    pe = np.zeros((S, 7))
    sc = np.zeros((S, 4))
    tot = C.c_double(0)
    soa = np.ascontiguousarray(soa)
    R.oracle().tto_trace(C.byref(sk), C.byref(DEV), R.ptr(soa, R.i32p), soa.shape[1], i, toggles, R.ptr(sy, R.i64p),
                         R.ptr(pe, R.f64p), R.ptr(sc, R.f64p), C.byref(tot))
    return sy, pe, sc, tot.value


# ------------------------------------------------------------ reference KATs --

def test_kat_symbols_gemm128():
    # test_draft.cpp:19-53
    sk = make_sketch(make_gemm(128, 128, 128))
    sy, _, _, _ = o_trace(sk, ref_gemm_schedule())
    assert (sy[:, 0] == 24).all() and (sy[:, 1] == 2048).all() and (sy[:, 2] == 2048).all()
    assert (sy[:, 3] == 64).all() and (sy[:, 5] == 16).all()
    assert sy[0, 4] == 65536 and sy[0, 6] == 32 and sy[1, 4] == 65536 and sy[1, 6] == 32
    assert sy[2, 4] == 0 and sy[2, 6] == 1 and sy[3, 6] == 4
    assert sy[4, 7] == 2097152 and sy[4, 4] == 0
    assert sy[5, 4] == 16384 and sy[5, 6] == 4


def test_kat_symbols_degenerate():
    # test_draft.cpp:55-70
    sk = make_sketch(make_gemm(1, 1, 1))
    soa = np.ones((12, 1), np.int32)
    sy, _, _, _ = o_trace(sk, soa)
    assert (sy[:, 0] == 3).all() and (sy[:, 1] == 1).all() and (sy[:, 2] == 2).all()
    assert (sy[:, 3] == 1).all() and (sy[:, 5] == 1).all()
    assert sy[0, 4] == 1 and sy[1, 4] == 1 and sy[4, 7] == 1


def test_kat_draft_total_and_statement_costs():
    # test_draft.cpp:160-183 + the goldens the reference printed
    sk = make_sketch(make_gemm(128, 128, 128))
    _, pe, sc, tot = o_trace(sk, ref_gemm_schedule())
    assert tot == 2.6700226718146717e-06
    assert sc[0, 1] == 6.5535999999999996e-07 and sc[1, 1] == 6.5535999999999996e-07
    assert sc[4, 0] == 4.8582671814671819e-08
    assert sc[5, 1] == 1.3107199999999999e-06
    assert sc[4, 2] == 43166666666666.664
    # penalties of the l0 terms (test_draft.cpp:98-106)
    assert pe[0, 0] == 1.0 and abs(pe[0, 1] - (1.0 + 2048.0 / 24.0)) < 1e-15 * pe[0, 1]


def test_kat_random_init_seed42_first_three():
    # RngStream(42) GEMM-128 first three schedules + their costs
    sk = make_sketch(make_gemm(128, 128, 128))
    pop = R.O_random_init(sk, 42, 3)
    want = [([8, 1, 8, 2], [1, 4, 16, 2], [2, 4, 16], 4, 8.6325815153715799e-06),
            ([1, 1, 16, 8], [16, 2, 1, 4], [1, 128, 1], 16, 5.0353117619099428e-05),
            ([2, 1, 16, 4], [4, 2, 16, 1], [1, 128, 1], 4, 1.807849353250212e-05)]
    cost = R.O_draft_cost(sk, DEV, pop)
    for j, (m, n, k, u, c) in enumerate(want):
        assert pop[:, j].tolist() == m + n + k + [u]
        assert cost[j] == c


def test_kat_init_params_score():
    # init_params(64, RngStream(7)) score of the reference schedule
    sk = make_sketch(make_gemm(128, 128, 128))
    st, bl = R.O_features(sk, DEV, ref_gemm_schedule(), np.array([0]))
    p = R.O_init_params(64, 7)
    assert R.O_score(p, 64, st, bl)[0] == 0.75490836797299699


def test_kat_zero_params_score_zero():
    # test_ranker.cpp:32-36
    sk = make_sketch(make_gemm(128, 128, 128))
    st, bl = R.O_features(sk, DEV, ref_gemm_schedule(), np.array([0]))
    assert R.O_score(np.zeros_like(R.O_init_params(16, 1)), 16, st, bl)[0] == 0.0


def test_kat_select_top():
    # test_ranker.cpp:268-288
    scores = np.array([1.0, 3.0, 3.0, 2.0])
    drafts = np.array([0.5, 0.9, 0.2, 0.1])
    assert R.O_select_top(scores, drafts, None, 4).tolist() == [2, 1, 3, 0]
    assert R.O_select_top(np.zeros(4), drafts, None, 2).tolist() == [3, 2]
    ex = np.array([0, 0, 1, 0], np.uint8)
    assert R.O_select_top(scores, drafts, ex, 3).tolist() == [1, 3, 0]
    with pytest.raises(RuntimeError):
        R.O_select_top(scores, drafts, ex, 4)


def test_kat_momentum_endpoints():
    # test_momentum.cpp:69-99
    phi, tgt = R.O_init_params(8, 113), R.O_init_params(8, 114)
    p = phi.copy()
    R.oracle().tto_momentum_update(R.ptr(p, R.f64p), R.ptr(tgt, R.f64p), len(p), 0.0)
    assert (bits(p) == bits(tgt)).all()
    p = phi.copy()
    R.oracle().tto_momentum_update(R.ptr(p, R.f64p), R.ptr(phi, R.f64p), len(p), 1.0 - 1e-9)
    assert (bits(p) == bits(phi)).all()
    z, ones = np.zeros_like(phi), np.ones_like(phi)
    R.oracle().tto_momentum_update(R.ptr(z, R.f64p), R.ptr(ones, R.f64p), len(z), 0.99)
    assert np.abs(z - 0.01).max() <= 1e-12 * 0.01 + 1e-15


def test_kat_momentum_geometric_convergence():
    # test_momentum.cpp:122-132
    tgt, phi = R.O_init_params(8, 118), R.O_init_params(8, 119)
    d0 = np.sqrt(((phi - tgt) ** 2).sum())
    for k in range(1, 51):
        R.oracle().tto_momentum_update(R.ptr(phi, R.f64p), R.ptr(tgt, R.f64p), len(phi), 0.9)
        assert abs(np.sqrt(((phi - tgt) ** 2).sum()) - 0.9 ** k * d0) <= 1e-10 * 0.9 ** k * d0


def test_kat_divisibility_unity():
    # test_draft.cpp:115-131: p_l2_c == 1 exactly iff pu_l2 divides s6
    sk = make_sketch(make_gemm(4096, 1, 1))
    for b0 in [1, 2, 3, 4, 6, 8, 16, 24, 32, 64]:
        soa = np.array([[b0], [4096 // b0], [1], [1], [1], [1], [1], [1], [1], [1], [1], [1]], np.int32)
        _, pe, _, _ = o_trace(sk, soa)
        assert (pe[0, 5] == 1.0) == (b0 % DEV.pu_l2 == 0)


# --------------------------------------------------- reference golden vectors --

@pytest.mark.parametrize("name", SHAPES)
def test_golden_population(G, name):
    sk = sketch_of(name)
    assert (R.O_random_init(sk, 42, 256) == G[f"{name}/pop"]).all()
    # counter-based: the shard [100, 256) drawn on its own is the same stream
    assert (R.O_random_init(sk, 42, 156, first=100) == G[f"{name}/pop"][:, 100:]).all()


@pytest.mark.parametrize("name", SHAPES)
def test_golden_draft_cost(G, name):
    sk = sketch_of(name)
    pop = G[f"{name}/pop"]
    for t in (1, 2, 3):
        assert (bits(R.O_draft_cost(sk, DEV, pop, t)) == bits(G[f"{name}/cost_t{t}"])).all()


@pytest.mark.parametrize("name", SHAPES)
def test_golden_trace(G, name):
    sk = sketch_of(name)
    sy, pe, sc, tot = o_trace(sk, G[f"{name}/pop"])
    assert (sy == G[f"{name}/trace_symbols"]).all()
    assert (bits(pe) == bits(G[f"{name}/trace_penalties"])).all()
    assert (bits(sc) == bits(G[f"{name}/trace_stmt_cost"])).all()
    assert tot == G[f"{name}/trace_total"][0]


@pytest.mark.parametrize("name", SHAPES)
def test_golden_explore_topk(G, name):
    # explore(op, dev, 1, 64, 2048, RngStream(43)) == random_init + SA + dedup top-K
    sk = sketch_of(name)
    pop = R.O_random_init(sk, 43, 2048)
    cost = R.O_draft_cost(sk, DEV, pop)
    idx, c = R.O_draft_topk(sk, cost, pop, 64)
    assert (bits(c) == bits(G[f"{name}/ex_cost"])).all()
    assert (pop[:, idx] == G[f"{name}/ex_soa"]).all()


@pytest.mark.parametrize("name", SHAPES)
def test_golden_features_scores_select(G, name):
    sk = sketch_of(name)
    st, bl = R.O_features(sk, DEV, G[f"{name}/pop"], np.arange(16))
    assert np.abs(st - G[f"{name}/st"]).max() <= 1e-13 * max(1.0, np.abs(G[f"{name}/st"]).max())
    assert np.abs(bl - G[f"{name}/bl"]).max() <= 1e-13 * max(1.0, np.abs(G[f"{name}/bl"]).max())
    p = G["params_h64"]
    assert (bits(R.O_init_params(64, derive_seed(42, TAG_INIT))) == bits(p)).all()
    sc = R.O_score(p, 64, G[f"{name}/st"], G[f"{name}/bl"])
    assert np.abs(sc - G[f"{name}/score"]).max() <= 1e-12
    sci = R.O_score(p, 64, G[f"{name}/st"], G[f"{name}/bl"], identity=True)
    assert np.abs(sci - G[f"{name}/score_identity_attn"]).max() <= 1e-12
    sel = R.O_select_top(G[f"{name}/score"], G[f"{name}/cost_t3"][:16], None, 5)
    assert (sel == G[f"{name}/sel"]).all()


def test_golden_momentum(G):
    for m in (0.0, 0.5, 0.9, 0.99):
        p = G["moa/phi"].copy()
        R.oracle().tto_momentum_update(R.ptr(p, R.f64p), R.ptr(G["moa/target"], R.f64p), len(p), m)
        assert (bits(p) == bits(G[f"moa/phi_m{m}"])).all()


def test_host_init_params_matches_reference(G):
    # the product's host-side init_params (numpy) == init_params (ranker.cpp:305-326)
    from paper_2402_02361_b200.tiletune import init_params
    assert (bits(init_params(64, derive_seed(42, TAG_INIT))) == bits(G["params_h64"])).all()


def test_oracle_space_and_draws():
    sk = make_sketch(make_gemm(1024, 1024, 1024))
    assert R.oracle().tto_space_size(C.byref(sk)) == 16195608
    assert R.oracle().tto_draws_per_schedule(C.byref(sk)) == 4


@pytest.mark.parametrize("name", SHAPES)
def test_golden_explore_genetic(G, name):
    # explore(op, dev, 8, 64, 128, RngStream(44)): 8 generations of mutate()
    sk = sketch_of(name)
    soa, c = R.O_explore(sk, DEV, 128, 64, 44, 8)
    assert (bits(c) == bits(G[f"{name}/ga_cost"])).all()
    assert (soa == G[f"{name}/ga_soa"]).all()


# ------------------------------------------ live reference (when built here) --

live = pytest.mark.skipif(not R.ref_available(), reason="oracle/_ref not built (no /root/reference here)")


@live
@pytest.mark.parametrize("name", ["gemm1024", "r50_c3x3_64", "r50_c3x3_512", "bert_ffn2", "bert_bmm_pv"])
def test_live_population_cost_explore(name):
    sk = make_sketch(WORKLOADS[name]())
    pop = R.O_random_init(sk, 7, 20000)
    assert (pop == R.R_random_init(sk, 7, 20000)).all()
    assert (bits(R.O_draft_cost(sk, DEV, pop)) == bits(R.R_draft_cost(sk, DEV, pop))).all()
    cost = R.O_draft_cost(sk, DEV, pop)
    idx, c = R.O_draft_topk(sk, cost, pop, 512)
    rs, rc = R.R_explore(sk, DEV, 20000, 512, 7)
    assert (bits(c) == bits(rc)).all() and (pop[:, idx] == rs).all()


@live
@pytest.mark.parametrize("name,n,k,steps", [("gemm1024", 512, 512, 32), ("r50_c3x3_64", 512, 128, 32),
                                            ("bert_ffn1", 300, 1000, 12), ("elementwise", 64, 16, 40),
                                            ("gemm4", 256, 64, 20)])
def test_live_explore_genetic(name, n, k, steps):
    # the reference's real per-round explore: n_steps generations, pool trim, mutate()
    sk = make_sketch(make_gemm(4, 4, 4)) if name == "gemm4" else sketch_of(name)
    soa, c = R.O_explore(sk, DEV, n, k, 11, steps)
    rs, rc = R.R_explore(sk, DEV, n, k, 11, n_steps=steps)
    assert len(c) == len(rc) and (bits(c) == bits(rc)).all() and (soa == rs).all()


@live
def test_live_heavy_duplicates():
    # conv 512@7 at N=65,536 carries 648 duplicate schedules
    sk = make_sketch(make_conv(512, 7, 7, 512, 9))
    pop = R.O_random_init(sk, 42, 65536)
    cost = R.O_draft_cost(sk, DEV, pop)
    idx, c = R.O_draft_topk(sk, cost, pop, 512)
    rs, rc = R.R_explore(sk, DEV, 65536, 512, 42)
    assert (bits(c) == bits(rc)).all() and (pop[:, idx] == rs).all()


@live
@pytest.mark.parametrize("h", [8, 64])
def test_live_scores(h):
    sk = make_sketch(WORKLOADS["r50_c3x3_64"]())
    pop = R.O_random_init(sk, 3, 300)
    idx = np.arange(300)
    st, bl = R.O_features(sk, DEV, pop, idx)
    rst, rbl = R.R_features(sk, DEV, pop, idx)
    assert np.abs(st - rst).max() <= 1e-13 * np.abs(rst).max()
    assert np.abs(bl - rbl).max() <= 1e-13 * np.abs(rbl).max()
    p = R.O_init_params(h, 11)
    assert (bits(p) == bits(R.R_init_params(h, 11))).all()
    assert np.abs(R.O_score(p, h, st, bl) - R.R_score(p, h, rst, rbl)).max() <= 1e-12


# ---- lambda_rank_loss (ranker.cpp:394-441): the oracle against the reference's
# closed forms (test_ranker.cpp "rank loss closed forms") and, live, bit for bit
def test_rank_loss_closed_forms():
    import math
    r = R.O_rank_loss([40.0, 30.0, 20.0, 10.0], [1.0, 2.0, 3.0, 4.0])
    assert r[0] < 1e-4
    loss, g = R.O_rank_loss([0.0, 0.0], [1.0, 2.0])
    g0, g1 = 2.0 - 1.0, 2.0 ** 0.5 - 1.0
    max_dcg = g0 / math.log2(2.0) + g1 / math.log2(3.0)
    w = abs(g0 - g1) * abs(1.0 / math.log2(2.0) - 1.0 / math.log2(3.0)) / max_dcg
    assert abs(loss - w * math.log(2.0)) <= 1e-12 * w * math.log(2.0)
    assert g[0] == -g[1]
    assert R.O_rank_loss([1.0], [1.0]) is None
    assert R.O_rank_loss([1.0, 2.0], [1.0, 0.0]) is None


@pytest.mark.skipif(not R.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("n,ties", [(2, False), (16, False), (64, True), (300, True)])
def test_rank_loss_matches_reference(n, ties):
    rng = np.random.default_rng(n)
    sc = rng.normal(size=n)
    lat = rng.uniform(1e-4, 1e-3, size=n)
    if ties:  # repeated scores and latencies: index tie-breaks and skipped pairs
        sc[::3] = sc[0]
        lat[::4] = lat[1]
    o, r = R.O_rank_loss(sc, lat), R.R_rank_loss(sc, lat)
    assert o[0] == r[0] and (o[1] == r[1]).all()


@pytest.mark.skipif(not R.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", ["gemm1024", "r50_c3x3_64"])
def test_strict_cpu_round_selects_what_the_reference_round_selects(name):
    """bench.py's strict CPU bound (ref_round_strict: the reference's own
    per-schedule functions without explore's string keys) must select the
    same schedules as the reference's round on the same population."""
    import ctypes as C
    from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device
    sk, dev = make_sketch(WORKLOADS[name]()), reference_device()
    n, k, b, seed = 4096, 256, 10, 5
    params = R.R_init_params(64, derive_seed(seed, TAG_INIT))
    sel, sc, cnt, secs = np.zeros(b, np.int64), np.zeros(b), C.c_int64(0), np.zeros(4)
    dsoa, dcost = np.zeros((sk.cols, k), np.int32), np.zeros(k)
    R.check(R.ref().ref_round(C.byref(sk), C.byref(dev), n, k, b, seed, R.ptr(params, R.f64p), 64, 4,
                              R.ptr(sel, R.i64p), R.ptr(sc, R.f64p), R.ptr(dsoa, R.i32p), R.ptr(dcost, R.f64p),
                              C.byref(cnt), R.ptr(secs, R.f64p)))
    pop = R.R_random_init(sk, seed, n)
    sel2 = np.zeros(b, np.int64)
    R.check(R.ref().ref_round_strict(C.byref(sk), C.byref(dev), R.ptr(pop, R.i32p), pop.shape[1], n, k, b,
                                     R.ptr(params, R.f64p), 64, 4, R.ptr(sel2, R.i64p), R.ptr(secs, R.f64p)))
    assert (pop[:, sel2] == dsoa[:, sel]).all()
