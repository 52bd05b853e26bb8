"""PaCM training on the device against the reference's own
train() (ranker.cpp:459-512): the golden run dumped from the compiled
reference (tests/golden: h = 8, 32 records, 2 epochs, batch 16, lr 1e-2)
and, when oracle/_ref is present, live runs at h = 64.

Bar: parameters after training within 1e-12 relative (max |Δ| / max |p|)
and losses within 1e-12 relative: the sums follow the reference's order;
only CUDA vs glibc tanh/exp ulps differ.
"""
import os

import numpy as np
import pytest
import torch

from paper_2402_02361_b200 import tiletune as tt
from paper_2402_02361_b200.types import WORKLOADS, make_sketch, reference_device
from tests import _refs as R

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300)


def test_train_matches_reference_golden(ctx):
    G = np.load(GOLDEN)
    p = torch.from_numpy(G["train/p0"].copy()).cuda()
    st = torch.from_numpy(G["train/st"]).cuda()
    bl = torch.from_numpy(G["train/bl"]).cuda()
    l0, l1 = tt.train(ctx, p, 8, st, bl, G["train/lat"], epochs=2, lr=1e-2, batch=16, seed=99)
    assert rel(p.cpu().numpy(), G["train/p1"]) <= 1e-12
    assert abs(l0 - G["train/loss"][0]) <= 1e-12 * abs(G["train/loss"][0])
    assert abs(l1 - G["train/loss"][1]) <= 1e-12 * abs(G["train/loss"][1])


def test_train_lr_zero_is_identity(ctx):
    G = np.load(GOLDEN)
    p0 = G["train/p0"].copy()
    p = torch.from_numpy(p0.copy()).cuda()
    l0, l1 = tt.train(ctx, p, 8, torch.from_numpy(G["train/st"]).cuda(), torch.from_numpy(G["train/bl"]).cuda(),
                      G["train/lat"], epochs=3, lr=0.0, batch=16, seed=5)
    assert (p.cpu().numpy() == p0).all() and l0 == l1


@pytest.mark.skipif(not R.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("n,batch,identity", [(100, 64, False), (40, 256, False), (60, 32, True)])
def test_train_matches_live_reference(ctx, n, batch, identity):
    import ctypes as C
    sk = make_sketch(WORKLOADS["r50_c3x3_64"]())
    dev = reference_device()
    pop = R.O_random_init(sk, 17, n)
    st, bl = R.O_features(sk, dev, pop, np.arange(n))
    lat = R.O_draft_cost(sk, dev, pop) * (1.0 + 0.1 * np.sin(np.arange(n)))
    p0 = R.O_init_params(64, 23)
    pr = p0.copy()
    l0r, l1r = C.c_double(0), C.c_double(0)
    if identity:
        pytest.skip("ref_train wrapper scores without attention_identity")
    R.check(R.ref().ref_train(R.ptr(pr, R.f64p), 64, st.shape[1], bl.shape[1], R.ptr(st, R.f64p), R.ptr(bl, R.f64p),
                              R.ptr(lat, R.f64p), n, 4, 1e-2, batch, 31, C.byref(l0r), C.byref(l1r)))
    p = torch.from_numpy(p0.copy()).cuda()
    l0, l1 = tt.train(ctx, p, 64, torch.from_numpy(st).cuda(), torch.from_numpy(bl).cuda(), lat, epochs=4, lr=1e-2,
                      batch=batch, seed=31)
    assert rel(p.cpu().numpy(), pr) <= 1e-11
    assert abs(l0 - l0r.value) <= 1e-11 * abs(l0r.value) and abs(l1 - l1r.value) <= 1e-11 * abs(l1r.value)


def test_momentum_adapt_composes(ctx):
    G = np.load(GOLDEN)
    phi = torch.from_numpy(G["train/p0"].copy()).cuda()
    phi0 = phi.clone()
    target, (l0, l1) = tt.momentum_adapt(ctx, phi, 0.99, 8, torch.from_numpy(G["train/st"]).cuda(),
                                         torch.from_numpy(G["train/bl"]).cuda(), G["train/lat"], epochs=2, lr=1e-2,
                                         batch=16, seed=99)
    assert rel(target.cpu().numpy(), G["train/p1"]) <= 1e-12
    want = target.cpu().numpy() + 0.99 * (phi0.cpu().numpy() - target.cpu().numpy())
    assert (phi.cpu().numpy() == want).all()


@pytest.mark.parametrize("n,ties", [(2, False), (16, False), (256, True), (1000, True)])
def test_rank_loss_matches_oracle(ctx, n, ties):
    """tt_rank_loss (device LambdaRank) against the oracle's literal
    ranker.cpp:394-441: the pair terms are the same expressions, only the
    summation order differs (per-item gradient, fixed chunk order), so the
    bar is 1e-13 relative to the largest |gradient| / the loss."""
    rng = np.random.default_rng(100 + n)
    sc = rng.normal(size=n)
    lat = rng.uniform(1e-4, 1e-3, size=n)
    if ties:
        sc[::3] = sc[0]
        lat[::4] = lat[1]
    loss, g = tt.rank_loss(ctx, torch.from_numpy(sc).cuda(), torch.from_numpy(lat).cuda())
    lo, go = R.O_rank_loss(sc, lat)
    assert abs(loss - lo) <= 1e-13 * abs(lo)
    assert np.abs(g.cpu().numpy() - go).max() <= 1e-13 * np.abs(go).max()


def test_rank_loss_closed_forms_and_errors(ctx):
    import math
    loss, g = tt.rank_loss(ctx, torch.tensor([0.0, 0.0], dtype=torch.float64, device="cuda"),
                           torch.tensor([1.0, 2.0], dtype=torch.float64, device="cuda"))
    g0, g1 = 1.0, 2.0 ** 0.5 - 1.0
    max_dcg = g0 / math.log2(2.0) + g1 / math.log2(3.0)
    w = abs(g0 - g1) * abs(1.0 / math.log2(2.0) - 1.0 / math.log2(3.0)) / max_dcg
    assert abs(loss - w * math.log(2.0)) <= 1e-12 * w * math.log(2.0)
    g = g.cpu().numpy()
    assert g[0] == -g[1]  # both endpoints evaluate the same slope
    for sc, lat in [([1.0], [1.0]), ([1.0, 2.0], [1.0, 0.0])]:
        with pytest.raises(tt.TTError) as e:
            tt.rank_loss(ctx, torch.tensor(sc, dtype=torch.float64, device="cuda"),
                         torch.tensor(lat, dtype=torch.float64, device="cuda"))
        assert e.value.code == "E_STATE"
