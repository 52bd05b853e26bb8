"""Loaders for the CHECKERS: the C restatement (oracle/_build/libtt_oracle.so)
and the compiled reference (oracle/_ref/libtiletune_ref.so).

Test infrastructure only. The product (paper_2402_02361_b200) never imports
this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2402_02361_b200.types import DeviceSpec, OracleSpec, Sketch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "libtt_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libtiletune_ref.so")

P = C.POINTER
i32p, i64p, u64p, f64p, u8p = P(C.c_int32), P(C.c_int64), P(C.c_uint64), P(C.c_double), P(C.c_uint8)


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t) if a is not None else None


_oracle = None
_ref = None


def oracle():
    global _oracle
    if _oracle is None:
        lib = C.CDLL(ORACLE_SO)
        sk, dv = P(Sketch), P(DeviceSpec)
        sig = {
            "tto_derive_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "tto_draws_per_schedule": (C.c_int, [sk]),
            "tto_space_size": (C.c_uint64, [sk]),
            "tto_random_init": (None, [sk, C.c_uint64, C.c_int64, C.c_int64, i32p, C.c_int64]),
            "tto_draft_cost": (None, [sk, dv, i32p, C.c_int64, C.c_int64, C.c_int, f64p]),
            "tto_trace": (C.c_int, [sk, dv, i32p, C.c_int64, C.c_int64, C.c_int, i64p, f64p, f64p, f64p]),
            "tto_identity": (C.c_uint64, [sk, i32p, C.c_int64, C.c_int64, P(C.c_int)]),
            "tto_draft_topk": (C.c_int64, [sk, f64p, i32p, C.c_int64, C.c_int64, C.c_int64, i64p, f64p]),
            "tto_explore": (C.c_int64, [sk, dv, C.c_int, C.c_int64, C.c_int64, C.c_uint64, C.c_int, i32p, f64p]),
            "tto_features": (None, [sk, dv, i32p, C.c_int64, i64p, C.c_int64, f64p, f64p]),
            "tto_init_params": (None, [C.c_int, C.c_uint64, f64p]),
            "tto_score": (None, [f64p, C.c_int, C.c_int, C.c_int, f64p, f64p, C.c_int64, C.c_int, f64p]),
            "tto_select_top": (C.c_int, [f64p, f64p, u8p, C.c_int64, C.c_int64, i64p]),
            "tto_momentum_update": (None, [f64p, f64p, C.c_int64, C.c_double]),
            "tto_gd_step": (None, [f64p, f64p, C.c_int64, C.c_double]),
            "tto_rank_loss": (C.c_int, [f64p, f64p, C.c_int64, f64p, f64p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype, f.argtypes = res, args
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        sk, dv = P(Sketch), P(DeviceSpec)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_random_init": (C.c_int, [sk, C.c_uint64, C.c_int64, i32p, C.c_int64]),
            "ref_draft_cost": (C.c_int, [sk, dv, i32p, C.c_int64, C.c_int64, C.c_int, C.c_int, f64p]),
            "ref_trace": (C.c_int, [sk, dv, i32p, C.c_int64, C.c_int64, i64p, f64p, f64p, f64p]),
            "ref_explore": (C.c_int, [sk, dv, C.c_int, C.c_int64, C.c_int64, C.c_uint64, C.c_int, i32p, f64p, i64p, u64p]),
            "ref_features": (C.c_int, [sk, dv, i32p, C.c_int64, i64p, C.c_int64, f64p, f64p]),
            "ref_init_params": (C.c_int, [C.c_int, C.c_uint64, f64p]),
            "ref_score_batch": (C.c_int, [f64p, C.c_int, C.c_int, C.c_int, f64p, f64p, C.c_int64, C.c_int, C.c_int, f64p, u64p]),
            "ref_select_top": (C.c_int, [f64p, f64p, u8p, C.c_int64, C.c_int64, i64p]),
            "ref_momentum_update": (C.c_int, [f64p, f64p, C.c_int, C.c_double]),
            "ref_rank_loss": (C.c_int, [f64p, f64p, C.c_int64, f64p, f64p]),
            "ref_train": (C.c_int, [f64p, C.c_int, C.c_int, C.c_int, f64p, f64p, f64p, C.c_int64, C.c_int, C.c_double, C.c_int, C.c_uint64, f64p, f64p]),
            "ref_noiseless_latency": (C.c_int, [sk, dv, C.c_double, C.c_double, C.c_double, i32p, C.c_int64, C.c_int64, f64p]),
            "ref_measure": (C.c_int, [sk, P(OracleSpec), i32p, C.c_int64, C.c_int64, C.c_uint64, C.c_uint64, f64p,
                                      f64p]),
            "ref_oracle_best": (C.c_int, [sk, P(OracleSpec), C.c_uint64, i32p, f64p]),
            "ref_round_strict": (C.c_int, [sk, dv, i32p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, f64p, C.c_int,
                                           C.c_int, i64p, f64p]),
            "ref_round": (C.c_int, [sk, dv, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, f64p, C.c_int, C.c_int, i64p, f64p, i32p, f64p, i64p, f64p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype, f.argtypes = res, args
        _ref = lib
    return _ref


def check(rc):
    if rc != 0:
        raise RuntimeError(ref().ref_last_error().decode())


# ---- numpy conveniences over the oracle (O_*) and the reference (R_*) ----

def O_random_init(sk, seed, n, first=0):
    soa = np.zeros((sk.cols, n), np.int32)
    oracle().tto_random_init(C.byref(sk), seed, first, n, ptr(soa, i32p), n)
    return soa


def R_random_init(sk, seed, n):
    soa = np.zeros((sk.cols, n), np.int32)
    check(ref().ref_random_init(C.byref(sk), seed, n, ptr(soa, i32p), n))
    return soa


def O_draft_cost(sk, dev, soa, toggles=3):
    soa = np.ascontiguousarray(soa)
    n = soa.shape[1]
    out = np.zeros(n)
    oracle().tto_draft_cost(C.byref(sk), C.byref(dev), ptr(soa, i32p), n, n, toggles, ptr(out, f64p))
    return out


def R_draft_cost(sk, dev, soa, toggles=3, threads=1):
    soa = np.ascontiguousarray(soa)
    n = soa.shape[1]
    out = np.zeros(n)
    check(ref().ref_draft_cost(C.byref(sk), C.byref(dev), ptr(soa, i32p), n, n, toggles, threads, ptr(out, f64p)))
    return out


def O_identity(sk, soa):
    soa = np.ascontiguousarray(soa)
    ok = C.c_int(0)
    n = soa.shape[1]
    ids = np.array([oracle().tto_identity(C.byref(sk), ptr(soa, i32p), n, i, C.byref(ok)) for i in range(n)], np.uint64)
    return ids, bool(ok.value)


def O_draft_topk(sk, cost, soa, k):
    soa = np.ascontiguousarray(soa)
    n = soa.shape[1]
    idx = np.zeros(k, np.int64)
    c = np.zeros(k)
    m = oracle().tto_draft_topk(C.byref(sk), ptr(cost, f64p), ptr(soa, i32p), n, n, k, ptr(idx, i64p), ptr(c, f64p))
    return idx[:m], c[:m]


def R_explore(sk, dev, n, k, seed, n_steps=1, threads=1):
    soa = np.zeros((sk.cols, k), np.int32)
    cost = np.zeros(k)
    cnt = C.c_int64(0)
    ev = C.c_uint64(0)
    check(ref().ref_explore(C.byref(sk), C.byref(dev), n_steps, k, n, seed, threads, ptr(soa, i32p), ptr(cost, f64p), C.byref(cnt), C.byref(ev)))
    m = cnt.value
    return np.ascontiguousarray(soa[:, :m]), cost[:m]


def O_explore(sk, dev, n, k, seed, n_steps, toggles=3):
    soa = np.zeros((sk.cols, k), np.int32)
    cost = np.zeros(k)
    m = oracle().tto_explore(C.byref(sk), C.byref(dev), n_steps, k, n, seed, toggles, ptr(soa, i32p), ptr(cost, f64p))
    return np.ascontiguousarray(soa[:, :m]), cost[:m]


def O_features(sk, dev, soa, idx):
    soa = np.ascontiguousarray(soa)
    S, B = sk.op.n_statements, sk.op.n_blocks
    idx = np.ascontiguousarray(idx, np.int64)
    st = np.zeros((len(idx), S, 24))
    bl = np.zeros((len(idx), B, 23))
    oracle().tto_features(C.byref(sk), C.byref(dev), ptr(soa, i32p), soa.shape[1], ptr(idx, i64p), len(idx), ptr(st, f64p), ptr(bl, f64p))
    return st, bl


def R_features(sk, dev, soa, idx):
    soa = np.ascontiguousarray(soa)
    S, B = sk.op.n_statements, sk.op.n_blocks
    idx = np.ascontiguousarray(idx, np.int64)
    st = np.zeros((len(idx), S, 24))
    bl = np.zeros((len(idx), B, 23))
    check(ref().ref_features(C.byref(sk), C.byref(dev), ptr(soa, i32p), soa.shape[1], ptr(idx, i64p), len(idx), ptr(st, f64p), ptr(bl, f64p)))
    return st, bl


def O_init_params(h, seed):
    from paper_2402_02361_b200.types import C as _  # noqa: F401
    n = 24 * h + h + h * h + h + 23 * h + h + 3 * (h * h + h) + 2 * h * h + h + h + 1
    p = np.zeros(n)
    oracle().tto_init_params(h, seed, ptr(p, f64p))
    return p


def R_init_params(h, seed):
    n = 24 * h + h + h * h + h + 23 * h + h + 3 * (h * h + h) + 2 * h * h + h + h + 1
    p = np.zeros(n)
    check(ref().ref_init_params(h, seed, ptr(p, f64p)))
    return p


def O_score(params, h, st, bl, identity=False):
    st = np.ascontiguousarray(st)
    bl = np.ascontiguousarray(bl)
    k = st.shape[0]
    out = np.zeros(k)
    oracle().tto_score(ptr(params, f64p), h, st.shape[1], bl.shape[1], ptr(st, f64p), ptr(bl, f64p), k, int(identity), ptr(out, f64p))
    return out


def R_score(params, h, st, bl, identity=False, threads=1):
    st = np.ascontiguousarray(st)
    bl = np.ascontiguousarray(bl)
    k = st.shape[0]
    out = np.zeros(k)
    calls = C.c_uint64(0)
    check(ref().ref_score_batch(ptr(params, f64p), h, st.shape[1], bl.shape[1], ptr(st, f64p), ptr(bl, f64p), k, int(identity), threads, ptr(out, f64p), C.byref(calls)))
    return out


def O_select_top(scores, drafts, excluded, b):
    out = np.zeros(b, np.int64)
    ex = None if excluded is None else np.ascontiguousarray(excluded, np.uint8)
    rc = oracle().tto_select_top(ptr(scores, f64p), ptr(drafts, f64p), ptr(ex, u8p), len(scores), b, ptr(out, i64p))
    if rc != 0:
        raise RuntimeError("select_top: not enough unmeasured candidates")
    return out


def R_select_top(scores, drafts, excluded, b):
    out = np.zeros(b, np.int64)
    ex = None if excluded is None else np.ascontiguousarray(excluded, np.uint8)
    check(ref().ref_select_top(ptr(scores, f64p), ptr(drafts, f64p), ptr(ex, u8p), len(scores), b, ptr(out, i64p)))
    return out


def R_measure(sk, oracle, soa, task_hash, trial0):
    soa = np.ascontiguousarray(soa)
    n = soa.shape[1]
    lat, nl = np.zeros(n), np.zeros(n)
    check(ref().ref_measure(C.byref(sk), C.byref(oracle), ptr(soa, i32p), n, n, task_hash, trial0, ptr(lat, f64p),
                            ptr(nl, f64p)))
    return lat, nl


def R_oracle_best(sk, oracle, cap=1 << 30):
    soa = np.zeros((sk.cols, 1), np.int32)
    lat = C.c_double(0)
    check(ref().ref_oracle_best(C.byref(sk), C.byref(oracle), cap, ptr(soa, i32p), C.byref(lat)))
    return soa, lat.value


def O_rank_loss(scores, lat):
    """lambda_rank_loss via the C restatement: (loss, grad) or None (kState)."""
    scores, lat = np.ascontiguousarray(scores, np.float64), np.ascontiguousarray(lat, np.float64)
    g = np.zeros(len(scores))
    loss = C.c_double(0)
    rc = oracle().tto_rank_loss(ptr(scores, f64p), ptr(lat, f64p), len(scores), C.byref(loss), ptr(g, f64p))
    return None if rc else (loss.value, g)


def R_rank_loss(scores, lat):
    """lambda_rank_loss of the compiled reference: (loss, grad) or None (Error)."""
    scores, lat = np.ascontiguousarray(scores, np.float64), np.ascontiguousarray(lat, np.float64)
    g = np.zeros(len(scores))
    loss = C.c_double(0)
    rc = ref().ref_rank_loss(ptr(scores, f64p), ptr(lat, f64p), len(scores), C.byref(loss), ptr(g, f64p))
    return None if rc else (loss.value, g)
