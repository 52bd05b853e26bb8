"""Wire formats (CPU): the model and Siamese checkpoints
written here load in the reference (oracle/_ref: parse_params /
parse_siamese) to the same bits and vice versa, and round-trip exactly
(test_ranker.cpp:290-297, test_momentum.cpp:161-172). Error codes mirror
the reference's.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2402_02361_b200 import checkpoint as ck
from paper_2402_02361_b200._capi import TTError
from paper_2402_02361_b200.tiletune import init_params
from tests import _refs as R

live = pytest.mark.skipif(not R.ref_available(), reason="oracle/_ref not built")


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def _ref_fn(name, res, args):
    f = getattr(R.ref(), name)
    f.restype, f.argtypes = res, args
    return f


def ref_serialize(p, h, siamese=None):
    buf = C.create_string_buffer(1 << 22)
    n = C.c_int64(0)
    if siamese is None:
        f = _ref_fn("ref_serialize_params", C.c_int, [R.f64p, C.c_int, C.c_char_p, C.c_int64, R.i64p])
        R.check(f(R.ptr(p, R.f64p), h, buf, len(buf), C.byref(n)))
    else:
        m, ev = siamese
        f = _ref_fn("ref_serialize_siamese", C.c_int, [R.f64p, C.c_int, C.c_double, C.c_int, C.c_char_p, C.c_int64,
                                                        R.i64p])
        R.check(f(R.ptr(p, R.f64p), h, m, int(ev), buf, len(buf), C.byref(n)))
    return buf.value.decode()


def ref_parse(text, n_params, siamese=False):
    p = np.zeros(n_params)
    h = C.c_int(0)
    if not siamese:
        f = _ref_fn("ref_parse_params", C.c_int, [C.c_char_p, R.f64p, C.POINTER(C.c_int)])
        R.check(f(text.encode(), R.ptr(p, R.f64p), C.byref(h)))
        return p, h.value
    m, ev = C.c_double(0), C.c_int(0)
    f = _ref_fn("ref_parse_siamese", C.c_int, [C.c_char_p, R.f64p, C.POINTER(C.c_int), C.POINTER(C.c_double),
                                               C.POINTER(C.c_int)])
    R.check(f(text.encode(), R.ptr(p, R.f64p), C.byref(h), C.byref(m), C.byref(ev)))
    return p, h.value, m.value, "evolved" if ev.value else "pretrained"


@pytest.mark.parametrize("h", [1, 8, 64])
def test_params_round_trip_exact(h):
    p = init_params(h, 107) * 1.2345678901234567 + 1e-310  # subnormals and full mantissas
    q, h2 = ck.parse_params(ck.serialize_params(p, h))
    assert h2 == h and (bits(q) == bits(p)).all()


@live
@pytest.mark.parametrize("h", [8, 64])
def test_params_interchange_with_reference(h):
    p = init_params(h, 11) * np.pi
    ours = ck.serialize_params(p, h)
    q, h2 = ref_parse(ours, p.size)
    assert h2 == h and (bits(q) == bits(p)).all()
    theirs = ref_serialize(p, h)
    r, h3 = ck.parse_params(theirs)
    assert h3 == h and (bits(r) == bits(p)).all()


@live
def test_siamese_interchange_with_reference():
    p = init_params(16, 3)
    for m, prov in [(0.99, "pretrained"), (0.5, "evolved")]:
        q, h, m2, prov2 = ref_parse(ck.serialize_siamese(p, 16, m, prov), p.size, siamese=True)
        assert (bits(q) == bits(p)).all() and h == 16 and m2 == m and prov2 == prov
        r, h3, m3, prov3 = ck.parse_siamese(ref_serialize(p, 16, (m, prov == "evolved")))
        assert (bits(r) == bits(p)).all() and h3 == 16 and m3 == m and prov3 == prov


def test_checkpoint_errors():
    with pytest.raises(TTError) as e:
        ck.parse_params('{"format_version":2}')
    assert e.value.code == "E_PARSE"
    with pytest.raises(TTError) as e:
        ck.parse_params("not json")
    assert e.value.code == "E_PARSE"
    bad = ck.serialize_params(init_params(4, 1), 4).replace('"rows":24', '"rows":23', 1)
    with pytest.raises(TTError) as e:
        ck.parse_params(bad)
    assert e.value.code == "E_PARSE"
    with pytest.raises(TTError) as e:
        ck.parse_siamese(ck.serialize_siamese(init_params(4, 1), 4, 0.5).replace('"momentum":0.5', '"momentum":1.5'))
    assert e.value.code == "E_VALIDATE"


@live
@pytest.mark.parametrize("h", [8, 64])
def test_params_text_layout_matches_reference(h):
    # nlohmann::json's number layout (plain notation for decimal-point
    # positions in (-4, 15], else d.ddde+XX): byte-identical text on values
    # whose shortest digits are unique. (For arbitrary doubles the reference's
    # Grisu2 may pick a different last digit of equal length; both texts parse
    # to the same bits — test_params_interchange_with_reference.)
    nice = np.array([1.0, 1e-5, 1234567890123456.0, 1e15, 123.25, -0.0, 5e-324, 1e300, 0.1, 2.5e-7, 100.0, -3.0e16,
                     0.001, 123456789012345.0])
    n = init_params(h, 5).size
    p = nice[np.arange(n) % nice.size] * np.where(np.arange(n) % 3 == 0, -1.0, 1.0)
    assert ck.serialize_params(p, h) == ref_serialize(p, h)
    assert ck.serialize_siamese(p, h, 0.5, "evolved") == ref_serialize(p, h, (0.5, True))


# ------------------------------------------------------- records JSONL --

def _records(sk, n, seed):
    rng = np.random.default_rng(seed)
    soa = R.O_random_init(sk, seed, n)
    cols = [soa[:, i].tolist() for i in range(n)]
    nice = [0.00025, 1.5e-6, 3.0, 1234567890123456.0, 1e16, 0.125, 7e-5, 42.0]
    recs = [{"task": "op", "round": int(i // 3), "schedule": cols[i],
             "latency_s": float(rng.lognormal(-8, 2)), "draft_cost": float(rng.random() * 10.0 ** int(rng.integers(-6, 18))),
             "model_score": float(rng.normal())} for i in range(n)]
    seen, out = set(), []
    for r in recs:  # the reference rejects duplicate (task, schedule) pairs
        if tuple(r["schedule"]) not in seen:
            seen.add(tuple(r["schedule"]))
            out.append(r)
    for i in range(0, len(out), 2):  # values with unique shortest digits: byte-identical text expected
        out[i].update(latency_s=nice[i % 8], draft_cost=nice[(i + 3) % 8], model_score=-nice[(i + 5) % 8])
    return out


def _names(sk):
    # the axis names the reference wrapper (oracle/ref_capi.cpp) gives the op
    return [f"s{a}" for a in range(sk.op.n_spatial)] + [f"r{r}" for r in range(sk.op.n_reduction)]


def ref_records_to_jsonl(sk, recs):
    n = len(recs)
    soa = np.ascontiguousarray(np.array([r["schedule"] for r in recs], np.int32).T)
    rounds = np.array([r["round"] for r in recs], np.int32)
    lat, dc, ms = (np.array([r[k] for r in recs]) for k in ("latency_s", "draft_cost", "model_score"))
    buf = C.create_string_buffer(1 << 22)
    ln = C.c_int64(0)
    f = _ref_fn("ref_records_to_jsonl", C.c_int, [C.c_void_p, C.c_char_p, R.i32p, C.c_int64, C.c_int64, R.i32p,
                                                   R.f64p, R.f64p, R.f64p, C.c_char_p, C.c_int64, R.i64p])
    R.check(f(C.byref(sk), b"op", R.ptr(soa, R.i32p), n, n, R.ptr(rounds, R.i32p), R.ptr(lat, R.f64p),
              R.ptr(dc, R.f64p), R.ptr(ms, R.f64p), buf, len(buf), C.byref(ln)))
    return buf.value.decode()


def ref_records_from_jsonl(sk, text, cap):
    soa = np.zeros((sk.cols, cap), np.int32)
    rounds = np.zeros(cap, np.int32)
    lat, dc, ms = np.zeros(cap), np.zeros(cap), np.zeros(cap)
    n = C.c_int64(0)
    f = _ref_fn("ref_records_from_jsonl", C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p, R.i32p, C.c_int64, R.i32p,
                                                     R.f64p, R.f64p, R.f64p, C.c_int64, R.i64p])
    rc = f(C.byref(sk), b"op", text.encode(), R.ptr(soa, R.i32p), cap, R.ptr(rounds, R.i32p), R.ptr(lat, R.f64p),
           R.ptr(dc, R.f64p), R.ptr(ms, R.f64p), cap, C.byref(n))
    if rc:
        return None
    m = n.value
    return [{"task": "op", "round": int(rounds[i]), "schedule": soa[:, i].tolist(), "latency_s": float(lat[i]),
             "draft_cost": float(dc[i]), "model_score": float(ms[i])} for i in range(m)]


@live
@pytest.mark.parametrize("name", ["gemm1024", "r50_c3x3_64", "elementwise"])
def test_records_jsonl_interchange_with_reference(name):
    from paper_2402_02361_b200.types import WORKLOADS, make_elementwise, make_sketch
    sk = make_sketch(make_elementwise(64, 48) if name == "elementwise" else WORKLOADS[name]())
    recs = _records(sk, 40, 9)
    tasks = {"op": (sk, _names(sk))}
    ours = ck.records_to_jsonl(recs, tasks)
    theirs = ref_records_to_jsonl(sk, recs)
    # byte-identical lines where every double has unique shortest digits (even
    # records); elsewhere the reference's Grisu2 may pick another last digit
    for i, (lo, lt) in enumerate(zip(ours.splitlines(), theirs.splitlines())):
        if i % 2 == 0:
            assert lo == lt
    assert ck.records_from_jsonl(ours, tasks) == recs  # our text, our parser: exact
    assert ck.records_from_jsonl(theirs, tasks) == recs  # their text, our parser: exact
    assert ref_records_from_jsonl(sk, ours, len(recs) + 1) == recs  # our text, their parser: exact


@live
def test_records_jsonl_errors_match_reference():
    from paper_2402_02361_b200.types import make_gemm, make_sketch
    sk = make_sketch(make_gemm(64, 64, 64))
    tasks = {"op": (sk, _names(sk))}
    recs = _records(sk, 4, 2)
    good = ck.records_to_jsonl(recs, tasks)
    dup = good + good.splitlines()[0] + "\n"
    bad_sched = good.replace('"unroll":', '"unroll":3', 1)  # 1 -> 31 / 4 -> 34 / 16 -> 316: not a choice
    unknown = good.replace('"task":"op"', '"task":"zz"', 1)
    for text, code in [(dup, "E_VALIDATE"), (bad_sched, "E_VALIDATE"), (unknown, "E_PARSE"), ("{oops\n", "E_PARSE")]:
        with pytest.raises(TTError) as e:
            ck.records_from_jsonl(text, tasks)
        assert e.value.code == code
        assert ref_records_from_jsonl(sk, text, 16) is None  # the reference rejects it too


@live
def test_records_jsonl_axis_structure_matches_reference():
    """validate_schedule's per-axis rules (schedule.cpp:242-278): 4 factors per
    spatial axis, 3 per reduction axis (a shifted list with the right total is
    rejected), and element-wise (arity-2) slots admit only (b, t, 1, 1)."""
    import json as _json

    from paper_2402_02361_b200.types import make_elementwise, make_gemm, make_sketch
    sk = make_sketch(make_gemm(64, 64, 64))
    names = _names(sk)
    tasks = {"op": (sk, names)}
    line = ck.records_to_jsonl(_records(sk, 1, 3), tasks).splitlines()[0]
    j = _json.loads(line)
    ax = j["schedule"]["axes"]
    a0, a1 = names[0], names[1]
    ax[a0], ax[a1] = ax[a0] + [1], ax[a1][:3]  # products unchanged, tuple sizes 5 and 3
    shifted = _json.dumps(j, separators=(",", ":")) + "\n"
    esk = make_sketch(make_elementwise(64, 48))
    enames = _names(esk)
    etasks = {"op": (esk, enames)}
    je = _json.loads(ck.records_to_jsonl(_records(esk, 1, 3), etasks).splitlines()[0])
    e0 = je["schedule"]["axes"][enames[0]]
    je["schedule"]["axes"][enames[0]] = [1, 1, e0[0] * e0[1], 1]  # extent 64 in the o slot
    degenerate = _json.dumps(je, separators=(",", ":")) + "\n"
    for s_, t_, text in [(sk, tasks, shifted), (esk, etasks, degenerate)]:
        with pytest.raises(TTError) as e:
            ck.records_from_jsonl(text, t_)
        assert e.value.code == "E_VALIDATE"
        assert ref_records_from_jsonl(s_, text, 4) is None
