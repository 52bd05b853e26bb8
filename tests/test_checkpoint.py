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
