"""Wire formats of the PaCM parameters: the reference's model
checkpoint (ranker.cpp:265-303, 534-554; JSON, format_version 1) and its
Siamese/MoA checkpoint (momentum.cpp:58-92), so parameters trained or adapted
on the device round-trip into the reference CLI / tuner unchanged.

Parameters are the flattened RankerParams of include/tt/tt_types.h
(for_each_tensor order). Doubles are written in shortest round-trip form,
so save -> load is exact. Errors mirror the reference's codes (E_PARSE,
E_VALIDATE) via TTError.
"""
from __future__ import annotations

import json
import math

import numpy as np

from ._capi import TTError

# for_each_tensor (ranker.cpp:336-353): name, (rows, cols) as functions of h
TENSORS = [("stmt_w1", lambda h: (24, h)), ("stmt_b1", lambda h: (1, h)), ("stmt_w2", lambda h: (h, h)),
           ("stmt_b2", lambda h: (1, h)), ("embed_w", lambda h: (23, h)), ("embed_b", lambda h: (1, h)),
           ("attn_wq", lambda h: (h, h)), ("attn_bq", lambda h: (1, h)), ("attn_wk", lambda h: (h, h)),
           ("attn_bk", lambda h: (1, h)), ("attn_wv", lambda h: (h, h)), ("attn_bv", lambda h: (1, h)),
           ("head_w1", lambda h: (2 * h, h)), ("head_b1", lambda h: (1, h)), ("head_w2", lambda h: (h, 1)),
           ("head_b2", lambda h: (1, 1))]


def _num(x: float) -> str:
    """A JSON number that parses back to exactly x (the reference's json writer
    is also shortest round-trip); non-finite values are not representable."""
    if not math.isfinite(x):
        raise TTError("E_VALIDATE", "checkpoint: non-finite parameter")
    r = repr(float(x))
    return r


def _params_obj(params, h: int) -> str:
    p = np.ascontiguousarray(np.asarray(params, np.float64)).ravel()
    parts, off = [], 0
    for name, shape in TENSORS:
        r, c = shape(h)
        data = ",".join(_num(v) for v in p[off:off + r * c])
        parts.append(f'"{name}":{{"rows":{r},"cols":{c},"data":[{data}]}}')
        off += r * c
    if off != p.size:
        raise TTError("E_STATE", f"checkpoint: {p.size} parameters for hidden width {h}, expected {off}")
    return f'"format_version":1,"hidden":{h},"tensors":{{' + ",".join(parts) + "}"


def serialize_params(params, h: int) -> str:
    """serialize_params (ranker.cpp:534-538)."""
    return "{" + _params_obj(params, h) + "}\n"


def _params_from(j) -> tuple[np.ndarray, int]:
    """params_from_json (ranker.cpp:280-303)."""
    if not isinstance(j, dict) or j.get("format_version") != 1:
        raise TTError("E_PARSE", "model file: unsupported format_version")
    h = j.get("hidden")
    if not isinstance(h, int) or h < 1:
        raise TTError("E_PARSE", "model file: hidden must be >= 1")
    tensors = j.get("tensors")
    if not isinstance(tensors, dict):
        raise TTError("E_PARSE", "model file: missing tensors")
    out = []
    for name, shape in TENSORS:
        if name not in tensors:
            raise TTError("E_PARSE", "model file: missing tensor " + name)
        jt = tensors[name]
        r, c = shape(h)
        if jt.get("rows") != r or jt.get("cols") != c:
            raise TTError("E_PARSE", f"model file: tensor {name} has shape {jt.get('rows')}x{jt.get('cols')}, "
                                     f"expected {r}x{c}")
        data = jt.get("data")
        if not isinstance(data, list) or len(data) != r * c:
            raise TTError("E_PARSE", f"model file: tensor {name} size")
        out.append(np.asarray(data, np.float64))
    return np.concatenate(out), h


def parse_params(text: str) -> tuple[np.ndarray, int]:
    """parse_params (ranker.cpp:540-548): (flattened params, hidden width)."""
    try:
        j = json.loads(text)
    except ValueError as e:
        raise TTError("E_PARSE", f"model file parse failure: {e}") from None
    return _params_from(j)


def serialize_siamese(params, h: int, momentum: float = 0.99, provenance: str = "pretrained") -> str:
    """serialize_siamese (momentum.cpp:58-64)."""
    if provenance not in ("pretrained", "evolved"):
        raise TTError("E_PARSE", "unknown provenance tag " + provenance)
    return "{" + _params_obj(params, h) + f',"momentum":{_num(momentum)},"provenance":"{provenance}"' + "}\n"


def parse_siamese(text: str) -> tuple[np.ndarray, int, float, str]:
    """parse_siamese (momentum.cpp:66-86): (params, hidden, momentum, provenance)."""
    try:
        j = json.loads(text)
    except ValueError as e:
        raise TTError("E_PARSE", f"siamese checkpoint parse failure: {e}") from None
    p, h = _params_from(j)
    m = j.get("momentum", 0.99)
    if not (isinstance(m, (int, float)) and 0.0 <= m < 1.0):
        raise TTError("E_VALIDATE", f"momentum must lie in [0, 1), got {m}")
    prov = j.get("provenance", "pretrained")
    if prov not in ("pretrained", "evolved"):
        raise TTError("E_PARSE", "unknown provenance tag " + str(prov))
    return p, h, float(m), prov


def save_params(params, h: int, path: str) -> None:
    with open(path, "w") as f:
        f.write(serialize_params(params, h))


def load_params(path: str) -> tuple[np.ndarray, int]:
    with open(path) as f:
        return parse_params(f.read())
