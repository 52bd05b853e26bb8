"""Wire formats: the reference's model checkpoint
(ranker.cpp:265-303, 534-554; JSON, format_version 1), its Siamese/MoA
checkpoint (momentum.cpp:58-92) and its measurement records JSONL
(tuner.cpp:577-645), so parameters and records produced on the device
round-trip into the reference CLI / tuner unchanged.

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
from .types import TT_OP_ELEMENTWISE

# for_each_tensor (ranker.cpp:336-353): name, (rows, cols) as functions of h
TENSORS = [("stmt_w1", lambda h: (24, h)), ("stmt_b1", lambda h: (1, h)), ("stmt_w2", lambda h: (h, h)),
           ("stmt_b2", lambda h: (1, h)), ("embed_w", lambda h: (23, h)), ("embed_b", lambda h: (1, h)),
           ("attn_wq", lambda h: (h, h)), ("attn_bq", lambda h: (1, h)), ("attn_wk", lambda h: (h, h)),
           ("attn_bk", lambda h: (1, h)), ("attn_wv", lambda h: (h, h)), ("attn_bv", lambda h: (1, h)),
           ("head_w1", lambda h: (2 * h, h)), ("head_b1", lambda h: (1, h)), ("head_w2", lambda h: (h, 1)),
           ("head_b2", lambda h: (1, 1))]


def _num(x: float) -> str:
    """x as the reference's JSON writer prints a double: the shortest digits
    that round-trip (as Python's repr), laid out by nlohmann::json's rules —
    plain notation for decimal-point positions -4 < n <= 15, else d.ddde+XX.
    Non-finite values are not representable."""
    if not math.isfinite(x):
        raise TTError("E_VALIDATE", "checkpoint: non-finite parameter")
    r = repr(float(x))
    sign = "-" if r.startswith("-") else ""
    r = r.lstrip("-")
    mant, _, exp = r.partition("e")
    whole, _, frac = mant.partition(".")
    digits = (whole + frac).lstrip("0")
    e10 = int(exp or 0) + len(whole)  # decimal-point position of whole.frac
    if not digits:  # zero
        return sign + "0.0"
    e10 -= len(whole + frac) - len((whole + frac).lstrip("0"))
    digits = digits.rstrip("0")
    k, n = len(digits), e10
    if k <= n <= 15:
        body = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        body = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        body = "0." + "0" * (-n) + digits
    else:
        e = n - 1
        body = digits[0] + ("." + digits[1:] if k > 1 else "") + "e" + ("-" if e < 0 else "+") + f"{abs(e):02d}"
    return sign + body


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


# ------------------------------------------------------------ records --
# A record: {"task": str, "round": int, "schedule": int sequence in the
# tt_types.h column order (4 per spatial axis, 3 per reduction axis, unroll),
# "latency_s", "draft_cost", "model_score": float}. `tasks` maps a task name to
# (sketch, axis names: spatial then reduction, as the op declares them).

def records_to_jsonl(records, tasks) -> str:
    """records_to_jsonl (tuner.cpp:577-601): one JSON object per line."""
    out = []
    for rec in records:
        if rec["task"] not in tasks:
            raise TTError("E_STATE", "record references unknown task " + rec["task"])
        sk, names = tasks[rec["task"]]
        n_sp, n_red = sk.op.n_spatial, sk.op.n_reduction
        f = [int(v) for v in rec["schedule"]]
        axes = []
        for a in range(n_sp):
            axes.append(f'{json.dumps(names[a])}:[{",".join(str(v) for v in f[4 * a:4 * a + 4])}]')
        for r in range(n_red):
            c = 4 * n_sp + 3 * r
            axes.append(f'{json.dumps(names[n_sp + r])}:[{",".join(str(v) for v in f[c:c + 3])}]')
        out.append(f'{{"task":{json.dumps(rec["task"])},"round":{int(rec["round"])},'
                   f'"schedule":{{"axes":{{{",".join(axes)}}},"unroll":{f[4 * n_sp + 3 * n_red]}}},'
                   f'"latency_s":{_num(rec["latency_s"])},"draft_cost":{_num(rec["draft_cost"])},'
                   f'"model_score":{_num(rec["model_score"])}}}\n')
    return "".join(out)


def _valid(sk, f) -> bool:
    """validate_schedule (schedule.cpp:242-278): every axis' factors multiply
    to its extent, element-wise (arity-2) spatial slots are (b, t, 1, 1),
    unroll is one of the sketch's choices."""
    n_sp, n_red = sk.op.n_spatial, sk.op.n_reduction
    for a in range(n_sp + n_red):
        c, w = (4 * a, 4) if a < n_sp else (4 * n_sp + 3 * (a - n_sp), 3)
        if any(v < 1 for v in f[c:c + w]) or math.prod(f[c:c + w]) != sk.op.extent[a]:
            return False
        if a < n_sp and sk.op.kind == TT_OP_ELEMENTWISE and (f[c + 2] != 1 or f[c + 3] != 1):
            return False
    return f[4 * n_sp + 3 * n_red] in [sk.unroll[u] for u in range(sk.n_unroll)]


def records_from_jsonl(text: str, tasks) -> list:
    """records_from_jsonl (tuner.cpp:603-645): parse, validate each schedule,
    reject duplicate (task, schedule) pairs (E_VALIDATE) and unknown tasks
    (E_PARSE)."""
    records, seen = [], set()
    for lineno, line in enumerate(text.split("\n"), 1):
        if not line:
            continue
        try:
            j = json.loads(line)
            task = j["task"]
        except (ValueError, KeyError, TypeError) as e:
            raise TTError("E_PARSE", f"records line {lineno}: {e}") from None
        if task not in tasks:
            raise TTError("E_PARSE", f"records line {lineno}: unknown task {task}")
        sk, names = tasks[task]
        n_sp, n_red = sk.op.n_spatial, sk.op.n_reduction
        try:
            axes = j["schedule"]["axes"]
            f = []
            for a in range(n_sp + n_red):
                tup = [int(v) for v in axes[names[a]]]
                if len(tup) != (4 if a < n_sp else 3):  # schedule.cpp:249,265: 4 per spatial, 3 per reduction
                    raise TTError("E_VALIDATE", f"records line {lineno}: axis {names[a]} has {len(tup)} factors")
                f += tup
            f.append(int(j["schedule"]["unroll"]))
            rec = {"task": task, "round": int(j["round"]), "schedule": f, "latency_s": float(j["latency_s"]),
                   "draft_cost": float(j["draft_cost"]), "model_score": float(j["model_score"])}
        except (KeyError, TypeError, ValueError) as e:
            raise TTError("E_PARSE", f"records line {lineno}: {e}") from None
        if len(f) != sk.cols or not _valid(sk, f):
            raise TTError("E_VALIDATE", f"records line {lineno}: schedule does not satisfy validate_schedule")
        key = (task, tuple(f))
        if key in seen:
            raise TTError("E_VALIDATE", f"records line {lineno}: duplicate (task, schedule) pair")
        seen.add(key)
        records.append(rec)
    return records
