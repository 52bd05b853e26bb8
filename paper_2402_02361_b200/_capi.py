"""ctypes binding of the C ABI (include/tt/tt.h).

Loads the in-tree sm_100a library paper_2402_02361_b200/_lib/libtt_b200.so.
There is no fallback: a missing library raises, and every compute call
fails with E_CUDA when no GPU is usable.
"""
from __future__ import annotations

import ctypes as C
import os

from .types import DeviceSpec, OpSpec, OracleSpec, Sketch

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libtt_b200.so")

P = C.POINTER
vp = C.c_void_p
i64p = P(C.c_int64)
f64p = P(C.c_double)
u64p = P(C.c_uint64)


class RoundConfig(C.Structure):
    _fields_ = [("n", C.c_int64), ("k", C.c_int64), ("b", C.c_int64), ("toggles", C.c_int32),
                ("precision", C.c_int32), ("band", C.c_double), ("first", C.c_int64)]


class RoundResult(C.Structure):
    _fields_ = [("selected", C.c_int64), ("drafted", C.c_int64), ("rescored", C.c_int64),
                ("status", C.c_int32), ("retries", C.c_int32), ("band_err", C.c_double)]


TT_PREC_FP64, TT_PREC_BF16 = 0, 1
TT_ROUND_BAND_RERUN = 1 << 16
# default certification band for bf16 rounds: a bound on |bf16 - fp64| scores
# at h = 64 (measured max 3.2e-2 on random-init weights)
TT_BF16_BAND = 6e-2

# (name, restype, argtypes) — exactly the declarations of include/tt/tt.h
_SIGS = [
    ("tt_status_code", C.c_char_p, [C.c_int]),
    ("tt_version", C.c_char_p, []),
    ("tt_kernel_launches", C.c_uint64, []),
    ("tt_ctx_create", C.c_int, [C.c_int, P(vp)]),
    ("tt_ctx_destroy", None, [vp]),
    ("tt_last_error", C.c_char_p, [vp]),
    ("tt_ctx_set_stream", C.c_int, [vp, vp]),
    ("tt_ctx_stream", vp, [vp]),
    ("tt_ctx_sync", C.c_int, [vp]),
    ("tt_sketch_from_op", C.c_int, [P(OpSpec), C.c_int, P(Sketch)]),
    ("tt_validate_device", C.c_int, [P(DeviceSpec)]),
    ("tt_space_size", C.c_uint64, [P(Sketch)]),
    ("tt_draws_per_schedule", C.c_int, [P(Sketch)]),
    ("tt_population_generate", C.c_int, [vp, P(Sketch), C.c_uint64, C.c_int64, C.c_int64, vp, C.c_int64, vp]),
    ("tt_schedule_identity", C.c_int, [vp, P(Sketch), vp, C.c_int64, C.c_int64, vp]),
    ("tt_schedule_from_identity", C.c_int, [vp, P(Sketch), vp, C.c_int64, vp, C.c_int64]),
    ("tt_draft_cost", C.c_int, [vp, P(Sketch), P(DeviceSpec), vp, C.c_int64, C.c_int64, C.c_int, vp]),
    ("tt_draft_topk", C.c_int, [vp, P(Sketch), P(DeviceSpec), vp, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                C.c_int64, vp, vp, vp, i64p]),
    ("tt_explore1", C.c_int, [vp, P(Sketch), P(DeviceSpec), C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                              vp, vp, vp, i64p]),
    ("tt_explore", C.c_int, [vp, P(Sketch), P(DeviceSpec), C.c_int, C.c_int64, C.c_int64, C.c_uint64, C.c_int,
                             vp, vp, vp, i64p, C.POINTER(C.c_uint64)]),
    ("tt_draft_set", C.c_int, [vp, P(Sketch), P(DeviceSpec), C.c_int, C.c_int64, C.c_int64, C.c_double, C.c_uint64,
                               C.c_uint64, C.c_int, vp, vp, i64p, C.POINTER(C.c_uint64)]),
    ("tt_tuner_round", C.c_int, [vp, P(Sketch), P(DeviceSpec), C.c_int, C.c_int64, C.c_int64, C.c_double,
                                 C.c_uint64, C.c_uint64, C.c_int64, C.c_int, vp, vp, vp, i64p]),
    ("tt_topk_merge", C.c_int, [vp, vp, vp, vp, C.c_int64, C.c_int64, vp, vp, vp, i64p]),
    ("tt_features", C.c_int, [vp, P(Sketch), P(DeviceSpec), vp, C.c_int64, vp, vp]),
    ("tt_features_soa", C.c_int, [vp, P(Sketch), P(DeviceSpec), vp, C.c_int64, vp, C.c_int64, vp, vp]),
    ("tt_pacm_load", C.c_int, [vp, vp, C.c_int]),
    ("tt_pacm_score", C.c_int, [vp, P(Sketch), P(DeviceSpec), vp, C.c_int64, C.c_int, vp]),
    ("tt_pacm_score_features", C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int64, C.c_int, vp]),
    ("tt_forward_calls", C.c_uint64, []),
    ("tt_reset_forward_calls", None, []),
    ("tt_select_top", C.c_int, [vp, vp, vp, vp, C.c_int64, C.c_int64, i64p]),
    ("tt_oracle_latency", C.c_int, [vp, P(Sketch), P(OracleSpec), vp, C.c_int64, C.c_int64, vp]),
    ("tt_oracle_measure", C.c_int, [vp, P(Sketch), P(OracleSpec), vp, C.c_int64, C.c_int64, C.c_uint64, C.c_uint64,
                                    vp, vp]),
    ("tt_oracle_best", C.c_int, [vp, P(Sketch), P(OracleSpec), u64p, f64p]),
    ("tt_pacm_train", C.c_int, [vp, vp, C.c_int, vp, vp, C.c_int, C.c_int, f64p, C.c_int64, C.c_int, C.c_double,
                                 C.c_int, C.c_uint64, C.c_int, f64p, f64p]),
    ("tt_rank_loss", C.c_int, [vp, vp, vp, C.c_int64, f64p, vp]),
    ("tt_gd_step", C.c_int, [vp, vp, vp, C.c_int64, C.c_double]),
    ("tt_momentum_update", C.c_int, [vp, vp, vp, C.c_int64, C.c_double]),
    ("tt_round", C.c_int, [vp, P(Sketch), P(DeviceSpec), P(RoundConfig), vp, C.c_int64, C.c_uint64, i64p, f64p,
                           f64p, u64p, P(RoundResult)]),
    ("tt_round_async", C.c_int, [vp, P(Sketch), P(DeviceSpec), P(RoundConfig), vp, C.c_int64, C.c_uint64]),
    ("tt_round_collect", C.c_int, [vp, C.c_int64, i64p, f64p, f64p, u64p, P(RoundResult)]),
    ("tt_round_finish_merged", C.c_int, [vp, P(Sketch), P(DeviceSpec), P(RoundConfig), vp, vp, vp, C.c_int64,
                                         i64p, f64p, f64p, u64p, P(RoundResult)]),
    ("tt_round_drafted", C.c_int, [vp, P(vp), P(vp), P(vp), P(vp)]),
    ("tt_round_local_async", C.c_int, [vp, P(Sketch), P(DeviceSpec), P(RoundConfig), vp, C.c_int64, C.c_uint64,
                                       vp, vp, vp]),
    ("tt_comm_unique_id", C.c_int, [vp]),
    ("tt_comm_init", C.c_int, [vp, C.c_int, C.c_int, vp]),
    ("tt_comm_destroy", C.c_int, [vp]),
    ("tt_round_sharded", C.c_int, [vp, P(Sketch), P(DeviceSpec), P(RoundConfig), vp, C.c_int64, C.c_uint64,
                                   i64p, f64p, f64p, u64p, P(RoundResult)]),
    ("tt_round_local", C.c_int, [vp, P(Sketch), P(DeviceSpec), P(RoundConfig), vp, C.c_int64, C.c_uint64,
                                 vp, vp, vp]),
    ("tt_round_finish_merged_async", C.c_int, [vp, P(Sketch), P(DeviceSpec), P(RoundConfig), vp, vp, vp,
                                               C.c_int64]),
    ("tt_profile_enable", C.c_int, [vp, C.c_int]),
    ("tt_profile_read", C.c_int, [vp, f64p, i64p, C.c_int]),
]

EXPORTED = [name for name, _, _ in _SIGS]

_lib = None


def lib():
    """The loaded library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2402_02361_b200.build` "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in _SIGS:
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


class TTError(RuntimeError):
    """A non-zero tt status; .code is the reference's code string (E_VALIDATE, ...)."""

    def __init__(self, code: str, message: str):
        super().__init__(f"{code}: {message}")
        self.code = code
