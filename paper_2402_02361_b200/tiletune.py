"""Host-side mirror of the reference tiletune API for the draft+verify path.

Names, argument meaning and error behaviour follow the reference's free
functions (proj/core/include/tiletune/*.hpp) so call sites read the same;
data lives on the GPU (torch tensors as device memory) and every compute
call goes through the C ABI (include/tt/tt.h) into sm_100a kernels.

    reference                              here
    random_init(sketch, n, rng)            random_init(ctx, sketch, n, seed)
    draft_cost(sketch, s, dev).total       draft_cost(ctx, sketch, dev, population)
    explore(op, dev, 1, K, N, rng)         explore1(ctx, sketch, dev, seed, N, K)
    extract_features(sketch, s, dev)       extract_features(ctx, sketch, dev, identities)
    score_batch(params, feats)             PaCM.score_batch / PaCM.score
    select_top(scores, drafts, excl, b)    select_top(ctx, scores, drafts, excluded, b)
    momentum_update(state, target)         momentum_update(ctx, phi, target, m)
    train's GD update                      gd_step(ctx, params, grads, lr)
    Engine::round_draft_verify             draft_verify_round(ctx, ...)
"""
from __future__ import annotations

import collections
import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi
from ._capi import TTError, RoundConfig, RoundResult, TT_BF16_BAND, TT_PREC_BF16, TT_PREC_FP64, TT_ROUND_BAND_RERUN, lib
from .types import DeviceSpec, OpSpec, OracleSpec, Sketch, TT_TOGGLES_ALL

__all__ = ["Context", "TTError", "TT_PREC_FP64", "TT_PREC_BF16", "random_init", "draft_cost", "draft_topk",
           "explore1", "explore", "draft_set", "tuner_round", "topk_merge", "schedule_identity", "schedule_from_identity", "extract_features",
           "extract_features_soa", "PaCM", "select_top", "gd_step", "momentum_update", "draft_verify_round",
           "init_params", "param_count", "generate_sketch", "forward_calls", "reset_forward_calls",
           "oracle_latency", "oracle_measure", "oracle_best", "train", "momentum_adapt"]


def _p(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


class Context:
    """Owns a tt_ctx (stream + scratch) on one GPU. By default it adopts
    torch's current stream so torch-allocated buffers are ordered with the
    kernels."""

    def __init__(self, device: int = 0, use_torch_stream: bool = True):
        self.device = device
        h = C.c_void_p()
        rc = lib().tt_ctx_create(device, C.byref(h))
        if rc != 0:
            raise TTError(lib().tt_status_code(rc).decode(), f"tt_ctx_create({device}) failed (no usable CUDA device?)")
        self.h = h
        self.torch_device = torch.device("cuda", device)
        # gathered lists of merged rounds in flight (the device reads them until
        # the round is collected); None for the rounds that need nothing kept
        self._inflight = collections.deque()
        if use_torch_stream:
            s = torch.cuda.current_stream(self.torch_device)
            # torch's default stream has handle 0 = the legacy default stream;
            # pass cudaStreamLegacy (0x1) explicitly (NULL means "ctx stream")
            self.check(lib().tt_ctx_set_stream(self.h, C.c_void_p(s.cuda_stream or 1)))

    def stream_handle(self) -> int:
        """The raw cudaStream_t this context enqueues on."""
        return int(lib().tt_ctx_stream(self.h) or 0)

    def check(self, rc: int):
        if rc != 0:
            raise TTError(lib().tt_status_code(rc).decode(), lib().tt_last_error(self.h).decode())

    def sync(self):
        self.check(lib().tt_ctx_sync(self.h))

    def close(self):
        if getattr(self, "h", None):
            lib().tt_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def empty(self, shape, dtype):
        return torch.empty(shape, dtype=dtype, device=self.torch_device)


def generate_sketch(op: OpSpec, elementwise_fallback: bool = True) -> Sketch:
    """generate_sketch (schedule.cpp:150-164) incl. validate_op."""
    sk = Sketch()
    rc = lib().tt_sketch_from_op(C.byref(op), int(elementwise_fallback), C.byref(sk))
    if rc != 0:
        raise TTError(lib().tt_status_code(rc).decode(), "generate_sketch: invalid op"
                      if rc != 2 or op.kind == 0 or elementwise_fallback else "elementwise ops take the trivial sketch")
    return sk


def random_init(ctx: Context, sketch: Sketch, n: int, seed: int, first: int = 0,
                with_identity: bool = False):
    """random_init(sketch, n, RngStream(seed)) schedules [first, first+n) as
    int32 SoA [cols, n] on the GPU (+ identities)."""
    soa = ctx.empty((sketch.cols, n), torch.int32)
    ids = ctx.empty((n,), torch.int64) if with_identity else None
    ctx.check(lib().tt_population_generate(ctx.h, C.byref(sketch), seed & (2**64 - 1), first, n, _p(soa), n, _p(ids)))
    return (soa, ids) if with_identity else soa


def schedule_identity(ctx: Context, sketch: Sketch, soa: torch.Tensor) -> torch.Tensor:
    n = soa.shape[1]
    ids = ctx.empty((n,), torch.int64)
    ctx.check(lib().tt_schedule_identity(ctx.h, C.byref(sketch), _p(soa), soa.stride(0), n, _p(ids)))
    return ids


def schedule_from_identity(ctx: Context, sketch: Sketch, ids: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """schedule_from_key's replacement: exact identities -> SoA factor columns (async)."""
    n = ids.shape[0]
    soa = ctx.empty((sketch.cols, n), torch.int32) if out is None else out
    ctx.check(lib().tt_schedule_from_identity(ctx.h, C.byref(sketch), _p(ids), n, _p(soa), n))
    return soa


def draft_cost(ctx: Context, sketch: Sketch, dev: DeviceSpec, soa: torch.Tensor,
               toggles: int = TT_TOGGLES_ALL) -> torch.Tensor:
    """draft_cost(...).total per schedule (draft.cpp:129-154), bit-exact fp64."""
    n = soa.shape[1]
    out = ctx.empty((n,), torch.float64)
    ctx.check(lib().tt_draft_cost(ctx.h, C.byref(sketch), C.byref(dev), _p(soa), soa.stride(0), n, toggles, _p(out)))
    return out


def _topk_out(ctx, k):
    return ctx.empty((k,), torch.int64), ctx.empty((k,), torch.float64), ctx.empty((k,), torch.int64)


def draft_topk(ctx: Context, sketch: Sketch, dev: DeviceSpec, soa: torch.Tensor, k: int,
               toggles: int = TT_TOGGLES_ALL, index_base: int = 0):
    """explore(n_steps=1) PriorFilter over an explicit population: the k
    lowest unique schedules by (cost, first index). Returns (index, cost,
    identity) trimmed to the unique count."""
    idx, cost, ids = _topk_out(ctx, k)
    cnt = C.c_int64(0)
    ctx.check(lib().tt_draft_topk(ctx.h, C.byref(sketch), C.byref(dev), _p(soa), soa.stride(0), soa.shape[1], k,
                                  toggles, index_base, _p(idx), _p(cost), _p(ids), C.byref(cnt)))
    m = cnt.value
    return idx[:m], cost[:m], ids[:m]


def explore1(ctx: Context, sketch: Sketch, dev: DeviceSpec, seed: int, n: int, k: int, first: int = 0,
             toggles: int = TT_TOGGLES_ALL):
    """explore(op, dev, 1, k, n, RngStream(seed)) over the counter-based
    population, fused (never materialised)."""
    idx, cost, ids = _topk_out(ctx, k)
    cnt = C.c_int64(0)
    ctx.check(lib().tt_explore1(ctx.h, C.byref(sketch), C.byref(dev), seed & (2**64 - 1), first, n, k, toggles,
                                _p(idx), _p(cost), _p(ids), C.byref(cnt)))
    m = cnt.value
    return idx[:m], cost[:m], ids[:m]


def explore(ctx: Context, sketch: Sketch, dev: DeviceSpec, n_steps: int, draft_size: int, pop_size: int, seed: int,
            toggles: int = TT_TOGGLES_ALL, with_soa: bool = True):
    """explore(op, dev, n_steps, draft_size, pop_size, RngStream(seed), toggles)
    (draft.cpp:156-221): the genetic draft loop. Returns host numpy arrays
    (soa [cols, count] int32, cost [count], identity [count] uint64,
    evaluations), sorted by (cost, discovery) like ExploreResult.drafted.
    with_soa=False returns soa None: the identities already encode every
    schedule exactly (schedule_from_identity)."""
    cols = sketch.cols
    soa = np.zeros((cols, draft_size), np.int32)
    cost = np.zeros(draft_size, np.float64)
    ids = np.zeros(draft_size, np.uint64)
    cnt, ev = C.c_int64(0), C.c_uint64(0)
    ctx.check(lib().tt_explore(ctx.h, C.byref(sketch), C.byref(dev), n_steps, draft_size, pop_size,
                               seed & (2**64 - 1), toggles, soa.ctypes.data if with_soa else None, cost.ctypes.data,
                               ids.ctypes.data, C.byref(cnt), C.byref(ev)))
    m = cnt.value
    return (np.ascontiguousarray(soa[:, :m]) if with_soa else None), cost[:m], ids[:m], ev.value


def draft_set(ctx: Context, sketch: Sketch, dev: DeviceSpec, n_steps: int, draft_size: int, pop_size: int,
              random_mix: float, explore_seed: int, mix_seed: int, toggles: int = TT_TOGGLES_ALL):
    """Tuner::build_draft_set (tuner.cpp:294-323): the GA explore pool of
    n_spec schedules then the unseen random-mix schedules. Returns host numpy
    (identity uint64 [count], draft cost [count], evaluations)."""
    ids = np.zeros(draft_size, np.uint64)
    cost = np.zeros(draft_size, np.float64)
    cnt, ev = C.c_int64(0), C.c_uint64(0)
    ctx.check(lib().tt_draft_set(ctx.h, C.byref(sketch), C.byref(dev), n_steps, draft_size, pop_size, random_mix,
                                 explore_seed & (2**64 - 1), mix_seed & (2**64 - 1), toggles, ids.ctypes.data,
                                 cost.ctypes.data, C.byref(cnt), C.byref(ev)))
    m = cnt.value
    return ids[:m], cost[:m], ev.value


def tuner_round(ctx: Context, sketch: Sketch, dev: DeviceSpec, n_steps: int, draft_size: int, pop_size: int,
                random_mix: float, explore_seed: int, mix_seed: int, b: int, precision: int = TT_PREC_FP64):
    """One tuner round (tuner.cpp:294-396): the draft set, features + PaCM
    scores on the device, select_top(b). Needs a loaded PaCM (PaCM(ctx, ...)).
    Returns (picked indices into the draft set int64 [b], their scores
    float64 [b], their identities uint64 [b], draft-set size)."""
    sel = np.zeros(b, np.int64)
    sc = np.zeros(b, np.float64)
    ids = np.zeros(b, np.uint64)
    cnt = C.c_int64(0)
    ctx.check(lib().tt_tuner_round(ctx.h, C.byref(sketch), C.byref(dev), n_steps, draft_size, pop_size, random_mix,
                                   explore_seed & (2**64 - 1), mix_seed & (2**64 - 1), b, precision,
                                   sel.ctypes.data, sc.ctypes.data, ids.ctypes.data, C.byref(cnt)))
    return sel, sc, ids, cnt.value


def topk_merge(ctx: Context, cost: torch.Tensor, gidx: torch.Tensor, ids: torch.Tensor, k: int):
    idx, c, i = _topk_out(ctx, k)
    cnt = C.c_int64(0)
    ctx.check(lib().tt_topk_merge(ctx.h, _p(cost), _p(gidx), _p(ids), cost.shape[0], k, _p(idx), _p(c), _p(i),
                                  C.byref(cnt)))
    m = cnt.value
    return idx[:m], c[:m], i[:m]


def extract_features(ctx: Context, sketch: Sketch, dev: DeviceSpec, ids: torch.Tensor):
    """extract_features (features.cpp:98-257) for schedules given by identity:
    (stmt [k, S, 24], block [k, B, 23]) fp64."""
    k = ids.shape[0]
    S, B = sketch.op.n_statements, sketch.op.n_blocks
    st = ctx.empty((k, S, 24), torch.float64)
    bl = ctx.empty((k, B, 23), torch.float64)
    ctx.check(lib().tt_features(ctx.h, C.byref(sketch), C.byref(dev), _p(ids), k, _p(st), _p(bl)))
    return st, bl


def extract_features_soa(ctx: Context, sketch: Sketch, dev: DeviceSpec, soa: torch.Tensor, idx: torch.Tensor):
    k = idx.shape[0]
    S, B = sketch.op.n_statements, sketch.op.n_blocks
    st = ctx.empty((k, S, 24), torch.float64)
    bl = ctx.empty((k, B, 23), torch.float64)
    ctx.check(lib().tt_features_soa(ctx.h, C.byref(sketch), C.byref(dev), _p(soa), soa.stride(0), _p(idx), k,
                                    _p(st), _p(bl)))
    return st, bl


def param_count(h: int) -> int:
    return 24 * h + h + h * h + h + 23 * h + h + 3 * (h * h + h) + 2 * h * h + h + h + 1


_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def _scramble(x: np.ndarray) -> np.ndarray:
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def init_params(h: int, seed: int) -> np.ndarray:
    """init_params(h, RngStream(seed)) (ranker.cpp:305-326): Xavier-uniform
    weights drawn in tensor order, zero biases; flattened in
    for_each_tensor order."""
    if h < 1:
        raise TTError("E_STATE", "hidden width must be >= 1")
    shapes = [(24, h), (1, h), (h, h), (1, h), (23, h), (1, h), (h, h), (1, h), (h, h), (1, h), (h, h), (1, h),
              (2 * h, h), (1, h), (h, 1), (1, 1)]
    n_draw = sum(r * c for i, (r, c) in enumerate(shapes) if i % 2 == 0)
    s0 = np.uint64(seed if seed else int(_GOLDEN))
    with np.errstate(over="ignore"):
        g = np.arange(1, n_draw + 1, dtype=np.uint64)
        u = (_scramble(s0 + g * _GOLDEN) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    out, pos = [], 0
    for i, (r, c) in enumerate(shapes):
        if i % 2 == 0:
            lim = np.sqrt(6.0 / (r + c))
            out.append((2.0 * u[pos:pos + r * c] - 1.0) * lim)
            pos += r * c
        else:
            out.append(np.zeros(r * c))
    return np.concatenate(out)


class PaCM:
    """The learned cost model bound to a context (RankerParams on the GPU)."""

    def __init__(self, ctx: Context, params, h: int):
        self.ctx, self.h = ctx, h
        self.load(params)

    def load(self, params):
        if isinstance(params, torch.Tensor):
            t = params.detach().to(torch.float64).contiguous()
        else:
            t = torch.from_numpy(np.ascontiguousarray(params, np.float64))
        if t.numel() != param_count(self.h):
            raise TTError("E_STATE", f"expected {param_count(self.h)} parameters for h={self.h}")
        self._host = t  # keep alive during the async copy
        self.ctx.check(lib().tt_pacm_load(self.ctx.h, C.c_void_p(t.data_ptr()), self.h))
        if not t.is_cuda:
            self.ctx.sync()

    def score(self, sketch: Sketch, dev: DeviceSpec, ids: torch.Tensor, precision: int = TT_PREC_FP64) -> torch.Tensor:
        out = self.ctx.empty((ids.shape[0],), torch.float64)
        self.ctx.check(lib().tt_pacm_score(self.ctx.h, C.byref(sketch), C.byref(dev), _p(ids), ids.shape[0], precision,
                                           _p(out)))
        return out

    def score_batch(self, stmt: torch.Tensor, block: torch.Tensor, attention_identity: bool = False) -> torch.Tensor:
        """score_batch(params, feats, opts) (ranker.cpp:375-381)."""
        stmt, block = stmt.contiguous(), block.contiguous()
        k = stmt.shape[0]
        out = self.ctx.empty((k,), torch.float64)
        self.ctx.check(lib().tt_pacm_score_features(self.ctx.h, _p(stmt), _p(block), stmt.shape[1], block.shape[1], k,
                                                    int(attention_identity), _p(out)))
        return out


def forward_calls() -> int:
    return int(lib().tt_forward_calls())


def reset_forward_calls() -> None:
    lib().tt_reset_forward_calls()


def select_top(ctx: Context, scores: torch.Tensor, drafts: torch.Tensor, excluded: torch.Tensor | None, b: int):
    """select_top (ranker.cpp:514-532); raises E_STATE when < b available."""
    out = (C.c_int64 * b)()
    ex = None if excluded is None else excluded.to(torch.uint8).contiguous()
    ctx.check(lib().tt_select_top(ctx.h, _p(scores), _p(drafts), _p(ex), scores.shape[0], b, out))
    return np.frombuffer(out, dtype=np.int64).copy()


def oracle_latency(ctx: Context, sketch: Sketch, oracle: OracleSpec, soa: torch.Tensor) -> torch.Tensor:
    """noiseless_latency (oracle.cpp:105-111) per schedule, bit-exact fp64."""
    n = soa.shape[1]
    out = ctx.empty((n,), torch.float64)
    ctx.check(lib().tt_oracle_latency(ctx.h, C.byref(sketch), C.byref(oracle), _p(soa), soa.stride(0), n, _p(out)))
    return out


def oracle_measure(ctx: Context, sketch: Sketch, oracle: OracleSpec, soa: torch.Tensor, task_hash: int, trial0: int):
    """measure (oracle.cpp:113-121) with the tuner's per-trial streams
    (tuner.cpp:202-203): schedule i is trial trial0 + i. Returns (latency, noiseless)."""
    n = soa.shape[1]
    lat, nl = ctx.empty((n,), torch.float64), ctx.empty((n,), torch.float64)
    ctx.check(lib().tt_oracle_measure(ctx.h, C.byref(sketch), C.byref(oracle), _p(soa), soa.stride(0), n,
                                      task_hash & (2**64 - 1), trial0, _p(lat), _p(nl)))
    return lat, nl


def oracle_best(ctx: Context, sketch: Sketch, oracle: OracleSpec):
    """oracle_best (oracle.cpp:123-135): (identity of a minimiser, minimal noiseless latency)."""
    ident, lat = C.c_uint64(0), C.c_double(0)
    ctx.check(lib().tt_oracle_best(ctx.h, C.byref(sketch), C.byref(oracle), C.byref(ident), C.byref(lat)))
    return int(ident.value), float(lat.value)


def train(ctx: Context, params: torch.Tensor, h: int, stmt: torch.Tensor, block: torch.Tensor, latencies,
          epochs: int = 8, lr: float = 1e-2, batch: int = 256, seed: int = 0, attention_identity: bool = False):
    """train(params, {one task}, cfg) (ranker.cpp:459-512) on the device, in
    place on `params` (flattened RankerParams, fp64 CUDA tensor). Returns
    (initial_loss, final_loss)."""
    if params.dtype != torch.float64 or not params.is_cuda or params.numel() != param_count(h):
        raise TTError("E_STATE", f"params must be {param_count(h)} fp64 values on the GPU")
    stmt, block = stmt.contiguous(), block.contiguous()
    lat = np.ascontiguousarray(np.asarray(latencies, np.float64))
    l0, l1 = C.c_double(0), C.c_double(0)
    ctx.check(lib().tt_pacm_train(ctx.h, _p(params), h, _p(stmt), _p(block), stmt.shape[1], block.shape[1],
                                  lat.ctypes.data_as(C.POINTER(C.c_double)), stmt.shape[0], epochs, float(lr), batch,
                                  seed & (2**64 - 1), int(attention_identity), C.byref(l0), C.byref(l1)))
    return l0.value, l1.value


def rank_loss(ctx: Context, scores: torch.Tensor, latencies: torch.Tensor, with_grad: bool = True):
    """lambda_rank_loss(scores, latencies) (ranker.cpp:394-441) on the device:
    (loss, d loss / d score or None)."""
    scores, latencies = scores.contiguous(), latencies.contiguous()
    grad = ctx.empty((scores.shape[0],), torch.float64) if with_grad else None
    loss = C.c_double(0)
    ctx.check(lib().tt_rank_loss(ctx.h, _p(scores), _p(latencies), scores.shape[0], C.byref(loss), _p(grad)))
    return loss.value, grad


def momentum_adapt(ctx: Context, phi: torch.Tensor, m: float, h: int, stmt: torch.Tensor, block: torch.Tensor,
                   latencies, **cfg):
    """momentum_adapt (momentum.cpp:48-56): target = phi, train(target),
    phi <- target + m (phi - target). Returns (target, (initial, final) loss)."""
    target = phi.clone()
    report = train(ctx, target, h, stmt, block, latencies, **cfg)
    momentum_update(ctx, phi, target, m)
    return target, report


def gd_step(ctx: Context, params: torch.Tensor, grads: torch.Tensor, lr: float):
    ctx.check(lib().tt_gd_step(ctx.h, _p(params), _p(grads), params.numel(), float(lr)))


def momentum_update(ctx: Context, phi: torch.Tensor, target: torch.Tensor, m: float):
    """In-place phi <- target + m (phi - target) (momentum.cpp:28-46)."""
    if phi.shape != target.shape:
        raise TTError("E_STATE", "model tensor shape mismatch")
    ctx.check(lib().tt_momentum_update(ctx.h, _p(phi), _p(target), phi.numel(), float(m)))


@dataclass
class RoundOutput:
    index: np.ndarray      # population index of each selected candidate
    score: np.ndarray      # PaCM score (fp64; certified for the fast path)
    cost: np.ndarray       # draft cost
    identity: np.ndarray   # exact schedule identity
    drafted: int
    rescored: int
    status: int
    retries: int = 0
    band_err: float = 0.0

    @property
    def selected(self) -> int:
        return len(self.index)


def _round_cfg(n, k, b, precision, band, first, toggles):
    if band is None:  # the bf16 path needs an explicit bound; fp64 ignores it
        band = TT_BF16_BAND if precision == TT_PREC_BF16 else 0.0
    return RoundConfig(n, k, b, toggles, precision, band, first)


def _round_out(b, res, ix, sc, co, ids):
    m = res.selected
    return RoundOutput(np.frombuffer(ix, np.int64)[:m].copy(), np.frombuffer(sc, np.float64)[:m].copy(),
                       np.frombuffer(co, np.float64)[:m].copy(), np.frombuffer(ids, np.uint64)[:m].copy(),
                       res.drafted, res.rescored, res.status, res.retries, res.band_err)


def draft_verify_round(ctx: Context, sketch: Sketch, dev: DeviceSpec, n: int, k: int, b: int, seed: int = 0,
                       soa: torch.Tensor | None = None, precision: int = TT_PREC_FP64, band: float | None = None,
                       first: int = 0, toggles: int = TT_TOGGLES_ALL) -> RoundOutput:
    """Engine::round_draft_verify's compute (tuner.cpp:361-396): SA draft over
    n candidates -> dedup top-k -> features + PaCM -> select_top(b). Needs a
    PaCM loaded on ctx."""
    cfg = _round_cfg(n, k, b, precision, band, first, toggles)
    ix, sc, co, ids = (C.c_int64 * b)(), (C.c_double * b)(), (C.c_double * b)(), (C.c_uint64 * b)()
    res = RoundResult()
    ld = soa.stride(0) if soa is not None else 0
    ctx.check(lib().tt_round(ctx.h, C.byref(sketch), C.byref(dev), C.byref(cfg), _p(soa), ld, seed & (2**64 - 1),
                             ix, sc, co, ids, C.byref(res)))
    return _round_out(b, res, ix, sc, co, ids)


def round_async(ctx: Context, sketch: Sketch, dev: DeviceSpec, n: int, k: int, b: int, seed: int = 0,
                soa: torch.Tensor | None = None, precision: int = TT_PREC_FP64, band: float | None = None, first: int = 0,
                toggles: int = TT_TOGGLES_ALL):
    cfg = _round_cfg(n, k, b, precision, band, first, toggles)
    ld = soa.stride(0) if soa is not None else 0
    ctx.check(lib().tt_round_async(ctx.h, C.byref(sketch), C.byref(dev), C.byref(cfg), _p(soa), ld,
                                   seed & (2**64 - 1)))
    ctx._inflight.append(None)


def round_collect(ctx: Context, b: int) -> RoundOutput:
    ix, sc, co, ids = (C.c_int64 * b)(), (C.c_double * b)(), (C.c_double * b)(), (C.c_uint64 * b)()
    res = RoundResult()
    ctx.check(lib().tt_round_collect(ctx.h, b, ix, sc, co, ids, C.byref(res)))
    if ctx._inflight:
        ctx._inflight.popleft()
    return _round_out(b, res, ix, sc, co, ids)


def round_finish_merged(ctx: Context, sketch: Sketch, dev: DeviceSpec, cost: torch.Tensor, gidx: torch.Tensor,
                        ids: torch.Tensor, n: int, k: int, b: int, precision: int = TT_PREC_FP64,
                        band: float | None = None) -> RoundOutput:
    cfg = _round_cfg(n, k, b, precision, band, 0, TT_TOGGLES_ALL)
    ix, sc, co, idv = (C.c_int64 * b)(), (C.c_double * b)(), (C.c_double * b)(), (C.c_uint64 * b)()
    res = RoundResult()
    ctx.check(lib().tt_round_finish_merged(ctx.h, C.byref(sketch), C.byref(dev), C.byref(cfg), _p(cost), _p(gidx),
                                           _p(ids), cost.shape[0], ix, sc, co, idv, C.byref(res)))
    return _round_out(b, res, ix, sc, co, idv)


def round_local_async(ctx: Context, sketch: Sketch, dev: DeviceSpec, n: int, k: int, b: int, first: int,
                      out: torch.Tensor, seed: int = 0, soa: torch.Tensor | None = None,
                      toggles: int = TT_TOGGLES_ALL):
    """Draft half of a sharded round into `out` (int64 [3, k]: cost bits,
    global index (-1 = empty), identity) — the all-gather payload."""
    cfg = _round_cfg(n, k, b, TT_PREC_FP64, 0.0, first, toggles)
    ld = soa.stride(0) if soa is not None else 0
    ctx.check(lib().tt_round_local_async(ctx.h, C.byref(sketch), C.byref(dev), C.byref(cfg), _p(soa), ld,
                                         seed & (2**64 - 1), _p(out[0]), _p(out[1]), _p(out[2])))


def comm_unique_id() -> bytes:
    """NCCL unique id for tt_comm_init (create on rank 0, share out of band)."""
    buf = (C.c_uint8 * 128)()
    rc = lib().tt_comm_unique_id(buf)
    if rc:
        raise TTError("E_NCCL", "tt_comm_unique_id failed (libnccl.so.2 missing?)")
    return bytes(buf)


def comm_init(ctx: Context, nranks: int, rank: int, uid: bytes):
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    ctx.check(lib().tt_comm_init(ctx.h, nranks, rank, buf))


def comm_destroy(ctx: Context):
    ctx.check(lib().tt_comm_destroy(ctx.h))


def round_sharded(ctx: Context, sketch: Sketch, dev: DeviceSpec, n: int, k: int, b: int, seed: int = 0,
                  soa_shard: torch.Tensor | None = None, precision: int = TT_PREC_FP64, band: float | None = None,
                  first: int = 0, toggles: int = TT_TOGGLES_ALL) -> RoundOutput:
    """tt_round_sharded: the whole sharded round (n = global population) over
    the context's NCCL communicator; every rank gets the same selection."""
    cfg = _round_cfg(n, k, b, precision, band, first, toggles)
    ix, sc, co, idv = (C.c_int64 * b)(), (C.c_double * b)(), (C.c_double * b)(), (C.c_uint64 * b)()
    res = RoundResult()
    ld = soa_shard.stride(0) if soa_shard is not None else 0
    ctx.check(lib().tt_round_sharded(ctx.h, C.byref(sketch), C.byref(dev), C.byref(cfg), _p(soa_shard), ld,
                                     seed & (2**64 - 1), ix, sc, co, idv, C.byref(res)))
    return _round_out(b, res, ix, sc, co, idv)


def round_local(ctx: Context, sketch: Sketch, dev: DeviceSpec, n: int, k: int, b: int, first: int,
                out: torch.Tensor, seed: int = 0, soa: torch.Tensor | None = None, toggles: int = TT_TOGGLES_ALL):
    """Synchronous draft half (tt_round_local): the same payload with the
    selector's host-driven retries (margin, hash path) and the population
    check; raises where draft_verify_round would."""
    cfg = _round_cfg(n, k, b, TT_PREC_FP64, 0.0, first, toggles)
    ld = soa.stride(0) if soa is not None else 0
    ctx.check(lib().tt_round_local(ctx.h, C.byref(sketch), C.byref(dev), C.byref(cfg), _p(soa), ld,
                                   seed & (2**64 - 1), _p(out[0]), _p(out[1]), _p(out[2])))


def unpack_gathered(gathered: torch.Tensor, world: int, k: int) -> torch.Tensor:
    """The all-gather output (world consecutive [3, k] payloads) as one
    [3, world * k] table: row 0 cost bits, row 1 global index, row 2 identity."""
    if gathered.numel() != world * 3 * k:
        raise TTError("E_STATE", f"gathered {gathered.numel()} entries, expected {world * 3 * k}")
    return gathered.reshape(world, 3, k).permute(1, 0, 2).contiguous().reshape(3, world * k)


def round_finish_merged_async(ctx: Context, sketch: Sketch, dev: DeviceSpec, gathered: torch.Tensor, n: int, k: int,
                              b: int, precision: int = TT_PREC_FP64, band: float | None = None):
    """Verify half of a sharded round over the all-gathered [R, 3, k] lists."""
    g = unpack_gathered(gathered, gathered.numel() // (3 * k), k)
    cfg = _round_cfg(n, k, b, precision, band, 0, TT_TOGGLES_ALL)
    ctx.check(lib().tt_round_finish_merged_async(ctx.h, C.byref(sketch), C.byref(dev), C.byref(cfg), _p(g[0]),
                                                 _p(g[1]), _p(g[2]), g.shape[1]))
    ctx._inflight.append(g)  # kept alive until collected


STAGES = ["select", "pacm", "certify", "finish", "merge", "pacm_kernel", "features", "draft_cost"]


def profile_enable(ctx: Context, on: bool = True):
    ctx.check(lib().tt_profile_enable(ctx.h, int(on)))


def profile_read(ctx: Context) -> dict:
    ms = (C.c_double * 8)()
    cnt = (C.c_int64 * 8)()
    ctx.check(lib().tt_profile_read(ctx.h, ms, cnt, 8))
    return {STAGES[i]: (ms[i], cnt[i]) for i in range(len(STAGES)) if cnt[i]}


def kernel_launches() -> int:
    return int(lib().tt_kernel_launches())


def round_drafted(ctx: Context, k: int):
    """Device views (index, cost, identity, score) of the last round's drafted set."""
    ptrs = [C.c_void_p() for _ in range(4)]
    ctx.check(lib().tt_round_drafted(ctx.h, *[C.byref(p) for p in ptrs]))
    return ptrs
