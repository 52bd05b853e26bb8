"""Multi-GPU draft+verify round: the population sharded by global index
range across ranks (one process per GPU), one all-gather of every rank's
local top-K, a deterministic merge, and a replicated verify.

The reference has no multi-GPU path; this is the B200
design of SURVEY.md §8e:

1. rank r owns global indices [first_r, first_r + n_r) (``shard_range``);
   the counter-based population makes the union bit-identical to one GPU;
2. each rank runs K1 + K2 locally into a K-entry list of (cost bits,
   global index, identity) — int64 [3, K], index -1 = empty slot. K per rank
   suffices without a margin: a schedule's rank in its first-occurrence
   shard's unique list is never worse than its global rank;
3. one all-gather of the [3, K] payloads (NCCL over NVLink on the box,
   gloo in the CPU tests) — 24 B per entry, ≈12 KB per rank at K = 512;
4. every rank merges the R·K entries (dedup by identity, keep the lowest
   (cost, global index)), then runs features → PaCM → select_top on
   identical data, so every rank returns the same selection, equal to R = 1.
"""
from __future__ import annotations

import torch

from . import tiletune as tt
from .tiletune import unpack_gathered  # noqa: F401  (re-exported: the payload layout)
from .types import DeviceSpec, Sketch, TT_TOGGLES_ALL


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """(first, n) of rank's contiguous slice of [0, n_total); the first
    n_total % world ranks take one extra candidate."""
    if world < 1 or not 0 <= rank < world:
        raise tt.TTError("E_CONFIG", f"rank {rank} outside world {world}")
    base, extra = divmod(n_total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


class ShardedRound:
    """draft_verify_round over a population sharded across a process group.

    ``weak`` scaling (the bench): every rank drafts n candidates, rank r the
    slice [r n, (r + 1) n) of the global stream. ``strong`` scaling: n is the
    global population, split with shard_range."""

    def __init__(self, ctx: tt.Context, group=None):
        import torch.distributed as dist
        self.ctx, self.group, self.dist = ctx, group, dist
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._bufs = {}

    def _buffers(self, k):
        if k not in self._bufs:
            self._bufs[k] = (self.ctx.empty((3, k), torch.int64), self.ctx.empty((self.world * 3 * k,), torch.int64))
        return self._bufs[k]

    def local(self, sketch: Sketch, dev: DeviceSpec, first: int, n: int, k: int, b: int = 1, seed: int = 0,
              soa: torch.Tensor | None = None, toggles: int = TT_TOGGLES_ALL, sync: bool = False) -> torch.Tensor:
        """Draft half: this rank's [3, k] payload (async on the ctx stream;
        sync=True: tt_round_local, with the selector's host-driven retries)."""
        payload, _ = self._buffers(k)
        fn = tt.round_local if sync else tt.round_local_async
        fn(self.ctx, sketch, dev, n, k, b, first, payload, seed=seed, soa=soa, toggles=toggles)
        return payload

    def run_async(self, sketch: Sketch, dev: DeviceSpec, n: int, k: int, b: int, seed: int = 0,
                  soa: torch.Tensor | None = None, precision: int = tt.TT_PREC_FP64, band: float | None = None,
                  scaling: str = "strong", toggles: int = TT_TOGGLES_ALL, sync_local: bool = False):
        if scaling == "strong":
            first, n_local = shard_range(n, self.rank, self.world)
            n_total = n
        else:
            first, n_local, n_total = self.rank * n, n, n * self.world
        payload = self.local(sketch, dev, first, n_local, k, b, seed=seed, soa=soa, toggles=toggles, sync=sync_local)
        _, gathered = self._buffers(k)
        if self.dist.get_backend(self.group) == "nccl":
            self.dist.all_gather_into_tensor(gathered, payload.reshape(-1), group=self.group)
        else:  # gloo (CPU tests, single-GPU multi-rank emulation): list form
            parts = list(gathered.view(self.world, -1).unbind(0))
            self.dist.all_gather(parts, payload.reshape(-1).contiguous(), group=self.group)
        tt.round_finish_merged_async(self.ctx, sketch, dev, gathered, n_total, k, b, precision=precision, band=band)

    def run(self, *a, **kw) -> tt.RoundOutput:
        """One sharded round, collected. A rank whose device selector could
        not certify its list marks its payload; every rank then sees the same
        merged E_STATE and re-runs the draft half synchronously (host-driven
        retries, hash path) — no extra agreement step is needed."""
        b = a[4] if len(a) > 4 else kw["b"]
        self.run_async(*a, **kw)
        try:
            return tt.round_collect(self.ctx, b)
        except tt.TTError as e:
            if e.code != "E_STATE" or "tt_round_local" not in str(e) or kw.get("sync_local"):
                raise
        self.run_async(*a, **dict(kw, sync_local=True))
        return tt.round_collect(self.ctx, b)
