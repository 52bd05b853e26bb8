"""The N > 1 path's host logic on CPU: world_size 2 (and 3) over gloo.

Each rank plays its GPU's part with the oracle standing in for K0+K1+K2 on
its shard (tests may call the checker): it builds the same [3, K] payload
the device writes (cost bits, global index, identity; -1 = empty slot),
the payloads go through a real torch.distributed all-gather, the product's
``unpack_gathered`` lays them out, and the merge semantics (dedup by
identity, lowest (cost, global index), ascending) must reproduce the
single-rank explore(n_steps=1) top-K exactly — on every rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2402_02361_b200.sharded import shard_range
from paper_2402_02361_b200.tiletune import unpack_gathered
from paper_2402_02361_b200.types import WORKLOADS, make_conv, make_sketch, reference_device


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def local_payload(sk, seed, first, n, k):
    """What tt_round_local_async writes for this shard (via the oracle)."""
    from tests import _refs as R
    pop = R.O_random_init(sk, seed, n, first=first)
    cost = R.O_draft_cost(sk, reference_device(), pop)
    idx, c = R.O_draft_topk(sk, cost, pop, k)
    ids, ok = R.O_identity(sk, pop[:, idx])
    assert ok
    out = np.zeros((3, k), np.int64)
    out[1, :] = -1
    m = len(idx)
    out[0, :m] = c.view(np.int64)
    out[1, :m] = idx + first
    out[2, :m] = ids.view(np.int64)
    return out


def merge(table, k):
    """Merge semantics of k_merge (tt_topk_merge): unique identities, each at
    its lowest (cost, global index), the k lowest ascending."""
    cost = table[0].view(np.float64)
    gidx, ids = table[1], table[2]
    live = gidx >= 0
    order = np.lexsort((gidx[live], cost[live]))
    seen, out = set(), []
    for j in order:
        i = int(ids[live][j])
        if i in seen:
            continue
        seen.add(i)
        out.append((cost[live][j], int(gidx[live][j])))
        if len(out) == k:
            break
    return out


def _worker(rank, world, port, name, n_total, k, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sk = make_sketch(WORKLOADS[name]() if name in WORKLOADS else make_conv(512, 7, 7, 512, 9))
        first, n = shard_range(n_total, rank, world)
        payload = torch.from_numpy(local_payload(sk, seed, first, n, k))
        parts = [torch.empty_like(payload) for _ in range(world)]
        dist.all_gather(parts, payload)
        gathered = torch.cat([p.reshape(-1) for p in parts])
        table = unpack_gathered(gathered, world, k).numpy()
        q.put((rank, merge(table, k)))
    finally:
        dist.destroy_process_group()


def run_world(world, name, n_total, k, seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, n_total, k, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    return res


def test_shard_range_partitions():
    for n, w in [(1 << 20, 8), (1000, 3), (7, 8), (0, 2), (65536, 1)]:
        spans = [shard_range(n, r, w) for r in range(w)]
        assert sum(s[1] for s in spans) == n
        pos = 0
        for first, cnt in spans:
            assert first == pos
            pos += cnt


def test_unpack_gathered_layout():
    k, world = 4, 3
    parts = [torch.arange(3 * k, dtype=torch.int64).reshape(3, k) + 100 * r for r in range(world)]
    t = unpack_gathered(torch.cat([p.reshape(-1) for p in parts]), world, k)
    for row in range(3):
        assert t[row].tolist() == sum([parts[r][row].tolist() for r in range(world)], [])


@pytest.mark.parametrize("world,name,n_total,k", [(2, "gemm1024", 8192, 512), (3, "dups", 30000, 256)])
def test_sharded_merge_equals_single_rank(world, name, n_total, k):
    from tests import _refs as R
    seed = 42
    res = run_world(world, name, n_total, k, seed)
    sk = make_sketch(WORKLOADS[name]() if name in WORKLOADS else make_conv(512, 7, 7, 512, 9))
    pop = R.O_random_init(sk, seed, n_total)
    cost = R.O_draft_cost(sk, reference_device(), pop)
    idx, c = R.O_draft_topk(sk, cost, pop, k)
    want = list(zip(c.tolist(), idx.tolist()))
    for r in range(world):
        got = [(float(a), b) for a, b in res[r]]
        assert got == want, f"rank {r}"
