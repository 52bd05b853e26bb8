"""The sharded round on a real device: two ranks (processes) share cuda:0
over a gloo group — the exact ShardedRound code path the NCCL bench runs
(local draft half -> all-gather of the [3, K] payloads -> merge + verify),
minus the NVLink transport. Every rank must return the single-GPU round's
selection bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, n, k, b, seed, prec, q):
    import torch.distributed as dist
    from paper_2402_02361_b200 import tiletune as tt
    from paper_2402_02361_b200.sharded import ShardedRound
    from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = tt.Context(0)
        tt.PaCM(ctx, tt.init_params(64, derive_seed(seed, TAG_INIT)), 64)
        out = ShardedRound(ctx).run(make_sketch(WORKLOADS[name]()), reference_device(), n, k, b, seed=seed,
                                    precision=prec)
        q.put((rank, out.index.tolist(), out.score.tolist(), out.identity.tolist()))
        ctx.close()
    except Exception as e:  # report instead of leaving the parent waiting
        q.put((rank, "error", repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,n,prec", [("gemm1024", 20000, 0), ("r50_c3x3_512", 65536, 1)])
def test_sharded_two_ranks_equal_single(name, n, prec):
    from paper_2402_02361_b200 import tiletune as tt
    from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device
    k, b, seed, world = 512, 10, 42, 2
    ctx = tt.Context(0)
    tt.PaCM(ctx, tt.init_params(64, derive_seed(seed, TAG_INIT)), 64)
    ref = tt.draft_verify_round(ctx, make_sketch(WORKLOADS[name]()), reference_device(), n, k, b, seed=seed,
                                precision=prec)
    ctx.close()
    c = mp.get_context("spawn")
    q = c.Queue()
    port = _port()
    procs = [c.Process(target=_worker, args=(r, world, port, name, n, k, b, seed, prec, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, rest) for r, *rest in (q.get(timeout=180) for _ in procs))
    assert all(v[0] != "error" for v in res.values()), res
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for r in range(world):
        idx, sc, ids = res[r]
        assert idx == ref.index.tolist(), r
        assert np.abs(np.array(sc) - ref.score).max() <= (1e-12 if prec == 0 else 6e-2)
        assert ids == ref.identity.tolist()
