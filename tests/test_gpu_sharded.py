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


def _worker(rank, world, port, name, n, k, b, seed, prec, q, backend="gloo"):
    import torch.distributed as dist
    from paper_2402_02361_b200 import tiletune as tt
    from paper_2402_02361_b200.sharded import ShardedRound
    from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev_id = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev_id)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev_id))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = tt.Context(dev_id)
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


def _run_ranks(world, name, n, k, b, seed, prec, backend):
    c = mp.get_context("spawn")
    q = c.Queue()
    port = _port()
    procs = [c.Process(target=_worker, args=(r, world, port, name, n, k, b, seed, prec, q, backend))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, rest) for r, *rest in (q.get(timeout=180) for _ in procs))
    assert all(v[0] != "error" for v in res.values()), res
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    return res


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs for an NCCL group")
@pytest.mark.parametrize("name", ["bert_ffn1", "bert_bmm_qk"])
def test_sharded_nccl_equal_single(name):
    """The bench's N > 1 transport: ranks on distinct GPUs, NCCL all-gather
    (NVLink), config-3 shape (strong-sharded population), selection equal to
    the single-GPU round bit for bit on every rank."""
    from paper_2402_02361_b200 import tiletune as tt
    from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device
    n, k, b, seed = 1 << 20, 512, 10, 42
    world = min(torch.cuda.device_count(), 8)
    ctx = tt.Context(0)
    tt.PaCM(ctx, tt.init_params(64, derive_seed(seed, TAG_INIT)), 64)
    ref = tt.draft_verify_round(ctx, make_sketch(WORKLOADS[name]()), reference_device(), n, k, b, seed=seed)
    ctx.close()
    res = _run_ranks(world, name, n, k, b, seed, 0, "nccl")
    for r in range(world):
        idx, sc, ids = res[r]
        assert idx == ref.index.tolist(), r
        assert np.abs(np.array(sc) - ref.score).max() <= 1e-12
        assert ids == ref.identity.tolist()


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


def _two_rank_payloads(tt, ctx, sk, dev, n, k, b, seed, soa=None, sync=False):
    outs = []
    for r in range(2):
        o = torch.empty((3, k), dtype=torch.int64, device="cuda")
        fn = tt.round_local if sync else tt.round_local_async
        fn(ctx, sk, dev, n, k, b, r * n, o, seed=seed, soa=None if soa is None else soa[r])
        outs.append(o)
    return torch.cat([o.reshape(-1) for o in outs])


def test_local_sync_equals_async_and_single():
    """tt_round_local (host-driven retries) emits the same payload as the
    async draft half; merged, both equal the single-GPU round."""
    from paper_2402_02361_b200 import tiletune as tt
    from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device
    ctx = tt.Context(0)
    tt.PaCM(ctx, tt.init_params(64, derive_seed(3, TAG_INIT)), 64)
    sk, dev = make_sketch(WORKLOADS["bert_qkv"]()), reference_device()
    n, k, b = 30000, 512, 10
    ga = _two_rank_payloads(tt, ctx, sk, dev, n, k, b, 3)
    gs = _two_rank_payloads(tt, ctx, sk, dev, n, k, b, 3, sync=True)
    assert torch.equal(ga, gs)
    tt.round_finish_merged_async(ctx, sk, dev, gs, 2 * n, k, b)
    got = tt.round_collect(ctx, b)
    want = tt.draft_verify_round(ctx, sk, dev, 2 * n, k, b, seed=3)
    assert (got.index == want.index).all() and (got.identity == want.identity).all()
    ctx.close()


def test_failed_rank_fails_every_merged_round():
    """A payload marked by a failed selector (index -2) or by an invalid
    explicit population (-3, written by the draft half itself) makes the
    merged round fail loudly instead of returning a short selection."""
    from paper_2402_02361_b200 import tiletune as tt
    from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device
    ctx = tt.Context(0)
    tt.PaCM(ctx, tt.init_params(64, derive_seed(3, TAG_INIT)), 64)
    sk, dev = make_sketch(WORKLOADS["gemm1024"]()), reference_device()
    n, k, b = 20000, 512, 10
    g = _two_rank_payloads(tt, ctx, sk, dev, n, k, b, 5)
    g2 = g.clone().view(2, 3, k)
    g2[1, 1, 0] = -2
    tt.round_finish_merged_async(ctx, sk, dev, g2.reshape(-1), 2 * n, k, b)
    with pytest.raises(tt.TTError) as e:
        tt.round_collect(ctx, b)
    assert e.value.code == "E_STATE" and "tt_round_local" in str(e.value)
    # explicit populations: rank 1's holds a schedule whose factors do not multiply to the extent
    pops = [tt.random_init(ctx, sk, n, 5, first=r * n) for r in range(2)]
    pops[1][0, 17] += 1
    g3 = _two_rank_payloads(tt, ctx, sk, dev, n, k, b, 0, soa=pops)
    assert int(g3.view(2, 3, k)[1, 1, 0]) == -3
    tt.round_finish_merged_async(ctx, sk, dev, g3, 2 * n, k, b)
    with pytest.raises(tt.TTError) as e:
        tt.round_collect(ctx, b)
    assert e.value.code == "E_VALIDATE"
    with pytest.raises(tt.TTError) as e:  # the synchronous half reports it directly
        _two_rank_payloads(tt, ctx, sk, dev, n, k, b, 0, soa=pops, sync=True)
    assert e.value.code == "E_VALIDATE"
    ctx.close()


def test_c_abi_sharded_round_single_rank():
    """tt_comm_init + tt_round_sharded (the collective inside the C ABI,
    NCCL loaded at run time) on a one-rank communicator: equal to tt_round."""
    from paper_2402_02361_b200 import tiletune as tt
    from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device
    ctx = tt.Context(0)
    tt.PaCM(ctx, tt.init_params(64, derive_seed(9, TAG_INIT)), 64)
    tt.comm_init(ctx, 1, 0, tt.comm_unique_id())
    sk, dev = make_sketch(WORKLOADS["bert_ffn2"]()), reference_device()
    n, k, b = 100000, 512, 10
    got = tt.round_sharded(ctx, sk, dev, n, k, b, seed=9)
    want = tt.draft_verify_round(ctx, sk, dev, n, k, b, seed=9)
    assert (got.index == want.index).all() and (got.identity == want.identity).all()
    soa = tt.random_init(ctx, sk, n, 9)
    got2 = tt.round_sharded(ctx, sk, dev, n, k, b, soa_shard=soa)
    assert (got2.index == want.index).all()
    tt.comm_destroy(ctx)
    ctx.close()


def _c_abi_worker(rank, world, uid_q, name, n, k, b, seed, q):
    from paper_2402_02361_b200 import tiletune as tt
    from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device
    try:
        torch.cuda.set_device(rank)
        ctx = tt.Context(rank)
        tt.PaCM(ctx, tt.init_params(64, derive_seed(seed, TAG_INIT)), 64)
        if rank == 0:
            uid = tt.comm_unique_id()
            for _ in range(world - 1):
                uid_q.put(uid)
        else:
            uid = uid_q.get(timeout=60)
        tt.comm_init(ctx, world, rank, uid)
        out = tt.round_sharded(ctx, make_sketch(WORKLOADS[name]()), reference_device(), n, k, b, seed=seed)
        q.put((rank, out.index.tolist()))
        tt.comm_destroy(ctx)
        ctx.close()
    except Exception as e:
        q.put((rank, "error " + repr(e)))
        raise


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs for an NCCL group")
def test_c_abi_sharded_round_multi_gpu():
    """The C-ABI collective over R GPUs (no torch.distributed): every rank's
    selection equals the one-GPU round over the whole population."""
    from paper_2402_02361_b200 import tiletune as tt
    from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device
    name, n, k, b, seed = "bert_qkv", 1 << 20, 512, 10, 21
    world = min(torch.cuda.device_count(), 8)
    ctx = tt.Context(0)
    tt.PaCM(ctx, tt.init_params(64, derive_seed(seed, TAG_INIT)), 64)
    want = tt.draft_verify_round(ctx, make_sketch(WORKLOADS[name]()), reference_device(), n, k, b, seed=seed)
    ctx.close()
    c = mp.get_context("spawn")
    q, uq = c.Queue(), c.Queue()
    procs = [c.Process(target=_c_abi_worker, args=(r, world, uq, name, n, k, b, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(120)
    for r in range(world):
        assert res[r] == want.index.tolist(), (r, res[r])
