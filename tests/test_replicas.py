"""CPU: the N>1 (replicas) path with world_size 2 over gloo on 127.0.0.1.

Each rank takes its shard of C4's 28 Pearson pairs (paper_2508_12093_b200/replicas.py),
computes them (the C oracle stands in for the per-rank GPU work: this exercises the
sharding, the host-side gather of decrypted scalars and the max-over-ranks timing),
and the gathered result must equal the single-process sweep bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle_abi import Params, ST_PEARSON, bits, oracle

S = 1024


def _columns():
    rng = np.random.default_rng(4)
    z = rng.standard_normal(S)
    return [np.sqrt(0.6) * z + np.sqrt(0.4) * rng.standard_normal(S) for _ in range(8)]


def _pearson(cols, pair):
    i, j = pair
    r = oracle().stat(Params(slot_count=S), ST_PEARSON, cols[i], 20.0, y=cols[j])
    assert r.rc == 0
    return float(r.out[0])


def _worker(rank, world, port, out_q):
    import torch.distributed as dist
    from paper_2508_12093_b200 import replicas as R
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cols = _columns()
        pairs = R.c4_pairs()
        mine = [pairs[k] for k in R.shard(len(pairs), world, rank)]
        local = [(p, _pearson(cols, p)) for p in mine]
        allres = R.gather_results(local, world, rank)
        t = R.max_over_ranks(float(rank + 1), world)
        if rank == 0:
            out_q.put((allres, t))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_balanced():
    from paper_2508_12093_b200 import replicas as R
    for n in (0, 1, 7, 28, 64):
        for w in (1, 2, 3, 8):
            got = [k for r in range(w) for k in R.shard(n, w, r)]
            assert got == list(range(n))
            sizes = [len(R.shard(n, w, r)) for r in range(w)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        R.shard(4, 2, 2)


def test_two_rank_gloo_pearson_sweep():
    from paper_2508_12093_b200 import replicas as R
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    allres, t = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cols = _columns()
    ref = [(p, _pearson(cols, p)) for p in R.c4_pairs()]
    assert [p for p, _ in allres] == [p for p, _ in ref]
    assert np.array_equal(bits(np.array([v for _, v in allres])), bits(np.array([v for _, v in ref])))
    assert t == 2.0  # max over ranks


def _gpu_worker(rank, world, port, out_q):
    """The same sweep with the GPU product as each rank's work (both ranks on cuda:0: replicas
    never wait on each other's kernels, so one device stands in for two without a cross-rank
    dependency; the data path has no collective)."""
    import sys
    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    from paper_2508_12093_b200 import hestat as H
    from paper_2508_12093_b200 import replicas as R
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        H.init(0)
        cols = _columns()
        ctx = H.EvalContext(H.CkksParams(slot_count=S), rng_seed=rank)
        enc = [H.encode_column(ctx, c) for c in cols]
        pairs = R.c4_pairs()
        mine = [pairs[k] for k in R.shard(len(pairs), world, rank)]
        local = [(p, float(ctx.decrypt(H.pearson(ctx, enc[p[0]], enc[p[1]], 20.0), 1)[0])) for p in mine]
        allres = R.gather_results(local, world, rank)
        meters = R.gather_results([ctx.meter().as_tuple()], world, rank)
        if rank == 0:
            out_q.put((allres, meters, [len(R.shard(len(pairs), world, r)) for r in range(world)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_gpu_replicas_pearson_sweep():
    from paper_2508_12093_b200 import replicas as R
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    allres, meters, sizes = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cols = _columns()
    ref = [(p, _pearson(cols, p)) for p in R.c4_pairs()]
    assert [p for p, _ in allres] == [p for p, _ in ref]
    assert np.array_equal(bits(np.array([v for _, v in allres])), bits(np.array([v for _, v in ref])))
    # each rank's meter = its share of pearson calls x one pearson's ledger
    one = oracle().stat(Params(slot_count=S), ST_PEARSON, cols[0], 20.0, y=cols[1]).meter
    for m, n in zip(meters, sizes):
        assert tuple(m) == tuple(n * v for v in one)
