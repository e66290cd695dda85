"""Multi-process (gloo, world_size 2) coverage of the layer-sharded path.

The GPU path shards (layer, role) units across ranks with no data-path
collective; these CPU tests check the placement logic and the
off-hot-path collectives with the oracle standing in for the per-rank encode
(checker only): the per-rank digests gathered to every rank must equal the
single-process digests of the same units, unit for unit.
"""

import hashlib
import os
import socket

import numpy as np
import pytest

from paper_2605_27646_b200.errors import InvalidArgument
from paper_2605_27646_b200.shard import ShardPlan, head_split


def test_strong_plan_partitions_every_unit():
    for layers, world in [(80, 1), (80, 2), (80, 4), (80, 8), (32, 3), (5, 8)]:
        seen = []
        for r in range(world):
            p = ShardPlan(layers, world, r)
            lr = p.layer_range()
            assert lr.step == 1  # contiguous layer blocks
            seen += p.units()
        assert sorted(seen) == sorted((l, ro) for l in range(layers) for ro in "KV")
        assert ShardPlan(layers, world, 0).total_units() == 2 * layers
    # C5 at 8 GPUs: 10 contiguous layers x (K, V) per rank
    assert ShardPlan(80, 8, 3).units()[:2] == [(30, "K"), (30, "V")]
    assert len(ShardPlan(80, 8, 7).units()) == 20


def test_weak_plan_replicates():
    p = ShardPlan(32, 4, 2, "weak")
    assert len(p.units()) == 64 and p.total_units() == 256


def test_plan_validation():
    with pytest.raises(InvalidArgument):
        ShardPlan(8, 2, 2)
    with pytest.raises(InvalidArgument):
        ShardPlan(8, 2, 0, "diagonal")
    assert head_split(8, 4, 3) == (6, 2)
    with pytest.raises(InvalidArgument):
        head_split(8, 3, 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _unit_digest(layer, role, heads, tokens):
    import hqmq_oracle as O

    x = O.gen_gaussian((1, heads, tokens, 16), seed=2 * layer + (role == "V"))
    x = x.astype(np.float16).astype(np.float64)
    enc = O.encode(x, 4, 3, multiplier=3.0, layer=layer, role=role)
    return O.digest(enc)


def _worker(rank, world, port, layers, q):
    import torch.distributed as dist

    from paper_2605_27646_b200 import shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = ShardPlan(layers, world, rank)
        mine = {f"{l}{r}": _unit_digest(l, r, 2, 8) for l, r in plan.units()}
        stats = shard.gather_stats({"rank": rank, "digests": mine, "n": len(mine)})
        t = shard.max_over_ranks([float(rank + 1), -float(rank)])
        s = shard.sum_over_ranks([float(len(mine))])
        q.put((rank, stats, t, s))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_digests_match_single_process():
    import multiprocessing as mp

    layers, world = 3, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, layers, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = {f"{l}{r}": _unit_digest(l, r, 2, 8) for l in range(layers) for r in "KV"}
    for rank, stats, t, s in res:
        assert [st["rank"] for st in stats] == [0, 1]
        merged = {}
        for st in stats:
            assert not set(merged) & set(st["digests"])  # disjoint ownership
            merged.update(st["digests"])
        assert merged == single
        assert t == [2.0, 0.0]
        assert s == [2.0 * layers]
    # checksum of checksums is order-independent of the rank that computed each unit
    h = hashlib.sha256("".join(single[k] for k in sorted(single)).encode()).hexdigest()
    assert len(h) == 64
