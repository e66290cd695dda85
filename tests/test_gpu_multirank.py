"""The product's N > 1 path on the one available GPU: bench.py self-launches
two ranks (torch.distributed.run; gloo process group, since NCCL needs one GPU
per rank) on the layer-sharded c5 configuration at test size.  Checks: the
line reports n_gpus = 2 and strong scaling, the ranks own disjoint contiguous
layer blocks that cover the cache, and each rank's first-unit section digest
equals a single-process encode of the same unit (no data-path collective:
sharding does not change a single byte)."""

import hashlib
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_layer_shard(cuda):
    import torch

    env = dict(os.environ, HQMQ_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--workload", "c5s", "--steps", "2", "--warmup", "1", "--no-attn",
                          "--no-cpu", "--no-e2e", "--graph", "off"],
                         env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    res = json.loads(lines[0])
    assert res["n_gpus"] == 2 and res["scaling"] == "strong"
    ranks = sorted(res["ranks"], key=lambda r: r["rank"])
    assert [r["layers"] for r in ranks] == [[0, 3], [4, 7]]
    assert sum(r["units"] for r in ranks) == 16

    import paper_2605_27646_b200 as m
    sys.path.insert(0, ROOT)
    import bench

    wl = bench.WORKLOADS["c5s"]
    cfg = m.CodecConfig(wl["S"], wl["br"])
    bank = m.CodebookBank(0, wl["S"])
    for r in ranks:
        layer = r["layers"][0]
        x = bench.make_input(torch, wl, layer, "K", cuda)
        qt = m.encode_tensor(x, cfg, layer=layer, role="K", bank=bank)
        want = hashlib.sha256(b"".join(qt.section_bytes())).hexdigest()[:16]
        assert r["first_unit_digest"] == want
