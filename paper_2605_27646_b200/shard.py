"""Multi-GPU placement of codec units (one process per GPU, torch.distributed).

A *unit* is one (layer, role) call of encode_tensor: the reference pools the
Med3x median over every head of that call (codec.py:208-219,
outliers.py:5-7), and keys codebooks by (layer, head, role)
(codebook.py:98-118), so units are fully independent.  Sharding by layer
therefore needs no collective on the data path:

* ``ShardPlan.strong``: the units of one cache are split across ranks in
  contiguous layer blocks (rank r owns layers [r*L/N, (r+1)*L/N), K and V of
  each), so a rank's codebook tables are its own layers only;
* ``ShardPlan.weak``: every rank owns a full cache of its own (replicas).

Splitting a unit by KV head is exchange-free only with per-head median
pooling; with "batch" pooling the exact median would need the bracket
counts and histograms all-reduced per narrowing pass.  ``head_split`` exposes the per-head variant
(head_base offsets keep the codebook keys of the unsplit call,
codec.py:133-135).

Collectives appear only off the hot path: ``gather_stats`` all-gathers the
per-rank unit statistics (coded / payload counts, fixups, digests) to every
rank, and ``max_over_ranks`` reduces the timing.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import InvalidArgument

ROLES = ("K", "V")


@dataclass(frozen=True)
class ShardPlan:
    layers: int
    world: int
    rank: int
    mode: str = "strong"  # "strong" (split one cache) | "weak" (replicas)

    def __post_init__(self):
        if self.layers < 1 or self.world < 1:
            raise InvalidArgument("layers and world size must be positive")
        if not 0 <= self.rank < self.world:
            raise InvalidArgument(f"rank {self.rank} outside world {self.world}")
        if self.mode not in ("strong", "weak"):
            raise InvalidArgument("shard mode must be 'strong' or 'weak'")

    def layer_range(self) -> range:
        if self.mode == "weak":
            return range(self.layers)
        base, extra = divmod(self.layers, self.world)
        lo = self.rank * base + min(self.rank, extra)
        return range(lo, lo + base + (1 if self.rank < extra else 0))

    def units(self) -> list[tuple[int, str]]:
        return [(layer, role) for layer in self.layer_range() for role in ROLES]

    def total_units(self) -> int:
        return 2 * self.layers * (self.world if self.mode == "weak" else 1)


def head_split(heads: int, world: int, rank: int) -> tuple[int, int]:
    """(head_base, n_heads) of rank's contiguous block of KV heads; valid for
    per-head median pooling or extraction off (no cross-head statistic)."""
    if heads % world:
        raise InvalidArgument(f"{heads} KV heads do not split over {world} ranks")
    n = heads // world
    return rank * n, n


def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


def gather_stats(stats: dict, device=None) -> list[dict]:
    """All-gather one rank's stats dict (numbers / short strings) to every rank.

    Off the hot path: called once after the timed region.  Works with NCCL
    (device tensors) and gloo (CPU tensors) process groups.
    """
    dist = _dist()
    if dist is None:
        return [dict(stats)]
    obj: list = [None] * dist.get_world_size()
    dist.all_gather_object(obj, dict(stats))
    return obj


def max_over_ranks(values: list[float], device=None) -> list[float]:
    """Element-wise max over ranks (timings: the slowest rank defines the step)."""
    dist = _dist()
    if dist is None:
        return list(values)
    import torch

    t = torch.tensor(values, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def sum_over_ranks(values: list[float], device=None) -> list[float]:
    dist = _dist()
    if dist is None:
        return list(values)
    import torch

    t = torch.tensor(values, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.tolist()
