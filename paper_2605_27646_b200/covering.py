"""Monte-Carlo covering analysis of a joint codebook on the GPU (SURVEY.md
§8(f) rank 4): the reference's packing.estimate_covering (packing.py:59-83)
with its nearest-codeword scan (_kernels.nearest_scan) on the device.

The probes are the reference's Haar directions from the keyed probe stream
(rng.py:109-111, quat.py:76-91), generated on the host in 8192-probe blocks
exactly as the reference slices them (PROBE_BLOCK, packing.py:29); each block
runs hqmq_nearest_scan, the exact fp64 twin of the Cython scan (same dot
association, no FMA, lowest index on ties), so the cosines are bit-identical;
the worst cosine and the per-block arccos sums are then reduced on the host in
the reference's order, so rho_hat and mean_angle equal the reference's
bit for bit (tests/test_gpu_covering.py against tests/golden/covering.json).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .codebook import JointCodebook, RandomStream, haar_quaternions
from .errors import InvalidArgument
from .scan import nearest_scan

PROBE_BLOCK = 8192
TAG_PROBE = 0x50524F42  # rng.py:32


@dataclass(frozen=True)
class CoveringEstimate:
    """packing.py:32-39."""

    codebook_size: int
    seed: int
    n_probes: int
    probe_seed: int
    rho_hat: float
    mean_angle: float


def probe_stream(probe_seed: int) -> RandomStream:
    """rng.py:109-111."""
    return RandomStream(TAG_PROBE, probe_seed)


def estimate_covering(joint: JointCodebook, n_probes: int, probe_seed: int = 0,
                      device=None) -> CoveringEstimate:
    """Max and mean nearest-codeword angle over Haar probes (packing.py:59-83)."""
    import torch

    if n_probes < 1:
        raise InvalidArgument("need at least one probe")
    stream = probe_stream(probe_seed)
    dev = torch.device(device) if device is not None else torch.device("cuda")
    cw = torch.from_numpy(np.ascontiguousarray(joint.codewords, dtype=np.float64)).to(dev)
    worst_cos = 2.0
    total = 0.0
    done = 0
    while done < n_probes:
        block = min(PROBE_BLOCK, n_probes - done)
        probes = haar_quaternions(stream, block)
        _, cos = nearest_scan(probes, cw, device=dev)
        cos = cos.cpu().numpy()
        worst_cos = min(worst_cos, float(cos.min()))
        total += float(np.arccos(np.clip(cos, -1.0, 1.0)).sum())
        done += block
    return CoveringEstimate(
        codebook_size=joint.size,
        seed=joint.secondary.seed,
        n_probes=n_probes,
        probe_seed=probe_seed,
        rho_hat=float(np.arccos(np.clip(worst_cos, -1.0, 1.0))),
        mean_angle=total / n_probes,
    )


@dataclass(frozen=True)
class RateFit:
    """Least-squares fit of log rho_hat against log codeword count (packing.py:47-54)."""

    points: tuple
    slope: float
    intercept: float
    residual: float


def fit_points(points) -> RateFit:
    """packing.py:117-126."""
    pts = tuple((float(x), float(y)) for x, y in points)
    if len(pts) < 2:
        raise InvalidArgument("need at least two points to fit a rate")
    x = np.array([p[0] for p in pts])
    y = np.array([p[1] for p in pts])
    slope, intercept = np.polyfit(x, y, 1)
    residual = float(((y - (slope * x + intercept)) ** 2).sum())
    return RateFit(points=pts, slope=float(slope), intercept=float(intercept), residual=residual)


def fit_covering_rate(size_values, seed: int = 0, n_probes: int = 100_000, probe_seed: int = 0,
                      device=None):
    """packing.py:129-152: estimates over secondary sizes (layer 0, head 0,
    role K of `seed`) plus the log-log rate fit."""
    import math

    from .codebook import build_joint, build_secondary

    sizes = sorted(set(int(s) for s in size_values))
    if any(s < 1 for s in sizes):
        raise InvalidArgument("codebook sizes must be >= 1")
    estimates = [estimate_covering(build_joint(build_secondary(seed, 0, 0, "K", size)), n_probes,
                                   probe_seed, device=device) for size in sizes]
    fit = fit_points((math.log(24.0 * e.codebook_size), math.log(e.rho_hat)) for e in estimates)
    return fit, estimates


def covering_csv(estimates, sink) -> None:
    """packing.py:240-247."""
    import csv

    writer = csv.writer(sink)
    writer.writerow(["S", "seed", "n_probes", "rho_hat_rad", "mean_rad"])
    for e in estimates:
        writer.writerow([e.codebook_size, e.seed, e.n_probes, f"{e.rho_hat:.8f}",
                         f"{e.mean_angle:.8f}"])
