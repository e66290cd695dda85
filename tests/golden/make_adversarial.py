"""Adversarial encode fixtures: chunks that sit on (or within a few ulps of) a
decision boundary of the nearest-codeword search, encoded by the REFERENCE.

Run in the build container (where /root/reference exists), after
`python oracle/build.py`:

    python tests/golden/make_adversarial.py

Why: the sm_100a encode searches in fp32 (FFMA2 on the CUDA cores, or split-fp16
rotations on tcgen05) and certifies each index against a margin (kDelta /
kDeltaTc in csrc/encode.cu), re-scoring uncertain chunks in exact fp64 with the
reference's lowest-index tie-break (_kernels.pyx:27-45: strict `>`).  Random
inputs almost never land inside that margin; these fixtures are built to.

Construction (per head, against that head's joint table, reference arithmetic:
u = x / r, score = ((u0 c0 + u1 c1) + u2 c2) + u3 c3 in fp64):
  * cross-secondary boundaries: random directions are projected onto the
    bisector of their two best codewords (those always sit in different
    secondaries' cosets for S >= 16), scaled, rounded to fp16, then every
    +-1-ulp perturbation of the 4 components is tried and the one with the
    smallest top-2 score gap is kept (gaps down to ~1e-8);
  * within-coset crossovers (S = 1, where the 24-cell's own Voronoi cells
    decide): points on the axis-vs-half bisector v0 = v1 + v2 + v3 and on
    half-vs-half bisectors in the secondary's frame (v = u * conj(s)), rotated
    back, rounded and refined the same way;
  * fp64 input (the generic encode path): bisector points without rounding
    (exact-tie gaps ~1e-16).
Each fixture records the input, the reference's QuantizedTensor fields, its
kvpack digest, and the top-2 gap of every chunk.
"""

from __future__ import annotations

import hashlib
import itertools
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

import hqmq  # noqa: E402  (the reference)
from hqmq.codebook import CodebookBank  # noqa: E402
from hqmq.codec import CodecConfig, encode_tensor  # noqa: E402
from hqmq.kernels import COMPILED_AVAILABLE  # noqa: E402
from hqmq.kvpack import to_bytes  # noqa: E402
from hqmq.quat import hamilton  # noqa: E402

assert COMPILED_AVAILABLE
assert os.path.realpath(hqmq.__file__).startswith(os.path.join(ROOT, "oracle", "_ref"))

D = 128
C = D // 4


def scores(x: np.ndarray, cw: np.ndarray) -> np.ndarray:
    """Reference arithmetic for (n, 4) chunks x against (m, 4) codewords."""
    s = ((x[:, 0:1] * x[:, 0:1] + x[:, 1:2] * x[:, 1:2]) + x[:, 2:3] * x[:, 2:3]) + x[:, 3:4] * x[:, 3:4]
    r = np.sqrt(s)
    u = x / r
    return ((u[:, 0:1] * cw[None, :, 0] + u[:, 1:2] * cw[None, :, 1]) + u[:, 2:3] * cw[None, :, 2]) \
        + u[:, 3:4] * cw[None, :, 3]


def top2_gap(x: np.ndarray, cw: np.ndarray):
    sc = scores(x, cw)
    order = np.argsort(-sc, axis=1, kind="stable")
    a, b = order[:, 0], order[:, 1]
    rows = np.arange(x.shape[0])
    return sc[rows, a] - sc[rows, b], a, b


def refine_fp16(x16: np.ndarray, cw: np.ndarray) -> np.ndarray:
    """For each fp16 chunk, the +-1-ulp neighbour (81 candidates) with the
    smallest top-2 gap."""
    steps = np.array(list(itertools.product((-1, 0, 1), repeat=4)), dtype=np.int16)
    bits = x16.view(np.uint16).astype(np.int32)
    best = x16.copy()
    best_gap = np.full(x16.shape[0], np.inf)
    for st in steps:
        cand_bits = bits.copy()
        for i in range(4):
            # move one ulp along the real line (sign-magnitude encoding)
            neg = (cand_bits[:, i] & 0x8000) != 0
            mag = cand_bits[:, i] & 0x7FFF
            d = int(st[i])
            mag = np.where(neg, mag - d, mag + d)
            flip = mag < 0
            mag = np.abs(mag)
            neg = neg ^ flip
            cand_bits[:, i] = (mag & 0x7FFF) | np.where(neg, 0x8000, 0)
        cand = cand_bits.astype(np.uint16).view(np.float16)
        xf = cand.astype(np.float64)
        ok = np.isfinite(xf).all(axis=1) & (np.abs(xf).sum(axis=1) > 0)
        gap, _, _ = top2_gap(np.where(ok[:, None], xf, 1.0), cw)
        gap = np.where(ok, gap, np.inf)
        better = gap < best_gap
        best[better] = cand[better]
        best_gap[better] = gap[better]
    return best


def haar(rng, n):
    q = rng.standard_normal((n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def bisector_points(rng, cw, n):
    """Directions on the bisector of their two best codewords."""
    u = haar(rng, n)
    _, a, b = top2_gap(u, cw)
    d = cw[a] - cw[b]
    u = u - ((u * d).sum(1) / (d * d).sum(1))[:, None] * d
    return u / np.linalg.norm(u, axis=1, keepdims=True)


def coset_crossovers(rng, sec, n):
    """S = 1: points of the 24-cell's own Voronoi boundaries (axis vs half:
    |v0| = (|v0|+|v1|+|v2|+|v3|)/2; half vs half: one component ~ 0), in the
    secondary's frame, rotated back: u = v * s."""
    v = np.abs(rng.standard_normal((n, 4))) + 0.05
    kind = rng.integers(0, 2, n)
    # axis-vs-half: v0 = v1 + v2 + v3
    v[kind == 0, 0] = v[kind == 0, 1:].sum(1)
    # half-vs-half: a zero component (the two half units differing in its sign tie)
    v[kind == 1, rng.integers(0, 4, int((kind == 1).sum()))] = 0.0
    perm = np.array([rng.permutation(4) for _ in range(n)])
    v = np.take_along_axis(v, perm, axis=1)
    v *= rng.choice([-1.0, 1.0], size=(n, 4))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return hamilton(v, np.broadcast_to(sec, v.shape))


def make_tensor(rng, heads, tokens, table_for, gen, fp16=True):
    x = np.zeros((1, heads, tokens, D))
    gaps = np.zeros((1, heads, tokens, C))
    for h in range(heads):
        cw = table_for(h)
        n = tokens * C
        u = gen(h, cw, 4 * n)
        g0, _, _ = top2_gap(u, cw)
        u = u[np.argsort(g0)[:n]]  # keep the tightest
        rad = rng.uniform(0.25, 6.0, n)
        pts = u * rad[:, None]
        if fp16:
            p16 = refine_fp16(pts.astype(np.float16), cw)
            pts = p16.astype(np.float64)
        gap, _, _ = top2_gap(pts, cw)
        order = rng.permutation(n)
        x[0, h] = pts[order].reshape(tokens, D)
        gaps[0, h] = gap[order].reshape(tokens, C)
    return x, gaps


def save(name, x, gaps, cfg, cast, layer=0, role="K"):
    packed = encode_tensor(x, cfg, layer=layer, role=role)
    blob = to_bytes(packed)
    meta = dict(name=name, cast=cast, codebook_size=cfg.codebook_size, radius_bits=cfg.radius_bits,
                seed=cfg.seed, layer=layer, role=role, digest=hashlib.sha256(blob).hexdigest(),
                min_gap=float(gaps.min()), n_gap_below_1e5=int((gaps < 1e-5).sum()),
                n_gap_below_1e7=int((gaps < 1e-7).sum()), n_chunks=int(gaps.size))
    np.savez_compressed(os.path.join(HERE, f"adv_{name}.npz"), data=x, gaps=gaps,
                        scales=packed.scales, indices=packed.indices, quanta=packed.quanta,
                        blob=np.frombuffer(blob, dtype=np.uint8), meta=json.dumps(meta))
    print(json.dumps(meta))
    return meta


def main():
    metas = []
    rng = np.random.default_rng(0xAD7)
    for S, layer, role in ((16, 3, "K"), (64, 1, "V"), (256, 7, "K")):
        cfg = CodecConfig(codebook_size=S, radius_bits=4, seed=S)
        bank = CodebookBank(seed=cfg.seed, size=S)
        tab = lambda h, bank=bank, layer=layer, role=role: bank.joint(layer, h, role).codewords  # noqa: E731
        x, gaps = make_tensor(rng, 2, 32, tab, lambda h, cw, n: bisector_points(rng, cw, n))
        metas.append(save(f"s{S}", x, gaps, cfg, "f16", layer=layer, role=role))
    # within-coset crossovers at S = 1 (the 24-cell decides)
    cfg = CodecConfig(codebook_size=1, radius_bits=4, seed=5)
    bank = CodebookBank(seed=cfg.seed, size=1)
    tab = lambda h: bank.joint(0, h, "K").codewords  # noqa: E731
    sec = lambda h: bank.joint(0, h, "K").secondary.entries[0]  # noqa: E731
    x, gaps = make_tensor(rng, 2, 32, tab, lambda h, cw, n: coset_crossovers(rng, sec(h), n))
    metas.append(save("s1_coset", x, gaps, cfg, "f16"))
    # fp64 input, exact bisector points (generic encode path), S = 64
    cfg = CodecConfig(codebook_size=64, radius_bits=5, seed=9)
    bank = CodebookBank(seed=cfg.seed, size=64)
    tab = lambda h: bank.joint(2, h, "K").codewords  # noqa: E731
    x, gaps = make_tensor(rng, 2, 8, tab, lambda h, cw, n: bisector_points(rng, cw, n), fp16=False)
    metas.append(save("f64_s64", x, gaps, cfg, "f64", layer=2))
    with open(os.path.join(HERE, "ADVERSARIAL.json"), "w") as f:
        json.dump(metas, f, indent=1)


if __name__ == "__main__":
    main()
