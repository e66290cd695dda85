"""Randomised parity sweep: random shapes / codebook sizes / radius bits / Med3x
multipliers / pooling / input dtypes / head_base / roles, the sm_100a encode +
kvpack bytes against the oracle (bit-exact) and the fp64 decode against the
oracle's decode (bit-exact).  Test infrastructure (imports oracle/).

    python tools/fuzz_parity.py --cases 200 --seed 1
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import hqmq_oracle as O  # noqa: E402
import paper_2605_27646_b200 as m  # noqa: E402


def one(rs, dev, threads):
    S = int(rs.choice([16, 24, 32, 48, 64, 96, 128, 256]))
    br = int(rs.integers(1, 9))
    C = [None, None, 2.5, 3.0][int(rs.integers(0, 4))]
    pooling = "per_head" if rs.random() < 0.3 else "batch"
    D = int(rs.choice([4, 12, 64, 126, 128, 128, 128]))
    B, H = int(rs.integers(1, 3)), int(rs.integers(1, 5))
    T = int(rs.integers(1, 400)) if rs.random() < 0.8 else int(rs.integers(400, 3000))
    dt = [torch.float16, torch.float16, torch.bfloat16, torch.float32, torch.float64][int(rs.integers(0, 5))]
    role = "K" if rs.random() < 0.5 else "V"
    layer, head_base, seed = int(rs.integers(0, 80)), int(rs.integers(0, 4)), int(rs.integers(0, 3))
    x = rs.standard_normal((B, H, T, D))
    if rs.random() < 0.3:  # outlier-heavy chunks
        idx = rs.random(x.shape) < 0.02
        x[idx] *= 40.0
    if rs.random() < 0.1:  # all-zero tokens
        x[:, :, : max(1, T // 7)] = 0.0
    xt = torch.from_numpy(x).to(dev).to(dt)
    x64 = xt.double().cpu().numpy()
    cfg = m.CodecConfig(codebook_size=S, radius_bits=br, seed=seed, outlier_multiplier=C,
                        median_pooling=pooling)
    bank = m.CodebookBank(seed, S)
    qt = m.encode_tensor(xt, cfg, layer=layer, role=role, bank=bank, head_base=head_base)
    ref = O.encode(x64, S, br, seed=seed, multiplier=C, pooling=pooling, layer=layer, role=role,
                   head_base=head_base, threads=threads)
    desc = f"S={S} br={br} C={C} pool={pooling} shape={(B, H, T, D)} {dt} {role} L{layer} hb{head_base} seed{seed}"
    if m.to_bytes(qt) != O.to_bytes(ref):
        return False, desc + " : kvpack bytes differ"
    dec = m.decode_tensor(qt, bank, dtype=torch.float64).cpu().numpy()
    if not np.array_equal(dec, O.decode(ref)):
        return False, desc + " : fp64 decode differs"
    return True, desc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=100)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    rs = np.random.default_rng(args.seed)
    threads = os.cpu_count() or 1
    t0 = time.time()
    bad = 0
    for i in range(args.cases):
        ok, desc = one(rs, dev, threads)
        print(("ok   " if ok else "FAIL ") + desc, flush=True)
        bad += not ok
    print(f"{args.cases - bad}/{args.cases} cases bit-exact ({time.time() - t0:.0f} s)")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
