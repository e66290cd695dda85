"""Randomised attention parity: fused_attend (decode steps, chunked / full prefill,
causal or not, GQA groups 1-8, Med3x or not, S in {16, 64, 256}) against the
ORACLE's dense fp64 attention (oracle.reference_attend, attention.py:80-101) over
the fp64 decode of the cache (bit-exact against the oracle's decode), tolerance
2e-3 relative to |out| where that exceeds 1 (fp16 P and V); for decode steps also
the paged cache (same tolerance) -- with Med3x a prefill append (own median) and a
frozen-threshold append, referenced against the contiguous encodes of the same
two calls with the same thresholds.

    python tools/fuzz_attention.py --cases 100 --seed 1
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import hqmq_oracle as O  # noqa: E402  (checker only)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_27646_b200 as m  # noqa: E402


def one(rs, dev):
    S = int(rs.choice([16, 64, 64, 256]))
    C = None if rs.random() < 0.7 else 3.0
    g = int(rs.choice([1, 2, 4, 8]))
    HKV = int(rs.integers(1, 4))
    B = int(rs.integers(1, 3))
    TK = int(rs.integers(1, 3000)) if rs.random() < 0.8 else int(rs.integers(4096, 7000))
    decode = rs.random() < 0.5
    TQ = 1 if decode else int(rs.integers(1, TK + 1))
    causal = True if decode else bool(rs.random() < 0.8)
    cfg = m.CodecConfig(S, 4, outlier_multiplier=C)
    bank = m.CodebookBank(0, S)
    gen = torch.Generator(device=dev).manual_seed(int(rs.integers(0, 1 << 30)))
    k = torch.randn((B, HKV, TK, 128), generator=gen, device=dev).half()
    v = torch.randn((B, HKV, TK, 128), generator=gen, device=dev).half()
    q = torch.randn((B, HKV * g, TQ, 128), generator=gen, device=dev)
    pk = m.encode_tensor(k, cfg, role="K", bank=bank)
    pv = m.encode_tensor(v, cfg, role="V", bank=bank)
    acfg = m.AttentionConfig(B, HKV * g, HKV, TQ, TK, 128, causal=causal)
    out = m.fused_attend(q, pk, pv, bank, acfg)

    def dense_of(kd, vd):
        return torch.from_numpy(O.reference_attend(q.double().cpu().numpy(), kd.cpu().numpy(),
                                                   vd.cpu().numpy(), g, causal=causal)).to(dev)

    dense = dense_of(m.decode_tensor(pk, bank, dtype=torch.float64),
                     m.decode_tensor(pv, bank, dtype=torch.float64))
    # fp16 P and V: a row that sees few keys returns ~v rounded to fp16, so the
    # bound is 2e-3 relative to |out| where that exceeds 1 (Med3x payload rows)
    diff = (out.double() - dense).abs()
    err = diff.max().item()
    rel = (diff / dense.abs().clamp_min(1.0)).max().item()
    desc = f"S={S} C={C} B={B} Hkv={HKV} g={g} Tq={TQ} Tkv={TK} causal={causal}: err {err:.2e} (scaled {rel:.2e})"
    if not rel < 2e-3:
        return False, desc
    if decode and g <= 8 and (C is None or (TK >= 2 and S <= 170)):
        cache = m.PagedKVCache(cfg, B, HKV, TK, bank=bank, device=dev,
                               page_order_seed=int(rs.integers(0, 100)))
        cut = int(rs.integers(1 if C else 0, TK + (0 if C else 1)))
        if cut:
            cache.append(k[:, :, :cut], v[:, :, :cut])
        if cut < TK:
            cache.append(k[:, :, cut:], v[:, :, cut:])
        paged = cache.attend(q)
        if C is not None:  # the reference: the same two calls, the second frozen
            parts = []
            for role, x in (("K", k), ("V", v)):
                a = m.encode_tensor(x[:, :, :cut], cfg, role=role, bank=bank)
                segs = [m.decode_tensor(a, bank, dtype=torch.float64)]
                if cut < TK:
                    b2 = m.encode_tensor(x[:, :, cut:], cfg, role=role, bank=bank,
                                         outlier_thresholds=a.outlier_thresholds)
                    segs.append(m.decode_tensor(b2, bank, dtype=torch.float64))
                parts.append(torch.cat(segs, dim=2))
            dense = dense_of(*parts)
        perr = ((paged.double() - dense).abs() / dense.abs().clamp_min(1.0)).max().item()
        d = (paged - out).abs().max().item()
        # the contiguous call may take another kernel (fp32 CUDA-core when
        # T_kv % 8 != 0) or another split of the keys, so only the tolerance
        # against the dense reference is required of the paged cache
        desc += f" | paged err {perr:.2e} (vs contiguous {d:.1e})"
        if not perr < 2e-3:
            return False, desc
    return True, desc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=100)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    rs = np.random.default_rng(args.seed)
    t0 = time.time()
    bad = 0
    for _ in range(args.cases):
        ok, desc = one(rs, dev)
        print(("ok   " if ok else "FAIL ") + desc, flush=True)
        bad += not ok
    print(f"{args.cases - bad}/{args.cases} attention cases within tolerance ({time.time() - t0:.0f} s)")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
