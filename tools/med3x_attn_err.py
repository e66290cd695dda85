"""Error anatomy of the Med3x tensor-core decode attention vs the oracle."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np, torch
import paper_2605_27646_b200 as m
import hqmq_oracle as O
from test_gpu_med3x_serving import heavy, np64

dev = torch.device("cuda", 0)
for (S, br, B, HQ, HKV, TQ, T, causal, C) in [(64, 6, 2, 8, 2, 1, 2048, True, 3.0),
                                                (64, 6, 2, 8, 2, 1, 2048, True, None)]:
    gen = torch.Generator(device=dev).manual_seed(T + S)
    cfg = m.CodecConfig(S, br, outlier_multiplier=C)
    bank = m.CodebookBank(0, S)
    k = heavy((B, HKV, T, 128), gen, dev); v = heavy((B, HKV, T, 128), gen, dev)
    pk = m.encode_tensor(k, cfg, role="K", bank=bank, layer=4)
    pv = m.encode_tensor(v, cfg, role="V", bank=bank, layer=4)
    q = torch.randn((B, HQ, TQ, 128), generator=gen, device=dev)
    acfg = m.AttentionConfig(B, HQ, HKV, TQ, T, 128, causal=causal)
    kd = m.decode_tensor(pk, bank, dtype=torch.float64).cpu().numpy()
    vd = m.decode_tensor(pv, bank, dtype=torch.float64).cpu().numpy()
    dense = O.reference_attend(np64(q), kd, vd, HQ // HKV, causal=causal)
    print("C", C, "kernel", m.attention_kernel(q, pk, pv, bank, acfg), "|dense| max", np.abs(dense).max())
    for name, kw in [("fast", {}), ("precise", {"precise": True})]:
        out = np64(m.fused_attend(q, pk, pv, bank, acfg, **kw))
        e = np.abs(out - dense); rel = e / np.maximum(1, np.abs(dense))
        i = np.unravel_index(rel.argmax(), rel.shape)
        print(f"  {name}: abs max {e.max():.3e} rel max {rel.max():.3e} at {i} dense {dense[i]:.4f} "
              f"mean abs {e.mean():.3e}")

# timing: C3-shaped decode step (Qwen2.5-7B: H_q 28, H_kv 4), Med3x tensor-core
# kernel vs the fp32 CUDA-core kernel vs the same cache without extraction
def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(reps):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

B, HQ, HKV, T = 16, 28, 4, 32768
gen = torch.Generator(device=dev).manual_seed(1)
for C in (3.0, None):
    cfg = m.CodecConfig(64, 6, outlier_multiplier=C)
    bank = m.CodebookBank(0, 64)
    pk = m.encode_tensor(heavy((B, HKV, T, 128), gen, dev), cfg, role="K", bank=bank)
    pv = m.encode_tensor(heavy((B, HKV, T, 128), gen, dev), cfg, role="V", bank=bank)
    q = torch.randn((B, HQ, 1, 128), generator=gen, device=dev)
    acfg = m.AttentionConfig(B, HQ, HKV, 1, T, 128)
    out = torch.empty((B, HQ, 1, 128), device=dev)
    tf = timeit(lambda: m.fused_attend(q, pk, pv, bank, acfg, out=out))
    tp = timeit(lambda: m.fused_attend(q, pk, pv, bank, acfg, precise=True, out=out))
    print(f"C={C} B={B} HQ={HQ} HKV={HKV} T={T}: {m.attention_kernel(q, pk, pv, bank, acfg)} "
          f"{tf:.4f} ms, fp32 CUDA-core kernel {tp:.4f} ms")
    del pk, pv
