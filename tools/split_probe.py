import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2605_27646_b200 as hq
dev = torch.device("cuda", 0)
xs = [torch.randn((1, 8, 32768, 128), device=dev).half() for _ in range(16)]
cfg = hq.CodecConfig(64, 4); bank = hq.CodebookBank(0, 64)
out = [torch.empty_like(xs[0]) for _ in range(2)]
def one(with_dec, n=32):
    recs = []
    for i in range(n):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e2 = torch.cuda.Event(enable_timing=True)
        e0.record()
        qt = hq.encode_tensor(xs[i % 16], cfg, layer=i, role="K", bank=bank, sync=False)
        e1.record()
        if with_dec: hq.decode_tensor(qt, bank, dtype=torch.float16, out=out[i & 1], check=False)
        e2.record()
        recs.append((e0, e1, e2))
    torch.cuda.synchronize()
    enc = [a.elapsed_time(b) for a, b, _ in recs]
    return sum(enc) / n, max(enc), min(enc)
for layer_var in (False, True):
    pass
one(True); one(False)
print("enc+dec loop: avg/max/min enc ms", one(True))
print("enc-only loop: avg/max/min enc ms", one(False))
