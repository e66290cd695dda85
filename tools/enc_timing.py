"""Per-call host time and device time of encode_tensor / decode_tensor on one
C2 unit (1, 8, 32768, 128) fp16, S=64, b_r=4, single stream."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27646_b200 as hq

dev = torch.device("cuda", 0)
S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
x = torch.randn((1, 8, 32768, 128), device=dev).half()
cfg = hq.CodecConfig(S, 4)
bank = hq.CodebookBank(0, S)
out = torch.empty_like(x)
for _ in range(3):
    qt = hq.encode_tensor(x, cfg, bank=bank, sync=False)
    hq.decode_tensor(qt, bank, dtype=torch.float16, out=out, check=False)
torch.cuda.synchronize()
# host time per call (GPU saturated by a long first kernel is not guaranteed: report both)
n = 20
t0 = time.perf_counter()
for _ in range(n):
    qt = hq.encode_tensor(x, cfg, bank=bank, sync=False)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"encode host {1e6*(t1-t0)/n:.1f} us/call, wall incl. drain {1e3*(t2-t0)/n:.3f} ms/call")
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(n):
    qt = hq.encode_tensor(x, cfg, bank=bank, sync=False)
b.record(); torch.cuda.synchronize()
print(f"encode device back-to-back {a.elapsed_time(b)/n:.4f} ms/call")
evs = []
for _ in range(n):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); qt = hq.encode_tensor(x, cfg, bank=bank, sync=False); e1.record(); evs.append((e0, e1))
torch.cuda.synchronize()
print("encode per-call events", [round(p.elapsed_time(q), 4) for p, q in evs[:8]])
a.record()
for _ in range(n):
    hq.decode_tensor(qt, bank, dtype=torch.float16, out=out, check=False)
b.record(); torch.cuda.synchronize()
print(f"decode device back-to-back {a.elapsed_time(b)/n:.4f} ms/call")
t0 = time.perf_counter()
for _ in range(n):
    hq.decode_tensor(qt, bank, dtype=torch.float16, out=out, check=False)
t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"decode host {1e6*(t1-t0)/n:.1f} us/call")
