"""C2 split-pass diagnostic: per-pass encode / decode time of all 64 units back
to back on one stream, repeated, with the SM clock sampled around each pass."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27646_b200 as hq

dev = torch.device("cuda", 0)
units = [(l, r) for l in range(32) for r in ("K", "V")]
cfg = hq.CodecConfig(64, 4)
bank = hq.CodebookBank(0, 64)
inputs = []
for l, r in units:
    g = torch.Generator(device=dev).manual_seed(1000 + 2 * l + (r == "V"))
    inputs.append(torch.randn((1, 8, 32768, 128), generator=g, device=dev).half())
    bank.device_tables(l, 0, 8, r, dev)
outs = [torch.empty_like(inputs[0]) for _ in range(2)]

def clk():
    return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                           "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()

for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    qts = [hq.encode_tensor(x, cfg, layer=l, role=r, bank=bank, sync=False) for (l, r), x in zip(units, inputs)]
    e[1].record()
    for i, qt in enumerate(qts):
        hq.decode_tensor(qt, bank, dtype=torch.float16, out=outs[i % 2], check=False)
    e[2].record()
    c = clk()
    torch.cuda.synchronize()
    print(f"pass {rep}: enc {e[0].elapsed_time(e[1]):.2f} ms dec {e[1].elapsed_time(e[2]):.3f} ms | {c}", flush=True)
    del qts
