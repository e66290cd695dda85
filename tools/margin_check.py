"""Certification-margin experiment: encode the 64 C2 units (or 160 C5 units with
--c5) of the bench, report encode time, fixup count and a digest of every
unit's index / radius streams (to compare builds with different margins)."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27646_b200 as hq
from bench import WORKLOADS, make_input
dev = torch.device("cuda", 0)
wl = WORKLOADS["c5" if "--c5" in sys.argv else "c2"]
S = wl["S"]
cfg = hq.CodecConfig(S, wl["br"])
bank = hq.CodebookBank(0, S)
layers = wl["layers"] if "--c5" not in sys.argv else 16
units = [(l, r) for l in range(layers) for r in ("K", "V")]
h = hashlib.sha256()
fix = 0
tot_ms = 0.0
for (l, r) in units:
    x = make_input(torch, wl, l, r, dev)
    bank.device_tables(l, 0, wl["heads"], r, dev)
    for rep in range(2):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        qt = hq.encode_tensor(x, cfg, layer=l, role=r, bank=bank, sync=False)
        b.record()
        qt.synchronize()
    tot_ms += a.elapsed_time(b)
    fix += qt.n_fixup
    h.update(qt.index_words.cpu().numpy().tobytes())
    h.update(qt.radius_words.cpu().numpy().tobytes())
    h.update(qt.scales.cpu().numpy().tobytes())
    del x, qt
print(f"units {len(units)} encode {tot_ms:.2f} ms fixups {fix} digest {h.hexdigest()[:32]}")
