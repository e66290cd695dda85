"""Med3x decode output check: fp16 / bf16 / fp32 decode against the bit-exact fp64 decode."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_27646_b200 as m

dev = torch.device("cuda", 0)
for S, br in ((16, 4), (64, 6)):
    g = torch.Generator(device=dev).manual_seed(S)
    x = torch.randn((1, 8, 256, 128), generator=g, device=dev).half()
    x[:, :, ::7, 12:16] *= 30
    cfg = m.CodecConfig(S, br, outlier_multiplier=3.0)
    bank = m.CodebookBank(0, S)
    qt = m.encode_tensor(x, cfg, bank=bank)
    d64 = m.decode_tensor(qt, bank, dtype=torch.float64)
    ref16 = d64.half().double()
    for dt in (torch.float16, torch.bfloat16, torch.float32):
        d = m.decode_tensor(qt, bank, dtype=dt).double()
        rel = ((d - d64).abs() / (d64.abs() + 1e-6)).max().item()
        i = ((d - d64).abs() / (d64.abs() + 1e-6)).argmax().item()
        print(f"S={S} b_r={br} {dt}: max rel err {rel:.3e} at {i}: got {d.flatten()[i].item():.6f} "
              f"want {d64.flatten()[i].item():.6f}; mismatches vs fp16(fp64): "
              f"{(d != ref16).sum().item() if dt == torch.float16 else '-'}")
    # non-Med3x fast decode, for comparison
    qn = m.encode_tensor(x, m.CodecConfig(S, br), bank=bank)
    dn64 = m.decode_tensor(qn, bank, dtype=torch.float64)
    dn = m.decode_tensor(qn, bank, dtype=torch.float16).double()
    print(f"  no-Med3x fp16: max rel err {((dn - dn64).abs() / (dn64.abs() + 1e-6)).max().item():.3e}, "
          f"mismatches vs fp16(fp64) {(dn != dn64.half().double()).sum().item()} of {dn.numel()}")
