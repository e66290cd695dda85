"""Decode attention at the BASELINE config shapes, against the oracle
(VERDICT r01 parity items 1(b) and 1(c)).

* C4: Llama-3-8B decode step, B = 32, H_q = 32, H_kv = 8, T_q = 1, d = 128,
  S = 64, b_r = 4, at 32k keys (and 128k), the serving path (fp32 out,
  tensor cores) within the reference's fp32 bound 1e-3
  (test_attention.py:97-102) and the fp64 path within 1e-10
  (test_attention.py:83-87);
* C3: Qwen2.5-7B shape (H_q = 28, H_kv = 4, GQA 7) over an outlier-heavy cache
  encoded with Med3x (S = 64, b_r = 6, C = 3) at 32k keys.

The comparison is the oracle's dense fp64 attention (oracle.reference_attend,
attention.py:80-101) over the fp64 decode of sampled batch rows (the fp64
decode is bit-exact against the oracle's, test_gpu_parity.py), so the kernel is
never compared with itself.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def decoded_rows(m, packed, bank, rows, chunk=4096):
    """fp64 decode of batch rows `rows`, token chunk by token chunk."""
    T = packed.shape.tokens
    parts = []
    for t0 in range(0, T, chunk):
        t1 = min(T, t0 + chunk)
        d = m.decode_token_range(packed, bank, t0, t1, dtype=torch.float64)
        parts.append(d[rows].cpu().numpy())
        del d
    return np.concatenate(parts, axis=2)


def check_rows(m, oracle, q, out, pk, pv, bank, rows, group, tol, rel=False):
    kd = decoded_rows(m, pk, bank, rows)
    vd = decoded_rows(m, pv, bank, rows)
    qr = q[rows].double().cpu().numpy()
    dense = oracle.reference_attend(qr, kd, vd, group, causal=True)
    got = out[rows].double().cpu().numpy()
    err = np.abs(got - dense)
    if rel:
        err = err / np.maximum(1.0, np.abs(dense))
    assert err.max() <= tol, err.max()
    return err.max()


@pytest.mark.parametrize("T,rows", [(32768, [0, 13, 31]), (131072, [5, 30])])
def test_c4_decode_attention_full_shape(cuda, oracle, T, rows):
    import paper_2605_27646_b200 as m

    B, HQ, HKV, D = 32, 32, 8, 128
    g = torch.Generator(device=cuda).manual_seed(T)
    cfg = m.CodecConfig(64, 4)
    bank = m.CodebookBank(0, 64)
    k = torch.randn((B, HKV, T, D), generator=g, device=cuda, dtype=torch.float16)
    pk = m.encode_tensor(k, cfg, role="K", bank=bank, layer=7)
    del k
    v = torch.randn((B, HKV, T, D), generator=g, device=cuda, dtype=torch.float16)
    pv = m.encode_tensor(v, cfg, role="V", bank=bank, layer=7)
    del v
    q = torch.randn((B, HQ, 1, D), generator=g, device=cuda)
    acfg = m.AttentionConfig(B, HQ, HKV, 1, T, D)
    fast = m.fused_attend(q, pk, pv, bank, acfg)
    assert fast.dtype == torch.float32
    check_rows(m, oracle, q, fast, pk, pv, bank, rows, HQ // HKV, 1e-3)
    if T == 32768:
        exact = m.fused_attend(q.double(), pk, pv, bank, acfg)
        assert exact.dtype == torch.float64
        check_rows(m, oracle, q, exact, pk, pv, bank, rows, HQ // HKV, 1e-10)


def test_c3_med3x_decode_attention(cuda, oracle):
    import paper_2605_27646_b200 as m

    B, HQ, HKV, T, D = 4, 28, 4, 32768, 128
    g = torch.Generator(device=cuda).manual_seed(3)
    cfg = m.CodecConfig(64, 6, outlier_multiplier=3.0)
    bank = m.CodebookBank(0, 64)

    def heavy():
        x = torch.randn((B, HKV, T, D // 4, 4), generator=g, device=cuda)
        mark = torch.rand((B, HKV, T, D // 4, 1), generator=g, device=cuda) < 0.02
        mult = torch.exp(np.log(25.0) + 0.6 * torch.randn((B, HKV, T, D // 4, 1), generator=g,
                                                          device=cuda))
        return torch.where(mark, x * mult, x).reshape(B, HKV, T, D).half()

    pk = m.encode_tensor(heavy(), cfg, role="K", bank=bank, layer=2)
    pv = m.encode_tensor(heavy(), cfg, role="V", bank=bank, layer=2)
    assert pk.n_payload > 0.01 * pk.shape.n_chunks and pv.n_payload > 0
    q = torch.randn((B, HQ, 1, D), generator=g, device=cuda)
    acfg = m.AttentionConfig(B, HQ, HKV, 1, T, D)
    rows = [0, 3]
    fast = m.fused_attend(q, pk, pv, bank, acfg)
    # outlier payload rows can exceed 1 in magnitude: bound relative to |out| > 1
    check_rows(m, oracle, q, fast, pk, pv, bank, rows, HQ // HKV, 1e-3, rel=True)
    exact = m.fused_attend(q.double(), pk, pv, bank, acfg)
    check_rows(m, oracle, q, exact, pk, pv, bank, rows, HQ // HKV, 1e-10)
