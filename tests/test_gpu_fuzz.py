"""Randomised parity (tools/fuzz_parity.py): random shapes, codebook sizes, radius
bits, Med3x multipliers, pooling, dtypes, roles and head_base; kvpack bytes and
fp64 decode bit-exact against the oracle.  The round's evidence run covers 2000
cases (profiles/r01g_fuzz_parity.log); this keeps 60 in the GPU suite."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fuzz_parity(cuda):
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_parity.py"),
                          "--cases", "60", "--seed", "2024"], capture_output=True, text=True,
                         timeout=900)
    assert res.returncode == 0, (res.stdout[-3000:], res.stderr[-2000:])
    assert "60/60 cases bit-exact" in res.stdout


def test_fuzz_attention(cuda):
    """tools/fuzz_attention.py: decode / prefill / paged attention over random shapes,
    GQA groups, causal masks, Med3x and codebook sizes within 2e-3 of the dense
    fp64 attention over the decoded cache (1000 cases in
    profiles/r01g_fuzz_attention.log; 80 here)."""
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_attention.py"),
                          "--cases", "80", "--seed", "77"], capture_output=True, text=True,
                         timeout=900)
    assert res.returncode == 0, (res.stdout[-3000:], res.stderr[-2000:])
    assert "80/80 attention cases within tolerance" in res.stdout
