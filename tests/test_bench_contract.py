"""bench.py's reference arm (the reference's own CPU path, oracle/_ref) keeps the
driver's JSON contract.  CPU-only; the GPU arm is exercised on the B200."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

REF = os.path.join(ROOT, "oracle", "_ref")


@pytest.mark.skipif(not os.path.isdir(REF), reason="oracle/_ref not built")
def test_reference_arm_json_line():
    res = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
         "--warmup", "0", "--ref-step-seconds", "0.5"],
        capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    line = [ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s"
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_clock_sampler_summary():
    """The clocks object of the JSON line: median SM clock, max clock, and the
    throttle reasons seen by any sample (NVML bitmask or nvidia-smi CSV)."""
    sys.path.insert(0, ROOT)
    import bench

    class FakeNvml:
        nvmlClocksEventReasonHwSlowdown = 0x8
        nvmlClocksEventReasonHwThermalSlowdown = 0x40
        nvmlClocksEventReasonSwThermalSlowdown = 0x20
        nvmlClocksEventReasonSwPowerCap = 0x4

    cs = bench.ClockSampler(0)
    cs.nvml, cs.source = (FakeNvml, None), "nvml, 10 ms period"
    cs.samples = [(1965, 1965, 0), (1890, 1965, 0x4), (1965, 1965, 0)]
    s = cs.summary()
    assert s["sm_mhz"] == 1965 and s["sm_max_mhz"] == 1965 and s["samples"] == 3
    assert s["reasons"] == ["sw_power_cap"] and s["source"].startswith("nvml")
    cs2 = bench.ClockSampler(0)
    cs2.lines = ["1965, 1965, 700.0, Not Active, Not Active, Active, Not Active"]
    s2 = cs2.summary()
    assert s2["reasons"] == ["sw_thermal_slowdown"] and s2["samples"] == 1
    assert bench.ClockSampler(0).summary()["samples"] == 0
