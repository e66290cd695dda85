"""Summarise gpurun_out/ ncu artefacts into tracked text files under profiles/.

    python tools/summarize_profiles.py <tag>            # e.g. r01a

Reads (whatever exists):
  gpurun_out/launches.csv     ncu --metrics gpu__time_duration.sum launch list
  gpurun_out/prof_*.ncu-rep   ncu --set full captures
  gpurun_out/bench.log        bench.py JSON line
and writes profiles/<tag>_launches.txt, profiles/<tag>_ncu_<name>.txt,
profiles/<tag>_bench.json.
"""

import collections
import csv
import glob
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "lts__t_sectors_srcunit_tex_op_write.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "sm__cycles_elapsed.avg.per_second",
]


def launches(tag):
    path = os.path.join(OUT, "launches.csv")
    if not os.path.exists(path):
        return
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        agg[r[ki][:110]][0] += 1
        agg[r[ki][:110]][1] += v
    tot = sum(a[1] for a in agg.values()) or 1.0
    lines = ["# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised;",
             "# compare SHARES, not absolutes).  count  total_ms  share  avg_us  kernel"]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{c:6d} {t / 1e6:10.3f} {100 * t / tot:6.1f}% {t / c / 1e3:10.1f}  {n}")
    with open(os.path.join(PROF, f"{tag}_launches.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")


def ncu_reports(tag):
    for rep in sorted(glob.glob(os.path.join(OUT, "prof_*.ncu-rep"))):
        name = os.path.basename(rep)[5:-8]
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            continue
        h, units = rows[0], rows[1]
        lines = [f"# ncu --set full --clock-control none capture: {os.path.basename(rep)}"]
        for r in rows[2:]:
            if len(r) < len(h):
                continue
            lines.append("")
            lines.append(f"kernel: {r[h.index('Kernel Name')]}")
            for m in METRICS:
                if m in h:
                    i = h.index(m)
                    lines.append(f"  {m:66s} {r[i]:>16s} {units[i]}")
            if "dram__bytes_read.sum" in h:
                def to_bytes(i):
                    u = units[i]
                    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                    return float(r[i].replace(",", "")) * mul
                t = to_bytes(h.index("dram__bytes_read.sum")) + to_bytes(h.index("dram__bytes_write.sum"))
                lines.append(f"  {'traffic (dram read+write)':66s} {t:16.0f} byte")
        with open(os.path.join(PROF, f"{tag}_ncu_{name}.txt"), "w") as f:
            f.write("\n".join(lines) + "\n")


def bench(tag):
    for log in sorted(glob.glob(os.path.join(OUT, "bench*.log"))):
        for line in open(log):
            if line.startswith("{"):
                base = os.path.basename(log)[:-4]
                with open(os.path.join(PROF, f"{tag}_{base}.json"), "w") as f:
                    json.dump(json.loads(line), f, indent=1)
                    f.write("\n")


if __name__ == "__main__":
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    launches(tag)
    ncu_reports(tag)
    bench(tag)
    print(sorted(os.listdir(PROF)))
