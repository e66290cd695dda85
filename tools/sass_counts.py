"""Count the Blackwell-specific SASS mnemonics per kernel of the built library
(cuobjdump -sass): tcgen05 MMA (UTCHMMA / UTCQMMA), TMEM loads / stores (LDTM /
STTM), TMA bulk copies (UBLKCP), L2 bulk prefetch (UBLKPF), DSMEM async stores
(STAS), legacy mma.sync (HMMA), packed fp32 (FFMA2 / FMUL2 / FADD2).

    python tools/sass_counts.py > profiles/r02_sass_counts.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_27646_b200", "_lib", "libhqmq_b200.so")
OPS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UBLKPF", "SYNCS", "STAS", "HMMA",
       "FFMA2", "FMUL2", "FADD2", "DFMA", "DMUL"]

sass = subprocess.run(["cuobjdump", "-sass", sys.argv[1] if len(sys.argv) > 1 else LIB],
                      capture_output=True, text=True).stdout
counts = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
    if m:
        op = m.group(1)
        for o in OPS:
            if op == o or op.startswith(o + "."):
                counts[cur][o] += 1
print("# SASS mnemonic counts per kernel (cuobjdump -sass of the built library, sm_100a)")
print("# " + " ".join(OPS))
for fn, c in counts.items():
    if any(c.values()):
        demangled = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip()
        print(f"{demangled[:110]}")
        print("    " + "  ".join(f"{o}={c[o]}" for o in OPS if c[o]))
