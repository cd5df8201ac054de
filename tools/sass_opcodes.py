#!/usr/bin/env python
"""Opcode histogram per kernel of the built library (cuobjdump -sass), the evidence that the hot
kernels are Blackwell-native: UTCHMMA (tcgen05.mma), LDTM / STTM (tcgen05.ld / st), UTMALDG /
UTMASTG / UBLKCP (TMA loads / stores / bulk copies), FFMA2 (packed FP32 FMA), SYNCS (mbarrier).

    python tools/sass_opcodes.py [out.md]
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2010_08486_b200" / "libdogblob_b200.so"
KEY = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "UTMAPF", "SYNCS", "FFMA2", "FFMA",
       "HMMA", "LDGSTS", "LDG", "STG", "LDS", "STS", "R2UR", "ELECT", "DFMA", "DADD", "DMUL", "ATOMG", "RED",
       "SHFL", "VOTE", "BAR"]

sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
kernels = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"\(anonymous namespace\)::|dogblob::|void ", "", name)
        cur = kernels.setdefault(name.split("(")[0], collections.Counter())
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\d+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and cur is not None:
        cur[m.group(1)] += 1
out = ["# SASS opcode histogram per kernel (`cuobjdump -sass libdogblob_b200.so`, sm_100a)", "",
       "Counts of static instructions. tcgen05.mma = `UTCHMMA`, tcgen05.commit = `UTCBAR`, tcgen05.ld/st = `LDTM`/`STTM`, "
       "TMA = `UTMALDG`/`UTMASTG`/`UBLKCP`, mbarrier = `SYNCS`, packed FP32 FMA = `FFMA2`.", "",
       "| kernel | total | " + " | ".join(KEY) + " |", "|---|---:|" + "---:|" * len(KEY)]
for name, c in kernels.items():
    out.append(f"| `{name}` | {sum(c.values())} | " + " | ".join(str(c.get(k, 0)) if c.get(k, 0) else "" for k in KEY) + " |")
text = "\n".join(out) + "\n"
if len(sys.argv) > 1:
    Path(sys.argv[1]).write_text(text)
print(text)
