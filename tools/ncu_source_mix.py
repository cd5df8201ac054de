#!/usr/bin/env python
"""Instruction mix and stall samples per opcode from `ncu -i rep --page source --csv`.

  ncu -i gpurun_out/x.ncu-rep --page source --csv > src.csv; python tools/ncu_source_mix.py src.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
kern = []
cur = None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        kern.append(cur)
        continue
    if cur is None:
        continue
    if r and r[0] == "Address":
        cur["hdr"] = r
        continue
    if r and r[0].startswith("0x"):
        cur["rows"].append(r)
for k in kern:
    h = k["hdr"]
    ix = {n: i for i, n in enumerate(h)}
    print(k["name"][:70], len(k["rows"]), "SASS lines")
    tot = collections.Counter()
    opc = collections.Counter()
    opi = collections.Counter()
    stall_cols = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
    totsamp = 0
    for r in k["rows"]:
        s = int(r[ix["# Samples"]])
        totsamp += s
        ins = int(r[ix["Instructions Executed"]])
        op = [o for o in r[ix["Source"]].split() if not o.startswith("@")][0].rstrip(";")
        op = "FFMA2" if op.startswith("FFMA2") else op.split(".")[0]
        opc[op] += s
        opi[op] += ins
        for c in stall_cols:
            tot[c] += int(r[ix[c]])
    ti = sum(opi.values())
    print("  samples", totsamp, "warp-instructions", ti)
    print("  stalls  :", [(c[6:], round(100 * v / totsamp, 1)) for c, v in tot.most_common(9)])
    print("  mix %   :", [(o, round(100 * v / ti, 1)) for o, v in opi.most_common(16)])
    print("  samples%:", [(o, round(100 * v / totsamp, 1)) for o, v in opc.most_common(10)])
