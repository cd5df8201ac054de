#!/usr/bin/env python
"""Turn the files tools/round_profiles.sh brought back in gpurun_out/ into the tracked summaries under
profiles/ (bench lines, config timings, launch lists with DRAM bytes, ncu summaries, role cycles,
sanitizer tails, traffic json, SASS opcodes).

    python tools/write_round_profiles.py r02
"""
import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
G, P = ROOT / "gpurun_out", ROOT / "profiles"
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"

for src, dst in (("bench.json", f"{tag}_bench.json"), ("bench_reference.json", f"{tag}_bench_reference.json"),
                 ("bench_2ranks_1gpu.json", f"{tag}_bench_2ranks_on_1gpu.json"),
                 ("config_timings.jsonl", f"{tag}_config_timings.jsonl"), ("r02_parity.json", f"{tag}_parity.json")):
    if (G / src).exists():
        shutil.copy(G / src, P / dst)

with open(P / f"{tag}_umma_role_cycles.md", "w") as f:
    f.write(f"# Round {tag[1:]} - per-role cycle counters and CTA timeline of the tensor-core passes "
            "(DOGBLOB_UMMA_PROF=1 python tools/umma_masks.py <config> 0)\n\n```\n")
    for c in ("C2", "C4"):
        if (G / f"roles_{c}.txt").exists():
            f.write(f"== {c}\n" + (G / f"roles_{c}.txt").read_text())
    f.write("```\n")

with open(P / f"{tag}_sanitizer.md", "w") as f:
    f.write(f"# Round {tag[1:]} - compute-sanitizer memcheck (tools/sanitize_run.py: ragged shapes, dense frame, preprocessing)\n")
    for name, title in (("san_memcheck.log", "Default engine choice"), ("san_memcheck_umma.log", "Tensor-core engine forced (DOGBLOB_CONV=umma)")):
        if (G / name).exists():
            f.write(f"\n{title}:\n```\n" + "\n".join((G / name).read_text().splitlines()[-4:]) + "\n```\n")

if (G / "stress_engines.txt").exists():
    txt = (G / "stress_engines.txt").read_text().splitlines()
    (P / f"{tag}_stress_engines.md").write_text(
        f"# Round {tag[1:]} - randomised engine cross-check (tools/stress_engines.py 120 5): random ragged shapes, ladders, "
        "thresholds; tensor-core DoG slices vs the FP32 engine's, detector vs stage functions on the same stack, frame "
        "sequences through one slot (stale slice memory)\n\n```\n" + "\n".join(txt[:12] + ["..."] + txt[-3:]) + "\n```\n")
    extra = [(n, c) for n, c in (("stress_400.txt", "python tools/stress_engines.py 400 77"),
                                 ("stress_large.txt", "python tools/stress_engines.py 60 78 large        # frames up to 2600 px, sigma up to 60"))
             if (G / n).exists()]
    if extra:
        with open(P / f"{tag}_stress_engines.md", "a") as f:
            f.write("\nExtended runs with the final build (FAIL lines: "
                    + str(sum((G / n).read_text().count("FAIL") for n, _ in extra)) + "):\n\n```\n")
            for n, c in extra:
                f.write(c + "\n" + (G / n).read_text().splitlines()[-1] + "\n")
            f.write("```\n")

rows = list(csv.reader(open(G / "launches_one_frame.csv")))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
cols = rows[h]
ki, mi, vi = cols.index("Kernel Name"), cols.index("Metric Name"), cols.index("Metric Value")
cur, order = {}, []
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    k = (int(r[0]), r[ki].split("(")[0].replace("void ", "").split("::")[-1])
    if k not in cur:
        order.append(k)
    cur.setdefault(k, {})[r[mi]] = float(r[vi].replace(",", ""))
lines = [f"# Round {tag[1:]} - kernels of one C2 frame (tools/profile_run.py --frames 5, last frame), tensor-core engine", "",
         "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none` (per-launch "
         "times are cold-cache and serialised: compare shares, not absolutes)", "",
         "| # | kernel | us | DRAM read MB | DRAM write MB |", "|---:|---|---:|---:|---:|"]
tot, traffic = 0.0, {}
for k in order:
    v = cur[k]
    us = v["gpu__time_duration.sum"] / 1e3
    tot += us
    lines.append(f"| {k[0]} | `{k[1]}` | {us:.2f} | {v['dram__bytes_read.sum'] / 1e6:.1f} | {v['dram__bytes_write.sum'] / 1e6:.1f} |")
    traffic[k[1]] = v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]
lines.append(f"| | total | {tot:.1f} | | |")
(P / f"{tag}_launches_one_frame.md").write_text("\n".join(lines) + "\n")
old = json.loads((P / "ncu_traffic.json").read_text())
old.update({"source": f"profiles/{tag}_launches_one_frame.md (ncu dram__bytes_read.sum + dram__bytes_write.sum per launch, C2 frame)",
            "umma_col_dog_kernel_dram_bytes_per_launch": next((v for k, v in traffic.items() if k.startswith("umma_pass_kernel<1")), None),
            "umma_row_kernel_dram_bytes_per_launch": next((v for k, v in traffic.items() if k.startswith("umma_pass_kernel<0")), None),
            "nms_kernel_dram_bytes_per_launch": next((v for k, v in traffic.items() if k.startswith("nms_")), None)})
(P / "ncu_traffic.json").write_text(json.dumps(old, indent=1) + "\n")

py = sys.executable
subprocess.run([py, str(ROOT / "tools" / "summarize_ncu.py"), "launches", str(G / "launches_bench.csv"),
                str(P / f"{tag}_launches_bench.md"),
                f"Round {tag[1:]} - kernels of bench.py --steps 2 --warmup 1 (DOGBLOB_BENCH_BATCH=16, tensor-core engine)"],
               stdout=subprocess.DEVNULL)
subprocess.run([py, str(ROOT / "tools" / "summarize_ncu.py"), "full", str(G / "umma_full.ncu-rep"),
                str(P / f"{tag}_ncu_umma_nms_kernels.md"),
                f"Round {tag[1:]} - ncu --set full of the tensor-core passes and the extrema kernel (C2 frame)"],
               stdout=subprocess.DEVNULL)
subprocess.run([py, str(ROOT / "tools" / "sass_opcodes.py"), str(P / f"{tag}_sass_opcodes.md")], stdout=subprocess.DEVNULL)
print("profiles written:", sorted(p.name for p in P.glob(f"{tag}_*")))
