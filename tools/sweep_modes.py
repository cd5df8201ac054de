#!/usr/bin/env python
"""Experiment driver: times the row pass and the fused column+DoG pass for every sweep
variant (DOGBLOB_SWEEP, see csrc/scale_space.cu SweepCfg) in a fresh process each, and checks
that every variant returns the same blobs bit for bit.

    python tools/sweep_modes.py [--configs C2,C4] [--modes 0,1,3,...] [--groups G]
"""
import argparse
import hashlib
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def child(config):
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import torch
    import paper_2010_08486_b200 as P
    from paper_2010_08486_b200 import detector as D, synth
    kw = synth.config_params(config)
    frames = [synth.config_frame("C3", i) for i in range(4)] if config == "C2" else [synth.config_frame(config)]
    params = P.DetectionParams(preprocess=False, **kw)
    det = P.Detector(params, slots=1)
    H, W = frames[0].shape
    eng = det.plan_for((H, W))
    dev = torch.device("cuda", det.device)
    resident = []
    for f in frames:
        d = torch.zeros((H, eng.plan.pitch), dtype=torch.float32, device=dev)
        d[:, :W] = torch.from_numpy(f).to(dev)
        resident.append(d)
    slot = eng.slots[0]
    for _ in range(3):
        for d in resident:
            slot.launch_device(d, params, True)
    torch.cuda.synchronize()
    reps = 8
    sets = [D.new_events() for _ in range(reps * len(resident))]
    k = 0
    for _ in range(reps):
        for d in resident:
            slot.launch_device(d, params, True, events=sets[k])
            k += 1
    torch.cuda.synchronize()
    iv = np.array([D.event_intervals_ms(es) for es in sets])
    h = hashlib.sha256()
    for f in frames:
        r = det.run(f)
        h.update(repr([(b.x, b.y, b.sigma, b.radius, b.response, b.at_scale_boundary) for b in r.blobs.blobs]).encode())
    print(json.dumps({"row_ms": float(np.median(iv[:, 0])), "col_ms": float(np.median(iv[:, 1])),
                      "row_min": float(iv[:, 0].min()), "col_min": float(iv[:, 1].min()),
                      "extrema_ms": float(np.median(iv[:, 2])), "prune_ms": float(np.median(iv[:, 3])),
                      "blobs_sha": h.hexdigest()[:12]}))
    det.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C4")
    ap.add_argument("--modes", default="0,1,3,4,6,8,9,11,12,14")
    ap.add_argument("--groups", default="")
    ap.add_argument("--child", default="")
    a = ap.parse_args()
    if a.child:
        child(a.child)
        return
    for cfg in a.configs.split(","):
        for g in (a.groups.split(",") if a.groups else [""]):
            for m in a.modes.split(","):
                env = dict(os.environ, DOGBLOB_SWEEP=m)
                if g:
                    env["DOGBLOB_GROUPS"] = g
                r = subprocess.run([sys.executable, __file__, "--child", cfg], env=env, capture_output=True, text=True)
                line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-400:]
                print(cfg, "groups", g or "auto", "mode", m, line, flush=True)


if __name__ == "__main__":
    main()
