#!/usr/bin/env python
"""Timing experiments on the tensor-core passes: DOGBLOB_UMMA_DEBUG masks (results are garbage for
most masks, only the stage times matter).  Test tooling only.

    python tools/umma_masks.py C2 0 1 2 8 ...
"""
import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("DOGBLOB_UMMA_DEBUG", "0")      # the library only honours the masks if this exists at load time

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2010_08486_b200 as P  # noqa: E402
from paper_2010_08486_b200 import detector as D, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
masks = [int(x) for x in sys.argv[2:]] or [0]
frame, kw = synth.config_frame(name), synth.config_params(name)
if os.environ.get("UMMA_MASKS_SHAPE"):      # HxW: the config's frame cropped / tiled to another shape
    hh, ww = (int(v) for v in os.environ["UMMA_MASKS_SHAPE"].split("x"))
    frame = np.ascontiguousarray(np.tile(frame, (hh // frame.shape[0] + 1, ww // frame.shape[1] + 1))[:hh, :ww])
params = P.DetectionParams(preprocess=False, **kw)
import dataclasses  # noqa: E402
# garbage planes under a mask: nothing may be flagged; UMMA_MASKS_THR=<threshold> times the real detection path (mask 0 only)
run_params = dataclasses.replace(params, threshold=float(os.environ.get("UMMA_MASKS_THR", "inf")))
H, W = frame.shape
det = P.Detector(params, slots=1)
eng = det.plan_for((H, W))
slot = eng.slots[0]
dev = torch.device("cuda", torch.cuda.current_device())
d_img = torch.zeros((H, eng.plan.pitch), dtype=torch.float32, device=dev)
d_img[:, :W] = torch.from_numpy(frame).to(dev)
for m in masks:
    os.environ["DOGBLOB_UMMA_DEBUG"] = str(m)
    for _ in range(3):
        slot.launch_device(d_img, run_params, True)
    torch.cuda.synchronize()
    sets = [D.new_events() for _ in range(12)]
    for es in sets:
        slot.launch_device(d_img, run_params, True, events=es)
    torch.cuda.synchronize()
    med = np.median(np.array([D.event_intervals_ms(es) for es in sets]), axis=0)
    print(f"{name} mask {m:3d}: row {med[0]:.4f}  col+dog {med[1]:.4f}  extrema {med[2]:.4f}  prune {med[3]:.4f} ms", flush=True)
os.environ["DOGBLOB_UMMA_DEBUG"] = "0"
det.close()
