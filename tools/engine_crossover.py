#!/usr/bin/env python
"""Where the tensor-core engine starts to beat the FP32 engine: scale-space time of both for a grid of frame sizes and
ladders (the plan's own choice is marked).  Test tooling only.

    python tools/engine_crossover.py [HxW ...]
"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2010_08486_b200 as P  # noqa: E402
from paper_2010_08486_b200 import synth  # noqa: E402


def conv_ms(frame, kw, engine):
    if engine:
        os.environ["DOGBLOB_CONV"] = engine
    else:
        os.environ.pop("DOGBLOB_CONV", None)
    det = P.Detector(P.DetectionParams(preprocess=False, **kw), slots=1)
    try:
        used = det.plan_for(frame.shape).plan.conv_engine
        ts = []
        for i in range(12):
            r = det.run(frame)
            if i >= 4:
                ts.append(r.timings_ms["convolve_ms"])
        return float(np.median(ts)), used, len(r.blobs)
    finally:
        det.close()
        os.environ.pop("DOGBLOB_CONV", None)


shapes = [(int(a), int(b)) for a, b in (s.split("x") for s in sys.argv[1:])] or [(n, n) for n in (512, 768, 1024, 1536)]
for Hh, Ww in shapes:
    size = f"{Hh}x{Ww}"
    frame = synth.sensor_noise(synth.droplet_scene(Ww, Hh, 40, (3.0, min(20.0, Hh / 12, Ww / 12)), seed=3), seed=4).image
    assert frame.shape == (Hh, Ww)
    for max_sigma, n_bin in ((3, 6), (6, 12), (10, 20), (15, 30), (20, 40), (30, 58)):
        kw = dict(min_sigma=1.0, max_sigma=float(max_sigma), n_bin=n_bin)
        f, _, nb = conv_ms(frame, kw, "fma")
        try:
            u, _, nb2 = conv_ms(frame, kw, "umma")
        except Exception as e:      # the tensor engine cannot stage this plan
            u, nb2 = float("nan"), -1
        _, chosen, _ = conv_ms(frame, kw, None)
        print(f"{size} sigma<={max_sigma:2d} n_bin {n_bin:2d}: fp32 {f:.4f} ms  tensor {u:.4f} ms  "
              f"ratio {f / u:.2f}  plan chooses {'tensor' if chosen == 2 else 'fp32'}  blobs {nb}/{nb2}", flush=True)
