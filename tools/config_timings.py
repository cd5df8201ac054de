#!/usr/bin/env python
"""Per-configuration timings of the BASELINE.json configs (C1, C2, C4, C5): device stage
times (CUDA events, single stream), single-frame end-to-end latency, blob counts.
Prints one JSON line per config; used for the tables in DESIGN.md / profiles/."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2010_08486_b200 as P  # noqa: E402
from paper_2010_08486_b200 import synth  # noqa: E402

for name in (sys.argv[1:] or ["C1", "C2", "C4", "C5"]):
    extra = {}
    if name == "C5b":
        frame, kw, extra = synth.config_frame("C5"), synth.config_params("C5"), {"overlap": 0.1}
    elif name == "P1000":   # "typical blobs per sample ~1000": 1000 droplets, package default ladder
        frame = synth.sensor_noise(synth.droplet_scene(1024, 1024, 1000, (3.0, 12.0), seed=21,
                                                       allow_overlap=True), seed=22).image
        kw = dict(min_sigma=1.0, max_sigma=10.0, n_bin=18)
    else:
        frame, kw = synth.config_frame(name), synth.config_params(name)
    det = P.Detector(P.DetectionParams(preprocess=False, **kw, **extra), slots=1)
    pinned = torch.from_numpy(frame).pin_memory()
    for _ in range(5):
        res = det.run(pinned)
    lat, stages = [], []
    for _ in range(30):
        t0 = time.perf_counter()
        res = det.run(pinned)
        lat.append((time.perf_counter() - t0) * 1e3)
        stages.append([res.timings_ms[k] for k in ("convolve_ms", "extrema_ms", "prune_ms")])
    st = np.median(np.array(stages), axis=0)
    H, W = frame.shape
    L = len(det.ladder.sigmas)
    taps = int(sum(2 * int(r) + 1 for r in det.bank.radii))
    flops = 2.0 * H * W * 2 * taps + 2.0 * H * W * (L - 1)
    nbytes = 4.0 * H * W * (4 * (L - 1) + 3)
    print(json.dumps({
        "config": name, "shape": [H, W], "levels": L, "taps": taps,
        "blobs": len(res.blobs), **res.stats,
        "latency_ms_median": float(np.median(lat)), "latency_ms_p90": float(np.percentile(lat, 90)),
        "convolve_ms": float(st[0]), "extrema_ms": float(st[1]), "prune_ms": float(st[2]),
        "conv_tflops_useful": flops / (st[0] * 1e-3) / 1e12,
        "frame_hbm_gbs_algorithmic": nbytes / (float(st.sum()) * 1e-3) / 1e9,
    }), flush=True)
    det.close()
