#!/usr/bin/env python
"""Where the host-side time of Detector.run goes (launch call, wait, decode, timings, histogram)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import paper_2010_08486_b200 as P  # noqa: E402
from paper_2010_08486_b200 import synth  # noqa: E402

for name in (sys.argv[1:] or ["C1", "C2"]):
    det = P.Detector(P.DetectionParams(preprocess=False, **synth.config_params(name)), slots=1)
    frame = torch.from_numpy(synth.config_frame(name)).pin_memory()
    for _ in range(20):
        det.run(frame)
    eng = det.plan_for(tuple(frame.shape))
    acc = np.zeros(6)
    n = 200
    for _ in range(n):
        t0 = time.perf_counter()
        slot = eng.free.get()
        t1 = time.perf_counter()
        slot.launch(frame, det.params, True)
        t2 = time.perf_counter()
        hdr, recs = slot.collect()
        t3 = time.perf_counter()
        tm = slot.stage_times_ms(hdr)
        t4 = time.perf_counter()
        eng.free.put(slot)
        res = det._finish(slot, hdr, recs, tuple(frame.shape), tm)
        t5 = time.perf_counter()
        acc += [t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t5 - t0]
    acc *= 1e6 / n
    dev = sum(tm.values()) * 1e3
    print(f"{name}: slot {acc[0]:.1f} us | launch call {acc[1]:.1f} | wait+decode {acc[2]:.1f} | stage times {acc[3]:.1f} "
          f"| finish (BlobSet, histogram) {acc[4]:.1f} | total {acc[5]:.1f} us | device stages {dev:.1f} us")
    det.close()
