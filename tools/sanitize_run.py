#!/usr/bin/env python
"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / initcheck):
ragged shapes, a dense frame that takes the grid-bucketed pruning path, preprocessing."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2010_08486_b200 as P  # noqa: E402
from paper_2010_08486_b200 import synth  # noqa: E402

rng = np.random.default_rng(0)
for shape, kw in (((97, 131), dict(min_sigma=1.0, max_sigma=4.0, n_bin=6)),
                  ((256, 200), dict(min_sigma=2.0, max_sigma=9.0, n_bin=7)),
                  ((33, 300), dict(min_sigma=3.0, max_sigma=12.0, n_bin=3))):
    frame = synth.sensor_noise(synth.droplet_scene(shape[1], shape[0], 6, (2.0, 6.0), seed=3,
                                                   allow_overlap=True), seed=4).image
    for pre in (False, True):
        det = P.Detector(P.DetectionParams(preprocess=pre, **kw))
        res = det.run(frame)
        print(shape, pre, len(res.blobs), res.stats)
        det.close()
dense = synth.sensor_noise(synth.droplet_scene(384, 384, 1900, (2.0, 5.0), seed=5, allow_overlap=True), seed=6).image
det = P.Detector(P.DetectionParams(preprocess=False, min_sigma=1.0, max_sigma=6.0, n_bin=10, overlap=0.3))
res = det.run(dense)
print("dense", len(res.blobs), res.stats)
det.close()
big = synth.sensor_noise(synth.droplet_scene(700, 600, 30, (3.0, 9.0), seed=7, allow_overlap=True), seed=8).image
det = P.Detector(P.DetectionParams(preprocess=False, min_sigma=1.0, max_sigma=5.0, n_bin=4))
print("streamed upload", [len(det.run(big).blobs) for _ in range(2)])     # >= 1 MiB: row chunks + gate word
det.close()
sl = (rng.random((2, 60, 70)) * 0.05).astype(np.float32)
sl[0, 10:30, 20:50] = 0.9
print("plateau", len(P.find_extrema(P.DoGStack(sl, np.array([1.5, 2.5])), threshold=0.1)))
bank = P.build_kernel_bank(P.build_ladder(1.0, 4.0, 3))
print("levels", P.convolve_bank(rng.random((45, 67)).astype(np.float32), bank).levels.shape)
