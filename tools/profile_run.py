#!/usr/bin/env python
"""Tiny driver for ncu: N frames of the bench workload through Detector.run
(the same call bench.py's latency leg times).  Usage under gpurun:

  ncu --metrics gpu__time_duration.sum --clock-control none -s 36 -c 9 --csv \
      --log-file gpurun_out/launches.csv python tools/profile_run.py --frames 5
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2010_08486_b200 as P  # noqa: E402
from paper_2010_08486_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=5)
ap.add_argument("--config", default="C2")
args = ap.parse_args()
name = args.config
det = P.Detector(P.DetectionParams(preprocess=False, **synth.config_params(name)), slots=1)
frames = [synth.config_frame("C3", i) if name == "C2" else synth.config_frame(name) for i in range(2)]
for i in range(args.frames):
    r = det.run(frames[i % 2])
torch.cuda.synchronize()
print(len(r.blobs), r.timings_ms, r.stats)
det.close()
