#!/usr/bin/env python
"""Precision / recall and throughput sweep entirely on the device: frames are
generated on the GPU (perf-only random streams), detected as resident frames and scored by the
device matcher - thousands of frames per minute, no host image ever exists.

    python tools/sweep_pr.py --frames 512 --thresholds 0.05,0.1,0.2
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2010_08486_b200 as P  # noqa: E402
from paper_2010_08486_b200 import evaluate as ev, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=256)
ap.add_argument("--size", type=int, default=1024)
ap.add_argument("--droplets", type=int, default=160)
ap.add_argument("--thresholds", default="0.05,0.1,0.2")
ap.add_argument("--seed", type=int, default=1)
args = ap.parse_args()

t0 = time.perf_counter()
frames, truths = synth.device_frames(args.frames, args.size, args.size, args.droplets, (3.0, 40.0), args.seed)
torch.cuda.synchronize()
gen_s = time.perf_counter() - t0
truth_sets = [[synth.Droplet(*t) for t in truths[k]] for k in range(args.frames)]
for thr in (float(v) for v in args.thresholds.split(",")):
    det = P.Detector(P.DetectionParams(min_sigma=1.0, max_sigma=30.0, n_bin=58, threshold=thr, preprocess=False), slots=4)
    det.run(frames[0])
    t0 = time.perf_counter()
    blobs = [r.blobs for r in det.run_batch([frames[k] for k in range(args.frames)])]
    det_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    reps = ev.match_voc_batch(blobs, truth_sets, 0.5)
    match_s = time.perf_counter() - t0
    det.close()
    print(json.dumps({"threshold": thr, "frames": args.frames, "generate_s": round(gen_s, 3),
                      "detect_fps": round(args.frames / det_s, 1), "match_s": round(match_s, 3),
                      "precision_mean": float(np.mean([r.precision for r in reps])),
                      "recall_mean": float(np.mean([r.recall for r in reps])),
                      "blobs_per_frame": float(np.mean([len(b) for b in blobs]))}), flush=True)
