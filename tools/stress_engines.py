#!/usr/bin/env python
"""Randomised cross-check of the two convolution engines and of the detection path that skips stores:
random frame shapes (ragged, odd widths), ladders and thresholds; the tensor-core engine's fused DoG
slices against the FP32 engine's (within 2e-6 sigma) and the detected blob lists of both engines on
frame SEQUENCES through one detector (stale slice memory must never show).  Test tooling only.

    python tools/stress_engines.py [n_cases] [seed] [large]        # large: frames up to 2600 px, sigma up to 60
"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2010_08486_b200 as P  # noqa: E402
from paper_2010_08486_b200 import synth  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
large = len(sys.argv) > 3 and sys.argv[3] == "large"
worst, n_tensor, n_list_diff, failures = 0.0, 0, 0, 0
for case in range(n_cases):
    H, W = (int(rng.integers(600, 2600)), int(rng.integers(600, 2600))) if large else \
           (int(rng.integers(140, 1300)), int(rng.integers(140, 1300)))
    if rng.random() < 0.3:
        W = W // 8 * 8
    if rng.random() < 0.2:
        H, W = H // 128 * 128 + 128, W // 128 * 128 + 128
    lo = float(rng.choice([1.0, 1.5, 2.0, 3.0]))
    hi = float(min(lo + rng.uniform(4, 58 if large else 28), min(H, W) / 6.0))
    n_bin = int(rng.integers(3, 40))
    kw = dict(min_sigma=lo, max_sigma=max(hi, lo + 1.0), n_bin=n_bin)
    thr = float(rng.choice([0.02, 0.05, 0.1, 0.2]))
    frames = [synth.sensor_noise(synth.droplet_scene(W, H, int(rng.integers(3, 60)), (2.0, float(min(H, W)) / 12.0),
                                                     seed=int(rng.integers(1 << 30)), allow_overlap=True),
                                 seed=int(rng.integers(1 << 30))).image for _ in range(3)]
    frames.append(np.zeros((H, W), np.float32))
    bank = P.build_kernel_bank(P.build_ladder(kw["min_sigma"], kw["max_sigma"], kw["n_bin"]), 5.0)
    out = {}
    for eng in ("fma", "umma"):
        os.environ["DOGBLOB_CONV"] = eng
        det = P.Detector(P.DetectionParams(preprocess=False, threshold=thr, **kw), slots=1)
        used = det.plan_for((H, W)).plan.conv_engine
        seq = [0, 1, 3, 0, 2, 1, 0]
        dog = P.fused_dog(frames[0], bank)
        # the stage functions on the fully stored stack (no hit flags, nothing skipped) must give the
        # detector's list for the same frame exactly: same DoG bits, same extrema, same pruning
        staged = P.prune_overlaps(P.find_extrema(dog, thr, 3, source_shape=(W, H)), 0.5)
        out[eng] = (used, dog.slices,
                    [[(b.x, b.y, b.sigma) for b in det.run(frames[i]).blobs.blobs] for i in seq],
                    [(b.x, b.y, b.sigma) for b in staged.blobs])
        det.close()
    if out["umma"][0] != 2:
        print(f"case {case}: {H}x{W} sigma {lo}..{kw['max_sigma']:.1f} n_bin {n_bin}: tensor engine not available, skipped")
        continue
    n_tensor += 1
    sig = np.asarray(bank.ladder.sigmas[:-1], dtype=np.float64)[:, None, None]
    err = float((np.abs(out["fma"][1].astype(np.float64) - out["umma"][1]) / sig).max())
    worst = max(worst, err)
    same_seq = out["umma"][2][0] == out["umma"][2][3] == out["umma"][2][6] and out["umma"][2][1] == out["umma"][2][5]
    diff = sum(len(set(a) ^ set(b)) for a, b in zip(out["fma"][2], out["umma"][2]))
    n_list_diff += diff
    print(f"case {case}: {H}x{W} sigma {lo}..{kw['max_sigma']:.1f} n_bin {n_bin} thr {thr}: max |dDoG|/sigma = {err:.2e}, "
          f"blobs {len(out['umma'][2][0])}, engine list differences {diff}, repeat-stable {same_seq}", flush=True)
    tol = 2e-6 if int(bank.radii.max()) <= 150 else 3e-6      # two float32 results: rounding grows with the taps
    if err >= tol:
        failures += 1
        d = np.abs(out["fma"][1].astype(np.float64) - out["umma"][1]) / sig
        per = d.reshape(d.shape[0], -1).max(axis=1)
        bad = np.nonzero(per >= tol)[0]
        print("   DoG slices differ: slices", bad.tolist(), "radii", [int(bank.radii[i]) for i in bad], [int(bank.radii[i + 1]) for i in bad])
        for i in bad[:4]:
            ys, xs = np.nonzero(d[i] >= tol)
            print(f"   slice {i}: err {per[i]:.2e}, {ys.size} px, rows {ys.min()}..{ys.max()}, cols {xs.min()}..{xs.max()}")
        continue
    for eng in ("fma", "umma"):
        assert out[eng][3] == out[eng][2][0], f"{eng}: detector and stage functions disagree on the same stack"
    assert same_seq, "a frame's result depends on what the slot saw before"
    assert out["umma"][2][2] == [], "blank frame produced blobs"
print(f"{failures} FAILED cases") if failures else None
print(f"{n_tensor} tensor-engine cases, worst |dDoG|/sigma = {worst:.2e}, {n_list_diff} near-tie list differences between the engines")
sys.exit(1 if failures else 0)
