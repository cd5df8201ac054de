#!/usr/bin/env python
"""Generate tests/golden/* by running the REAL reference in the build container.

    python tools/make_golden.py [--only small,C1,...] [--skip C4,C5]

The reference (`/root/reference/pkg/src/dogblob`, pure Python) is imported
read-only; it does not exist on the GPU box, so its outputs are committed as
small fixtures and everything in tests/ compares against those.  Nothing here
is imported by the product package.

Fixture formats (npz):
  blobs arrays  : bx, by (int64), bsigma, bradius, bresponse (float64), bedge (bool)
  suffix _cand  : before pruning, suffix _kept: after pruning
  prefix t0_    : reference fft backend, float32 (production default, tier T0)
  prefix t1_    : reference fft backend, float64 (tie-breaking truth, tier T1)
"""

from __future__ import annotations

import argparse
import hashlib
import json
import shutil
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF_SRC = Path("/root/reference/pkg/src")
GOLD = ROOT / "tests" / "golden"
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(ROOT))

import dogblob  # noqa: E402  (the reference)
from dogblob.detector import DoGStack  # noqa: E402

from paper_2010_08486_b200 import synth  # noqa: E402


def blob_arrays(blobset, prefix):
    bl = blobset.blobs if hasattr(blobset, "blobs") else blobset
    return {
        prefix + "bx": np.array([b.x for b in bl], dtype=np.int64),
        prefix + "by": np.array([b.y for b in bl], dtype=np.int64),
        prefix + "bsigma": np.array([b.sigma for b in bl], dtype=np.float64),
        prefix + "bradius": np.array([b.radius for b in bl], dtype=np.float64),
        prefix + "bresponse": np.array([b.response for b in bl], dtype=np.float64),
        prefix + "bedge": np.array([b.at_scale_boundary for b in bl], dtype=bool),
    }


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_frame(name, index=None):
    if name == "C3":
        w, h, n, rr, _ = synth.CONFIGS["C2"]
        s1, s2 = 1000 + index, 2000 + index
    else:
        w, h, n, rr, _ = synth.CONFIGS[name]
        s1, s2 = synth._CONFIG_SEEDS[name]
    return dogblob.add_noise(dogblob.render_scene(w, h, n, rr, seed=s1, allow_overlap=True),
                             seed=s2).image


def run_tiers(img, params_kw, tiers=("t0", "t1")):
    out = {}
    base = dict(preprocess=False, backend="fft")
    base.update(params_kw)
    for tier in tiers:
        dtype = np.float32 if tier == "t0" else np.float64
        det = dogblob.Detector(dogblob.DetectionParams(**{**base, "prune": False}))
        t0 = time.perf_counter()
        res = det.run(img, dtype=dtype)
        cand = res.blobs
        t1 = time.perf_counter()
        kept = dogblob.prune_overlaps(cand, base.get("overlap", 0.5))
        t2 = time.perf_counter()
        hist = dogblob.histogram(kept, det.ladder)
        out.update(blob_arrays(cand, f"{tier}_cand_"))
        out.update(blob_arrays(kept, f"{tier}_kept_"))
        out[f"{tier}_hist_counts"] = hist.counts
        out[f"{tier}_hist_volumes"] = hist.volume_weights
        out[f"{tier}_hist_centers"] = hist.bin_centers
        out[f"{tier}_ms"] = np.array([res.timings_ms["convolve_ms"], res.timings_ms["extrema_ms"],
                                      (t2 - t1) * 1e3])
        print(f"    {tier}: {len(cand)} candidates -> {len(kept)} kept "
              f"({t1 - t0:.1f}s detect, {t2 - t1:.1f}s prune)", flush=True)
    return out


def gen_frames():
    """sha256 of every generated frame: pins paper_2010_08486_b200.synth to the reference."""
    doc = {}
    for name in ("C1", "C2", "C5"):
        ref = ref_frame(name)
        mine = synth.config_frame(name)
        assert np.array_equal(ref, mine), name
        doc[name] = {"sha256": sha(ref), "shape": list(ref.shape), "sum": float(ref.sum(dtype=np.float64))}
    for f in range(4):
        ref = ref_frame("C3", f)
        assert np.array_equal(ref, synth.config_frame("C3", f)), f
        doc[f"C3_{f}"] = {"sha256": sha(ref), "shape": list(ref.shape), "sum": float(ref.sum(dtype=np.float64))}
    ref = ref_frame("C4")
    assert np.array_equal(ref, synth.config_frame("C4"))
    doc["C4"] = {"sha256": sha(ref), "shape": list(ref.shape), "sum": float(ref.sum(dtype=np.float64))}
    d = dogblob.render_disk(128, 96, 64.25, 40.5, 10.0)
    assert np.array_equal(d, synth.flat_disk(128, 96, 64.25, 40.5, 10.0))
    doc["disk_128x96"] = {"sha256": sha(d), "shape": list(d.shape), "sum": float(d.sum(dtype=np.float64))}
    sc = dogblob.render_scene(200, 160, 10, (4.0, 12.0), seed=7)  # no-overlap placement path
    mine = synth.droplet_scene(200, 160, 10, (4.0, 12.0), seed=7)
    assert np.array_equal(sc.image, mine.image)
    doc["scene_nooverlap_200x160"] = {"sha256": sha(sc.image), "shape": list(sc.image.shape),
                                      "sum": float(sc.image.sum(dtype=np.float64))}
    (GOLD / "frames.json").write_text(json.dumps(doc, indent=1) + "\n")
    print("frames.json written (synth is bit-identical to the reference)")


def gen_small():
    """Per-stage arrays on small inputs: levels, DoG, masks, blobs."""
    out = {}
    # (a) random 48x64 image, ladder (1, 4, 3): levels / DoG in both precisions, both backends
    rng = np.random.default_rng(21)
    img = rng.random((48, 64)).astype(np.float32)
    ladder = dogblob.build_ladder(1.0, 4.0, 3)
    bank = dogblob.build_kernel_bank(ladder)
    out["a_img"] = img
    out["a_sigmas"] = ladder.sigmas
    out["a_radii"] = bank.radii
    for backend in ("fft", "direct"):
        for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
            st = dogblob.convolve_bank(img, bank, backend, dtype=dt)
            out[f"a_levels_{backend}_{tag}"] = st.levels
            if backend == "fft":
                out[f"a_dog_{tag}"] = dogblob.dog_stack(st, ladder).slices
    cand = dogblob.find_extrema(dogblob.dog_stack(dogblob.convolve_bank(img, bank, "fft"), ladder),
                                threshold=0.02)
    out.update(blob_arrays(cand, "a_cand_"))
    # (b) kernel wider than the image (tests/test_convolve.py:70-83)
    rng = np.random.default_rng(25)
    imgb = rng.random((32, 32))
    ladder_b = dogblob.build_ladder(5.0, 10.0, 1)
    bank_b = dogblob.build_kernel_bank(ladder_b)
    out["b_img"] = imgb
    out["b_sigmas"] = ladder_b.sigmas
    out["b_radii"] = bank_b.radii
    out["b_levels_fft_f64"] = dogblob.convolve_bank(imgb, bank_b, "fft", dtype=np.float64).levels
    out["b_levels_fft_f32"] = dogblob.convolve_bank(imgb.astype(np.float32), bank_b, "fft").levels
    # (c) ragged tiny shapes incl. 1-pixel axes
    for tag, shape in (("c1", (1, 37)), ("c2", (29, 1)), ("c3", (5, 3)), ("c4", (1, 1))):
        rng = np.random.default_rng(100 + shape[0] * 7 + shape[1])
        im = rng.random(shape).astype(np.float32)
        lad = dogblob.build_ladder(0.8, 2.4, 2)
        bk = dogblob.build_kernel_bank(lad)
        out[f"{tag}_img"] = im
        out[f"{tag}_sigmas"] = lad.sigmas
        out[f"{tag}_radii"] = bk.radii
        out[f"{tag}_levels_fft_f64"] = dogblob.convolve_bank(im, bk, "fft", dtype=np.float64).levels
    # (d) extrema on hand-made stacks: random (tests/test_detector.py:167-180), plateau, corner
    rng = np.random.default_rng(43)
    sl = rng.random((3, 24, 31)).astype(np.float32)
    out["d_slices"] = sl
    cand = dogblob.find_extrema(DoGStack(slices=sl, sigmas=np.array([1.0, 2.0, 3.0])), threshold=0.2)
    out.update(blob_arrays(cand, "d_cand_"))
    pl = np.zeros((2, 21, 21), dtype=np.float32)
    pl[0, 9:12, 8:14] = 0.5          # 3x6 plateau  (tests/test_detector.py:126-134)
    pl[1, 2:4, 15:20] = 0.75         # 2x5 plateau -> centroid (2.5, 17) half-even rounding
    pl[1, 15, 3] = 0.75
    pl[1, 16, 4] = 0.75              # diagonal pair (8-connectivity)
    pl[0, 0, 0] = 1.0                # corner voxel
    out["e_slices"] = pl
    cand = dogblob.find_extrema(DoGStack(slices=pl, sigmas=np.array([2.0, 3.0])), threshold=0.1)
    out.update(blob_arrays(cand, "e_cand_"))
    for n in (1, 5):                 # other neighbourhood sizes
        cand = dogblob.find_extrema(DoGStack(slices=sl, sigmas=np.array([1.0, 2.0, 3.0])),
                                    threshold=0.2, neighborhood=n)
        out.update(blob_arrays(cand, f"d_n{n}_cand_"))
    np.savez_compressed(GOLD / "small_stages.npz", **out)
    print("small_stages.npz written")


def gen_prune():
    """prune_overlaps / histogram on synthetic blob lists (tests/test_detector.py:254-269 style)."""
    out = {}
    params = dogblob.DetectionParams()
    case = 0
    for seed, n, span, thr in ((47, 15, 60, 0.5), (48, 60, 80, 0.5), (49, 200, 160, 0.3),
                               (50, 400, 200, 0.1), (51, 120, 60, 0.0), (52, 50, 40, 1.0),
                               (53, 600, 300, 0.5)):
        rng = np.random.default_rng(seed)
        blobs = []
        for _ in range(n):
            x = int(rng.integers(0, span))
            y = int(rng.integers(0, span))
            r = float(rng.uniform(2, 9))
            resp = float(np.float32(rng.uniform(0.1, 1.0)))
            blobs.append(dogblob.Blob(x=x, y=y, sigma=r / np.sqrt(2.0), radius=r, response=resp,
                                      at_scale_boundary=bool(rng.integers(0, 2))))
        bs = dogblob.BlobSet(blobs=tuple(blobs), source_shape=(span, span), params=params)
        t0 = time.perf_counter()
        kept = dogblob.prune_overlaps(bs, thr)
        print(f"    prune case {case}: n={n} thr={thr} -> {len(kept)} ({time.perf_counter() - t0:.1f}s)",
              flush=True)
        ladder = dogblob.build_ladder(1.0, 8.0, 10)
        hist = dogblob.histogram(kept, ladder)
        out.update(blob_arrays(bs, f"p{case}_in_"))
        out.update(blob_arrays(kept, f"p{case}_out_"))
        out[f"p{case}_thr"] = np.array(thr)
        out[f"p{case}_hist_counts"] = hist.counts
        out[f"p{case}_hist_volumes"] = hist.volume_weights
        case += 1
    out["n_cases"] = np.array(case)
    np.savez_compressed(GOLD / "prune_cases.npz", **out)
    print("prune_cases.npz written")


def gen_scene256():
    """tests/test_detector.py:328-337 scene, with and without the default preprocessing."""
    scene = dogblob.add_noise(dogblob.render_scene(256, 256, 12, (4.0, 12.0), seed=5), seed=6)
    mine = synth.sensor_noise(synth.droplet_scene(256, 256, 12, (4.0, 12.0), seed=5), seed=6)
    assert np.array_equal(scene.image, mine.image)
    kw = dict(min_sigma=2.5, max_sigma=9.0, n_bin=10)
    out = {"frame_sha": np.array(sha(scene.image))}
    out.update(run_tiers(scene.image, kw))
    res = dogblob.Detector(dogblob.DetectionParams(**kw)).run(scene.image)  # preprocess=True default
    out.update(blob_arrays(res.blobs, "pre_kept_"))
    out["pre_image"] = dogblob.preprocess(scene.image)
    np.savez_compressed(GOLD / "scene256.npz", **out)
    print("scene256.npz written")


def gen_config(name):
    img = ref_frame(name)
    kw = synth.config_params(name)
    print(f"  {name}: {img.shape} {kw}", flush=True)
    out = {"frame_sha": np.array(sha(img))}
    tiers = ("t0", "t1")
    out.update(run_tiers(img, kw, tiers))
    if name == "C5":
        # the merge-heavy variant: prune the T0 candidates at overlap 0.1
        det = dogblob.Detector(dogblob.DetectionParams(preprocess=False, prune=False, **kw))
        # (the reference's dense N x N matrix per merge makes all ~10k candidates
        # impractical at 0.1, so the strongest 2000 are used)
        cand = det.run(img).blobs
        top = dogblob.BlobSet(blobs=cand.blobs[:2000], source_shape=cand.source_shape,
                              params=cand.params)
        t0 = time.perf_counter()
        kept = dogblob.prune_overlaps(top, 0.1)
        print(f"    overlap=0.1 top-2000: {len(top)} -> {len(kept)} ({time.perf_counter() - t0:.1f}s)",
              flush=True)
        out.update(blob_arrays(kept, "t0_top2000_kept01_"))
    np.savez_compressed(GOLD / f"config_{name}.npz", **out)
    print(f"config_{name}.npz written")


def gen_c3():
    out = {}
    kw = synth.config_params("C3")
    for f in range(4):
        img = ref_frame("C3", f)
        r = run_tiers(img, kw, ("t0",))
        for k, v in r.items():
            out[f"f{f}_{k}"] = v
        out[f"f{f}_frame_sha"] = np.array(sha(img))
    np.savez_compressed(GOLD / "config_C3.npz", **out)
    print("config_C3.npz written")


def gen_demo03():
    """The reference's own committed golden vector (pkg/demos/output/03_*)."""
    src = Path("/root/reference/pkg/demos/output")
    shutil.copyfile(src / "03_blobs.json", GOLD / "ref_demo03_blobs.json")
    shutil.copyfile(src / "03_histogram.csv", GOLD / "ref_demo03_histogram.csv")
    print("ref_demo03_* copied")


JOBS = {
    "frames": gen_frames,
    "small": gen_small,
    "prune": gen_prune,
    "scene256": gen_scene256,
    "demo03": gen_demo03,
    "C1": lambda: gen_config("C1"),
    "C2": lambda: gen_config("C2"),
    "C3": gen_c3,
    "C4": lambda: gen_config("C4"),
    "C5": lambda: gen_config("C5"),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--skip", default="")
    args = ap.parse_args()
    only = [s for s in args.only.split(",") if s]
    skip = [s for s in args.skip.split(",") if s]
    GOLD.mkdir(parents=True, exist_ok=True)
    for name, fn in JOBS.items():
        if (only and name not in only) or name in skip:
            continue
        t0 = time.perf_counter()
        print(f"[{name}]", flush=True)
        fn()
        print(f"[{name}] done in {time.perf_counter() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
