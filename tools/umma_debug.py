"""Compare the tensor-core (tcgen05) convolution passes with the FP32 sliding-window passes.

    python tools/umma_debug.py [C1|C2|C4|C5|small] [--time]

For each engine (DOGBLOB_CONV=fma / umma) the levels of one frame are computed through the stage
API and compared with a float64 separable correlation (scipy, reflect boundary); then the full
detector runs with both and the blob lists are compared.  Test tooling only.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

os.environ.setdefault("DOGBLOB_STREAMED_UPLOAD", "0")   # the gated row pass is FP32 only

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2010_08486_b200 as P  # noqa: E402
from paper_2010_08486_b200 import synth  # noqa: E402
from paper_2010_08486_b200.scale_space import gaussian_taps  # noqa: E402


def truth_levels(img, bank):
    from scipy import ndimage
    out = []
    x = np.asarray(img, dtype=np.float64)
    for s, r in zip(bank.ladder.sigmas, bank.radii):
        w = gaussian_taps(float(s), int(r))
        t = ndimage.correlate1d(x, w, axis=0, mode="reflect")
        out.append(ndimage.correlate1d(t, w, axis=1, mode="reflect"))
    return np.stack(out)


def main():
    name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "C1"
    do_time = "--time" in sys.argv
    if name == "small":
        rng = np.random.default_rng(5)
        img = rng.random((200, 150)).astype(np.float32)
        kw = dict(min_sigma=1.0, max_sigma=4.0, n_bin=3)
    else:
        img = synth.config_frame(name)
        kw = synth.config_params(name)
    kw = dict(kw, preprocess=False)
    params = P.DetectionParams(**kw)
    ladder = P.build_ladder(params.min_sigma, params.max_sigma, params.n_bin)
    bank = P.build_kernel_bank(ladder, params.truncate)
    print(f"{name}: image {img.shape}, {len(ladder.sigmas)} levels, radii {int(bank.radii[0])}..{int(bank.radii[-1])}",
          flush=True)
    t0 = time.time()
    truth = truth_levels(img, bank)
    print(f"float64 truth in {time.time() - t0:.1f} s", flush=True)

    results = {}
    for eng in ("fma", "umma"):
        os.environ["DOGBLOB_CONV"] = eng
        lev = P.convolve_bank(img, bank, "cuda").levels
        err = np.abs(lev - truth).reshape(len(lev), -1).max(axis=1)
        bias = (lev - truth).reshape(len(lev), -1).mean(axis=1)
        print(f"[{eng}] levels: max |err| = {err.max():.3e} (level {int(err.argmax())}); "
              f"per level: {np.array2string(err[::max(1, len(err) // 8)], precision=2)}", flush=True)
        print(f"[{eng}] mean signed err per level (bias): "
              f"{np.array2string(bias[::max(1, len(bias) // 8)], precision=2)}", flush=True)
        dog = P.fused_dog(img, bank).slices
        dtruth = (truth[:-1] - truth[1:]) * np.asarray(ladder.sigmas[:-1], dtype=np.float64)[:, None, None]
        derr = (np.abs(dog - dtruth).reshape(len(dog), -1).max(axis=1) / np.asarray(ladder.sigmas[:-1]))
        print(f"[{eng}] fused DoG: max |err| / sigma = {derr.max():.3e} (slice {int(derr.argmax())})", flush=True)
        det = P.Detector(params)
        res = det.run(img)
        results[eng] = res
        print(f"[{eng}] detect: {len(res.blobs)} blobs, timings {res.timings_ms}", flush=True)
        if do_time:
            import torch
            for _ in range(3):
                det.run(img)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            n = 20
            for _ in range(n):
                det.run(img)
            torch.cuda.synchronize()
            print(f"[{eng}] Detector.run: {(time.perf_counter() - t0) / n * 1e3:.3f} ms per frame; "
                  f"last timings {det.run(img).timings_ms}", flush=True)
        det.close()
    a = results["fma"].blobs.yxs()
    b = results["umma"].blobs.yxs()
    sa = {tuple(r) for r in a.tolist()}
    sb = {tuple(r) for r in b.tolist()}
    print(f"blob sets: fma {len(sa)}, umma {len(sb)}, common {len(sa & sb)}, "
          f"only fma {sorted(sa - sb)[:5]}, only umma {sorted(sb - sa)[:5]}")


if __name__ == "__main__":
    main()
