"""Synthetic PLIF-like droplet frames (host side, numpy) for benches and tests.

The frames are bit-identical to the reference generator for the same seeds
(`pkg/src/dogblob/synth.py:89-162`): bright sphere-cap droplets
v(d) = sqrt(1 - (d/r)^2) on black, rim antialiased by 4x4 sub-pixel coverage,
then Poisson(255 v)/255 shot noise + N(0, 0.01) read noise, clamped at zero.
Bit-identity matters because blob-set parity is judged on identical float32
inputs; it is pinned by sha256 fixtures in `tests/golden/frames.json`
(generated from the reference by `tools/make_golden.py`).

This is an input generator, not part of the detector hot path.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np

SUBSAMPLES = 4          # per axis, synth.py:27
MAX_TRIES = 2000        # per droplet when overlap is disallowed, synth.py:28


class Droplet(NamedTuple):
    x: float
    y: float
    r: float


class Frame(NamedTuple):
    image: np.ndarray            # float32 (H, W)
    truths: tuple                # Droplet, ...
    seed: int


def _sub_offsets() -> np.ndarray:
    return (np.arange(SUBSAMPLES) + 0.5) / SUBSAMPLES - 0.5


def _footprint(c: float, r: float, n: int) -> tuple[int, int]:
    lo = max(int(np.floor(c - r - 1)), 0)
    hi = min(int(np.ceil(c + r + 1)) + 1, n)
    return lo, hi


def _coverage_grid(lo: int, hi: int, c: float) -> np.ndarray:
    """Squared sub-pixel distances to c along one axis, length (hi-lo)*SUBSAMPLES."""
    pos = (np.arange(lo, hi)[:, None] + _sub_offsets()[None, :]).reshape(-1)
    return (pos - c) ** 2


def _box_average(fine: np.ndarray, ny: int, nx: int) -> np.ndarray:
    return fine.reshape(ny, SUBSAMPLES, nx, SUBSAMPLES).mean(axis=(1, 3))


def paint_droplet(img: np.ndarray, d: Droplet, peak: float = 1.0) -> None:
    h, w = img.shape
    y0, y1 = _footprint(d.y, d.r, h)
    x0, x1 = _footprint(d.x, d.r, w)
    if y0 >= y1 or x0 >= x1:
        return
    dist2 = _coverage_grid(y0, y1, d.y)[:, None] + _coverage_grid(x0, x1, d.x)[None, :]
    shade = peak * np.sqrt(np.clip(1.0 - dist2 / (d.r * d.r), 0.0, None))
    tile = _box_average(shade, y1 - y0, x1 - x0).astype(img.dtype)
    view = img[y0:y1, x0:x1]
    np.maximum(view, tile, out=view)


def flat_disk(width: int, height: int, cx: float, cy: float, r: float) -> np.ndarray:
    """Unit-intensity antialiased disk (reference render_disk, synth.py:70-86)."""
    img = np.zeros((height, width), dtype=np.float32)
    y0, y1 = _footprint(cy, r, height)
    x0, x1 = _footprint(cx, r, width)
    off = _sub_offsets()
    ys = (np.arange(y0, y1)[:, None] + off[None, :]).reshape(-1)
    xs = (np.arange(x0, x1)[:, None] + off[None, :]).reshape(-1)
    dist2 = (ys - cy)[:, None] ** 2 + (xs - cx)[None, :] ** 2
    inside = (dist2 <= r * r).astype(np.float32)
    img[y0:y1, x0:x1] = _box_average(inside, y1 - y0, x1 - x0)
    return img


def droplet_scene(width: int, height: int, count: int, r_range, seed: int,
                  allow_overlap: bool = False, peak: float = 1.0) -> Frame:
    """Noise-free scene; consumes the default_rng(seed) stream in the order
    r, cx, cy per placement attempt (synth.py:111-126)."""
    r_lo, r_hi = r_range
    if r_lo <= 0 or r_hi < r_lo:
        raise ValueError(f"bad radius range {r_range}")
    if count < 0:
        raise ValueError("count must be >= 0")
    if min(width, height) < 2 * r_hi + 3:
        raise ValueError(f"radius {r_hi} cannot fit inside {width}x{height}")
    rng = np.random.default_rng(seed)
    placed: list[Droplet] = []
    for n in range(count):
        ok = False
        for _ in range(MAX_TRIES):
            r = float(rng.uniform(r_lo, r_hi))
            cx = float(rng.uniform(r + 1, width - 1 - r - 1))
            cy = float(rng.uniform(r + 1, height - 1 - r - 1))
            if allow_overlap or all(np.hypot(cx - t.x, cy - t.y) > r + t.r + 2 for t in placed):
                placed.append(Droplet(cx, cy, r))
                ok = True
                break
        if not ok:
            raise RuntimeError(f"could not place droplet {n + 1}/{count} without overlap")
    img = np.zeros((height, width), dtype=np.float32)
    for d in placed:
        paint_droplet(img, d, peak)
    return Frame(img, tuple(placed), seed)


def sensor_noise(frame: Frame, photons: float = 255.0, read_sigma: float = 0.01,
                 seed: int = 0) -> Frame:
    """Shot noise then read noise, clamped at zero (synth.py:136-162)."""
    if photons <= 0:
        raise ValueError("photons must be > 0")
    if read_sigma < 0:
        raise ValueError("read_sigma must be >= 0")
    rng = np.random.default_rng(seed)
    lam = np.clip(frame.image.astype(np.float64), 0, None) * photons
    out = rng.poisson(lam).astype(np.float64) / photons
    if read_sigma > 0:
        out += rng.normal(0.0, read_sigma, size=out.shape)
    return Frame(np.clip(out, 0.0, None).astype(np.float32), frame.truths, frame.seed)


# ---- the BASELINE.json configurations -------------------------

CONFIGS = {
    # name: (width, height, droplets, r_range, detector kwargs)
    "C1": (512, 512, 40, (3.0, 15.0), dict(min_sigma=1.0, max_sigma=10.0, n_bin=18)),
    "C2": (1024, 1024, 160, (3.0, 40.0), dict(min_sigma=1.0, max_sigma=30.0, n_bin=58)),
    "C4": (2048, 2048, 300, (3.0, 80.0), dict(min_sigma=1.0, max_sigma=60.0, n_bin=59)),
    "C5": (1024, 1024, 13500, (2.0, 5.0), dict(min_sigma=1.0, max_sigma=6.0, n_bin=10)),
}
_CONFIG_SEEDS = {"C1": (1, 2), "C2": (1, 2), "C4": (1, 2), "C5": (5, 6)}


def config_frame(name: str, index: int | None = None) -> np.ndarray:
    """The float32 frame of configuration `name`; `index` selects frame f of the
    C3 batch (scene seed 1000+f, noise seed 2000+f, C2 geometry)."""
    if name == "C3":
        if index is None:
            raise ValueError("C3 needs a frame index")
        w, h, n, rr, _ = CONFIGS["C2"]
        s_scene, s_noise = 1000 + index, 2000 + index
    else:
        w, h, n, rr, _ = CONFIGS[name]
        s_scene, s_noise = _CONFIG_SEEDS[name]
    return sensor_noise(droplet_scene(w, h, n, rr, s_scene, allow_overlap=True), seed=s_noise).image


def config_params(name: str) -> dict:
    return dict(CONFIGS["C2" if name == "C3" else name][4])


def write_truth_csv(path, frame: Frame) -> None:
    """synth.py:165-171 layout: `# seed=`, header `x,y,r`, one repr() row per droplet."""
    with open(path, "w") as f:
        f.write(f"# seed={frame.seed}\nx,y,r\n")
        for d in frame.truths:
            f.write(f"{float(d.x)!r},{float(d.y)!r},{float(d.r)!r}\n")


def read_truth_csv(path) -> tuple:
    """synth.py:174-182"""
    out = []
    with open(path) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#") or line.startswith("x,"):
                continue
            x, y, r = (float(v) for v in line.split(","))
            out.append(Droplet(x=x, y=y, r=r))
    return tuple(out)


def device_frames(n_frames: int, width: int, height: int, count: int, r_range, seed: int,
                  photons: float = 255.0, read_sigma: float = 0.01, device: int | None = None):
    """PLIF-like frames generated ON the device for throughput / precision-recall sweeps over
    thousands of frames: same scene model as droplet_scene(allow_overlap=True) +
    sensor_noise, but counter-based random streams - PERF ONLY, never bit-identical to the
    reference's numpy streams; parity is always judged on host frames.

    Returns (frames, truths): a float32 CUDA tensor [n_frames][height][pitch] (pitch = width rounded
    up to 128, the detector's device layout: frames[f] can go straight into dogblob_detect) and a
    float64 array [n_frames][count][3] of (x, y, r)."""
    import torch
    from . import _lib
    lib = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    pitch = (int(width) + 127) // 128 * 128
    frames = torch.empty((int(n_frames), int(height), pitch), dtype=torch.float32, device=dev)
    truth = torch.zeros((int(n_frames), max(int(count), 1), 3), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev)
        _lib.check(lib.dogblob_synth_frames(int(n_frames), int(height), int(width), pitch, int(count),
                                            float(r_range[0]), float(r_range[1]), int(seed) & (2**64 - 1),
                                            float(photons), float(read_sigma), frames.data_ptr(),
                                            truth.data_ptr(), st.cuda_stream))
    return frames, truth[:, :int(count)].cpu().numpy()
