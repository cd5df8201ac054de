"""Pre-processing used before detection, on the GPU (reference `images.py:112-157`).

`smooth` + `contrast_stretch` = `preprocess`, with the reference's argument checks.
The numerics run in libdogblob_b200.so (`csrc/preprocess.cu`): scipy's float64
line filter restated bit for bit, then an exact radix-select for the two
nearest-rank quantiles.  Host code here only derives the filter taps and the two
ranks, exactly as scipy / the reference derive them.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib

__all__ = ["preprocess", "smooth_taps", "stretch_ranks", "PREPROCESS_TRUNCATE"]

PREPROCESS_TRUNCATE = 5.0   # images.py:148


def smooth_taps(sigma: float) -> tuple[int, np.ndarray]:
    """(radius, taps[0..radius]) of scipy.ndimage.gaussian_filter1d(sigma, truncate=5):
    radius = int(truncate * sigma + 0.5), phi = exp(-0.5 / sigma^2 * x^2) / sum (float64)."""
    if sigma < 0:
        raise ValueError(f"smoothing sigma must be >= 0, got {sigma}")
    if sigma == 0:
        return 0, np.ones(1, dtype=np.float64)
    sd = float(sigma)
    radius = int(PREPROCESS_TRUNCATE * sd + 0.5)
    x = np.arange(-radius, radius + 1)
    phi = np.exp(-0.5 / (sd * sd) * x ** 2)
    phi = phi / phi.sum()
    return radius, np.ascontiguousarray(phi[radius:], dtype=np.float64)


def stretch_ranks(n: int, saturation: float) -> tuple[int, int]:
    """0-based nearest ranks of the saturation/2 and 1 - saturation/2 quantiles (images.py:112-131)."""
    if not 0.0 <= saturation < 0.5:
        raise ValueError(f"saturation must be in [0, 0.5), got {saturation}")

    def rank(q):
        return min(max(math.ceil(q * n) - 1, 0), n - 1)

    return rank(saturation / 2.0), rank(1.0 - saturation / 2.0)


def preprocess(img, smooth_sigma: float = 1.0, saturation: float = 0.0035) -> np.ndarray:
    """Smooth, then contrast stretch to [0, 1]; float32 in, float32 out (images.py:153-157)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("backend='cuda' needs a CUDA device; there is no CPU fallback")
    arr = np.asarray(img)
    if arr.ndim != 2:
        raise ValueError(f"expected a single-channel 2-D image, got shape {arr.shape}")
    if arr.size == 0:
        raise ValueError("empty image")
    arr = np.ascontiguousarray(arr, dtype=np.float32)
    H, W = arr.shape
    radius, taps = smooth_taps(smooth_sigma)
    lo, hi = stretch_ranks(H * W, saturation)
    lib = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    src = torch.from_numpy(arr).to(dev)
    dst = torch.empty_like(src)
    scratch = torch.zeros(int(lib.dogblob_preprocess_bytes(H, W)), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream(dev)
    _lib.check(lib.dogblob_preprocess(H, W, src.data_ptr(), W, radius, _lib.ptr(taps), lo, hi,
                                      scratch.data_ptr(), dst.data_ptr(), W, st.cuda_stream))
    status = _read_status(lib, scratch, st)
    if status & 1:
        raise ValueError("image contains NaN or Inf values")
    return dst.cpu().numpy()


def _read_status(lib, scratch, stream) -> int:
    import torch
    host = torch.zeros(1, dtype=torch.int32).pin_memory()
    _lib.check(lib.dogblob_preprocess_status(scratch.data_ptr(), host.data_ptr(), stream.cuda_stream))
    stream.synchronize()
    return int(host.item()) & 0xFFFFFFFF
