"""CPU oracle for the DoG blob-detector hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference package's detector
path (`/root/reference/pkg/src/dogblob`).  It exists so that the CUDA path can
be checked on a GPU box where the reference itself is not present.  Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu-baseline /
`--impl reference` legs may import it; the product package
(`paper_2010_08486_b200`) never does.

Parity status: PINNED.  `tools/make_golden.py` runs the real reference in the
build container and commits its outputs under `tests/golden/`;
`tests/test_oracle.py` checks this restatement against those fixtures and
against the reference's own golden vector `pkg/demos/output/03_blobs.json`
(copied as a fixture by the same script).

Third-party arithmetic the reference delegates to (not under /root/reference,
`pkg/pyproject.toml:10-14` pins numpy>=1.24, scipy>=1.10; installed here
numpy 2.3.5 / scipy 1.18.1): `scipy.fft.rfft2/irfft2` (pocketfft) is called
here exactly as the reference calls it; `scipy.ndimage.maximum_filter`,
`label` and `center_of_mass` are restated in plain numpy below;
`scipy.ndimage.gaussian_filter` (pre-processing only) is called as-is.

Each function cites the reference lines it follows (paths relative to
`pkg/src/dogblob/`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy import fft as _sfft
from scipy import ndimage as _ndi

SQRT2 = math.sqrt(2.0)


# --------------------------------------------------------------------------
# scale-space definition
# --------------------------------------------------------------------------

def ladder_sigmas(min_sigma: float, max_sigma: float, n_bin: int) -> np.ndarray:
    """n_bin+1 arithmetic scales; same guards as scale_space.py:54-73."""
    if not min_sigma > 0:
        raise ValueError(f"min_sigma must be > 0, got {min_sigma}")
    if max_sigma < min_sigma:
        raise ValueError(f"max_sigma {max_sigma} < min_sigma {min_sigma}")
    if n_bin < 1:
        raise ValueError(f"n_bin must be >= 1, got {n_bin}")
    if max_sigma == min_sigma:
        raise ValueError("degenerate ladder: max_sigma == min_sigma")
    return np.linspace(min_sigma, max_sigma, n_bin + 1)


def tap_radii(sigmas: np.ndarray, truncate: float = 5.0) -> np.ndarray:
    """radius_i = ceil(truncate * sigma_i)  (scale_space.py:95-97)."""
    if not truncate > 0:
        raise ValueError(f"truncate must be > 0, got {truncate}")
    return np.array([math.ceil(truncate * float(s)) for s in sigmas], dtype=np.int64)


def gauss_profile(sigma: float, radius: int) -> np.ndarray:
    """Un-normalised 1-D profile exp(-x^2 / 2 sigma^2), x in [-r, r] (scale_space.py:78-79)."""
    x = np.arange(-radius, radius + 1, dtype=np.float64)
    return np.exp(-(x * x) / (2.0 * sigma * sigma))


def kernel_2d(sigma: float, radius: int) -> np.ndarray:
    """outer(g, g) / sum, float64 -- scale_space.py:76-81."""
    g = gauss_profile(sigma, radius)
    k = np.outer(g, g)
    return k / k.sum()


def kernel_1d(sigma: float, radius: int) -> np.ndarray:
    """w = g / sum(g): the exact separable factor of kernel_2d (k == w (x) w up to rounding)."""
    g = gauss_profile(sigma, radius)
    return g / g.sum()


# --------------------------------------------------------------------------
# convolution backends
# --------------------------------------------------------------------------

def _check_image(img) -> np.ndarray:
    img = np.asarray(img)
    if img.ndim != 2 or img.shape[0] < 1 or img.shape[1] < 1:
        raise ValueError(f"expected a non-empty 2-D image, got shape {img.shape}")
    return img


def fft_spectra(shape, sigmas, radii, dtype=np.float32) -> np.ndarray:
    """Real kernel spectra at the (2H, 2W) period -- convolve.py:118-146.

    The reference wrap-accumulates the zero-framed max_width kernel with
    np.add.at in row-major order; adding the zero frame is exact, so the
    trimmed kernel accumulated in the same order gives identical float64 sums.
    """
    H, W = shape
    P, Q = 2 * H, 2 * W
    out = np.empty((len(sigmas), P, Q // 2 + 1), dtype=dtype)
    for i, (s, r) in enumerate(zip(sigmas, radii)):
        r = int(r)
        k = kernel_2d(float(s), r)
        offs = np.arange(-r, r + 1)
        yy = np.broadcast_to((offs % P)[:, None], k.shape)
        xx = np.broadcast_to((offs % Q)[None, :], k.shape)
        placed = np.zeros((P, Q))
        np.add.at(placed, (yy, xx), k)
        out[i] = _sfft.rfft2(placed).real.astype(dtype)
    return out


def levels_fft(img, sigmas, radii, dtype=np.float32, spectra=None) -> np.ndarray:
    """FFT backend: half-sample symmetric extension to (2H,2W), one circular
    convolution per level, crop -- convolve.py:161-186."""
    img = _check_image(img)
    dtype = np.dtype(dtype)
    H, W = img.shape
    if spectra is None:
        spectra = fft_spectra((H, W), sigmas, radii, dtype)
    work = img.astype(dtype, copy=False)
    ext = np.empty((2 * H, 2 * W), dtype=dtype)
    ext[:H, :W] = work
    ext[H:, :W] = work[::-1, :]
    ext[:H, W:] = work[:, ::-1]
    ext[H:, W:] = work[::-1, ::-1]
    fwd = _sfft.rfft2(ext)
    levels = np.empty((len(sigmas), H, W), dtype=dtype)
    for i in range(len(sigmas)):
        full = _sfft.irfft2(fwd * spectra[i], s=(2 * H, 2 * W))
        levels[i] = full[:H, :W]
    return levels


def fold_index(idx: np.ndarray, n: int) -> np.ndarray:
    """Reflect ("symmetric", edge sample repeated) index map of period 2n (convolve.py:4,94)."""
    m = np.mod(idx, 2 * n)
    return np.where(m < n, m, 2 * n - 1 - m)


def _correlate_axis0(a: np.ndarray, w: np.ndarray) -> np.ndarray:
    """out[y] = sum_k w[k] a[fold(y + k - r)] along axis 0, in a's dtype (float64)."""
    r = (w.size - 1) // 2
    n = a.shape[0]
    out = np.zeros_like(a)
    base = np.arange(n)
    # accumulate from the outermost (smallest) taps inwards
    order = sorted(range(w.size), key=lambda k: (-abs(k - r), k))
    for k in order:
        out += w[k] * a[fold_index(base + (k - r), n)]
    return out


def levels_separable(img, sigmas, radii, dtype=np.float64) -> np.ndarray:
    """Separable float64 evaluation of the same sampled, truncated kernels with
    the same boundary rule; the tie-breaking "truth" tier."""
    img = _check_image(img).astype(np.float64)
    out = np.empty((len(sigmas),) + img.shape, dtype=dtype)
    for i, (s, r) in enumerate(zip(sigmas, radii)):
        w = kernel_1d(float(s), int(r))
        tmp = _correlate_axis0(img, w)
        out[i] = _correlate_axis0(tmp.T, w).T
    return out


def level_values_at(img, sigma: float, radius: int, ys, xs) -> np.ndarray:
    """float64 level values L_sigma[y, x] at scattered pixels, straight from the
    2-D definition (kernel_2d correlated with the reflect-extended image)."""
    img = np.asarray(img, dtype=np.float64)
    H, W = img.shape
    k = kernel_2d(float(sigma), int(radius))
    offs = np.arange(-radius, radius + 1)
    out = np.empty(len(ys), dtype=np.float64)
    for n, (y, x) in enumerate(zip(ys, xs)):
        rows = fold_index(y + offs, H)
        cols = fold_index(x + offs, W)
        out[n] = float(np.sum(k * img[np.ix_(rows, cols)]))
    return out


def scale_space(img, sigmas, radii, backend="fft", dtype=np.float32,
                stack_element_cap: int = 2 ** 28) -> np.ndarray:
    """convolve_bank guards (convolve.py:189-218) + the chosen backend."""
    img = _check_image(img)
    if backend not in ("fft", "separable"):
        raise ValueError(f"unknown backend {backend!r}")
    if img.shape[0] * img.shape[1] * len(sigmas) > stack_element_cap:
        raise ValueError(
            f"stack of {len(sigmas)} x {img.shape} exceeds element cap {stack_element_cap}")
    if backend == "fft":
        return levels_fft(img, sigmas, radii, dtype)
    return levels_separable(img, sigmas, radii, dtype)


# --------------------------------------------------------------------------
# DoG, extrema
# --------------------------------------------------------------------------

def dog_slices(levels: np.ndarray, sigmas: np.ndarray) -> np.ndarray:
    """slices[i] = sigma_i * (L_i - L_{i+1}) in the stack dtype (detector.py:117-126)."""
    if levels.shape[0] != len(sigmas):
        raise ValueError(f"stack has {levels.shape[0]} levels, ladder expects {len(sigmas)}")
    lower = np.asarray(sigmas)[:-1]
    return (levels[:-1] - levels[1:]) * lower[:, None, None].astype(levels.dtype)


def box_max(data: np.ndarray, size: int) -> np.ndarray:
    """Maximum over the size^ndim block with -inf outside the volume -- the
    ndimage.maximum_filter(mode="constant", cval=-inf) call of detector.py:165."""
    h = size // 2
    out = data
    for axis in range(data.ndim):
        pad = [(0, 0)] * data.ndim
        pad[axis] = (h, h)
        padded = np.pad(out, pad, mode="constant", constant_values=-np.inf)
        n = data.shape[axis]
        acc = None
        for d in range(size):
            sl = [slice(None)] * data.ndim
            sl[axis] = slice(d, d + n)
            piece = padded[tuple(sl)]
            acc = piece.copy() if acc is None else np.maximum(acc, piece)
        out = acc
    return out


def flagged_mask(slices: np.ndarray, threshold: float, neighborhood: int = 3) -> np.ndarray:
    """(data == boxmax) & (data > threshold)  (detector.py:162-166).

    Under numpy 2 promotion the Python-float threshold is compared in the
    array dtype, i.e. against float32(threshold) for a float32 stack.
    """
    if neighborhood < 1 or neighborhood % 2 == 0:
        raise ValueError(f"neighborhood must be odd and >= 1, got {neighborhood}")
    thr = slices.dtype.type(threshold)
    return (slices == box_max(slices, neighborhood)) & (slices > thr)


def components_8(mask2d: np.ndarray):
    """8-connected components of a 2-D boolean mask, labelled in raster order of
    their first pixel (what ndimage.label with a full 3x3 structure returns)."""
    H, W = mask2d.shape
    seen = np.zeros_like(mask2d, dtype=bool)
    comps = []
    ys, xs = np.nonzero(mask2d)
    for y0, x0 in zip(ys.tolist(), xs.tolist()):
        if seen[y0, x0]:
            continue
        seen[y0, x0] = True
        stack = [(y0, x0)]
        members = []
        while stack:
            y, x = stack.pop()
            members.append((y, x))
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    yy, xx = y + dy, x + dx
                    if 0 <= yy < H and 0 <= xx < W and mask2d[yy, xx] and not seen[yy, xx]:
                        seen[yy, xx] = True
                        stack.append((yy, xx))
        members.sort()
        comps.append(members)
    return comps


def coalesce_slice(mask2d: np.ndarray, values: np.ndarray):
    """One (x, y, response) per component at the half-even rounded centroid;
    response is the value at the raster-first member (detector.py:129-146)."""
    out = []
    for members in components_8(mask2d):
        n = float(len(members))
        cy = float(sum(m[0] for m in members)) / n
        cx = float(sum(m[1] for m in members)) / n
        fy, fx = members[0]
        out.append((int(round(cx)), int(round(cy)), float(values[fy, fx])))
    return out


@dataclass(frozen=True)
class OBlob:
    """Field-for-field the reference's Blob (detector.py:67-76)."""
    x: int
    y: int
    sigma: float
    radius: float
    response: float
    at_scale_boundary: bool = False


def sort_key(b: OBlob):
    return (-b.response, b.y, b.x, b.sigma)  # detector.py:191-193


def extrema(slices: np.ndarray, slice_sigmas: np.ndarray, threshold: float = 0.1,
            neighborhood: int = 3) -> list[OBlob]:
    """find_extrema (detector.py:149-188) returning the sorted blob list."""
    mask = flagged_mask(slices, threshold, neighborhood)
    S = slices.shape[0]
    blobs = []
    for i in range(S):
        if not mask[i].any():
            continue
        sigma = float(slice_sigmas[i])
        edge = i == 0 or i == S - 1
        for x, y, val in coalesce_slice(mask[i], slices[i]):
            blobs.append(OBlob(x, y, sigma, SQRT2 * sigma, val, edge))
    return sorted(blobs, key=sort_key)


# --------------------------------------------------------------------------
# overlap pruning, histogram
# --------------------------------------------------------------------------

def lens_area(x1, y1, r1, x2, y2, r2) -> float:
    """Scalar disk-intersection area (detector.py:196-209)."""
    d = math.hypot(x2 - x1, y2 - y1)
    if d >= r1 + r2:
        return 0.0
    rmin = min(r1, r2)
    if d <= abs(r1 - r2):
        return math.pi * rmin * rmin
    a1 = r1 * r1 * math.acos((d * d + r1 * r1 - r2 * r2) / (2.0 * d * r1))
    a2 = r2 * r2 * math.acos((d * d + r2 * r2 - r1 * r1) / (2.0 * d * r2))
    s = 0.5 * math.sqrt((-d + r1 + r2) * (d + r1 - r2) * (d - r1 + r2) * (d + r1 + r2))
    return a1 + a2 - s


def normalized_overlap(b1: OBlob, b2: OBlob) -> float:
    rmin = min(b1.radius, b2.radius)  # detector.py:212-218
    if rmin <= 0:
        return 0.0
    return lens_area(b1.x, b1.y, b1.radius, b2.x, b2.y, b2.radius) / (math.pi * rmin * rmin)


def overlap_pairs(x1, y1, r1, x2, y2, r2) -> np.ndarray:
    """Normalised overlap of matrix entries [row][col] for row blobs (x1, y1, r1) and column
    blobs (x2, y2, r2), element-wise on equally shaped arrays: the vector arithmetic of
    _overlap_matrix (detector.py:221-247), float64, same operand order."""
    d = np.hypot(x1 - x2, y1 - y2)
    rmin = np.minimum(r1, r2)
    rmax = np.maximum(r1, r2)
    out = np.zeros(d.shape)
    contained = d <= rmax - rmin
    out[contained] = 1.0
    partial = (~contained) & (d < r1 + r2) & (d > 0)
    if partial.any():
        dd, p1, p2 = d[partial], r1[partial], r2[partial]
        a1 = p1 * p1 * np.arccos(np.clip((dd * dd + p1 * p1 - p2 * p2) / (2 * dd * p1), -1, 1))
        a2 = p2 * p2 * np.arccos(np.clip((dd * dd + p2 * p2 - p1 * p1) / (2 * dd * p2), -1, 1))
        s = 0.5 * np.sqrt(np.clip(
            (-dd + p1 + p2) * (dd + p1 - p2) * (dd - p1 + p2) * (dd + p1 + p2), 0, None))
        rm = np.minimum(p1, p2)
        out[partial] = (a1 + a2 - s) / (np.pi * rm * rm)
    return out


def overlap_row(xs, ys, rs, i: int, js: np.ndarray) -> np.ndarray:
    """Entries [i][js] of the overlap matrix (diagonal zeroed, detector.py:246)."""
    js = np.asarray(js)
    out = overlap_pairs(np.full(js.shape, xs[i]), np.full(js.shape, ys[i]), np.full(js.shape, rs[i]),
                        xs[js], ys[js], rs[js])
    out[js == i] = 0.0
    return out


def overlap_col(xs, ys, rs, ks: np.ndarray, i: int) -> np.ndarray:
    """Entries [ks][i] of the overlap matrix (row blob = k, column blob = i)."""
    ks = np.asarray(ks)
    out = overlap_pairs(xs[ks], ys[ks], rs[ks], np.full(ks.shape, xs[i]), np.full(ks.shape, ys[i]),
                        np.full(ks.shape, rs[i]))
    out[ks == i] = 0.0
    return out


def prune(blobs: list[OBlob], overlap_threshold: float = 0.5) -> list[OBlob]:
    """Sequential greedy coalescing with the reference's visiting order
    (detector.py:250-280): repeatedly take the row-major-first pair (i < j) of
    the response-sorted list whose overlap exceeds the threshold, keep i's
    centre/response, radius <- mean, sigma <- radius / sqrt 2, OR the boundary
    flags, delete j, re-sort.

    Restated without the dense N x N matrix per merge: `first[i]` caches the
    smallest offending j > i and only rows a merge can change are recomputed
    (pairs not touching i or j keep their radii and hence their overlap).
    """
    if not 0.0 <= overlap_threshold <= 1.0:
        raise ValueError(f"overlap threshold must be in [0, 1], got {overlap_threshold}")
    blobs = sorted(blobs, key=sort_key)
    n = len(blobs)
    if n < 2:
        return blobs
    xs = np.array([b.x for b in blobs], dtype=np.float64)
    ys = np.array([b.y for b in blobs], dtype=np.float64)
    rs = np.array([b.radius for b in blobs], dtype=np.float64)

    def first_partner(i, alive_idx):
        js = alive_idx[alive_idx > i]
        if js.size == 0:
            return -1
        hit = overlap_row(xs, ys, rs, i, js) > overlap_threshold
        return int(js[np.argmax(hit)]) if hit.any() else -1

    alive = np.ones(n, dtype=bool)
    alive_idx = np.arange(n)
    first = np.array([first_partner(i, alive_idx) for i in range(n)], dtype=np.int64)
    while True:
        cand = np.nonzero(alive & (first >= 0))[0]
        if cand.size == 0:
            break
        i = int(cand[0])
        j = int(first[i])
        strong, weak = blobs[i], blobs[j]
        new_r = 0.5 * (strong.radius + weak.radius)
        merged = OBlob(strong.x, strong.y, new_r / SQRT2, new_r, strong.response,
                       strong.at_scale_boundary or weak.at_scale_boundary)
        # re-sort: only sigma (last key) of blob i changed; order can change only
        # among exact (response, y, x) ties, which we handle by a full rebuild.
        blobs[i] = merged
        rs[i] = new_r
        alive[j] = False
        tie = [k for k in np.nonzero(alive)[0]
               if k != i and blobs[k].response == merged.response
               and blobs[k].y == merged.y and blobs[k].x == merged.x]
        if tie:
            return prune([blobs[k] for k in np.nonzero(alive)[0]], overlap_threshold)
        alive_idx = np.nonzero(alive)[0]
        first[i] = first_partner(i, alive_idx)
        # rows k < i had no offending partner (i was the first row with one); the
        # only pair of theirs whose overlap changed is (k, i).
        lower = alive_idx[alive_idx < i]
        if lower.size:
            first[lower[overlap_col(xs, ys, rs, lower, i) > overlap_threshold]] = i
        # rows k > i only lose j as a partner
        for k in alive_idx[(alive_idx > i) & (first[alive_idx] == j)]:
            first[int(k)] = first_partner(int(k), alive_idx)
    return [blobs[k] for k in np.nonzero(alive)[0]]


def prune_dense(blobs: list[OBlob], overlap_threshold: float = 0.5) -> list[OBlob]:
    """Literal form of detector.py:259-280 (dense matrix per merge, re-sort);
    O(N^2) per merge -- used to validate `prune` on small inputs."""
    if not 0.0 <= overlap_threshold <= 1.0:
        raise ValueError(f"overlap threshold must be in [0, 1], got {overlap_threshold}")
    blobs = sorted(blobs, key=sort_key)
    while len(blobs) > 1:
        xs = np.array([b.x for b in blobs], dtype=np.float64)
        ys = np.array([b.y for b in blobs], dtype=np.float64)
        rs = np.array([b.radius for b in blobs], dtype=np.float64)
        n = len(blobs)
        hit = None
        for i in range(n - 1):
            js = np.arange(i + 1, n)
            over = overlap_row(xs, ys, rs, i, js) > overlap_threshold
            if over.any():
                hit = (i, int(js[np.argmax(over)]))
                break
        if hit is None:
            break
        i, j = hit
        strong, weak = blobs[i], blobs[j]
        new_r = 0.5 * (strong.radius + weak.radius)
        blobs[i] = OBlob(strong.x, strong.y, new_r / SQRT2, new_r, strong.response,
                         strong.at_scale_boundary or weak.at_scale_boundary)
        del blobs[j]
        blobs = sorted(blobs, key=sort_key)
    return blobs


@dataclass(frozen=True)
class OHistogram:
    bin_centers: np.ndarray = field(repr=False)
    counts: np.ndarray = field(repr=False)
    volume_weights: np.ndarray = field(repr=False)


def radius_histogram(blobs: list[OBlob], sigmas: np.ndarray) -> OHistogram:
    """Nearest ladder-radius bin, ties low; counts and sum 4/3 pi r^3 (detector.py:283-299)."""
    centers = SQRT2 * np.asarray(sigmas, dtype=np.float64)
    counts = np.zeros(centers.size, dtype=np.int64)
    volumes = np.zeros(centers.size, dtype=np.float64)
    if blobs:
        radii = np.array([b.radius for b in blobs])
        mid = 0.5 * (centers[:-1] + centers[1:])
        idx = np.searchsorted(mid, radii, side="left")
        np.add.at(counts, idx, 1)
        np.add.at(volumes, idx, (4.0 / 3.0) * np.pi * radii ** 3)
    return OHistogram(centers, counts, volumes)


# --------------------------------------------------------------------------
# pre-processing (reference default preprocess=True; images.py:112-157)
# --------------------------------------------------------------------------

def smooth(img: np.ndarray, sigma: float) -> np.ndarray:
    img = np.asarray(img).astype(np.float32, copy=False)
    if sigma < 0:
        raise ValueError(f"smoothing sigma must be >= 0, got {sigma}")
    if sigma == 0:
        return img
    return _ndi.gaussian_filter(img, sigma, mode="reflect", truncate=5.0).astype(
        np.float32, copy=False)


def contrast_stretch(img: np.ndarray, saturation: float = 0.0035) -> np.ndarray:
    img = np.asarray(img).astype(np.float32, copy=False)
    if not 0.0 <= saturation < 0.5:
        raise ValueError(f"saturation must be in [0, 0.5), got {saturation}")
    flat = np.sort(img, axis=None)
    n = flat.size

    def rank(q):
        return float(flat[min(max(math.ceil(q * n) - 1, 0), n - 1)])

    lo, hi = rank(saturation / 2.0), rank(1.0 - saturation / 2.0)
    if hi <= lo:
        return np.zeros_like(img)
    return np.clip((img - np.float32(lo)) / np.float32(hi - lo), 0.0, 1.0)


def preprocess(img, smooth_sigma=1.0, saturation=0.0035) -> np.ndarray:
    return contrast_stretch(smooth(img, smooth_sigma), saturation)


# --------------------------------------------------------------------------
# whole pipeline (Detector.run, detector.py:333-360)
# --------------------------------------------------------------------------

@dataclass
class OResult:
    candidates: list          # sorted blobs before pruning
    blobs: list               # after pruning (== candidates when prune=False)
    histogram: OHistogram
    sigmas: np.ndarray
    radii: np.ndarray
    timings_ms: dict


class OracleDetector:
    """Reusable oracle pipeline; caches kernel spectra per image shape the way
    Detector.plan_for / FftPlan.kernel_spectra do (detector.py:323-331)."""

    def __init__(self, min_sigma=1.0, max_sigma=10.0, n_bin=18, truncate=5.0, threshold=0.1,
                 overlap=0.5, neighborhood=3, backend="fft", preprocess=True, smooth_sigma=1.0,
                 saturation=0.0035, prune=True):
        self.threshold = threshold
        self.overlap = overlap
        self.neighborhood = neighborhood
        self.backend = backend
        self.do_preprocess = preprocess
        self.smooth_sigma = smooth_sigma
        self.saturation = saturation
        self.do_prune = prune
        self.sigmas = ladder_sigmas(min_sigma, max_sigma, n_bin)
        self.radii = tap_radii(self.sigmas, truncate)
        if 2 * int(self.radii.max()) + 1 > 4097:  # scale_space.py:21,100-104
            raise ValueError("kernel width exceeds cap 4097")
        self._spectra = {}

    def spectra_for(self, shape, dtype):
        key = (tuple(shape), np.dtype(dtype).name)
        if key not in self._spectra:
            self._spectra[key] = fft_spectra(shape, self.sigmas, self.radii, dtype)
        return self._spectra[key]

    def run(self, img, dtype=np.float32) -> OResult:
        import time
        t = {}
        t0 = time.perf_counter()
        if self.do_preprocess:
            img = preprocess(img, self.smooth_sigma, self.saturation)
        t["preprocess_ms"] = (time.perf_counter() - t0) * 1e3
        t0 = time.perf_counter()
        img = _check_image(img)
        if img.shape[0] * img.shape[1] * len(self.sigmas) > 2 ** 28:
            raise ValueError("stack exceeds element cap")
        if self.backend == "fft":
            levels = levels_fft(img, self.sigmas, self.radii, dtype,
                                self.spectra_for(img.shape, dtype))
        else:
            levels = levels_separable(img, self.sigmas, self.radii, dtype)
        t["convolve_ms"] = (time.perf_counter() - t0) * 1e3
        t0 = time.perf_counter()
        slices = dog_slices(levels, self.sigmas)
        cands = extrema(slices, self.sigmas[:-1], self.threshold, self.neighborhood)
        t["extrema_ms"] = (time.perf_counter() - t0) * 1e3
        t0 = time.perf_counter()
        kept = prune(cands, self.overlap) if self.do_prune else list(cands)
        t["prune_ms"] = (time.perf_counter() - t0) * 1e3
        return OResult(cands, kept, radius_histogram(kept, self.sigmas), self.sigmas,
                       self.radii, t)


# --------------------------------------------------------------------------
# pointwise float64 evidence for near-tie classification
# --------------------------------------------------------------------------

def dog_neighbourhood_f64(img, sigmas, radii, s: int, y: int, x: int, half: int = 1) -> np.ndarray:
    """float64 DoG values on the (2h+1)^3 block around voxel (s, y, x); entries
    outside the volume are -inf.  Evaluated from the 2-D kernel definition."""
    img = np.asarray(img, dtype=np.float64)
    H, W = img.shape
    S = len(sigmas) - 1
    n = 2 * half + 1
    out = np.full((n, n, n), -np.inf)
    ys, xs, pos = [], [], []
    for dy in range(-half, half + 1):
        for dx in range(-half, half + 1):
            if 0 <= y + dy < H and 0 <= x + dx < W:
                ys.append(y + dy)
                xs.append(x + dx)
                pos.append((dy + half, dx + half))
    lv = {}
    for ds in range(-half, half + 1):
        for lev in (s + ds, s + ds + 1):
            if 0 <= s + ds < S and lev not in lv:
                lv[lev] = level_values_at(img, sigmas[lev], int(radii[lev]), ys, xs)
    for ds in range(-half, half + 1):
        si = s + ds
        if not 0 <= si < S:
            continue
        d = float(sigmas[si]) * (lv[si] - lv[si + 1])
        for (py, px), v in zip(pos, d):
            out[ds + half, py, px] = v
    return out
