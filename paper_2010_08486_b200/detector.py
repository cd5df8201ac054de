"""Drop-in detector API over the sm_100a CUDA hot path.

Mirrors the reference detector module (`pkg/src/dogblob/detector.py`) and the
stage function of `pkg/src/dogblob/convolve.py`: same names, argument meaning,
result types and error behaviour, with `backend="cuda"` as the only backend.
Everything numeric runs in libdogblob_b200.so (include/dogblob_b200.h); this
file is plumbing: parameter records, device buffers (torch), streams, result
decoding.  There is no CPU fallback - without the CUDA library and a GPU every
compute entry point raises.

Layout on the device (per frame slot):
  image      [H][Wp]            float32, Wp = W rounded up to 128
  rows^T     [L][Wp][Hp]        row-filtered planes, stored x-major
  DoG^T      [S][Wp][Hp]        sigma_i (L_i - L_{i+1}), x-major (never transposed back)
  blob space candidate lists, sort/prune scratch
  result     header + blob records (dogblob_blob), sorted by (-response, y, x, sigma)
"""

from __future__ import annotations

import ctypes as C
import math
import os
import queue
import threading
import time
from dataclasses import asdict, dataclass, field

import numpy as np

from . import _lib
from .scale_space import SigmaLadder, TapBank, build_kernel_bank, build_ladder

__all__ = [
    "BACKENDS", "ScaleStack", "DoGStack", "Blob", "BlobSet", "RadiusHistogram", "DetectionParams",
    "DetectResult", "Detector", "convolve_bank", "dog_stack", "find_extrema", "prune_overlaps",
    "normalized_overlap", "disk_intersection_area", "histogram", "detect",
]

BACKENDS = ("cuda",)
RADIUS_PER_SIGMA = math.sqrt(2.0)
DEFAULT_STACK_ELEMENT_CAP = 2 ** 28   # convolve.py:37 (the reference's host-RAM guard)
DEFAULT_MAX_BLOBS = 1 << 16
HOST_RESULT_BLOBS = 4096              # records copied back with the header in one D2H
# FP32 engine only: frames of at least 8 MiB upload in row chunks under the running row pass (below
# that the gate only delays a row pass that is shorter than the copy: C1 0.21 vs 0.16 ms, C5 0.88
# vs 0.84 ms).  The tensor-core engine needs the whole frame's maximum (scale of its fp16 operand
# split) before its first MMA and always uploads in one piece; its 4 MiB copy is 15 % of a C2
# frame's latency and overlaps the kernels of the other slots in run_batch.
STREAM_MIN_BYTES_FP32 = 8 << 20
STREAMED_UPLOAD = os.environ.get("DOGBLOB_STREAMED_UPLOAD", "1") != "0"


# --------------------------------------------------------------------------
# records (field-for-field the reference's)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class ScaleStack:
    """convolve.py:40-53."""
    levels: np.ndarray = field(repr=False)
    sigmas: np.ndarray = field(repr=False)

    @property
    def n_levels(self) -> int:
        return self.levels.shape[0]

    @property
    def shape(self) -> tuple[int, int]:
        return self.levels.shape[1], self.levels.shape[2]


@dataclass(frozen=True)
class DoGStack:
    """detector.py:55-64; slices[i] = sigmas[i] * (L_i - L_{i+1})."""
    slices: np.ndarray = field(repr=False)
    sigmas: np.ndarray = field(repr=False)

    @property
    def n_slices(self) -> int:
        return self.slices.shape[0]


@dataclass(frozen=True)
class Blob:
    """detector.py:67-76."""
    x: int
    y: int
    sigma: float
    radius: float
    response: float
    at_scale_boundary: bool = False


@dataclass(frozen=True)
class DetectionParams:
    """detector.py:79-95; only the backend default differs ("cuda")."""
    min_sigma: float = 1.0
    max_sigma: float = 10.0
    n_bin: int = 18
    truncate: float = 5.0
    threshold: float = 0.1
    overlap: float = 0.5
    neighborhood: int = 3
    backend: str = "cuda"
    preprocess: bool = True
    smooth_sigma: float = 1.0
    saturation: float = 0.0035
    prune: bool = True

    def to_dict(self) -> dict:
        return asdict(self)


class BlobSet:
    """detector.py:98-105, backed by the device result records.

    `blobs` (tuple of Blob) is materialised on first access so that batch
    throughput is not bounded by Python object construction; `records`,
    `yxs()` and `radii` expose the same data as arrays.
    """

    def __init__(self, blobs=None, source_shape=(0, 0), params=None, records=None):
        if records is None:
            blobs = tuple(blobs or ())
            records = np.zeros(len(blobs), dtype=_lib.BLOB_DTYPE)
            for i, b in enumerate(blobs):
                records[i] = (b.x, b.y, b.sigma, b.radius, b.response, -1,
                              _lib.BLOB_SCALE_EDGE if b.at_scale_boundary else 0)
            self._blobs = blobs
        else:
            self._blobs = None
        self.records = records
        self.source_shape = tuple(source_shape)   # (width, height)
        self.params = params if params is not None else DetectionParams()

    @property
    def blobs(self) -> tuple:
        if self._blobs is None:
            r = self.records
            integral = bool(np.all(r["x"] == np.rint(r["x"])) and np.all(r["y"] == np.rint(r["y"])))
            xs = r["x"].astype(np.int64).tolist() if integral else r["x"].tolist()
            ys = r["y"].astype(np.int64).tolist() if integral else r["y"].tolist()
            edge = ((r["flags"] & _lib.BLOB_SCALE_EDGE) != 0).tolist()
            self._blobs = tuple(
                Blob(x, y, s, rad, resp, e)
                for x, y, s, rad, resp, e in zip(xs, ys, r["sigma"].tolist(), r["radius"].tolist(),
                                                 r["response"].tolist(), edge))
        return self._blobs

    def yxs(self) -> np.ndarray:
        """(N, 3) float64 array of (y, x, sigma) rows, strongest first."""
        r = self.records
        return np.stack([r["y"], r["x"], r["sigma"]], axis=1) if len(r) else np.zeros((0, 3))

    @property
    def radii(self) -> np.ndarray:
        return self.records["radius"].copy()

    def __len__(self) -> int:
        return len(self.records)

    def __eq__(self, other):
        if not isinstance(other, BlobSet):
            return NotImplemented
        return (self.blobs == other.blobs and self.source_shape == other.source_shape
                and self.params == other.params)

    def __repr__(self):
        return f"BlobSet(n={len(self)}, source_shape={self.source_shape})"


@dataclass(frozen=True)
class RadiusHistogram:
    """detector.py:108-114."""
    bin_centers: np.ndarray = field(repr=False)
    counts: np.ndarray = field(repr=False)
    volume_weights: np.ndarray = field(repr=False)


class DetectResult:
    """detector.py:55-64 `DetectResult(blobs, histogram, timings_ms)`, plus `stats`.

    `histogram` may be given as a zero-argument callable: it is then evaluated on first access
    (the single-frame latency path does not pay for a histogram nobody reads)."""
    __slots__ = ("blobs", "_histogram", "timings_ms", "stats")

    def __init__(self, blobs, histogram, timings_ms, stats=None):
        self.blobs = blobs
        self._histogram = histogram
        self.timings_ms = timings_ms
        self.stats = {} if stats is None else stats   # n_flagged / n_plateau / n_candidates / n_merges

    @property
    def histogram(self) -> "RadiusHistogram":
        h = self._histogram
        if callable(h):
            h = self._histogram = h()
        return h

    def __repr__(self):
        return f"DetectResult(blobs={self.blobs!r}, timings_ms={self.timings_ms!r})"


# --------------------------------------------------------------------------
# device plumbing
# --------------------------------------------------------------------------

def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("backend='cuda' needs a CUDA device; there is no CPU fallback")
    return torch


def _check_image(img) -> np.ndarray:
    img = np.asarray(img)
    if img.ndim != 2 or img.shape[0] < 1 or img.shape[1] < 1:
        raise ValueError(f"expected a non-empty 2-D image, got shape {img.shape}")
    return img


def _check_backend(backend: str) -> None:
    if backend not in BACKENDS:
        raise ValueError(f"unknown backend {backend!r}; expected one of {BACKENDS}")


def _check_dtype(dtype) -> np.dtype:
    """float32 (production kernels) or float64 (the oracle-grade tier, convolve.py:76-77)."""
    dt = np.dtype(dtype)
    if dt not in (np.dtype(np.float32), np.dtype(np.float64)):
        raise ValueError(f"backend='cuda' computes the scale space in float32 or float64; dtype={dt.name} "
                         "is not available")
    return dt


def _f64_tables(bank: TapBank):
    """host tables of the float64 entry points: sigmas, radii, float64 taps, offsets"""
    return (np.ascontiguousarray(bank.ladder.sigmas, dtype=np.float64),
            np.ascontiguousarray(bank.radii, dtype=np.int32),
            np.ascontiguousarray(bank.taps64, dtype=np.float64),
            np.ascontiguousarray(bank.offsets, dtype=np.int64))


class _Plan:
    """Owns one dogblob_plan (ladder + taps for one image shape on one device)."""

    def __init__(self, bank: TapBank, shape, device: int, max_blobs: int):
        lib = _lib.load()
        H, W = int(shape[0]), int(shape[1])
        self.shape = (H, W)
        self.device = device
        self.max_blobs = int(max_blobs)
        self.n_levels = bank.ladder.n_levels
        sig = np.ascontiguousarray(bank.ladder.sigmas, dtype=np.float64)
        radii = np.ascontiguousarray(bank.radii, dtype=np.int32)
        taps = np.ascontiguousarray(bank.taps32, dtype=np.float32)
        offs = np.ascontiguousarray(bank.offsets, dtype=np.int64)
        handle = C.c_void_p()
        _lib.check(lib.dogblob_plan_create(device, H, W, self.n_levels, _lib.ptr(sig),
                                           _lib.ptr(radii), _lib.ptr(taps), _lib.ptr(offs),
                                           self.max_blobs, C.byref(handle)))
        self.handle = handle
        self.workspace_bytes = int(lib.dogblob_workspace_bytes(handle))
        self.result_bytes = int(lib.dogblob_result_bytes(handle))
        self.pitch = int(lib.dogblob_image_pitch(handle))
        self.conv_engine = int(lib.dogblob_plan_conv_engine(handle))   # 0 FP32 kernels, 1 tcgen05 (2: fp16 build)
        import ctypes
        buf = (ctypes.c_int32 * 400)()
        n = int(lib.dogblob_plan_conv_groups(handle, buf, 400))
        self.conv_groups = [int(buf[i]) for i in range(n + 1)]        # level groups of the fused column pass

    def close(self):
        if self.handle is not None:
            _lib.load().dogblob_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


N_EVENTS = 5   # DOGBLOB_N_EVENTS: start | row pass | column+DoG pass | extrema | prune+pack


def new_events():
    lib = _lib.load()
    events = (C.c_void_p * N_EVENTS)()
    for k in range(N_EVENTS):
        e = C.c_void_p()
        _lib.check(lib.dogblob_event_create(C.byref(e)))
        events[k] = e
    return events


def free_events(events) -> None:
    lib = _lib.load()
    for k in range(N_EVENTS):
        if events[k]:
            lib.dogblob_event_destroy(events[k])
            events[k] = None


def event_intervals_ms(events) -> list:
    """[row pass, column+DoG pass, extrema, prune+pack] in milliseconds."""
    out = (C.c_float * (N_EVENTS - 1))()
    _lib.check(_lib.load().dogblob_event_intervals_ms(events, N_EVENTS, out))
    return list(out)


class _Slot:
    """Buffers + stream of one in-flight frame (one per concurrent caller)."""

    def __init__(self, plan: _Plan):
        torch = _torch()
        lib = _lib.load()
        dev = torch.device("cuda", plan.device)
        H, W = plan.shape
        self.plan = plan
        self.stream = torch.cuda.Stream(device=dev)
        self.d_image = torch.zeros((H, plan.pitch), dtype=torch.float32, device=dev)
        self.d_work = torch.zeros(plan.workspace_bytes, dtype=torch.uint8, device=dev)
        self.d_result = torch.zeros(plan.result_bytes, dtype=torch.uint8, device=dev)
        self.h_image = torch.empty((H, W), dtype=torch.float32).pin_memory()
        self.d_raw = None          # raw frame + scratch, allocated on first preprocess=True use
        self.d_pre = None
        self.h_status = torch.zeros(1, dtype=torch.int32).pin_memory()
        # streamed upload (frames of at least STREAM_MIN_BYTES): second stream, gate, frame event
        self.copy_stream = torch.cuda.Stream(device=dev)
        self.h_gate = torch.zeros(_lib.GATE_INTS, dtype=torch.int32).pin_memory()
        done = C.c_void_p()
        _lib.check(lib.dogblob_event_create(C.byref(done)))
        self.frame_done = done
        self.pre_events = None
        n_host = min(HOST_RESULT_BLOBS, plan.max_blobs)
        self.h_result = torch.zeros(_lib.RESULT_HEADER_BYTES + n_host * _lib.BLOB_DTYPE.itemsize,
                                    dtype=torch.uint8).pin_memory()
        self.h_result_np = self.h_result.numpy()
        self.h_image_np = self.h_image.numpy()
        self.n_host = n_host
        torch.cuda.synchronize(dev)
        self.pending = None     # bookkeeping of run_batch
        self.streamed = False   # whether the last launch() used the streamed upload

    # ---- one frame --------------------------------------------------------------
    def launch(self, frame, params: DetectionParams, prune: bool) -> None:
        """H2D + all kernels + D2H of header/records, asynchronously on self.stream."""
        lib = _lib.load()
        torch = _torch()
        if isinstance(frame, torch.Tensor) and frame.device.type == "cuda":
            self._launch_resident(frame, params, prune)
            return
        src = self._host_pointer(frame)
        self.preprocessed = bool(params.preprocess)
        if params.preprocess:
            self._launch_with_preprocess(src, params, prune)
            return
        H, W = self.plan.shape
        self.streamed = (STREAMED_UPLOAD and self.plan.conv_engine == 0
                         and H * W * 4 >= STREAM_MIN_BYTES_FP32)
        if self.streamed:
            # row chunks on the copy stream while the row pass already runs
            _lib.check(lib.dogblob_detect_host_streamed(
                self.plan.handle, src, float(np.float32(params.threshold)), int(params.neighborhood),
                float(params.overlap), 1 if prune else 0, self.d_image.data_ptr(),
                self.d_work.data_ptr(), self.d_result.data_ptr(), self.h_result.data_ptr(),
                self.n_host, self.stream.cuda_stream, self.copy_stream.cuda_stream,
                self.h_gate.data_ptr(), self.frame_done, None))
            return
        _lib.check(lib.dogblob_detect_host(
            self.plan.handle, src, float(np.float32(params.threshold)), int(params.neighborhood),
            float(params.overlap), 1 if prune else 0, self.d_image.data_ptr(),
            self.d_work.data_ptr(), self.d_result.data_ptr(), self.h_result.data_ptr(),
            self.n_host, self.stream.cuda_stream, None))   # stage times come back in the header

    def _launch_with_preprocess(self, src: int, params: DetectionParams, prune: bool) -> None:
        """raw frame H2D -> smooth + stretch on the device (images.py:153-157) -> detect."""
        from .images import smooth_taps, stretch_ranks
        torch = _torch()
        lib = _lib.load()
        H, W = self.plan.shape
        if self.d_raw is None:
            dev = self.d_image.device
            self.d_raw = torch.zeros((H, self.plan.pitch), dtype=torch.float32, device=dev)
            self.d_pre = torch.zeros(int(lib.dogblob_preprocess_bytes(H, W)), dtype=torch.uint8,
                                     device=dev)
            self.pre_events = (C.c_void_p * 2)()
            for k in range(2):
                e = C.c_void_p()
                _lib.check(lib.dogblob_event_create(C.byref(e)))
                self.pre_events[k] = e
        radius, taps = smooth_taps(params.smooth_sigma)
        lo, hi = stretch_ranks(H * W, params.saturation)
        st = self.stream.cuda_stream
        _lib.check(lib.dogblob_event_record(self.pre_events[0], st))
        _lib.check(lib.dogblob_upload_image(self.plan.handle, src, self.d_raw.data_ptr(), st))
        _lib.check(lib.dogblob_preprocess(H, W, self.d_raw.data_ptr(), self.plan.pitch, radius,
                                          _lib.ptr(taps), lo, hi, self.d_pre.data_ptr(),
                                          self.d_image.data_ptr(), self.plan.pitch, st))
        _lib.check(lib.dogblob_preprocess_status(self.d_pre.data_ptr(), self.h_status.data_ptr(), st))
        _lib.check(lib.dogblob_event_record(self.pre_events[1], st))
        self.launch_device(self.d_image, params, prune)
        n = min(self.n_host, self.plan.max_blobs)
        _lib.check(lib.dogblob_fetch_result(self.d_result.data_ptr(), n, self.h_result.data_ptr(), st))

    def _launch_resident(self, frame, params: DetectionParams, prune: bool) -> None:
        """A frame that already lives on the device (float32 CUDA tensor [H][W], e.g. from
        synth.device_frames or an upstream GPU stage): no host round trip for the pixels."""
        torch = _torch()
        lib = _lib.load()
        H, W = self.plan.shape
        if params.preprocess:
            raise ValueError("device-resident frames are detected as they are: use preprocess=False")
        if frame.dtype != torch.float32 or tuple(frame.shape) != (H, W) or frame.device.index != self.plan.device:
            raise ValueError(f"expected a float32 CUDA tensor of shape {(H, W)} on device {self.plan.device}")
        self.preprocessed = False
        self.streamed = False
        self.stream.wait_stream(torch.cuda.current_stream(frame.device))     # the producer's work is ordered first
        with torch.cuda.stream(self.stream):
            if W == self.plan.pitch and frame.is_contiguous():
                src = frame                                   # the detector's own layout: zero copy
                self._keepalive = frame
            else:
                self.d_image[:, :W].copy_(frame, non_blocking=True)
                src = self.d_image
        self.launch_device(src, params, prune)
        n = min(self.n_host, self.plan.max_blobs)
        _lib.check(lib.dogblob_fetch_result(self.d_result.data_ptr(), n, self.h_result.data_ptr(),
                                            self.stream.cuda_stream))

    def launch_device(self, d_frame, params: DetectionParams, prune: bool, events=None) -> None:
        """Same, for a frame that is already resident: a float32 CUDA tensor [H][pitch]."""
        lib = _lib.load()
        _lib.check(lib.dogblob_detect(
            self.plan.handle, d_frame.data_ptr(), float(np.float32(params.threshold)),
            int(params.neighborhood), float(params.overlap), 1 if prune else 0,
            self.d_work.data_ptr(), self.d_result.data_ptr(), self.stream.cuda_stream, events))

    def _host_pointer(self, frame) -> int:
        torch = _torch()
        H, W = self.plan.shape
        if isinstance(frame, torch.Tensor):
            if frame.device.type != "cpu":
                raise ValueError("expected a host frame")
            if (frame.dtype == torch.float32 and frame.is_contiguous() and frame.is_pinned()
                    and tuple(frame.shape) == (H, W)):
                self._keepalive = frame
                return frame.data_ptr()
            frame = frame.numpy()
        np.copyto(self.h_image_np, np.asarray(frame), casting="same_kind")
        return self.h_image.data_ptr()

    def collect(self):
        """Wait for the frame and decode header + records (numpy structured array)."""
        lib = _lib.load()
        self.stream.synchronize()
        if getattr(self, "preprocessed", False) and (int(self.h_status.item()) & 1):
            raise ValueError("image contains NaN or Inf values")
        hdr = self.h_result_np[:_lib.RESULT_HEADER_BYTES].view(_lib.HEADER_DTYPE)[0].copy()
        n = int(hdr["n_blobs"])
        if int(hdr["flags"]) & _lib.FLAG_OVERFLOW:
            return hdr, None
        recs = np.empty(n, dtype=_lib.BLOB_DTYPE)
        k = min(n, self.n_host)
        body = self.h_result_np[_lib.RESULT_HEADER_BYTES:]
        recs[:k] = body[:k * _lib.BLOB_DTYPE.itemsize].view(_lib.BLOB_DTYPE)
        if n > k:
            _lib.check(lib.dogblob_fetch_blobs(self.d_result.data_ptr(), k, n - k,
                                               recs[k:].ctypes.data, self.stream.cuda_stream))
            self.stream.synchronize()
        return hdr, recs

    def stage_times_ms(self, hdr) -> dict:
        """timings_ms of the frame just collected: device-side stamps from the result header
        (no event calls on the latency path); pre-processing is bracketed by two events."""
        pre = 0.0
        if getattr(self, "preprocessed", False):
            ms = C.c_float()
            _lib.check(_lib.load().dogblob_event_elapsed_ms(self.pre_events[0], self.pre_events[1],
                                                            C.byref(ms)))
            pre = float(ms.value)
        return {"preprocess_ms": pre, "convolve_ms": int(hdr["conv_ns"]) * 1e-6,
                "extrema_ms": int(hdr["extrema_ns"]) * 1e-6, "prune_ms": int(hdr["prune_ns"]) * 1e-6}

    def close(self):
        if self.frame_done is not None:
            _lib.load().dogblob_event_destroy(self.frame_done)
            self.frame_done = None
        if self.pre_events is not None:
            lib = _lib.load()
            for k in range(2):
                if self.pre_events[k]:
                    lib.dogblob_event_destroy(self.pre_events[k])
                    self.pre_events[k] = None


class _Engine:
    """Plan + slot pool for one image shape.

    `users` counts the calls that currently hold a lease on the engine (Detector._lease); an engine
    that has been replaced (candidate capacity grown) is only marked `retired` and is closed by
    the last call that still uses it, so no plan or slot is destroyed under a concurrent caller.
    """

    def __init__(self, bank: TapBank, shape, device: int, max_blobs: int, n_slots: int):
        self.plan = _Plan(bank, shape, device, max_blobs)
        try:
            self._check_memory(n_slots)
            self.slots = [_Slot(self.plan) for _ in range(n_slots)]
        except Exception:
            self.plan.close()
            raise
        self.free = queue.Queue()
        for s in self.slots:
            self.free.put(s)
        self.users = 0
        self.retired = False

    def _check_memory(self, n_slots: int) -> None:
        """The slot pool must fit the device: a parameter error like the reference's stack cap
        (convolve.py:209-212), not an out-of-memory failure half way through the allocation."""
        torch = _torch()
        H, W = self.plan.shape
        need = n_slots * (self.plan.workspace_bytes + self.plan.result_bytes + H * self.plan.pitch * 4)
        free, _total = torch.cuda.mem_get_info(self.plan.device)
        if need > 0.9 * free:
            raise ValueError(f"scale-space workspace of {need / 2**30:.1f} GiB ({n_slots} slots of "
                             f"{self.plan.workspace_bytes / 2**30:.1f} GiB) exceeds the device memory "
                             f"available ({free / 2**30:.1f} GiB free)")

    def close(self):
        for s in self.slots:
            s.close()
        self.plan.close()


# --------------------------------------------------------------------------
# the reusable pipeline
# --------------------------------------------------------------------------

def histogram(blobset: BlobSet, ladder: SigmaLadder) -> RadiusHistogram:
    """Nearest ladder-radius bin, ties to the smaller (detector.py:283-299).

    Evaluated on the host in float64 over the <= ~10^4 surviving radii so that
    counts and volume weights are bit-identical to the reference's numpy
    arithmetic (np.add.at order, libm pow).
    """
    centers = RADIUS_PER_SIGMA * ladder.sigmas
    counts = np.zeros(centers.size, dtype=np.int64)
    volumes = np.zeros(centers.size, dtype=np.float64)
    if len(blobset) > 0:
        radii = blobset.radii
        mid = 0.5 * (centers[:-1] + centers[1:])
        idx = np.searchsorted(mid, radii, side="left")
        np.add.at(counts, idx, 1)
        np.add.at(volumes, idx, (4.0 / 3.0) * np.pi * radii ** 3)
    return RadiusHistogram(bin_centers=centers, counts=counts, volume_weights=volumes)


class Detector:
    """Reusable detection pipeline for a fixed parameter set (detector.py:302-360).

    Immutable after construction apart from lock-guarded, append-only per-shape
    engines, so one Detector may serve many images and threads concurrently
    (each concurrent `run` borrows its own slot: stream + workspace).
    """

    def __init__(self, params: DetectionParams, device: int | None = None,
                 max_blobs: int = DEFAULT_MAX_BLOBS, slots: int = 2):
        _check_backend(params.backend)
        self.params = params
        self.ladder = build_ladder(params.min_sigma, params.max_sigma, params.n_bin)
        self.bank = build_kernel_bank(self.ladder, params.truncate)
        if params.neighborhood < 1 or params.neighborhood % 2 == 0:
            raise ValueError(f"neighborhood must be odd and >= 1, got {params.neighborhood}")
        if not 0.0 <= params.overlap <= 1.0:
            raise ValueError(f"overlap threshold must be in [0, 1], got {params.overlap}")
        self._device = device
        self._max_blobs = int(max_blobs)
        self._n_slots = max(1, int(slots))
        self._engines: dict = {}
        self._lock = threading.Lock()

    # -- plumbing ---------------------------------------------------------------
    @property
    def device(self) -> int:
        if self._device is None:
            self._device = _torch().cuda.current_device()
        return self._device

    def plan_for(self, shape) -> _Engine:
        """Per-shape engine, double-checked like the reference's plan cache (detector.py:323-331)."""
        key = (int(shape[0]), int(shape[1]))
        eng = self._engines.get(key)
        if eng is None:
            with self._lock:
                eng = self._engines.get(key)
                if eng is None:
                    eng = _Engine(self.bank, key, self.device, self._max_blobs, self._n_slots)
                    self._engines[key] = eng
        return eng

    def _lease(self, shape) -> _Engine:
        """The per-shape engine with a use count; every _lease needs one _release."""
        key = (int(shape[0]), int(shape[1]))
        with self._lock:
            eng = self._engines.get(key)
            if eng is None:
                eng = _Engine(self.bank, key, self.device, self._max_blobs, self._n_slots)
                self._engines[key] = eng
            eng.users += 1
            return eng

    def _release(self, eng: _Engine) -> None:
        with self._lock:
            eng.users -= 1
            close_now = eng.retired and eng.users == 0
        if close_now:
            eng.close()

    def _grow(self, shape, seen: _Engine) -> None:
        """Candidate capacity exceeded on engine `seen`: replace it by one with 4x the room, once
        (concurrent overflows of the same engine grow it a single time).  The caller still holds its
        lease; the retired engine is closed by the last _release."""
        key = (int(shape[0]), int(shape[1]))
        with self._lock:
            if self._engines.get(key) is seen:
                del self._engines[key]
                self._max_blobs *= 4
            seen.retired = True

    def close(self) -> None:
        with self._lock:
            engines = list(self._engines.values())
            self._engines.clear()
            idle = []
            for eng in engines:
                eng.retired = True
                if eng.users == 0:
                    idle.append(eng)
        for eng in idle:                # engines still in use are closed by their last user
            eng.close()

    def _prepare(self, img, dtype):
        if _check_dtype(dtype) == np.float64:
            return np.ascontiguousarray(_check_image(img), dtype=np.float64)
        torch = _torch()
        if isinstance(img, torch.Tensor):
            if img.ndim != 2 or img.shape[0] < 1 or img.shape[1] < 1:
                raise ValueError(f"expected a non-empty 2-D image, got shape {tuple(img.shape)}")
            return img
        img = _check_image(img)
        if img.dtype != np.float32:
            img = img.astype(np.float32)
        return img

    def _finish(self, slot: _Slot, hdr, recs, shape, timings) -> DetectResult:
        blobs = BlobSet(records=recs, source_shape=(shape[1], shape[0]), params=self.params)
        stats = {k: int(hdr[k]) for k in ("n_flagged", "n_plateau", "n_candidates", "n_merges", "n_seeds")}
        prof = [int(v) & 0xFFFFFFFF for v in hdr["prune_profile"]]
        if prof[3]:                      # whole-GPU pruning kernel ran: its phase profile
            r = [prof[0] & 0xFFFF, prof[0] >> 16, prof[1] & 0xFFFF, prof[1] >> 16, prof[2] & 0xFFFF, prof[2] >> 16]
            stats["prune_profile"] = {"order_us": r[0], "grid_first_us": r[1] - r[0], "bound_us": r[2] - r[1],
                                      "parts_us": r[3] - r[2], "merge_us": r[4] - r[3], "pack_us": r[5] - r[4],
                                      "total_us": r[5], "sweeps": prof[3] >> 24, "parts": prof[3] & 0xFFFFFF}
        ladder = self.ladder
        return DetectResult(blobs=blobs, histogram=lambda: histogram(blobs, ladder),
                            timings_ms=timings, stats=stats)

    # -- public API -------------------------------------------------------------
    def run(self, img, dtype=np.float32) -> DetectResult:
        """Full pipeline on one frame; per-stage timings are CUDA-event milliseconds."""
        p = self.params
        img = self._prepare(img, dtype)
        shape = tuple(img.shape)
        if np.dtype(dtype) == np.float64:
            return self._run_f64(img)
        while True:
            eng = self._lease(shape)     # ValueError if the slot pool cannot fit the device
            try:
                slot = eng.free.get()
                try:
                    slot.launch(img, p, p.prune)
                    hdr, recs = slot.collect()
                    timings = slot.stage_times_ms(hdr)
                finally:
                    eng.free.put(slot)
                if recs is not None:
                    return self._finish(slot, hdr, recs, shape, timings)
                self._grow(shape, eng)   # candidate capacity exceeded: retry with 4x the room
            finally:
                self._release(eng)

    def _run_f64(self, img: np.ndarray) -> DetectResult:
        """The float64 tier (detector.py:333 with dtype=np.float64): every stage in float64 on the
        device, buffers allocated per call - the oracle-grade path, ~100x slower than float32."""
        torch = _torch()
        lib = _lib.load()
        p = self.params
        t0 = time.perf_counter()
        if p.preprocess:                  # host float64, like the reference (images.py:112-157)
            from .images import preprocess
            img = np.ascontiguousarray(preprocess(img, p.smooth_sigma, p.saturation), dtype=np.float64)
        pre_ms = (time.perf_counter() - t0) * 1e3
        H, W = img.shape
        sig, rad, taps, offs = _f64_tables(self.bank)
        L = int(sig.size)
        dev = torch.device("cuda", self.device)
        max_blobs = self._max_blobs
        with torch.cuda.device(dev):
            st = torch.cuda.current_stream(dev)
            d_img = torch.from_numpy(img).to(dev)
            while True:
                need = int(lib.dogblob_f64_workspace_bytes(H, W, L, max_blobs))
                free, _total = torch.cuda.mem_get_info(dev)
                if need > 0.9 * free:
                    raise ValueError(f"float64 scale-space workspace of {need / 2**30:.1f} GiB exceeds the device "
                                     f"memory available ({free / 2**30:.1f} GiB free)")
                work = torch.empty(need, dtype=torch.uint8, device=dev)
                res = torch.zeros(int(lib.dogblob_result_bytes_for(max_blobs)), dtype=torch.uint8, device=dev)
                _lib.check(lib.dogblob_detect_f64(H, W, L, _lib.ptr(sig), _lib.ptr(rad), _lib.ptr(taps), _lib.ptr(offs),
                                                  d_img.data_ptr(), float(p.threshold), int(p.neighborhood),
                                                  float(p.overlap), 1 if p.prune else 0, max_blobs,
                                                  work.data_ptr(), res.data_ptr(), st.cuda_stream))
                hdr, recs = _read_result(res, max_blobs)
                if recs is not None:
                    break
                max_blobs *= 4
        timings = {"preprocess_ms": pre_ms, "convolve_ms": int(hdr["conv_ns"]) * 1e-6,
                   "extrema_ms": int(hdr["extrema_ns"]) * 1e-6, "prune_ms": int(hdr["prune_ns"]) * 1e-6}
        return self._finish(None, hdr, recs, (H, W), timings)

    def run_batch(self, frames, timings: bool = False) -> list:
        """Detect over a sequence of equally shaped host frames, pipelined over the
        slot pool: the H2D copy and kernels of frame f+1 overlap the D2H/decode of f."""
        p = self.params
        frames = [self._prepare(f, np.float32) for f in frames]
        if not frames:
            return []
        shape = tuple(frames[0].shape)
        for f in frames:
            if tuple(f.shape) != shape:
                raise ValueError("run_batch needs equally shaped frames")
        eng = self._lease(shape)
        # one slot for certain, the others only if they are free right now: concurrent callers
        # (batches or single frames) share the pool instead of waiting for each other's slots
        slots = [eng.free.get()]
        while len(slots) < len(eng.slots):
            try:
                slots.append(eng.free.get_nowait())
            except queue.Empty:
                break
        results = [None] * len(frames)
        retry = []
        try:
            def drain(slot):
                idx = slot.pending
                slot.pending = None
                hdr, recs = slot.collect()
                if recs is None:
                    retry.append(idx)
                    return
                t = slot.stage_times_ms(hdr) if timings else {}
                results[idx] = self._finish(slot, hdr, recs, shape, t)

            for i, frame in enumerate(frames):
                slot = slots[i % len(slots)]
                if slot.pending is not None:
                    drain(slot)
                slot.launch(frame, p, p.prune)
                slot.pending = i
            for slot in slots:
                if slot.pending is not None:
                    drain(slot)
        finally:
            for s in slots:
                s.pending = None
                eng.free.put(s)
            if retry:
                self._grow(shape, eng)
            self._release(eng)
        for idx in retry:
            results[idx] = self.run(frames[idx])
        return results


def detect(img, params: DetectionParams) -> tuple:
    """One-shot detection (detector.py:363-366)."""
    det = Detector(params)
    try:
        result = det.run(img)
    finally:
        det.close()
    return result.blobs, result.histogram


# --------------------------------------------------------------------------
# stage functions (convolve.py:189-218, detector.py:117-299) on the CUDA library
# --------------------------------------------------------------------------

_stage_lock = threading.Lock()


def _stage_stream():
    torch = _torch()
    return torch.cuda.current_stream()


def convolve_bank(img, bank: TapBank, backend: str = "cuda", dtype=np.float32, plan=None,
                  stack_element_cap: int = DEFAULT_STACK_ELEMENT_CAP) -> ScaleStack:
    """Scale-space stack levels[i] = k_i * img, reflect boundary, float32 [L][H][W].

    Stage entry point for tests and diagnostics: it materialises every level,
    which the fused production path (`Detector.run`) never does.
    """
    img = _check_image(img)
    _check_backend(backend)
    n_levels = bank.ladder.n_levels
    if img.shape[0] * img.shape[1] * n_levels > stack_element_cap:
        raise ValueError(f"stack of {n_levels} x {img.shape} exceeds element cap {stack_element_cap}")
    if _check_dtype(dtype) == np.float64:
        return _convolve_bank_f64(img, bank)
    if isinstance(plan, _Engine):        # the reference idiom: plan=det.plan_for(img.shape)
        plan = plan.plan
    if plan is not None and tuple(plan.shape) != tuple(img.shape):
        raise ValueError(f"plan built for {plan.shape[1]}x{plan.shape[0]}, "
                         f"image is {img.shape[1]}x{img.shape[0]}")
    torch = _torch()
    lib = _lib.load()
    device = torch.cuda.current_device()
    own = plan is None
    if own:
        plan = _Plan(bank, img.shape, device, 1024)
    try:
        dev = torch.device("cuda", plan.device)
        H, W = img.shape
        d_img = torch.zeros((H, plan.pitch), dtype=torch.float32, device=dev)
        d_img[:, :W] = torch.from_numpy(np.ascontiguousarray(img, dtype=np.float32)).to(dev)
        work = torch.zeros(plan.workspace_bytes, dtype=torch.uint8, device=dev)
        out = torch.empty((n_levels, H, W), dtype=torch.float32, device=dev)
        st = torch.cuda.current_stream(dev)
        _lib.check(lib.dogblob_scale_space(plan.handle, d_img.data_ptr(), work.data_ptr(),
                                           out.data_ptr(), st.cuda_stream))
        levels = out.cpu().numpy()
    finally:
        if own:
            plan.close()
    return ScaleStack(levels=levels, sigmas=bank.ladder.sigmas)


def _convolve_bank_f64(img, bank: TapBank) -> ScaleStack:
    """float64 levels (convolve.py:76-77 with dtype=np.float64) on the FP64 pipe"""
    torch = _torch()
    lib = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    sig, rad, taps, offs = _f64_tables(bank)
    H, W = img.shape
    d_img = torch.from_numpy(np.ascontiguousarray(img, dtype=np.float64)).to(dev)
    d_tmp = torch.empty((H, W), dtype=torch.float64, device=dev)
    out = torch.empty((int(sig.size), H, W), dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev)
    _lib.check(lib.dogblob_scale_space_f64(H, W, int(sig.size), _lib.ptr(rad), _lib.ptr(taps), _lib.ptr(offs),
                                           d_img.data_ptr(), d_tmp.data_ptr(), out.data_ptr(), st.cuda_stream))
    return ScaleStack(levels=out.cpu().numpy(), sigmas=bank.ladder.sigmas)


def fused_dog(img, bank: TapBank) -> DoGStack:
    """DoG slices exactly as the production kernels compute them (row pass, then
    column pass with the subtraction fused), transposed back to [S][H][W]."""
    img = _check_image(img)
    torch = _torch()
    lib = _lib.load()
    plan = _Plan(bank, img.shape, torch.cuda.current_device(), 1024)
    try:
        dev = torch.device("cuda", plan.device)
        H, W = img.shape
        d_img = torch.zeros((H, plan.pitch), dtype=torch.float32, device=dev)
        d_img[:, :W] = torch.from_numpy(np.ascontiguousarray(img, dtype=np.float32)).to(dev)
        work = torch.zeros(plan.workspace_bytes, dtype=torch.uint8, device=dev)
        out = torch.empty((bank.ladder.n_levels - 1, H, W), dtype=torch.float32, device=dev)
        st = torch.cuda.current_stream(dev)
        _lib.check(lib.dogblob_dog(plan.handle, d_img.data_ptr(), work.data_ptr(), out.data_ptr(),
                                   st.cuda_stream))
        slices = out.cpu().numpy()
    finally:
        plan.close()
    return DoGStack(slices=slices, sigmas=bank.ladder.sigmas[:-1])


def dog_stack(stack: ScaleStack, ladder: SigmaLadder) -> DoGStack:
    """Adjacent differences scaled by the lower sigma of each pair (detector.py:117-126)."""
    if stack.n_levels != ladder.n_levels:
        raise ValueError(f"stack has {stack.n_levels} levels, ladder expects {ladder.n_levels}")
    torch = _torch()
    lib = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    L, H, W = stack.levels.shape
    if stack.levels.dtype == np.float64:
        d_lv = torch.from_numpy(np.ascontiguousarray(stack.levels)).to(dev)
        sig = np.ascontiguousarray(ladder.sigmas, dtype=np.float64)
        _lib.check(lib.dogblob_dog_inplace_f64(L, H, W, d_lv.data_ptr(), _lib.ptr(sig),
                                               torch.cuda.current_stream(dev).cuda_stream))
        return DoGStack(slices=d_lv[:L - 1].cpu().numpy(), sigmas=ladder.sigmas[:-1])
    if stack.levels.dtype != np.float32:
        raise ValueError("backend='cuda' differences float32 and float64 stacks only")
    d_lv = torch.from_numpy(np.ascontiguousarray(stack.levels)).to(dev)
    out = torch.empty((L - 1, H, W), dtype=torch.float32, device=dev)
    sig = np.ascontiguousarray(ladder.sigmas, dtype=np.float64)
    st = torch.cuda.current_stream(dev)
    _lib.check(lib.dogblob_dog_from_levels(L, H, W, d_lv.data_ptr(), _lib.ptr(sig), out.data_ptr(),
                                           st.cuda_stream))
    return DoGStack(slices=out.cpu().numpy(), sigmas=ladder.sigmas[:-1])


def _read_result(d_result, max_blobs):
    host = d_result.cpu().numpy()
    hdr = host[:_lib.RESULT_HEADER_BYTES].view(_lib.HEADER_DTYPE)[0]
    if int(hdr["flags"]) & _lib.FLAG_OVERFLOW:
        return hdr, None
    n = int(hdr["n_blobs"])
    body = host[_lib.RESULT_HEADER_BYTES:_lib.RESULT_HEADER_BYTES + n * _lib.BLOB_DTYPE.itemsize]
    return hdr, body.view(_lib.BLOB_DTYPE).copy()


def find_extrema(dog: DoGStack, threshold: float = 0.1, neighborhood: int = 3,
                 source_shape=None, params: DetectionParams | None = None,
                 max_blobs: int = DEFAULT_MAX_BLOBS) -> BlobSet:
    """Voxels equal to the max of their n^3 block and above threshold, plateaus
    coalesced to their centroid, sorted (detector.py:149-193)."""
    if neighborhood < 1 or neighborhood % 2 == 0:
        raise ValueError(f"neighborhood must be odd and >= 1, got {neighborhood}")
    data = np.asarray(dog.slices)
    if data.ndim != 3:
        raise ValueError(f"expected (n_slices, height, width) slices, got shape {data.shape}")
    if data.dtype not in (np.float32, np.float64):
        raise ValueError("backend='cuda' searches float32 and float64 stacks only")
    f64 = data.dtype == np.float64
    torch = _torch()
    lib = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    S, H, W = data.shape
    d_sl = torch.from_numpy(np.ascontiguousarray(data)).to(dev)
    sig = np.ascontiguousarray(dog.sigmas, dtype=np.float64)
    st = torch.cuda.current_stream(dev)
    while True:
        space = torch.zeros(int(lib.dogblob_blobspace_bytes(max_blobs)), dtype=torch.uint8, device=dev)
        res = torch.zeros(int(lib.dogblob_result_bytes_for(max_blobs)), dtype=torch.uint8, device=dev)
        if f64:      # the comparison `data > threshold` promotes to float64 (detector.py:166)
            _lib.check(lib.dogblob_extrema_f64(S, H, W, d_sl.data_ptr(), _lib.ptr(sig), float(threshold),
                                               int(neighborhood), max_blobs, space.data_ptr(), res.data_ptr(),
                                               st.cuda_stream))
        else:
            _lib.check(lib.dogblob_extrema(S, H, W, d_sl.data_ptr(), _lib.ptr(sig),
                                           float(np.float32(threshold)), int(neighborhood), max_blobs,
                                           space.data_ptr(), res.data_ptr(), st.cuda_stream))
        hdr, recs = _read_result(res, max_blobs)
        if recs is not None:
            break
        max_blobs *= 4
    shape = source_shape if source_shape is not None else (W, H)
    return BlobSet(records=recs, source_shape=shape, params=params or DetectionParams())


def disk_intersection_area(x1, y1, r1, x2, y2, r2) -> float:
    """Exact lens area of two disks (detector.py:196-209); scalar host helper."""
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


def normalized_overlap(b1: Blob, b2: Blob) -> float:
    """Lens area over the smaller disk's area (detector.py:212-218)."""
    rmin = min(b1.radius, b2.radius)
    if rmin <= 0:
        return 0.0
    return disk_intersection_area(b1.x, b1.y, b1.radius, b2.x, b2.y, b2.radius) / (
        math.pi * rmin * rmin)


def prune_overlaps(blobset: BlobSet, overlap_threshold: float = 0.5) -> BlobSet:
    """Coalesce blob pairs whose normalised overlap exceeds the threshold, in the
    reference's visiting order (detector.py:250-280), on the GPU."""
    if not 0.0 <= overlap_threshold <= 1.0:
        raise ValueError(f"overlap threshold must be in [0, 1], got {overlap_threshold}")
    torch = _torch()
    lib = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    recs = np.ascontiguousarray(blobset.records)
    n = len(recs)
    cap = max(n, 1)
    d_in = torch.from_numpy(recs.view(np.uint8).reshape(-1).copy()).to(dev) if n else None
    space = torch.zeros(int(lib.dogblob_blobspace_bytes(cap)), dtype=torch.uint8, device=dev)
    res = torch.zeros(int(lib.dogblob_result_bytes_for(cap)), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream(dev)
    _lib.check(lib.dogblob_prune(n, d_in.data_ptr() if n else None, float(overlap_threshold), cap,
                                 space.data_ptr(), res.data_ptr(), st.cuda_stream))
    hdr, out = _read_result(res, cap)
    if out is None:
        raise RuntimeError("prune result overflow")
    return BlobSet(records=out, source_shape=blobset.source_shape, params=blobset.params)
