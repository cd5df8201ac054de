"""Per-image analysis over HTTP with the CUDA backend.

Same wire contract as the reference service (`service.py:199-260`): `POST /detect` takes image
bytes (raw float format with `Content-Type: application/octet-stream`; PNG / TIFF when imageio
is installed), query parameters override detector settings within the reference's bounds, and the
answer is the blob set + radius histogram + per-stage timings as `json.dumps(doc, indent=2)`;
`GET /healthz` answers outside the worker pool; 400 / 404 / 413 / 503 as in the reference.

What is different, because the detector now lives on a GPU:
  * `backend` accepts `"cuda"` only (`_PARAM_SPECS`, reference `service.py:57`);
  * a raw body is decoded straight into a pinned staging buffer owned by the worker slot
    (`formats.raw_into_pinned`), so the H2D copy starts from the request bytes' only copy;
  * `DetectorCache` hands out LEASES: an evicted detector frees its device memory
    (`Detector.close`) only once the last request using it has finished;
  * `POST /detect_batch` takes several raw frames back to back in one body and runs them
    through `Detector.run_batch` (H2D / kernels / D2H of consecutive frames overlap);
  * the JSON text is assembled from the record array (`formats.blobs_json_text`).
"""

from __future__ import annotations

import io
import json
import struct
import threading
import time
from collections import OrderedDict
from contextlib import contextmanager
from dataclasses import dataclass, field, replace
from http.server import BaseHTTPRequestHandler, ThreadingHTTPServer
from urllib.parse import parse_qs, urlparse

import numpy as np

from . import formats
from .detector import DetectionParams, Detector

__all__ = ["ServiceConfig", "DetectorCache", "AnalysisServer", "make_server", "serve"]


_TRUE, _FALSE = ("1", "true", "yes", "on"), ("0", "false", "no", "off")


def _flag(text: str) -> bool:
    t = text.lower()
    if t in _TRUE or t in _FALSE:
        return t in _TRUE
    raise ValueError(f"not a boolean: {text!r}")


@dataclass(frozen=True)
class _Range:
    """Closed interval with optionally open ends; the reference's per-request bounds
    (service.py:49-62) written as data."""
    cast: type
    lo: float = float("-inf")
    hi: float = float("inf")
    open_lo: bool = False
    open_hi: bool = False
    odd: bool = False

    def parse(self, text: str):
        return self.cast(text)

    def accepts(self, v) -> bool:
        if v < self.lo or (self.open_lo and v == self.lo):
            return False
        if v > self.hi or (self.open_hi and v == self.hi):
            return False
        return not self.odd or v % 2 == 1


@dataclass(frozen=True)
class _Choice:
    options: tuple

    def parse(self, text: str):
        return text

    def accepts(self, v) -> bool:
        return v in self.options


@dataclass(frozen=True)
class _Switch:
    def parse(self, text: str):
        return _flag(text)

    def accepts(self, v) -> bool:
        return True


# query parameters a request may override (backend: only the CUDA implementation lives here)
_PARAM_SPECS = {
    "min_sigma": _Range(float, 0, 100, open_lo=True),
    "max_sigma": _Range(float, 0, 100, open_lo=True),
    "n_bin": _Range(int, 1, 256),
    "truncate": _Range(float, 0, 10, open_lo=True),
    "threshold": _Range(float, 0, 1e6),
    "overlap": _Range(float, 0, 1),
    "neighborhood": _Range(int, 1, odd=True),
    "backend": _Choice(("cuda",)),
    "preprocess": _Switch(),
    "smooth_sigma": _Range(float, 0, 50),
    "saturation": _Range(float, 0, 0.5, open_hi=True),
    "prune": _Switch(),
}
_IGNORED_QUERY_KEYS = frozenset({"name"})


@dataclass(frozen=True)
class ServiceConfig:
    host: str = "127.0.0.1"
    port: int = 8750
    params: DetectionParams = DetectionParams()
    max_request_bytes: int = 16 * 1024 * 1024
    request_timeout_s: float = 120.0
    workers: int = 1
    backlog: int = 4
    detector_cache_size: int = 4
    device: int | None = None          # CUDA device of every detector this service builds
    max_batch_frames: int = 64         # frames accepted by one POST /detect_batch
    detector_factory: object = field(default=None, compare=False)   # tests inject a stub


class DetectorCache:
    """LRU of detectors keyed by parameter set, single-flight builds, leased entries.

    `lease(params)` is a context manager; while at least one lease is open the detector is
    never closed.  Eviction (capacity exceeded) closes an idle detector immediately and a busy
    one when its last lease ends, so the device memory of cold parameter sets is returned."""

    def __init__(self, capacity: int = 4, factory=None):
        self.capacity = max(1, int(capacity))
        self._factory = factory or Detector
        self._cache: OrderedDict = OrderedDict()      # key -> entry
        self._lock = threading.Lock()
        self._building: dict = {}
        self.closed = 0                               # detectors released so far (healthz)

    class _Entry:
        __slots__ = ("det", "leases", "evicted")

        def __init__(self, det):
            self.det, self.leases, self.evicted = det, 0, False

    @staticmethod
    def key_of(params: DetectionParams) -> tuple:
        return tuple(sorted(params.to_dict().items()))

    def _acquire(self, params: DetectionParams):
        key = self.key_of(params)
        while True:
            with self._lock:
                entry = self._cache.get(key)
                if entry is not None:
                    self._cache.move_to_end(key)
                    entry.leases += 1
                    return entry
                pending = self._building.get(key)
                if pending is None:
                    self._building[key] = threading.Event()
                    break
            pending.wait()
        try:
            det = self._factory(params)
        except Exception:
            with self._lock:
                self._building.pop(key).set()
            raise
        to_close = []
        with self._lock:
            entry = self._Entry(det)
            entry.leases = 1
            self._cache[key] = entry
            while len(self._cache) > self.capacity:
                _, old = self._cache.popitem(last=False)
                old.evicted = True
                if old.leases == 0:
                    to_close.append(old)
            self._building.pop(key).set()
        for old in to_close:
            self._close(old)
        return entry

    def _close(self, entry) -> None:
        close = getattr(entry.det, "close", None)
        if close is not None:
            close()
        with self._lock:
            self.closed += 1

    def _release(self, entry) -> None:
        with self._lock:
            entry.leases -= 1
            last = entry.evicted and entry.leases == 0
        if last:
            self._close(entry)

    @contextmanager
    def lease(self, params: DetectionParams):
        entry = self._acquire(params)
        try:
            yield entry.det
        finally:
            self._release(entry)

    def get(self, params: DetectionParams):
        """Reference-compatible accessor (service.py:86-111): the detector without a lease."""
        with self.lease(params) as det:
            return det

    def __len__(self) -> int:
        with self._lock:
            return len(self._cache)

    def clear(self) -> None:
        with self._lock:
            entries = list(self._cache.values())
            self._cache.clear()
            for e in entries:
                e.evicted = True
        for e in entries:
            if e.leases == 0:
                self._close(e)


class _State:
    def __init__(self, config: ServiceConfig):
        self.config = config
        factory = config.detector_factory
        if factory is None:
            def factory(params, _cfg=config):
                return Detector(params, device=_cfg.device, slots=max(2, _cfg.workers))
        self.cache = DetectorCache(config.detector_cache_size, factory)
        self.started = time.monotonic()
        self.requests_served = 0
        self.frames_served = 0
        self.counter_lock = threading.Lock()
        # admission: workers computing + backlog waiting; beyond that, 503
        self.admission = threading.BoundedSemaphore(config.workers + config.backlog)
        self.compute = threading.BoundedSemaphore(config.workers)
        self._staging = []                            # idle pinned staging tensors
        self._staging_lock = threading.Lock()

    @contextmanager
    def staging(self, n_floats: int):
        """A pinned float32 buffer of at least n_floats for the duration of one request;
        None when pinned memory is unavailable (no CUDA runtime: stub detectors in tests)."""
        buf = None
        with self._staging_lock:
            for i, b in enumerate(self._staging):
                if b.numel() >= n_floats:
                    buf = self._staging.pop(i)
                    break
        if buf is None:
            try:
                import torch
                buf = torch.empty(max(n_floats, 1 << 20), dtype=torch.float32).pin_memory()
            except Exception:
                buf = None
        try:
            yield buf
        finally:
            if buf is not None:
                with self._staging_lock:
                    if len(self._staging) < self.config.workers + 1:
                        self._staging.append(buf)


class _HttpError(Exception):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status
        self.message = message


_INT_SCALE = {np.dtype(np.uint8): 255.0, np.dtype(np.uint16): 65535.0}


def _media_type(header: str) -> str:
    return (header or "").partition(";")[0].strip().lower()


def _decode_file_image(body) -> np.ndarray:
    """8/16-bit single-channel PNG or TIFF scaled by the dtype maximum (images.py:70-98)."""
    try:
        import imageio.v3 as iio
    except ImportError:
        raise ValueError("PNG/TIFF decoding needs imageio; send the raw float format "
                         "as application/octet-stream") from None
    pixels = iio.imread(io.BytesIO(body))
    if pixels.ndim != 2:
        raise ValueError(f"multi-channel image (shape {pixels.shape})")
    scale = _INT_SCALE.get(pixels.dtype)
    if scale is None:
        raise ValueError(f"unsupported bit depth {pixels.dtype}")
    return pixels.astype(np.float32) / scale


def _decode_image(body: bytes, content_type: str, staging=None):
    """Request body -> image the detector accepts (a pinned tensor for raw frames)."""
    kind = _media_type(content_type)
    try:
        if kind == "application/octet-stream":
            if staging is None:
                return formats.raw_from_bytes(body, label="request body")
            return formats.raw_into_pinned(body, label="request body", out=staging)
        if kind in ("", "image/png", "image/tiff", "image/tif"):
            return _decode_file_image(body)
        raise ValueError(f"unsupported content type {kind!r}")
    except Exception as exc:
        raise _HttpError(400, f"cannot decode image: {exc}") from exc


def _split_frames(body: bytes, limit: int) -> list:
    """A /detect_batch body is raw frames back to back, each with its own 8-byte header."""
    frames, pos = [], 0
    while pos < len(body):
        if len(body) - pos < formats.RAW_HEADER_LEN:
            raise _HttpError(400, f"cannot decode image: frame {len(frames)}: truncated raw header")
        w, h = struct.unpack_from("<II", body, pos)
        size = formats.RAW_HEADER_LEN + 4 * w * h
        if w < 1 or h < 1 or pos + size > len(body):
            raise _HttpError(400, f"cannot decode image: frame {len(frames)}: bad raw frame "
                                  f"({w}x{h}, {len(body) - pos} bytes left)")
        frames.append(memoryview(body)[pos:pos + size])
        pos += size
        if len(frames) > limit:
            raise _HttpError(413, f"more than {limit} frames in one batch")
    if not frames:
        raise _HttpError(400, "empty request body")
    return frames


def _apply_overrides(params: DetectionParams, query: dict) -> DetectionParams:
    """Detector parameters of one request: service defaults + validated query overrides."""
    changed = {}
    for key in query.keys() - _IGNORED_QUERY_KEYS:
        spec = _PARAM_SPECS.get(key)
        if spec is None:
            raise _HttpError(400, f"unknown parameter {key!r}")
        text = query[key][-1]
        try:
            value = spec.parse(text)
        except ValueError:
            raise _HttpError(400, f"bad value for {key!r}: {text!r}") from None
        if not spec.accepts(value):
            raise _HttpError(400, f"value out of bounds for {key!r}: {value!r}")
        changed[key] = value
    if changed:
        params = replace(params, **changed)
        if not params.min_sigma < params.max_sigma:
            raise _HttpError(400, "max_sigma must exceed min_sigma")
    return params


def _result_text(result, name: str) -> str:
    extra = {"histogram": formats.histogram_to_doc(result.histogram),
             "timing_ms": {k: round(v, 3) for k, v in result.timings_ms.items()}}
    return formats.blobs_json_text(result.blobs, name, extra=extra)


class _Handler(BaseHTTPRequestHandler):
    protocol_version = "HTTP/1.1"
    disable_nagle_algorithm = True   # replies are single small writes: no 40 ms delayed-ACK stalls
    state: _State   # bound by make_server

    def log_message(self, fmt, *args):   # requests are not logged
        return

    # -- replies ------------------------------------------------------------------
    def _reply(self, status: int, text: str) -> None:
        data = (text + "\n").encode()
        self.send_response(status)
        self.send_header("Content-Type", "application/json")
        self.send_header("Content-Length", str(len(data)))
        if status >= 400:                    # unread body bytes may follow: drop the socket
            self.send_header("Connection", "close")
            self.close_connection = True
        self.end_headers()
        self.wfile.write(data)

    def _reply_doc(self, status: int, doc: dict) -> None:
        self._reply(status, json.dumps(doc, indent=2))

    def _fail(self, status: int, message: str) -> None:
        self._reply_doc(status, {"error": message})

    # -- GET ----------------------------------------------------------------------
    def do_GET(self):
        path = urlparse(self.path).path
        if path not in ("/healthz", "/health"):
            return self._fail(404, f"no such path {path!r}")
        st = self.state
        with st.counter_lock:
            requests, frames = st.requests_served, st.frames_served
        self._reply_doc(200, {
            "status": "ok",
            "params": st.config.params.to_dict(),
            "uptime_s": time.monotonic() - st.started,
            "requests_served": requests,
            "workers": st.config.workers,
            "frames_served": frames,
            "detectors_cached": len(st.cache),
            "detectors_released": st.cache.closed,
        })

    # -- POST ---------------------------------------------------------------------
    _ROUTES = {"/detect": "_detect_one", "/detect_batch": "_detect_many"}

    def do_POST(self):
        url = urlparse(self.path)
        route = self._ROUTES.get(url.path)
        if route is None:
            return self._fail(404, f"no such path {url.path!r}")
        st = self.state
        try:
            size = int(self.headers.get("Content-Length", "0"))
            cap = st.config.max_request_bytes
            if route == "_detect_many":
                cap *= st.config.max_batch_frames
            if size > cap:
                raise _HttpError(413, f"payload {size} exceeds limit {cap}")
            if size <= 0:
                raise _HttpError(400, "empty request body")
            with self._admitted(st):
                body = self.rfile.read(size)
                query = parse_qs(url.query)
                params = _apply_overrides(st.config.params, query)
                label = query.get("name", ["request"])[-1]
                with self._worker(st):
                    text, n_frames = getattr(self, route)(st, body, params, label)
            with st.counter_lock:
                st.requests_served += 1
                st.frames_served += n_frames
            self._reply(200, text)
        except _HttpError as err:
            self._fail(err.status, err.message)
        except ValueError as exc:            # detector argument errors (ladder, image shape, ...)
            self._fail(400, str(exc))
        except Exception as exc:             # never drop the connection silently
            self._fail(500, f"internal error: {exc}")

    @staticmethod
    @contextmanager
    def _admitted(st: _State):
        """workers + backlog requests may be inside; the next one is turned away at once"""
        if not st.admission.acquire(blocking=False):
            raise _HttpError(503, "detection queue full, retry later")
        try:
            yield
        finally:
            st.admission.release()

    @staticmethod
    @contextmanager
    def _worker(st: _State):
        """at most `workers` requests decode and compute; the others hold raw bytes only"""
        if not st.compute.acquire(timeout=st.config.request_timeout_s):
            raise _HttpError(503, "timed out waiting for a worker")
        try:
            yield
        finally:
            st.compute.release()

    def _detect_one(self, st: _State, body: bytes, params: DetectionParams, label: str):
        n_floats = max(0, (len(body) - formats.RAW_HEADER_LEN) // 4)
        with st.staging(n_floats) as pinned:
            image = _decode_image(body, self.headers.get("Content-Type", ""), pinned)
            with st.cache.lease(params) as detector:
                result = detector.run(image)
        return _result_text(result, label), 1

    def _detect_many(self, st: _State, body: bytes, params: DetectionParams, label: str):
        if _media_type(self.headers.get("Content-Type", "")) != "application/octet-stream":
            raise _HttpError(400, "cannot decode image: /detect_batch takes raw frames "
                                  "(application/octet-stream)")
        try:
            images = [formats.raw_from_bytes(v, label=f"frame {i}")
                      for i, v in enumerate(_split_frames(body, st.config.max_batch_frames))]
        except ValueError as exc:
            raise _HttpError(400, f"cannot decode image: {exc}") from exc
        with st.cache.lease(params) as detector:
            same_shape = len({im.shape for im in images}) == 1
            if same_shape and hasattr(detector, "run_batch"):
                results = detector.run_batch(images, timings=True)
            else:
                results = [detector.run(im) for im in images]
        docs = [_result_text(r, f"{label}[{i}]").replace("\n", "\n    ") for i, r in enumerate(results)]
        return '{\n  "frames": [\n    ' + ",\n    ".join(docs) + "\n  ]\n}", len(results)


class AnalysisServer(ThreadingHTTPServer):
    daemon_threads = True

    def server_close(self):
        super().server_close()
        state = getattr(self, "state", None)
        if state is not None:
            state.cache.clear()       # return the device memory of every cached detector


def make_server(config: ServiceConfig) -> AnalysisServer:
    """Build (but do not start) the HTTP server; call serve_forever() to run."""
    state = _State(config)
    handler = type("BoundHandler", (_Handler,), {"state": state})
    server = AnalysisServer((config.host, config.port), handler)
    server.state = state
    return server


def serve(config: ServiceConfig) -> None:
    server = make_server(config)
    host, port = server.server_address[:2]
    print(f"dogblob (cuda) service listening on {host}:{port}")
    try:
        server.serve_forever()
    except KeyboardInterrupt:
        pass
    finally:
        server.server_close()
