"""Wire and disk formats around the hot path, unchanged from the reference.

  raw frames   `<u32 width><u32 height><f32 * w * h>` little endian
               (reference images.py:45-68: raw_from_bytes / read_raw / write_raw)
  blob JSON    {"image", "params", "blobs": [{x, y, sigma, radius, response,
               at_scale_boundary}]}, json.dump(indent=2) + "\n" (detector.py:394-439)
  histogram    CSV `bin_center_px,count,volume_weight` with repr() floats, and the
               JSON form used by the service (detector.py:441-452)

Two things differ from the reference, neither visible in the bytes:
  * a raw frame is decoded straight into PINNED host memory (`raw_into_pinned`,
    `read_raw_pinned`), so `Detector.run` can start its H2D copy without another pass
    over the pixels;
  * the writers are fed from the record ARRAY that comes back from the GPU
    (`BlobSet.records`), not from per-blob Python objects: `blobs_json_text` emits exactly
    the text `json.dump(blobset_to_doc(...), indent=2)` would.
"""

from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np

from . import _lib

RAW_HEADER_LEN = 8   # u32 width + u32 height, little-endian (images.py:17)

__all__ = [
    "RAW_HEADER_LEN", "raw_from_bytes", "raw_into_pinned", "read_raw", "read_raw_pinned", "write_raw",
    "raw_to_bytes", "blobset_to_doc", "blobset_from_doc", "blobs_json_text", "write_blobset_json",
    "read_blobset_json", "histogram_to_doc", "histogram_csv_text", "write_histogram_csv",
]


# ---------------------------------------------------------------------------------
# raw float frames
# ---------------------------------------------------------------------------------
def _raw_shape(data, label: str) -> tuple[int, int]:
    """(height, width) after the reference's header checks (images.py:45-55)."""
    if len(data) < RAW_HEADER_LEN:
        raise ValueError(f"{label}: truncated raw header")
    width, height = struct.unpack_from("<II", data, 0)
    expected = RAW_HEADER_LEN + 4 * width * height
    if width < 1 or height < 1:
        raise ValueError(f"{label}: invalid raw dimensions {width}x{height}")
    if len(data) != expected:
        raise ValueError(f"{label}: expected {expected} bytes, found {len(data)}")
    return height, width


def _check_finite(arr: np.ndarray) -> None:
    if not np.isfinite(arr).all():
        raise ValueError("image contains NaN or Inf values")    # images.py:40-41


def raw_from_bytes(data, label: str = "raw image") -> np.ndarray:
    """Decode the raw float format into a float32 [height, width] array (images.py:45-57)."""
    h, w = _raw_shape(data, label)
    img = np.frombuffer(data, dtype="<f4", offset=RAW_HEADER_LEN).reshape(h, w)
    _check_finite(img)
    return img.astype(np.float32, copy=False)


def raw_into_pinned(data, label: str = "raw image", out=None):
    """Decode a raw frame into pinned host memory; returns a float32 torch tensor [h, w].

    `out` may be a pinned float32 tensor of at least h*w elements to re-use (a staging
    ring); the pixels are copied exactly once, from the request / file buffer into it."""
    import torch
    h, w = _raw_shape(data, label)
    src = np.frombuffer(data, dtype="<f4", offset=RAW_HEADER_LEN).reshape(h, w)
    _check_finite(src)
    if out is None:
        out = torch.empty((h, w), dtype=torch.float32).pin_memory()
        dst = out
    else:
        if out.dtype != torch.float32 or out.numel() < h * w or not out.is_contiguous():
            raise ValueError("staging tensor must be contiguous float32 with at least h*w elements")
        dst = out.view(-1)[: h * w].view(h, w)
    np.copyto(dst.numpy(), src)
    return dst


def read_raw(path) -> np.ndarray:
    return raw_from_bytes(Path(path).read_bytes(), label=str(path))


def read_raw_pinned(path, out=None):
    """File -> pinned float32 tensor: header read first, then the pixels are read by the OS
    directly into the pinned pages (no intermediate bytes object)."""
    import torch
    p = Path(path)
    size = p.stat().st_size
    with open(p, "rb") as f:
        head = f.read(RAW_HEADER_LEN)
        if len(head) < RAW_HEADER_LEN:
            raise ValueError(f"{path}: truncated raw header")
        width, height = struct.unpack("<II", head)
        expected = RAW_HEADER_LEN + 4 * width * height
        if width < 1 or height < 1:
            raise ValueError(f"{path}: invalid raw dimensions {width}x{height}")
        if size != expected:
            raise ValueError(f"{path}: expected {expected} bytes, found {size}")
        if out is None:
            out = torch.empty((height, width), dtype=torch.float32).pin_memory()
            dst = out
        else:
            if out.dtype != torch.float32 or out.numel() < height * width or not out.is_contiguous():
                raise ValueError("staging tensor must be contiguous float32 with at least h*w elements")
            dst = out.view(-1)[: height * width].view(height, width)
        view = dst.numpy().reshape(-1).view(np.uint8)
        got = f.readinto(memoryview(view))
        if got != view.size:
            raise ValueError(f"{path}: expected {expected} bytes, found {RAW_HEADER_LEN + got}")
    _check_finite(dst.numpy())
    return dst


def raw_to_bytes(img) -> bytes:
    arr = np.asarray(img)
    if arr.ndim != 2:
        raise ValueError(f"expected a single-channel 2-D image, got shape {arr.shape}")
    if arr.size == 0:
        raise ValueError("empty image")
    arr = np.ascontiguousarray(arr, dtype="<f4")
    _check_finite(arr)
    h, w = arr.shape
    return struct.pack("<II", w, h) + arr.tobytes()


def write_raw(path, img) -> None:
    with open(path, "wb") as f:
        f.write(raw_to_bytes(img))


# ---------------------------------------------------------------------------------
# blob sets
# ---------------------------------------------------------------------------------
def _columns(blobset):
    """Python scalars per column, straight from the record array (no Blob objects)."""
    r = blobset.records
    integral = bool(np.all(r["x"] == np.rint(r["x"])) and np.all(r["y"] == np.rint(r["y"])))
    xs = r["x"].astype(np.int64).tolist() if integral else r["x"].tolist()
    ys = r["y"].astype(np.int64).tolist() if integral else r["y"].tolist()
    edge = ((r["flags"] & _lib.BLOB_SCALE_EDGE) != 0).tolist()
    return xs, ys, r["sigma"].tolist(), r["radius"].tolist(), r["response"].tolist(), edge


def blobset_to_doc(blobset, image_name: str = "image") -> dict:
    """detector.py:397-412."""
    xs, ys, sg, rad, resp, edge = _columns(blobset)
    return {
        "image": image_name,
        "params": blobset.params.to_dict(),
        "blobs": [{"x": x, "y": y, "sigma": s, "radius": r, "response": v, "at_scale_boundary": e}
                  for x, y, s, r, v, e in zip(xs, ys, sg, rad, resp, edge)],
    }


def blobs_json_text(blobset, image_name: str = "image", extra: dict | None = None) -> str:
    """The text `json.dumps(doc, indent=2)` yields for blobset_to_doc(...) (+ `extra` top-level
    keys, e.g. the service's histogram and timing), assembled from the columns."""
    head = json.dumps({"image": image_name, "params": blobset.params.to_dict()}, indent=2)
    xs, ys, sg, rad, resp, edge = _columns(blobset)
    fr = float.__repr__
    if xs:
        items = ",\n".join(
            '    {\n      "x": %s,\n      "y": %s,\n      "sigma": %s,\n      "radius": %s,\n'
            '      "response": %s,\n      "at_scale_boundary": %s\n    }'
            % (_num(x), _num(y), fr(s), fr(r), fr(v), "true" if e else "false")
            for x, y, s, r, v, e in zip(xs, ys, sg, rad, resp, edge))
        blobs = '  "blobs": [\n' + items + "\n  ]"
    else:
        blobs = '  "blobs": []'
    text = head[:-2] + ",\n" + blobs          # head ends with "\n}"
    for key, value in (extra or {}).items():
        body = json.dumps({key: value}, indent=2)
        text += ",\n" + body[2:-2]            # strip "{\n" and "\n}"
    return text + "\n}"


def _num(v) -> str:
    return repr(v) if isinstance(v, int) else float.__repr__(v)


def blobset_from_doc(doc: dict):
    """detector.py:415-429."""
    from .detector import Blob, BlobSet, DetectionParams
    params = DetectionParams(**doc.get("params", {}))
    blobs = tuple(
        Blob(x=int(b["x"]), y=int(b["y"]), sigma=float(b["sigma"]), radius=float(b["radius"]),
             response=float(b["response"]), at_scale_boundary=bool(b.get("at_scale_boundary", False)))
        for b in doc.get("blobs", []))
    shape = tuple(doc.get("source_shape", (0, 0)))
    return BlobSet(blobs=blobs, source_shape=shape, params=params)


def write_blobset_json(path, blobset, image_name: str = "image") -> None:
    """Byte-identical to the reference's json.dump(..., indent=2) + newline (detector.py:432-435)."""
    with open(path, "w") as f:
        f.write(blobs_json_text(blobset, image_name))
        f.write("\n")


def read_blobset_json(path):
    with open(path) as f:
        return blobset_from_doc(json.load(f))


# ---------------------------------------------------------------------------------
# histogram
# ---------------------------------------------------------------------------------
def histogram_to_doc(hist) -> dict:
    """detector.py:441-446."""
    return {
        "bin_center_px": np.asarray(hist.bin_centers, dtype=np.float64).tolist(),
        "count": np.asarray(hist.counts, dtype=np.int64).tolist(),
        "volume_weight": np.asarray(hist.volume_weights, dtype=np.float64).tolist(),
    }


def histogram_csv_text(hist) -> str:
    d = histogram_to_doc(hist)
    rows = ["bin_center_px,count,volume_weight\n"]
    rows += [f"{c!r},{n},{v!r}\n" for c, n, v in zip(d["bin_center_px"], d["count"], d["volume_weight"])]
    return "".join(rows)


def write_histogram_csv(path, hist) -> None:
    """detector.py:449-453."""
    with open(path, "w") as f:
        f.write(histogram_csv_text(hist))
