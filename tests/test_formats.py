"""Wire/disk formats: bytes identical to the reference's writers, pinned by the
reference's own committed outputs (pkg/demos/output/03_blobs.json, 03_histogram.csv ->
tests/golden/ref_demo03_*) and by json.dump on the reference's document layout."""

import json
import struct
from pathlib import Path

import numpy as np
import pytest

import paper_2010_08486_b200 as P
from paper_2010_08486_b200 import formats as F

GOLD = Path(__file__).parent / "golden"


def test_blob_json_round_trip_is_byte_identical_to_the_reference_file():
    raw = (GOLD / "ref_demo03_blobs.json").read_bytes()
    bs = F.read_blobset_json(GOLD / "ref_demo03_blobs.json")
    assert len(bs) == 100 and bs.params.backend == "fft" and bs.params.n_bin == 25
    text = F.blobs_json_text(bs, "demo_scene") + "\n"
    assert text.encode() == raw


def test_write_read_files(tmp_path):
    bs = F.read_blobset_json(GOLD / "ref_demo03_blobs.json")
    F.write_blobset_json(tmp_path / "b.json", bs, image_name="demo_scene")
    assert (tmp_path / "b.json").read_bytes() == (GOLD / "ref_demo03_blobs.json").read_bytes()
    again = F.read_blobset_json(tmp_path / "b.json")
    assert again.blobs == bs.blobs and again.params == bs.params


def test_histogram_csv_is_byte_identical_to_the_reference_file(tmp_path):
    bs = F.read_blobset_json(GOLD / "ref_demo03_blobs.json")
    hist = P.histogram(bs, P.build_ladder(2.5, 15.0, 25))
    F.write_histogram_csv(tmp_path / "h.csv", hist)
    assert (tmp_path / "h.csv").read_bytes() == (GOLD / "ref_demo03_histogram.csv").read_bytes()
    d = F.histogram_to_doc(hist)
    assert set(d) == {"bin_center_px", "count", "volume_weight"}
    assert all(isinstance(c, int) for c in d["count"]) and sum(d["count"]) == 100


@pytest.mark.parametrize("n,floats", [(0, False), (1, False), (37, False), (12, True)])
def test_json_text_equals_json_dump_of_the_reference_document(n, floats):
    rng = np.random.default_rng(n + 5)
    blobs = []
    for _ in range(n):
        x = float(rng.uniform(0, 900)) if floats else int(rng.integers(0, 900))
        y = float(rng.uniform(0, 900)) if floats else int(rng.integers(0, 900))
        s = float(rng.choice([1.0, 2.5, 1e-7, 3.3333333333333335, 1e22]))
        blobs.append(P.Blob(x, y, s, s * 2 ** 0.5, float(np.float32(rng.uniform(0.1, 2.0))), bool(rng.integers(0, 2))))
    bs = P.BlobSet(blobs=blobs, source_shape=(900, 900), params=P.DetectionParams(backend="cuda", n_bin=7))
    doc = F.blobset_to_doc(bs, "frame 7 \"quoted\" é")
    want = {
        "image": "frame 7 \"quoted\" é",
        "params": bs.params.to_dict(),
        "blobs": [{"x": b.x, "y": b.y, "sigma": b.sigma, "radius": b.radius, "response": b.response,
                   "at_scale_boundary": b.at_scale_boundary} for b in bs.blobs],
    }
    assert doc == want
    assert F.blobs_json_text(bs, "frame 7 \"quoted\" é") == json.dumps(want, indent=2)
    extra = {"histogram": {"count": [1, 2]}, "timing_ms": {"convolve_ms": 0.25}}
    assert F.blobs_json_text(bs, "f", extra=extra) == json.dumps(
        {**want, "image": "f", **extra}, indent=2)
    assert F.blobset_from_doc(json.loads(F.blobs_json_text(bs))).blobs == tuple(
        P.Blob(int(b.x), int(b.y), b.sigma, b.radius, b.response, b.at_scale_boundary) for b in bs.blobs)


def test_raw_round_trip_and_layout(tmp_path):
    img = np.random.default_rng(3).random((37, 53), dtype=np.float32)
    F.write_raw(tmp_path / "a.raw", img)
    data = (tmp_path / "a.raw").read_bytes()
    assert struct.unpack_from("<II", data) == (53, 37)            # width first (images.py:65)
    assert len(data) == 8 + 4 * 37 * 53
    assert np.array_equal(np.frombuffer(data, "<f4", offset=8).reshape(37, 53), img)
    back = F.read_raw(tmp_path / "a.raw")
    assert back.dtype == np.float32 and np.array_equal(back, img)
    assert np.array_equal(F.raw_from_bytes(F.raw_to_bytes(img)), img)


def test_raw_errors_match_the_reference_messages():
    img = np.ones((4, 5), np.float32)
    good = F.raw_to_bytes(img)
    with pytest.raises(ValueError, match="truncated raw header"):
        F.raw_from_bytes(good[:5])
    with pytest.raises(ValueError, match="expected 88 bytes, found 87"):
        F.raw_from_bytes(good[:-1])
    with pytest.raises(ValueError, match="invalid raw dimensions 0x4"):
        F.raw_from_bytes(struct.pack("<II", 0, 4))
    bad = bytearray(good)
    bad[8:12] = struct.pack("<f", float("nan"))
    with pytest.raises(ValueError, match="NaN or Inf"):
        F.raw_from_bytes(bytes(bad))
    with pytest.raises(ValueError, match="single-channel 2-D"):
        F.raw_to_bytes(np.ones((2, 2, 3), np.float32))
    with pytest.raises(ValueError, match="empty image"):
        F.raw_to_bytes(np.ones((0, 3), np.float32))
