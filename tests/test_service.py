"""HTTP service around the detector: request validation, admission control and
the leased detector cache, exercised with a stub detector so that no GPU is needed; the
end-to-end equivalence with the offline detector is in test_gpu_pipeline.py::TestService."""

import http.client
import json
import threading
import time

import numpy as np
import pytest

import paper_2010_08486_b200 as P
from paper_2010_08486_b200 import formats as F
from paper_2010_08486_b200 import service as S


class StubDetector:
    """Stands in for the CUDA detector: one blob at the brightest pixel."""
    built = []

    def __init__(self, params, gate=None):
        self.params = params
        self.ladder = P.build_ladder(params.min_sigma, params.max_sigma, params.n_bin)
        self.closed = False
        self.gate = gate
        StubDetector.built.append(self)

    def run(self, img):
        if self.gate is not None:
            self.gate.wait(5)
        if self.closed:
            raise RuntimeError("detector used after close")
        a = img.numpy() if hasattr(img, "numpy") else np.asarray(img)
        y, x = np.unravel_index(int(np.argmax(a)), a.shape)
        s = float(self.ladder.sigmas[0])
        bs = P.BlobSet(blobs=[P.Blob(int(x), int(y), s, s * 2 ** 0.5, float(a[y, x]), True)],
                       source_shape=(a.shape[1], a.shape[0]), params=self.params)
        return P.DetectResult(blobs=bs, histogram=P.histogram(bs, self.ladder),
                              timings_ms={"preprocess_ms": 0.0, "convolve_ms": 0.12345, "extrema_ms": 0.5,
                                          "prune_ms": 0.25})

    def close(self):
        self.closed = True


@pytest.fixture
def server():
    made = []

    def start(**kw):
        kw.setdefault("detector_factory", StubDetector)
        srv = S.make_server(S.ServiceConfig(port=0, **kw))
        t = threading.Thread(target=srv.serve_forever, daemon=True)
        t.start()
        made.append(srv)
        return srv, srv.server_address[1]

    yield start
    for srv in made:
        srv.shutdown()
        srv.server_close()


def call(port, method, path, body=None, ctype="application/octet-stream"):
    c = http.client.HTTPConnection("127.0.0.1", port, timeout=10)
    c.request(method, path, body=body, headers={"Content-Type": ctype} if body is not None else {})
    r = c.getresponse()
    data = r.read()
    c.close()
    return r.status, data


def frame(h=12, w=20, peak=(3, 7)):
    img = np.zeros((h, w), np.float32)
    img[peak] = 0.75
    return img


class TestOverrides:
    def test_values_and_bounds(self):
        base = P.DetectionParams()
        p = S._apply_overrides(base, {"min_sigma": ["2.5"], "n_bin": ["7"], "prune": ["off"], "name": ["x"]})
        assert (p.min_sigma, p.n_bin, p.prune, p.backend) == (2.5, 7, False, "cuda")
        assert S._apply_overrides(base, {}) is base
        for q in ({"n_bin": ["0"]}, {"n_bin": ["257"]}, {"max_sigma": ["100.5"]}, {"min_sigma": ["0"]},
                  {"truncate": ["11"]}, {"overlap": ["1.5"]}, {"neighborhood": ["4"]}, {"saturation": ["0.5"]},
                  {"backend": ["fft"]}, {"n_bin": ["3.5"]}, {"preprocess": ["maybe"]}, {"bogus": ["1"]},
                  {"max_sigma": ["0.5"]}):
            with pytest.raises(S._HttpError) as e:
                S._apply_overrides(base, q)
            assert e.value.status == 400, q
        assert S._apply_overrides(base, {"saturation": ["0"], "overlap": ["1"], "neighborhood": ["5"],
                                         "backend": ["cuda"], "threshold": ["0"]}).neighborhood == 5

    def test_last_value_wins(self):
        assert S._apply_overrides(P.DetectionParams(), {"n_bin": ["3", "9"]}).n_bin == 9


class TestDetectorCache:
    def test_lru_eviction_closes_idle_detectors(self):
        StubDetector.built.clear()
        cache = S.DetectorCache(2, StubDetector)
        ps = [P.DetectionParams(n_bin=n) for n in (3, 4, 5)]
        a = cache.get(ps[0]); b = cache.get(ps[1])
        assert cache.get(ps[0]) is a and len(StubDetector.built) == 2
        c = cache.get(ps[2])                       # evicts ps[1], the least recently used
        assert b.closed and not a.closed and not c.closed and len(cache) == 2 and cache.closed == 1
        assert cache.get(ps[1]) is not b           # rebuilt on demand
        cache.clear()
        assert all(d.closed for d in StubDetector.built)

    def test_busy_detector_is_closed_when_its_last_lease_ends(self):
        cache = S.DetectorCache(1, StubDetector)
        p1, p2 = P.DetectionParams(n_bin=3), P.DetectionParams(n_bin=4)
        with cache.lease(p1) as d1:
            with cache.lease(p1) as again:
                assert again is d1
                cache.get(p2)                       # evicts p1 while two leases are open
                assert not d1.closed
            assert not d1.closed
            d1.run(frame())                         # still usable
        assert d1.closed

    def test_single_flight_build(self):
        built = []
        gate = threading.Event()

        def slow_factory(params):
            gate.wait(5)
            built.append(params)
            return StubDetector(params)

        cache = S.DetectorCache(2, slow_factory)
        out = []
        ts = [threading.Thread(target=lambda: out.append(cache.get(P.DetectionParams()))) for _ in range(6)]
        [t.start() for t in ts]
        time.sleep(0.1)
        gate.set()
        [t.join() for t in ts]
        assert len(built) == 1 and all(o is out[0] for o in out)

    def test_failed_build_is_not_cached(self):
        calls = []

        def factory(params):
            calls.append(1)
            if len(calls) == 1:
                raise ValueError("max_sigma must exceed min_sigma")
            return StubDetector(params)

        cache = S.DetectorCache(2, factory)
        with pytest.raises(ValueError):
            cache.get(P.DetectionParams())
        assert cache.get(P.DetectionParams()) is not None and len(calls) == 2


class TestHttp:
    def test_health_and_unknown_paths(self, server):
        _, port = server(workers=2)
        st, data = call(port, "GET", "/healthz")
        doc = json.loads(data)
        assert st == 200 and doc["status"] == "ok" and doc["workers"] == 2 and doc["requests_served"] == 0
        assert doc["params"] == P.DetectionParams().to_dict()
        assert call(port, "GET", "/nope")[0] == 404
        assert call(port, "POST", "/nope", b"x")[0] == 404

    def test_detect_matches_the_reference_document_layout(self, server):
        srv, port = server()
        st, data = call(port, "POST", "/detect?name=f17&min_sigma=2&max_sigma=6&n_bin=4", F.raw_to_bytes(frame()))
        assert st == 200
        doc = json.loads(data)
        assert list(doc) == ["image", "params", "blobs", "histogram", "timing_ms"]
        assert doc["image"] == "f17" and doc["params"]["n_bin"] == 4 and doc["params"]["backend"] == "cuda"
        assert doc["blobs"] == [{"x": 7, "y": 3, "sigma": 2.0, "radius": 2.0 * 2 ** 0.5, "response": 0.75,
                                 "at_scale_boundary": True}]
        assert doc["timing_ms"] == {"preprocess_ms": 0.0, "convolve_ms": 0.123, "extrema_ms": 0.5, "prune_ms": 0.25}
        assert sum(doc["histogram"]["count"]) == 1 and len(doc["histogram"]["bin_center_px"]) == 5
        assert data == (json.dumps(doc, indent=2) + "\n").encode()      # same text as json.dumps(indent=2)
        assert json.loads(call(port, "GET", "/healthz")[1])["requests_served"] == 1

    def test_bad_requests(self, server):
        _, port = server(max_request_bytes=4096)
        raw = F.raw_to_bytes(frame())
        assert call(port, "POST", "/detect", b"")[0] == 400
        assert call(port, "POST", "/detect", raw[:-3])[0] == 400
        assert call(port, "POST", "/detect", raw, ctype="text/plain")[0] == 400
        assert call(port, "POST", "/detect?n_bin=999", raw)[0] == 400
        assert call(port, "POST", "/detect?backend=fft", raw)[0] == 400
        st, data = call(port, "POST", "/detect", F.raw_to_bytes(np.zeros((40, 40), np.float32)))
        assert st == 413 and "exceeds limit" in json.loads(data)["error"]
        nan = frame(); nan[0, 0] = np.nan
        st, data = call(port, "POST", "/detect", b"\x14\x00\x00\x00\x0c\x00\x00\x00" + nan.tobytes())
        assert st == 400 and "NaN or Inf" in json.loads(data)["error"]

    def test_queue_full_is_503(self, server):
        gate = threading.Event()
        srv, port = server(workers=1, backlog=0, detector_factory=lambda p: StubDetector(p, gate))
        raw = F.raw_to_bytes(frame())
        first = []
        t = threading.Thread(target=lambda: first.append(call(port, "POST", "/detect", raw)))
        t.start()
        for _ in range(100):                       # wait until the first request holds the worker
            if not srv.state.compute.acquire(blocking=False):
                break
            srv.state.compute.release()
            time.sleep(0.01)
        st, data = call(port, "POST", "/detect", raw)
        assert st == 503 and "queue full" in json.loads(data)["error"]
        assert call(port, "GET", "/healthz")[0] == 200            # health stays outside the pool
        gate.set()
        t.join()
        assert first[0][0] == 200

    def test_detect_batch(self, server):
        _, port = server()
        frames = [frame(peak=(1 + i, 2 + i)) for i in range(3)]
        body = b"".join(F.raw_to_bytes(f) for f in frames)
        st, data = call(port, "POST", "/detect_batch?name=b", body)
        assert st == 200
        doc = json.loads(data)
        assert [f["image"] for f in doc["frames"]] == ["b[0]", "b[1]", "b[2]"]
        assert [(f["blobs"][0]["x"], f["blobs"][0]["y"]) for f in doc["frames"]] == [(2, 1), (3, 2), (4, 3)]
        assert data == (json.dumps(doc, indent=2) + "\n").encode()
        assert call(port, "POST", "/detect_batch", body[:-1])[0] == 400
        assert call(port, "POST", "/detect_batch", body, ctype="image/png")[0] == 400
        mixed = body + F.raw_to_bytes(frame(5, 6, (1, 1)))          # ragged shapes: frame by frame
        assert len(json.loads(call(port, "POST", "/detect_batch", mixed)[1])["frames"]) == 4
        assert json.loads(call(port, "GET", "/healthz")[1])["frames_served"] == 7
