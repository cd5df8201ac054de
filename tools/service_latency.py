#!/usr/bin/env python
"""Service latency: POST /detect round trips of a 1000x1000 raw frame through the
HTTP service on localhost, parameters of the reference's recorded figure (sigma 2.5..9, n_bin 13,
preprocessing on: 1827 ms p50 on its desk CPU, pkg/test_output.txt:46), plus the C2 parameters."""
import http.client
import json
import socket
import sys
import threading
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2010_08486_b200 as P  # noqa: E402
from paper_2010_08486_b200 import formats as F, service as S, synth  # noqa: E402


def measure(params, frame, n=60, warm=10):
    srv = S.make_server(S.ServiceConfig(port=0, params=params, workers=1))
    threading.Thread(target=srv.serve_forever, daemon=True).start()
    port = srv.server_address[1]
    body = F.raw_to_bytes(frame)
    conn = http.client.HTTPConnection("127.0.0.1", port, timeout=60)
    conn.connect()
    conn.sock.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)   # headers and body are two writes
    lat, dev = [], []
    for i in range(warm + n):
        t0 = time.perf_counter()
        conn.request("POST", "/detect", body=body, headers={"Content-Type": "application/octet-stream"})
        r = conn.getresponse()
        data = r.read()
        dt = (time.perf_counter() - t0) * 1e3
        assert r.status == 200, data[:200]
        if i >= warm:
            lat.append(dt)
            dev.append(sum(json.loads(data)["timing_ms"].values()))
    conn.close()
    srv.shutdown()
    srv.server_close()
    return {"p50_ms": float(np.median(lat)), "p10_ms": float(np.percentile(lat, 10)),
            "p90_ms": float(np.percentile(lat, 90)), "device_ms_median": float(np.median(dev)),
            "request_bytes": len(body), "response_bytes": len(data), "blobs": len(json.loads(data)["blobs"])}


frame = synth.sensor_noise(synth.droplet_scene(1000, 1000, 100, (4.0, 20.0), seed=123), seed=124).image
print(json.dumps({"case": "1000x1000, sigma 2.5..9, n_bin 13, preprocess on (reference: 1827 ms p50)",
                  **measure(P.DetectionParams(min_sigma=2.5, max_sigma=9.0, n_bin=13), frame)}))
print(json.dumps({"case": "C2 1024x1024, sigma 1..30, n_bin 58, preprocess off",
                  **measure(P.DetectionParams(preprocess=False, **synth.config_params("C2")),
                            synth.config_frame("C2"))}))
