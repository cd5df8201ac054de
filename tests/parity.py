"""Helpers shared by the parity tests: golden decoding and the near-tie classifier.

Blob-set parity rule (BASELINE.json north_star): indices and sigma levels are
bit-exact, except for peaks whose DoG response lies within a stated float32
epsilon of the threshold or of a neighbour tie; those are reported.

EPS_REL is that epsilon: a candidate in slice i is "fragile" when, in float64
arithmetic, its DoG value is within sigma_i * EPS_REL of the threshold or of the
largest value among its 26 neighbours.  sigma_i scales the bound because
D_i = sigma_i (L_i - L_{i+1}) amplifies the absolute error of the two float32
levels (the reference's own fft/float32 levels carry ~4e-7, pkg/test_output.txt:15).
"""

from __future__ import annotations

import numpy as np

from oracle import dog_oracle as O

EPS_REL = 2.0e-6


def golden_blobs(g, prefix):
    """[(x, y, sigma, radius, response, edge)] from a golden npz."""
    return list(zip(g[prefix + "bx"].tolist(), g[prefix + "by"].tolist(),
                    g[prefix + "bsigma"].tolist(), g[prefix + "bradius"].tolist(),
                    g[prefix + "bresponse"].tolist(), g[prefix + "bedge"].tolist()))


def golden_oblobs(g, prefix):
    return [O.OBlob(int(x), int(y), float(s), float(r), float(v), bool(e))
            for x, y, s, r, v, e in golden_blobs(g, prefix)]


def oblob_tuples(blobs):
    return [(b.x, b.y, b.sigma, b.radius, b.response, b.at_scale_boundary) for b in blobs]


def records_tuples(recs):
    """dogblob_blob records -> same tuple form (x, y as int when integral)."""
    out = []
    for r in recs:
        x, y = float(r["x"]), float(r["y"])
        if x == int(x):
            x = int(x)
        if y == int(y):
            y = int(y)
        out.append((x, y, float(r["sigma"]), float(r["radius"]), float(r["response"]),
                    bool(r["flags"] & 1)))
    return out


def slice_of(sigma, sigmas):
    idx = np.nonzero(np.asarray(sigmas) == sigma)[0]
    assert idx.size == 1, f"sigma {sigma} is not a ladder scale"
    return int(idx[0])


def classify_candidates(img, sigmas, radii, threshold, got, want, neighborhood=3):
    """Compare two candidate lists (tuples as above, integer centres).

    Returns dict(common, only_got, only_want, explained, unexplained, max_resp_diff);
    every voxel in the symmetric difference is looked up in float64.
    """
    key = lambda t: (slice_of(t[2], sigmas), t[1], t[0])
    gk = {key(t): t for t in got}
    wk = {key(t): t for t in want}
    common = sorted(set(gk) & set(wk))
    only_got = sorted(set(gk) - set(wk))
    only_want = sorted(set(wk) - set(gk))
    explained, unexplained = [], []
    half = neighborhood // 2
    for k in only_got + only_want:
        s, y, x = k
        block = O.dog_neighbourhood_f64(img, sigmas, radii, s, y, x, half)
        c = block[half, half, half]
        others = block.copy()
        others[half, half, half] = -np.inf
        margin = min(abs(c - others.max()), abs(c - float(np.float32(threshold))))
        eps = float(sigmas[s]) * EPS_REL
        (explained if margin <= eps else unexplained).append((k, margin, eps))
    max_resp = 0.0
    for k in common:
        eps = float(sigmas[k[0]]) * EPS_REL
        d = abs(gk[k][4] - wk[k][4])
        max_resp = max(max_resp, d / eps)
    return dict(common=common, only_got=only_got, only_want=only_want, explained=explained,
                unexplained=unexplained, max_resp_diff_in_eps=max_resp)


# ---- the parity report (profiles/rNN_parity.json) ------------------------------------------------
# north_star: peaks whose DoG response lies within the stated epsilon of the threshold or of a
# neighbour tie "are reported".  The -m gpu configuration tests collect one entry per frame here
# and tests/conftest.py writes the file when the session ends.
REPORT = {}
ROUND_TAG = "r02"


def _voxel_rows(items):
    return [{"slice": int(k[0]), "y": int(k[1]), "x": int(k[2]), "float64_margin": float(m), "eps": float(e)}
            for k, m, e in items]


def report_entry(rep, n_got, n_want):
    return {"candidates_gpu": int(n_got), "candidates_ref": int(n_want), "common": len(rep["common"]),
            "only_gpu": len(rep["only_got"]), "only_ref": len(rep["only_want"]),
            "fragile": _voxel_rows(rep["explained"]), "unexplained": _voxel_rows(rep["unexplained"]),
            "max_response_diff_in_eps": float(rep["max_resp_diff_in_eps"])}


def reference_t0_vs_t1(img, sigmas, radii, threshold, t0, t1):
    """The reference against itself: float32 / fft (T0, production) versus float64 / direct (T1)
    candidates of the same frame, every differing voxel classified like a GPU difference."""
    rep = classify_candidates(img, sigmas, radii, threshold, t0, t1)
    e = report_entry(rep, len(t0), len(t1))
    e["candidates_t0"], e["candidates_t1"] = e.pop("candidates_gpu"), e.pop("candidates_ref")
    e["only_t0"], e["only_t1"] = e.pop("only_gpu"), e.pop("only_ref")
    return e


def write_report(root):
    """profiles/<round>_parity.json (+ a copy under gpurun_out/, the only directory a GPU box returns)"""
    import json
    from pathlib import Path
    if not REPORT:
        return None
    doc = {"rule": "centres and sigma levels bit-exact except peaks whose float64 DoG margin to the threshold "
                   "or to the largest of the 26 neighbours is <= sigma_i * EPS_REL (BASELINE.json north_star)",
           "EPS_REL": EPS_REL,
           "reference_noise": "the reference's own float32 fft levels differ from its float64 levels by up to "
                              "4.17e-7 (pkg/test_output.txt:15), i.e. 8e-7 * sigma_i on a DoG value",
           "frames": REPORT,
           "totals": {"frames": len(REPORT),
                      "fragile": sum(len(v["gpu_vs_reference"]["fragile"]) for v in REPORT.values()),
                      "unexplained": sum(len(v["gpu_vs_reference"]["unexplained"]) for v in REPORT.values())}}
    out = None
    for d in (Path(root) / "profiles", Path(root) / "gpurun_out"):
        try:
            d.mkdir(exist_ok=True)
            out = d / f"{ROUND_TAG}_parity.json"
            out.write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")
        except OSError:
            pass
    return out
