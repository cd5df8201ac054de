"""Precision / recall scoring of blob sets and detector-configuration parity statistics.

Mirrors the reference's `evaluate` module (pkg/src/dogblob/evaluate.py:24-182: `EvalReport`,
`ParityStats`, `box_iou`, `match_voc`, `parity`, `write_report_json`, `write_parity_csv`) with the
same conventions: PASCAL VOC 2012 matching on the circles' bounding boxes (inclusive pixel
extents, side 2 r + 1), predictions visited in descending response order, each claiming the
unmatched truth with the highest IoU if that IoU reaches the threshold; empty denominators score
1.0.  `match_voc` is host code over the (small) record arrays; `match_voc_batch` scores many
frames at once on the device (csrc/evaluate.cu: one CTA per frame, identical
matches) for sweeps over thousands of frames.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .detector import BlobSet, DetectionParams, Detector

__all__ = ["EvalReport", "ParityStats", "box_iou", "match_voc", "match_voc_batch", "parity",
           "write_report_json", "write_parity_csv"]


@dataclass(frozen=True)
class EvalReport:
    tp: int
    fp: int
    fn: int
    precision: float
    recall: float
    iou_threshold: float
    matches: tuple      # ((pred index, truth index, iou), ...)


@dataclass(frozen=True)
class ParityStats:
    precision_a: np.ndarray = field(repr=False)
    recall_a: np.ndarray = field(repr=False)
    precision_b: np.ndarray = field(repr=False)
    recall_b: np.ndarray = field(repr=False)
    dp: np.ndarray = field(repr=False)
    dr: np.ndarray = field(repr=False)
    mean_dp: float
    mean_dr: float
    std_dp: float
    std_dr: float


def box_iou(x1: float, y1: float, r1: float, x2: float, y2: float, r2: float) -> float:
    """IoU of the circles' bounding boxes, inclusive-pixel side lengths (evaluate.py:48-58)."""
    iw = min(x1 + r1, x2 + r2) - max(x1 - r1, x2 - r2) + 1.0
    ih = min(y1 + r1, y2 + r2) - max(y1 - r1, y2 - r2) + 1.0
    if iw <= 0 or ih <= 0:
        return 0.0
    inter = iw * ih
    return inter / ((2.0 * r1 + 1.0) ** 2 + (2.0 * r2 + 1.0) ** 2 - inter)


def _pred_arrays(preds: BlobSet):
    """(x, y, radius) rows in visiting order and the permutation that produced it."""
    rec = preds.records
    n = len(rec)
    if n == 0:
        return np.zeros((0, 3)), np.zeros(0, dtype=np.int64)
    # sorted(range(n), key=(-response, y, x)), stable
    order = np.lexsort((rec["x"], rec["y"], -rec["response"]))
    xyr = np.stack([rec["x"][order], rec["y"][order], rec["radius"][order]], axis=1).astype(np.float64)
    return np.ascontiguousarray(xyr), order


def _truth_array(truths) -> np.ndarray:
    t = np.array([(t.x, t.y, t.r) for t in truths], dtype=np.float64).reshape(-1, 3)
    return np.ascontiguousarray(t)


def _iou_row(p, t):
    """box IoU of one prediction row against truth rows, the reference's operation order"""
    iw = np.minimum(p[0] + p[2], t[:, 0] + t[:, 2]) - np.maximum(p[0] - p[2], t[:, 0] - t[:, 2]) + 1.0
    ih = np.minimum(p[1] + p[2], t[:, 1] + t[:, 2]) - np.maximum(p[1] - p[2], t[:, 1] - t[:, 2]) + 1.0
    inter = iw * ih
    with np.errstate(divide="ignore", invalid="ignore"):
        iou = inter / ((2.0 * p[2] + 1.0) ** 2 + (2.0 * t[:, 2] + 1.0) ** 2 - inter)
    return np.where((iw <= 0) | (ih <= 0), 0.0, iou)


def _report(n_pred, n_truth, matches, iou_threshold) -> EvalReport:
    tp = len(matches)
    fp, fn = n_pred - tp, n_truth - tp
    return EvalReport(tp=tp, fp=fp, fn=fn, precision=tp / (tp + fp) if tp + fp > 0 else 1.0,
                      recall=tp / (tp + fn) if tp + fn > 0 else 1.0, iou_threshold=iou_threshold,
                      matches=tuple(matches))


def match_voc(preds: BlobSet, truths, iou_threshold: float = 0.5) -> EvalReport:
    """Greedy one-to-one matching of predictions to ground-truth circles (evaluate.py:61-109)."""
    if not 0.0 < iou_threshold <= 1.0:
        raise ValueError(f"iou_threshold must be in (0, 1], got {iou_threshold}")
    truths = list(truths)
    p, order = _pred_arrays(preds)
    t = _truth_array(truths)
    free = np.ones(len(truths), dtype=bool)
    matches = []
    for k in range(len(p)):
        if not free.any():
            break
        iou = np.where(free, _iou_row(p[k], t), 0.0)
        ti = int(np.argmax(iou))                    # first index among equal maxima, like the scan
        if iou[ti] > 0.0 and iou[ti] >= iou_threshold:
            free[ti] = False
            matches.append((int(order[k]), ti, float(iou[ti])))
    return _report(len(p), len(truths), matches, iou_threshold)


def match_voc_batch(pred_sets, truth_sets, iou_threshold: float = 0.5, device: int | None = None) -> list:
    """`match_voc` for many frames at once on the device (one CTA per frame); same reports."""
    if not 0.0 < iou_threshold <= 1.0:
        raise ValueError(f"iou_threshold must be in (0, 1], got {iou_threshold}")
    import torch
    lib = _lib.load()
    pred_sets, truth_sets = list(pred_sets), [list(t) for t in truth_sets]
    if len(pred_sets) != len(truth_sets):
        raise ValueError("need one truth list per prediction set")
    if not pred_sets:
        return []
    pa = [_pred_arrays(p) for p in pred_sets]
    ta = [_truth_array(t) for t in truth_sets]
    pb = np.concatenate([[0], np.cumsum([len(a[0]) for a in pa])]).astype(np.int32)
    tb = np.concatenate([[0], np.cumsum([len(a) for a in ta])]).astype(np.int32)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    d_pred = to(np.concatenate([a[0] for a in pa]) if pb[-1] else np.zeros((1, 3)))
    d_truth = to(np.concatenate(ta) if tb[-1] else np.zeros((1, 3)))
    d_pb, d_tb = to(pb), to(tb)
    d_taken = torch.zeros(max(int(tb[-1]), 1), dtype=torch.uint8, device=dev)
    d_match = torch.full((max(int(pb[-1]), 1),), -1, dtype=torch.int32, device=dev)
    d_iou = torch.zeros(max(int(pb[-1]), 1), dtype=torch.float64, device=dev)
    d_tp = torch.zeros(len(pa), dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev)
        _lib.check(lib.dogblob_match_voc(len(pa), d_pred.data_ptr(), d_pb.data_ptr(), d_truth.data_ptr(),
                                         d_tb.data_ptr(), float(iou_threshold), d_taken.data_ptr(),
                                         d_match.data_ptr(), d_iou.data_ptr(), d_tp.data_ptr(), st.cuda_stream))
        match, iou = d_match.cpu().numpy(), d_iou.cpu().numpy()
    out = []
    for j, (p, order) in enumerate(pa):
        m, q = match[pb[j]:pb[j + 1]], iou[pb[j]:pb[j + 1]]
        matches = [(int(order[k]), int(m[k]), float(q[k])) for k in range(len(m)) if m[k] >= 0]
        out.append(_report(len(p), len(ta[j]), matches, iou_threshold))
    return out


def parity(imgs, params_a: DetectionParams, params_b: DetectionParams, truths_per_image,
           iou_threshold: float = 0.5, dtype_a=np.float32, dtype_b=np.float32) -> ParityStats:
    """Per-image precision / recall differences between two detector configurations
    (evaluate.py:112-152).  The reference compares its `direct` and `fft` backends; here both
    sides run on the device and may differ in numeric options or in the arithmetic tier
    (`dtype_a` / `dtype_b`: float32 production kernels versus the float64 tier)."""
    ladder_a = (params_a.min_sigma, params_a.max_sigma, params_a.n_bin)
    ladder_b = (params_b.min_sigma, params_b.max_sigma, params_b.n_bin)
    if ladder_a != ladder_b:
        raise ValueError(f"parity requires one ladder, got {ladder_a} vs {ladder_b}")
    det_a, det_b = Detector(params_a), Detector(params_b)
    try:
        imgs, truths = list(imgs), [list(t) for t in truths_per_image]
        blobs_a = [det_a.run(img, dtype=dtype_a).blobs for img in imgs]
        blobs_b = [det_b.run(img, dtype=dtype_b).blobs for img in imgs]
    finally:
        det_a.close()
        det_b.close()
    rep_a = match_voc_batch(blobs_a, truths, iou_threshold)
    rep_b = match_voc_batch(blobs_b, truths, iou_threshold)
    pa, ra = np.array([r.precision for r in rep_a]), np.array([r.recall for r in rep_a])
    pb, rb = np.array([r.precision for r in rep_b]), np.array([r.recall for r in rep_b])
    dp, dr = pa - pb, ra - rb
    return ParityStats(precision_a=pa, recall_a=ra, precision_b=pb, recall_b=rb, dp=dp, dr=dr,
                       mean_dp=float(dp.mean()) if dp.size else 0.0, mean_dr=float(dr.mean()) if dr.size else 0.0,
                       std_dp=float(dp.std()) if dp.size else 0.0, std_dr=float(dr.std()) if dr.size else 0.0)


def write_report_json(path, report: EvalReport) -> None:
    doc = {"tp": report.tp, "fp": report.fp, "fn": report.fn, "precision": report.precision,
           "recall": report.recall, "iou_threshold": report.iou_threshold,
           "matches": [[p, t, iou] for p, t, iou in report.matches]}
    with open(path, "w") as f:
        json.dump(doc, f, indent=2)
        f.write("\n")


def write_parity_csv(path, stats: ParityStats, names=None) -> None:
    n = stats.dp.size
    names = list(names) if names is not None else [f"scene_{i:03d}" for i in range(n)]
    with open(path, "w") as f:
        f.write("image,precision_a,recall_a,precision_b,recall_b,dp,dr\n")
        for i in range(n):
            f.write(f"{names[i]},{float(stats.precision_a[i])!r},{float(stats.recall_a[i])!r},"
                    f"{float(stats.precision_b[i])!r},{float(stats.recall_b[i])!r},"
                    f"{float(stats.dp[i])!r},{float(stats.dr[i])!r}\n")
        f.write(f"# mean_dp={stats.mean_dp!r} std_dp={stats.std_dp!r}\n")
        f.write(f"# mean_dr={stats.mean_dr!r} std_dr={stats.std_dr!r}\n")
