"""Scoring (evaluate.py) - host matcher against the reference's own implementation and its
documented properties; the device matcher and generator are in the -m gpu part."""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2010_08486_b200 as P
from paper_2010_08486_b200 import evaluate as ev, synth

REF_SRC = Path("/root/reference/pkg/src")


def mk(x, y, r, resp):
    return P.Blob(x, y, r / np.sqrt(2.0), r, resp, False)


def bset(*blobs):
    return P.BlobSet(blobs=tuple(blobs), source_shape=(100, 100), params=P.DetectionParams(backend="cuda"))


T = synth.Droplet


def random_case(rng, n_pred, n_truth, span=60, integer=False):
    pick = (lambda: float(rng.integers(0, span))) if integer else (lambda: float(rng.uniform(0, span)))
    truths = [T(pick(), pick(), float(rng.choice([2.0, 3.0, 4.5, 6.0]))) for _ in range(n_truth)]
    preds = [mk(pick(), pick(), float(rng.choice([2.0, 3.0, 4.5, 6.0])), float(rng.choice([0.2, 0.4, 0.6, 0.8])))
             for _ in range(n_pred)]
    return bset(*preds), truths


class TestBoxIou:
    def test_matches_pixel_counting_on_integer_boxes(self):
        rng = np.random.default_rng(3)
        for _ in range(50):
            x1, y1, x2, y2 = (int(v) for v in rng.integers(10, 30, 4))
            r1, r2 = (int(v) for v in rng.integers(1, 8, 2))
            a = np.zeros((60, 60), bool); b = np.zeros((60, 60), bool)
            a[y1 - r1:y1 + r1 + 1, x1 - r1:x1 + r1 + 1] = True
            b[y2 - r2:y2 + r2 + 1, x2 - r2:x2 + r2 + 1] = True
            want = (a & b).sum() / (a | b).sum()
            assert ev.box_iou(x1, y1, r1, x2, y2, r2) == pytest.approx(want, abs=1e-12)

    def test_disjoint_boxes(self):
        assert ev.box_iou(0, 0, 2, 10, 10, 2) == 0.0


class TestMatchVoc:
    def test_exact_match_gives_perfect_scores(self):
        truths = [T(10, 10, 4), T(30, 30, 6)]
        rep = ev.match_voc(bset(mk(10, 10, 4, 0.9), mk(30, 30, 6, 0.8)), truths)
        assert (rep.tp, rep.fp, rep.fn, rep.precision, rep.recall) == (2, 0, 0, 1.0, 1.0)

    def test_empty_sides_score_one(self):
        assert ev.match_voc(bset(), [T(5, 5, 2)]).precision == 1.0
        assert ev.match_voc(bset(), [T(5, 5, 2)]).recall == 0.0
        assert ev.match_voc(bset(mk(5, 5, 2, 0.5)), []).recall == 1.0
        assert ev.match_voc(bset(mk(5, 5, 2, 0.5)), []).precision == 0.0

    def test_each_truth_matched_at_most_once_and_strongest_claims_it(self):
        rep = ev.match_voc(bset(mk(10, 10, 4, 0.5), mk(10, 10, 4, 0.9)), [T(10, 10, 4)])
        assert (rep.tp, rep.fp) == (1, 1)
        assert rep.matches[0][0] == 1           # the stronger prediction (index 1) got the truth

    def test_lowering_threshold_never_decreases_tp(self):
        rng = np.random.default_rng(9)
        preds, truths = random_case(rng, 30, 25)
        tps = [ev.match_voc(preds, truths, thr).tp for thr in (0.9, 0.7, 0.5, 0.3, 0.1)]
        assert tps == sorted(tps) and tps[-1] <= min(30, 25)

    def test_threshold_validation(self):
        for bad in (0.0, -0.1, 1.5):
            with pytest.raises(ValueError):
                ev.match_voc(bset(), [], bad)

    def test_report_json_and_parity_csv_layout(self, tmp_path):
        rep = ev.match_voc(bset(mk(10, 10, 4, 0.9)), [T(11, 10, 4)])
        ev.write_report_json(tmp_path / "r.json", rep)
        doc = json.loads((tmp_path / "r.json").read_text())
        assert list(doc) == ["tp", "fp", "fn", "precision", "recall", "iou_threshold", "matches"]
        assert doc["matches"][0][:2] == [0, 0]
        z = np.zeros(2)
        st = ev.ParityStats(z + 1, z + 1, z + 1, z + 1, z, z, 0.0, 0.0, 0.0, 0.0)
        ev.write_parity_csv(tmp_path / "p.csv", st)
        lines = (tmp_path / "p.csv").read_text().splitlines()
        assert lines[0] == "image,precision_a,recall_a,precision_b,recall_b,dp,dr"
        assert lines[1] == "scene_000,1.0,1.0,1.0,1.0,0.0,0.0" and lines[-1] == "# mean_dr=0.0 std_dr=0.0"

    @pytest.mark.skipif(not REF_SRC.exists(), reason="the reference sources are not on this machine")
    def test_identical_to_the_reference_implementation(self, tmp_path):
        """random sets full of equal IoUs and equal responses (integer grids, few radii): every
        report field and every match of the reference's own match_voc"""
        sys.path.insert(0, str(REF_SRC))
        try:
            from dogblob import evaluate as rev
            from dogblob.detector import Blob as RBlob, BlobSet as RBlobSet, DetectionParams as RParams
            from dogblob.synth import GroundTruthCircle
        finally:
            sys.path.remove(str(REF_SRC))
        rng = np.random.default_rng(21)
        for trial in range(40):
            preds, truths = random_case(rng, int(rng.integers(0, 40)), int(rng.integers(0, 40)),
                                        span=25 if trial % 2 else 60, integer=trial % 3 == 0)
            rpreds = RBlobSet(blobs=tuple(RBlob(b.x, b.y, b.sigma, b.radius, b.response, False) for b in preds.blobs),
                              source_shape=(100, 100), params=RParams())
            rtruths = [GroundTruthCircle(t.x, t.y, t.r) for t in truths]
            for thr in (0.5, 0.2):
                a, b = ev.match_voc(preds, truths, thr), rev.match_voc(rpreds, rtruths, thr)
                assert (a.tp, a.fp, a.fn, a.precision, a.recall) == (b.tp, b.fp, b.fn, b.precision, b.recall)
                assert a.matches == b.matches


def test_truth_csv_round_trip(tmp_path):
    frame = synth.droplet_scene(64, 64, 5, (2.0, 6.0), seed=4)
    synth.write_truth_csv(tmp_path / "t.csv", frame)
    back = synth.read_truth_csv(tmp_path / "t.csv")
    assert [(d.x, d.y, d.r) for d in back] == [(float(d.x), float(d.y), float(d.r)) for d in frame.truths]


def test_cli_evaluate(tmp_path, capsys):
    from paper_2010_08486_b200 import cli, formats
    preds = bset(mk(10, 10, 4, 0.9), mk(40, 40, 3, 0.5))
    formats.write_blobset_json(tmp_path / "b.json", preds)
    (tmp_path / "t.csv").write_text("# seed=1\nx,y,r\n10.0,10.0,4.0\n")
    rc = cli.main(["evaluate", "--pred", str(tmp_path / "b.json"), "--truth", str(tmp_path / "t.csv"),
                   "--out", str(tmp_path / "rep.json")])
    assert rc == 0 and "precision=0.5000 recall=1.0000 (tp=1 fp=1 fn=0)" in capsys.readouterr().out
    assert json.loads((tmp_path / "rep.json").read_text())["tp"] == 1
