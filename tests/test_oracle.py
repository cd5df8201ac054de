"""Pins oracle/dog_oracle.py to the reference: committed outputs of the real
reference (tools/make_golden.py) and the reference's own golden vector."""

import json

import numpy as np
import pytest

from oracle import dog_oracle as O
from paper_2010_08486_b200 import synth
from parity import golden_blobs, golden_oblobs, oblob_tuples


@pytest.fixture(scope="module")
def small(golden):
    return golden("small_stages.npz")


class TestStages:
    def test_fft_levels_bit_exact_float32(self, small):
        lv = O.levels_fft(small["a_img"], small["a_sigmas"], small["a_radii"], np.float32)
        assert np.array_equal(lv, small["a_levels_fft_f32"])

    def test_fft_levels_bit_exact_float64(self, small):
        lv = O.levels_fft(small["a_img"], small["a_sigmas"], small["a_radii"], np.float64)
        assert np.array_equal(lv, small["a_levels_fft_f64"])

    def test_dog_bit_exact(self, small):
        lv = O.levels_fft(small["a_img"], small["a_sigmas"], small["a_radii"], np.float32)
        assert np.array_equal(O.dog_slices(lv, small["a_sigmas"]), small["a_dog_f32"])

    def test_separable_truth_matches_both_reference_backends(self, small):
        sep = O.levels_separable(small["a_img"], small["a_sigmas"], small["a_radii"])
        assert np.abs(sep - small["a_levels_fft_f64"]).max() < 1e-14
        assert np.abs(sep - small["a_levels_direct_f64"]).max() < 1e-14

    def test_kernel_wider_than_image(self, small):
        sep = O.levels_separable(small["b_img"], small["b_sigmas"], small["b_radii"])
        assert np.abs(sep - small["b_levels_fft_f64"]).max() < 1e-14
        fft = O.levels_fft(small["b_img"], small["b_sigmas"], small["b_radii"], np.float64)
        assert np.array_equal(fft, small["b_levels_fft_f64"])

    @pytest.mark.parametrize("tag", ["c1", "c2", "c3", "c4"])
    def test_ragged_shapes(self, small, tag):
        sep = O.levels_separable(small[tag + "_img"], small[tag + "_sigmas"], small[tag + "_radii"])
        assert np.abs(sep - small[tag + "_levels_fft_f64"]).max() < 1e-14

    def test_pointwise_level_evaluator(self, small):
        ys, xs = [0, 5, 47, 20], [0, 63, 10, 31]
        for i in range(4):
            v = O.level_values_at(small["a_img"], small["a_sigmas"][i], int(small["a_radii"][i]), ys, xs)
            assert np.abs(v - small["a_levels_fft_f64"][i][ys, xs]).max() < 1e-14

    def test_dog_neighbourhood_block(self, small):
        dog64 = O.dog_slices(small["a_levels_fft_f64"], small["a_sigmas"])
        blk = O.dog_neighbourhood_f64(small["a_img"], small["a_sigmas"], small["a_radii"], 1, 10, 0)
        assert np.all(np.isneginf(blk[:, :, 0]))            # x = -1 is outside
        assert np.abs(blk[:, :, 1:] - dog64[0:3, 9:12, 0:2]).max() < 1e-13


class TestExtrema:
    def test_random_stack(self, small):
        got = O.extrema(small["d_slices"], np.array([1.0, 2.0, 3.0]), 0.2)
        assert oblob_tuples(got) == golden_blobs(small, "d_cand_")

    @pytest.mark.parametrize("n", [1, 5])
    def test_other_neighbourhoods(self, small, n):
        got = O.extrema(small["d_slices"], np.array([1.0, 2.0, 3.0]), 0.2, n)
        assert oblob_tuples(got) == golden_blobs(small, f"d_n{n}_cand_")

    def test_plateaus_corner_and_half_even_centroid(self, small):
        got = O.extrema(small["e_slices"], np.array([2.0, 3.0]), 0.1)
        assert oblob_tuples(got) == golden_blobs(small, "e_cand_")
        assert (10, 10) in [(b.x, b.y) for b in got]         # 3x6 plateau, centroid (10.5, 10)

    def test_on_reference_dog(self, small):
        got = O.extrema(small["a_dog_f32"], small["a_sigmas"][:-1], 0.02)
        assert oblob_tuples(got) == golden_blobs(small, "a_cand_")

    def test_even_neighbourhood_rejected(self, small):
        with pytest.raises(ValueError):
            O.extrema(small["d_slices"], np.array([1.0, 2.0, 3.0]), 0.2, 4)


class TestPruneAndHistogram:
    def test_cases(self, golden):
        p = golden("prune_cases.npz")
        for c in range(int(p["n_cases"])):
            out = O.prune(golden_oblobs(p, f"p{c}_in_"), float(p[f"p{c}_thr"]))
            assert oblob_tuples(out) == golden_blobs(p, f"p{c}_out_"), c
            h = O.radius_histogram(out, O.ladder_sigmas(1.0, 8.0, 10))
            assert np.array_equal(h.counts, p[f"p{c}_hist_counts"])
            assert np.array_equal(h.volume_weights, p[f"p{c}_hist_volumes"])

    def test_incremental_equals_literal_form(self, golden):
        p = golden("prune_cases.npz")
        for c in (0, 1, 2, 4):
            blobs = golden_oblobs(p, f"p{c}_in_")
            thr = float(p[f"p{c}_thr"])
            assert O.prune(blobs, thr) == O.prune_dense(blobs, thr)

    def test_dense_c5_candidates(self, golden):
        """9,714 reference candidates of the dense frame -> the reference's 9,023 survivors
        (691 merges; the reference's dense-matrix loop needs 75 minutes for this)"""
        g = golden("config_C5.npz")
        out = O.prune(golden_oblobs(g, "t0_cand_"), 0.5)
        assert oblob_tuples(out) == golden_blobs(g, "t0_kept_")
        h = O.radius_histogram(out, O.ladder_sigmas(1.0, 6.0, 10))
        assert np.array_equal(h.counts, g["t0_hist_counts"])
        assert np.array_equal(h.volume_weights, g["t0_hist_volumes"])

    def test_threshold_bounds(self):
        with pytest.raises(ValueError):
            O.prune([], 1.5)


def _run(name, frame, tier="t0", **extra):
    kw = dict(synth.config_params(name), preprocess=False, **extra)
    det = O.OracleDetector(**kw)
    return det, det.run(frame, dtype=np.float32 if tier == "t0" else np.float64)


class TestPipeline:
    def test_scene256(self, golden):
        g = golden("scene256.npz")
        frame = synth.sensor_noise(synth.droplet_scene(256, 256, 12, (4.0, 12.0), seed=5), seed=6).image
        det = O.OracleDetector(min_sigma=2.5, max_sigma=9.0, n_bin=10, preprocess=False)
        for tier, dt in (("t0", np.float32), ("t1", np.float64)):
            res = det.run(frame, dtype=dt)
            assert oblob_tuples(res.candidates) == golden_blobs(g, f"{tier}_cand_")
            assert oblob_tuples(res.blobs) == golden_blobs(g, f"{tier}_kept_")
        pre = O.OracleDetector(min_sigma=2.5, max_sigma=9.0, n_bin=10)   # preprocess=True default
        assert np.array_equal(O.preprocess(frame), g["pre_image"])
        assert oblob_tuples(pre.run(frame).blobs) == golden_blobs(g, "pre_kept_")

    def test_reference_demo_golden_vector(self):
        """pkg/demos/output/03_blobs.json + 03_histogram.csv, the reference's own fixture
        (scene + params of pkg/demos/03_detect_and_histogram.py:24-28, preprocess on)."""
        from conftest import GOLDEN
        doc = json.loads((GOLDEN / "ref_demo03_blobs.json").read_text())
        frame = synth.sensor_noise(synth.droplet_scene(1000, 1000, 100, (4.0, 20.0), seed=123),
                                   seed=124).image
        p = doc["params"]
        det = O.OracleDetector(**{k: v for k, v in p.items()})
        res = det.run(frame)
        want = [(b["x"], b["y"], b["sigma"], b["radius"], b["response"], b["at_scale_boundary"])
                for b in doc["blobs"]]
        assert oblob_tuples(res.blobs) == want
        rows = (GOLDEN / "ref_demo03_histogram.csv").read_text().strip().splitlines()[1:]
        for row, c, n, v in zip(rows, res.histogram.bin_centers, res.histogram.counts,
                                res.histogram.volume_weights):
            assert row == f"{float(c)!r},{int(n)},{float(v)!r}"

    def test_config_c1(self, golden):
        g = golden("config_C1.npz")
        det, res = _run("C1", synth.config_frame("C1"))
        assert oblob_tuples(res.candidates) == golden_blobs(g, "t0_cand_")
        assert oblob_tuples(res.blobs) == golden_blobs(g, "t0_kept_")
        assert np.array_equal(res.histogram.counts, g["t0_hist_counts"])
        assert np.array_equal(res.histogram.volume_weights, g["t0_hist_volumes"])

    def test_config_c2(self, golden):
        g = golden("config_C2.npz")
        det, res = _run("C2", synth.config_frame("C2"))
        assert oblob_tuples(res.candidates) == golden_blobs(g, "t0_cand_")
        assert oblob_tuples(res.blobs) == golden_blobs(g, "t0_kept_")
        assert len(res.blobs) == 129 and len(res.candidates) == 138


def tie_cases():
    """Blob sets full of exact (response, y, x) ties: same-pixel twins / triplets in different
    slices (equal float32 DoG values in neighbouring slices are all flagged, detector.py:165-166),
    alone, next to overlapping neighbours, and mixed into random sets."""
    import math
    r2 = math.sqrt(2.0)
    mk = lambda x, y, sigma, resp, edge=False: O.OBlob(x, y, sigma, sigma * r2, float(np.float32(resp)), edge)
    cases = [
        [mk(10, 10, 2.0, 0.5), mk(10, 10, 3.0, 0.5)],
        [mk(10, 10, 2.0, 0.5), mk(10, 10, 3.0, 0.5), mk(10, 10, 9.0, 0.5)],
        # twins with a stronger and a weaker overlapping neighbour on either side
        [mk(10, 10, 2.0, 0.5), mk(10, 10, 6.0, 0.5), mk(12, 10, 4.0, 0.9), mk(9, 11, 5.0, 0.2), mk(30, 30, 3.0, 0.5)],
        # the absorbed twin is the larger / the smaller one; boundary flags travel
        [mk(20, 20, 8.0, 0.7, True), mk(20, 20, 1.5, 0.7), mk(26, 20, 8.0, 0.7), mk(20, 26, 1.5, 0.7)],
        # two pairs of twins overlapping each other
        [mk(15, 15, 3.0, 0.4), mk(15, 15, 5.0, 0.4), mk(17, 15, 3.5, 0.4), mk(17, 15, 4.5, 0.4), mk(16, 15, 4.0, 0.4)],
    ]
    rng = np.random.default_rng(5)
    for _ in range(6):
        blobs = []
        for _k in range(25):
            x, y = int(rng.integers(0, 40)), int(rng.integers(0, 40))
            resp = float(rng.choice([0.25, 0.5, 0.75]))
            for sigma in rng.choice([1.5, 2.0, 3.0, 4.5, 6.0], size=int(rng.integers(1, 4)), replace=False):
                blobs.append(mk(x, y, float(sigma), resp, bool(rng.integers(0, 2))))
        cases.append(blobs)
    return cases


class TestPruneTies:
    @pytest.mark.parametrize("thr", [0.5, 0.1, 0.99, 1.0])
    def test_cached_partner_form_equals_literal_resorting_form_on_exact_ties(self, thr):
        for blobs in tie_cases():
            assert O.prune(blobs, thr) == O.prune_dense(blobs, thr)
