"""Host-side logic that needs no GPU: ladder/taps (ported from the reference's
tests/test_scale_space.py), records, histogram, synthetic frames, and the C-ABI
library's load + symbol table."""

import ctypes
import hashlib
import json
import math
import re

import numpy as np
import pytest

import paper_2010_08486_b200 as P
from paper_2010_08486_b200 import _lib, synth
from conftest import GOLDEN, ROOT


class TestBuildLadder:
    def test_simple_progression(self):
        ladder = P.build_ladder(1.0, 3.0, 2)
        assert np.allclose(ladder.sigmas, [1.0, 2.0, 3.0])
        assert ladder.delta_sigma == 1.0 and ladder.n_levels == 3

    def test_endpoints_exact(self):
        ladder = P.build_ladder(0.7, 13.3, 17)
        assert ladder.sigmas[0] == 0.7 and ladder.sigmas[-1] == 13.3
        assert np.allclose(np.diff(ladder.sigmas), ladder.delta_sigma)

    def test_degenerate_equal_sigmas_rejected(self):
        with pytest.raises(ValueError, match="degenerate"):
            P.build_ladder(2.0, 2.0, 1)

    @pytest.mark.parametrize("args", [(0.0, 3.0, 2), (-1.0, 3.0, 2), (3.0, 1.0, 2), (1.0, 3.0, 0)])
    def test_invalid_arguments(self, args):
        with pytest.raises(ValueError):
            P.build_ladder(*args)


class TestTapBank:
    def test_width_formula_and_padding(self):
        bank = P.build_kernel_bank(P.build_ladder(0.5, 2.0, 1), truncate=5.0)
        assert list(bank.radii) == [3, 10] and bank.max_width == 21
        k = bank.kernels
        assert k.shape == (2, 21, 21)
        frame = k[0].copy()
        frame[10 - 3:10 + 4, 10 - 3:10 + 4] = 0.0
        assert np.all(frame == 0.0) and k[0, 10, 10] > 0.0

    def test_unit_sums_and_separability(self):
        bank = P.build_kernel_bank(P.build_ladder(0.5, 6.0, 10))
        for i in range(bank.ladder.n_levels):
            w = bank.level_taps(i)
            assert abs(w.sum() - 1.0) < 1e-12
            r = int(bank.radii[i]); c = bank.max_width // 2
            assert np.abs(np.outer(w, w) - bank.kernels[i, c - r:c + r + 1, c - r:c + r + 1]).max() < 1e-15

    def test_center_value_matches_direct_evaluation(self):
        bank = P.build_kernel_bank(P.build_ladder(1.0, 2.0, 1))
        total = sum(math.exp(-(x * x + y * y) / 2.0) for x in range(-5, 6) for y in range(-5, 6))
        c = bank.max_width // 2
        assert bank.kernels[0, c, c] == pytest.approx(1.0 / total, rel=1e-12)
        assert bank.kernels[0, c + 1, c + 2] == pytest.approx(math.exp(-2.5) / total, rel=1e-12)

    def test_matches_oracle_definition(self):
        from oracle import dog_oracle as O
        ladder = P.build_ladder(1.0, 30.0, 58)
        bank = P.build_kernel_bank(ladder)
        assert np.array_equal(ladder.sigmas, O.ladder_sigmas(1.0, 30.0, 58))
        assert np.array_equal(bank.radii, O.tap_radii(ladder.sigmas))
        assert bank.taps64.size == 9233
        for i in (0, 17, 58):
            assert np.array_equal(bank.level_taps(i), O.kernel_1d(ladder.sigmas[i], int(bank.radii[i])))

    def test_width_cap_guard(self):
        with pytest.raises(ValueError, match="cap"):
            P.build_kernel_bank(P.build_ladder(1.0, 500.0, 2))

    def test_truncate_must_be_positive(self):
        with pytest.raises(ValueError):
            P.build_kernel_bank(P.build_ladder(1.0, 2.0, 1), truncate=0.0)


def mk(x, y, radius, response, sigma=None):
    return P.Blob(x=x, y=y, sigma=sigma if sigma is not None else radius / math.sqrt(2),
                  radius=radius, response=response)


def bset(*blobs):
    return P.BlobSet(blobs=tuple(blobs), source_shape=(100, 100), params=P.DetectionParams())


class TestRecordsAndHistogram:
    def test_blobset_round_trip(self):
        a, b = mk(3, 4, 5.0, 0.9), mk(7, 8, 2.5, 0.5)
        s = bset(a, b)
        assert len(s) == 2 and s.blobs == (a, b)
        again = P.BlobSet(records=s.records, source_shape=(100, 100), params=P.DetectionParams())
        assert again.blobs == (a, b) and again == s
        assert np.array_equal(again.yxs(), [[4, 3, a.sigma], [8, 7, b.sigma]])

    def test_empty_blobset_all_zero(self):
        ladder = P.build_ladder(1.0, 3.0, 2)
        hist = P.histogram(bset(), ladder)
        assert np.all(hist.counts == 0) and np.all(hist.volume_weights == 0)
        assert hist.bin_centers == pytest.approx(math.sqrt(2) * ladder.sigmas)

    def test_exact_center_and_midpoint_tie(self):
        ladder = P.build_ladder(1.0, 5.0, 4)
        centers = math.sqrt(2) * ladder.sigmas
        hist = P.histogram(bset(mk(5, 5, centers[3], 0.5)), ladder)
        assert hist.counts[3] == 1 and hist.counts.sum() == 1
        assert hist.volume_weights[3] == pytest.approx(4.0 / 3.0 * math.pi * centers[3] ** 3)
        mid = 0.5 * (centers[1] + centers[2])
        assert P.histogram(bset(mk(5, 5, mid, 0.5)), ladder).counts[1] == 1

    def test_histogram_bit_identical_to_reference(self, golden):
        p = golden("prune_cases.npz")
        ladder = P.build_ladder(1.0, 8.0, 10)
        for c in range(int(p["n_cases"])):
            pre = f"p{c}_out_"
            blobs = [P.Blob(int(x), int(y), float(s), float(r), float(v), bool(e))
                     for x, y, s, r, v, e in zip(p[pre + "bx"], p[pre + "by"], p[pre + "bsigma"],
                                                 p[pre + "bradius"], p[pre + "bresponse"], p[pre + "bedge"])]
            h = P.histogram(bset(*blobs), ladder)
            assert np.array_equal(h.counts, p[f"p{c}_hist_counts"])
            assert np.array_equal(h.volume_weights, p[f"p{c}_hist_volumes"])

    def test_overlap_helpers(self):
        assert P.disk_intersection_area(0, 0, 1, 5, 0, 1) == 0.0
        assert P.disk_intersection_area(0, 0, 2, 0, 0, 1) == pytest.approx(math.pi)
        assert P.normalized_overlap(mk(20, 20, 10.0, 0.5), mk(22, 20, 2.0, 0.9)) == pytest.approx(1.0)


class TestParamsAndErrors:
    def test_defaults_match_reference(self):
        d = P.DetectionParams().to_dict()
        assert d == dict(min_sigma=1.0, max_sigma=10.0, n_bin=18, truncate=5.0, threshold=0.1,
                         overlap=0.5, neighborhood=3, backend="cuda", preprocess=True,
                         smooth_sigma=1.0, saturation=0.0035, prune=True)

    def test_unknown_backend(self):
        with pytest.raises(ValueError, match="backend"):
            P.Detector(P.DetectionParams(backend="fft"))
        with pytest.raises(ValueError, match="backend"):
            P.convolve_bank(np.ones((4, 4)), P.build_kernel_bank(P.build_ladder(1, 2, 1)), "gpu")

    def test_bad_parameters(self):
        with pytest.raises(ValueError):
            P.Detector(P.DetectionParams(neighborhood=4))
        with pytest.raises(ValueError):
            P.Detector(P.DetectionParams(overlap=1.5))
        with pytest.raises(ValueError):
            P.Detector(P.DetectionParams(max_sigma=0.5))
        with pytest.raises(ValueError):
            P.convolve_bank(np.ones((0, 4)), P.build_kernel_bank(P.build_ladder(1, 2, 1)))
        with pytest.raises(ValueError, match="cap"):
            P.convolve_bank(np.ones((64, 64), np.float32),
                            P.build_kernel_bank(P.build_ladder(1, 4, 3)), stack_element_cap=1000)
        with pytest.raises(ValueError):
            P.prune_overlaps(bset(), 1.5)
        with pytest.raises(ValueError):
            P.find_extrema(P.DoGStack(np.zeros((1, 8, 8), np.float32), np.array([1.0])), neighborhood=4)

    def test_no_cpu_fallback(self):
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
        det = P.Detector(P.DetectionParams(preprocess=False))
        with pytest.raises(RuntimeError, match="no CPU fallback"):
            det.run(np.zeros((16, 16), np.float32))


class TestSynth:
    def test_frames_match_reference_hashes(self):
        doc = json.loads((GOLDEN / "frames.json").read_text())
        for name in ("C1", "C2", "C5"):
            f = synth.config_frame(name)
            assert hashlib.sha256(f.tobytes()).hexdigest() == doc[name]["sha256"], name
        f = synth.config_frame("C3", 2)
        assert hashlib.sha256(f.tobytes()).hexdigest() == doc["C3_2"]["sha256"]
        d = synth.flat_disk(128, 96, 64.25, 40.5, 10.0)
        assert hashlib.sha256(d.tobytes()).hexdigest() == doc["disk_128x96"]["sha256"]
        s = synth.droplet_scene(200, 160, 10, (4.0, 12.0), seed=7)
        assert hashlib.sha256(s.image.tobytes()).hexdigest() == doc["scene_nooverlap_200x160"]["sha256"]

    def test_deterministic_and_guarded(self):
        a = synth.droplet_scene(64, 64, 3, (2.0, 5.0), seed=9).image
        b = synth.droplet_scene(64, 64, 3, (2.0, 5.0), seed=9).image
        assert np.array_equal(a, b)
        with pytest.raises(ValueError):
            synth.droplet_scene(16, 16, 1, (10.0, 12.0), seed=1)


class TestCAbi:
    def test_library_loads_and_exports_every_declared_symbol(self):
        header = (ROOT / "include" / "dogblob_b200.h").read_text()
        declared = set(re.findall(r"\b(dogblob_[a-z0-9_]+)\s*\(", header))
        assert len(declared) >= 20
        lib = _lib.load()
        raw = ctypes.CDLL(str(_lib.LIB_PATH))
        for name in sorted(declared):
            assert hasattr(raw, name), f"{name} declared in the header but not exported"
        assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
        assert lib.dogblob_abi_version() == 1

    def test_struct_sizes(self):
        lib = _lib.load()
        assert _lib.BLOB_DTYPE.itemsize == 48
        assert lib.dogblob_result_bytes_for(10) == 64 + 10 * 48
        assert lib.dogblob_blobspace_bytes(1000) > 1000 * 48 * 2

    def test_argument_errors_without_touching_the_gpu(self):
        lib = _lib.load()
        handle = ctypes.c_void_p()
        rc = lib.dogblob_plan_create(0, 0, 16, 2, None, None, None, None, 16, ctypes.byref(handle))
        assert rc == _lib.EINVAL
        with pytest.raises(ValueError, match="non-empty"):
            _lib.check(rc)
        assert lib.dogblob_prune(5, None, 2.0, 8, None, None, None) == _lib.EINVAL
