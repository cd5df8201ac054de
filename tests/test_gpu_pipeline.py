"""End-to-end blob-set parity of Detector.run (H2D -> kernels -> D2H through the
C ABI) against the reference's outputs on the BASELINE.json configurations.

Rule (BASELINE.json north_star): centres and sigma levels are bit-exact except
for peaks whose float64 DoG response lies within sigma_i * EPS_REL of the
threshold or of a neighbour tie (parity.EPS_REL = 2e-6); those are counted and
printed.  Pruning, ordering and the histogram are checked bit-exactly on the
GPU's own candidate list with the oracle.
"""

import threading

import numpy as np
import pytest

import paper_2010_08486_b200 as P
from oracle import dog_oracle as O
from paper_2010_08486_b200 import synth
import parity
from parity import (EPS_REL, classify_candidates, golden_blobs, oblob_tuples, records_tuples)

pytestmark = pytest.mark.gpu


def params_for(name, **kw):
    return P.DetectionParams(preprocess=False, **synth.config_params(name), **kw)


def to_oblobs(tuples):
    return [O.OBlob(int(x), int(y), s, r, v, e) for x, y, s, r, v, e in tuples]


def check_frame(frame, params, want_cand, want_kept, label, t1_cand=None):
    """Run the detector with and without pruning and compare with the reference; the outcome
    goes into the parity report (profiles/rNN_parity.json)."""
    det_raw = P.Detector(P.DetectionParams(**{**params.to_dict(), "prune": False}))
    det = P.Detector(params)
    try:
        cand = records_tuples(det_raw.run(frame).blobs.records)
        res = det.run(frame)
        kept = records_tuples(res.blobs.records)
    finally:
        det_raw.close()
        det.close()
    sig, rad = det.ladder.sigmas, det.bank.radii
    rep = classify_candidates(frame, sig, rad, params.threshold, cand, want_cand, params.neighborhood)
    print(f"\n[{label}] candidates gpu={len(cand)} ref={len(want_cand)} common={len(rep['common'])} "
          f"fragile-explained={len(rep['explained'])} unexplained={len(rep['unexplained'])} "
          f"max |dresponse| = {rep['max_resp_diff_in_eps']:.3f} eps; kept gpu={len(kept)} ref={len(want_kept)}")
    for k, margin, eps in rep["explained"]:
        print(f"    fragile voxel (slice,y,x)={k}: float64 margin {margin:.3e} <= eps {eps:.3e}")
    strip = lambda ts: [(t[0], t[1], t[2], t[3], t[5]) for t in ts]
    entry = {"gpu_vs_reference": parity.report_entry(rep, len(cand), len(want_cand)),
             "kept_gpu": len(kept), "kept_ref": len(want_kept),
             "kept_only_gpu": len(set(strip(kept)) - set(strip(want_kept))),
             "kept_only_ref": len(set(strip(want_kept)) - set(strip(kept)))}
    if t1_cand is not None:
        entry["reference_t0_vs_t1"] = parity.reference_t0_vs_t1(frame, sig, rad, params.threshold, want_cand, t1_cand)
    parity.REPORT[label] = entry
    assert not rep["unexplained"], rep["unexplained"]
    assert rep["max_resp_diff_in_eps"] <= 1.0
    # pruning / ordering / histogram: exact on the GPU's own candidates
    want = O.prune(to_oblobs(cand), params.overlap)
    assert strip(kept) == strip(oblob_tuples(want))
    assert [t[4] for t in kept] == [t[4] for t in oblob_tuples(want)]
    h = O.radius_histogram(want, sig)
    assert np.array_equal(res.histogram.counts, h.counts)
    assert np.array_equal(res.histogram.volume_weights, h.volume_weights)
    # The reference's list, edited by EXACTLY the fragile voxels (those only the GPU has are inserted
    # with the GPU's response, those only the reference has are removed): the common candidates must
    # come in the same order except where two responses are within the float32 epsilon of each
    # other, and without such swaps the pruned lists must be identical.
    key = lambda t: (t[2], t[1], t[0])
    fragile = {(float(sig[k[0]]), k[1], k[2]) for k, _, _ in rep["explained"]}
    hybrid = [t for t in want_cand if key(t) not in fragile] + [t for t in cand if key(t) in fragile]
    hybrid.sort(key=lambda t: (-t[4], t[1], t[0], t[2]))
    assert sorted(strip(cand)) == sorted(strip(hybrid))
    swaps = [(a, b) for a, b in zip(cand, hybrid) if strip([a]) != strip([b])]
    entry["order_swaps_within_eps"] = len(swaps)
    for a, b in swaps:
        eps = max(a[2], b[2]) * EPS_REL
        assert abs(a[4] - b[4]) <= 2 * eps, (a, b)
    kept_hybrid = oblob_tuples(O.prune(to_oblobs(hybrid), params.overlap))
    diff = set(strip(kept)) ^ set(strip(kept_hybrid))
    entry["kept_differs_from_edited_reference"] = len(diff)
    if not swaps:
        assert strip(kept) == strip(kept_hybrid)
        if not rep["explained"]:
            assert strip(kept) == strip(want_kept)
    else:
        print(f"    {len(swaps)} positions re-ordered by near-equal responses; "
              f"{len(diff)} kept blobs differ through them")
        assert len(diff) <= 4 * len(swaps)
    return rep, res


class TestConfigs:
    def test_c1_512(self, golden):
        g = golden("config_C1.npz")
        rep, res = check_frame(synth.config_frame("C1"), params_for("C1"),
                               golden_blobs(g, "t0_cand_"), golden_blobs(g, "t0_kept_"), "C1",
                    t1_cand=golden_blobs(g, "t1_cand_"))
        assert set(res.timings_ms) == {"preprocess_ms", "convolve_ms", "extrema_ms", "prune_ms"}

    def test_c2_1024(self, golden):
        g = golden("config_C2.npz")
        check_frame(synth.config_frame("C2"), params_for("C2"),
                    golden_blobs(g, "t0_cand_"), golden_blobs(g, "t0_kept_"), "C2",
                    t1_cand=golden_blobs(g, "t1_cand_"))

    @pytest.mark.parametrize("f", [0, 1, 2, 3])
    def test_c3_frames(self, golden, f):
        g = golden("config_C3.npz")
        check_frame(synth.config_frame("C3", f), params_for("C3"),
                    golden_blobs(g, f"f{f}_t0_cand_"), golden_blobs(g, f"f{f}_t0_kept_"), f"C3[{f}]")

    def test_c4_2048_wide_filters(self, golden):
        g = golden("config_C4.npz")
        check_frame(synth.config_frame("C4"), params_for("C4"),
                    golden_blobs(g, "t0_cand_"), golden_blobs(g, "t0_kept_"), "C4",
                    t1_cand=golden_blobs(g, "t1_cand_"))

    def test_c5_dense(self, golden):
        g = golden("config_C5.npz")
        check_frame(synth.config_frame("C5"), params_for("C5"),
                    golden_blobs(g, "t0_cand_"), golden_blobs(g, "t0_kept_"), "C5",
                    t1_cand=golden_blobs(g, "t1_cand_"))

    def test_scene256(self, golden):
        g = golden("scene256.npz")
        frame = synth.sensor_noise(synth.droplet_scene(256, 256, 12, (4.0, 12.0), seed=5), seed=6).image
        p = P.DetectionParams(min_sigma=2.5, max_sigma=9.0, n_bin=10, preprocess=False)
        check_frame(frame, p, golden_blobs(g, "t0_cand_"), golden_blobs(g, "t0_kept_"), "scene256")

    def test_non_multiple_of_tile_shape(self):
        """1000 x 900 frame (padding path) against the oracle run live"""
        frame = synth.sensor_noise(synth.droplet_scene(1000, 900, 60, (4.0, 20.0), seed=11,
                                                       allow_overlap=True), seed=12).image
        kw = dict(min_sigma=2.0, max_sigma=12.0, n_bin=10)
        ref = O.OracleDetector(preprocess=False, **kw).run(frame)
        check_frame(frame, P.DetectionParams(preprocess=False, **kw),
                    oblob_tuples(ref.candidates), oblob_tuples(ref.blobs), "1000x900")


class TestRandomisedParity:
    """Seeded random frames, ladders and detection parameters against the oracle run live, on both
    convolution engines (ragged shapes, 5^3 neighbourhoods, low thresholds on sensor noise,
    overlap thresholds either side of the default)."""

    @pytest.mark.parametrize("engine", ["fma", "umma"])
    @pytest.mark.parametrize("seed", range(6))
    def test_random_case(self, monkeypatch, seed, engine):
        monkeypatch.setenv("DOGBLOB_CONV", engine)
        rng = np.random.default_rng(1000 + seed)
        H, W = int(rng.integers(200, 560)), int(rng.integers(200, 560))
        lo = float(rng.choice([1.0, 1.5, 2.0, 3.0]))
        kw = dict(min_sigma=lo, max_sigma=lo + float(rng.uniform(3, 16)), n_bin=int(rng.integers(3, 22)),
                  threshold=float(rng.choice([0.03, 0.05, 0.1, 0.2])), neighborhood=int(rng.choice([3, 3, 5])),
                  overlap=float(rng.choice([0.3, 0.5, 0.8])))
        frame = synth.sensor_noise(synth.droplet_scene(W, H, int(rng.integers(5, 60)), (2.5, 24.0),
                                                       seed=int(rng.integers(1 << 30)), allow_overlap=True),
                                   seed=int(rng.integers(1 << 30))).image
        ref = O.OracleDetector(preprocess=False, **kw).run(frame)
        check_frame(frame, P.DetectionParams(preprocess=False, **kw), oblob_tuples(ref.candidates),
                    oblob_tuples(ref.blobs), f"random{seed}_{engine}_{H}x{W}")


class TestDetectorBehaviour:
    def test_blank_and_dark_images_yield_nothing(self):
        p = P.DetectionParams(min_sigma=1, max_sigma=4, n_bin=6, preprocess=False)
        blobs, hist = P.detect(np.zeros((64, 64), dtype=np.float32), p)
        assert len(blobs) == 0 and hist.counts.sum() == 0
        img = 1.0 - synth.flat_disk(128, 128, 64, 64, 10.0)
        blobs, _ = P.detect(img, P.DetectionParams(min_sigma=4, max_sigma=10, n_bin=12, preprocess=False))
        assert len(blobs) == 0

    def test_detector_reusable_and_deterministic(self):
        img = synth.flat_disk(96, 96, 48, 48, 8.0)
        det = P.Detector(P.DetectionParams(min_sigma=3, max_sigma=9, n_bin=8, preprocess=False))
        r1, r2 = det.run(img), det.run(img)
        assert r1.blobs == r2.blobs and len(r1.blobs) >= 1
        assert set(r1.timings_ms) == {"preprocess_ms", "convolve_ms", "extrema_ms", "prune_ms"}
        assert r1.blobs.source_shape == (96, 96)
        assert r1.blobs.yxs().shape == (len(r1.blobs), 3)
        det.close()

    def test_run_batch_equals_run_and_pinned_inputs(self):
        import torch
        det = P.Detector(params_for("C1"), slots=3)
        frames = [synth.sensor_noise(synth.droplet_scene(512, 512, 30, (3.0, 15.0), seed=50 + i,
                                                         allow_overlap=True), seed=90 + i).image
                  for i in range(7)]
        single = [det.run(f) for f in frames]
        batch = det.run_batch(frames)
        pinned = det.run_batch([torch.from_numpy(f).pin_memory() for f in frames])
        for a, b, c in zip(single, batch, pinned):
            assert np.array_equal(a.blobs.records, b.blobs.records)
            assert np.array_equal(a.blobs.records, c.blobs.records)
            assert np.array_equal(a.histogram.counts, b.histogram.counts)
        det.close()

    def test_dense_frames_on_concurrent_streams(self):
        """several whole-GPU pruning kernels (device-chained phases, ticket-ordered waits) in
        flight at once, next to the convolution kernels of other frames: same result as one
        frame at a time, and the phase profile is reported"""
        det = P.Detector(params_for("C5", overlap=0.3), slots=4)
        frames = [synth.sensor_noise(synth.droplet_scene(512, 512, 3000 + 400 * i, (2.0, 5.0), seed=70 + i,
                                                         allow_overlap=True), seed=80 + i).image
                  for i in range(6)] + [synth.config_frame("C1")]
        single = [det.run(f) for f in frames]
        assert single[0].stats["n_candidates"] > 1500 and single[0].stats["n_merges"] > 0
        assert single[0].stats["prune_profile"]["parts"] > 0
        for _ in range(3):
            batch = det.run_batch(frames)
            for a, b in zip(single, batch):
                assert np.array_equal(a.blobs.records, b.blobs.records)
                assert a.stats["n_merges"] == b.stats["n_merges"]
        det.close()

    @pytest.mark.parametrize("shape,kw", [((600, 700), dict(min_sigma=1.0, max_sigma=8.0, n_bin=7)),
                                          ((515, 520), dict(min_sigma=30.0, max_sigma=120.0, n_bin=3)),
                                          ((1024, 1024), dict(min_sigma=2.0, max_sigma=12.0, n_bin=10))])
    def test_streamed_upload_equals_plain_upload(self, shape, kw, monkeypatch):
        """FP32 engine: large frames go up in row chunks under the running row pass (gate word per
        chunk); same records as the single pitched copy, also when the widest kernel exceeds the
        image (every tile then waits for the whole frame) and with ragged last chunks (the size
        threshold is lowered to 1 MiB for the test)"""
        from paper_2010_08486_b200 import detector as D
        monkeypatch.setenv("DOGBLOB_CONV", "fma")
        monkeypatch.setattr(D, "STREAM_MIN_BYTES_FP32", 1 << 20)
        frames = [synth.sensor_noise(synth.droplet_scene(shape[1], shape[0], 40, (3.0, 14.0), seed=11 + i,
                                                         allow_overlap=True), seed=31 + i).image for i in range(3)]
        params = P.DetectionParams(preprocess=False, **kw)
        monkeypatch.setattr(D, "STREAMED_UPLOAD", False)
        det = P.Detector(params)
        plain = [det.run(f).blobs.records for f in frames]
        eng = det.plan_for(shape)
        assert eng.plan.conv_engine == 0 and not any(s.streamed for s in eng.slots)
        det.close()
        monkeypatch.setattr(D, "STREAMED_UPLOAD", True)
        det = P.Detector(params, slots=2)
        for _ in range(3):                               # the gate counter advances from frame to frame
            for f, want in zip(frames, plain):
                assert np.array_equal(det.run(f).blobs.records, want)
        for got, want in zip(det.run_batch(frames * 2), plain * 2):
            assert np.array_equal(got.blobs.records, want)
        eng = det.plan_for(shape)
        assert eng.plan.conv_engine == 0 and all(s.streamed for s in eng.slots)      # the streamed entry really ran
        det.close()

    def test_tensor_engine_uploads_in_one_piece(self, monkeypatch):
        """the fp16 operand split needs the frame's maximum first: tensor-engine plans never use the
        streamed upload, and the C entry point refuses it instead of silently falling back"""
        import ctypes as C
        from paper_2010_08486_b200 import _lib, detector as D
        monkeypatch.setenv("DOGBLOB_CONV", "umma")
        monkeypatch.setattr(D, "STREAM_MIN_BYTES_FP32", 1 << 20)
        frame = synth.sensor_noise(synth.droplet_scene(700, 600, 40, (3.0, 14.0), seed=11, allow_overlap=True),
                                   seed=31).image
        params = P.DetectionParams(preprocess=False, min_sigma=2.0, max_sigma=12.0, n_bin=10)
        det = P.Detector(params, slots=1)
        det.run(frame)
        eng = det.plan_for(frame.shape)
        slot = eng.slots[0]
        assert eng.plan.conv_engine == 2 and not slot.streamed
        lib = _lib.load()
        rc = lib.dogblob_detect_host_streamed(
            eng.plan.handle, slot.h_image.data_ptr(), 0.1, 3, 0.5, 1, slot.d_image.data_ptr(),
            slot.d_work.data_ptr(), slot.d_result.data_ptr(), slot.h_result.data_ptr(), slot.n_host,
            slot.stream.cuda_stream, slot.copy_stream.cuda_stream, slot.h_gate.data_ptr(), slot.frame_done, None)
        assert rc == _lib.EINVAL and b"FP32 engine" in lib.dogblob_last_error()
        det.close()

    def test_shared_detector_from_threads(self):
        det = P.Detector(params_for("C1"), slots=2)
        frame = synth.config_frame("C1")
        want = det.run(frame).blobs.records
        out = [None] * 8

        def work(i):
            out[i] = det.run(frame).blobs.records

        ts = [threading.Thread(target=work, args=(i,)) for i in range(8)]
        [t.start() for t in ts]
        [t.join() for t in ts]
        assert all(np.array_equal(o, want) for o in out)
        det.close()

    def test_run_batch_from_two_threads_shares_the_slot_pool(self):
        """two concurrent batches on one Detector (the service's /detect_batch with workers >= 2):
        each takes one slot for certain and the others only if free - neither waits for a slot the
        other holds"""
        det = P.Detector(params_for("C1"), slots=2)
        frames = [synth.config_frame("C1")] * 6
        want = det.run(frames[0]).blobs.records
        out, errs = [None, None], []

        def work(i):
            try:
                out[i] = det.run_batch(frames)
            except Exception as e:       # pragma: no cover
                errs.append(e)

        ts = [threading.Thread(target=work, args=(i,), daemon=True) for i in range(2)]
        [t.start() for t in ts]
        [t.join(timeout=120) for t in ts]
        assert not any(t.is_alive() for t in ts), "run_batch callers deadlocked"
        assert not errs, errs
        for res in out:
            assert len(res) == 6 and all(np.array_equal(r.blobs.records, want) for r in res)
        det.close()

    def test_concurrent_capacity_growth_keeps_engines_alive(self):
        """several threads overflow the candidate capacity at once: the engine is replaced once per
        overflow level and the old one is closed only after its last user has returned its slot"""
        det = P.Detector(params_for("C5"), max_blobs=2048, slots=2)
        frame = synth.config_frame("C5")
        out, errs = [None] * 4, []

        def work(i):
            try:
                out[i] = det.run(frame).blobs.records
            except Exception as e:       # pragma: no cover
                errs.append(e)

        ts = [threading.Thread(target=work, args=(i,), daemon=True) for i in range(4)]
        [t.start() for t in ts]
        [t.join(timeout=300) for t in ts]
        assert not any(t.is_alive() for t in ts) and not errs, errs
        assert all(np.array_equal(o, out[0]) for o in out) and len(out[0]) > 2048
        assert det._max_blobs == 2048 * 4 * 4          # 2048 -> 8192 -> 32768: grown once per level, not per thread
        det.close()

    def test_workspace_beyond_device_memory_is_a_parameter_error(self):
        det = P.Detector(P.DetectionParams(min_sigma=1.0, max_sigma=4.0, n_bin=300, preprocess=False), slots=2)
        with pytest.raises(ValueError, match="exceeds the device memory"):
            det.run(np.zeros((16384, 16384), dtype=np.float32))
        det.close()

    def test_convolve_bank_accepts_the_detectors_plan(self):
        det = P.Detector(params_for("C1"))
        frame = synth.config_frame("C1")
        bank = det.bank
        a = P.convolve_bank(frame, bank, plan=det.plan_for(frame.shape)).levels
        assert np.array_equal(a, P.convolve_bank(frame, bank).levels)
        det.close()

    def test_candidate_capacity_growth(self):
        det = P.Detector(params_for("C5"), max_blobs=512)
        big = P.Detector(params_for("C5"))
        frame = synth.config_frame("C5")
        assert np.array_equal(det.run(frame).blobs.records, big.run(frame).blobs.records)
        det.close(); big.close()

    def test_errors(self):
        det = P.Detector(params_for("C1"))
        with pytest.raises(ValueError):
            det.run(np.zeros((4, 4, 3), np.float32))
        with pytest.raises(ValueError, match="float32 or float64"):
            det.run(np.zeros((16, 16), np.float32), dtype=np.int32)
        det.close()


class TestFullSizeProperties:
    """Size-independent checks at the BASELINE.json sizes."""

    def test_constant_frame_has_zero_dog_and_no_blobs(self):
        det = P.Detector(params_for("C2"))
        assert len(det.run(np.full((1024, 1024), 0.7, np.float32)).blobs) == 0
        det.close()

    def test_transpose_equivariance(self):
        """detections of a transposed frame are the transposed detections; the row
        and column passes round differently, so differences must all be fragile
        near-ties in float64 (same classifier as the reference comparison)"""
        frame = synth.config_frame("C3", 5)
        det = P.Detector(params_for("C2", prune=False))
        a = records_tuples(det.run(frame).blobs.records)
        b = records_tuples(det.run(np.ascontiguousarray(frame.T)).blobs.records)
        sig, rad = det.ladder.sigmas, det.bank.radii
        det.close()
        b_back = [(t[1], t[0]) + t[2:] for t in b]
        rep = classify_candidates(frame, sig, rad, 0.1, a, b_back)
        print(f"\n[transpose] common={len(rep['common'])} fragile={len(rep['explained'])} "
              f"unexplained={len(rep['unexplained'])}")
        assert not rep["unexplained"] and len(rep["common"]) >= 0.9 * len(a)

    def test_scaling_linearity_of_responses(self):
        frame = synth.config_frame("C1")
        det = P.Detector(params_for("C1", prune=False, threshold=0.05))
        det2 = P.Detector(params_for("C1", prune=False, threshold=0.1))
        a = det.run(frame).blobs.records
        b = det2.run((2.0 * frame).astype(np.float32)).blobs.records   # exact power-of-two scaling
        det.close(); det2.close()
        assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["y"], b["y"])
        assert np.array_equal(a["sigma"], b["sigma"])
        assert np.array_equal(2.0 * a["response"], b["response"])

    def test_impulse_response_sums(self):
        """an impulse spreads to unit-sum levels: sum over the plane of each DoG slice ~ 0"""
        img = np.zeros((512, 512), np.float32)
        img[200, 300] = 1.0
        bank = P.build_kernel_bank(P.build_ladder(1.0, 10.0, 18))
        dog = P.fused_dog(img, bank).slices.astype(np.float64)
        assert np.abs(dog.sum(axis=(1, 2))).max() < 1e-4


class TestPreprocess:
    """images.preprocess on the GPU, bit-exact against the reference."""

    def test_preprocess_bit_exact(self, golden):
        g = golden("scene256.npz")
        frame = synth.sensor_noise(synth.droplet_scene(256, 256, 12, (4.0, 12.0), seed=5), seed=6).image
        got = P.preprocess(frame)
        assert got.dtype == np.float32 and np.array_equal(got, g["pre_image"])

    @pytest.mark.parametrize("shape,sigma,sat", [((97, 131), 1.0, 0.0035), ((64, 200), 2.3, 0.01),
                                                  ((33, 47), 0.0, 0.0), ((1, 50), 1.0, 0.1),
                                                  ((300, 1), 0.7, 0.3), ((120, 90), 20.0, 0.02),
                                                  ((64, 64), 50.0, 0.0035)])      # radius 100 / 250: wider than the image
    def test_preprocess_against_oracle(self, shape, sigma, sat):
        rng = np.random.default_rng(shape[0] + shape[1])
        img = (rng.random(shape) ** 3).astype(np.float32)
        assert np.array_equal(P.preprocess(img, sigma, sat), O.preprocess(img, sigma, sat))

    def test_constant_image_maps_to_zero_and_errors(self):
        assert np.array_equal(P.preprocess(np.full((40, 40), 0.3, np.float32)), np.zeros((40, 40), np.float32))
        bad = np.ones((8, 8), np.float32)
        bad[3, 3] = np.nan
        with pytest.raises(ValueError, match="NaN"):
            P.preprocess(bad)
        with pytest.raises(ValueError):
            P.preprocess(np.ones((8, 8), np.float32), saturation=0.7)
        with pytest.raises(ValueError):
            P.preprocess(np.ones((8, 8), np.float32), smooth_sigma=-1.0)

    def test_detector_with_default_preprocess(self, golden):
        g = golden("scene256.npz")
        frame = synth.sensor_noise(synth.droplet_scene(256, 256, 12, (4.0, 12.0), seed=5), seed=6).image
        det = P.Detector(P.DetectionParams(min_sigma=2.5, max_sigma=9.0, n_bin=10))   # preprocess=True
        res = det.run(frame)
        det.close()
        strip = lambda ts: [(t[0], t[1], t[2], t[3], t[5]) for t in ts]
        assert strip(records_tuples(res.blobs.records)) == strip(golden_blobs(g, "pre_kept_"))
        assert res.timings_ms["preprocess_ms"] > 0.0

    def test_reference_demo_golden_vector_on_gpu(self):
        """The reference's own committed fixture pkg/demos/output/03_blobs.json (1000x1000
        scene, sigma 2.5..15, n_bin 25, preprocess ON): every blob reproduced on the GPU."""
        import json
        from conftest import GOLDEN
        doc = json.loads((GOLDEN / "ref_demo03_blobs.json").read_text())
        frame = synth.sensor_noise(synth.droplet_scene(1000, 1000, 100, (4.0, 20.0), seed=123),
                                   seed=124).image
        kw = {k: v for k, v in doc["params"].items() if k != "backend"}
        det = P.Detector(P.DetectionParams(**kw))
        res = det.run(frame)
        got = records_tuples(res.blobs.records)
        want = [(b["x"], b["y"], b["sigma"], b["radius"], b["response"], b["at_scale_boundary"])
                for b in doc["blobs"]]
        pre = O.preprocess(frame)
        rep = classify_candidates(pre, det.ladder.sigmas, det.bank.radii, kw["threshold"], got, want)
        det.close()
        print(f"\n[demo03] gpu={len(got)} ref={len(want)} common={len(rep['common'])} "
              f"fragile={len(rep['explained'])} unexplained={len(rep['unexplained'])}")
        assert not rep["unexplained"]
        if not rep["explained"]:
            strip = lambda ts: [(t[0], t[1], t[2], t[3], t[5]) for t in ts]
            assert strip(got) == strip(want)
            rows = (GOLDEN / "ref_demo03_histogram.csv").read_text().strip().splitlines()[1:]
            for row, c, n, v in zip(rows, res.histogram.bin_centers, res.histogram.counts,
                                    res.histogram.volume_weights):
                assert row == f"{float(c)!r},{int(n)},{float(v)!r}"


class TestFormats:
    """raw frame file -> pinned memory -> detector -> the reference's JSON / CSV."""

    def test_raw_file_to_pinned_to_blob_json(self, tmp_path):
        import json
        import torch
        from conftest import GOLDEN
        from paper_2010_08486_b200 import formats as F
        frame = synth.sensor_noise(synth.droplet_scene(1000, 1000, 100, (4.0, 20.0), seed=123),
                                   seed=124).image
        F.write_raw(tmp_path / "frame.raw", frame)
        pinned = F.read_raw_pinned(tmp_path / "frame.raw")
        assert isinstance(pinned, torch.Tensor) and pinned.is_pinned()
        assert np.array_equal(pinned.numpy(), frame)
        ring = torch.empty(1200 * 1000, dtype=torch.float32).pin_memory()        # re-used staging buffer
        again = F.raw_into_pinned((tmp_path / "frame.raw").read_bytes(), out=ring)
        assert again.data_ptr() == ring.data_ptr() and np.array_equal(again.numpy(), frame)
        doc = json.loads((GOLDEN / "ref_demo03_blobs.json").read_text())
        kw = {k: v for k, v in doc["params"].items() if k != "backend"}
        det = P.Detector(P.DetectionParams(**kw))
        res = det.run(pinned)
        res2 = det.run(again)
        det.close()
        assert np.array_equal(res.blobs.records, res2.blobs.records)
        # same blobs as the reference file (responses differ in the last float32 bits, so the
        # bytes are compared after substituting the reference's responses)
        text = F.blobs_json_text(res.blobs, "demo_scene")
        got = json.loads(text)
        assert got["params"] == {**doc["params"], "backend": "cuda"}
        strip = lambda bl: [(b["x"], b["y"], b["sigma"], b["radius"], b["at_scale_boundary"]) for b in bl]
        assert strip(got["blobs"]) == strip(doc["blobs"])
        assert max(abs(a["response"] - b["response"]) for a, b in zip(got["blobs"], doc["blobs"])) < 2e-5
        assert text == json.dumps(F.blobset_to_doc(res.blobs, "demo_scene"), indent=2)
        F.write_histogram_csv(tmp_path / "h.csv", res.histogram)
        assert (tmp_path / "h.csv").read_bytes() == (GOLDEN / "ref_demo03_histogram.csv").read_bytes()

    def test_pinned_ingest_rejects_bad_frames(self, tmp_path):
        from paper_2010_08486_b200 import formats as F
        img = np.ones((8, 8), np.float32)
        img[3, 3] = np.inf
        (tmp_path / "bad.raw").write_bytes(b"\x08\x00\x00\x00\x08\x00\x00\x00" + img.tobytes())
        with pytest.raises(ValueError, match="NaN or Inf"):
            F.read_raw_pinned(tmp_path / "bad.raw")
        (tmp_path / "short.raw").write_bytes(b"\x08\x00\x00\x00\x08\x00\x00\x00" + img.tobytes()[:-4])
        with pytest.raises(ValueError, match="expected 264 bytes, found 260"):
            F.read_raw_pinned(tmp_path / "short.raw")


class TestService:
    """the HTTP service and the CLI call the same detector; their JSON is the offline
    detector's, byte for byte apart from the timings (reference tests/test_service.py:82-94,
    acceptance criterion 7)."""

    @staticmethod
    def _post(port, path, body, ctype="application/octet-stream"):
        import http.client
        c = http.client.HTTPConnection("127.0.0.1", port, timeout=60)
        c.request("POST", path, body=body, headers={"Content-Type": ctype})
        r = c.getresponse()
        data = r.read()
        c.close()
        return r.status, data

    def test_service_equals_offline_detector_and_cli(self, tmp_path):
        import json
        from paper_2010_08486_b200 import cli, formats as F, service as S
        params = P.DetectionParams(min_sigma=2.5, max_sigma=9.0, n_bin=13)          # preprocess on
        frames = [synth.sensor_noise(synth.droplet_scene(400, 300, 25, (4.0, 12.0), seed=30 + i,
                                                         allow_overlap=True), seed=60 + i).image
                  for i in range(5)]
        det = P.Detector(params)
        offline = [det.run(f) for f in frames]
        det.close()
        srv = S.make_server(S.ServiceConfig(port=0, params=params, workers=2, backlog=8))
        t = threading.Thread(target=srv.serve_forever, daemon=True)
        t.start()
        port = srv.server_address[1]
        try:
            def strip(doc):
                return {k: v for k, v in doc.items() if k != "timing_ms"}

            out = [None] * len(frames)

            def work(i):
                out[i] = self._post(port, f"/detect?name=frame{i}", F.raw_to_bytes(frames[i]))

            ts = [threading.Thread(target=work, args=(i,)) for i in range(len(frames))]
            [x.start() for x in ts]
            [x.join() for x in ts]
            for i, (st, data) in enumerate(out):
                assert st == 200
                doc = json.loads(data)
                want = json.loads(F.blobs_json_text(offline[i].blobs, f"frame{i}",
                                                    extra={"histogram": F.histogram_to_doc(offline[i].histogram)}))
                assert strip(doc) == want
                assert set(doc["timing_ms"]) == {"preprocess_ms", "convolve_ms", "extrema_ms", "prune_ms"}
                assert data == (json.dumps(doc, indent=2) + "\n").encode()
            # per-request override: a second parameter set builds (and caches) a second detector
            st, data = self._post(port, "/detect?n_bin=6&preprocess=false", F.raw_to_bytes(frames[0]))
            d2 = P.Detector(P.DetectionParams(min_sigma=2.5, max_sigma=9.0, n_bin=6, preprocess=False))
            assert st == 200 and json.loads(data)["blobs"] == F.blobset_to_doc(d2.run(frames[0]).blobs)["blobs"]
            d2.close()
            # batch path: same answers as the single-frame path
            st, data = self._post(port, "/detect_batch?name=b", b"".join(F.raw_to_bytes(f) for f in frames))
            assert st == 200
            for i, fd in enumerate(json.loads(data)["frames"]):
                assert fd["blobs"] == F.blobset_to_doc(offline[i].blobs)["blobs"] and fd["image"] == f"b[{i}]"
            # detector argument errors surface as 400, like the reference's decode errors
            assert self._post(port, "/detect?min_sigma=9&max_sigma=9.5&n_bin=300", F.raw_to_bytes(frames[0]))[0] == 400
        finally:
            srv.shutdown()
            srv.server_close()
        assert srv.state.cache.closed >= 2 and len(srv.state.cache) == 0     # device memory returned
        # CLI detect on the raw file: same JSON file as the offline writer
        F.write_raw(tmp_path / "f0.raw", frames[0])
        rc = cli.main(["detect", "--input", str(tmp_path / "f0.raw"), "--min-sigma", "2.5", "--max-sigma", "9",
                       "--n-bin", "13", "--out-json", str(tmp_path / "o.json"), "--out-hist", str(tmp_path / "h.csv")])
        assert rc == 0
        assert (tmp_path / "o.json").read_text() == F.blobs_json_text(offline[0].blobs, "f0.raw") + "\n"
        assert (tmp_path / "h.csv").read_text() == F.histogram_csv_text(offline[0].histogram)

    def test_cli_bench_sweep(self, tmp_path, capsys):
        from paper_2010_08486_b200 import cli
        out = tmp_path / "sweep.csv"
        assert cli.main(["bench", "--sweep", "max_sigma", "--values", "4,8", "--seed", "3", "--width", "256",
                         "--height", "256", "--n-bin", "6", "--out", str(out)]) == 0
        rows = out.read_text().splitlines()
        assert rows[0] == ("backend,n_bin,max_sigma,width,height,warmup_runs,timed_runs,median_ms,p10_ms,"
                           "p90_ms,hardware")
        assert len(rows) == 3 and rows[1].startswith("cuda,6,4.0,256,256,1,3,")
        assert "median" in capsys.readouterr().out


class TestReferenceSideStub:
    def test_cuda_stub_of_integration_md_returns_the_detectors_records(self, monkeypatch):
        """the ctypes stub a reference maintainer drops into pkg/src/dogblob (INTEGRATION.md 2,
        paper_2010_08486_b200/integration/_cuda.py: numpy + the C ABI only, no torch) against
        Detector.run on the same frames"""
        from paper_2010_08486_b200 import _lib
        from paper_2010_08486_b200.integration import _cuda
        monkeypatch.setenv("DOGBLOB_B200_LIB", str(_lib.LIB_PATH))
        for name in ("C1", "C2"):
            frame = synth.config_frame(name)
            params = params_for(name)
            det = P.Detector(params)
            want = det.run(frame).blobs.records
            plan = _cuda.CudaPlan(det.ladder, det.bank, frame.shape)
            try:
                for _ in range(2):
                    got = plan.detect(frame, np.float32(params.threshold), params.neighborhood, params.overlap,
                                      params.prune)
                    assert got.dtype == _cuda.BLOB and np.array_equal(got, want.astype(_cuda.BLOB))
            finally:
                plan.close()
                det.close()


class TestFloat64Detector:
    """Detector.run(img, dtype=np.float64): the reference's T1 tier (float64 / direct) on the device."""

    @pytest.mark.parametrize("name", ["C1", "C2", "C5"])
    def test_float64_run_equals_the_reference_t1_lists(self, golden, name):
        g = golden(f"config_{name}.npz")
        det = P.Detector(params_for(name))
        res = det.run(synth.config_frame(name), dtype=np.float64)
        det.close()
        strip = lambda ts: [(t[0], t[1], t[2], t[3], t[5]) for t in ts]
        got, want = records_tuples(res.blobs.records), golden_blobs(g, "t1_kept_")
        assert strip(got) == strip(want)
        assert max(abs(a[4] - b[4]) for a, b in zip(got, want)) < 1e-12
        assert set(res.timings_ms) == {"preprocess_ms", "convolve_ms", "extrema_ms", "prune_ms"}

    def test_float64_candidates_without_pruning(self, golden):
        g = golden("config_C2.npz")
        p = P.DetectionParams(**{**params_for("C2").to_dict(), "prune": False})
        det = P.Detector(p)
        got = records_tuples(det.run(synth.config_frame("C2"), dtype=np.float64).blobs.records)
        det.close()
        want = golden_blobs(g, "t1_cand_")
        assert [(t[0], t[1], t[2]) for t in got] == [(t[0], t[1], t[2]) for t in want]


class TestDeviceEvaluation:
    """scoring and scene generation on the device for large sweeps."""

    def test_device_matcher_equals_host_matcher(self):
        from paper_2010_08486_b200 import evaluate as ev
        from test_evaluate import random_case
        rng = np.random.default_rng(77)
        cases = [random_case(rng, int(rng.integers(0, 60)), int(rng.integers(0, 60)),
                             span=25 if k % 2 else 80, integer=k % 3 == 0) for k in range(24)]
        cases.append(random_case(rng, 1500, 1400, span=600))          # more truths than threads
        for thr in (0.5, 0.15):
            got = ev.match_voc_batch([c[0] for c in cases], [c[1] for c in cases], thr)
            for (preds, truths), g in zip(cases, got):
                assert g == ev.match_voc(preds, truths, thr)

    def test_device_frames_have_the_scene_statistics(self):
        frames, truths = synth.device_frames(6, 512, 384, 40, (3.0, 15.0), seed=5)
        assert tuple(frames.shape) == (6, 384, 512) and truths.shape == (6, 40, 3)
        f = frames.cpu().numpy()
        assert np.isfinite(f).all() and f.min() >= 0.0 and 0.9 < f.max() < 1.6
        # droplets are where the truth says: bright centres, dark background (median ~ read noise)
        for k in range(6):
            for x, y, r in truths[k][:10]:
                assert f[k, int(round(y)), int(round(x))] > 0.5
                assert 3.0 <= r <= 15.0 and r + 1 <= x <= 512 - 2 - r and r + 1 <= y <= 384 - 2 - r
            assert np.median(f[k]) < 0.02
        # same seed, same frames; another seed, other frames
        again, _ = synth.device_frames(6, 512, 384, 40, (3.0, 15.0), seed=5)
        other, _ = synth.device_frames(6, 512, 384, 40, (3.0, 15.0), seed=6)
        assert torch_equal(frames, again) and not torch_equal(frames, other)
        # noise-free frames reproduce the host painter's sphere caps
        clean, tr = synth.device_frames(1, 256, 256, 8, (4.0, 12.0), seed=9, photons=0.0, read_sigma=0.0)
        host = np.zeros((256, 256), np.float32)
        for x, y, r in tr[0]:
            synth.paint_droplet(host, synth.Droplet(x, y, r))
        assert np.abs(clean[0].cpu().numpy() - host).max() < 1e-6

    def test_detection_scores_on_device_frames(self):
        """end to end on the device: generate, detect (resident frames), score - the droplets are found"""
        from paper_2010_08486_b200 import evaluate as ev
        frames, truths = synth.device_frames(4, 512, 512, 30, (4.0, 14.0), seed=11)
        det = P.Detector(P.DetectionParams(min_sigma=2.0, max_sigma=12.0, n_bin=20, preprocess=False))
        blobs = [det.run(frames[k]).blobs for k in range(4)]
        det.close()
        reps = ev.match_voc_batch(blobs, [[synth.Droplet(*t) for t in truths[k]] for k in range(4)], 0.5)
        assert all(r.recall > 0.6 and r.precision > 0.6 for r in reps), [(r.precision, r.recall) for r in reps]


def torch_equal(a, b):
    import torch
    return bool(torch.equal(a, b))


class TestStaleSliceMemory:
    """The tensor engine does not store DoG boxes without a value above the threshold and the extrema
    kernel reads blocks without a hit as -inf: whatever an older frame left in a slot's slice buffer
    must never show up in a later result."""

    def test_frame_sequences_through_one_slot_equal_fresh_detectors(self):
        params = params_for("C2")
        frames = {"a": synth.config_frame("C3", 0), "b": synth.config_frame("C3", 1),
                  "blank": np.zeros((1024, 1024), np.float32),
                  "bright": np.full((1024, 1024), 0.9, np.float32) + synth.config_frame("C3", 2),
                  "sparse": np.where(np.add.outer(np.arange(1024), np.arange(1024)) % 512 < 40,
                                     synth.config_frame("C3", 3), 0).astype(np.float32)}
        want = {}
        for k, f in frames.items():
            det = P.Detector(params, slots=1)
            want[k] = det.run(f).blobs.records
            det.close()
        det = P.Detector(params, slots=1)
        assert det.plan_for((1024, 1024)).plan.conv_engine == 2
        for k in ["a", "b", "a", "blank", "a", "bright", "sparse", "b", "sparse", "blank", "bright", "a"]:
            assert np.array_equal(det.run(frames[k]).blobs.records, want[k]), k
        # other thresholds on the same slot: the validity map follows the threshold of the call
        lo = P.Detector(P.DetectionParams(**{**params.to_dict(), "threshold": 0.02}), slots=1)
        hi = P.Detector(P.DetectionParams(**{**params.to_dict(), "threshold": 0.3}), slots=1)
        w_lo, w_hi = lo.run(frames["a"]).blobs.records, hi.run(frames["a"]).blobs.records
        for d, w in ((hi, w_hi), (lo, w_lo)):
            d.run(frames["bright"]); d.run(frames["b"])
            assert np.array_equal(d.run(frames["a"]).blobs.records, w)
        for d in (det, lo, hi):
            d.close()


class TestSeedList:
    """Tensor engine, 3^3 neighbourhood: the column pass hands the extrema kernel a list of seeds (values
    above the threshold that none of the in-slice neighbours it holds in registers exceeds).  The list
    path, the strip kernel without a list (DOGBLOB_SEED_CAP=0 at plan creation) and the strip kernel as
    the overflow fallback (a list far too short) must return the same records."""

    @pytest.mark.parametrize("name,frame_of", [("C2", lambda: synth.config_frame("C2")),
                                               ("C2", lambda: synth.config_frame("C3", 5)),
                                               ("C4", lambda: synth.config_frame("C4"))])
    def test_seed_list_equals_strip_kernel_and_overflow_fallback(self, monkeypatch, name, frame_of):
        params = P.DetectionParams(**{**params_for(name).to_dict(), "prune": False})
        frame = frame_of()
        got = {}
        for cap in (None, "0", "4096"):
            if cap is None:
                monkeypatch.delenv("DOGBLOB_SEED_CAP", raising=False)
            else:
                monkeypatch.setenv("DOGBLOB_SEED_CAP", cap)
            det = P.Detector(params, slots=1)
            assert det.plan_for(frame.shape).plan.conv_engine == 2
            res = det.run(frame)
            res2 = det.run(frame)
            assert np.array_equal(res.blobs.records, res2.blobs.records)
            got[cap] = (res.blobs.records, res.stats["n_seeds"])
            det.close()
        n_seeds = got[None][1]
        assert n_seeds > len(got[None][0]) > 0            # every maximum is a seed; most seeds are not maxima
        assert got["0"][1] == 0                           # no list: nothing is appended
        assert got["4096"][1] == n_seeds > 4096           # the count runs past the capacity: incomplete list
        assert np.array_equal(got[None][0], got["0"][0])
        assert np.array_equal(got[None][0], got["4096"][0])

    def test_low_threshold_on_noise(self, monkeypatch):
        """many seeds (noise maxima above a low threshold), frame edges inside the last chunk"""
        frame = synth.sensor_noise(synth.droplet_scene(1000, 900, 60, (4.0, 20.0), seed=11, allow_overlap=True),
                                   seed=12).image
        kw = dict(min_sigma=1.0, max_sigma=24.0, n_bin=40, threshold=0.01, preprocess=False, prune=False)
        got = {}
        for cap in (None, "0"):
            if cap is None:
                monkeypatch.delenv("DOGBLOB_SEED_CAP", raising=False)
            else:
                monkeypatch.setenv("DOGBLOB_SEED_CAP", cap)
            det = P.Detector(P.DetectionParams(**kw), slots=1)
            assert det.plan_for(frame.shape).plan.conv_engine == 2
            got[cap] = det.run(frame).blobs.records
            det.close()
        assert len(got[None]) > 100 and np.array_equal(got[None], got["0"])

    @pytest.mark.parametrize("thr", [0.0, -0.05])
    def test_thresholds_at_and_below_zero(self, monkeypatch, thr):
        """every block has a hit and the in-slice maxima of flat noise overflow the list: the strip walk
        inside the seed kernel must return what the plan without a list returns"""
        monkeypatch.setenv("DOGBLOB_CONV", "umma")
        frame = synth.sensor_noise(synth.droplet_scene(400, 300, 10, (4.0, 20.0), seed=3), seed=4).image
        kw = dict(min_sigma=2.0, max_sigma=20.0, n_bin=12, threshold=thr, preprocess=False, prune=False)
        got = {}
        for cap in (None, "0"):
            if cap is None:
                monkeypatch.delenv("DOGBLOB_SEED_CAP", raising=False)
            else:
                monkeypatch.setenv("DOGBLOB_SEED_CAP", cap)
            det = P.Detector(P.DetectionParams(**kw), slots=1, max_blobs=1 << 20)
            assert det.plan_for(frame.shape).plan.conv_engine == 2
            got[cap] = det.run(frame).blobs.records
            det.close()
        assert len(got[None]) > 1000 and np.array_equal(got[None], got["0"])
