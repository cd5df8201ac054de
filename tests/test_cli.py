"""CLI of the CUDA backend: flags, exit codes (0 / 1 usage / 2 runtime) and the
backend-independent subcommands, without a GPU; `detect` and `bench` run in test_gpu_pipeline.py."""

import numpy as np

from paper_2010_08486_b200 import cli, formats, synth


def test_usage_errors_exit_1(capsys):
    assert cli.main([]) == 1
    assert cli.main(["detect", "--input", "x.raw"]) == 1                 # ladder + --out-json required
    assert cli.main(["detect", "--input", "x.raw", "--min-sigma", "1", "--max-sigma", "5", "--n-bin", "4",
                     "--out-json", "o.json", "--backend", "fft"]) == 1   # only cuda lives here
    assert cli.main(["bench", "--sweep", "n_bin", "--values", "", "--seed", "1", "--out", "o.csv"]) == 1
    assert cli.main(["bench", "--sweep", "n_bin", "--values", "a,b", "--seed", "1", "--out", "o.csv"]) == 1
    assert cli.main(["serve", "--listen", "nonsense"]) == 1
    assert "error:" in capsys.readouterr().err


def test_runtime_errors_exit_2(tmp_path, capsys):
    common = ["--min-sigma", "1", "--max-sigma", "5", "--n-bin", "4", "--out-json", str(tmp_path / "o.json")]
    assert cli.main(["detect", "--input", str(tmp_path / "missing.raw")] + common) == 2
    (tmp_path / "short.raw").write_bytes(b"\x01\x02\x03")
    assert cli.main(["detect", "--input", str(tmp_path / "short.raw")] + common) == 2
    assert cli.main(["evaluate"]) == 1 and cli.main(["parity"]) == 1          # usage errors, like the reference
    assert cli.main(["evaluate", "--pred", str(tmp_path / "nope.json"), "--truth", str(tmp_path / "nope.csv"),
                     "--out", str(tmp_path / "r.json")]) == 2
    assert cli.main(["simulate", "--r-min", "3", "--r-max", "9", "--seed", "1", "--out-image",
                     str(tmp_path / "s.png"), "--out-truth", str(tmp_path / "s.csv")]) == 2
    err = capsys.readouterr().err
    assert "no such image" in err and "truncated raw header" in err and "nope.json" in err


def test_simulate_writes_the_reference_scene(tmp_path, capsys):
    img, truth = tmp_path / "scene.raw", tmp_path / "scene.csv"
    assert cli.main(["simulate", "--width", "200", "--height", "160", "--n-spheres", "9", "--r-min", "4",
                     "--r-max", "12", "--seed", "7", "--gaussian-sigma", "0.02", "--allow-overlap",
                     "--out-image", str(img), "--out-truth", str(truth)]) == 0
    assert "scene with 9 spheres" in capsys.readouterr().out
    want = synth.sensor_noise(synth.droplet_scene(200, 160, 9, (4.0, 12.0), seed=7, allow_overlap=True),
                              read_sigma=0.02, seed=7)
    assert np.array_equal(formats.read_raw(img), want.image)
    lines = truth.read_text().splitlines()
    assert lines[:2] == ["# seed=7", "x,y,r"] and len(lines) == 11
    assert lines[2] == f"{want.truths[0].x!r},{want.truths[0].y!r},{want.truths[0].r!r}"


def test_parameter_mapping():
    args = cli.build_parser().parse_args(["serve", "--n-bin", "7", "--no-preprocess", "--overlap", "0.3"])
    p = cli._params(args)
    assert (p.n_bin, p.preprocess, p.overlap, p.min_sigma, p.backend) == (7, False, 0.3, 1.0, "cuda")
