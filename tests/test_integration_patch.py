"""INTEGRATION.md sections 2 and 3, exercised: the patch is applied to a temporary copy of the
reference package (read from /root/reference, which only exists in the build container: the
tests skip elsewhere) and the patched package is imported in a subprocess.

Without a GPU the run reaches libdogblob_b200.so's plan creation and fails there with the
library's own error; with one (the same container never has one) it returns the blob list."""
import json
import os
import subprocess
import sys
import textwrap
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_PKG = Path("/root/reference/pkg/src/dogblob")
LIB = ROOT / "paper_2010_08486_b200" / "libdogblob_b200.so"

pytestmark = pytest.mark.skipif(not REF_PKG.exists(), reason="the reference sources are not on this machine")


@pytest.fixture(scope="module")
def patched(tmp_path_factory):
    from paper_2010_08486_b200.integration import patch_reference
    dst = tmp_path_factory.mktemp("patched_ref") / "dogblob"
    patch_reference(REF_PKG, dst)
    return dst


def run_py(patched, code):
    env = dict(os.environ, PYTHONPATH=str(patched.parent), DOGBLOB_B200_LIB=str(LIB))
    return subprocess.run([sys.executable, "-c", textwrap.dedent(code)], env=env, capture_output=True, text=True,
                          timeout=300)


def test_patch_touches_exactly_the_cited_places(patched):
    import difflib
    changed = {}
    for f in sorted(REF_PKG.glob("*.py")):
        a, b = f.read_text().splitlines(), (patched / f.name).read_text().splitlines()
        n = sum(1 for l in difflib.unified_diff(a, b, lineterm="") if l.startswith(("+", "-")) and not l.startswith(("+++", "---")))
        if n:
            changed[f.name] = n
    assert set(changed) == {"convolve.py", "cli.py", "service.py", "detector.py"}
    assert changed["cli.py"] == 8 and changed["service.py"] == 2          # four lines / one line
    assert (patched / "_cuda.py").exists()


def test_allow_lists_accept_cuda_and_other_backends_are_untouched(patched):
    r = run_py(patched, """
        import json, numpy as np
        import dogblob
        from dogblob import convolve, cli, service
        from dogblob.detector import Detector, DetectionParams
        out = {"backends": list(convolve.BACKENDS)}
        args = cli.build_parser().parse_args(["detect", "--input", "x.raw", "--out-json", "o.json", "--min-sigma", "1",
                                              "--max-sigma", "4", "--n-bin", "3", "--backend", "cuda"])
        out["cli"] = args.backend
        caster, ok = service._PARAM_SPECS["backend"]
        out["service"] = bool(ok(caster("cuda")))
        # the CPU path of the patched package is the reference's own
        img = np.zeros((48, 48), np.float32); img[20:28, 20:28] = 1.0
        res = Detector(DetectionParams(min_sigma=2, max_sigma=6, n_bin=4, preprocess=False)).run(img)
        out["fft_blobs"] = len(res.blobs.blobs)
        print(json.dumps(out))
        """)
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["backends"] == ["direct", "fft", "cuda"] and out["service"] is True
    assert out["cli"] == "cuda" and out["fft_blobs"] >= 1


def test_cuda_backend_reaches_the_library(patched):
    """Detector.run(backend='cuda') of the patched reference goes through _cuda.py into
    dogblob_plan_create: blobs on a GPU box, the library's own device error here."""
    r = run_py(patched, """
        import json, numpy as np
        from dogblob.detector import Detector, DetectionParams
        img = np.zeros((64, 64), np.float32); img[24:40, 24:40] = 1.0
        det = Detector(DetectionParams(min_sigma=2, max_sigma=8, n_bin=6, preprocess=False, backend="cuda"))
        try:
            res = det.run(img)
            ref = Detector(DetectionParams(min_sigma=2, max_sigma=8, n_bin=6, preprocess=False)).run(img)
            same = [(b.x, b.y, b.sigma) for b in res.blobs.blobs] == [(b.x, b.y, b.sigma) for b in ref.blobs.blobs]
            print(json.dumps({"ran": True, "n": len(res.blobs.blobs), "same_as_fft": same}))
        except (RuntimeError, ValueError) as e:
            print(json.dumps({"ran": False, "error": str(e)}))
        """)
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    if out["ran"]:
        assert out["n"] >= 1 and out["same_as_fft"]
    else:       # no CUDA device in this container: the message is the library's (dogblob_last_error)
        assert "CUDA" in out["error"] or "cuda" in out["error"] or "device" in out["error"], out
    # direct convolve_bank calls are told to use the fused path
    r = run_py(patched, """
        import numpy as np
        from dogblob.convolve import convolve_bank
        from dogblob.scale_space import build_ladder, build_kernel_bank
        bank = build_kernel_bank(build_ladder(1, 3, 2), 5.0)
        try:
            convolve_bank(np.zeros((8, 8), np.float32), bank, backend="cuda")
        except ValueError as e:
            print("ValueError", e)
        """)
    assert r.returncode == 0 and "Detector.run" in r.stdout, r.stderr
