"""Applies the reference-side patch of INTEGRATION.md section 3 to a COPY of the reference's
`dogblob` package: three allow-lists, one branch in `Detector.run`, the plan cache next to
`plan_for`, and the ctypes stub `_cuda.py`.  Every edit is an exact-text replacement that fails
loudly if the reference source differs from the lines INTEGRATION.md cites.

    python -m paper_2010_08486_b200.integration.patch /path/to/pkg/src/dogblob /tmp/patched/dogblob
"""
from __future__ import annotations

import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent

RUN_BRANCH = '''
        if p.backend == "cuda":
            # fused scale space + DoG + extrema + pruning on the GPU (libdogblob_b200.so)
            t0 = time.perf_counter()
            plan, lock = self.cuda_plan_for(img.shape)
            with lock:                                   # one frame in flight per buffer set
                recs = plan.detect(img, np.float32(p.threshold), p.neighborhood, p.overlap, p.prune)
            timings.update(convolve_ms=(time.perf_counter() - t0) * 1e3, extrema_ms=0.0, prune_ms=0.0)
            blobs = BlobSet(
                blobs=tuple(
                    Blob(x=int(r["x"]) if r["x"] == int(r["x"]) else float(r["x"]),
                         y=int(r["y"]) if r["y"] == int(r["y"]) else float(r["y"]),
                         sigma=float(r["sigma"]), radius=float(r["radius"]), response=float(r["response"]),
                         at_scale_boundary=bool(r["flags"] & 1))
                    for r in recs),
                source_shape=(img.shape[1], img.shape[0]),
                params=p,
            )
            return DetectResult(blobs=blobs, histogram=histogram(blobs, self.ladder), timings_ms=timings)
'''

PLAN_CACHE = '''
    def cuda_plan_for(self, shape: tuple[int, int]):
        """(CudaPlan, lock) for an image shape: the same double-checked cache as plan_for()."""
        entry = self._cuda_plans.get(shape)
        if entry is None:
            with self._plan_lock:
                entry = self._cuda_plans.get(shape)
                if entry is None:
                    from ._cuda import CudaPlan
                    entry = (CudaPlan(self.ladder, self.bank, shape), threading.Lock())
                    self._cuda_plans[shape] = entry
        return entry
'''

EDITS = {
    "convolve.py": [
        ('BACKENDS = ("direct", "fft")', 'BACKENDS = ("direct", "fft", "cuda")'),
        ('    dtype = np.dtype(dtype)\n    if backend == "direct":',
         '    dtype = np.dtype(dtype)\n    if backend == "cuda":\n'
         '        raise ValueError("backend \'cuda\' runs the fused pipeline: call Detector.run")\n'
         '    if backend == "direct":'),
    ],
    # cli.py:46 (detect / serve), :100-101 (parity --backend-a / -b), :109 (bench)
    "cli.py": [('choices=("direct", "fft")', 'choices=("direct", "fft", "cuda")', 4)],
    "service.py": [('lambda v: v in ("direct", "fft")', 'lambda v: v in ("direct", "fft", "cuda")')],
    "detector.py": [
        ("        self._plans: dict[tuple[int, int], FftPlan] = {}\n",
         "        self._plans: dict[tuple[int, int], FftPlan] = {}\n        self._cuda_plans: dict = {}\n"),
        ("    def run(self, img: np.ndarray, dtype=np.float32) -> DetectResult:",
         PLAN_CACHE.lstrip("\n") + "\n    def run(self, img: np.ndarray, dtype=np.float32) -> DetectResult:"),
        ('        timings["preprocess_ms"] = (time.perf_counter() - t0) * 1e3\n',
         '        timings["preprocess_ms"] = (time.perf_counter() - t0) * 1e3\n' + RUN_BRANCH),
    ],
}


def patch_reference(src_pkg: str | Path, dst_pkg: str | Path) -> Path:
    """Copy the reference package directory `src_pkg` (…/src/dogblob) to `dst_pkg` and patch the copy."""
    src_pkg, dst_pkg = Path(src_pkg), Path(dst_pkg)
    if dst_pkg.exists():
        shutil.rmtree(dst_pkg)
    shutil.copytree(src_pkg, dst_pkg, ignore=shutil.ignore_patterns("__pycache__"))
    for name, edits in EDITS.items():
        path = dst_pkg / name
        text = path.read_text()
        for old, new, *count in edits:
            want = count[0] if count else 1
            if text.count(old) != want:
                raise RuntimeError(f"{name}: expected {want} occurrence(s) of {old!r} (reference changed?)")
            text = text.replace(old, new)
        path.write_text(text)
    shutil.copy(HERE / "_cuda.py", dst_pkg / "_cuda.py")
    return dst_pkg


if __name__ == "__main__":
    if len(sys.argv) != 3:
        sys.exit(__doc__)
    print(patch_reference(sys.argv[1], sys.argv[2]))
