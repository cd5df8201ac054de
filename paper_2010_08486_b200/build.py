"""Builds libdogblob_b200.so in-tree with nvcc for sm_100a (no torch involved).

    python -m paper_2010_08486_b200.build [--force]

The shared library is a plain C-ABI CUDA library (include/dogblob_b200.h); it
links cudart statically so that the only run-time dependency is the driver.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libdogblob_b200.so"
STAMP = PKG / "csrc" / ".build_stamp"
SOURCES = ["api.cu", "scale_space.cu", "scale_space_umma.cu", "extrema.cu", "prune.cu", "preprocess.cu", "fp64.cu", "evaluate.cu", "synth_device.cu"]
HEADERS = [CSRC / "common.cuh", PKG.parent / "include" / "dogblob_b200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-std=c++17", "-lineinfo",
    "-fmad=false",              # every FMA in this library is written explicitly
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "--cudart", "static",
]


# experiment knobs of the tensor-core passes (compile-time): DOGBLOB_UMMA_ISSUERS, DOGBLOB_UMMA_STAGEK
for _k in ("DOGBLOB_UMMA_ISSUERS", "DOGBLOB_UMMA_STAGEK", "DOGBLOB_UMMA_DRAIN_GROUPS", "DOGBLOB_UMMA_F16", "DOGBLOB_UMMA_ROWS1", "DOGBLOB_UMMA_TOEP1", "DOGBLOB_UMMA_TOEP2", "DOGBLOB_UMMA_STAGING1", "DOGBLOB_UMMA_BACKOFF"):
    if os.environ.get(_k):
        NVCC_FLAGS.append(f"-D{_k}={os.environ[_k]}")


def _nvcc() -> str:
    cand = os.environ.get("NVCC") or shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; cannot build libdogblob_b200.so")
    return cand


def _fingerprint(sources) -> str:
    h = hashlib.sha256()
    for p in list(sources) + HEADERS:
        h.update(Path(p).read_bytes())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def build_library(force: bool = False, verbose: bool = False) -> Path:
    sources = [CSRC / s for s in SOURCES if (CSRC / s).exists()]
    fp = _fingerprint(sources)
    if not force and LIB.exists() and STAMP.exists() and STAMP.read_text().strip() == fp:
        return LIB
    nvcc = _nvcc()
    objs = []
    procs = []
    for src in sources:
        obj = CSRC / (src.stem + ".o")
        cmd = [nvcc, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    for src, p in procs:
        out, _ = p.communicate()
        if verbose and out:
            print(out)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{out}")
    link = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "--cudart", "static",
            "-Xcompiler", "-fPIC", *map(str, objs), "-o", str(LIB)]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}")
    STAMP.write_text(fp + "\n")
    return LIB


if __name__ == "__main__":
    path = build_library(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(path)
