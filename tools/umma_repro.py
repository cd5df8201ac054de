"""Run-to-run reproducibility of the fused DoG slices of one frame (tensor-core engine forced):
prints the largest difference against the first run.  python tools/umma_repro.py [C2|C4]"""
import os, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2010_08486_b200 as P
from paper_2010_08486_b200 import synth
os.environ["DOGBLOB_CONV"] = "umma"
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
img = synth.config_frame(name); kw = synth.config_params(name)
ladder = P.build_ladder(kw["min_sigma"], kw["max_sigma"], kw["n_bin"]); bank = P.build_kernel_bank(ladder, 5.0)
ref = None
for it in range(6):
    dog = P.fused_dog(img, bank).slices
    if ref is None:
        ref = dog
        continue
    d = np.abs(dog - ref)
    bad = np.argwhere(d > 1e-6)
    print(it, "max diff vs run 0:", d.max(), "n bad", len(bad), "first", bad[:3].tolist(), "slices", sorted(set(bad[:, 0].tolist()))[:10], flush=True)
