#!/usr/bin/env python
"""Row / column pass throughput versus sweep length: ladders whose levels all have (nearly) the
same radius, so that every sweep has the same number of 16-row chunks."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import paper_2010_08486_b200 as P  # noqa: E402
from paper_2010_08486_b200 import detector as D, synth  # noqa: E402

frame = synth.config_frame("C2")
H, W = frame.shape
for lo, hi, n_bin in ((1.0, 1.5, 40), (3.0, 3.5, 40), (6.0, 6.5, 40), (12.0, 12.5, 40), (20.0, 20.5, 40), (29.5, 30.0, 40),
                      (44.0, 44.5, 40), (1.0, 30.0, 58)):
    params = P.DetectionParams(preprocess=False, min_sigma=lo, max_sigma=hi, n_bin=n_bin)
    det = P.Detector(params, slots=1)
    eng = det.plan_for((H, W))
    d = torch.zeros((H, eng.plan.pitch), dtype=torch.float32, device="cuda")
    d[:, :W] = torch.from_numpy(frame).cuda()
    slot = eng.slots[0]
    for _ in range(3):
        slot.launch_device(d, params, True)
    torch.cuda.synchronize()
    sets = [D.new_events() for _ in range(10)]
    for es in sets:
        slot.launch_device(d, params, True, events=es)
    torch.cuda.synchronize()
    iv = np.median(np.array([D.event_intervals_ms(es) for es in sets]), axis=0)
    rpad = np.maximum(8, (det.bank.radii + 7) // 8 * 8)
    chunks = (2 * rpad + 16) // 16
    fma_groups = (chunks - 2) * 256 + 272          # per 16 outputs x 1 column
    issued = 2.0 * H * W * float(fma_groups.sum()) / 16.0
    useful = 2.0 * H * W * float((2 * det.bank.radii + 1).sum())
    print(json.dumps({"sigma": [lo, hi], "levels": len(rpad), "chunks_per_sweep": float(chunks.mean()),
                      "row_ms": float(iv[0]), "col_ms": float(iv[1]),
                      "row_issued_tflops": issued / iv[0] / 1e9, "col_issued_tflops": issued / iv[1] / 1e9,
                      "useful_over_issued": useful / issued}), flush=True)
    det.close()
