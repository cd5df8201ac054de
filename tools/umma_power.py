#!/usr/bin/env python
"""Board power and SM clock while the scale-space passes of one frame run back to back (DOGBLOB_UMMA_DEBUG masks:
results are garbage under a mask, only power / clocks / time matter).  Test tooling only.

    python tools/umma_power.py C2 0 8 1 32
"""
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

os.environ.setdefault("DOGBLOB_UMMA_DEBUG", "0")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import pynvml  # noqa: E402
import torch  # noqa: E402

import paper_2010_08486_b200 as P  # noqa: E402
from paper_2010_08486_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
masks = [int(x) for x in sys.argv[2:]] or [0]
frame, kw = synth.config_frame(name), synth.config_params(name)
params = P.DetectionParams(preprocess=False, **kw)
import dataclasses  # noqa: E402
run_params = dataclasses.replace(params, threshold=float(os.environ.get("UMMA_MASKS_THR", "inf")))
H, W = frame.shape
det = P.Detector(params, slots=1)
eng = det.plan_for((H, W))
slot = eng.slots[0]
dev = torch.device("cuda", torch.cuda.current_device())
d_img = torch.zeros((H, eng.plan.pitch), dtype=torch.float32, device=dev)
d_img[:, :W] = torch.from_numpy(frame).to(dev)
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
for m in masks:
    os.environ["DOGBLOB_UMMA_DEBUG"] = str(m)
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetPowerUsage(h) / 1e3, pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
            time.sleep(0.05)
    n = int(os.environ.get("UMMA_POWER_FRAMES", "20000"))
    for _ in range(200):
        slot.launch_device(d_img, run_params, True)
    torch.cuda.synchronize()
    th = threading.Thread(target=sample)
    th.start()
    t0 = time.perf_counter()
    for _ in range(n):
        slot.launch_device(d_img, run_params, True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    stop.set()
    th.join()
    s = np.array(samples[len(samples) // 3:])
    print(f"{name} mask {m:4d}: {dt / n * 1e3:.4f} ms/frame, power median {np.median(s[:, 0]):.0f} W, SM clock median {np.median(s[:, 1]):.0f} MHz, "
          f"{dt / n * np.median(s[:, 0]):.4f} mJ... J/frame = {dt / n * np.median(s[:, 0]):.4f}", flush=True)
os.environ["DOGBLOB_UMMA_DEBUG"] = "0"
det.close()
