"""Timing experiments on the tensor-core convolution passes (DOGBLOB_UMMA_DEBUG masks) through the
DoG stage entry point (row pass + column/DoG pass + untranspose); results are garbage for most
masks, only the time matters.  Test tooling only.

    python tools/umma_probe.py C2 [mask ...]
"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2010_08486_b200 as P  # noqa: E402
from paper_2010_08486_b200 import _lib, detector as D, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
masks = [int(x) for x in sys.argv[2:]]
frame, kw = synth.config_frame(name), synth.config_params(name)
params = P.DetectionParams(preprocess=False, **kw)
ladder = P.build_ladder(params.min_sigma, params.max_sigma, params.n_bin)
bank = P.build_kernel_bank(ladder, params.truncate)
lib = _lib.load()
dev = torch.device("cuda", torch.cuda.current_device())
H, W = frame.shape
plan = D._Plan(bank, frame.shape, dev.index, 1024)
d_img = torch.zeros((H, plan.pitch), dtype=torch.float32, device=dev)
d_img[:, :W] = torch.from_numpy(frame).to(dev)
work = torch.zeros(plan.workspace_bytes, dtype=torch.uint8, device=dev)
out = torch.empty((ladder.n_levels - 1, H, W), dtype=torch.float32, device=dev)
st = torch.cuda.current_stream(dev)


def run(label):
    ts = []
    for i in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        _lib.check(lib.dogblob_dog(plan.handle, d_img.data_ptr(), work.data_ptr(), out.data_ptr(), st.cuda_stream))
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{label:24s} rows + cols + untranspose: {np.median(ts[2:]):.4f} ms", flush=True)


def stage_times(label):
    """row / column+DoG / extrema / prune from CUDA events of the detect entry point"""
    det = P.Detector(params, slots=1)
    eng = det.plan_for((H, W))
    slot = eng.slots[0]
    for _ in range(5):
        slot.launch_device(d_img, params, True)
    torch.cuda.synchronize()
    sets = [D.new_events() for _ in range(20)]
    for es in sets:
        slot.launch_device(d_img, params, True, events=es)
    torch.cuda.synchronize()
    med = np.median(np.array([D.event_intervals_ms(es) for es in sets]), axis=0)
    print(f"{label:24s} row {med[0]:.4f}  col+dog {med[1]:.4f}  extrema {med[2]:.4f}  prune {med[3]:.4f} ms",
          flush=True)
    det.close()


os.environ["DOGBLOB_CONV"] = "fma"
stage_times("fma")
os.environ["DOGBLOB_CONV"] = "umma"
stage_times("umma")
os.environ["DOGBLOB_CONV"] = "fma"
run("fma")
os.environ["DOGBLOB_CONV"] = "umma"
os.environ.pop("DOGBLOB_UMMA_DEBUG", None)
run("umma")
for m in masks:
    os.environ["DOGBLOB_UMMA_DEBUG"] = str(m)
    run(f"umma debug={m}")
if os.environ.get("UMMA_PROF_MASKS"):
    os.environ["DOGBLOB_UMMA_PROF"] = "1"
    for m in os.environ["UMMA_PROF_MASKS"].split(","):
        os.environ["DOGBLOB_UMMA_DEBUG"] = m
        print(f"--- per-role cycles, debug={m}", flush=True)
        sys.stdout.flush()
        _lib.check(lib.dogblob_dog(plan.handle, d_img.data_ptr(), work.data_ptr(), out.data_ptr(), st.cuda_stream))
        torch.cuda.synchronize()
