#!/usr/bin/env python
"""Headline benchmark: frames/s and single-frame latency of the 1024^2 DoG detector.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

Workload (BASELINE.json configs[1] as the batch of configs[2], SURVEY 8d "C2" / "C3"):
1024x1024 PLIF-like synthetic frames, sigma in [1, 30], n_bin = 58 (59 levels, radii
5..150), threshold 0.1, overlap 0.5, pruning on, preprocess off.  A step is one pass of
the hot path over the C3 batch: BATCH = 256 distinct frames per GPU (scene seed 1000+f,
noise seed 2000+f; frame f of the global batch runs on rank f mod N).

  value  : frames/s, kernels only, frames resident in HBM (CUDA events, max over ranks)
  e2e    : frames/s through Detector.run_batch with pinned HOST frames: H2D copy of
           every frame and D2H + decoding of every blob list inside the timed region
  latency: Detector.run on one pinned host frame, median wall-clock ms
  roofline: the fused column+DoG kernel (dominant), CUDA-event duration per launch
  cpu_baseline: the oracle port of the reference CPU path timed on this host

Multi-GPU: frames shard by index, frame f -> rank f mod N, no collective on the data
path (weak scaling: BATCH frames per GPU per step).  Under torchrun the ranks come from
the environment; `python bench.py --gpus N` without one spawns the N ranks itself (one per
device, wrapping around on a box with fewer devices) and relays rank 0's line.
`--impl reference` times the reference CPU algorithm (oracle port) on all host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOAD = "C2"
BATCH = int(os.environ.get("DOGBLOB_BENCH_BATCH", "256"))   # frames per GPU per step (the C3 batch)
KERNELS_PER_FRAME = 8    # FP32 engine: reset, row pass, column+DoG, edge DoG, nms, plateau, finalize_small, prune_large
KERNELS_PER_FRAME_TENSOR = 8   # tensor engine: frame max (+ counter reset), operand split, row pass, column+DoG, nms, plateau, finalize_small, prune_large
METRIC = "frames/sec, 1024x1024 DoG detector (sigma<=30, n_bin=58)"


def bench_config(world):
    """The `config` object of both arms (identical keys and values for the same N)."""
    return {"workload": f"{WORKLOAD}: 1024x1024 PLIF-like frames, sigma 1..30, n_bin 58, threshold 0.1, "
                        f"overlap 0.5, prune on, preprocess off; batch C3 (scene seed 1000+f, noise seed 2000+f)",
            "frames_per_step": BATCH * world, "frames_per_gpu": BATCH,
            "sharding": "frame f -> rank f mod N, no collective",
            "l2": f"per-frame working set 490 MB (59 + 58 planes of 4 MB) exceeds the 126 MB L2; "
                  f"{BATCH} distinct frames per GPU rotate"}


def params_kw():
    from paper_2010_08486_b200 import synth
    return synth.config_params(WORKLOAD)


def _make_frame(f):
    from paper_2010_08486_b200 import synth
    return synth.config_frame("C3", int(f))


def make_frames(indices):
    """Frames of the C3 batch; generated in parallel worker processes (0.2 s each on one core).
    Must run before CUDA is initialised in this process (fork)."""
    indices = [int(f) for f in indices]
    if len(indices) < 8:
        return [_make_frame(f) for f in indices]
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    procs = max(1, min(32, cores // max(1, min(world, 8))))
    if procs == 1:
        return [_make_frame(f) for f in indices]
    with mp.get_context("fork").Pool(procs) as pool:
        return pool.map(_make_frame, indices, chunksize=4)


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.idx)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); mx.append(float(f[2])); power.append(float(f[3]))
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "power_w_max": float(max(power)), "samples": len(sm), "reasons": sorted(reasons)}


# --------------------------------------------------------------------------------
def oracle_fps_single_core():
    """cpu_baseline of the `ours` line: the oracle port of the reference CPU path
    (fft backend, float32, as-is = 1 core) on one frame of the workload."""
    from oracle import dog_oracle as O
    frame = make_frames([0])[0]
    det = O.OracleDetector(preprocess=False, **params_kw())
    det.spectra_for(frame.shape, np.float32)     # amortised state, like bench.py:57-62 of the reference
    t0 = time.perf_counter()
    res = det.run(frame)
    dt = time.perf_counter() - t0
    return {"value": 1.0 / dt, "unit": "frames/s", "cores": 1, "kind": "port",
            "sample": f"1 frame of {WORKLOAD} (1024x1024, 59 levels) after building kernel spectra; "
                      f"{dt * 1e3:.0f} ms, {len(res.blobs)} blobs",
            "stage_ms": {k: round(v, 1) for k, v in res.timings_ms.items()}}


_WORKER = {}


def _ref_worker_init():
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import dog_oracle as O
    det = O.OracleDetector(preprocess=False, **params_kw())
    det.spectra_for((1024, 1024), np.float32)
    _WORKER["det"] = det


def _ref_worker_run(frame_index):
    frame = make_frames([frame_index])[0]
    t0 = time.perf_counter()
    res = _WORKER["det"].run(frame)
    return time.perf_counter() - t0, len(res.blobs)


def run_reference(args):
    """The reference CPU implementation of the path (oracle port: /root/reference is pure
    Python and does not exist on the GPU box), frame-parallel over all host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    procs = max(1, min(cores, 32))
    ctx = mp.get_context("fork")
    with ctx.Pool(procs, initializer=_ref_worker_init) as pool:
        per_step = procs                                     # one frame per worker per step
        for w in range(args.warmup):
            pool.map(_ref_worker_run, range(per_step))
        t0 = time.perf_counter()
        for k in range(args.steps):
            pool.map(_ref_worker_run, [k * per_step + i for i in range(per_step)])
        dt = time.perf_counter() - t0
    fps = per_step * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC,
        "value": fps, "unit": "frames/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(args.gpus),
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": procs, "kind": "port",
                         "sample": f"bounded sample of the batch: {per_step} frames per step (frames "
                                   f"{0}..{per_step * args.steps - 1} of C3), one per worker process "
                                   f"({procs} processes, fft backend, float32)"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2010_08486_b200 as P
    from paper_2010_08486_b200 import detector as D

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # frame f of the global batch goes to rank f mod world; generated in forked workers, so
    # before this process touches CUDA
    my_frames = [f for f in range(BATCH * world) if f % world == rank]
    frames = make_frames(my_frames)
    if not torch.cuda.is_available():
        raise RuntimeError("bench.py --impl ours needs a CUDA device (no CPU fallback)")
    n_dev = torch.cuda.device_count()
    local = local % n_dev                           # (a 1-GPU box can still exercise N > 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ctl = None
    if world > 1:
        # control plane only (barrier + max of one scalar): the data path has no collective.  With one
        # device per rank the NCCL backend is registered as the contract asks (never used on the hot
        # path); ranks that share a device (N > devices) cannot form an NCCL communicator: gloo only.
        dist.init_process_group("cpu:gloo,cuda:nccl" if n_dev >= world else "gloo")
        ctl = dist.new_group(backend="gloo")

    kw = params_kw()
    params = P.DetectionParams(preprocess=False, **kw)
    n_slots = int(os.environ.get("DOGBLOB_BENCH_SLOTS", "8"))   # frame slots = concurrent streams
    det = P.Detector(params, device=local, slots=n_slots)
    H, W = frames[0].shape
    eng = det.plan_for((H, W))
    pitch = eng.plan.pitch
    pinned = [torch.from_numpy(f).pin_memory() for f in frames]
    resident = []
    for f in frames:
        d = torch.zeros((H, pitch), dtype=torch.float32, device=dev)
        d[:, :W] = torch.from_numpy(f).to(dev)
        resident.append(d)
    slots = eng.slots
    main = torch.cuda.current_stream(dev)
    event_sets = [D.new_events() for _ in range(len(frames))]

    def device_step(record_sets=None):
        for i, d in enumerate(resident):
            s = slots[i % len(slots)]
            s.launch_device(d, params, True, events=None if record_sets is None else record_sets[i])

    def fenced(fn, reps):
        """reps x fn() on the slot streams, bracketed by events on the main stream."""
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier(group=ctl)
            torch.cuda.synchronize(dev)
        start.record(main)
        for s in slots:
            s.stream.wait_event(start)
        for r in range(reps):
            fn(r)
        for s in slots:
            done = torch.cuda.Event()
            done.record(s.stream)
            main.wait_event(done)
        end.record(main)
        torch.cuda.synchronize(dev)
        ms = start.elapsed_time(end)
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=ctl)
            ms = float(t.item())
        return ms

    # ---- kernels only, frames resident in HBM ----
    for _ in range(max(args.warmup, 3)):
        device_step()
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
        time.sleep(0.25)
    ms_total = fenced(lambda r: device_step(event_sets if r == args.steps - 1 else None), args.steps)
    clocks = sampler.stop() if rank == 0 else None
    frames_per_step = BATCH * world
    value = frames_per_step * args.steps / (ms_total * 1e-3)
    stage = np.array([D.event_intervals_ms(es) for es in event_sets])   # [frame][row, col, extrema, prune]

    # ---- isolated kernel durations: one stream, frames back to back ----
    iso_sets = [D.new_events() for _ in range(len(frames))]
    for i, d in enumerate(resident):
        slots[0].launch_device(d, params, True, events=iso_sets[i])
    torch.cuda.synchronize(dev)
    iso = np.array([D.event_intervals_ms(es) for es in iso_sets])

    # ---- end to end through the public API, pinned host frames ----
    for _ in range(3):
        det.run_batch(pinned)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier(group=ctl)
    t0 = time.perf_counter()
    n_blobs = 0
    for _ in range(args.steps):
        out = det.run_batch(pinned)
        n_blobs = sum(len(r.blobs) for r in out)
    torch.cuda.synchronize(dev)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s, float(n_blobs)], dtype=torch.float64)
        dist.all_reduce(t[:1], op=dist.ReduceOp.MAX, group=ctl)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM, group=ctl)
        e2e_s, n_blobs = float(t[0].item()), int(t[1].item())
    e2e_value = frames_per_step * args.steps / e2e_s
    h2d = frames_per_step * H * W * 4
    d2h = frames_per_step * (64 + slots[0].n_host * 48)

    # ---- single-frame latency (batch 1), pinned host frame in, decoded blobs out ----
    lat = []
    for i in range(10 + 100):
        t0 = time.perf_counter()
        res = det.run(pinned[i % len(pinned)])
        dt = (time.perf_counter() - t0) * 1e3
        if i >= 10:
            lat.append(dt)
    lat = np.array(lat)

    if rank == 0:
        L = len(det.ladder.sigmas)
        S = L - 1
        taps = int(sum(2 * int(r) + 1 for r in det.bank.radii))
        col_bytes = 4.0 * H * W * (L + S)                  # read L row-filtered planes, write S slices
        col_flops = 2.0 * H * W * taps + 2.0 * H * W * S
        frame_bytes = 4.0 * H * W * (4 * (L - 1) + 3)      # SURVEY 8d algorithmic bytes per frame
        frame_flops = 2.0 * H * W * 2 * taps + 2.0 * H * W * S
        peak, peak_src = measured_peaks()
        col_ms = float(stage[:, 1].mean())
        col_ms_iso = float(iso[:, 1].mean())
        achieved = col_bytes / (col_ms_iso * 1e-3) / 1e9
        traffic = None
        tp = ROOT / "profiles" / "ncu_traffic.json"
        if tp.exists():
            try:
                traffic = json.loads(tp.read_text()).get(
                    "umma_col_dog_kernel_dram_bytes_per_launch" if eng.plan.conv_engine >= 1
                    else "col_dog_kernel_dram_bytes_per_launch")
            except Exception:
                traffic = None
        tensor_engine = eng.plan.conv_engine >= 1
        fp16_engine = eng.plan.conv_engine == 2
        if tensor_engine:
            # tcgen05 Toeplitz GEMM: per 128 x 128 tile a level spends (128 + 2 rpad) / 16 k-steps of two
            # kind::f16 MMAs (M = 128, K = 16): [main | small] += T_hi * [X_hi | X_lo] with N = 256 and
            # small += T_lo * X_hi with N = 128.  The tensor pipe spends 64 cycles per 128 columns of N
            # (tools/ubench_umma_ss.cu).  The column pass computes the first level of every group but the
            # first twice.
            rpads = [max(8, (int(r) + 7) // 8 * 8) for r in det.bank.radii]
            tiles = ((H + 127) // 128) * ((W + 127) // 128)
            groups = eng.plan.conv_groups
            levels = []
            for g in range(len(groups) - 1):
                levels += list(range(groups[g], min(groups[g + 1] + (1 if g + 2 < len(groups) else 0), L)))
            n_mma, mma_flops = 0, 0.0
            for lv in levels:
                rp2 = 2 * rpads[lv]
                n_k = (128 + rp2) // 16
                n_mma += 2 * n_k
                mma_flops += n_k * 2.0 * 128 * (256 + 128) * 16
            n_mma *= tiles
            mma_flops *= tiles
            try:
                f16_peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["bf16_tflops"]
            except Exception:
                f16_peak = 2250.0
            sm_hz = 1e6 * ((clocks or {}).get("sm_mhz") or 1965.0)
            engine_roof = {
                "note": "tcgen05 kind::f16 Toeplitz GEMM, float32 accuracy from a hi/lo split of both operands "
                        "(2 MMAs per k-step: N = 256 and N = 128); see DESIGN.md 3a for what bounds it",
                "useful_flops_per_launch": col_flops,
                "useful_tflops": col_flops / (col_ms_iso * 1e-3) / 1e12,
                "mma_instructions_per_launch": n_mma,
                "issued_mma_flops_per_launch": mma_flops,
                "issued_mma_tflops": mma_flops / (col_ms_iso * 1e-3) / 1e12,
                "mma_peak_tflops": f16_peak,
                "mma_peak_source": "MEASURED_PEAKS.json bf16_tflops (kind::f16 rate)",
                "frac_of_mma_peak": mma_flops / (col_ms_iso * 1e-3) / 1e12 / f16_peak,
                "tensor_pipe_busy_estimate": n_mma * 96.0 / 148.0 / (col_ms_iso * 1e-3 * sm_hz),
                "level_groups": groups,
            }
            kernel_name = ("umma_pass_kernel<kModeDog> (tcgen05 Toeplitz-GEMM column pass + fused DoG + in-slice part of "
                           "the extrema search: seed list)")
        else:
            engine_roof = {"note": "this kernel is FP32-FMA bound, not HBM bound (SURVEY 7, 8d): "
                                   "arithmetic intensity 38 FLOP/B",
                           "flops_per_launch": col_flops,
                           "achieved_tflops": col_flops / (col_ms_iso * 1e-3) / 1e12,
                           "peak_tflops": 71.9,
                           "peak_source": "tools/ubench_fma.cu on this pool's B200 (FFMA, 1965 MHz)",
                           "frac": col_flops / (col_ms_iso * 1e-3) / 1e12 / 71.9}
            kernel_name = "col_pass_kernel<true> (fused column pass + DoG)"
        roofline = {"bound": "hbm", "kernel": kernel_name,
                    "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": traffic, "peak_source": peak_src,
                    "bytes_per_launch": col_bytes, "ms_per_launch_isolated": col_ms_iso,
                    "ms_per_launch_in_timed_region": col_ms,
                    "tensor" if tensor_engine else "fp32": engine_roof,
                    # the kernel also does the in-slice half of the extrema search (DESIGN 3a, seeds), which is what lets
                    # the extrema stage skip its 4HWS-byte read of the slices: the pair against the pair's bytes
                    "column_pass_plus_extrema": {
                        "bytes": col_bytes + 4.0 * H * W * S,
                        "ms_isolated": col_ms_iso + float(iso[:, 2].mean()),
                        "frac": (col_bytes + 4.0 * H * W * S) / ((col_ms_iso + float(iso[:, 2].mean())) * 1e-3) / 1e9 / peak},
                    "whole_frame": {"bytes": frame_bytes, "flops": frame_flops,
                                    "hbm_frac_at_value": frame_bytes * value / world / 1e9 / peak}}
        line = {
            "metric": METRIC,
            "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": bench_config(world),
            "streams_per_gpu": len(slots), "devices": n_dev,
            "latency_ms": {"single_frame_e2e_median": float(np.median(lat)),
                           "p10": float(np.percentile(lat, 10)), "p90": float(np.percentile(lat, 90)),
                           "what": "Detector.run(pinned host frame): H2D + kernels + D2H + decode, batch 1",
                           "device_stage_ms_isolated": {"row_pass": float(iso[:, 0].mean()),
                                                        "col_dog_pass": col_ms_iso,
                                                        "extrema": float(iso[:, 2].mean()),
                                                        "prune_pack": float(iso[:, 3].mean())}},
            "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "blobs_per_step": n_blobs,
                    "what": "Detector.run_batch over pinned host frames, wall clock"},
            "gpu_launches": (KERNELS_PER_FRAME_TENSOR if tensor_engine else KERNELS_PER_FRAME) * BATCH * world * args.steps,
            "roofline": roofline,
            "clocks": clocks,
        }
        if world == 1:
            line["cpu_baseline"] = oracle_fps_single_core()
        print(json.dumps(line), flush=True)
    det.close()
    if world > 1:
        dist.barrier(group=ctl)
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    args = ap.parse_args()
    if args.impl == "reference":
        args.steps = 3 if args.steps is None else args.steps
        args.warmup = 1 if args.warmup is None else args.warmup
        run_reference(args)
    else:
        args.steps = 30 if args.steps is None else args.steps
        args.warmup = 3 if args.warmup is None else args.warmup
        if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
            sys.exit(spawn_ranks(args))
        run_ours(args)


def spawn_ranks(args):
    """`python bench.py --gpus N` outside torchrun: launch the N ranks the way the driver does
    (one process per GPU, rendezvous on 127.0.0.1) and pass their output through."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()),
           "--gpus", str(args.gpus), "--steps", str(args.steps), "--warmup", str(args.warmup), "--impl", args.impl]
    return subprocess.call(cmd)


if __name__ == "__main__":
    main()
