"""Command line of the CUDA backend: detect, simulate, evaluate, parity, bench, serve.

Flags, outputs and exit codes follow the reference CLI (`cli.py:38-136,288-301`): 0 on
success, 1 on usage errors, 2 on runtime failures; `--backend` accepts `cuda` only.  `parity`
compares the float32 production kernels with the float64 tier (`--dtype-a / --dtype-b`) where the
reference compares its two CPU backends.

    python -m paper_2010_08486_b200 detect --input f.raw --min-sigma 1 --max-sigma 30 --n-bin 58 \
        --out-json blobs.json [--out-hist hist.csv]
    python -m paper_2010_08486_b200 serve --listen 127.0.0.1:8750 --workers 2
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import sys
from pathlib import Path

import numpy as np

from . import formats, synth
from .detector import BACKENDS, DetectionParams, Detector

USAGE_ERROR, RUNTIME_ERROR = 1, 2
RAW_SUFFIXES = (".raw", ".bin")


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        self.print_usage(sys.stderr)
        print(f"error: {message}", file=sys.stderr)
        raise SystemExit(USAGE_ERROR)


# (flag, DetectionParams field, type): the detector options every subcommand shares
_LADDER_FLAGS = (("--min-sigma", "min_sigma", float), ("--max-sigma", "max_sigma", float),
                 ("--n-bin", "n_bin", int))
_TUNING_FLAGS = (("--truncate", "truncate", float), ("--threshold", "threshold", float),
                 ("--overlap", "overlap", float), ("--neighborhood", "neighborhood", int),
                 ("--smooth-sigma", "smooth_sigma", float), ("--saturation", "saturation", float))


def _add_detector_flags(p: argparse.ArgumentParser, ladder_required: bool) -> None:
    defaults = DetectionParams()
    for flag, _, kind in _LADDER_FLAGS:
        p.add_argument(flag, type=kind, required=ladder_required, default=None)
    for flag, name, kind in _TUNING_FLAGS:
        p.add_argument(flag, type=kind, default=getattr(defaults, name))
    p.add_argument("--backend", choices=BACKENDS, default=BACKENDS[0])
    p.add_argument("--no-preprocess", action="store_true")
    p.add_argument("--device", type=int, default=None, help="CUDA device index")


def _params(args) -> DetectionParams:
    values = DetectionParams().to_dict()
    for _, name, _ in _LADDER_FLAGS + _TUNING_FLAGS:
        given = getattr(args, name)
        if given is not None:
            values[name] = given
    values.update(backend=args.backend, preprocess=not args.no_preprocess)
    return DetectionParams(**values)


def build_parser() -> _Parser:
    parser = _Parser(prog="dogblob-b200", description=__doc__,
                     formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = parser.add_subparsers(dest="command", required=True)

    p = sub.add_parser("detect", help="detect blobs in one image")
    p.add_argument("--input", required=True)
    _add_detector_flags(p, ladder_required=True)
    p.add_argument("--out-json", required=True)
    p.add_argument("--out-hist", default=None)

    p = sub.add_parser("simulate", help="render a synthetic droplet scene (raw float output)")
    p.add_argument("--width", type=int, default=1000)
    p.add_argument("--height", type=int, default=1000)
    p.add_argument("--n-spheres", type=int, default=100)
    p.add_argument("--r-min", type=float, required=True)
    p.add_argument("--r-max", type=float, required=True)
    p.add_argument("--seed", type=int, required=True)
    p.add_argument("--poisson-scale", type=float, default=None)
    p.add_argument("--gaussian-sigma", type=float, default=None)
    p.add_argument("--allow-overlap", action="store_true")
    p.add_argument("--out-image", required=True)
    p.add_argument("--out-truth", required=True)

    p = sub.add_parser("bench", help="runtime scaling sweeps (device time of convolve -> dog -> extrema)")
    p.add_argument("--sweep", choices=("n_bin", "max_sigma"), required=True)
    p.add_argument("--values", required=True, help="comma-separated sweep values")
    p.add_argument("--backend", choices=BACKENDS, default=BACKENDS[0])
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=1)
    p.add_argument("--width", type=int, default=512)
    p.add_argument("--height", type=int, default=512)
    p.add_argument("--seed", type=int, required=True, help="seed for the benchmark scene")
    p.add_argument("--min-sigma", type=float, default=1.0)
    p.add_argument("--max-sigma", type=float, default=10.0, help="fixed value for n_bin sweeps")
    p.add_argument("--n-bin", type=int, default=10, help="fixed value for max_sigma sweeps")
    p.add_argument("--device", type=int, default=None)
    p.add_argument("--out", required=True)

    p = sub.add_parser("serve", help="run the analysis HTTP service")
    p.add_argument("--listen", default=os.environ.get("DROPLET_LISTEN", "127.0.0.1:8750"),
                   help="ADDR:PORT (env DROPLET_LISTEN)")
    p.add_argument("--workers", type=int, default=int(os.environ.get("DROPLET_WORKERS", "1")),
                   help="concurrent detection workers (env DROPLET_WORKERS)")
    p.add_argument("--backlog", type=int, default=4)
    p.add_argument("--max-request-mb", type=float, default=16.0)
    _add_detector_flags(p, ladder_required=False)

    p = sub.add_parser("evaluate", help="score a blob set against ground truth")
    p.add_argument("--pred", required=True)
    p.add_argument("--truth", required=True)
    p.add_argument("--iou", type=float, default=0.5)
    p.add_argument("--out", required=True)

    p = sub.add_parser("parity", help="compare two arithmetic tiers over a scene directory")
    p.add_argument("--scenes", required=True, help="directory of .raw image files + <stem>.csv truths")
    # the reference compares its direct and fft backends (--backend-a / --backend-b); both sides run on
    # the device here and differ in the arithmetic tier
    p.add_argument("--dtype-a", choices=("float32", "float64"), default="float64")
    p.add_argument("--dtype-b", choices=("float32", "float64"), default="float32")
    _add_detector_flags(p, ladder_required=True)
    p.add_argument("--iou", type=float, default=0.5)
    p.add_argument("--out", required=True)
    return parser


# ---------------------------------------------------------------------------------
def load_image(path):
    """Raw float frames go straight to pinned memory; 8/16-bit PNG/TIFF need imageio
    (same scaling and checks as the reference's images.load_image, images.py:70-98)."""
    p = Path(path)
    if not p.is_file():
        raise FileNotFoundError(f"no such image: {path}")
    if p.suffix.lower() in RAW_SUFFIXES:
        try:
            return formats.read_raw_pinned(p)
        except RuntimeError:                       # no CUDA runtime for pinned pages
            return formats.read_raw(p)
    try:
        import imageio.v3 as iio
    except ImportError:
        raise ValueError(f"{path}: PNG/TIFF input needs imageio; use the raw float format") from None
    try:
        arr = iio.imread(p)
    except Exception as exc:
        raise ValueError(f"unreadable image {path}: {exc}") from exc
    if arr.ndim != 2:
        raise ValueError(f"{path}: multi-channel image (shape {arr.shape}); convert to grayscale first")
    scale = {np.dtype(np.uint8): 255.0, np.dtype(np.uint16): 65535.0}.get(arr.dtype)
    if scale is None:
        raise ValueError(f"{path}: unsupported bit depth {arr.dtype}; expected uint8 or uint16")
    return arr.astype(np.float32) / scale


def _cmd_detect(args) -> int:
    image = load_image(args.input)
    detector = Detector(_params(args), device=args.device)
    try:
        result = detector.run(image)
    finally:
        detector.close()
    formats.write_blobset_json(args.out_json, result.blobs, image_name=Path(args.input).name)
    if args.out_hist:
        formats.write_histogram_csv(args.out_hist, result.histogram)
    print(f"{len(result.blobs)} blobs -> {args.out_json}")
    return 0


def _cmd_simulate(args) -> int:
    frame = synth.droplet_scene(args.width, args.height, args.n_spheres, (args.r_min, args.r_max),
                                seed=args.seed, allow_overlap=args.allow_overlap)
    if args.poisson_scale is not None or args.gaussian_sigma is not None:
        frame = synth.sensor_noise(frame,
                                   photons=255.0 if args.poisson_scale is None else args.poisson_scale,
                                   read_sigma=0.01 if args.gaussian_sigma is None else args.gaussian_sigma,
                                   seed=args.seed)
    if Path(args.out_image).suffix.lower() not in RAW_SUFFIXES:
        raise ValueError("simulate writes the raw float format: use an --out-image ending in .raw or .bin")
    formats.write_raw(args.out_image, frame.image)
    synth.write_truth_csv(args.out_truth, synth.Frame(frame.image, frame.truths, args.seed))
    print(f"scene with {len(frame.truths)} spheres -> {args.out_image}")
    return 0


def time_detection_core(image, params: DetectionParams, reps: int, warmup: int = 1, device=None) -> dict:
    """One sweep point: device milliseconds of convolve -> dog -> extrema (CUDA events),
    the region the reference's bench.time_detection_core times on the host (bench.py:46-86)."""
    if reps < 3:
        raise ValueError(f"timed_runs must be >= 3, got {reps}")
    if warmup < 1:
        raise ValueError(f"warmup must be >= 1, got {warmup}")
    detector = Detector(params, device=device, slots=1)
    try:
        for _ in range(warmup):
            detector.run(image)
        times = []
        for _ in range(reps):
            t = detector.run(image).timings_ms
            times.append(t["convolve_ms"] + t["extrema_ms"])
    finally:
        detector.close()
    times = np.array(times)
    try:
        import torch
        hardware = torch.cuda.get_device_name(detector.device).replace(",", " ")
    except Exception:
        hardware = platform.machine()
    return {"backend": params.backend, "n_bin": params.n_bin, "max_sigma": params.max_sigma,
            "width": int(image.shape[1]), "height": int(image.shape[0]), "warmup_runs": warmup,
            "timed_runs": reps, "median_ms": float(np.median(times)),
            "p10_ms": float(np.percentile(times, 10)), "p90_ms": float(np.percentile(times, 90)),
            "hardware": f"{hardware}/py{platform.python_version()}"}


_BENCH_COLUMNS = ("backend", "n_bin", "max_sigma", "width", "height", "warmup_runs", "timed_runs",
                  "median_ms", "p10_ms", "p90_ms", "hardware")


def _cmd_bench(args) -> int:
    try:
        values = [float(v) for v in args.values.split(",") if v.strip()]
    except ValueError:
        print(f"error: bad --values list {args.values!r}", file=sys.stderr)
        return USAGE_ERROR
    if not values:
        print("error: --values is empty", file=sys.stderr)
        return USAGE_ERROR
    # the reference's benchmark scene (cli.py:233-243): realistic content, not ground-truthed
    count = max(4, int(40 * args.width * args.height / 512 ** 2))
    r_hi = min(15.0, (min(args.width, args.height) - 4) / 4)
    image = synth.droplet_scene(args.width, args.height, count, (min(3.0, r_hi / 2), r_hi),
                                seed=args.seed, allow_overlap=True).image
    rows = []
    for v in values:
        point = {"n_bin": int(v)} if args.sweep == "n_bin" else {"max_sigma": float(v)}
        params = DetectionParams(**{"min_sigma": args.min_sigma, "max_sigma": args.max_sigma,
                                    "n_bin": args.n_bin, "backend": args.backend, "preprocess": False,
                                    "prune": False, **point})
        rows.append(time_detection_core(image, params, args.reps, args.warmup, args.device))
    with open(args.out, "w") as f:
        f.write(",".join(_BENCH_COLUMNS) + "\n")
        for r in rows:
            f.write(",".join(repr(r[c]) if isinstance(r[c], float) else str(r[c]) for c in _BENCH_COLUMNS) + "\n")
    for r in rows:
        print(f"{r['backend']} n_bin={r['n_bin']} max_sigma={r['max_sigma']}: "
              f"median {r['median_ms']:.3f} ms [{r['p10_ms']:.3f}, {r['p90_ms']:.3f}]")
    return 0


def _cmd_serve(args) -> int:
    from .service import ServiceConfig, serve
    host, _, port = args.listen.rpartition(":")
    if not host or not port.isdigit():
        print(f"error: bad --listen value {args.listen!r}", file=sys.stderr)
        return USAGE_ERROR
    serve(ServiceConfig(host=host, port=int(port), params=_params(args),
                        max_request_bytes=int(args.max_request_mb * 1024 * 1024),
                        workers=max(1, args.workers), backlog=max(0, args.backlog), device=args.device))
    return 0


def _cmd_evaluate(args) -> int:
    """cli.py:166-181 of the reference: score a blob JSON against a truth CSV"""
    from . import evaluate as ev
    preds = formats.read_blobset_json(args.pred)
    truths = synth.read_truth_csv(args.truth)
    report = ev.match_voc(preds, truths, args.iou)
    ev.write_report_json(args.out, report)
    print(f"precision={report.precision:.4f} recall={report.recall:.4f} "
          f"(tp={report.tp} fp={report.fp} fn={report.fn})")
    return 0


def _cmd_parity(args) -> int:
    """cli.py:184-213 of the reference, with arithmetic tiers in place of CPU backends"""
    from . import evaluate as ev
    scene_dir = Path(args.scenes)
    if not scene_dir.is_dir():
        raise FileNotFoundError(f"scene directory not found: {scene_dir}")
    paths = sorted(p for p in scene_dir.iterdir() if p.suffix.lower() in (".png", ".tif", ".tiff", ".raw"))
    if not paths:
        raise FileNotFoundError(f"no scene images in {scene_dir}")
    imgs, truths, names = [], [], []
    for p in paths:
        truth_path = p.with_suffix(".csv")
        if not truth_path.is_file():
            raise FileNotFoundError(f"missing truth file {truth_path}")
        imgs.append(np.asarray(load_image(p)))
        truths.append(synth.read_truth_csv(truth_path))
        names.append(p.stem)
    if args.device is not None:
        import torch
        torch.cuda.set_device(args.device)
    params = _params(args)
    stats = ev.parity(imgs, params, params, truths, args.iou, dtype_a=np.dtype(args.dtype_a),
                      dtype_b=np.dtype(args.dtype_b))
    ev.write_parity_csv(args.out, stats, names)
    print(f"{len(imgs)} scenes: mean dP={stats.mean_dp:+.2e} mean dR={stats.mean_dr:+.2e}")
    return 0


_COMMANDS = {"detect": _cmd_detect, "simulate": _cmd_simulate, "bench": _cmd_bench, "serve": _cmd_serve,
             "evaluate": _cmd_evaluate, "parity": _cmd_parity}


def main(argv=None) -> int:
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as exc:
        return USAGE_ERROR if exc.code is None else exc.code
    try:
        return _COMMANDS[args.command](args)
    except (ValueError, FileNotFoundError, json.JSONDecodeError, RuntimeError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return RUNTIME_ERROR


if __name__ == "__main__":
    sys.exit(main())
