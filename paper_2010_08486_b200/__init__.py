"""B200-native Difference-of-Gaussians blob detector (arXiv 2010.08486 hot path).

Keeps the reference `dogblob` detector API (DetectionParams / Detector.run ->
blobs (y, x, sigma), radius = sqrt(2) sigma, radius/volume histogram) with
`backend="cuda"`: hand-written sm_100a kernels behind a C ABI
(include/dogblob_b200.h).  See DESIGN.md and INTEGRATION.md.
"""

from .scale_space import KernelBank, SigmaLadder, TapBank, build_kernel_bank, build_ladder
from .detector import (
    BACKENDS,
    Blob,
    BlobSet,
    DetectionParams,
    DetectResult,
    Detector,
    DoGStack,
    RadiusHistogram,
    ScaleStack,
    convolve_bank,
    detect,
    disk_intersection_area,
    dog_stack,
    find_extrema,
    fused_dog,
    histogram,
    normalized_overlap,
    prune_overlaps,
)

from .images import preprocess
from .formats import (
    blobset_from_doc,
    blobset_to_doc,
    histogram_to_doc,
    raw_from_bytes,
    read_blobset_json,
    read_raw,
    read_raw_pinned,
    write_blobset_json,
    write_histogram_csv,
    write_raw,
)

__version__ = "0.1.0"

__all__ = [
    "SigmaLadder", "KernelBank", "TapBank", "build_ladder", "build_kernel_bank",
    "BACKENDS", "ScaleStack", "DoGStack", "Blob", "BlobSet", "RadiusHistogram",
    "DetectionParams", "DetectResult", "Detector", "convolve_bank", "dog_stack", "fused_dog",
    "find_extrema", "prune_overlaps", "normalized_overlap", "disk_intersection_area",
    "histogram", "detect", "preprocess", "raw_from_bytes", "read_raw", "read_raw_pinned", "write_raw",
    "blobset_to_doc", "blobset_from_doc", "write_blobset_json", "read_blobset_json",
    "histogram_to_doc", "write_histogram_csv", "__version__",
]
