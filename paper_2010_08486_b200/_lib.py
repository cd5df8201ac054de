"""ctypes binding of libdogblob_b200.so (include/dogblob_b200.h).

There is no CPU fallback: if the library cannot be loaded, every call that
needs it raises RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libdogblob_b200.so"
ABI_VERSION = 1

OK, EINVAL, ECUDA, ENOMEM = 0, 1, 2, 3
FLAG_OVERFLOW = 1
BLOB_SCALE_EDGE = 1
BLOB_MERGED = 2
RESULT_HEADER_BYTES = 64
GATE_INTS = 16

# numpy mirrors of the C structs
BLOB_DTYPE = np.dtype([("x", "<f8"), ("y", "<f8"), ("sigma", "<f8"), ("radius", "<f8"),
                       ("response", "<f8"), ("slice", "<i4"), ("flags", "<u4")])
HEADER_DTYPE = np.dtype([("n_blobs", "<i4"), ("n_candidates", "<i4"), ("n_flagged", "<i4"),
                         ("n_plateau", "<i4"), ("n_merges", "<i4"), ("flags", "<u4"),
                         ("capacity", "<i4"), ("conv_ns", "<i4"), ("extrema_ns", "<i4"),
                         ("prune_ns", "<i4"), ("prune_profile", "<i4", (4,)), ("n_seeds", "<i4"), ("reserved", "<i4")])
assert BLOB_DTYPE.itemsize == 48 and HEADER_DTYPE.itemsize == RESULT_HEADER_BYTES

# every symbol include/dogblob_b200.h declares: name -> (restype, argtypes)
_vp, _i, _f, _d, _sz, _i64 = C.c_void_p, C.c_int, C.c_float, C.c_double, C.c_size_t, C.c_int64
SIGNATURES = {
    "dogblob_abi_version": (_i, []),
    "dogblob_last_error": (C.c_char_p, []),
    "dogblob_plan_create": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, _i, C.POINTER(_vp)]),
    "dogblob_plan_destroy": (None, [_vp]),
    "dogblob_workspace_bytes": (_sz, [_vp]),
    "dogblob_result_bytes": (_sz, [_vp]),
    "dogblob_image_pitch": (_i64, [_vp]),
    "dogblob_plan_conv_engine": (C.c_int, [_vp]),
    "dogblob_plan_conv_groups": (C.c_int, [_vp, C.POINTER(C.c_int32), C.c_int]),
    "dogblob_detect": (_i, [_vp, _vp, _f, _i, _d, _i, _vp, _vp, _vp, _vp]),
    "dogblob_detect_host": (_i, [_vp, _vp, _f, _i, _d, _i, _vp, _vp, _vp, _vp, _i, _vp, _vp]),
    "dogblob_detect_host_streamed": (_i, [_vp, _vp, _f, _i, _d, _i, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp,
                                          _vp, _vp]),
    "dogblob_upload_image": (_i, [_vp, _vp, _vp, _vp]),
    "dogblob_fetch_blobs": (_i, [_vp, _i, _i, _vp, _vp]),
    "dogblob_fetch_result": (_i, [_vp, _i, _vp, _vp]),
    "dogblob_scale_space": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "dogblob_dog": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "dogblob_dog_from_levels": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp]),
    "dogblob_blobspace_bytes": (_sz, [_i]),
    "dogblob_result_bytes_for": (_sz, [_i]),
    "dogblob_extrema": (_i, [_i, _i, _i, _vp, _vp, _f, _i, _i, _vp, _vp, _vp]),
    "dogblob_prune": (_i, [_i, _vp, _d, _i, _vp, _vp, _vp]),
    "dogblob_preprocess_bytes": (_sz, [_i, _i]),
    "dogblob_preprocess": (_i, [_i, _i, _vp, _i64, _i, _vp, _i64, _i64, _vp, _vp, _i64, _vp]),
    "dogblob_preprocess_status": (_i, [_vp, _vp, _vp]),
    "dogblob_event_record": (_i, [_vp, _vp]),
    "dogblob_event_create": (_i, [C.POINTER(_vp)]),
    "dogblob_event_destroy": (_i, [_vp]),
    "dogblob_event_elapsed_ms": (_i, [_vp, _vp, C.POINTER(_f)]),
    "dogblob_event_intervals_ms": (_i, [_vp, _i, _vp]),
    "dogblob_stream_sync": (_i, [_vp]),
    "dogblob_device_count": (_i, [C.POINTER(_i)]),
    "dogblob_f64_workspace_bytes": (C.c_size_t, [_i, _i, _i, _i]),
    "dogblob_scale_space_f64": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "dogblob_dog_inplace_f64": (_i, [_i, _i, _i, _vp, _vp, _vp]),
    "dogblob_extrema_f64": (_i, [_i, _i, _i, _vp, _vp, C.c_double, _i, _i, _vp, _vp, _vp]),
    "dogblob_detect_f64": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, C.c_double, _i, C.c_double, _i, _i,
                                _vp, _vp, _vp]),
    "dogblob_match_voc": (_i, [_i, _vp, _vp, _vp, _vp, C.c_double, _vp, _vp, _vp, _vp, _vp]),
    "dogblob_synth_frames": (_i, [_i, _i, _i, _i64, _i, C.c_double, C.c_double, C.c_uint64, C.c_double, C.c_double,
                                  _vp, _vp, _vp]),
    "dogblob_device_alloc": (_i, [_i, C.c_size_t, C.POINTER(_vp)]),
    "dogblob_device_free": (_i, [_i, _vp]),
    "dogblob_pinned_alloc": (_i, [C.c_size_t, C.POINTER(_vp)]),
    "dogblob_pinned_free": (_i, [_vp]),
}

_lock = threading.Lock()
_lib = None


def load():
    """Load the shared library once; raise RuntimeError if it is missing or stale."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH.name} is not built; run `python -m paper_2010_08486_b200.build` "
                "(nvcc, sm_100a). There is no CPU fallback for backend='cuda'.")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)      # AttributeError if the header and library disagree
            fn.restype = res
            fn.argtypes = args
        if lib.dogblob_abi_version() != ABI_VERSION:
            raise RuntimeError("libdogblob_b200.so ABI version mismatch; rebuild it")
        _lib = lib
        return lib


def check(rc: int) -> None:
    """Map the C status to the reference's exception conventions."""
    if rc == OK:
        return
    msg = load().dogblob_last_error().decode("utf-8", "replace")
    if rc == EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"dogblob_b200 (status {rc}): {msg}")


def ptr(array: np.ndarray) -> int:
    return array.ctypes.data
