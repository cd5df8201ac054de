"""ctypes binding of libdogblob_b200.so for the reference `dogblob` package.

Dropped into `pkg/src/dogblob/` as `_cuda.py`; needs nothing but numpy and the shared library
(`DOGBLOB_B200_LIB` or the default loader path).  One `CudaPlan` = plan handle + one buffer set
(one frame in flight); `Detector.cuda_plan_for` keeps one per image shape behind the detector's
plan lock.  The complete host layer with slot pools, batching and preprocessing on the device is
`paper_2010_08486_b200.detector`.
"""
import ctypes as C
import os

import numpy as np

BLOB = np.dtype([("x", "<f8"), ("y", "<f8"), ("sigma", "<f8"), ("radius", "<f8"),
                 ("response", "<f8"), ("slice", "<i4"), ("flags", "<u4")])   # dogblob_blob, 48 bytes
HEADER_BYTES = 64
_lib = None


def lib():
    """The shared library, loaded on first use (so that importing dogblob never needs it)."""
    global _lib
    if _lib is None:
        so = C.CDLL(os.environ.get("DOGBLOB_B200_LIB", "libdogblob_b200.so"))
        so.dogblob_last_error.restype = C.c_char_p
        so.dogblob_workspace_bytes.restype = so.dogblob_result_bytes.restype = C.c_size_t
        so.dogblob_workspace_bytes.argtypes = so.dogblob_result_bytes.argtypes = [C.c_void_p]
        so.dogblob_image_pitch.restype = C.c_int64
        so.dogblob_image_pitch.argtypes = [C.c_void_p]
        so.dogblob_plan_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        so.dogblob_plan_destroy.argtypes = [C.c_void_p]
        so.dogblob_plan_destroy.restype = None
        so.dogblob_detect_host.argtypes = [C.c_void_p, C.c_void_p, C.c_float, C.c_int, C.c_double, C.c_int,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                           C.c_void_p]
        so.dogblob_fetch_blobs.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        so.dogblob_stream_sync.argtypes = [C.c_void_p]
        so.dogblob_device_alloc.argtypes = [C.c_int, C.c_size_t, C.POINTER(C.c_void_p)]
        so.dogblob_device_free.argtypes = [C.c_int, C.c_void_p]
        so.dogblob_pinned_alloc.argtypes = [C.c_size_t, C.POINTER(C.c_void_p)]
        so.dogblob_pinned_free.argtypes = [C.c_void_p]
        _lib = so
    return _lib


def _check(rc):
    if rc == 1:
        raise ValueError(lib().dogblob_last_error().decode())
    if rc:
        raise RuntimeError(lib().dogblob_last_error().decode())


class CudaPlan:
    """Plan + buffers for one image shape (one frame in flight; guard with a lock to share)."""

    def __init__(self, ladder, bank, shape, max_blobs=65536, device=0):
        so = lib()
        taps = [np.exp(-np.arange(-r, r + 1.0) ** 2 / (2 * s * s)) for s, r in zip(ladder.sigmas, bank.radii)]
        taps = [(t / t.sum()).astype(np.float32) for t in taps]               # w_i, k_i == outer(w_i, w_i)
        offs = np.cumsum([0] + [t.size for t in taps[:-1]]).astype(np.int64)
        flat = np.concatenate(taps)
        sig = np.ascontiguousarray(ladder.sigmas, dtype=np.float64)
        rad = np.ascontiguousarray(bank.radii, dtype=np.int32)
        self.device, self.shape, self.max_blobs = device, (int(shape[0]), int(shape[1])), max_blobs
        self.h = C.c_void_p()
        self._dev, self._pin = [], None
        _check(so.dogblob_plan_create(device, self.shape[0], self.shape[1], len(sig), sig.ctypes.data,
                                      rad.ctypes.data, flat.ctypes.data, offs.ctypes.data, max_blobs,
                                      C.byref(self.h)))
        try:
            pitch = so.dogblob_image_pitch(self.h)
            self.d_image = self._device(self.shape[0] * pitch * 4)
            self.d_work = self._device(so.dogblob_workspace_bytes(self.h))
            self.d_result = self._device(so.dogblob_result_bytes(self.h))
            self.n_host = min(4096, max_blobs)
            nbytes = HEADER_BYTES + BLOB.itemsize * self.n_host
            pin = C.c_void_p()
            _check(so.dogblob_pinned_alloc(nbytes, C.byref(pin)))
            self._pin = pin
            self.h_result = np.ctypeslib.as_array(C.cast(pin, C.POINTER(C.c_uint8)), shape=(nbytes,))
        except Exception:
            self.close()
            raise

    def _device(self, nbytes):
        p = C.c_void_p()
        _check(lib().dogblob_device_alloc(self.device, nbytes, C.byref(p)))
        self._dev.append(p)
        return p

    def close(self):
        so = lib()
        for p in self._dev:
            so.dogblob_device_free(self.device, p)
        self._dev = []
        if self._pin is not None:
            so.dogblob_pinned_free(self._pin)
            self._pin = None
        if self.h:
            so.dogblob_plan_destroy(self.h)
            self.h = C.c_void_p()

    def detect(self, img, threshold, neighborhood, overlap, prune, stream=None):
        """Records (BLOB dtype) sorted by (-response, y, x, sigma), exactly _sort_blobs' order."""
        so = lib()
        img = np.ascontiguousarray(img, dtype=np.float32)
        if img.shape != self.shape:
            raise ValueError(f"plan built for {self.shape[1]}x{self.shape[0]}, image is {img.shape[1]}x{img.shape[0]}")
        _check(so.dogblob_detect_host(self.h, img.ctypes.data, C.c_float(threshold), neighborhood,
                                      C.c_double(overlap), int(prune), self.d_image, self.d_work, self.d_result,
                                      self.h_result.ctypes.data, self.n_host, stream, None))
        _check(so.dogblob_stream_sync(stream))
        n = int(self.h_result[:4].view("<i4")[0])
        flags = int(self.h_result[20:24].view("<u4")[0])
        if flags & 1:
            raise RuntimeError("candidate capacity exceeded; rebuild the plan with a larger max_blobs")
        recs = np.empty(n, BLOB)
        k = min(n, self.n_host)
        recs[:k] = self.h_result[HEADER_BYTES:HEADER_BYTES + BLOB.itemsize * k].view(BLOB)
        if n > k:
            _check(so.dogblob_fetch_blobs(self.d_result, k, n - k, recs[k:].ctypes.data, stream))
            _check(so.dogblob_stream_sync(stream))
        return recs
