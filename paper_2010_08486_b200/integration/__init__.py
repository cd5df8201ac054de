"""Files a maintainer of the reference `dogblob` package adds to get `backend="cuda"`
(INTEGRATION.md): `_cuda.py` is dropped into `pkg/src/dogblob/` unchanged, `patch_reference()`
applies the four edits of INTEGRATION.md section 3 to a copy of the package."""
from .patch import patch_reference  # noqa: F401
