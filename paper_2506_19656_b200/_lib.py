"""ctypes binding of ``lib/libcvb200.so`` (the C ABI declared in include/cvb200.h).

There is no CPU fallback: if the library is missing every entry point raises.
The binding only passes integers (device pointers, sizes, flags) and the
current torch CUDA stream handle.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import ConfigurationError

LIB_PATH = Path(os.environ.get("CVB200_LIB", Path(__file__).resolve().parent / "lib" / "libcvb200.so"))

# dtype / layout / status codes (mirror include/cvb200.h)
CV_U8, CV_U16, CV_F32, CV_F64 = 0, 1, 2, 3
CV_LAYOUT_CHANNEL_LAST, CV_LAYOUT_PLANAR = 0, 1
CV_PAD_REPEAT, CV_PAD_ZERO = 0, 1
CV_OK, CV_ERR_ARG, CV_ERR_SHAPE, CV_ERR_UNSUPPORTED, CV_ERR_CUDA = 0, 1, 2, 3, 4
CV_FLAG_NONFINITE, CV_FLAG_NAN, CV_FLAG_RANGE, CV_FLAG_INT_RANGE = 1, 2, 4, 8

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_F32 = ctypes.c_float
_SZ = ctypes.c_size_t
_INT = ctypes.c_int

# name -> (argtypes, restype); keep in the order of include/cvb200.h
SIGNATURES = {
    "cv_version": ([], _INT),
    "cv_status_string": ([_INT], ctypes.c_char_p),
    "cv_last_error": ([], ctypes.c_char_p),
    "cv_max_channels": ([], _INT),
    "cv_launch_count": ([], ctypes.c_ulonglong),
    "cv_set_variant": ([ctypes.c_char_p, _INT], _INT),
    "cv_stats_ws_bytes": ([_I64, _I32], _SZ),
    "cv_num_segments": ([_I64, _I32], _I64),
    "cv_stats_reset": ([_P, _I64, _I32, _P], _INT),
    "cv_stats": ([_P, _I32, _I64, _I64, _I64, _I32, _I32, _I32, _P, _P, _P, _P], _INT),
    "cv_stats_finalize": ([_P, _I64, _I32, _I32, _F32, _P, _P, _P, _P], _INT),
    "cv_stats_lead_flags": ([_P, _I64, _I32, _P, _P], _INT),
    "cv_forward_fill": ([_P, _I64, _I64, _I64, _F32, _I32, _P, _P, _P, _P, _P, _P], _INT),
    "cv_quantize": ([_P, _I32, _I64, _I64, _I64, _I32, _P, _P, _I32, _I32, _I32, _F32, _I32, _P,
                     _P, _P, _P, _I32, _I32, _I32, _P, _P, _P, _P], _INT),
    "cv_dequantize": ([_P, _I32, _I64, _I64, _I64, _I32, _I32, _P, _P, _I32, _P, _I32, _P, _P], _INT),
    "cv_gram_ws_bytes": ([_I64, _I32], _SZ),
    "cv_pca_gram": ([_P, _I32, _I64, _I32, _P, _P, _P, _P, _P], _INT),
    "cv_pca_project": ([_P, _I32, _I64, _I64, _I32, _P, _P, _I32, _P, _I32, _P, _P, _P], _INT),
    "cv_pca_inverse": ([_P, _I32, _I64, _I64, _I32, _P, _P, _I32, _P, _I32, _P], _INT),
    "cv_eval_ws_bytes": ([_I64, _I64, _I64, _I64, _I32, _I32], _SZ),
    "cv_eval": ([_P, _I32, _I32, _P, _P, _I32, _P, _P, _P, _I32, _P, _I32,
                 _I64, _I64, _I64, _I64, _I32, _P, _I32, _P, _P, _P, _P, _P, _P], _INT),
    "cv_select_stack": ([_P, _P, _I32, _I32, _I64, _I64, _I64, _P, _P], _INT),
    "cv_planar_pack": ([_P, _I32, _I64, _I64, _I32, _P, _P], _INT),
    "cv_planar_unpack": ([_P, _I32, _I64, _I64, _I32, _P, _P], _INT),
    "cv_angle_ws_bytes": ([], _SZ),
    "cv_spectral_angle": ([_P, _I32, _P, _I32, _I64, _I32, _P, _P, _P], _INT),
}

_lock = threading.Lock()
_lib = None


def load(path: Path | None = None) -> ctypes.CDLL:
    """Load (once) and type the library. Raises RuntimeError if it was not built."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise RuntimeError(
                f"{p} is missing: the B200 CUDA library is not built "
                "(run `python -c 'import __graft_entry__ as g; g.build()'`); "
                "there is no CPU fallback"
            )
        lib = ctypes.CDLL(str(p))
        for name, (argtypes, restype) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = restype
        if path is None:
            _lib = lib
        return lib


def check(status: int, what: str) -> None:
    """Map a CV_ERR_* status to the reference's exception convention."""
    if status == CV_OK:
        return
    lib = load()
    msg = lib.cv_last_error().decode() or lib.cv_status_string(status).decode()
    if status == CV_ERR_CUDA:
        raise RuntimeError(f"{what}: {msg}")
    raise ConfigurationError(msg)


def call(name: str, *args) -> None:
    fn = getattr(load(), name)
    check(fn(*args), name)


def set_variant(name: str, value: int) -> None:
    """Select a kernel variant (A/B measurements, tests); see cv_set_variant."""
    check(load().cv_set_variant(name.encode(), int(value)), "cv_set_variant")
