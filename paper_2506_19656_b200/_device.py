"""Device plumbing for the drop-in: host/device conversion, dtype codes,
current stream, and the device error word. PyTorch only provides device
memory and streams here; every computation runs in libcvb200."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import ConfigurationError

_NP_CODES = {
    np.dtype(np.uint8): _lib.CV_U8,
    np.dtype(np.uint16): _lib.CV_U16,
    np.dtype(np.float32): _lib.CV_F32,
    np.dtype(np.float64): _lib.CV_F64,
}
_TORCH_CODES = {
    torch.uint8: _lib.CV_U8,
    torch.float32: _lib.CV_F32,
    torch.float64: _lib.CV_F64,
}
if hasattr(torch, "uint16"):
    _TORCH_CODES[torch.uint16] = _lib.CV_U16


class Arr:
    """A device tensor plus how the caller handed it over.

    ``code`` is the element type the kernels see (u16 data travels in an
    int16/uint16 tensor: only the bytes matter), ``host`` tells the wrappers
    to hand numpy back, ``np_dtype`` is the caller's numpy dtype.
    """

    __slots__ = ("t", "code", "host", "np_dtype", "shape")

    def __init__(self, t, code, host, np_dtype, shape):
        self.t = t
        self.code = code
        self.host = host
        self.np_dtype = np_dtype
        self.shape = tuple(shape)

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    @property
    def device(self):
        return self.t.device


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 path needs a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def is_device_tensor(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def _code_of_np(dt: np.dtype) -> int | None:
    return _NP_CODES.get(np.dtype(dt))


def to_device(x, *, allow=("u8", "u16", "f32", "f64"), widen_ints=False) -> Arr:
    """Bring a numpy array or torch tensor onto the GPU, contiguous.

    float16 is widened to float32 (exact). With ``widen_ints`` other integer
    types are left for the caller (returned with code None).
    """
    if isinstance(x, torch.Tensor):
        t = x
        host = not t.is_cuda
        if t.dtype == torch.float16 or t.dtype == torch.bfloat16:
            t = t.float()
        if host:
            t = t.to(default_device())
        t = t.contiguous()
        code = _TORCH_CODES.get(t.dtype)
        if code is None and t.dtype == torch.int16:
            code = _lib.CV_U16  # uint16 payload carried in int16
        np_dtype = {
            _lib.CV_U8: np.dtype(np.uint8),
            _lib.CV_U16: np.dtype(np.uint16),
            _lib.CV_F32: np.dtype(np.float32),
            _lib.CV_F64: np.dtype(np.float64),
        }.get(code)
        return Arr(t, code, host, np_dtype, t.shape)
    a = np.asarray(x)
    dt = a.dtype
    if dt == np.float16:
        a = a.astype(np.float32)
        dt = a.dtype
    code = _code_of_np(dt)
    a = np.ascontiguousarray(a)
    if code is None:
        t = torch.from_numpy(a) if a.dtype != np.bool_ else torch.from_numpy(a.view(np.uint8))
    else:
        t = torch.from_numpy(a)
    t = t.to(default_device())
    return Arr(t, code, True, dt, a.shape)


def to_host_like(t: torch.Tensor, like: Arr, np_dtype=None):
    """Return ``t`` as numpy when the caller gave host data, else the tensor."""
    if not like.host:
        return t
    out = t.cpu().numpy()
    if np_dtype is not None and out.dtype != np_dtype:
        out = out.view(np_dtype)
    return out


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class ErrWord:
    """Device uint32 error word (CV_FLAG_*), read once per call."""

    def __init__(self, device):
        self.t = torch.zeros(1, dtype=torch.int32, device=device)

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    def flags(self) -> int:
        return int(self.t.item()) & 0xFFFFFFFF

    def reset(self) -> None:
        self.t.zero_()


def empty(shape, dtype, device) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=device)


def workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 8), dtype=torch.uint8, device=device)


def f64_tensor(values, device) -> torch.Tensor:
    return torch.as_tensor(np.asarray(values, dtype=np.float64), device=device)


def require_4d(shape, what="array"):
    if len(shape) != 4:
        raise ConfigurationError(f"expected a [t,y,x,c] array, got {len(shape)}-D")


def out_dtype_for_depth(bit_depth: int):
    return (torch.uint8, np.dtype(np.uint8)) if bit_depth == 8 else (torch.uint16, np.dtype(np.uint16))
