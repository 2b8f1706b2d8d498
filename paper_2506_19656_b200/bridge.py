"""Array side of the codec bridge: the planar byte streams an encoder reads and a
decoder returns (/root/reference/pkg/src/cubevid/codecs/bridge.py:157-174).

``_frames_to_planar_bytes`` / ``_planar_bytes_to_frames`` keep the reference's
names, arguments, dtypes and the ``CorruptStreamError`` of a truncated stream;
the ``[t,y,x,c] <-> [t,c,y,x]`` transposition runs on the device
(``cv_planar_pack`` / ``cv_planar_unpack``). Host inputs give host outputs
(``bytes`` / numpy); CUDA tensors stay on the device (a flat uint8 tensor is the
byte stream). The fused pipeline never needs these: ``cv_quantize`` writes the
planar layout directly and ``cv_eval`` reads it (pipeline.py).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as dev
from . import _lib
from .errors import ConfigurationError, CorruptStreamError


def _sample(bit_depth: int):
    return (torch.uint8, 1, _lib.CV_U8) if bit_depth == 8 else (torch.uint16, 2, _lib.CV_U16)


def _frames_to_planar_bytes(frames, bit_depth: int):
    """``[t,y,x,c]`` integer frames -> planar ``u1`` / ``<u2`` bytes (bridge.py:157-160)."""
    tdt, _, code = _sample(bit_depth)
    x = dev.to_device(frames)
    if len(x.shape) != 4:
        raise ConfigurationError(f"expected [t,y,x,c] frames, got {len(x.shape)}-D")
    t = x.t
    if t.dtype != tdt:
        if t.dtype == torch.int16 and tdt == torch.uint16:
            t = t.view(torch.uint16)
        else:  # astype(dtype) of the reference: value-preserving for in-range samples
            t = t.to(torch.int32).to(tdt)
    T, H, W, Cn = (int(v) for v in x.shape)
    out = torch.empty((T, Cn, H, W), dtype=tdt, device=t.device)
    _lib.call("cv_planar_pack", t.data_ptr(), code, T, H * W, Cn, out.data_ptr(), dev.stream_ptr(t.device))
    flat = out.view(torch.uint8).reshape(-1)
    return flat.cpu().numpy().tobytes() if x.host else flat


def _planar_bytes_to_frames(raw, h: int, w: int, n_planes: int, bit_depth: int):
    """Planar bytes -> ``[t,y,x,c]`` frames; a byte count that is not a whole number
    of frames is a ``CorruptStreamError`` (bridge.py:163-174)."""
    tdt, isz, code = _sample(bit_depth)
    on_device = isinstance(raw, torch.Tensor) and raw.is_cuda
    if isinstance(raw, torch.Tensor):
        buf = raw.contiguous().view(torch.uint8).reshape(-1)
        n = buf.numel()
    else:
        arr = np.frombuffer(raw, dtype=np.uint8) if not isinstance(raw, np.ndarray) else \
            np.ascontiguousarray(raw).view(np.uint8).reshape(-1)
        n = arr.size
    frame_bytes = h * w * n_planes * isz
    if frame_bytes == 0 or n % frame_bytes != 0:
        raise CorruptStreamError(f"decoded byte count {n} is not a whole number of "
                                 f"{h}x{w}x{n_planes} frames")
    if not isinstance(raw, torch.Tensor):
        buf = torch.from_numpy(arr.copy() if not arr.flags.writeable else arr)
    if not buf.is_cuda:
        buf = buf.to(dev.default_device())
    T = n // frame_bytes
    out = torch.empty((T, h, w, n_planes), dtype=tdt, device=buf.device)
    if T:
        _lib.call("cv_planar_unpack", buf.data_ptr(), code, T, h * w, n_planes, out.data_ptr(),
                  dev.stream_ptr(buf.device))
    return out if on_device else out.cpu().numpy()


frames_to_planar_bytes = _frames_to_planar_bytes
planar_bytes_to_frames = _planar_bytes_to_frames


def check_stream_bytes(n_bytes: int, h: int, w: int, n_planes: int, bit_depth: int) -> int:
    """Frames in a decoded stream of ``n_bytes``; raises like ``_planar_bytes_to_frames``."""
    frame_bytes = h * w * n_planes * (1 if bit_depth == 8 else 2)
    if frame_bytes == 0 or n_bytes % frame_bytes != 0:
        raise CorruptStreamError(f"decoded byte count {n_bytes} is not a whole number of "
                                 f"{h}x{w}x{n_planes} frames")
    return n_bytes // frame_bytes
