"""Drop-in for the array part of ``cubevid.cube``: ``forward_fill_time`` and
``ValidityMask`` (/root/reference/pkg/src/cubevid/cube.py:30-49, 213-246).

The fill runs as two sm_100a passes over the ``[outer][T][inner]`` view of the
array (no transpose is needed for any time axis): K1 records, per time segment,
the last observed value of every cell; the fill pass then walks each segment
with the carry in registers.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dev
from . import _lib
from .errors import ConfigurationError

FILL_SEGMENT = 32  # time steps per CTA in the fill passes


@dataclass(frozen=True)
class ValidityMask:
    """``True`` where the value was observed, ``False`` where the fill synthesised it."""

    mask: object

    def __post_init__(self):
        m = self.mask
        if isinstance(m, torch.Tensor):
            object.__setattr__(self, "mask", m.bool())
        else:
            view = np.asarray(m, dtype=bool).view()
            view.flags.writeable = False
            object.__setattr__(self, "mask", view)

    @property
    def n_synthesized(self) -> int:
        m = self.mask
        return int((~m).sum().item()) if isinstance(m, torch.Tensor) else int((~m).sum())

    @property
    def all_observed(self) -> bool:
        m = self.mask
        return bool(m.all().item()) if isinstance(m, torch.Tensor) else bool(m.all())


def segment_carries(x: dev.Arr, outer: int, T: int, inner: int, seg_len: int,
                    err: dev.ErrWord, C: int = 1):
    """K1 in fill mode: per-segment last-observed map [outer][n_seg][inner] (+ band stats)."""
    lib = _lib.load()
    nseg = lib.cv_num_segments(T, seg_len)
    seg_last = torch.empty((outer, nseg, inner), dtype=torch.float32, device=x.device)
    from .transform import band_stats  # local import: transform imports nothing from here

    mins, maxs, nans = band_stats(x, outer, T, inner, C, fill_mode=1, seg_len=seg_len,
                                  err=err, seg_last=seg_last)
    return seg_last, (mins, maxs, nans)


def forward_fill_time(arr, time_axis: int, fill_value_for_leading=0.0):
    """Hold the last valid value along ``time_axis``; leading gaps take the fill value."""
    x = dev.to_device(arr)
    nd = len(x.shape)
    if not -nd <= time_axis < nd:
        raise ConfigurationError(f"time axis {time_axis} does not exist on a {nd}-D array")
    t = x.t
    if not t.dtype.is_floating_point:
        out = t.clone()
        mask = torch.ones(x.shape, dtype=torch.bool, device=t.device)
        return dev.to_host_like(out, x, x.np_dtype), ValidityMask(dev.to_host_like(mask, x))
    if t.dtype != torch.float32:
        raise ConfigurationError(f"forward_fill_time on the B200 path supports float32 cubes, got {t.dtype}")
    ax = time_axis % nd
    outer = int(np.prod(x.shape[:ax], dtype=np.int64))
    T = int(x.shape[ax])
    inner = int(np.prod(x.shape[ax + 1:], dtype=np.int64))
    out = torch.empty_like(t)
    mask = torch.empty(x.shape, dtype=torch.bool, device=t.device)
    if t.numel():
        err = dev.ErrWord(t.device)
        seg_last, _ = segment_carries(x, outer, T, inner, FILL_SEGMENT, err)
        _lib.call("cv_forward_fill", x.ptr, outer, T, inner, float(fill_value_for_leading),
                  FILL_SEGMENT, seg_last.data_ptr(), None, out.data_ptr(), mask.data_ptr(), err.ptr,
                  dev.stream_ptr(t.device))
        if err.flags() & _lib.CV_FLAG_NONFINITE:
            raise ConfigurationError("array contains +/-inf; only NaN marks missing data")
    return dev.to_host_like(out, x), ValidityMask(dev.to_host_like(mask, x))
