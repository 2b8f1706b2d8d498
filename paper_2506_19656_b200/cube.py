"""Drop-in for the array part of ``cubevid.cube``: ``forward_fill_time``,
``ValidityMask`` and ``select_for_video`` with the ``DataCube`` it reads
(/root/reference/pkg/src/cubevid/cube.py:30-49, 52-158, 213-305).

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


class DataCube:
    """Named 3-D/4-D variables over named axes (cube.py:52-158), numpy arrays or
    CUDA tensors. Only what ``select_for_video`` and the container read is kept:
    variables, their ordered axis names, coordinate vectors and attributes; the
    reference's own DataCube works wherever this one does (same accessors)."""

    def __init__(self, variables, axes, coords=None, attrs=None, global_attrs=None):
        self._vars, self._axes, lengths = {}, {}, {}
        for name, arr in variables.items():
            if not isinstance(arr, torch.Tensor):
                arr = np.asarray(arr)
                if not (np.issubdtype(arr.dtype, np.number) or arr.dtype == bool):
                    raise ConfigurationError(f"variable {name!r} has non-numeric dtype {arr.dtype}")
            if arr.ndim not in (3, 4):
                raise ConfigurationError(f"variable {name!r} must be 3-D or 4-D, got {arr.ndim}-D")
            if name not in axes:
                raise ConfigurationError(f"variable {name!r} has no axes entry")
            ax = tuple(axes[name])
            if len(ax) != arr.ndim:
                raise ConfigurationError(f"variable {name!r}: {arr.ndim} dims but {len(ax)} axis names")
            if len(set(ax)) != len(ax):
                raise ConfigurationError(f"variable {name!r} repeats an axis name: {ax}")
            for axis_name, n in zip(ax, arr.shape):
                if lengths.setdefault(axis_name, int(n)) != int(n):
                    raise ConfigurationError(f"axis {axis_name!r} has conflicting lengths "
                                             f"{lengths[axis_name]} and {int(n)}")
            self._vars[name] = arr
            self._axes[name] = ax
        self._coords = {}
        for axis_name, vec in (coords or {}).items():
            vec = np.asarray(vec)
            if vec.ndim != 1:
                raise ConfigurationError(f"coordinate {axis_name!r} must be 1-D")
            if axis_name in lengths and len(vec) != lengths[axis_name]:
                raise ConfigurationError(f"coordinate {axis_name!r} has length {len(vec)}, "
                                         f"axis has length {lengths[axis_name]}")
            self._coords[axis_name] = vec
        self._attrs = {k: dict(v) for k, v in (attrs or {}).items()}
        self._global_attrs = dict(global_attrs or {})
        self._lengths = lengths

    variables = property(lambda self: dict(self._vars))
    axes = property(lambda self: dict(self._axes))
    coords = property(lambda self: dict(self._coords))
    attrs = property(lambda self: {k: dict(v) for k, v in self._attrs.items()})
    global_attrs = property(lambda self: dict(self._global_attrs))

    def __contains__(self, name) -> bool:
        return name in self._vars

    def __getitem__(self, name):
        return self._vars[name]

    def axes_of(self, name: str) -> tuple:
        return self._axes[name]

    def attrs_of(self, name: str) -> dict:
        return dict(self._attrs.get(name, {}))

    def axis_length(self, axis_name: str) -> int:
        return self._lengths[axis_name]

    def variable_names(self) -> tuple:
        return tuple(self._vars)


def channel_axis_of(cube, name: str, axis_order) -> str:
    """Name of the channel axis of a 4-D variable (cube.py:308-313)."""
    extra = [a for a in cube.axes_of(name) if a not in tuple(axis_order)]
    if len(extra) != 1:
        raise ConfigurationError(f"variable {name!r} has no unique channel axis")
    return extra[0]


def _strides_for(shape, var_axes, roles) -> list:
    """Element strides of a contiguous array of ``shape`` along the named roles."""
    st, acc = {}, 1
    for a, n in zip(reversed(var_axes), reversed(shape)):
        st[a] = acc
        acc *= int(n)
    return [st[a] for a in roles]


def select_for_video(cube, names, axis_order):
    """Stack variables into one contiguous ``[t, y, x, c]`` array (cube.py:249-305).

    ``names``: 3-D variables sharing the three axes of ``axis_order`` (one
    channel each, list order) or one 4-D variable whose extra axis becomes the
    channel axis. The transposition and the stacking are one gather kernel
    (``cv_select_stack``); numpy comes back for host variables, a CUDA tensor
    when any variable lives on the device.
    """
    names = [names] if isinstance(names, str) else list(names)
    axis_order = tuple(axis_order)
    if len(axis_order) != 3:
        raise ConfigurationError(f"axis_order must name 3 axes, got {axis_order}")
    if len(set(names)) != len(names):
        raise ConfigurationError(f"duplicate variable names in selection: {names}")
    if not names:
        raise ConfigurationError("empty variable selection")
    for n in names:
        if n not in cube:
            raise ConfigurationError(f"variable {n!r} not found in cube")
    ndims = {cube[n].ndim for n in names}
    if ndims == {4}:
        if len(names) != 1:
            raise ConfigurationError("a stream may use several 3-D variables or one 4-D variable, "
                                     f"got {len(names)} 4-D variables")
        name = names[0]
        var_axes = tuple(cube.axes_of(name))
        extra = [a for a in var_axes if a not in axis_order]
        if len(extra) != 1 or not all(a in var_axes for a in axis_order):
            raise ConfigurationError(f"variable {name!r} with axes {var_axes} does not match "
                                     f"axis order {axis_order} plus one channel axis")
        x = dev.to_device(cube[name])
        tyx = _strides_for(x.shape, var_axes, axis_order)
        sc = _strides_for(x.shape, var_axes, extra)[0]
        C = int(x.shape[var_axes.index(extra[0])])
        dims = [int(x.shape[var_axes.index(a)]) for a in axis_order]
        chans = [(x.t, c * sc, tyx) for c in range(C)]
        host = x.host
        np_dtype = x.np_dtype if x.np_dtype is not None else None
    elif ndims != {3}:
        raise ConfigurationError("cannot mix 3-D and 4-D variables in one stream")
    else:
        arrs, dims, host = [], None, True
        for n in names:
            var_axes = tuple(cube.axes_of(n))
            if set(var_axes) != set(axis_order):
                raise ConfigurationError(f"variable {n!r} has axes {var_axes}, expected a permutation "
                                         f"of {axis_order}")
            x = dev.to_device(cube[n])
            shp = tuple(int(x.shape[var_axes.index(a)]) for a in axis_order)
            if dims is None:
                dims = list(shp)
            elif shp != tuple(dims):
                raise ConfigurationError(f"variable {n!r} has shape {shp}, expected {tuple(dims)}")
            arrs.append((x, _strides_for(x.shape, var_axes, axis_order)))
            host = host and x.host
        # np.stack's dtype promotion when the variables differ
        dts = {a.t.dtype for a, _ in arrs}
        if len(dts) > 1:
            common = torch.result_type(arrs[0][0].t, arrs[1][0].t)
            for a, _ in arrs[2:]:
                common = torch.promote_types(common, a.t.dtype)
            for a, _ in arrs:
                a.t = a.t.to(common)
            np_dtype = None
        else:
            np_dtype = arrs[0][0].np_dtype
        chans = [(a.t, 0, st) for a, st in arrs]
        C = len(chans)
    T, H, W = dims
    lib = _lib.load()
    if C > lib.cv_max_channels():
        raise ConfigurationError(f"{C} channels in one stream (the B200 path supports up to "
                                 f"{lib.cv_max_channels()})")
    t0 = chans[0][0]
    esz = t0.element_size()
    out = torch.empty((T, H, W, C), dtype=t0.dtype, device=t0.device)
    import ctypes

    ptrs = (ctypes.c_void_p * C)(*[t.data_ptr() + off * esz for t, off, _ in chans])
    strides = (ctypes.c_int64 * (3 * C))(*[s for _, _, st in chans for s in st])
    _lib.call("cv_select_stack", ctypes.cast(ptrs, ctypes.c_void_p), ctypes.cast(strides, ctypes.c_void_p),
              C, esz, T, H, W, out.data_ptr(), dev.stream_ptr(t0.device))
    if not host:
        return out
    res = out.cpu().numpy()
    if np_dtype is not None and res.dtype != np_dtype:
        res = res.view(np_dtype)
    return res
