"""Drop-in for ``cubevid.transform`` (/root/reference/pkg/src/cubevid/transform.py)
on the B200: same names, argument meaning, return types and errors; the
arithmetic runs in libcvb200 (K1 stats, K4 quantiser, K5 dequantiser, K2/K3 PCA).

Inputs may be numpy arrays (results come back as numpy, like the reference)
or CUDA tensors (results stay on the device).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dev
from . import _lib
from .errors import ConfigurationError

SUPPORTED_BIT_DEPTHS = (8, 10, 12, 16)

_STATS_SEG = 64  # time segment of the stats pass when no forward fill is involved


@dataclass(frozen=True)
class QuantParams:
    """Per-channel [min, max] ranges and the target bit depth (transform.py:25-58)."""

    bit_depth: int
    mins: tuple
    maxs: tuple

    def __post_init__(self):
        if self.bit_depth not in SUPPORTED_BIT_DEPTHS:
            raise ConfigurationError(f"bit depth {self.bit_depth} not in {SUPPORTED_BIT_DEPTHS}")
        if len(self.mins) != len(self.maxs):
            raise ConfigurationError("mins and maxs must have equal length")
        for lo, hi in zip(self.mins, self.maxs):
            if not (np.isfinite(lo) and np.isfinite(hi)):
                raise ConfigurationError("quantization range must be finite")
            if lo > hi:
                raise ConfigurationError(f"channel min {lo} exceeds max {hi}")

    @property
    def levels(self) -> int:
        return (1 << self.bit_depth) - 1

    @property
    def n_channels(self) -> int:
        return len(self.mins)

    def is_constant(self, channel: int) -> bool:
        return self.mins[channel] == self.maxs[channel]

    def step(self, channel: int) -> float:
        return (self.maxs[channel] - self.mins[channel]) / self.levels


@dataclass(frozen=True)
class PcaModel:
    """Orthonormal channel transform, descending explained variance (transform.py:129-157)."""

    mean: np.ndarray
    components: np.ndarray
    explained_variance: np.ndarray
    n_input_channels: int
    per_component_quality: tuple | None = None

    def __post_init__(self):
        for name in ("mean", "components", "explained_variance"):
            object.__setattr__(self, name, np.asarray(getattr(self, name), dtype=np.float64))
        k, c = self.components.shape
        if c != self.n_input_channels or self.mean.shape != (c,):
            raise ConfigurationError("inconsistent PCA model shapes")
        if not np.allclose(self.components @ self.components.T, np.eye(k), atol=1e-10):
            raise ConfigurationError("PCA component rows are not orthonormal")
        ev = self.explained_variance
        if len(ev) != k or (np.diff(ev) > 1e-12 * max(ev[0], 1.0)).any():
            raise ConfigurationError("explained variance must be non-increasing")

    @property
    def n_kept(self) -> int:
        return self.components.shape[0]


# ----------------------------------------------------------------------------- helpers

def _raise_flags(flags: int, *, nonfinite_msg: str | None = None, range_msg: str | None = None,
                 int_msg: str | None = None) -> None:
    if flags & (_lib.CV_FLAG_NONFINITE | _lib.CV_FLAG_NAN) and nonfinite_msg:
        raise ConfigurationError(nonfinite_msg)
    if flags & _lib.CV_FLAG_RANGE and range_msg:
        raise ConfigurationError(range_msg)
    if flags & _lib.CV_FLAG_INT_RANGE and int_msg:
        raise ConfigurationError(int_msg)


def band_stats(x: dev.Arr, n_cubes: int, T: int, inner: int, C: int, *, fill_mode: int = 0,
               seg_len: int = _STATS_SEG, fill_value: float = 0.0, err: dev.ErrWord | None = None,
               seg_last: torch.Tensor | None = None):
    """K1 over ``[n_cubes][T][inner]``: returns device (mins, maxs, nan_counts) [n_cubes, C]."""
    d = x.device
    lib = _lib.load()
    ws = dev.workspace(lib.cv_stats_ws_bytes(n_cubes, C), d)
    s = dev.stream_ptr(d)
    _lib.call("cv_stats_reset", ws.data_ptr(), n_cubes, C, s)
    _lib.call("cv_stats", x.ptr, x.code, n_cubes, T, inner, C, fill_mode, seg_len, ws.data_ptr(),
              seg_last.data_ptr() if seg_last is not None else None,
              err.ptr if err is not None else None, s)
    mins = torch.empty((n_cubes, C), dtype=torch.float64, device=d)
    maxs = torch.empty_like(mins)
    nans = torch.empty((n_cubes, C), dtype=torch.int64, device=d)
    _lib.call("cv_stats_finalize", ws.data_ptr(), n_cubes, C, fill_mode, float(fill_value),
              mins.data_ptr(), maxs.data_ptr(), nans.data_ptr(), s)
    return mins, maxs, nans


def _params_device(params: QuantParams, device):
    return (dev.f64_tensor(params.mins, device), dev.f64_tensor(params.maxs, device))


# ----------------------------------------------------------------------------- quantisation

def fit_quant(arr, bit_depth: int) -> QuantParams:
    """Per-channel min/max over all (t, y, x) of a [t,y,x,c] array (transform.py:61-70)."""
    x = dev.to_device(arr)
    dev.require_4d(x.shape)
    if x.code is None:
        raise ConfigurationError(f"unsupported dtype {x.np_dtype} for the B200 path")
    T, H, W, C = x.shape
    if x.t.numel() == 0:
        raise ValueError("zero-size array to reduction operation minimum which has no identity")
    err = dev.ErrWord(x.device)
    mins, maxs, _ = band_stats(x, 1, T, H * W * C, C, fill_mode=0, err=err)
    _raise_flags(err.flags(), nonfinite_msg="cannot fit quantization on non-finite values")
    return QuantParams(bit_depth, tuple(mins[0].tolist()), tuple(maxs[0].tolist()))


def quantize(arr, params: QuantParams, clamp: bool = False):
    """q = round_half_away((v - min)/(max - min) * (2^B - 1)), bit-exact (transform.py:77-105)."""
    x = dev.to_device(arr)
    if len(x.shape) != 4 or x.shape[-1] != params.n_channels:
        raise ConfigurationError(f"array shape {x.shape} does not match {params.n_channels} channels")
    if x.code is None:
        raise ConfigurationError(f"unsupported dtype {x.np_dtype} for the B200 path")
    T, H, W, C = x.shape
    tdt, npdt = dev.out_dtype_for_depth(params.bit_depth)
    out = torch.empty((T, H, W, C), dtype=tdt, device=x.device)
    if out.numel():
        mins, maxs = _params_device(params, x.device)
        err = dev.ErrWord(x.device)
        _lib.call("cv_quantize", x.ptr, x.code, 1, T, H * W, C, mins.data_ptr(), maxs.data_ptr(),
                  params.bit_depth, int(bool(clamp)), 0, 0.0, _STATS_SEG, None, None, None, None, 0,
                  _lib.CV_LAYOUT_CHANNEL_LAST, _lib.CV_PAD_REPEAT, out.data_ptr(), None, err.ptr,
                  dev.stream_ptr(x.device))
        flags = err.flags()
        if flags & _lib.CV_FLAG_NAN:
            raise ConfigurationError("cannot quantize NaN values (forward-fill them first)")
        _raise_flags(flags, range_msg="values outside the quantization range (pass clamp=True to clip)")
    return dev.to_host_like(out, x, npdt)


def _as_unsigned_frames(q: dev.Arr, levels: int, bit_depth: int) -> dev.Arr:
    """Integer inputs other than u8/u16: check the range on the device, narrow to u16."""
    t = q.t
    if t.dtype.is_floating_point or t.dtype == torch.bool:
        raise ConfigurationError(f"dequantize expects integer frames, got {t.dtype}")
    if t.numel():
        lo, hi = int(t.min().item()), int(t.max().item())
        if lo < 0 or hi > levels:
            raise ConfigurationError(f"integer values outside [0, {levels}] for bit depth {bit_depth}")
    return dev.Arr(t.to(torch.uint16), _lib.CV_U16, q.host, np.dtype(np.uint16), q.shape)


def dequantize(q, params: QuantParams):
    """v = min + q/(2^B-1)*(max-min) in float64, bit-exact (transform.py:108-126)."""
    x = dev.to_device(q)
    if len(x.shape) != 4 or x.shape[-1] != params.n_channels:
        raise ConfigurationError(f"array shape {x.shape} does not match {params.n_channels} channels")
    if x.code not in (_lib.CV_U8, _lib.CV_U16):
        x = _as_unsigned_frames(x, params.levels, params.bit_depth)
    T, H, W, C = x.shape
    out = torch.empty((T, H, W, C), dtype=torch.float64, device=x.device)
    if out.numel():
        mins, maxs = _params_device(params, x.device)
        err = dev.ErrWord(x.device)
        _lib.call("cv_dequantize", x.ptr, x.code, 1, T, H * W, C, _lib.CV_LAYOUT_CHANNEL_LAST,
                  mins.data_ptr(), maxs.data_ptr(), params.bit_depth, out.data_ptr(), _lib.CV_F64,
                  err.ptr, dev.stream_ptr(x.device))
        _raise_flags(err.flags(), int_msg=(f"integer values outside [0, {params.levels}] for bit depth "
                                           f"{params.bit_depth}"))
    return dev.to_host_like(out, x)


# ----------------------------------------------------------------------------- PCA

def gram(x: dev.Arr, n_pix: int, C: int, stats: bool = False, err: dev.ErrWord | None = None):
    """K2: float64 (shift, sums, shifted Gram[, mins, maxs]) of [n_pix][C] spectra.

    Launch only: every result stays on the device (no host synchronisation).
    """
    d = x.device
    lib = _lib.load()
    s = dev.stream_ptr(d)
    ws = dev.workspace(lib.cv_gram_ws_bytes(n_pix, C), d)
    out = torch.empty(C + C * C, dtype=torch.float64, device=d)
    if err is None:
        err = dev.ErrWord(d)
    sws = None
    if stats:
        sws = dev.workspace(lib.cv_stats_ws_bytes(1, C), d)
        _lib.call("cv_stats_reset", sws.data_ptr(), 1, C, s)
    _lib.call("cv_pca_gram", x.ptr, x.code, n_pix, C, ws.data_ptr(), out.data_ptr(),
              sws.data_ptr() if sws is not None else None, err.ptr, s)
    res = {"out": out, "err": err, "shift": x.t.reshape(-1)[:C]}
    if stats:
        mins = torch.empty((1, C), dtype=torch.float64, device=d)
        maxs = torch.empty_like(mins)
        _lib.call("cv_stats_finalize", sws.data_ptr(), 1, C, 0, 0.0, mins.data_ptr(),
                  maxs.data_ptr(), None, s)
        res["mins"], res["maxs"] = mins[0], maxs[0]
    return res


def covariance_from_gram(shift: np.ndarray, out: np.ndarray, n: int, C: int):
    """mean and population covariance from the shifted one-pass sums."""
    sums = out[:C]
    G = out[C:].reshape(C, C)
    delta = sums / n
    mean = shift + delta
    cov = G / n - np.outer(delta, delta)
    cov = 0.5 * (cov + cov.T)
    return mean, cov


def eig_model(mean: np.ndarray, cov: np.ndarray, n_keep: int, C: int):
    """Host eigh + ordering + sign convention of transform.py:180-187."""
    eigvals, eigvecs = np.linalg.eigh(cov)
    order = np.argsort(eigvals)[::-1][:n_keep]
    variance = np.clip(eigvals[order], 0.0, None)
    comps = eigvecs[:, order].T
    lead = np.abs(comps).argmax(axis=1)
    signs = np.sign(comps[np.arange(n_keep), lead])
    signs[signs == 0] = 1.0
    comps = comps * signs[:, None]
    return PcaModel(mean, comps, variance, n_input_channels=C)


def pca_fit(arr, n_keep: int) -> PcaModel:
    """PCA over all pixel spectra of a [t,y,x,c] array (transform.py:160-188)."""
    x = dev.to_device(arr)
    dev.require_4d(x.shape)
    C = x.shape[-1]
    if not 1 <= n_keep <= C:
        raise ConfigurationError(f"n_keep={n_keep} outside [1, {C}]")
    n = int(np.prod(x.shape[:3]))
    if n < C:
        raise ConfigurationError(f"need at least {C} pixel samples to fit {C} channels")
    if x.code is None:
        raise ConfigurationError(f"unsupported dtype {x.np_dtype} for the B200 path")
    g = gram(x, n, C)
    flags = g["err"].flags()
    out = g["out"].cpu().numpy()
    shift = g["shift"].double().cpu().numpy()
    if flags & (_lib.CV_FLAG_NAN | _lib.CV_FLAG_NONFINITE):
        raise ConfigurationError("cannot fit a PCA on non-finite values")
    mean, cov = covariance_from_gram(shift, out, n, C)
    return eig_model(mean, cov, n_keep, C)


def pca_forward(arr, model: PcaModel):
    """(v - mean) @ components.T in float64 (transform.py:191-199)."""
    x = dev.to_device(arr)
    if len(x.shape) != 4 or x.shape[-1] != model.n_input_channels:
        raise ConfigurationError(
            f"array has {x.shape[-1] if len(x.shape) == 4 else '?'} channels, "
            f"model expects {model.n_input_channels}")
    if x.code is None:
        raise ConfigurationError(f"unsupported dtype {x.np_dtype} for the B200 path")
    T, H, W, C = x.shape
    k = model.n_kept
    out = torch.empty((T, H, W, k), dtype=torch.float64, device=x.device)
    if out.numel():
        mean = np.ascontiguousarray(model.mean, dtype=np.float64)
        comps = np.ascontiguousarray(model.components, dtype=np.float64)
        err = dev.ErrWord(x.device)
        _lib.call("cv_pca_project", x.ptr, x.code, 1, T * H * W, C, mean.ctypes.data,
                  comps.ctypes.data, k, out.data_ptr(), _lib.CV_F64, None, err.ptr,
                  dev.stream_ptr(x.device))
    return dev.to_host_like(out, x)


def pca_inverse(pc, model: PcaModel):
    """pc @ components + mean in float64 (transform.py:202-210)."""
    x = dev.to_device(pc)
    if len(x.shape) != 4 or x.shape[-1] != model.n_kept:
        raise ConfigurationError(
            f"array has {x.shape[-1] if len(x.shape) == 4 else '?'} components, "
            f"model keeps {model.n_kept}")
    if x.code not in (_lib.CV_F32, _lib.CV_F64):
        x = dev.Arr(x.t.double(), _lib.CV_F64, x.host, np.dtype(np.float64), x.shape)
    T, H, W, k = x.shape
    C = model.n_input_channels
    out = torch.empty((T, H, W, C), dtype=torch.float64, device=x.device)
    if out.numel():
        mean = np.ascontiguousarray(model.mean, dtype=np.float64)
        comps = np.ascontiguousarray(model.components, dtype=np.float64)
        _lib.call("cv_pca_inverse", x.ptr, x.code, 1, T * H * W, k, mean.ctypes.data,
                  comps.ctypes.data, C, out.data_ptr(), _lib.CV_F64, dev.stream_ptr(x.device))
    return dev.to_host_like(out, x)
