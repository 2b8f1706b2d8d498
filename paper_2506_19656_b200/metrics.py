"""Fidelity metrics of the paper as specified by the
(absent) reference metrics module, SPEC.md:400-477 — computed by the fused
K6 kernel (``cv_eval``) in float64 accumulation.

Conventions (BASELINE config 2 for the SSIM window):
  bpppb  = 8 * total_bytes / (t*h*w*c)
  PSNR_c = 10 log10(peak_c^2 / MSE_c), peak_c = max over (t, y, x) of the
           original channel; aggregate = mean of the finite per-band values;
           zero-peak channels are undefined and left out (with a warning).
  SSIM   = mean over frames and channels of the 11x11 Gaussian (sigma 1.5)
           SSIM map on the valid region (no padding), K1=0.01, K2=0.03,
           dynamic range = peak_c, population (co)variances.
"""

from __future__ import annotations

import math
import warnings

import numpy as np
import torch

from . import _device as dev
from . import _lib
from .errors import ConfigurationError

SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_K1 = 0.01
SSIM_K2 = 0.03


def bpppb(total_bytes: int, t: int, h: int, w: int, c: int) -> float:
    """Bits per pixel per band."""
    if min(t, h, w, c) < 1:
        raise ConfigurationError("bpppb needs all dimensions >= 1")
    return 8.0 * total_bytes / (t * h * w * c)


def psnr_from_sse(sse: np.ndarray, peaks: np.ndarray, n_per_band: int):
    """Per-band dB and the aggregate (mean of finite, defined bands)."""
    sse = np.asarray(sse, dtype=np.float64)
    peaks = np.asarray(peaks, dtype=np.float64)
    mse = sse / n_per_band
    db = np.empty_like(mse)
    for i, (m, p) in enumerate(zip(mse, peaks)):
        if p == 0.0:
            db[i] = np.nan
        elif m == 0.0:
            db[i] = np.inf
        else:
            db[i] = 10.0 * math.log10(p * p / m)
    if np.isnan(db).any():
        warnings.warn("PSNR undefined for channels with zero peak; excluded from the mean",
                      RuntimeWarning, stacklevel=3)
    finite = db[np.isfinite(db)]
    if finite.size:
        agg = float(finite.mean())
    elif np.isinf(db).any():
        agg = float("inf")
    else:
        agg = float("nan")
    return db, agg


def _prep_pair(orig, recon):
    o = dev.to_device(orig)
    r = dev.to_device(recon)
    if o.shape != r.shape:
        raise ConfigurationError(f"shape mismatch {o.shape} vs {r.shape}")
    dev.require_4d(o.shape)
    if o.code not in (_lib.CV_F32, _lib.CV_F64, _lib.CV_U16):
        o = dev.Arr(o.t.float(), _lib.CV_F32, o.host, np.dtype(np.float32), o.shape)
    if r.code not in (_lib.CV_F32, _lib.CV_F64):
        r = dev.Arr(r.t.double(), _lib.CV_F64, r.host, np.dtype(np.float64), r.shape)
    return o, r


def score(orig, recon, want_ssim: bool = True):
    """One fused pass: per-band SSE and (optionally) SSIM sums + peaks.

    Returns a dict with numpy per-band arrays: ``sse``, ``ssim_sum``, ``peaks``
    and the counts ``n_per_band`` / ``n_ssim_per_band``.
    """
    o, r = _prep_pair(orig, recon)
    T, H, W, C = o.shape
    if want_ssim and (H < SSIM_WINDOW or W < SSIM_WINDOW):
        raise ConfigurationError(f"spatial dims {H}x{W} smaller than the {SSIM_WINDOW}-px SSIM window")
    d = o.device
    from .transform import band_stats

    err = dev.ErrWord(d)
    _, maxs, _ = band_stats(o, 1, T, H * W * C, C, fill_mode=0, err=err)
    sse = torch.zeros(C, dtype=torch.float64, device=d)
    ssum = torch.zeros(C, dtype=torch.float64, device=d)
    lib = _lib.load()
    ws = dev.workspace(lib.cv_eval_ws_bytes(1, T, H, W, C, int(want_ssim)), d)
    _lib.call("cv_eval", None, 0, C, None, None, 8, None, None, r.ptr, r.code, o.ptr, o.code,
              1, T, H, W, C, maxs.data_ptr(), int(want_ssim), None, ws.data_ptr(),
              sse.data_ptr(), ssum.data_ptr(), err.ptr, dev.stream_ptr(d))
    if err.flags() & (_lib.CV_FLAG_NAN | _lib.CV_FLAG_NONFINITE):
        raise ConfigurationError("metrics need finite originals")
    return {
        "sse": sse.cpu().numpy(),
        "ssim_sum": ssum.cpu().numpy(),
        "peaks": maxs[0].cpu().numpy(),
        "n_per_band": T * H * W,
        "n_ssim_per_band": T * (H - SSIM_WINDOW + 1) * (W - SSIM_WINDOW + 1),
    }


def psnr(orig, recon):
    """(per-channel dB vector, aggregate dB) with peak_c = max of the original channel."""
    s = score(orig, recon, want_ssim=False)
    return psnr_from_sse(s["sse"], s["peaks"], s["n_per_band"])


def ssim_per_band(orig, recon) -> np.ndarray:
    s = score(orig, recon, want_ssim=True)
    return s["ssim_sum"] / s["n_ssim_per_band"]


def ssim(orig, recon) -> float:
    """Mean SSIM over frames and channels (11x11 Gaussian, sigma 1.5, valid region)."""
    return float(np.mean(ssim_per_band(orig, recon)))


def spectral_angle(orig, recon) -> tuple:
    """Mean spectral angle in degrees over pixels and the
    number of zero-norm pixels skipped: per pixel arccos(<o,r>/(|o||r|))."""
    o, r = _prep_pair(orig, recon)
    T, H, W, C = o.shape
    d = o.device
    n = T * H * W
    out = torch.zeros(3, dtype=torch.float64, device=d)
    if n:
        lib = _lib.load()
        ws = dev.workspace(lib.cv_angle_ws_bytes(), d)
        _lib.call("cv_spectral_angle", o.ptr, o.code, r.ptr, r.code, n, C, ws.data_ptr(),
                  out.data_ptr(), dev.stream_ptr(d))
    s, cnt, skipped = out.cpu().tolist()
    mean = s / cnt if cnt else float("nan")
    if skipped:
        warnings.warn(f"spectral angle: {int(skipped)} zero-norm pixels skipped", RuntimeWarning,
                      stacklevel=2)
    return mean, int(skipped)


def evaluate(orig, recon, total_bytes: int | None = None, want_ssim: bool = True) -> dict:
    """psnr + ssim (+ bpppb) of one reconstruction, one fused device pass."""
    s = score(orig, recon, want_ssim=want_ssim)
    db, agg = psnr_from_sse(s["sse"], s["peaks"], s["n_per_band"])
    rep = {"psnr_per_band": db, "psnr": agg}
    if want_ssim:
        per = s["ssim_sum"] / s["n_ssim_per_band"]
        rep["ssim_per_band"] = per
        rep["ssim"] = float(per.mean())
    rep["sa_degrees"], rep["sa_skipped"] = spectral_angle(orig, recon)
    if total_bytes is not None:
        t, h, w, c = np.asarray(orig).shape if not isinstance(orig, torch.Tensor) else orig.shape
        rep["bpppb"] = bpppb(total_bytes, t, h, w, c)
    return rep
