"""Float64 restatement of the metrics module the reference specifies but does not
ship. TEST INFRASTRUCTURE ONLY.

Pinned by SPEC's known answers and by the brute-force loop
implementations below (agreement to 1e-9 relative).

SSIM parameters: Gaussian window of ``win`` taps, sigma 1.5 (BASELINE config 2:
11x11), K1 = 0.01, K2 = 0.03, dynamic range = per-band peak (max of the
original), population (co)variances, valid region only (no padding), mean
over frames and channels.
"""

from __future__ import annotations

import math

import numpy as np
from scipy.ndimage import correlate1d


def gaussian_taps(win: int = 11, sigma: float = 1.5) -> np.ndarray:
    r = win // 2
    k = np.arange(-r, r + 1, dtype=np.float64)
    g = np.exp(-(k * k) / (2.0 * sigma * sigma))
    return g / g.sum()


def bpppb(total_bytes: int, t: int, h: int, w: int, c: int) -> float:
    """SPEC.md:412-418."""
    if min(t, h, w, c) < 1:
        raise ValueError("zero dims")
    return 8.0 * total_bytes / (t * h * w * c)


def psnr_per_band(orig: np.ndarray, recon: np.ndarray):
    """per band 10 log10(peak^2 / MSE), peak = max of the original."""
    o = np.asarray(orig, dtype=np.float64)
    r = np.asarray(recon, dtype=np.float64)
    mse = ((o - r) ** 2).mean(axis=(0, 1, 2))
    peak = o.max(axis=(0, 1, 2))
    out = np.empty_like(mse)
    for i in range(len(mse)):
        if peak[i] == 0:
            out[i] = np.nan
        elif mse[i] == 0:
            out[i] = np.inf
        else:
            out[i] = 10.0 * math.log10(peak[i] ** 2 / mse[i])
    return out


def psnr(orig, recon):
    """(per-band dB, mean over finite bands)."""
    db = psnr_per_band(orig, recon)
    fin = db[np.isfinite(db)]
    return db, (float(fin.mean()) if fin.size else (math.inf if np.isinf(db).any() else math.nan))


def _ssim_map(o, r, peak, win, sigma):
    g = gaussian_taps(win, sigma)
    rad = win // 2

    def filt(a):
        a = correlate1d(a, g, axis=1, mode="nearest")
        a = correlate1d(a, g, axis=2, mode="nearest")
        return a[:, rad:a.shape[1] - rad, rad:a.shape[2] - rad]

    mx, my = filt(o), filt(r)
    sxx = filt(o * o) - mx * mx
    syy = filt(r * r) - my * my
    sxy = filt(o * r) - mx * my
    c1 = (0.01 * peak) ** 2
    c2 = (0.03 * peak) ** 2
    num = (2 * mx * my + c1) * (2 * sxy + c2)
    den = (mx * mx + my * my + c1) * (sxx + syy + c2)
    with np.errstate(invalid="ignore", divide="ignore"):
        m = num / den
    return np.where(den == 0, 1.0, m)


def ssim_per_band(orig, recon, win: int = 11, sigma: float = 1.5) -> np.ndarray:
    """mean SSIM per band over frames and the valid region."""
    o = np.asarray(orig, dtype=np.float64)
    r = np.asarray(recon, dtype=np.float64)
    t, h, w, c = o.shape
    if h < win or w < win:
        raise ValueError("spatial dims smaller than window")
    peaks = o.max(axis=(0, 1, 2))
    out = np.empty(c)
    for b in range(c):
        out[b] = _ssim_map(o[..., b], r[..., b], peaks[b], win, sigma).mean()
    return out


def ssim(orig, recon, win: int = 11, sigma: float = 1.5) -> float:
    return float(ssim_per_band(orig, recon, win, sigma).mean())


def spectral_angle(orig, recon):
    """mean over pixels of arccos(<o,r>/(|o||r|)) in degrees;
    zero-norm pixels skipped. Returns (mean_degrees, skipped)."""
    o = np.asarray(orig, dtype=np.float64).reshape(-1, np.shape(orig)[-1])
    r = np.asarray(recon, dtype=np.float64).reshape(-1, np.shape(recon)[-1])
    no = np.sqrt((o * o).sum(axis=1))
    nr = np.sqrt((r * r).sum(axis=1))
    ok = (no > 0) & (nr > 0)
    cs = np.clip((o[ok] * r[ok]).sum(axis=1) / (no[ok] * nr[ok]), -1.0, 1.0)
    ang = np.degrees(np.arccos(cs))
    return (float(ang.mean()) if ang.size else math.nan), int((~ok).sum())


def spectral_angle_brute(orig, recon):
    o = np.asarray(orig, dtype=np.float64)
    r = np.asarray(recon, dtype=np.float64)
    c = o.shape[-1]
    o2, r2 = o.reshape(-1, c), r.reshape(-1, c)
    tot, n, skip = 0.0, 0, 0
    for i in range(o2.shape[0]):
        dot = sum(o2[i, k] * r2[i, k] for k in range(c))
        no = math.sqrt(sum(o2[i, k] ** 2 for k in range(c)))
        nr = math.sqrt(sum(r2[i, k] ** 2 for k in range(c)))
        if no == 0 or nr == 0:
            skip += 1
            continue
        tot += math.degrees(math.acos(max(-1.0, min(1.0, dot / (no * nr)))))
        n += 1
    return (tot / n if n else math.nan), skip


# --------------------------------------------------------------------------- brute force

def psnr_brute(orig, recon):
    o = np.asarray(orig, dtype=np.float64)
    r = np.asarray(recon, dtype=np.float64)
    t, h, w, c = o.shape
    res = []
    for b in range(c):
        se, peak, n = 0.0, -math.inf, 0
        for i in range(t):
            for y in range(h):
                for x in range(w):
                    d = o[i, y, x, b] - r[i, y, x, b]
                    se += d * d
                    peak = max(peak, o[i, y, x, b])
                    n += 1
        res.append(math.inf if se == 0 else 10 * math.log10(peak * peak / (se / n)))
    return np.array(res)


def ssim_brute(orig, recon, win: int = 11, sigma: float = 1.5):
    o = np.asarray(orig, dtype=np.float64)
    r = np.asarray(recon, dtype=np.float64)
    t, h, w, c = o.shape
    g = gaussian_taps(win, sigma)
    wts = np.outer(g, g)
    rad = win // 2
    res = []
    for b in range(c):
        peak = o[..., b].max()
        c1, c2 = (0.01 * peak) ** 2, (0.03 * peak) ** 2
        acc, n = 0.0, 0
        for i in range(t):
            for y in range(rad, h - rad):
                for x in range(rad, w - rad):
                    po = o[i, y - rad:y + rad + 1, x - rad:x + rad + 1, b]
                    pr = r[i, y - rad:y + rad + 1, x - rad:x + rad + 1, b]
                    mx, my = (wts * po).sum(), (wts * pr).sum()
                    vx = (wts * po * po).sum() - mx * mx
                    vy = (wts * pr * pr).sum() - my * my
                    cxy = (wts * po * pr).sum() - mx * my
                    den = (mx * mx + my * my + c1) * (vx + vy + c2)
                    acc += 1.0 if den == 0 else (2 * mx * my + c1) * (2 * cxy + c2) / den
                    n += 1
        res.append(acc / n)
    return np.array(res)
