"""CPU restatement (numpy, float64) of the reference's array path.

TEST INFRASTRUCTURE ONLY — imported by tests/, smoke() and the bench's CPU
baseline arm, never by the product package.

Every function restates the algorithm of the reference function named in its
docstring (paths relative to /root/reference/pkg/src/cubevid). numpy's
elementwise float64 arithmetic is IEEE round-to-nearest, so the integer
outputs are the reference's bit for bit; the PCA uses numpy's BLAS/LAPACK as
the reference does (unpinned third-party arithmetic: numpy 2.3 / OpenBLAS).
"""

from __future__ import annotations

import math

import numpy as np

LEVELS = {8: 255, 10: 1023, 12: 4095, 16: 65535}


class OracleError(ValueError):
    """Raised where the reference raises ConfigurationError."""


# --------------------------------------------------------------------------- cube.py

def forward_fill(arr: np.ndarray, time_axis: int, fill=0.0):
    """cube.py:213-246 — hold the last observed value along ``time_axis``.

    Returns (filled, observed_mask). Leading gaps take ``fill`` (cast to the
    array dtype, as numpy's weak-scalar promotion does in the reference).
    """
    a = np.asarray(arr)
    if not -a.ndim <= time_axis < a.ndim:
        raise OracleError("time axis does not exist")
    if not np.issubdtype(a.dtype, np.floating):
        return a.copy(), np.ones(a.shape, dtype=bool)
    if np.isinf(a).any():
        raise OracleError("array contains +/-inf")
    w = np.moveaxis(a, time_axis, 0)
    observed = ~np.isnan(w)
    steps = np.arange(w.shape[0]).reshape((-1,) + (1,) * (w.ndim - 1))
    last_seen = np.maximum.accumulate(np.where(observed, steps, -1), axis=0)
    held = np.take_along_axis(w, np.maximum(last_seen, 0), axis=0)
    held = np.where(last_seen >= 0, held, fill)
    held = np.where(observed, w, held)
    return (np.ascontiguousarray(np.moveaxis(held, 0, time_axis)),
            np.moveaxis(observed, 0, time_axis))


def select_for_video(variables: dict, axes: dict, names, axis_order) -> np.ndarray:
    """cube.py:249-305 — 3-D variables transposed to ``axis_order`` and stacked on a
    new last axis, or one 4-D variable transposed with its extra axis last."""
    names = [names] if isinstance(names, str) else list(names)
    order = tuple(axis_order)
    if len(order) != 3 or not names or len(set(names)) != len(names):
        raise OracleError("bad selection")
    if any(n not in variables for n in names):
        raise OracleError("unknown variable")
    nd = {np.ndim(variables[n]) for n in names}
    if nd == {4}:
        if len(names) != 1:
            raise OracleError("several 4-D variables")
        ax = tuple(axes[names[0]])
        rest = [a for a in ax if a not in order]
        if len(rest) != 1 or any(a not in ax for a in order):
            raise OracleError("axes do not match")
        perm = [ax.index(a) for a in order + (rest[0],)]
        return np.ascontiguousarray(np.transpose(variables[names[0]], perm))
    if nd != {3}:
        raise OracleError("mixed ranks")
    cols = []
    for n in names:
        ax = tuple(axes[n])
        if set(ax) != set(order):
            raise OracleError("axes do not match")
        cols.append(np.transpose(variables[n], [ax.index(a) for a in order]))
        if cols[-1].shape != cols[0].shape:
            raise OracleError("shape mismatch")
    return np.ascontiguousarray(np.stack(cols, axis=-1))


# --------------------------------------------------------------------------- transform.py

def fit_quant(arr: np.ndarray):
    """transform.py:61-70 — per-channel min/max over (t, y, x), as float64."""
    a = np.asarray(arr)
    if a.ndim != 4:
        raise OracleError("expected [t,y,x,c]")
    if np.issubdtype(a.dtype, np.floating) and not np.isfinite(a).all():
        raise OracleError("non-finite values")
    return (a.min(axis=(0, 1, 2)).astype(np.float64), a.max(axis=(0, 1, 2)).astype(np.float64))


def quantize(arr: np.ndarray, mins, maxs, bit_depth: int, clamp: bool = False) -> np.ndarray:
    """transform.py:77-105 — floor(((v - min)/span) * L + 0.5) in float64."""
    L = LEVELS[bit_depth]
    lo = np.asarray(mins, dtype=np.float64)
    hi = np.asarray(maxs, dtype=np.float64)
    v = np.asarray(arr).astype(np.float64, copy=False)
    if clamp:
        v = np.clip(v, lo, hi)
    elif np.any((v < lo) | (v > hi)):
        raise OracleError("values outside the quantization range")
    span = hi - lo
    flat = span == 0
    x = (v - lo) / np.where(flat, 1.0, span) * L
    q = np.floor(x + 0.5)
    q[..., flat] = 0
    return q.astype(np.uint8 if bit_depth == 8 else np.uint16)


def dequantize(q: np.ndarray, mins, maxs, bit_depth: int) -> np.ndarray:
    """transform.py:108-126 — min + q/L * (max - min), float64."""
    L = LEVELS[bit_depth]
    q = np.asarray(q)
    if q.size and (q.min() < 0 or q.max() > L):
        raise OracleError("integer values outside range")
    lo = np.asarray(mins, dtype=np.float64)
    hi = np.asarray(maxs, dtype=np.float64)
    out = lo + q.astype(np.float64) / L * (hi - lo)
    flat = (hi - lo) == 0
    if flat.any():
        out[..., flat] = lo[flat]
    return out


def pca_fit(arr: np.ndarray, n_keep: int):
    """transform.py:160-188 — covariance, eigh, descending order, sign rule.

    Returns (mean [c], components [k, c], explained_variance [k]).
    """
    a = np.asarray(arr)
    c = a.shape[-1]
    if not 1 <= n_keep <= c:
        raise OracleError("n_keep out of range")
    x = a.reshape(-1, c).astype(np.float64)
    if x.shape[0] < c:
        raise OracleError("too few samples")
    mu = x.mean(axis=0)
    xc = x - mu
    cov = xc.T @ xc / x.shape[0]
    w, v = np.linalg.eigh(cov)
    keep = np.argsort(w)[::-1][:n_keep]
    ev = np.clip(w[keep], 0.0, None)
    comps = v[:, keep].T
    pivot = np.abs(comps).argmax(axis=1)
    sgn = np.sign(comps[np.arange(n_keep), pivot])
    sgn[sgn == 0] = 1.0
    return mu, comps * sgn[:, None], ev


def pca_forward(arr, mean, comps) -> np.ndarray:
    """transform.py:191-199 — (v - mean) @ components.T in float64."""
    return (np.asarray(arr).astype(np.float64) - mean) @ np.asarray(comps).T


def pca_inverse(pc, mean, comps) -> np.ndarray:
    """transform.py:202-210 — pc @ components + mean in float64."""
    return np.asarray(pc).astype(np.float64) @ np.asarray(comps) + mean


# --------------------------------------------------------------------------- plan.py / bridge.py

def pack_groups(n: int):
    """plan.py:118-128 — ceil(n/3) slot triples, padding repeats the last real channel.

    Returns a list of (members, n_real).
    """
    if n < 1:
        raise OracleError("zero channels")
    groups = []
    for start in range(0, n, 3):
        real = list(range(start, min(start + 3, n)))
        groups.append((tuple(real + [real[-1]] * (3 - len(real))), len(real)))
    return groups


def planar_frames(q: np.ndarray, pad_zero: bool = False) -> np.ndarray:
    """plan.py:118-128 + bridge.py:157-160 — channel-last ints [t,y,x,e] to
    planar frames [g][t][3][y*x] (group members per pack_groups)."""
    t, h, w, e = q.shape
    out = []
    for members, n_real in pack_groups(e):
        planes = [q[..., m] for m in members]
        if pad_zero:
            planes = planes[:n_real] + [np.zeros_like(planes[0])] * (3 - n_real)
        out.append(np.stack(planes, axis=1).reshape(t, 3, h * w))
    return np.ascontiguousarray(np.stack(out, axis=0))


def planar_bytes(frames3: np.ndarray, bit_depth: int) -> bytes:
    """bridge.py:157-160 — [t,y,x,3] -> [t,3,y,x] little-endian bytes."""
    dt = "u1" if bit_depth == 8 else "<u2"
    return np.ascontiguousarray(np.moveaxis(frames3, -1, 1)).astype(dt, copy=False).tobytes()


def frames_from_planar_bytes(raw: bytes, h: int, w: int, n_planes: int, bit_depth: int):
    """bridge.py:163-174 — bytes -> [t,y,x,planes]."""
    dt = np.dtype("u1" if bit_depth == 8 else "<u2")
    fb = h * w * n_planes * dt.itemsize
    if fb == 0 or len(raw) % fb:
        raise OracleError("not a whole number of frames")
    a = np.frombuffer(raw, dtype=dt).reshape(len(raw) // fb, n_planes, h, w)
    return np.ascontiguousarray(np.moveaxis(a, 1, -1))


# --------------------------------------------------------------------------- composition

def encode_stream(cube: np.ndarray, bit_depth: int, n_pcs: int = 0, fill=0.0,
                  normalize: bool = False, pad_zero: bool = False):
    """fill -> [pca] -> fit_quant -> quantize -> planar frames.

    Returns a dict with the frames [g][t][3][h*w], mins/maxs, the PCA pieces
    and the filled cube.
    """
    filled, mask = forward_fill(cube, 0, fill)
    enc = {"filled": filled, "mask": mask}
    data = filled
    if n_pcs:
        z = filled.astype(np.float64)
        if normalize:
            lo = z.min(axis=(0, 1, 2))
            sc = z.max(axis=(0, 1, 2)) - lo
            sc = np.where(sc == 0, 1.0, sc)
            z = (z - lo) / sc
            enc["norm"] = (lo, sc)
        mean, comps, ev = pca_fit(z, n_pcs)
        enc["pca"] = (mean, comps, ev)
        data = pca_forward(z, mean, comps)
    mins, maxs = fit_quant(data)
    q = quantize(data, mins, maxs, bit_depth)
    enc.update(mins=mins, maxs=maxs, q=q, frames=planar_frames(q, pad_zero), encoded=data)
    return enc


def decode_stream(frames: np.ndarray, enc: dict, shape, bit_depth: int) -> np.ndarray:
    """frames -> drop padded planes -> dequantize -> [pca_inverse]."""
    t, h, w, c = shape
    e = len(enc["mins"])
    g = len(pack_groups(e))
    # frames [g][t][3][h*w] -> planes [g*3 + j][t][h*w]; real channel k sits at plane k
    planes = np.asarray(frames).reshape(g, t, 3, h * w).transpose(0, 2, 1, 3).reshape(3 * g, t, h * w)
    q = np.stack([planes[k] for k in range(e)], axis=-1).reshape(t, h, w, e)
    v = dequantize(q, enc["mins"], enc["maxs"], bit_depth)
    if "pca" in enc:
        mean, comps, _ = enc["pca"]
        v = pca_inverse(v, mean, comps)
        if "norm" in enc:
            lo, sc = enc["norm"]
            v = v * sc + lo
    return v


def decoded_frames_with_noise(frames: np.ndarray, bit_depth: int, amplitude_steps: int = 1):
    """Stand-in for a lossy codec: q' = clip(q + delta(i), 0, L) with
    delta(i) in {-1,0,1}*ceil(L/1023) from an integer hash of the linear index."""
    L = LEVELS[bit_depth]
    step = max(1, math.ceil(L / 1023)) * amplitude_steps
    i = np.arange(frames.size, dtype=np.uint64)
    h = (i * np.uint64(0x9E3779B97F4A7C15)) >> np.uint64(61)
    delta = (h.astype(np.int64) % 3) - 1
    out = np.clip(frames.reshape(-1).astype(np.int64) + delta * step, 0, L)
    return out.astype(frames.dtype).reshape(frames.shape)
