"""Full-size parity of the PCA configurations (BASELINE configs 3 and 5 at their
full T), against independent float64 references (VERDICT r1 "next" item 1).

* Gram / mean: a float64 torch restatement of transform.py:172-179 (shifted
  sums and ``X^T X`` accumulated over T-chunks with cuBLAS DGEMM) — not the
  repo's kernels. Mean within rel 1e-10, explained variance within rel 1e-9,
  components |cos| >= 1 - 1e-9 where the relative eigengap exceeds 1e-6
  (else the principal angles of the kept subspace <= 1e-6), SURVEY §8c.
* Frames on sampled T-slices: the oracle's pca_forward + quantize
  (transform.py:77-105, 191-199) fed the GPU's own model and ranges; <= 1 LSB
  on <= 2 % of samples (float32 projection vs the reference's float64).
* Recon on those slices: the oracle's dequantize + pca_inverse of the GPU
  frames; per-band PSNR within 0.01 dB and SSIM within 1e-5 of the oracle's.
* Metrics over the whole cube: per-band SSE and 11x11 SSIM sums recomputed in
  float64 torch from the GPU recon, PSNR within 0.01 dB, SSIM within 1e-5.
"""

import math

import numpy as np
import pytest
import torch

from oracle import cubevid_oracle as O
from oracle import metrics_oracle as M
from paper_2506_19656_b200 import pipeline as P
from paper_2506_19656_b200 import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _ref_cov(x: torch.Tensor, chunk: int):
    """float64 mean and covariance of the pixels of [T,H,W,C] (transform.py:172-179)."""
    T, H, W, C = x.shape
    shift = x[0, 0, 0].double()
    s = torch.zeros(C, dtype=torch.float64, device=x.device)
    q = torch.zeros((C, C), dtype=torch.float64, device=x.device)
    for t0 in range(0, T, chunk):
        v = x[t0:t0 + chunk].reshape(-1, C).double() - shift
        s += v.sum(dim=0)
        q += v.T @ v
    n = T * H * W
    m = s / n
    cov = q / n - torch.outer(m, m)
    return (shift + m).cpu().numpy(), cov.cpu().numpy()


def _check_model(model, mean, cov, k):
    ev, vec = np.linalg.eigh(cov)
    order = np.argsort(ev)[::-1]
    ev, vec = ev[order], vec[:, order]
    np.testing.assert_allclose(model.mean, mean, rtol=1e-10, atol=1e-12 * np.abs(mean).max())
    np.testing.assert_allclose(model.explained_variance, np.clip(ev[:k], 0, None), rtol=1e-9,
                               atol=1e-13 * ev[0])
    comps = np.asarray(model.components)
    for i in range(k):
        lo = abs(ev[i] - ev[i + 1]) if i + 1 < len(ev) else math.inf
        hi = abs(ev[i - 1] - ev[i]) if i > 0 else math.inf
        if min(lo, hi) / ev[0] > 1e-6:
            cos = abs(float(comps[i] @ vec[:, i]))
            assert cos >= 1 - 1e-9, (i, cos)
    # principal angles of the kept subspace
    if k < len(ev) and (ev[k - 1] - ev[k]) / ev[0] > 1e-9:
        sv = np.linalg.svd(comps @ vec[:, :k], compute_uv=False)
        assert np.arccos(np.clip(sv.min(), -1, 1)) <= 1e-6, sv


def _ssim_sse_fp64(x: torch.Tensor, rec: torch.Tensor, peaks: torch.Tensor, chunk: int):
    """Per-band SSE and SSIM sums over [T,H,W,C] in float64 (valid 11x11 Gaussian)."""
    T, H, W, C = x.shape
    g = torch.tensor(M.gaussian_taps(11, 1.5), dtype=torch.float64, device=x.device)
    c1 = ((0.01 * peaks) ** 2).view(1, C, 1, 1)
    c2 = ((0.03 * peaks) ** 2).view(1, C, 1, 1)

    def filt(a):
        w = a.shape[-1] - 10
        b = sum(g[k] * a[..., k:k + w] for k in range(11))
        h = b.shape[-2] - 10
        return sum(g[k] * b[..., k:k + h, :] for k in range(11))

    sse = torch.zeros(C, dtype=torch.float64, device=x.device)
    ss = torch.zeros(C, dtype=torch.float64, device=x.device)
    for t0 in range(0, T, chunk):
        o = x[t0:t0 + chunk].permute(0, 3, 1, 2).double()
        r = rec[t0:t0 + chunk].permute(0, 3, 1, 2).double()
        sse += ((o - r) ** 2).sum(dim=(0, 2, 3))
        mx, my = filt(o), filt(r)
        sxx = filt(o * o) - mx * mx
        syy = filt(r * r) - my * my
        sxy = filt(o * r) - mx * my
        num = (2 * mx * my + c1) * (2 * sxy + c2)
        den = (mx * mx + my * my + c1) * (sxx + syy + c2)
        m = torch.where(den == 0, torch.ones_like(den), num / den)
        ss += m.sum(dim=(0, 2, 3))
        del o, r, mx, my, sxx, syy, sxy, num, den, m
    return sse, ss


def _run(config: int, spec: P.StreamSpec, slices, gram_chunk: int, ssim_chunk: int):
    cuda = torch.device("cuda", 0)
    x = synth.make(config, device=cuda)
    T, H, W, C = x.shape
    enc, recon, sc = P.roundtrip(x, spec)
    enc.check()
    k = spec.n_pcs
    fold = enc.pca[0]
    model = fold.model

    # 1. Gram / mean / basis against float64 DGEMM over T-chunks
    mean, cov = _ref_cov(x, gram_chunk)
    if spec.normalize:
        lo = x.reshape(-1, C).amin(dim=0).double().cpu().numpy()
        hi = x.reshape(-1, C).amax(dim=0).double().cpu().numpy()
        sc_ = np.where(hi - lo == 0, 1.0, hi - lo)
        np.testing.assert_array_equal(fold.norm_offset, lo)
        mean, cov = (mean - lo) / sc_, cov / np.outer(sc_, sc_)
    _check_model(model, mean, cov, k)

    # 2. frames and recon on sampled T-slices against the oracle fed the GPU's model / ranges
    qmins = enc.qmins[0].cpu().numpy()
    qmaxs = enc.qmaxs[0].cpu().numpy()
    comps = np.asarray(model.components)
    for t in slices:
        xs = x[t:t + 1].cpu().numpy()
        z = xs.astype(np.float64)
        if spec.normalize:
            z = (z - fold.norm_offset) / fold.norm_scale
        pcs = O.pca_forward(z, model.mean, comps)
        q = O.quantize(pcs, qmins, qmaxs, spec.bit_depth, clamp=True)
        want = O.planar_frames(q)
        got = enc.frames[0][:, t:t + 1].cpu().numpy()
        d = np.abs(got.astype(np.int64) - want.astype(np.int64))
        assert d.max() <= 1 and (d > 0).mean() <= 0.02, (t, d.max(), (d > 0).mean())
        rec_o = O.dequantize(np.stack([got.reshape(-1, 1, 3, H * W)[j // 3, 0, j % 3] for j in range(k)],
                                      axis=-1).reshape(1, H, W, k), qmins, qmaxs, spec.bit_depth)
        rec_o = O.pca_inverse(rec_o, model.mean, comps)
        if spec.normalize:
            rec_o = rec_o * fold.norm_scale + fold.norm_offset
        rec_g = recon[t:t + 1].cpu().numpy()
        db_o = M.psnr_per_band(xs, rec_o)
        db_g = M.psnr_per_band(xs, rec_g)
        np.testing.assert_allclose(db_g, db_o, atol=0.01)
        np.testing.assert_allclose(M.ssim_per_band(xs, rec_g), M.ssim_per_band(xs, rec_o), atol=1e-5)

    # 3. whole-cube metrics recomputed in float64 from the GPU recon
    peaks = x.reshape(-1, C).amax(dim=0).double()
    np.testing.assert_array_equal(enc.peaks[0].cpu().numpy(), peaks.cpu().numpy())
    sse, ss = _ssim_sse_fp64(x, recon, peaks, ssim_chunk)
    rep = sc.report()[0]
    n = T * H * W
    db = (10 * torch.log10(peaks ** 2 / (sse / n))).cpu().numpy()
    np.testing.assert_allclose(rep["psnr_per_band"], db, atol=0.01)
    ssim = (ss / (T * (H - 10) * (W - 10))).cpu().numpy()
    np.testing.assert_allclose(rep["ssim_per_band"], ssim, atol=1e-5)
    return rep


def test_config3_full_size(cuda):
    rep = _run(3, P.StreamSpec(12, n_pcs=9), slices=(0, 31, 63), gram_chunk=16, ssim_chunk=4)
    assert rep["psnr"] > 40


def test_config5_full_size(cuda):
    rep = _run(5, P.StreamSpec(16, n_pcs=6, normalize=True), slices=(0, 371, 743), gram_chunk=24,
               ssim_chunk=2)
    # 12 independent fields per band: six components keep about half of the variance
    assert 20 < rep["psnr"] < 30
