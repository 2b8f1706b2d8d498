"""Pin the restated metrics oracle: SPEC.md known answers and brute-force loops
(SPEC.md:416-436, 455-458, 542, 548)."""

import math

import numpy as np
import pytest

from oracle import metrics_oracle as M


def test_bpppb_known_answers():
    assert M.bpppb(1000, 10, 10, 10, 1) == 8.0
    assert M.bpppb(2 * 10 * 10 * 10 * 3, 10, 10, 10, 3) == 16.0
    assert M.bpppb(4 * 2 * 3 * 4 * 5, 2, 3, 4, 5) == 32.0
    with pytest.raises(ValueError):
        M.bpppb(1, 0, 1, 1, 1)


def test_psnr_known_answer():
    o = np.array([0, 1, 2, 3], dtype=np.float64).reshape(1, 1, 4, 1)
    r = np.array([0, 1, 2, 2], dtype=np.float64).reshape(1, 1, 4, 1)
    db, agg = M.psnr(o, r)
    assert abs(db[0] - 10 * math.log10(36)) < 1e-12
    assert abs(agg - 15.563025007672874) < 1e-9
    db, agg = M.psnr(o, o)
    assert math.isinf(db[0]) and math.isinf(agg)


def test_psnr_excludes_infinite_band():
    rng = np.random.default_rng(1)
    o = rng.random((2, 4, 4, 2))
    r = o.copy()
    r[..., 1] += 0.01
    db, agg = M.psnr(o, r)
    assert math.isinf(db[0]) and np.isfinite(db[1]) and agg == db[1]


def test_psnr_scale_invariant():
    rng = np.random.default_rng(2)
    o = rng.random((3, 5, 5, 3)) + 0.1
    r = o + 0.01 * rng.normal(size=o.shape)
    np.testing.assert_allclose(M.psnr_per_band(o, r), M.psnr_per_band(7.5 * o, 7.5 * r), rtol=1e-12)


@pytest.mark.parametrize("seed", range(100))
def test_psnr_vs_brute(seed):
    rng = np.random.default_rng(seed)
    o = rng.random((4, 8, 8, 3))
    r = o + 0.05 * rng.normal(size=o.shape)
    np.testing.assert_allclose(M.psnr_per_band(o, r), M.psnr_brute(o, r), rtol=1e-9)


@pytest.mark.parametrize("seed", range(20))
@pytest.mark.parametrize("win", [7, 11])
def test_ssim_vs_brute(seed, win):
    rng = np.random.default_rng(100 + seed)
    o = rng.random((2, 13, 14, 3))
    r = o + 0.1 * rng.normal(size=o.shape)
    np.testing.assert_allclose(M.ssim_per_band(o, r, win), M.ssim_brute(o, r, win), rtol=1e-9)


def test_ssim_identities():
    rng = np.random.default_rng(3)
    o = rng.random((2, 16, 16, 2)) + 0.5
    assert abs(M.ssim(o, o) - 1.0) < 1e-12
    const = np.full((1, 12, 12, 1), 0.7)
    assert abs(M.ssim(const, const) - 1.0) < 1e-12
    # inverted zero-mean pattern (8x8 checkerboard tiled) -> negative structure term
    yy, xx = np.mgrid[0:16, 0:16]
    pat = (((yy // 2) + (xx // 2)) % 2 * 2 - 1).astype(np.float64)
    o = (1.0 + 0.5 * pat)[None, :, :, None]
    r = (1.0 - 0.5 * pat)[None, :, :, None]
    assert M.ssim(o, r) < 0
    with pytest.raises(ValueError):
        M.ssim(np.zeros((1, 8, 8, 1)), np.zeros((1, 8, 8, 1)))


def test_gaussian_taps():
    g = M.gaussian_taps(11, 1.5)
    assert g.shape == (11,) and abs(g.sum() - 1) < 1e-15
    np.testing.assert_allclose(g[5:], [0.26601172486179436, 0.2130055377112537, 0.10936068950970002,
                                      0.03600077212843083, 0.007598758135239185, 0.00102838008447911],
                               rtol=1e-12)


def test_spectral_angle_known_answers():
    o = np.array([1.0, 0.0]).reshape(1, 1, 1, 2)
    assert abs(M.spectral_angle(o, np.array([0.0, 1.0]).reshape(1, 1, 1, 2))[0] - 90.0) < 1e-12
    assert abs(M.spectral_angle(np.array([1.0, 1.0]).reshape(1, 1, 1, 2), o)[0] - 45.0) < 1e-12
    rng = np.random.default_rng(4)
    x = rng.random((2, 3, 4, 5)) + 0.1
    assert M.spectral_angle(x, x)[0] < 1e-5
    # invariant under per-pixel positive scaling
    s = rng.random((2, 3, 4, 1)) + 0.5
    np.testing.assert_allclose(M.spectral_angle(x, x * 1.1 + 0.01)[0],
                               M.spectral_angle(x * s, (x * 1.1 + 0.01) * s)[0], rtol=1e-9)
    z = x.copy()
    z[0, 0, 0] = 0
    assert M.spectral_angle(z, x)[1] == 1


@pytest.mark.parametrize("seed", range(20))
def test_spectral_angle_vs_brute(seed):
    rng = np.random.default_rng(200 + seed)
    o = rng.random((4, 8, 8, 3))
    r = o + 0.05 * rng.normal(size=o.shape)
    a, s = M.spectral_angle(o, r)
    b, t = M.spectral_angle_brute(o, r)
    assert s == t and abs(a - b) <= 1e-9 * abs(b)
