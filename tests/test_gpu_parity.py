"""GPU parity: every sm_100a entry point against the reference's golden vectors
and the CPU oracle. Integer outputs bit-exact; floats within the stated
tolerances (PSNR 0.01 dB, SSIM 1e-5 per band, PCA basis up to 1e-9 in |cos|)."""

import numpy as np
import pytest
import torch

from oracle import cubevid_oracle as O
from oracle import metrics_oracle as M
from paper_2506_19656_b200 import ConfigurationError
from paper_2506_19656_b200 import cube as G_cube
from paper_2506_19656_b200 import metrics as G_metrics
from paper_2506_19656_b200 import pipeline as G_pipe
from paper_2506_19656_b200 import transform as G

pytestmark = pytest.mark.gpu

PSNR_TOL_DB = 0.01
SSIM_TOL = 1e-5


# ------------------------------------------------------------------ forward fill

@pytest.mark.parametrize("name,fv", [("t0_f0", 0.0), ("t0_f01", 0.1), ("t0_fm3", -3.5)])
def test_forward_fill_golden(cuda, golden, name, fv):
    f, m = G_cube.forward_fill_time(golden["fill_in"], 0, fv)
    np.testing.assert_array_equal(f.view(np.uint32), golden[f"fill_{name}_out"].view(np.uint32))
    np.testing.assert_array_equal(m.mask, golden[f"fill_{name}_mask"])


def test_forward_fill_axes_ints_errors(cuda, golden, golden_errors):
    f, m = G_cube.forward_fill_time(golden["fill_ax2_in"], 2, 0.0)
    np.testing.assert_array_equal(f, golden["fill_ax2_out"])
    np.testing.assert_array_equal(m.mask, golden["fill_ax2_mask"])
    f, m = G_cube.forward_fill_time(golden["fill_ax2_in"], -2, 0.25)
    np.testing.assert_array_equal(f, golden["fill_axm2_out"])
    f, m = G_cube.forward_fill_time(golden["fill_int_in"], 0)
    np.testing.assert_array_equal(f, golden["fill_int_out"])
    assert m.all_observed
    bad = golden["fill_in"].copy()
    bad[1, 1, 1, 1] = np.inf
    with pytest.raises(ConfigurationError) as e:
        G_cube.forward_fill_time(bad, 0)
    assert str(e.value) == golden_errors["fill_inf"]
    with pytest.raises(ConfigurationError) as e:
        G_cube.forward_fill_time(golden["fill_in"], 4)
    assert str(e.value) == golden_errors["fill_axis"]


@pytest.mark.parametrize("shape,axis", [((70, 9, 11, 3), 0), ((5, 300, 7), 1), ((1, 4, 4, 2), 0),
                                        ((200, 3), 0)])
def test_forward_fill_long_runs_vs_oracle(cuda, shape, axis):
    rng = np.random.default_rng(7)
    x = rng.random(shape).astype(np.float32)
    x[rng.random(shape) < 0.6] = np.nan   # long gaps: exercises the segment carries
    f, m = G_cube.forward_fill_time(x, axis, 0.5)
    fo, mo = O.forward_fill(x, axis, 0.5)
    np.testing.assert_array_equal(f, fo)
    np.testing.assert_array_equal(m.mask, mo)
    assert m.n_synthesized == int((~mo).sum())


def test_forward_fill_device_tensor(cuda):
    x = torch.rand((40, 8, 8, 2), device=cuda)
    x[5:30] = float("nan")
    f, m = G_cube.forward_fill_time(x, 0)
    assert f.is_cuda
    fo, _ = O.forward_fill(x.cpu().numpy(), 0)
    np.testing.assert_array_equal(f.cpu().numpy(), fo)


# ------------------------------------------------------------------ quantisation

@pytest.mark.parametrize("B", [8, 10, 12, 16])
def test_fit_quant_quantize_dequantize_golden(cuda, golden, B):
    x = golden["q_in"]
    p = G.fit_quant(x, B)
    np.testing.assert_array_equal(np.array(p.mins), golden[f"q{B}_mins"])
    np.testing.assert_array_equal(np.array(p.maxs), golden[f"q{B}_maxs"])
    q = G.quantize(x, p)
    assert q.dtype == golden[f"q{B}_out"].dtype
    np.testing.assert_array_equal(q, golden[f"q{B}_out"])
    dq = G.dequantize(q, p)
    assert dq.dtype == np.float64
    np.testing.assert_array_equal(dq.view(np.uint64), golden[f"dq{B}_out"].view(np.uint64))


@pytest.mark.parametrize("B", [8, 10, 12, 16])
def test_quantize_ties_constant(cuda, golden, B):
    x = golden["ties_in"]
    p = G.fit_quant(x, B)
    np.testing.assert_array_equal(G.quantize(x, p), golden[f"ties{B}_out"])


def test_quantize_clamp_u16_f64_errors(cuda, golden, golden_errors):
    pc = G.QuantParams(12, (0.2, 0.0, 0.0), (0.8, 1.0, 1.0))
    np.testing.assert_array_equal(G.quantize(golden["q_in"], pc, clamp=True), golden["clamp12_out"])
    with pytest.raises(ConfigurationError) as e:
        G.quantize(golden["q_in"], pc)
    assert str(e.value) == golden_errors["quantize_range"]
    with pytest.raises(ConfigurationError) as e:
        G.fit_quant(golden["fill_in"], 8)
    assert str(e.value) == golden_errors["fit_nonfinite"]
    p = G.fit_quant(golden["u16_in"], 8)
    np.testing.assert_array_equal(np.array(p.mins), golden["u16_mins"])
    np.testing.assert_array_equal(G.quantize(golden["u16_in"], p), golden["u16_q8"])
    p = G.fit_quant(golden["f64_in"], 16)
    np.testing.assert_array_equal(np.array(p.maxs), golden["f64_maxs"])
    np.testing.assert_array_equal(G.quantize(golden["f64_in"], p), golden["f64_q16"])
    with pytest.raises(ConfigurationError) as e:
        G.dequantize(np.full((1, 1, 1, 3), 300, np.uint16), G.QuantParams(8, (0,) * 3, (1,) * 3))
    assert str(e.value) == golden_errors["dequant_range"]


@pytest.mark.parametrize("B", [8, 10, 12, 16])
def test_quantize_random_vs_oracle(cuda, B):
    """10^6 samples per depth (SPEC acceptance test 2 uses 10^6 at B=12/16)."""
    rng = np.random.default_rng(B)
    x = (rng.random((10, 100, 100, 10)) * rng.choice([1.0, 1e-3, 1e4], 10) +
         rng.normal(size=10) * 100).astype(np.float32)
    lo, hi = O.fit_quant(x)
    q = G.quantize(x, G.QuantParams(B, tuple(lo), tuple(hi)))
    np.testing.assert_array_equal(q, O.quantize(x, lo, hi, B))
    dq = G.dequantize(q, G.QuantParams(B, tuple(lo), tuple(hi)))
    np.testing.assert_array_equal(dq, O.dequantize(q, lo, hi, B))
    step = (hi - lo) / O.LEVELS[B]
    # exact-math bound step/2 plus the float64 rounding of the operands
    slack = 8 * np.spacing(np.maximum(np.abs(x), np.maximum(np.abs(lo), np.abs(hi))).astype(np.float64))
    assert (np.abs(dq - x) <= step / 2 + slack).all()


def test_quantize_exhaustive_8bit(cuda):
    """Every 8-bit level and every half-way point between levels (ties)."""
    L = 255
    v = np.arange(0, 2 * L + 1, dtype=np.float64) / (2 * L)
    x = np.stack([v, v * 3 - 1, v * 1e-6 + 2], axis=-1).reshape(1, 1, -1, 3)
    lo, hi = O.fit_quant(x)
    np.testing.assert_array_equal(G.quantize(x, G.QuantParams(8, tuple(lo), tuple(hi))),
                                  O.quantize(x, lo, hi, 8))


def test_quantize_nan_and_empty(cuda):
    x = np.zeros((2, 3, 3, 2), np.float32)
    x[0, 0, 0, 0] = np.nan
    with pytest.raises(ConfigurationError):
        G.quantize(x, G.QuantParams(8, (0.0, 0.0), (1.0, 1.0)))
    e = G.quantize(np.zeros((0, 3, 3, 2), np.float32), G.QuantParams(8, (0.0, 0.0), (1.0, 1.0)))
    assert e.shape == (0, 3, 3, 2) and e.dtype == np.uint8
    with pytest.raises(ValueError):
        G.fit_quant(np.zeros((0, 3, 3, 2), np.float32), 8)
    with pytest.raises(ConfigurationError):
        G.fit_quant(np.zeros((3, 3, 2), np.float32), 8)


# ------------------------------------------------------------------ PCA

def _cos_match(a, b, tol):
    cos = np.abs((a * b).sum(axis=1)) / (np.linalg.norm(a, axis=1) * np.linalg.norm(b, axis=1))
    assert (cos >= 1 - tol).all(), cos


def test_pca_golden(cuda, golden, golden_errors):
    x = golden["pca_in"]
    m = G.pca_fit(x, 3)
    np.testing.assert_allclose(m.mean, golden["pca_mean"], rtol=1e-12)
    _cos_match(m.components, golden["pca_comps"], 1e-9)
    np.testing.assert_allclose(m.components, golden["pca_comps"], atol=1e-8)  # same sign rule
    np.testing.assert_allclose(m.explained_variance, golden["pca_ev"], rtol=1e-9)
    pcs = G.pca_forward(x, m)
    np.testing.assert_allclose(pcs, golden["pca_fwd"], atol=1e-7)
    np.testing.assert_allclose(G.pca_inverse(pcs, m), golden["pca_inv"], atol=1e-7)
    full = G.pca_fit(x, 5)
    back = G.pca_inverse(G.pca_forward(x, full), full)
    np.testing.assert_allclose(back, x, atol=1e-6 * (x.max() - x.min()))
    np.testing.assert_allclose(full.explained_variance.sum(),
                               x.reshape(-1, 5).astype(np.float64).var(axis=0).sum(), rtol=1e-8)
    with pytest.raises(ConfigurationError) as e:
        G.pca_fit(x, 6)
    assert str(e.value) == golden_errors["pca_nkeep"]


def test_pca_rank1_and_mean_only(cuda):
    rng = np.random.default_rng(3)
    r = rng.normal(size=(3, 4, 5, 1))
    m = G.pca_fit(np.concatenate([r, 2 * r], axis=-1), 1)
    frac = m.explained_variance[0] / np.var(np.concatenate([r, 2 * r], -1).reshape(-1, 2), axis=0).sum()
    assert abs(frac - 1.0) < 1e-9
    const = np.ones((2, 3, 3, 4)) * np.array([1.0, 2.0, 3.0, 4.0])
    const[0, 0, 0] += 1e-3
    mc = G.pca_fit(const, 2)
    pcs = G.pca_forward(np.ones((1, 2, 2, 4)) * mc.mean, mc)
    assert np.abs(pcs).max() < 1e-12


@pytest.mark.parametrize("K", [6, 9, 4])
@pytest.mark.parametrize("shape", [(2, 9, 13, 12), (3, 40, 72, 12)])
def test_pca_forward_c12_vs_oracle(cuda, variant_sel, K, shape):
    """pca_forward on 12-band float32 cubes (k_pca_project12 for K in {6, 9}, the generic
    kernel for K = 4): float64 components against the oracle (transform.py:191-199), and
    bit for bit against the generic kernel; odd pixel counts exercise the two-pixel tail."""
    rng = np.random.default_rng(12 + K)
    x = (rng.standard_normal(shape) * 10.0 ** (np.arange(12) / 4) + 2.0).astype(np.float32)
    m = G.pca_fit(x, K)
    pcs = G.pca_forward(x, m)
    want = O.pca_forward(x, np.asarray(m.mean), np.asarray(m.components))
    np.testing.assert_allclose(pcs, want, rtol=0, atol=1e-9 * np.abs(want).max())
    variant_sel({"proj12": 0})
    np.testing.assert_array_equal(G.pca_forward(x, m), pcs)


# ------------------------------------------------------------------ metrics

@pytest.mark.parametrize("seed", range(5))
def test_metrics_vs_oracle(cuda, seed):
    rng = np.random.default_rng(seed)
    o = rng.random((3, 20, 24, 3)) + 0.1
    r = o + 0.02 * rng.normal(size=o.shape)
    db, agg = G_metrics.psnr(o, r)
    dbo, aggo = M.psnr(o, r)
    np.testing.assert_allclose(db, dbo, rtol=1e-12)
    np.testing.assert_allclose(G_metrics.ssim_per_band(o.astype(np.float32), r),
                               M.ssim_per_band(o.astype(np.float32), r), atol=SSIM_TOL)
    assert abs(G_metrics.ssim(o, o) - 1.0) < 1e-6


def test_metrics_known_answers(cuda):
    o = np.array([0, 1, 2, 3], dtype=np.float64).reshape(1, 1, 4, 1)
    r = np.array([0, 1, 2, 2], dtype=np.float64).reshape(1, 1, 4, 1)
    db, agg = G_metrics.psnr(o, r)
    assert abs(agg - 15.563025007672874) < 1e-9
    with pytest.raises(ConfigurationError):
        G_metrics.ssim(np.zeros((1, 8, 8, 1)), np.zeros((1, 8, 8, 1)))
    yy, xx = np.mgrid[0:16, 0:16]
    pat = (((yy // 2) + (xx // 2)) % 2 * 2 - 1).astype(np.float64)
    assert G_metrics.ssim((1.0 + 0.5 * pat)[None, :, :, None], (1.0 - 0.5 * pat)[None, :, :, None]) < 0


# ------------------------------------------------------------------ fused stream

@pytest.mark.parametrize("seg_len", [16, 3, 1])
def test_stream_golden(cuda, golden, seg_len):
    x = golden["stream_in"]
    spec = G_pipe.StreamSpec(10, seg_len=seg_len)
    enc, recon, sc = G_pipe.roundtrip(torch.from_numpy(x).to(cuda), spec)
    enc.check()
    np.testing.assert_array_equal(enc.qmins[0].cpu().numpy(), golden["stream_mins"])
    np.testing.assert_array_equal(enc.qmaxs[0].cpu().numpy(), golden["stream_maxs"])
    np.testing.assert_array_equal(enc.frames[0].cpu().numpy(), golden["stream_frames"])
    np.testing.assert_array_equal(recon.cpu().numpy(), golden["stream_recon"].astype(np.float32))
    rep = sc.report()[0]
    dbo, aggo = M.psnr(golden["stream_filled"], golden["stream_recon"])
    np.testing.assert_allclose(rep["psnr_per_band"], dbo, rtol=1e-9)
    so = M.ssim_per_band(golden["stream_filled"], golden["stream_recon"])
    np.testing.assert_allclose(rep["ssim_per_band"], so, atol=SSIM_TOL)
    assert int(enc.nan_counts.sum()) == int(np.isnan(x).sum())


def test_stream_zero_pad_and_noisy_frames(cuda, golden):
    x = golden["stream_in"]
    spec = G_pipe.StreamSpec(10, pad_mode="zero")
    enc = G_pipe.encode_prep(torch.from_numpy(x).to(cuda), spec)
    ref = O.encode_stream(x, 10, pad_zero=True)
    np.testing.assert_array_equal(enc.frames[0].cpu().numpy(), ref["frames"])
    noisy = O.decoded_frames_with_noise(ref["frames"], 10)
    recon, sc = G_pipe.decode_eval(enc, torch.from_numpy(x).to(cuda),
                                   frames=torch.from_numpy(noisy[None]).to(cuda))
    rec_o = O.decode_stream(noisy, ref, x.shape, 10)
    np.testing.assert_array_equal(recon.cpu().numpy(), rec_o.astype(np.float32))
    rep = sc.report()[0]
    np.testing.assert_allclose(rep["psnr_per_band"], M.psnr_per_band(ref["filled"], rec_o), rtol=1e-9)
    np.testing.assert_allclose(rep["ssim_per_band"], M.ssim_per_band(ref["filled"], rec_o), atol=SSIM_TOL)


@pytest.mark.parametrize("shape,C_pcs,B", [((6, 13, 17, 1), 0, 8), ((4, 12, 12, 32), 0, 12),
                                           ((3, 15, 19, 5), 0, 16), ((2, 21, 11, 12), 9, 12),
                                           ((5, 11, 30, 4), 2, 16),
                                           # W % 4 == 0: PCA inverse inside the vertical-first SSIM kernel
                                           ((2, 20, 132, 12), 9, 12), ((1, 16, 248, 5), 4, 16),
                                           ((1, 13, 128, 12), 12, 16)])
def test_stream_edge_shapes(cuda, shape, C_pcs, B):
    rng = np.random.default_rng(11)
    x = (rng.random(shape) * 3 - 1).astype(np.float32)
    if C_pcs == 0:
        x[rng.random(shape) < 0.1] = np.nan
    enc, recon, sc = G_pipe.roundtrip(torch.from_numpy(x).to(cuda), G_pipe.StreamSpec(B, n_pcs=C_pcs))
    enc.check()
    ref = O.encode_stream(x, B, n_pcs=C_pcs)
    if C_pcs == 0:
        np.testing.assert_array_equal(enc.frames[0].cpu().numpy(), ref["frames"])
        rec_o = O.decode_stream(ref["frames"], ref, x.shape, B)
        np.testing.assert_array_equal(recon.cpu().numpy(), rec_o.astype(np.float32))
    else:
        got = enc.frames[0].cpu().numpy().astype(np.int64)
        diff = np.abs(got - ref["frames"].astype(np.int64))
        assert diff.max() <= 1 and (diff > 0).mean() <= 0.02
        rec_o = O.decode_stream(ref["frames"], ref, x.shape, B)
    rep = sc.report()[0]
    np.testing.assert_allclose(rep["psnr_per_band"], M.psnr_per_band(ref["filled"], rec_o),
                               atol=PSNR_TOL_DB)
    np.testing.assert_allclose(rep["ssim_per_band"], M.ssim_per_band(ref["filled"], rec_o), atol=SSIM_TOL)


@pytest.mark.parametrize("normalize,bits,n_pcs", [(False, 12, 4), (True, 16, 4), (False, 10, 7)])
def test_stream_nan_then_pca(cuda, normalize, bits, n_pcs):
    """a cloudy cube is forward-filled before pca_fit / pca_forward
    (config-1 generator: 20 % NaN frames + 2 % NaN pixels, leading gaps)."""
    from paper_2506_19656_b200 import synth

    x = synth.minicube(19656, (20, 24, 36, 7)).numpy()
    assert np.isnan(x).any()
    enc, recon, sc = G_pipe.roundtrip(torch.from_numpy(x).to(cuda),
                                      G_pipe.StreamSpec(bits, n_pcs=n_pcs, normalize=normalize))
    enc.check()
    ref = O.encode_stream(x, bits, n_pcs=n_pcs, normalize=normalize)
    # the filled cube the PCA saw is forward_fill_time's output, bit for bit
    np.testing.assert_array_equal(enc.filled.cpu().numpy().view(np.uint32),
                                  ref["filled"].view(np.uint32))
    assert int(enc.nan_counts.sum()) == int(np.isnan(x).sum())
    mean_o, comps_o, ev_o = ref["pca"]
    m = enc.pca[0].model
    cos = np.abs(np.sum(m.components * comps_o, axis=1))
    assert (cos >= 1 - 1e-9).all(), cos
    got = enc.frames[0].cpu().numpy().astype(np.int64)
    diff = np.abs(got - ref["frames"].astype(np.int64))
    assert diff.max() <= 1 and (diff > 0).mean() <= 0.02
    rec_o = O.decode_stream(ref["frames"], ref, x.shape, bits)
    rep = sc.report()[0]
    np.testing.assert_allclose(rep["psnr_per_band"], M.psnr_per_band(ref["filled"], rec_o),
                               atol=PSNR_TOL_DB)
    np.testing.assert_allclose(rep["ssim_per_band"], M.ssim_per_band(ref["filled"], rec_o), atol=SSIM_TOL)


def test_pca_inf_raises(cuda):
    x = np.random.default_rng(4).random((3, 12, 12, 5)).astype(np.float32)
    x[1, 2, 3, 4] = np.inf
    with pytest.raises(ConfigurationError, match="inf"):
        G_pipe.encode_prep(torch.from_numpy(x).to(cuda), G_pipe.StreamSpec(12, n_pcs=3))


def test_all_nan_and_constant_bands(cuda):
    x = np.random.default_rng(1).random((8, 12, 12, 3)).astype(np.float32)
    x[..., 1] = np.nan          # never observed -> fill constant everywhere -> constant band
    x[..., 2] = 0.25            # constant
    x[:2, ..., 0] = np.nan      # leading gap -> fill enters the range
    enc, recon, sc = G_pipe.roundtrip(torch.from_numpy(x).to(cuda), G_pipe.StreamSpec(8, fill_value=0.5))
    ref = O.encode_stream(x, 8, fill=0.5)
    np.testing.assert_array_equal(enc.qmins[0].cpu().numpy(), ref["mins"])
    np.testing.assert_array_equal(enc.frames[0].cpu().numpy(), ref["frames"])
    rep = sc.report()[0]
    assert np.isinf(rep["psnr_per_band"][1]) and np.isinf(rep["psnr_per_band"][2])


def test_batch_matches_single(cuda):
    from paper_2506_19656_b200 import synth

    cubes = synth.minicube_batch(3, 100, (12, 16, 20, 7), device=cuda)
    spec = G_pipe.StreamSpec(10, seg_len=4)
    encb, reconb, scb = G_pipe.roundtrip(cubes, spec)
    for b in range(3):
        enc1, recon1, sc1 = G_pipe.roundtrip(cubes[b].contiguous(), spec)
        assert torch.equal(encb.frames[b], enc1.frames[0])
        assert torch.equal(reconb[b], recon1)
        np.testing.assert_array_equal(scb.report()[b]["psnr_per_band"], sc1.report()[0]["psnr_per_band"])


@pytest.mark.parametrize("seed", range(3))
def test_spectral_angle_vs_oracle(cuda, seed):
    rng = np.random.default_rng(seed)
    o = (rng.random((3, 10, 12, 5)) + 0.1).astype(np.float32)
    r = o + 0.02 * rng.normal(size=o.shape)
    o[0, 0, 0] = 0  # a zero-norm pixel, skipped
    with pytest.warns(RuntimeWarning):
        got, skipped = G_metrics.spectral_angle(o, r)
    want, wskip = M.spectral_angle(o, r)
    assert skipped == wskip == 1
    assert abs(got - want) <= 1e-9 * want
    assert G_metrics.spectral_angle(o[1:], o[1:])[0] < 1e-5


@pytest.mark.parametrize("shape,B", [((3, 11, 12, 2), 8), ((2, 37, 260, 3), 10), ((2, 20, 244, 5), 16),
                                     ((1, 130, 128, 7), 12), ((2, 16, 124, 1), 8), ((1, 12, 468, 4), 10),
                                     # 16-byte aligned rows: bulk-copy input path
                                     ((2, 24, 248, 3), 10), ((1, 16, 376, 5), 16), ((2, 40, 128, 8), 8),
                                     ((1, 13, 256, 7), 10), ((2, 11, 16, 2), 12)])
def test_ssim_column_groups(cuda, shape, B):
    """The vertical-first SSIM kernel (W % 4 == 0): CTAs of 118 output columns
    overlapping by 10 input columns, odd row counts, 8-bit (u8 frames) to
    16-bit, with and without the dequantisation table, per-lane and bulk-copy
    input paths; SSE and recon writes counted once per element."""
    rng = np.random.default_rng(sum(shape) + B)
    x = (rng.random(shape) * 2 + 0.5).astype(np.float32)
    x[rng.random(shape) < 0.05] = np.nan
    enc, recon, sc = G_pipe.roundtrip(torch.from_numpy(x).to(cuda), G_pipe.StreamSpec(B))
    enc.check()
    ref = O.encode_stream(x, B)
    rec_o = O.decode_stream(ref["frames"], ref, x.shape, B)
    np.testing.assert_array_equal(recon.cpu().numpy(), rec_o.astype(np.float32))
    rep = sc.report()[0]
    np.testing.assert_allclose(rep["psnr_per_band"], M.psnr_per_band(ref["filled"], rec_o), rtol=1e-9)
    np.testing.assert_allclose(rep["ssim_per_band"], M.ssim_per_band(ref["filled"], rec_o), atol=SSIM_TOL)


@pytest.mark.parametrize("shape,B,u16", [((5, 16, 20, 7), 12, False), ((3, 40, 36, 4), 16, False),
                                         ((4, 24, 28, 4), 8, True), ((2, 13, 12, 7), 10, True)])
def test_psnr_stream_kernel(cuda, shape, B, u16):
    """PSNR-only decode (streaming kernel for C in {4, 7}, H*W % 4 == 0): recon
    bit-exact and per-band PSNR against the oracle, f32 and u16 originals,
    table and computed dequantisation."""
    rng = np.random.default_rng(sum(shape) + B)
    if u16:
        x = rng.integers(0, 10001, size=shape).astype(np.uint16)
    else:
        x = (rng.random(shape) * 2 + 0.5).astype(np.float32)
        x[rng.random(shape) < 0.05] = np.nan
    enc, recon, sc = G_pipe.roundtrip(torch.from_numpy(x).to(cuda), G_pipe.StreamSpec(B), want_ssim=False)
    enc.check()
    ref = O.encode_stream(x, B)
    rec_o = O.decode_stream(ref["frames"], ref, x.shape, B)
    np.testing.assert_array_equal(recon.cpu().numpy(), rec_o.astype(np.float32))
    rep = sc.report()[0]
    np.testing.assert_allclose(rep["psnr_per_band"], M.psnr_per_band(ref["filled"], rec_o), rtol=1e-9)


# ------------------------------------------------------------------ Gram kernels

@pytest.mark.parametrize("C", [1, 5, 7, 12])
@pytest.mark.parametrize("n_pix", [1, 63, 64 * 5 + 3, 100_003])
@pytest.mark.parametrize("variant", [{}, {"gram12": 0}, {"gram12": 0, "gram_checks": 1}, {"gram12": 0, "gram_nt": 256},
                                     {"gram_tiles": 1}])
def test_gram_kernels_ragged(cuda, variant_sel, C, n_pix, variant):
    """k_gram_px (64- and 256-thread CTAs) and the tiled k_gram against a float64
    numpy shifted Gram (transform.py:177-179 restated as one-pass sums): ragged
    pixel counts, C below the 12-band register width; band extremes bit-exact."""
    from paper_2506_19656_b200 import _device as dev
    variant_sel(variant)
    rng = np.random.default_rng(1000 * C + n_pix % 997)
    x = (rng.standard_normal((n_pix, C)) * 10.0 ** np.arange(C) / 7 + 3.0).astype(np.float32)
    arr = dev.to_device(x)
    g = G.gram(arr, n_pix, C, stats=True)
    torch.cuda.synchronize()
    assert g["err"].flags() == 0
    out = g["out"].cpu().numpy()
    d = x.astype(np.float64) - x[0].astype(np.float64)
    want_sums = d.sum(axis=0)
    want_G = d.T @ d
    scale = np.sqrt(np.outer(np.diag(want_G), np.diag(want_G))) + 1e-300
    np.testing.assert_allclose(out[:C], want_sums, rtol=0, atol=1e-10 * np.abs(d).sum(axis=0).max() + 1e-300)
    assert np.all(np.abs(out[C:].reshape(C, C) - want_G) <= 1e-10 * scale + 1e-300)
    np.testing.assert_array_equal(g["mins"].cpu().numpy(), x.min(axis=0).astype(np.float64))
    np.testing.assert_array_equal(g["maxs"].cpu().numpy(), x.max(axis=0).astype(np.float64))


# ------------------------------------------------------------------ bulk-copy SSIM kernel edge cases

@pytest.mark.parametrize("shape,bits,n_pcs,noisy", [
    ((3, 11, 256, 7), 10, 0, False),     # minimum height, 3 strips, partial last strip, band groups 4+3
    ((2, 37, 128, 5), 8, 0, True),       # odd H, u8 frames (W % 16), groups 4+1, noisy frames
    ((2, 24, 240, 4), 12, 0, False),     # 12-bit without PCA (exact float64 dequantisation), C % 4 == 0
    ((2, 19, 136, 12), 16, 6, True),     # PCA 12->6, three band groups, odd H
    ((2, 16, 64, 12), 12, 9, False),     # PCA 12->9
    ((1, 21, 128, 8), 8, 5, False),      # 8-bit PCA planes, generic plane count
    ((2, 13, 128, 24), 12, 0, False),    # 24 bands: four input stages only (the dynamic-ring path), six band groups
    ((1, 23, 136, 24), 10, 0, True),     # same with the lookup table resident (fewer stages still)
])
@pytest.mark.parametrize("kernel", [7, 8])
def test_ssim_bulk_kernel_shapes(cuda, variant_sel, shape, bits, n_pcs, noisy, kernel):
    """Both bulk-copy SSIM kernels (k_eval_ssim7 / k_eval_ssim8) in every decode mode."""
    if kernel == 7 and shape[3] > 16:
        pytest.skip("k_eval_ssim7 (A/B only) has fixed-depth rings: they do not fit this many bands")
    variant_sel({"eval_kernel": kernel})
    rng = np.random.default_rng(sum(shape) + bits)
    T, H, W, C = shape
    yy, xx = np.mgrid[0:H, 0:W]
    base = np.stack([np.sin(yy / (3 + c) + xx / (5 + 2 * c)) for c in range(C)], -1)
    x = (base[None] * (1 + np.arange(C)) + 0.3 * rng.normal(size=shape)).astype(np.float32)
    if n_pcs == 0:
        x[rng.random(shape) < 0.05] = np.nan
    spec = G_pipe.StreamSpec(bits, n_pcs=n_pcs)
    xt = torch.from_numpy(x).to(cuda)
    enc = G_pipe.encode_prep(xt, spec)
    enc.check()
    ref = O.encode_stream(x, bits, n_pcs=n_pcs)
    frames_o = ref["frames"]
    if n_pcs == 0:
        np.testing.assert_array_equal(enc.frames[0].cpu().numpy(), frames_o)
    if noisy:
        frames_o = O.decoded_frames_with_noise(frames_o, bits)
    # decode the oracle's frames so that only the decode+metric path is compared
    fr = torch.from_numpy(frames_o[None]).to(cuda)
    if n_pcs:
        enc.qmins.copy_(torch.from_numpy(np.asarray(ref["mins"])[None]))
        enc.qmaxs.copy_(torch.from_numpy(np.asarray(ref["maxs"])[None]))
        mean_o, comps_o, ev_o = ref["pca"]
        m = G.PcaModel(mean_o, comps_o, ev_o, n_input_channels=C)
        enc.pca[0] = G_pipe._fold(m)
    recon, sc = G_pipe.decode_eval(enc, xt, frames=fr)
    rec_o = O.decode_stream(frames_o, ref, x.shape, bits)
    if n_pcs == 0:
        np.testing.assert_array_equal(recon.cpu().numpy(), rec_o.astype(np.float32))
    else:
        np.testing.assert_allclose(recon.cpu().numpy(), rec_o, rtol=1e-5, atol=1e-5 * np.abs(rec_o).max())
    rep = sc.report()[0]
    np.testing.assert_allclose(rep["psnr_per_band"], M.psnr_per_band(ref["filled"], rec_o), atol=PSNR_TOL_DB)
    np.testing.assert_allclose(rep["ssim_per_band"], M.ssim_per_band(ref["filled"], rec_o), atol=SSIM_TOL)
    # no recon output requested: same scores
    _, sc2 = G_pipe.decode_eval(enc, xt, frames=fr, want_recon=False)
    np.testing.assert_allclose(sc2.report()[0]["ssim_per_band"], rep["ssim_per_band"], rtol=0, atol=1e-12)


# ------------------------------------------------------------------ kernel variants agree bit for bit

@pytest.mark.parametrize("variant", [{"qp_runtime_c": 1}, {"qp_px1": 1}, {"proj12": 0}, {"proj12": 0, "proj_nopf": 1}])
@pytest.mark.parametrize("shape,n_pcs,bits", [((3, 40, 72, 12), 6, 16), ((2, 33, 64, 12), 9, 12)])
def test_pca_variants_bit_identical(cuda, variant_sel, variant, shape, n_pcs, bits):
    """The compile-time C = 12 PCA quantiser, the pixel-pair path and the prefetching
    projection produce exactly the frames / ranges of their generic counterparts
    (the 1-LSB parity bar cannot see a divergence between them)."""
    from paper_2506_19656_b200 import synth

    x = synth.era5(49656, shape, device=cuda)
    spec = G_pipe.StreamSpec(bits, n_pcs=n_pcs, normalize=True)
    a = G_pipe.encode_prep(x, spec)
    fa, ma = a.frames.clone(), a.qmins.clone()
    variant_sel(variant)
    b = G_pipe.encode_prep(x, spec)
    assert torch.equal(b.qmins, ma) and torch.equal(b.qmaxs, a.qmaxs)
    assert torch.equal(b.frames, fa)


@pytest.mark.parametrize("kind", ["f32_c7_fill", "u16_c4"])
def test_static_band_count_quantiser_bit_identical(cuda, variant_sel, kind):
    """The compile-time band-count quantisers (7 float32 bands with fill, 4 uint16 bands) write
    exactly the frames / filled cube of the runtime-count kernel ("qp_runtime_c")."""
    from paper_2506_19656_b200 import synth

    if kind == "f32_c7_fill":
        x = synth.minicube(77, (9, 24, 32, 7), device=cuda)
        spec = G_pipe.StreamSpec(10, seg_len=4)
    else:
        x = synth.dynamic_earthnet(78, (6, 32, 32, 4), device=cuda).contiguous()
        spec = G_pipe.StreamSpec(8)
    a = G_pipe.encode_prep(x, spec)
    fa = a.frames.clone()
    filled_a = a.filled.clone() if a.filled is not None else None
    variant_sel({"qp_runtime_c": 1})
    b = G_pipe.encode_prep(x, spec)
    assert torch.equal(b.frames, fa)
    assert torch.equal(b.qmins, a.qmins) and torch.equal(b.qmaxs, a.qmaxs)
    if filled_a is not None:
        assert torch.equal(b.filled, filled_a)
