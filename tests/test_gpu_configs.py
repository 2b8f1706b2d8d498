"""BASELINE.json configurations on the GPU: parity against the oracle at sizes
the oracle finishes in seconds (full H x W x C, truncated T), plus full-size
size-independent properties (round-trip error bound, shard/batch invariance)."""

import numpy as np
import pytest
import torch

from oracle import cubevid_oracle as O
from oracle import metrics_oracle as M
from paper_2506_19656_b200 import pipeline as P
from paper_2506_19656_b200 import synth

pytestmark = pytest.mark.gpu


def _parity(x_dev, spec, bit_exact=True, ssim=True):
    x = x_dev.cpu().numpy()
    enc, recon, sc = P.roundtrip(x_dev, spec, want_ssim=ssim)
    enc.check()
    ref = O.encode_stream(x, spec.bit_depth, n_pcs=spec.n_pcs, fill=spec.fill_value,
                          normalize=spec.normalize)
    got = enc.frames[0].cpu().numpy()
    if bit_exact:
        np.testing.assert_array_equal(enc.qmins[0].cpu().numpy(), ref["mins"])
        np.testing.assert_array_equal(got, ref["frames"])
    else:
        d = np.abs(got.astype(np.int64) - ref["frames"].astype(np.int64))
        assert d.max() <= 1 and (d > 0).mean() <= 0.02, (d.max(), (d > 0).mean())
    rec_o = O.decode_stream(ref["frames"], ref, x.shape, spec.bit_depth)
    rep = sc.report()[0]
    np.testing.assert_allclose(rep["psnr_per_band"], M.psnr_per_band(ref["filled"], rec_o), atol=0.01)
    if ssim:
        np.testing.assert_allclose(rep["ssim_per_band"], M.ssim_per_band(ref["filled"], rec_o), atol=1e-5)
    return enc, recon, rep


def test_config1_minicube(cuda):
    x = synth.make(1, device=cuda, T=60)
    _parity(x, P.StreamSpec(8), ssim=True)


def test_config1_full_T_bit_exact(cuda):
    x = synth.make(1, device=cuda)
    enc = P.encode_prep(x, P.StreamSpec(8))
    ref = O.encode_stream(x.cpu().numpy(), 8)
    np.testing.assert_array_equal(enc.frames[0].cpu().numpy(), ref["frames"])


def test_config2_batch(cuda):
    xb = synth.make(2, device=cuda, batch=3, T=40)
    enc, recon, sc = P.roundtrip(xb, P.StreamSpec(10))
    reps = sc.report()
    for b in range(3):
        ref = O.encode_stream(xb[b].cpu().numpy(), 10)
        np.testing.assert_array_equal(enc.frames[b].cpu().numpy(), ref["frames"])
        rec_o = O.decode_stream(ref["frames"], ref, xb[b].shape, 10)
        np.testing.assert_allclose(reps[b]["psnr_per_band"], M.psnr_per_band(ref["filled"], rec_o),
                                   atol=0.01)
        np.testing.assert_allclose(reps[b]["ssim_per_band"], M.ssim_per_band(ref["filled"], rec_o),
                                   atol=1e-5)


def test_config3_simple_s2(cuda):
    x = synth.make(3, device=cuda, T=3)
    _parity(x, P.StreamSpec(12, n_pcs=9), bit_exact=False)


def test_config4_dynamic_earthnet(cuda):
    x = synth.make(4, device=cuda, T=6)
    _parity(x, P.StreamSpec(8), ssim=False)


def test_config5_era5(cuda):
    x = synth.make(5, device=cuda, T=2)
    _parity(x, P.StreamSpec(16, n_pcs=6, normalize=True), bit_exact=False)


def test_config2_full_cube_properties(cuda):
    """A full 495-step minicube: round trip within half a step, bpppb, SSIM in range."""
    x = synth.make(1, device=cuda)
    spec = P.StreamSpec(10)
    enc, recon, sc = P.roundtrip(x, spec)
    enc.check()
    filled = torch.from_numpy(O.forward_fill(x.cpu().numpy(), 0, 0.0)[0]).to(cuda)
    step = (enc.qmaxs - enc.qmins)[0] / 1023
    err = (recon.double() - filled.double()).abs().amax(dim=(0, 1, 2))
    assert (err <= step / 2 + 1e-7).all()
    rep = sc.report()[0]
    assert abs(rep["bpppb"] - 8 * 2 * 9 / 7) < 1e-12
    assert 0.9 < rep["ssim"] <= 1.0 and rep["psnr"] > 50
