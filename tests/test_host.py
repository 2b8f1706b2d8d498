"""Host-side logic of the drop-in (no GPU): types, validation messages, plans,
metric aggregation, pipeline specs and the kernel-constant folds."""

import math

import numpy as np
import pytest

from paper_2506_19656_b200 import ConfigurationError
from paper_2506_19656_b200 import plan as P
from paper_2506_19656_b200 import transform as T
from paper_2506_19656_b200.metrics import bpppb, psnr_from_sse
from paper_2506_19656_b200.pipeline import StreamSpec, _fold


def test_quantparams_validation(golden_errors):
    with pytest.raises(ConfigurationError) as e:
        T.QuantParams(9, (0.0,), (1.0,))
    assert str(e.value) == golden_errors["bad_depth"]
    with pytest.raises(ConfigurationError):
        T.QuantParams(8, (0.0, 1.0), (1.0,))
    with pytest.raises(ConfigurationError):
        T.QuantParams(8, (float("nan"),), (1.0,))
    with pytest.raises(ConfigurationError):
        T.QuantParams(8, (2.0,), (1.0,))
    p = T.QuantParams(12, (0.0, 5.0), (1.0, 5.0))
    assert p.levels == 4095 and p.n_channels == 2 and p.is_constant(1) and not p.is_constant(0)
    assert p.step(0) == 1.0 / 4095


def test_pcamodel_validation(golden):
    m = T.PcaModel(golden["pca_mean"], golden["pca_comps"], golden["pca_ev"], 5)
    assert m.n_kept == 3
    with pytest.raises(ConfigurationError):
        T.PcaModel(golden["pca_mean"], 2 * golden["pca_comps"], golden["pca_ev"], 5)
    with pytest.raises(ConfigurationError):
        T.PcaModel(golden["pca_mean"], golden["pca_comps"], golden["pca_ev"][::-1], 5)
    with pytest.raises(ConfigurationError):
        T.PcaModel(golden["pca_mean"][:4], golden["pca_comps"], golden["pca_ev"], 5)


def test_eig_model_matches_reference_convention(golden):
    x = golden["pca_in"].reshape(-1, 5).astype(np.float64)
    mean = x.mean(axis=0)
    cov = (x - mean).T @ (x - mean) / x.shape[0]
    m = T.eig_model(mean, cov, 3, 5)
    np.testing.assert_allclose(m.components, golden["pca_comps"], atol=1e-10)
    np.testing.assert_allclose(m.explained_variance, golden["pca_ev"], rtol=1e-10)


def test_covariance_from_shifted_gram(golden):
    x = golden["pca_in"].reshape(-1, 5).astype(np.float64)
    shift = x[0]
    d = x - shift
    out = np.concatenate([d.sum(axis=0), (d.T @ d).reshape(-1)])
    mean, cov = T.covariance_from_gram(shift, out, x.shape[0], 5)
    ref_mean = x.mean(axis=0)
    np.testing.assert_allclose(mean, ref_mean, rtol=1e-13)
    np.testing.assert_allclose(cov, (x - ref_mean).T @ (x - ref_mean) / x.shape[0], rtol=1e-10, atol=1e-13)


def test_pack_groups_match_reference(golden_groups):
    for n in range(1, 65):
        got = [[list(g.members), g.n_real, g.video_index] for g in P.pack_groups(n)]
        assert got == golden_groups[str(n)]
    assert [g.members for g in P.pack_groups(4)] == [(0, 1, 2), (3, 3, 3)]
    assert len(P.plan_stream(9, 12)) == 3
    assert P.video_names("bands", P.pack_groups(4)) == ("bands_0001", "bands_0002")
    with pytest.raises(ConfigurationError):
        P.pack_groups(0)
    with pytest.raises(ConfigurationError):
        P.ChannelGroup(1, (0, 1, 2), 2)


def test_bpppb_and_psnr_aggregation():
    assert bpppb(1000, 10, 10, 10, 1) == 8.0
    with pytest.raises(ConfigurationError):
        bpppb(1, 0, 1, 1, 1)
    db, agg = psnr_from_sse(np.array([0.25 * 4]), np.array([3.0]), 4)
    assert abs(db[0] - 10 * math.log10(36)) < 1e-12 and agg == db[0]
    db, agg = psnr_from_sse(np.array([0.0, 1.0]), np.array([1.0, 1.0]), 1)
    assert math.isinf(db[0]) and agg == db[1] == 0.0
    with pytest.warns(RuntimeWarning):
        db, agg = psnr_from_sse(np.array([1.0, 1.0]), np.array([0.0, 2.0]), 1)
    assert np.isnan(db[0]) and agg == db[1]


def test_stream_spec():
    StreamSpec(10)
    with pytest.raises(ConfigurationError):
        StreamSpec(9)
    with pytest.raises(ConfigurationError):
        StreamSpec(8, pad_mode="mirror")


def test_normalised_pca_fold_is_exact_algebra(golden):
    rng = np.random.default_rng(5)
    x = rng.normal(size=(50, 4)) * np.array([1e3, 1.0, 1e-2, 10.0]) + 7.0
    lo, sc = x.min(axis=0), x.max(axis=0) - x.min(axis=0)
    z = (x - lo) / sc
    mu = z.mean(axis=0)
    w, v = np.linalg.eigh(np.cov(z.T, bias=True))
    model = T.PcaModel(mu, v[:, ::-1][:, :2].T, np.clip(w[::-1][:2], 0, None), 4)
    fold = _fold(model, lo, sc)
    pcs_ref = (z - mu) @ model.components.T
    pcs = (x - fold.fwd_mean) @ fold.fwd_comps.T
    np.testing.assert_allclose(pcs, pcs_ref, rtol=1e-9, atol=1e-12)
    back_ref = (pcs_ref @ model.components + mu) * sc + lo
    back = pcs @ fold.inv_comps + fold.inv_mean
    np.testing.assert_allclose(back, back_ref, rtol=1e-10, atol=1e-12)


def test_synth_small_shapes():
    import torch

    from paper_2506_19656_b200 import synth

    c = synth.minicube(1, (10, 16, 16, 7))
    assert c.shape == (10, 16, 16, 7) and c.dtype == torch.float32
    assert torch.isnan(c).any() and (c[~torch.isnan(c)] >= 0).all() and (c[~torch.isnan(c)] <= 1).all()
    assert torch.equal(torch.isnan(synth.minicube(1, (10, 16, 16, 7))), torch.isnan(c))
    d = synth.dynamic_earthnet(shape=(3, 32, 32, 4))
    assert d.dtype == torch.uint16 and int(d.to(torch.int32).max()) == 10000
    e = synth.era5(shape=(2, 19, 36, 12))
    assert e.shape == (2, 19, 36, 12) and float(e[..., 11].mean()) > 1e3 * float(e[..., 0].mean())
    s = synth.simple_s2(shape=(2, 32, 32, 12))
    assert s.shape == (2, 32, 32, 12)
