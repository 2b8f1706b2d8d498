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


def test_mapping_rule_and_plan_stream(golden_errors, golden_groups):
    ok = dict(stream_name="s", input_vars=("a",), axis_order=("t", "y", "x"))
    for key, kw in (("rule_noname", dict(ok, stream_name="")), ("rule_novars", dict(ok, input_vars=())),
                    ("rule_axes", dict(ok, axis_order=("t", "y"))), ("rule_npcs", dict(ok, n_pcs=-1)),
                    ("rule_depth", dict(ok, out_bit_depth=9))):
        with pytest.raises(ConfigurationError) as e:
            P.MappingRule(**kw)
        assert str(e.value) == golden_errors[key]
    rule = P.MappingRule("s", "a", ("time", "y", "x"), n_pcs=4)
    assert rule.input_vars == ("a",) and not rule.config_is_list
    got = [[g.video_index, list(g.members), g.n_real] for g in P.plan_stream(rule, 7)]
    assert got == golden_groups["rule_npcs4_of_7"]
    assert len(P.plan_stream(P.MappingRule("s", "a", ("time", "y", "x")), 7)) == 3


def test_select_for_video_validation(golden, golden_errors):
    from paper_2506_19656_b200 import cube as Cb

    dc = Cb.DataCube({"a": golden["sel_a"], "v4": golden["sel_4d"]},
                     {"a": ("time", "y", "x"), "v4": ("band", "time", "x2", "y2")})
    assert "a" in dc and dc.axis_length("x") == 130 and dc.variable_names() == ("a", "v4")
    assert Cb.channel_axis_of(dc, "v4", ("time", "y2", "x2")) == "band"
    for key, names, order in (("sel_axis3", ["a"], ("time", "y")), ("sel_dup", ["a", "a"], ("time", "y", "x")),
                              ("sel_empty", [], ("time", "y", "x")), ("sel_missing", ["zz"], ("time", "y", "x")),
                              ("sel_mix", ["a", "v4"], ("time", "y", "x")),
                              ("sel_axes", ["a"], ("time", "y", "lon")),
                              ("sel_4d_axes", ["v4"], ("time", "y", "x"))):
        with pytest.raises(ConfigurationError) as e:
            Cb.select_for_video(dc, names, order)
        assert str(e.value) == golden_errors[key], key
    with pytest.raises(ConfigurationError):
        Cb.DataCube({"a": golden["sel_a"]}, {"a": ("t", "y")})
    with pytest.raises(ConfigurationError):
        Cb.DataCube({"a": golden["sel_a"], "b": golden["sel_b"]}, {"a": ("t", "y", "x"), "b": ("t", "y", "x")})


def test_corrupt_stream_error(golden_errors):
    from paper_2506_19656_b200 import CodecError, CorruptStreamError
    from paper_2506_19656_b200.bridge import _planar_bytes_to_frames, check_stream_bytes

    with pytest.raises(CorruptStreamError) as e:
        _planar_bytes_to_frames(b"\x00" * 7, 4, 5, 3, 10)
    assert f"CorruptStreamError: {e.value}" == golden_errors["corrupt_stream"]
    assert issubclass(CorruptStreamError, CodecError)
    assert check_stream_bytes(4 * 5 * 3 * 2 * 6, 4, 5, 3, 10) == 6
    with pytest.raises(CorruptStreamError):
        check_stream_bytes(10, 0, 5, 3, 8)


def test_errors_are_the_reference_classes_when_importable():
    """With cubevid on the path the drop-in raises the reference's own classes."""
    import subprocess
    import sys
    from pathlib import Path

    ref = Path("/root/reference/pkg/src")
    if not ref.exists():
        pytest.skip("the reference tree only exists in the build container")
    root = Path(__file__).resolve().parents[1]
    code = ("import cubevid.errors as r, paper_2506_19656_b200.errors as e;"
            "assert e.SHARED_WITH_REFERENCE and e.ConfigurationError is r.ConfigurationError "
            "and e.CorruptStreamError is r.CorruptStreamError")
    subprocess.run([sys.executable, "-c", code], check=True, cwd=root,
                   env={"PYTHONPATH": f"{ref}:{root}", "PATH": "/usr/bin:/bin"})
