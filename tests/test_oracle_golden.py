"""Pin the CPU oracle against vectors produced by the reference itself
(tests/golden/make_golden.py ran cubevid unchanged)."""

import numpy as np
import pytest

from oracle import cubevid_oracle as O


def test_fill_time0(golden):
    x = golden["fill_in"]
    for name, fv in (("t0_f0", 0.0), ("t0_f01", 0.1), ("t0_fm3", -3.5)):
        f, m = O.forward_fill(x, 0, fv)
        assert f.dtype == golden[f"fill_{name}_out"].dtype
        np.testing.assert_array_equal(f.view(np.uint32), golden[f"fill_{name}_out"].view(np.uint32))
        np.testing.assert_array_equal(m, golden[f"fill_{name}_mask"])


def test_fill_other_axes_and_ints(golden):
    f, m = O.forward_fill(golden["fill_ax2_in"], 2, 0.0)
    np.testing.assert_array_equal(f, golden["fill_ax2_out"])
    np.testing.assert_array_equal(m, golden["fill_ax2_mask"])
    f, m = O.forward_fill(golden["fill_ax2_in"], -2, 0.25)
    np.testing.assert_array_equal(f, golden["fill_axm2_out"])
    np.testing.assert_array_equal(m, golden["fill_axm2_mask"])
    f, m = O.forward_fill(golden["fill_int_in"], 0)
    np.testing.assert_array_equal(f, golden["fill_int_out"])
    assert m.all()


def test_fill_idempotent_and_valid_cells(golden):
    x = golden["fill_in"]
    f, m = O.forward_fill(x, 0, 0.0)
    f2, m2 = O.forward_fill(f, 0, 0.0)
    np.testing.assert_array_equal(f, f2)
    assert m2.all()
    np.testing.assert_array_equal(f[m].view(np.uint32), x[m].view(np.uint32))


@pytest.mark.parametrize("B", [8, 10, 12, 16])
def test_quantize_bitexact(golden, B):
    x = golden["q_in"]
    mins, maxs = O.fit_quant(x)
    np.testing.assert_array_equal(mins, golden[f"q{B}_mins"])
    np.testing.assert_array_equal(maxs, golden[f"q{B}_maxs"])
    q = O.quantize(x, mins, maxs, B)
    assert q.dtype == golden[f"q{B}_out"].dtype
    np.testing.assert_array_equal(q, golden[f"q{B}_out"])
    dq = O.dequantize(q, mins, maxs, B)
    np.testing.assert_array_equal(dq.view(np.uint64), golden[f"dq{B}_out"].view(np.uint64))


@pytest.mark.parametrize("B", [8, 10, 12, 16])
def test_ties_and_constant(golden, B):
    x = golden["ties_in"]
    mins, maxs = O.fit_quant(x)
    np.testing.assert_array_equal(mins, golden[f"ties{B}_mins"])
    np.testing.assert_array_equal(O.quantize(x, mins, maxs, B), golden[f"ties{B}_out"])


def test_clamp_u16_f64(golden):
    q = O.quantize(golden["q_in"], (0.2, 0.0, 0.0), (0.8, 1.0, 1.0), 12, clamp=True)
    np.testing.assert_array_equal(q, golden["clamp12_out"])
    with pytest.raises(O.OracleError):
        O.quantize(golden["q_in"], (0.2, 0.0, 0.0), (0.8, 1.0, 1.0), 12)
    u = golden["u16_in"]
    mins, maxs = O.fit_quant(u)
    np.testing.assert_array_equal(mins, golden["u16_mins"])
    np.testing.assert_array_equal(O.quantize(u, mins, maxs, 8), golden["u16_q8"])
    d = golden["f64_in"]
    mins, maxs = O.fit_quant(d)
    np.testing.assert_array_equal(O.quantize(d, mins, maxs, 16), golden["f64_q16"])


def test_pca(golden):
    x = golden["pca_in"]
    mean, comps, ev = O.pca_fit(x, 3)
    np.testing.assert_allclose(mean, golden["pca_mean"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(comps, golden["pca_comps"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(ev, golden["pca_ev"], rtol=1e-10)
    pcs = O.pca_forward(x, mean, comps)
    np.testing.assert_allclose(pcs, golden["pca_fwd"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(O.pca_inverse(pcs, mean, comps), golden["pca_inv"], rtol=0, atol=1e-10)
    _, _, ev1 = O.pca_fit(np.concatenate([golden["pca_in"][..., :1]] * 2, axis=-1), 1)
    assert ev1.shape == (1,)
    np.testing.assert_allclose(golden["rank1_ev"].sum(), golden["rank1_ev"][0])


def test_pack_groups(golden_groups):
    for n in range(1, 65):
        got = [[list(m), r, i + 1] for i, (m, r) in enumerate(O.pack_groups(n))]
        assert got == golden_groups[str(n)]


def test_planar_layout(golden):
    assert O.planar_bytes(golden["planar_in8"], 8) == golden["planar_b8"].tobytes()
    assert O.planar_bytes(golden["planar_in10"], 10) == golden["planar_b10"].tobytes()
    back = O.frames_from_planar_bytes(golden["planar_b10"].tobytes(), 4, 5, 3, 10)
    np.testing.assert_array_equal(back, golden["planar_back10"])
    with pytest.raises(O.OracleError):
        O.frames_from_planar_bytes(b"\x00" * 7, 4, 5, 3, 10)


def test_stream_composition(golden):
    enc = O.encode_stream(golden["stream_in"], 10)
    np.testing.assert_array_equal(enc["filled"], golden["stream_filled"])
    np.testing.assert_array_equal(enc["mins"], golden["stream_mins"])
    np.testing.assert_array_equal(enc["frames"], golden["stream_frames"])
    rec = O.decode_stream(enc["frames"], enc, golden["stream_in"].shape, 10)
    np.testing.assert_array_equal(rec, golden["stream_recon"])


def test_select_for_video(golden):
    v = {k: golden[f"sel_{k}"] for k in ("a", "b", "c")}
    v["v4"] = golden["sel_4d"]
    ax = {"a": ("time", "y", "x"), "b": ("x", "time", "y"), "c": ("y", "x", "time"),
          "v4": ("band", "time", "x2", "y2")}
    np.testing.assert_array_equal(O.select_for_video(v, ax, ["a", "b", "c"], ("time", "y", "x")), golden["sel_abc"])
    np.testing.assert_array_equal(O.select_for_video(v, ax, ["c", "b"], ("y", "x", "time")), golden["sel_cb_yxt"])
    out = O.select_for_video(v, ax, "v4", ("time", "y2", "x2"))
    assert out.dtype == np.uint16
    np.testing.assert_array_equal(out, golden["sel_4d_out"])
    for names, order in ((["a"], ("time", "y")), (["a", "a"], ("time", "y", "x")), ([], ("time", "y", "x")),
                         (["zz"], ("time", "y", "x")), (["a", "v4"], ("time", "y", "x")),
                         (["a"], ("time", "y", "lon")), (["v4"], ("time", "y", "x"))):
        with pytest.raises(O.OracleError):
            O.select_for_video(v, ax, names, order)
