"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports cubevid.{cube,transform,plan,codecs.bridge} unchanged, feeds them
small seeded inputs and stores inputs + outputs in tests/golden/golden.npz
(and the exception messages in golden_errors.json). The oracle and the GPU
path are both checked against these fixtures; nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
if str(REF) not in sys.path:
    sys.path.insert(0, str(REF))

from cubevid import cube as rcube  # noqa: E402
from cubevid import plan as rplan  # noqa: E402
from cubevid import transform as rt  # noqa: E402
from cubevid.codecs import bridge as rbridge  # noqa: E402
from cubevid.errors import ConfigurationError  # noqa: E402

OUT = Path(__file__).resolve().parent


def nan_cube(rng, shape, frac_frames=0.2, frac_px=0.05, leading=True):
    t, h, w, c = shape
    x = rng.random(shape, dtype=np.float64).astype(np.float32)
    nt = max(1, int(round(frac_frames * t)))
    tt = rng.choice(t, nt, replace=False)
    x[tt] = np.nan
    x[rng.random((t, h, w)) < frac_px] = np.nan
    if leading:
        x[0, 0, 0, :] = np.nan
        x[:3, 1, 1, 0] = np.nan       # leading run of 3
        x[:, 2, 2, 1] = np.nan        # column never observed
    return x


def main():
    rng = np.random.default_rng(2506_19656)
    g = {}
    errors = {}

    # ---- forward_fill_time (cube.py:213-246)
    x = nan_cube(rng, (12, 5, 6, 3))
    g["fill_in"] = x
    for name, ax, fv in (("t0_f0", 0, 0.0), ("t0_f01", 0, 0.1), ("t0_fm3", 0, -3.5)):
        f, m = rcube.forward_fill_time(x, ax, fv)
        g[f"fill_{name}_out"], g[f"fill_{name}_mask"] = f, m.mask
    y = np.ascontiguousarray(np.moveaxis(x, 0, 2))  # time axis 2
    g["fill_ax2_in"] = y
    f, m = rcube.forward_fill_time(y, 2, 0.0)
    g["fill_ax2_out"], g["fill_ax2_mask"] = f, m.mask
    f, m = rcube.forward_fill_time(y, -2, 0.25)
    g["fill_axm2_out"], g["fill_axm2_mask"] = f, m.mask
    xi = rng.integers(0, 1000, (4, 3, 2, 2)).astype(np.uint16)
    f, m = rcube.forward_fill_time(xi, 0)
    g["fill_int_in"], g["fill_int_out"], g["fill_int_mask"] = xi, f, m.mask
    try:
        bad = x.copy()
        bad[1, 1, 1, 1] = np.inf
        rcube.forward_fill_time(bad, 0)
    except ConfigurationError as e:
        errors["fill_inf"] = str(e)
    try:
        rcube.forward_fill_time(x, 4)
    except ConfigurationError as e:
        errors["fill_axis"] = str(e)

    # ---- fit_quant / quantize / dequantize (transform.py:61-126)
    filled, _ = rcube.forward_fill_time(x, 0, 0.0)
    q_in = filled.copy()
    q_in[..., 2] = np.where(np.isfinite(q_in[..., 2]), q_in[..., 2], 0)
    g["q_in"] = q_in
    for B in (8, 10, 12, 16):
        p = rt.fit_quant(q_in, B)
        g[f"q{B}_mins"], g[f"q{B}_maxs"] = np.array(p.mins), np.array(p.maxs)
        q = rt.quantize(q_in, p)
        g[f"q{B}_out"] = q
        g[f"dq{B}_out"] = rt.dequantize(q, p)
    # constant channel + exact half ties: values k/(2L) at B=8 on [0,1]
    ties = (np.arange(2 * 255 + 1, dtype=np.float64) / (2 * 255)).astype(np.float32)
    tcube = np.zeros((1, 1, ties.size, 3), np.float32)
    tcube[0, 0, :, 0] = ties
    tcube[0, 0, :, 1] = 7.5
    tcube[0, 0, :, 2] = ties[::-1] * 10 - 5
    g["ties_in"] = tcube
    for B in (8, 10, 12, 16):
        p = rt.fit_quant(tcube, B)
        g[f"ties{B}_out"] = rt.quantize(tcube, p)
        g[f"ties{B}_mins"], g[f"ties{B}_maxs"] = np.array(p.mins), np.array(p.maxs)
    # clamp with a narrower range
    pc = rt.QuantParams(12, (0.2, 0.0, 0.0), (0.8, 1.0, 1.0))
    g["clamp12_out"] = rt.quantize(q_in, pc, clamp=True)
    try:
        rt.quantize(q_in, pc)
    except ConfigurationError as e:
        errors["quantize_range"] = str(e)
    try:
        rt.fit_quant(x, 8)
    except ConfigurationError as e:
        errors["fit_nonfinite"] = str(e)
    try:
        rt.QuantParams(9, (0.0,), (1.0,))
    except ConfigurationError as e:
        errors["bad_depth"] = str(e)
    try:
        rt.dequantize(np.full((1, 1, 1, 3), 300, np.uint16), rt.QuantParams(8, (0,) * 3, (1,) * 3))
    except ConfigurationError as e:
        errors["dequant_range"] = str(e)
    # u16 source (DynamicEarthNet-like) and f64 source (PC-like)
    u = rng.integers(0, 10001, (5, 4, 6, 4)).astype(np.uint16)
    g["u16_in"] = u
    p = rt.fit_quant(u, 8)
    g["u16_mins"], g["u16_maxs"], g["u16_q8"] = np.array(p.mins), np.array(p.maxs), rt.quantize(u, p)
    d = rng.normal(size=(4, 5, 6, 5)) * np.array([100.0, 10.0, 1.0, 0.1, 1e-3])
    g["f64_in"] = d
    p = rt.fit_quant(d, 16)
    g["f64_mins"], g["f64_maxs"], g["f64_q16"] = np.array(p.mins), np.array(p.maxs), rt.quantize(d, p)

    # ---- PCA (transform.py:160-210)
    base = rng.normal(size=(6, 8, 9, 2))
    mix = rng.normal(size=(2, 5))
    pcube = (base @ mix + 0.05 * rng.normal(size=(6, 8, 9, 5)) + 3.0).astype(np.float32)
    g["pca_in"] = pcube
    m = rt.pca_fit(pcube, 3)
    g["pca_mean"], g["pca_comps"], g["pca_ev"] = m.mean, m.components, m.explained_variance
    pcs = rt.pca_forward(pcube, m)
    g["pca_fwd"] = pcs
    g["pca_inv"] = rt.pca_inverse(pcs, m)
    mfull = rt.pca_fit(pcube, 5)
    g["pcafull_comps"], g["pcafull_ev"] = mfull.components, mfull.explained_variance
    # rank-1 2-channel
    r1 = rng.normal(size=(3, 4, 5, 1))
    r1 = np.concatenate([r1, 2 * r1], axis=-1)
    m1 = rt.pca_fit(r1, 1)
    g["rank1_ev"] = m1.explained_variance
    try:
        rt.pca_fit(pcube, 6)
    except ConfigurationError as e:
        errors["pca_nkeep"] = str(e)

    # ---- pack_groups (plan.py:118-128)
    groups = {str(n): [[list(gr.members), gr.n_real, gr.video_index] for gr in rplan.pack_groups(n)]
              for n in range(1, 65)}

    # ---- planar layout (bridge.py:157-174)
    fr8 = rng.integers(0, 256, (3, 4, 5, 3)).astype(np.uint8)
    fr10 = rng.integers(0, 1024, (3, 4, 5, 3)).astype(np.uint16)
    g["planar_in8"], g["planar_in10"] = fr8, fr10
    g["planar_b8"] = np.frombuffer(rbridge._frames_to_planar_bytes(fr8, 8), np.uint8)
    g["planar_b10"] = np.frombuffer(rbridge._frames_to_planar_bytes(fr10, 10), np.uint8)
    g["planar_back10"] = rbridge._planar_bytes_to_frames(g["planar_b10"].tobytes(), 4, 5, 3, 10)

    # ---- composed stream on a small NaN cube, C=7, 10-bit
    sc = nan_cube(rng, (20, 16, 16, 7), leading=True)
    g["stream_in"] = sc
    sf, smask = rcube.forward_fill_time(sc, 0, 0.0)
    sp = rt.fit_quant(sf, 10)
    sq = rt.quantize(sf, sp)
    vids = []
    for gr in rplan.pack_groups(7):
        vids.append(np.frombuffer(rbridge._frames_to_planar_bytes(sq[..., list(gr.members)], 10),
                                  np.uint16).reshape(20, 3, 16 * 16))
    g["stream_frames"] = np.stack(vids)
    g["stream_mins"], g["stream_maxs"] = np.array(sp.mins), np.array(sp.maxs)
    g["stream_recon"] = rt.dequantize(sq, sp)
    g["stream_filled"] = sf

    # ---- select_for_video (cube.py:249-305), MappingRule / plan_stream (plan.py:26-66, 131-139),
    # CorruptStreamError (bridge.py:163-171); own generator so the arrays above never change
    r2 = np.random.default_rng(2506_19656 + 1)
    va = r2.random((6, 9, 130)).astype(np.float32)            # (time, y, x)
    vb = r2.random((130, 6, 9)).astype(np.float32)            # (x, time, y)
    vc = r2.random((9, 130, 6)).astype(np.float32)            # (y, x, time)
    v4 = r2.integers(0, 60000, (5, 6, 7, 9)).astype(np.uint16)  # (band, time, x, y)
    g["sel_a"], g["sel_b"], g["sel_c"], g["sel_4d"] = va, vb, vc, v4
    dc = rcube.DataCube({"a": va, "b": vb, "c": vc, "v4": v4},
                        {"a": ("time", "y", "x"), "b": ("x", "time", "y"), "c": ("y", "x", "time"),
                         "v4": ("band", "time", "x2", "y2")})
    g["sel_abc"] = rcube.select_for_video(dc, ["a", "b", "c"], ("time", "y", "x"))
    g["sel_cb_yxt"] = rcube.select_for_video(dc, ["c", "b"], ("y", "x", "time"))
    g["sel_4d_out"] = rcube.select_for_video(dc, "v4", ("time", "y2", "x2"))
    for key, names, order in (("sel_axis3", ["a"], ("time", "y")), ("sel_dup", ["a", "a"], ("time", "y", "x")),
                              ("sel_empty", [], ("time", "y", "x")), ("sel_missing", ["zz"], ("time", "y", "x")),
                              ("sel_mix", ["a", "v4"], ("time", "y", "x")),
                              ("sel_axes", ["a"], ("time", "y", "lon")),
                              ("sel_4d_axes", ["v4"], ("time", "y", "x"))):
        try:
            rcube.select_for_video(dc, names, order)
        except ConfigurationError as e:
            errors[key] = str(e)
    for key, kw in (("rule_noname", dict(stream_name="", input_vars=("a",), axis_order=("t", "y", "x"))),
                    ("rule_novars", dict(stream_name="s", input_vars=(), axis_order=("t", "y", "x"))),
                    ("rule_axes", dict(stream_name="s", input_vars=("a",), axis_order=("t", "y"))),
                    ("rule_npcs", dict(stream_name="s", input_vars=("a",), axis_order=("t", "y", "x"), n_pcs=-1)),
                    ("rule_depth", dict(stream_name="s", input_vars=("a",), axis_order=("t", "y", "x"),
                                        out_bit_depth=9))):
        try:
            rplan.MappingRule(**kw)
        except ConfigurationError as e:
            errors[key] = str(e)
    rule = rplan.MappingRule("s", ("a", "b"), ("time", "y", "x"), n_pcs=4)
    groups["rule_npcs4_of_7"] = [[gr.video_index, list(gr.members), gr.n_real] for gr in rplan.plan_stream(rule, 7)]
    try:
        rbridge._planar_bytes_to_frames(b"\x00" * 7, 4, 5, 3, 10)
    except Exception as e:  # CorruptStreamError
        errors["corrupt_stream"] = f"{type(e).__name__}: {e}"

    np.savez_compressed(OUT / "golden.npz", **g)
    (OUT / "golden_groups.json").write_text(json.dumps(groups))
    (OUT / "golden_errors.json").write_text(json.dumps(errors, indent=1))
    print(f"wrote {len(g)} arrays, {len(errors)} error messages")


if __name__ == "__main__":
    main()
