"""GPU parity of the layout entry points either side of the hot path:
select_for_video (cube.py:249-305) and the planar byte streams of the codec
bridge (bridge.py:157-174), against the reference's golden outputs and the
oracle on seeded inputs. Pure data movement: bit-exact."""

import numpy as np
import pytest
import torch

from oracle import cubevid_oracle as O
from paper_2506_19656_b200 import CorruptStreamError
from paper_2506_19656_b200 import bridge as B
from paper_2506_19656_b200 import cube as Cb
from paper_2506_19656_b200 import pipeline as P
from paper_2506_19656_b200 import synth

pytestmark = pytest.mark.gpu

AXES = {"a": ("time", "y", "x"), "b": ("x", "time", "y"), "c": ("y", "x", "time"),
        "v4": ("band", "time", "x2", "y2")}


def _cube(golden, device=None):
    v = {k: golden[f"sel_{k}"] for k in ("a", "b", "c")}
    v["v4"] = golden["sel_4d"]
    if device is not None:
        v = {k: torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a).to(device)
             for k, a in v.items()}
    return Cb.DataCube(v, AXES)


def test_select_for_video_golden(cuda, golden):
    dc = _cube(golden)
    out = Cb.select_for_video(dc, ["a", "b", "c"], ("time", "y", "x"))
    assert isinstance(out, np.ndarray) and out.dtype == np.float32 and out.flags.c_contiguous
    np.testing.assert_array_equal(out, golden["sel_abc"])
    np.testing.assert_array_equal(Cb.select_for_video(dc, ["c", "b"], ("y", "x", "time")), golden["sel_cb_yxt"])
    out4 = Cb.select_for_video(dc, "v4", ("time", "y2", "x2"))
    assert out4.dtype == np.uint16
    np.testing.assert_array_equal(out4, golden["sel_4d_out"])


def test_select_for_video_device_tensors(cuda, golden):
    dc = _cube(golden, cuda)
    out = Cb.select_for_video(dc, ["a", "b", "c"], ("time", "y", "x"))
    assert out.is_cuda and out.is_contiguous()
    np.testing.assert_array_equal(out.cpu().numpy(), golden["sel_abc"])
    out4 = Cb.select_for_video(dc, "v4", ("time", "y2", "x2"))
    np.testing.assert_array_equal(out4.cpu().numpy().view(np.uint16), golden["sel_4d_out"])


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16, np.float32, np.float64])
@pytest.mark.parametrize("C", [1, 7, 32])
def test_select_stack_oracle(cuda, dtype, C):
    rng = np.random.default_rng(C * 7 + np.dtype(dtype).itemsize)
    T, H, W = 3, 5, 261  # ragged x tiles
    perms = [("t", "y", "x"), ("x", "y", "t"), ("y", "t", "x")]
    variables, axes = {}, {}
    for c in range(C):
        ax = perms[c % 3]
        shape = tuple({"t": T, "y": H, "x": W}[a] for a in ax)
        variables[f"v{c}"] = (rng.random(shape) * 200).astype(dtype)
        axes[f"v{c}"] = ax
    names = [f"v{c}" for c in range(C)]
    want = O.select_for_video(variables, axes, names, ("t", "y", "x"))
    got = Cb.select_for_video(Cb.DataCube(variables, axes), names, ("t", "y", "x"))
    assert got.dtype == want.dtype and got.shape == want.shape
    np.testing.assert_array_equal(got, want)


def test_select_feeds_the_pipeline(cuda):
    """select -> encode_prep equals encode_prep on the already stacked cube."""
    x = synth.minicube(7, (8, 32, 48, 5), device=cuda)
    variables = {f"b{c}": x[..., c].permute(1, 2, 0).contiguous() for c in range(5)}  # (y, x, t)
    dc = Cb.DataCube(variables, {k: ("y", "x", "t") for k in variables})
    sel = Cb.select_for_video(dc, list(variables), ("t", "y", "x"))
    assert torch.equal(sel.view(torch.int32), x.view(torch.int32))
    spec = P.StreamSpec(10, seg_len=4)
    a, b = P.encode_prep(sel, spec), P.encode_prep(x, spec)
    assert torch.equal(a.frames, b.frames)


def test_planar_bytes_golden(cuda, golden):
    assert B._frames_to_planar_bytes(golden["planar_in8"], 8) == golden["planar_b8"].tobytes()
    assert B._frames_to_planar_bytes(golden["planar_in10"], 10) == golden["planar_b10"].tobytes()
    back = B._planar_bytes_to_frames(golden["planar_b10"].tobytes(), 4, 5, 3, 10)
    assert back.dtype == np.uint16
    np.testing.assert_array_equal(back, golden["planar_back10"])
    with pytest.raises(CorruptStreamError):
        B._planar_bytes_to_frames(golden["planar_b10"].tobytes()[:-2], 4, 5, 3, 10)


@pytest.mark.parametrize("bits,planes", [(8, 1), (8, 3), (12, 3), (16, 4)])
def test_planar_round_trip_oracle(cuda, bits, planes):
    rng = np.random.default_rng(bits + planes)
    dt = np.uint8 if bits == 8 else np.uint16
    fr = rng.integers(0, 2 ** bits, (4, 37, 53, planes)).astype(dt)
    raw = B._frames_to_planar_bytes(fr, bits)
    assert raw == O.planar_bytes(fr, bits)
    np.testing.assert_array_equal(B._planar_bytes_to_frames(raw, 37, 53, planes, bits), fr)
    # device in, device out
    dflat = B._frames_to_planar_bytes(torch.from_numpy(fr.view(np.int16) if bits > 8 else fr).to(cuda), bits)
    assert dflat.is_cuda and dflat.dtype == torch.uint8
    assert dflat.cpu().numpy().tobytes() == raw
    dback = B._planar_bytes_to_frames(dflat, 37, 53, planes, bits)
    assert dback.is_cuda
    np.testing.assert_array_equal(dback.cpu().numpy().view(dt), fr)


def test_video_slices_are_the_bridge_bytes(cuda):
    """Each [g] slice of the fused encoder's frames is the byte stream the reference's
    bridge would hand the encoder for video g (bridge.py:157-160 on quantize's output)."""
    x = synth.minicube(3, (6, 16, 24, 7), device=cuda)
    enc = P.encode_prep(x, P.StreamSpec(12, seg_len=4))
    ref = O.encode_stream(x.cpu().numpy(), 12)
    q = ref["q"]
    for g, (members, _) in enumerate(O.pack_groups(7)):
        want = O.planar_bytes(q[..., list(members)], 12)
        assert enc.frames[0, g].cpu().numpy().tobytes() == want


def test_decode_rejects_truncated_stream(cuda):
    x = synth.minicube(5, (6, 16, 24, 4), device=cuda)
    enc = P.encode_prep(x, P.StreamSpec(8, seg_len=4))
    bad = enc.frames.reshape(-1)[:-5]
    with pytest.raises(CorruptStreamError):
        P.decode_eval(enc, x, frames=bad, want_ssim=False)
    short = enc.frames[:, :, :-1].contiguous()  # whole frames, but one too few
    with pytest.raises(CorruptStreamError):
        P.decode_eval(enc, x, frames=short, want_ssim=False)
    flat = enc.frames.reshape(-1).clone()  # right byte count, flat: accepted
    _, sc = P.decode_eval(enc, x, frames=flat, want_ssim=False)
    assert np.isfinite(sc.report()[0]["psnr"])
