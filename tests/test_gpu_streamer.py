"""HostStreamer (the bench's end-to-end path: pinned host cubes in, frame slices out to the
host and back, metric sums out) against the device-resident round trip and the oracle."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import cubevid_oracle as O  # noqa: E402
from oracle import metrics_oracle as M  # noqa: E402


@pytest.mark.parametrize("chunk,n_pcs,bits", [(2, 0, 10), (1, 0, 8), (3, 4, 12)])
def test_host_streamer_matches_roundtrip(cuda, chunk, n_pcs, bits):
    from paper_2506_19656_b200 import pipeline, synth

    B, shape = 4, (12, 32, 48, 7)
    x = synth.minicube_batch(B, 4242, shape, device=cuda)
    if n_pcs:
        x = torch.nan_to_num(x, nan=0.25)
    spec = pipeline.StreamSpec(bits, n_pcs=n_pcs, seg_len=4)
    host = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
    host.copy_(x)
    st = pipeline.HostStreamer(tuple(x.shape), x.dtype, spec, chunk=chunk, want_ssim=True, device=cuda)
    reps = st.run(host)
    assert len(reps) == B
    T, H, W, C = shape
    E = n_pcs or C
    planes = 3 * ((E + 2) // 3)
    fbytes = B * planes * T * H * W * (1 if bits == 8 else 2)
    assert st.d2h_bytes >= fbytes and st.h2d_bytes == x.numel() * 4 + fbytes
    # the same cubes through the device-resident round trip
    _, _, sc = pipeline.roundtrip(x, spec)
    want = sc.report()
    for got, ref in zip(reps, want):
        np.testing.assert_allclose(got["psnr_per_band"], ref["psnr_per_band"], rtol=0, atol=1e-9)
        np.testing.assert_allclose(got["ssim_per_band"], ref["ssim_per_band"], rtol=0, atol=1e-12)
    # and one cube against the oracle
    xn = x[1].cpu().numpy()
    ref = O.encode_stream(xn, bits, n_pcs=n_pcs)
    rec = O.decode_stream(ref["frames"], ref, xn.shape, bits)
    np.testing.assert_allclose(reps[1]["psnr_per_band"], M.psnr_per_band(ref["filled"], rec), atol=0.01)
    np.testing.assert_allclose(reps[1]["ssim_per_band"], M.ssim_per_band(ref["filled"], rec), atol=1e-5)
    # a second run reuses the buffers and reproduces the scores
    again = st.run(host)
    np.testing.assert_array_equal(again[3]["ssim_per_band"], reps[3]["ssim_per_band"])
