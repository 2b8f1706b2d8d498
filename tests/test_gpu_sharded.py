"""Time-sharded pipeline on the GPU: two ranks (gloo process group, both on
cuda:0 — the collectives are host-driven, no kernel waits on another rank)
each own half of the time axis; their frames must be the corresponding slices
of the single-process frames and the combined metrics must match."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _make(kind):
    from paper_2506_19656_b200 import synth

    if kind == "nan":
        return synth.minicube(123, (30, 24, 40, 7)), dict(bit_depth=10, seg_len=4)
    if kind == "nan_pca":
        return synth.minicube(321, (30, 24, 40, 7)), dict(bit_depth=12, n_pcs=4, seg_len=4)
    return synth.simple_s2(shape=(6, 32, 48, 12)), dict(bit_depth=12, n_pcs=5)


def _worker(rank, world, port, kind, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2506_19656_b200 import pipeline as P
        from paper_2506_19656_b200.dist import TimeShard

        dev = torch.device("cuda", 0)
        x, kw = _make(kind)
        spec = P.StreamSpec(**kw)
        T = x.shape[0]
        cut = [0, T // 2 - 1, T]
        xl = x[cut[rank]:cut[rank + 1]].contiguous().to(dev)
        enc = P.encode_prep(xl, spec, shard=TimeShard())
        enc.check()
        _, sc = P.decode_eval(enc, xl)
        rep = sc.report()[0]
        q.put((rank, ("ok", enc.frames[0].cpu().numpy(), enc.qmins.cpu().numpy(), rep["psnr_per_band"],
                      rep.get("ssim_per_band"))))
    except Exception as e:
        import traceback

        q.put((rank, ("err", traceback.format_exc())))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["nan", "pca", "nan_pca"])
def test_two_time_shards_match_single_gpu(cuda, kind):
    from paper_2506_19656_b200 import pipeline as P

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert res[r][0] == "ok", res[r][1]

    x, kw = _make(kind)
    enc, _, sc = P.roundtrip(x.to(cuda), P.StreamSpec(**kw))
    full = enc.frames[0].cpu().numpy()
    T = x.shape[0]
    cut = [0, T // 2 - 1, T]
    rep = sc.report()[0]
    for r in range(world):
        _, fr, qmins, psnr, ssim = res[r]
        part = full[:, cut[r]:cut[r + 1]]
        if kind == "nan":
            np.testing.assert_array_equal(qmins, enc.qmins.cpu().numpy())
            np.testing.assert_array_equal(fr, part)
        else:
            d = np.abs(fr.astype(np.int64) - part.astype(np.int64))
            assert d.max() <= 1 and (d > 0).mean() < 0.01
        np.testing.assert_allclose(psnr, rep["psnr_per_band"], atol=1e-6 if kind == "nan" else 0.01)
        np.testing.assert_allclose(ssim, rep["ssim_per_band"], atol=1e-7 if kind == "nan" else 1e-5)
