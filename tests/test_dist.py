"""Time-sharded (multi-GPU) combine logic, exercised with world_size=2 gloo
process groups on CPU: every combine must reproduce the single-process result
of the oracle on the whole cube."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cubevid_oracle as O


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cube():
    rng = np.random.default_rng(7)
    x = rng.random((13, 5, 6, 3)).astype(np.float32)
    x[rng.random(x.shape) < 0.35] = np.nan
    x[:9, 1, 1, 0] = np.nan          # leading gap crossing the shard boundary
    x[:, 2, 3, 1] = np.nan           # never observed
    x[7:, 4, 5, 2] = np.nan          # trailing gap fed by shard 0's carry
    return x


def _local_raw_stats(xs, first_shard):
    C = xs.shape[-1]
    flat = xs.reshape(xs.shape[0], -1, C)
    mins = np.array([np.nanmin(flat[..., c]) if np.isfinite(flat[..., c]).any() else np.inf for c in range(C)])
    maxs = np.array([np.nanmax(flat[..., c]) if np.isfinite(flat[..., c]).any() else -np.inf for c in range(C)])
    lead = np.isnan(xs[0]).reshape(-1, C).any(axis=0).astype(np.int32)
    nans = np.isnan(xs).reshape(-1, C).sum(axis=0)
    return mins, maxs, lead, nans


def _worker(rank, world, port, split, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2506_19656_b200.dist import TimeShard, last_observed

        sh = TimeShard()
        x = _cube()
        t0, t1 = split[rank], split[rank + 1]
        xs = x[t0:t1]
        C = x.shape[-1]

        # 1. band stats with the leading-fill rule
        mins, maxs, lead, nans = _local_raw_stats(xs, rank == 0)
        gm, gM, gn = sh.combine_band_stats(torch.tensor(mins), torch.tensor(maxs), torch.tensor(lead),
                                           torch.tensor(nans), 0.25)
        filled, _ = O.forward_fill(x, 0, 0.25)
        rm, rM = O.fit_quant(filled)
        np.testing.assert_array_equal(gm.numpy(), rm)
        np.testing.assert_array_equal(gM.numpy(), rM)
        assert int(gn.sum()) == int(np.isnan(x).sum())

        # 2. fill carries across the shard boundary
        inner = xs[0].size
        seg = xs.reshape(1, xs.shape[0], inner)  # one "segment" per time step
        last = last_observed(torch.tensor(seg))
        carry = sh.carry_in(last).numpy()[0]
        out = np.empty_like(xs)
        cur = np.where(np.isnan(carry), np.float32(0.25), carry).reshape(xs.shape[1:])
        for t in range(xs.shape[0]):
            cur = np.where(np.isnan(xs[t]), cur, xs[t])
            out[t] = cur
        np.testing.assert_array_equal(out, filled[t0:t1])

        # 3. PCA Gram re-centred on rank 0's shift
        v = filled[t0:t1].reshape(-1, C).astype(np.float64)
        shift = v[0]
        d = v - shift
        local = torch.tensor(np.concatenate([d.sum(axis=0), (d.T @ d).reshape(-1)]))
        s0, out_g, n = sh.combine_gram(torch.tensor(shift), local, v.shape[0], C)
        full = filled.reshape(-1, C).astype(np.float64)
        assert n == full.shape[0]
        np.testing.assert_array_equal(s0, full[0])
        mean = s0 + out_g[:C] / n
        cov = out_g[C:].reshape(C, C) / n - np.outer(out_g[:C] / n, out_g[:C] / n)
        np.testing.assert_allclose(mean, full.mean(axis=0), rtol=1e-12)
        np.testing.assert_allclose(cov, np.cov(full.T, bias=True), rtol=1e-9, atol=1e-14)

        # 4. metric partial sums
        a, b = sh.combine_scores(torch.full((1, C), float(rank + 1)), torch.full((1, C), 2.0))
        assert float(a[0, 0]) == sum(r + 1 for r in range(world)) and float(b[0, 0]) == 2.0 * world
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("split", [(0, 6, 13), (0, 1, 13), (0, 12, 13)])
def test_time_sharded_combines_gloo(split):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, split, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_last_observed_single_process():
    from paper_2506_19656_b200.dist import last_observed

    s = torch.tensor([[[1.0, np.nan, np.nan], [np.nan, 2.0, np.nan], [3.0, np.nan, np.nan]]])
    out = last_observed(s)
    assert out[0, 0] == 3.0 and out[0, 1] == 2.0 and torch.isnan(out[0, 2])
