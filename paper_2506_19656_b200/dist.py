"""Multi-GPU sharding of one cube along time (one process per GPU).

north_star: "Work is sharded along the time axis across the GPUs of one
8xB200 box, and only the per-band statistics, the C x C Gram partials and the
metric partial sums are combined" (BASELINE.json). Rank r holds the contiguous
time slice [t_r, t_{r+1}) of the cube. The exchanges, all tiny next to the
cube (NCCL over NVLink with backend "nccl"; gloo in the CPU tests):

  1. band stats      all_reduce MAX over [max, -min] (2C f64), SUM of NaN
                     counts, MAX of the leading-gap flag (rank 0's only: a
                     leading gap can only start at global t = 0);
  2. fill carries    all_gather of each rank's last-observed map [HW*C] f32
                     (only for float cubes with the fill policy); rank r takes,
                     per element, the last observation of ranks < r;
  3. PCA Gram        all_gather of (shift, sums, Gram, n) (C + C*C + 1 f64);
                     every rank re-centres them on rank 0's shift in float64
                     and runs the same eigh -> identical models everywhere;
  4. PC ranges       all_reduce as in 1 (2K f64);
  5. metrics         all_reduce SUM of the per-band SSE and SSIM sums (2C f64).

Frames are whole per t, so SSIM needs no spatial halo exchange. The combine
functions below are pure torch + torch.distributed and run on any backend.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _device as dev
from . import _lib


class TimeShard:
    """This process's place in a time-sharded cube."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        # gloo (CPU tests, or ranks sharing one GPU) moves CUDA tensors via the host
        self.host_staging = dist.is_initialized() and dist.get_backend(group) == "gloo"

    # -------------------------------------------------------------- collectives
    def all_reduce(self, t: torch.Tensor, op=dist.ReduceOp.SUM) -> torch.Tensor:
        if self.world > 1:
            if self.host_staging and t.is_cuda:
                h = t.cpu()
                dist.all_reduce(h, op=op, group=self.group)
                t.copy_(h)
            else:
                dist.all_reduce(t, op=op, group=self.group)
        return t

    def all_gather(self, t: torch.Tensor) -> list:
        if self.world == 1:
            return [t]
        src = t.contiguous()
        if self.host_staging and src.is_cuda:
            h = src.cpu()
            out = [torch.empty_like(h) for _ in range(self.world)]
            dist.all_gather(out, h, group=self.group)
            return [o.to(t.device) for o in out]
        out = [torch.empty_like(src) for _ in range(self.world)]
        dist.all_gather(out, src, group=self.group)
        return out

    # -------------------------------------------------------------- combines
    def combine_minmax(self, mins: torch.Tensor, maxs: torch.Tensor):
        """Global per-band min/max (bands a rank never observed carry +/-inf)."""
        n = mins.numel()
        t = torch.cat([maxs.reshape(-1), -mins.reshape(-1)]).to(torch.float64)
        self.all_reduce(t, dist.ReduceOp.MAX)
        return (-t[n:]).reshape(mins.shape), t[:n].reshape(maxs.shape)

    def combine_band_stats(self, mins, maxs, lead, nans, fill: float):
        """Raw local stats -> global fit_quant ranges with the leading-fill rule."""
        gmins, gmaxs = self.combine_minmax(mins, maxs)
        lead = lead.to(torch.int64) if self.rank == 0 else torch.zeros_like(lead, dtype=torch.int64)
        self.all_reduce(lead, dist.ReduceOp.MAX)
        nans = nans.to(torch.int64).clone()
        self.all_reduce(nans)
        f = float(np.float32(fill))
        has = lead > 0
        gmins = torch.where(has, torch.clamp(gmins, max=f), gmins)
        gmaxs = torch.where(has, torch.clamp(gmaxs, min=f), gmaxs)
        return gmins, gmaxs, nans

    def carry_in(self, last_map: torch.Tensor) -> torch.Tensor:
        """Per element, the last observation made by ranks < this one (NaN if none)."""
        maps = self.all_gather(last_map)
        carry = torch.full_like(last_map, float("nan"))
        for r in range(self.rank):
            m = maps[r]
            carry = torch.where(torch.isnan(m), carry, m)
        return carry

    def combine_gram(self, shift: torch.Tensor, out: torch.Tensor, n: int, C: int):
        """Re-centre every rank's shifted sums on rank 0's shift (float64, host)."""
        pack = torch.cat([shift.double().reshape(-1), out.double().reshape(-1),
                          torch.tensor([float(n)], dtype=torch.float64, device=out.device)])
        parts = [p.cpu().numpy() for p in self.all_gather(pack)]
        s0 = parts[0][:C]
        S = np.zeros(C)
        G = np.zeros((C, C))
        N = 0.0
        for p in parts:
            s_r, o_r, n_r = p[:C], p[C:C + C + C * C], p[-1]
            S_r, G_r = o_r[:C], o_r[C:].reshape(C, C)
            dlt = s_r - s0
            # sum (x - s0) = S_r + n_r d ; sum (x-s0)(x-s0)^T = G_r + d S_r^T + S_r d^T + n_r d d^T
            G += G_r + np.outer(dlt, S_r) + np.outer(S_r, dlt) + n_r * np.outer(dlt, dlt)
            S += S_r + n_r * dlt
            N += n_r
        return s0, np.concatenate([S, G.reshape(-1)]), int(round(N))

    def combine_flags(self, flags: int) -> int:
        """OR of every rank's device error flags (CV_FLAG_*), so that all ranks
        take the same branch (fill first, or raise together) instead of one rank
        raising while the others wait in a later collective."""
        bits = torch.tensor([(flags >> i) & 1 for i in range(8)], dtype=torch.int64)
        if not self.host_staging:
            bits = bits.to(torch.device("cuda", torch.cuda.current_device()))
        self.all_reduce(bits, dist.ReduceOp.MAX)
        return int(sum(int(b) << i for i, b in enumerate(bits.cpu().tolist())))

    def combine_scores(self, sse: torch.Tensor, ssim_sum: torch.Tensor):
        t = torch.cat([sse.reshape(-1), ssim_sum.reshape(-1)]).to(torch.float64)
        self.all_reduce(t)
        k = sse.numel()
        return t[:k].reshape(sse.shape), t[k:].reshape(ssim_sum.shape)


def last_observed(seg_last: torch.Tensor) -> torch.Tensor:
    """[B][n_seg][inner] per-segment last observations -> [B][inner] last overall."""
    valid = ~torch.isnan(seg_last)
    nseg = seg_last.shape[1]
    pos = torch.arange(1, nseg + 1, device=seg_last.device, dtype=torch.int32).view(1, nseg, 1)
    last = (valid.to(torch.int32) * pos).amax(dim=1)  # 1-based index of the last valid segment
    idx = (last - 1).clamp(min=0).to(torch.int64).unsqueeze(1)
    val = torch.gather(seg_last, 1, idx).squeeze(1)
    return torch.where(last > 0, val, torch.full_like(val, float("nan")))


def raw_band_stats(x: dev.Arr, B: int, T: int, inner: int, C: int, fill_mode: int, seg_len: int,
                   err: dev.ErrWord, seg_last: torch.Tensor | None):
    """K1 without the leading-fill adjustment: (mins, maxs, lead, nans) of this shard."""
    d = x.device
    lib = _lib.load()
    s = dev.stream_ptr(d)
    ws = dev.workspace(lib.cv_stats_ws_bytes(B, C), d)
    _lib.call("cv_stats_reset", ws.data_ptr(), B, C, s)
    _lib.call("cv_stats", x.ptr, x.code, B, T, inner, C, fill_mode, seg_len, ws.data_ptr(),
              seg_last.data_ptr() if seg_last is not None else None, err.ptr, s)
    mins = torch.empty((B, C), dtype=torch.float64, device=d)
    maxs = torch.empty_like(mins)
    nans = torch.empty((B, C), dtype=torch.int64, device=d)
    _lib.call("cv_stats_finalize", ws.data_ptr(), B, C, 0, 0.0, mins.data_ptr(), maxs.data_ptr(),
              nans.data_ptr(), s)
    lead = torch.empty((B, C), dtype=torch.int32, device=d)
    _lib.call("cv_stats_lead_flags", ws.data_ptr(), B, C, lead.data_ptr(), s)
    return mins, maxs, lead, nans
