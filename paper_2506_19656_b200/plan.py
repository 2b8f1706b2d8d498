"""Frame packing plan: ``ChannelGroup`` / ``pack_groups`` / ``plan_stream`` of
/root/reference/pkg/src/cubevid/plan.py:95-139 (host bookkeeping; the kernels
write the planes this plan describes)."""

from __future__ import annotations

import math
from dataclasses import dataclass

from .errors import ConfigurationError


@dataclass(frozen=True)
class ChannelGroup:
    """Three channel slots of one output video; padding repeats the last real channel."""

    video_index: int
    members: tuple
    n_real: int

    def __post_init__(self):
        if not 1 <= self.n_real <= 3:
            raise ConfigurationError("a group carries 1 to 3 real channels")
        real = tuple(self.members[: self.n_real])
        if tuple(self.members) != real + (real[-1],) * (3 - self.n_real):
            raise ConfigurationError("padding slots must repeat the group's last real channel")


def pack_groups(n_channels: int) -> list:
    """ceil(n/3) groups of three channel slots, last group padded by repetition."""
    if n_channels < 1:
        raise ConfigurationError("cannot plan a stream with zero channels")
    out = []
    for g in range(math.ceil(n_channels / 3)):
        first = 3 * g
        real = tuple(range(first, min(first + 3, n_channels)))
        out.append(ChannelGroup(g + 1, real + (real[-1],) * (3 - len(real)), len(real)))
    return out


def plan_stream(n_pcs: int, n_channels: int) -> list:
    """Groups of a stream; with PCA the encoded channels are the kept components."""
    return pack_groups(n_pcs if n_pcs > 0 else n_channels)


def video_names(stream_name: str, groups) -> tuple:
    return tuple(f"{stream_name}_{g.video_index:04d}" for g in groups)
