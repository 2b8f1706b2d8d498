"""Frame packing plan: ``ChannelGroup`` / ``pack_groups`` / ``plan_stream`` of
/root/reference/pkg/src/cubevid/plan.py:95-139 (host bookkeeping; the kernels
write the planes this plan describes), plus the array-side fields of
``MappingRule`` (plan.py:26-66)."""

from __future__ import annotations

import math
from dataclasses import dataclass, field

from .errors import ConfigurationError

_BIT_DEPTHS = (8, 10, 12, 16)


@dataclass(frozen=True)
class MappingRule:
    """Recipe of one output stream (plan.py:26-66). ``codec_config`` is carried
    as plain data: resolving it belongs to the codec layer, outside this path."""

    stream_name: str
    input_vars: tuple
    axis_order: tuple
    n_pcs: int = 0
    codec_config: dict | list = field(default_factory=dict)
    out_bit_depth: int = 12
    fill_value_for_leading: float = 0.0
    monochrome: bool = False

    def __post_init__(self):
        names = (self.input_vars,) if isinstance(self.input_vars, str) else tuple(self.input_vars)
        object.__setattr__(self, "input_vars", names)
        object.__setattr__(self, "axis_order", tuple(self.axis_order))
        if not self.stream_name:
            raise ConfigurationError("stream name must be non-empty")
        who = f"stream {self.stream_name!r}"
        if not names:
            raise ConfigurationError(f"{who} selects no variables")
        if len(self.axis_order) != 3:
            raise ConfigurationError(f"{who}: axis_order must name the (time, y, x) roles, "
                                     f"got {self.axis_order}")
        if self.n_pcs < 0:
            raise ConfigurationError(f"{who}: n_pcs must be >= 0")
        if self.out_bit_depth not in _BIT_DEPTHS:
            raise ConfigurationError(f"{who}: bit depth {self.out_bit_depth} not one of 8, 10, 12, 16")

    @property
    def config_is_list(self) -> bool:
        return isinstance(self.codec_config, (list, tuple))


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


def plan_stream(rule, n_channels: int) -> list:
    """Groups of a stream (plan.py:131-139); with PCA the encoded channels are the
    kept components. ``rule`` is a MappingRule (the reference's, or the one above:
    anything with ``n_pcs``); a bare component count is accepted too."""
    n_pcs = rule if isinstance(rule, int) else rule.n_pcs
    return pack_groups(n_pcs if n_pcs > 0 else n_channels)


def video_names(stream_name: str, groups) -> tuple:
    return tuple(f"{stream_name}_{g.video_index:04d}" for g in groups)
