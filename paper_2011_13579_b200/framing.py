"""Overlapping-window plan of a long stream (framing.py:21-83 of the reference).

Windows are computed in closed form; ``FramePlan.windows`` is a lazy
sequence, so planning 2^20 windows costs nothing (the reference builds one
Python object per window: 3.8 s at 2^20).
"""
from __future__ import annotations

import json
from collections.abc import Sequence
from dataclasses import dataclass

__all__ = ["Window", "FramePlan", "plan_frames", "DEFAULT_FRAME_LEN", "DEFAULT_OVERLAP"]

DEFAULT_FRAME_LEN = 256
DEFAULT_OVERLAP = 64


@dataclass(frozen=True)
class Window:
    start: int
    stop: int
    emit_start: int
    emit_stop: int

    @property
    def length(self) -> int:
        return self.stop - self.start


class _Windows(Sequence):
    """Window k: emit [kF, min((k+1)F, N)), span [max(0, emit_start-V), min(N, emit_stop+V))."""

    def __init__(self, n: int, f: int, v: int):
        self._n, self._f, self._v = n, f, v
        self._len = -(-n // f)

    def __len__(self) -> int:
        return self._len

    def __getitem__(self, k):
        if isinstance(k, slice):
            return tuple(self[i] for i in range(*k.indices(self._len)))
        if k < 0:
            k += self._len
        if not 0 <= k < self._len:
            raise IndexError(k)
        e0 = k * self._f
        e1 = min(e0 + self._f, self._n)
        return Window(max(0, e0 - self._v), min(self._n, e1 + self._v), e0, e1)

    def __eq__(self, other) -> bool:
        return tuple(self) == tuple(other)

    def __hash__(self) -> int:
        return hash((self._n, self._f, self._v))


@dataclass(frozen=True)
class FramePlan:
    total_stages: int
    frame_len: int
    overlap: int
    windows: Sequence[Window]

    def survivor_memory_estimate(self, spec) -> float:
        """Order-of-magnitude survivor storage in units of one entry (framing.py:45-47)."""
        return spec.num_states * self.total_stages * (1.0 + self.overlap / self.frame_len)

    def to_json(self) -> str:
        return json.dumps(
            {
                "total_stages": self.total_stages,
                "frame_len": self.frame_len,
                "overlap": self.overlap,
                "windows": [
                    {"start": w.start, "stop": w.stop, "emit_start": w.emit_start, "emit_stop": w.emit_stop}
                    for w in self.windows
                ],
            },
            indent=2,
        )


def plan_frames(total_stages: int, frame_len: int = DEFAULT_FRAME_LEN, overlap: int = DEFAULT_OVERLAP) -> FramePlan:
    """framing.py:68-83 plan_frames (same validation, closed-form windows)."""
    if total_stages < 1:
        raise ValueError("stream must have at least one stage")
    if frame_len < 1:
        raise ValueError("frame length must be >= 1")
    if overlap < 0:
        raise ValueError("overlap must be >= 0")
    return FramePlan(int(total_stages), int(frame_len), int(overlap),
                     _Windows(int(total_stages), int(frame_len), int(overlap)))
