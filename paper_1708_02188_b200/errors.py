"""Exception types shared by the runtime and the native binding."""

from __future__ import annotations


class CollectiveError(RuntimeError):
    """A collective failed; carries the offending rank and plan step when known
    (same shape as pkg/src/ringbox/runtime.py:42-48)."""

    def __init__(self, message: str, rank: int | None = None, phase: int | None = None):
        self.rank = rank
        self.phase = phase
        super().__init__(message)
