"""Host-side plumbing between ranks: handle exchange and shape agreement.

Replaces the reference's coordinator JSON lines (pkg/src/ringbox/runtime.py:
140-156, 496-553) and the peer plan-hash handshake (runtime.py:124-126,
374-386).  Everything here is small host metadata exchanged once per
buffer/shape over torch.distributed (gloo or nccl); no data-path traffic ever
goes through it.  Testable on CPU with the gloo backend (tests/test_exchange.py).
"""

from __future__ import annotations

import hashlib
import json

from .errors import CollectiveError


def allgather_objects(obj, group=None) -> list:
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return [obj]
    world = dist.get_world_size(group)
    if world == 1:
        return [obj]
    out = [None] * world
    dist.all_gather_object(out, obj, group=group)
    return out


def plan_fingerprint(dims, dtype: str, lengths) -> int:
    """Same fingerprint construction as the reference (runtime.py:124-126)."""
    blob = json.dumps([list(dims), dtype, list(lengths)]).encode()
    return int.from_bytes(hashlib.sha256(blob).digest()[:8], "little")


def agree(key, group=None, what: str = "shape") -> list:
    """Every rank contributes `key`; raise CollectiveError naming the first
    disagreeing rank unless all keys are equal (runtime.py:528-543)."""
    keys = allgather_objects(key, group)
    ref = keys[0]
    bad = [r for r, k in enumerate(keys) if k != ref]
    if bad:
        detail = ", ".join(f"rank {r} advertises {keys[r]!r}" for r in bad)
        raise CollectiveError(f"{what} mismatch: {detail} (rank 0 has {ref!r})", rank=bad[0])
    return keys
