"""Ring schedules as data (metadata only -- no data movement here).

API of pkg/src/ringbox/ring.py: `chunk_bounds` (57-70), `ring_pass_transfers`
(73-103), the single-ring reduce-scatter/allgather/allreduce schedules
(106-140), depth-first ring ordering on a topology tree (143-158) and the
`dump_schedule` listing (195-203).  On B200 these schedules are *not*
executed phase by phase: the runtime turns them into per-rank step tables
(paper_1708_02188_b200/csrc/rbx_plan.cpp) that fold whole chunks in one pass
with the same chunk boundaries and the same reduction order.
"""

from __future__ import annotations

from dataclasses import dataclass

from .topology import Topology

ADD = "add"
REPLACE = "replace"


@dataclass(frozen=True)
class Transfer:
    src: int
    dst: int
    chunk_index: int
    offset: int
    length: int
    combine: str


@dataclass(frozen=True)
class Phase:
    transfers: tuple


@dataclass(frozen=True)
class Schedule:
    ranks: int
    element_count: int
    phases: tuple
    kind: str


@dataclass(frozen=True)
class RingOrder:
    devices: tuple

    def __len__(self) -> int:
        return len(self.devices)

    def position_of(self, device: str) -> int:
        return self.devices.index(device)


def chunk_bounds(element_count: int, n_chunks: int, index: int) -> tuple[int, int]:
    """(offset, length) of chunk `index` when [0, element_count) is cut into
    n_chunks contiguous pieces, the first (count mod n) one element longer."""
    if n_chunks < 1:
        raise ValueError(f"n_chunks must be >= 1, got {n_chunks}")
    if not 0 <= index < n_chunks:
        raise ValueError(f"chunk index {index} out of range [0, {n_chunks})")
    small, extra = divmod(element_count, n_chunks)
    offset = index * small + min(index, extra)
    return offset, small + (1 if index < extra else 0)


def ring_pass_transfers(members: list, region_offset: int, region_length: int, kind: str) -> list:
    """Transfers of one ring pass, grouped by phase.  In reduce-scatter phase j
    the member at position p sends chunk (p - j) mod d to its successor (ADD),
    so position p ends up owning chunk (p + 1) mod d; allgather starts from that
    ownership and forwards chunk (p + 1 - j) mod d (REPLACE)."""
    d = len(members)
    rs = kind == "reduce_scatter"
    phases = []
    for j in range(d - 1):
        row = []
        for p, rank in enumerate(members):
            c = (p - j) % d if rs else (p + 1 - j) % d
            off, length = chunk_bounds(region_length, d, c)
            row.append(Transfer(rank, members[(p + 1) % d], c, region_offset + off, length, ADD if rs else REPLACE))
        phases.append(row)
    return phases


def _single_ring(order: RingOrder, element_count: int, kinds: tuple, label: str) -> Schedule:
    n = len(order)
    if n < 1:
        raise ValueError("ring needs at least one member")
    phases = []
    for kind in kinds:
        phases += [Phase(tuple(row)) for row in ring_pass_transfers(list(range(n)), 0, element_count, kind)]
    return Schedule(n, element_count, tuple(phases), label)


def reduce_scatter_schedule(order: RingOrder, element_count: int) -> Schedule:
    return _single_ring(order, element_count, ("reduce_scatter",), "reduce_scatter")


def allgather_schedule(order: RingOrder, element_count: int) -> Schedule:
    return _single_ring(order, element_count, ("allgather",), "allgather")


def allreduce_schedule(order: RingOrder, element_count: int) -> Schedule:
    return _single_ring(order, element_count, ("reduce_scatter", "allgather"), "composite")


def order_ranks_on_tree(t: Topology, devices: list) -> RingOrder:
    """Depth-first leaf order: every subtree is one contiguous arc of the ring."""
    for dev in devices:
        if dev not in t.nodes:
            raise ValueError(f"unknown device '{dev}'")
        if not t.is_leaf(dev) or t.nodes[dev].kind != "device":
            raise ValueError(f"'{dev}' is not a device leaf")
    wanted = set(devices)
    return RingOrder(tuple(leaf for leaf in t.dfs_leaves() if leaf in wanted))


def dump_schedule(schedule: Schedule) -> str:
    """`phase src dst chunk offset length combine`, one transfer per line."""
    rows = [
        f"{i} {t.src} {t.dst} {t.chunk_index} {t.offset} {t.length} {t.combine}"
        for i, ph in enumerate(schedule.phases)
        for t in ph.transfers
    ]
    return "".join(r + "\n" for r in rows)
