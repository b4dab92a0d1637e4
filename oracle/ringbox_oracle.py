"""CPU ORACLE for the multi-ring allreduce -- TEST INFRASTRUCTURE ONLY.

This module is a plain numpy restatement of the reference `ringbox` package's
hot-path semantics (reference: /root/reference/pkg/src/ringbox, v0.1.0).  It
is the *checker*: only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
CPU-baseline / `--impl reference` legs may import it.  The product package
(`paper_1708_02188_b200`) never imports, links or executes anything here.

Parity pinning: every function below is checked in `tests/test_oracle.py`
against the golden fixtures in `tests/golden/`, which were produced by
importing the reference itself (`tests/golden/make_golden.py`).  The
restatement is therefore pinned, not free-standing.

Functions and the reference code they restate:

* `chunk_bounds`          -- pkg/src/ringbox/ring.py:57-70 (remainder-first split)
* `Grid`                  -- pkg/src/ringbox/multiring.py:21-55 (mixed radix, dim 0 fastest)
* `ring_pass_transfers`   -- pkg/src/ringbox/ring.py:73-103
* `multiring_schedule`    -- pkg/src/ringbox/multiring.py:170-211
* `replay`                -- pkg/src/ringbox/ring.py:172-192 (phase-synchronous executor)
* `owned_region`          -- pkg/src/ringbox/runtime.py:187-196
* `generate_input`        -- pkg/src/ringbox/runtime.py:94-100
* `closed_form_allreduce` -- the nested rotated left fold that `replay` is
  equivalent to; vectorised so large buffers
  (25.6 M x 8) check in seconds.  Cross-checked against `replay` in tests.
* `bf16_allreduce`        -- bf16 policy (reference has no bf16,
  pkg/src/ringbox/runtime.py:37): replay over fp32-upcast inputs, one RNE to
  bf16 at the end (parity for bf16 is therefore *unpinned* by the reference).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

DTYPES = {"f32": np.float32, "f64": np.float64, "i64": np.int64}


def chunk_bounds(count: int, n: int, i: int) -> tuple[int, int]:
    # ring.py:57-70 -- the first (count mod n) chunks get one extra element.
    if n < 1 or not 0 <= i < n:
        raise ValueError("bad chunk request")
    q, r = divmod(count, n)
    if i < r:
        return i * (q + 1), q + 1
    return r * (q + 1) + (i - r) * q, q


@dataclass(frozen=True)
class Grid:
    # multiring.py:21-55
    dims: tuple

    @property
    def size(self) -> int:
        return int(np.prod(self.dims)) if self.dims else 1

    def coords(self, rank: int) -> tuple:
        out = []
        for d in self.dims:
            out.append(rank % d)
            rank //= d
        return tuple(out)

    def rank_of(self, coords) -> int:
        r, s = 0, 1
        for c, d in zip(coords, self.dims):
            r += c * s
            s *= d
        return r

    def rings(self, dim: int) -> list:
        groups: dict = {}
        for r in range(self.size):
            c = self.coords(r)
            groups.setdefault(c[:dim] + c[dim + 1:], []).append(r)
        return [sorted(g, key=lambda x: self.coords(x)[dim]) for g in groups.values()]


# A transfer is (src, dst, chunk, offset, length, is_add).
def ring_pass_transfers(members, off, length, kind):
    # ring.py:73-103: RS phase j: position p sends chunk (p-j) mod d; AG: (p+1-j) mod d.
    d = len(members)
    phases = []
    for j in range(d - 1):
        ts = []
        for p, rank in enumerate(members):
            c = (p - j) % d if kind == "rs" else (p + 1 - j) % d
            o, l = chunk_bounds(length, d, c)
            ts.append((rank, members[(p + 1) % d], c, off + o, l, kind == "rs"))
        phases.append(ts)
    return phases


def multiring_schedule(grid: Grid, count: int) -> list:
    # multiring.py:170-211: RS over dims 0..m-1 on a shrinking region, AG over m-1..0.
    n = grid.size
    region = {r: (0, count) for r in range(n)}
    saved = []
    phases = []
    for dim, d in enumerate(grid.dims):
        saved.append(dict(region))
        if d == 1:
            continue
        per = [[] for _ in range(d - 1)]
        for members in grid.rings(dim):
            off, length = region[members[0]]
            for j, ts in enumerate(ring_pass_transfers(members, off, length, "rs")):
                per[j].extend(ts)
            for p, rank in enumerate(members):
                o, l = chunk_bounds(length, d, (p + 1) % d)
                region[rank] = (off + o, l)
        phases.extend(per)
    for dim in range(len(grid.dims) - 1, -1, -1):
        d = grid.dims[dim]
        if d == 1:
            continue
        per = [[] for _ in range(d - 1)]
        for members in grid.rings(dim):
            off, length = saved[dim][members[0]]
            for j, ts in enumerate(ring_pass_transfers(members, off, length, "ag")):
                per[j].extend(ts)
        phases.extend(per)
    return phases


def replay(phases: list, buffers: list) -> list:
    # ring.py:172-192: every payload is staged from the pre-phase state, then applied.
    bufs = [np.array(b, copy=True) for b in buffers]
    for ph in phases:
        staged = [(t, bufs[t[0]][t[3]:t[3] + t[4]].copy()) for t in ph]
        for t, payload in staged:
            view = bufs[t[1]][t[3]:t[3] + t[4]]
            if t[5]:
                view += payload
            else:
                view[:] = payload
    return bufs


def owned_region(grid: Grid, rank: int, count: int) -> tuple[int, int]:
    # runtime.py:187-196
    off, length = 0, count
    for c, d in zip(grid.coords(rank), grid.dims):
        if d == 1:
            continue
        o, l = chunk_bounds(length, d, (c + 1) % d)
        off, length = off + o, l
    return off, length


def generate_input(seed: int, iteration: int, rank: int, length: int, dtype: str) -> np.ndarray:
    # runtime.py:94-100 (Workload(seed=...) -> generate_input(w, it, rank, length))
    rng = np.random.default_rng(seed * 100003 + iteration * 1009 + rank)
    if dtype == "i64":
        return rng.integers(-1000, 1001, size=length, dtype=np.int64)
    return rng.standard_normal(length).astype(DTYPES[dtype])


def sha256(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fold_order(grid: Grid, rank: int) -> list:
    """Ranks in the order the nested left fold visits them for `rank`'s owned
    region (dim 0 innermost; each dim's fold starts at the chunk index
    k_i = (c_i + 1) mod d_i and wraps, so the owner's own value is added last
    at every level).  Derived from ring.py:73-103 + multiring.py:170-211."""
    dims = list(grid.dims)
    ks = [(c + 1) % d for c, d in zip(grid.coords(rank), dims)]
    order = []

    def rec(level, outer):
        if level < 0:
            order.append(grid.rank_of(tuple(outer)))
            return
        d = dims[level]
        for j in range(d):
            outer[level] = (ks[level] + j) % d
            rec(level - 1, outer)

    rec(len(dims) - 1, [0] * len(dims))
    return order


def _nested_fold(vals: list, dims: list):
    """Left fold of `vals` (already in visit order) nested by dims (dim 0 innermost)."""
    level = list(vals)
    for d in dims:
        nxt = []
        for g in range(0, len(level), d):
            acc = level[g].copy()
            for v in level[g + 1:g + d]:
                acc += v
            nxt.append(acc)
        level = nxt
    return level[0]


def closed_form_allreduce(grid: Grid, buffers: list) -> np.ndarray:
    """Vectorised equivalent of replay(multiring_schedule(grid, n), buffers)[r]
    (identical on all ranks).  See SURVEY.md Appendix A.1/A.11."""
    n = len(buffers[0])
    out = np.empty_like(buffers[0])
    with np.errstate(over="ignore"):
        for r in range(grid.size):
            off, length = owned_region(grid, r, n)
            if length == 0:
                continue
            order = fold_order(grid, r)
            vals = [buffers[q][off:off + length] for q in order]
            out[off:off + length] = _nested_fold(vals, [d for d in grid.dims])
    return out


def bf16_round(x32: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bits (uint16), round-to-nearest-even (NaN kept quiet)."""
    u = x32.astype(np.float32).view(np.uint32).astype(np.uint64)
    nan = np.isnan(x32)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    rounded[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return rounded


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def bf16_allreduce(grid: Grid, buffers_bf16_bits: list) -> np.ndarray:
    """bf16 policy: fold fp32-upcast inputs in the reference order, round once."""
    up = [bf16_to_f32(b) for b in buffers_bf16_bits]
    return bf16_round(closed_form_allreduce(grid, up))


def f16_allreduce(grid: Grid, buffers_f16: list) -> np.ndarray:
    up = [b.astype(np.float32) for b in buffers_f16]
    return closed_form_allreduce(grid, up).astype(np.float16)


def factorizations(n: int, max_dims: int) -> list:
    # multiring.py:141-159 (ordered factor tuples, entries >= 2, plus (n,))
    found = {(n,)}

    def rec(rest, prefix):
        if rest == 1 and prefix:
            found.add(prefix)
            return
        if len(prefix) == max_dims:
            return
        for f in range(2, rest + 1):
            if rest % f == 0:
                rec(rest // f, prefix + (f,))

    rec(n, ())
    return sorted(found)
