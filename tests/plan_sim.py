"""Test-only CPU simulator of librbx's per-rank step tables.

Executes the plans produced by the native plan builder (rbx_plan_describe)
with `nb` simulated CTAs per rank, interleaved in a random order, honouring
exactly the kernel's wait/signal semantics (MATCHED = same block index, ALL =
every block of the peer).  Used to check on CPU that the tables (a) compute
the reference's reduction order bit-for-bit and (b) carry every dependency
(a missing wait shows up as a wrong result under some interleaving, or as a
deadlock)."""

from __future__ import annotations

import random

import numpy as np

from paper_1708_02188_b200 import _native


def _fold(vals, ctrl, nlev):
    acc = [None] * 4
    for x, c in zip(vals, ctrl):
        up = c >> 4
        acc[0] = x.copy() if c & 1 else acc[0] + x
        for L in range(1, nlev):
            if up >= L:
                acc[L] = acc[L - 1].copy() if c & (1 << L) else acc[L] + acc[L - 1]
    return acc[nlev - 1]


def simulate(dims, bufs, op="allreduce", mode="fused", nb=3, seed=0, dtype="f32"):
    n = len(bufs)
    count = len(bufs[0])
    plans = [_native.parse_plan(_native.plan_describe(dims, r, count, op, mode, dtype)) for r in range(n)]
    bufs = [b.copy() for b in bufs]
    inbox = {}  # MODE_PUSH: (owner, slot) -> element-offset-addressed array

    def resolve(me, idx):
        """Pointer-table entry -> array (rbx_plan.h table_entries layout)."""
        if idx < n:
            return bufs[idx]
        key = (me, idx - n) if idx < 2 * n else (idx - 2 * n, me)
        if key not in inbox:
            inbox[key] = np.full(count, np.nan if bufs[0].dtype.kind == "f" else -7, dtype=bufs[0].dtype)
        return inbox[key]

    flags = {}  # (dst_rank, slot, src_rank, block) -> 1
    pos = {(r, b): -1 for r in range(n) for b in range(nb)}  # -1: entry not yet signalled
    rng = random.Random(seed)
    units = list(pos)
    done = set()
    while len(done) < len(units):
        runnable = []
        for u in units:
            if u in done:
                continue
            r, b = u
            s = pos[u]
            if s == -1:
                runnable.append(u)
                continue
            st = plans[r]["steps"][s]
            ok = True
            for w in st["waits"]:
                blocks = range(nb) if w["all"] else [b]
                if not all(flags.get((r, w["slot"], w["peer"], k)) for k in blocks):
                    ok = False
                    break
            if ok:
                runnable.append(u)
        if not runnable:
            raise RuntimeError(f"deadlock: positions {pos}")
        u = rng.choice(runnable)
        r, b = u
        s = pos[u]
        if s == -1:
            for q in plans[r]["entry"]:
                flags[(q, 0, r, b)] = 1
        else:
            st = plans[r]["steps"][s]
            total = sum(sg["len"] for sg in st["segs"])
            lo, hi = total * b // nb, total * (b + 1) // nb
            base = 0
            for sg in st["segs"]:
                a, z = max(lo, base), min(hi, base + sg["len"])
                if a < z:
                    o0, o1 = sg["off"] + a - base, sg["off"] + z - base
                    vals = [resolve(r, q)[o0:o1] for q in sg["src"]]
                    res = vals[0].copy() if len(vals) == 1 else _fold(vals, sg["ctrl"], sg["nlev"])
                    for q in sg["dst"]:
                        resolve(r, q)[o0:o1] = res
                base += sg["len"]
            for q in st["sigs"]:
                flags[(q, s + 1, r, b)] = 1
        pos[u] = s + 1
        if pos[u] >= len(plans[r]["steps"]):
            done.add(u)
    return bufs
