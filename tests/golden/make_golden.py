"""Generate the committed golden fixtures by importing the REFERENCE package.

Run ONLY in the build container (the reference is mounted read-only at
/root/reference and does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every fixture is produced by the reference's own code -- `ringbox.ring.replay`
over `ringbox.multiring.multiring_schedule` (pkg/src/ringbox/ring.py:172-192,
pkg/src/ringbox/multiring.py:170-211), the reference runtime `launch`
(pkg/src/ringbox/runtime.py:435-589), the planner `plan`
(pkg/src/ringbox/multiring.py:278-318) and friends -- on the inputs of
`generate_input` (pkg/src/ringbox/runtime.py:94-100).  The tests compare the
oracle restatement (oracle/) and the GPU path against these files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

from ringbox import costmodel, topology  # noqa: E402
from ringbox.multiring import Grid, build_grid, factorizations, multiring_schedule, plan, ring_partner_pairs  # noqa: E402
from ringbox.ring import (  # noqa: E402
    RingOrder,
    allreduce_schedule,
    chunk_bounds,
    dump_schedule,
    reduce_scatter_schedule,
    replay,
)
from ringbox.runtime import Workload, generate_input, launch, owned_region  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
RANK_COUNTS = (1, 2, 3, 4, 6, 8, 12, 16)
LENGTHS = (0, 1, 17, 1000, 4099)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def dims_key(dims) -> str:
    return "x".join(str(d) for d in dims)


def chunk_kats():
    out = []
    for count in (0, 1, 3, 7, 8, 10, 17, 100, 1001):
        for n in (1, 2, 3, 4, 5, 8):
            for i in range(n):
                out.append([count, n, i, *chunk_bounds(count, n, i)])
    return out


def schedule_dumps():
    out = {}
    for dims, count in [((2,), 10), ((4,), 10), ((2, 2), 9), ((2, 4), 19), ((2, 2, 2), 23),
                        ((3, 2), 11), ((1, 4), 12), ((2, 1, 3), 13)]:
        out[f"{dims_key(dims)}:{count}"] = dump_schedule(multiring_schedule(Grid(dims=dims), count))
    out["rs_ring2:10"] = dump_schedule(reduce_scatter_schedule(RingOrder(devices=("a", "b")), 10))
    return out


def owned_regions():
    out = {}
    counts = (0, 1, 17, 1000, 4099, 25_600_000, 25_557_032, 6_250_000)
    for n in RANK_COUNTS:
        for dims in factorizations(n, 3):
            g = build_grid(n, dims)
            for count in counts:
                out[f"{dims_key(dims)}:{count}"] = [list(owned_region(g, r, count)) for r in range(n)]
    for dims in [(1, 4), (2, 1, 3), (2, 2, 2, 2)]:
        g = Grid(dims=dims)
        for count in counts:
            out[f"{dims_key(dims)}:{count}"] = [list(owned_region(g, r, count)) for r in range(g.size)]
    return out


def replay_digests():
    """sha256 of replay(...)[r] for Workload(lengths=LENGTHS, dtype, seed=N)."""
    out = {}
    extra_dims = {4: [(1, 4)], 6: [(2, 1, 3)], 16: [(2, 2, 2, 2)]}
    for n in RANK_COUNTS:
        for dims in list(factorizations(n, 3)) + extra_dims.get(n, []):
            g = build_grid(n, dims)
            for dtype in ("i64", "f32", "f64"):
                w = Workload(lengths=LENGTHS, dtype=dtype, seed=n)
                for it, length in enumerate(LENGTHS):
                    parts = [generate_input(w, it, r, length) for r in range(n)]
                    res = replay(multiring_schedule(g, length), [p.copy() for p in parts])
                    digs = {sha(x) for x in res}
                    assert len(digs) == 1, (n, dims, dtype, length)
                    out[f"{dims_key(dims)}:{dtype}:{it}:{length}"] = sha(res[0])
    return out


def input_digests():
    """Pins generate_input itself (numpy default_rng stream) for the inputs used above."""
    out = {}
    for dtype in ("i64", "f32", "f64"):
        w = Workload(lengths=LENGTHS, dtype=dtype, seed=8)
        for it, length in enumerate(LENGTHS):
            for r in range(8):
                out[f"{dtype}:8:{it}:{r}"] = sha(generate_input(w, it, r, length))
    return out


def small_vectors():
    """Full input/output vectors for a few small cases (for eyeballing and KATs)."""
    out = []
    for dims, dtype, length, seed in [((2, 2), "f32", 17, 3), ((2, 4), "f32", 37, 0),
                                      ((2, 2, 2), "f64", 29, 1), ((3, 2), "i64", 13, 5),
                                      ((8,), "f32", 19, 2)]:
        g = Grid(dims=dims)
        w = Workload(lengths=(length,), dtype=dtype, seed=seed)
        parts = [generate_input(w, 0, r, length) for r in range(g.size)]
        res = replay(multiring_schedule(g, length), [p.copy() for p in parts])[0]
        out.append({
            "dims": list(dims), "dtype": dtype, "length": length, "seed": seed,
            "inputs": [p.tolist() for p in parts],
            "inputs_hex": [p.tobytes().hex() for p in parts],
            "result_hex": res.tobytes().hex(),
        })
    return out


def runtime_digests():
    """The reference RUNTIME (forked workers over TCP) on a few grids: pins
    that runtime == replay for the exact cases the GPU tests replay."""
    out = {}
    lengths = (0, 1, 17, 1000)
    for n, dims in [(2, (2,)), (4, (2, 2)), (4, (4,)), (8, (2, 4)), (8, (2, 2, 2)), (8, (8,)), (6, (3, 2))]:
        for dtype in ("f32", "i64"):
            w = Workload(lengths=lengths, dtype=dtype, seed=n)
            rep = launch(n, dims, w, timeout_s=120)
            assert rep.ok, rep.error
            for it, length in enumerate(lengths):
                digs = {rep.results[r].digests[it] for r in range(n)}
                assert len(digs) == 1
                out[f"{dims_key(dims)}:{dtype}:{it}:{length}"] = digs.pop()
            out[f"{dims_key(dims)}:{dtype}:bytes_sent"] = [rep.results[r].bytes_sent for r in range(n)]
    return out


def large_digests():
    """Full-size configs 1/2 (25.6 M fp32, N=8) and exact ResNet-50 size."""
    out = {}
    for length in (25_600_000, 25_557_032):
        w = Workload(lengths=(length,), dtype="f32", seed=0)
        parts = [generate_input(w, 0, r, length) for r in range(8)]
        for dims in [(2, 4), (2, 2, 2), (8,), (4, 2)]:
            t0 = time.time()
            res = replay(multiring_schedule(Grid(dims=dims), length), [p.copy() for p in parts])[0]
            out[f"{dims_key(dims)}:f32:seed0:{length}"] = sha(res)
            print(f"  large {dims} {length}: {time.time() - t0:.1f}s", flush=True)
        out[f"inputs:f32:seed0:{length}"] = [sha(p) for p in parts]
    # i64 at full size too (exact integer sum)
    length = 25_600_000
    w = Workload(lengths=(length,), dtype="i64", seed=0)
    parts = [generate_input(w, 0, r, length) for r in range(8)]
    res = replay(multiring_schedule(Grid(dims=(2, 2, 2)), length), [p.copy() for p in parts])[0]
    out[f"2x2x2:i64:seed0:{length}"] = sha(res)
    return out


def planner_golden():
    out = {}
    topo_dir = "/root/reference/pkg/sample_topologies"
    for name in ("host4.json", "two_switch_4dev.json", "cluster_4x16x4.json"):
        t = topology.load_topology(os.path.join(topo_dir, name))
        devs = t.devices()
        cases = [(None, None, 0.35), ((2, 2), None, 0.1024)]
        if len(devs) >= 8:
            cases += [("first8", None, 0.1024), ("first8:2x4", (2, 4), 0.1024)]
        for tag, dims, size in cases:
            use = devs
            if tag and str(tag).startswith("first8"):
                use = devs[:8]
            if dims is not None and len(use) != int(np.prod(dims)):
                continue
            p = plan(t, use, size, dims=dims)
            out[f"{name}:{tag}:{size}"] = json.loads(p.to_json())
        out[f"{name}:serialize"] = t.serialize()
    for lat in (0.0, 5e-6, 5e-4):
        t = topology.build_tree(8, bandwidths_gbps=(900.0,), latencies_s=(lat,))
        p = plan(t, t.devices(), 0.1024)
        out[f"b200star:{lat}"] = json.loads(p.to_json())
    t = topology.build_tree(4, 2, 1, (20.0, 10.0), (0.0005, 0.0005))
    out["2hostx4"] = json.loads(plan(t, t.devices(), 0.1024).to_json())
    out["2hostx4:2x4"] = json.loads(plan(t, t.devices(), 0.1024, dims=(2, 4)).to_json())
    t = topology.build_tree(4, 16, 4, (20.0, 10.0, 9.5), (0.0005, 0.0005, 0.0005))
    out["cluster:auto:0.35"] = json.loads(plan(t, t.devices(), 0.35).to_json())
    out["factorizations"] = {str(n): [list(f) for f in factorizations(n, k)]
                             for n in (1, 2, 6, 7, 8, 12, 16, 36, 60) for k in (3,)}
    out["partner_pairs"] = {dims_key(d): sorted(list(p) for p in ring_partner_pairs(Grid(dims=d)))
                            for d in [(2, 2), (2, 4), (2, 2, 2), (8,), (3, 2)]}
    cm = {}
    cm["ring_reduction_time"] = vars(costmodel.ring_reduction_time(0.35, 256, 9.5, 0.0005))["total"]
    cm["allreduce_time"] = costmodel.allreduce_time(0.35, 256, 9.5, 0.0005).total
    cm["multiring_time"] = costmodel.multiring_time(0.35, [(4, 20.0), (16, 10.0), (4, 9.5)], 0.0005).total
    cm["multiring_b200_2x2x2"] = costmodel.multiring_time(0.1024, [(2, 900.0), (2, 900.0), (2, 900.0)], 0.0).total
    cm["parameter_server"] = costmodel.parameter_server_time(0.35, 256, 10.0).seconds
    out["costmodel"] = cm
    return out


def main():
    t0 = time.time()
    docs = {
        "chunk_kats.json": chunk_kats(),
        "schedules.json": schedule_dumps(),
        "owned_regions.json": owned_regions(),
        "input_digests.json": input_digests(),
        "small_vectors.json": small_vectors(),
        "planner.json": planner_golden(),
    }
    print(f"basic fixtures {time.time() - t0:.1f}s", flush=True)
    docs["replay_digests.json"] = replay_digests()
    print(f"replay digests {time.time() - t0:.1f}s", flush=True)
    docs["runtime_digests.json"] = runtime_digests()
    print(f"runtime digests {time.time() - t0:.1f}s", flush=True)
    docs["large_digests.json"] = large_digests()
    print(f"large digests {time.time() - t0:.1f}s", flush=True)
    for name, doc in docs.items():
        with open(os.path.join(OUT, name), "w", encoding="utf-8") as fh:
            json.dump({"generator": "tests/golden/make_golden.py (imports /root/reference/pkg/src ringbox 0.1.0)",
                       "data": doc}, fh, indent=1, sort_keys=True)
            fh.write("\n")
    print("done", time.time() - t0)


if __name__ == "__main__":
    main()
