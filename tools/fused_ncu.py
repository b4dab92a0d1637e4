"""Profilable view of the product's FUSED kernel (single process, 2 or 4 GPUs).

ncu must never wrap the multi-rank run (replaying a kernel that waits on a
peer's flags would hang).  This harness launches the SAME rbx_fused_kernel the
per-rank path uses (rbx_fused_harness: the plan and arguments of rank r's share
of a FUSED allreduce, flag protocol off) from one process: rank 0's share on
cuda:0 and rank 1's share on cuda:1, each reading the other's buffer and
writing its result into both over NVLink -- the bidirectional traffic pattern
of a real N=2 call, minus the entry/exit handshakes.  Outside ncu the two
launches run concurrently and are timed; the result is checked bit-exact.

With --gpus 4 the shares of a (2,2) allreduce run on cuda:0..3 the same way.

  python tools/fused_ncu.py [--gpus 2] [--elems 25600000] [--iters 20]
  ncu --set full ... python tools/fused_ncu.py --iters 1
"""

import argparse
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--elems", type=int, default=25_600_000)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--nblocks", type=int, default=148)
    ap.add_argument("--gpus", type=int, default=2, choices=[2, 4])
    args = ap.parse_args()
    import torch

    from paper_1708_02188_b200 import _native
    from paper_1708_02188_b200.runtime import Workload, generate_input

    L = _native.lib()
    G = args.gpus
    for a in range(G):
        for b in range(G):
            if a != b:
                _native.check(L.rbx_enable_peer_access(a, b))
    n = args.elems
    wl = Workload(lengths=(n,), dtype="f32", seed=0)
    parts = [generate_input(wl, 0, r, n) for r in range(G)]
    bufs = [torch.from_numpy(parts[r]).to(f"cuda:{r}") for r in range(G)]
    ptrs = (ctypes.c_void_p * G)(*[b.data_ptr() for b in bufs])
    grid = [2] if G == 2 else [2, 2]
    dims = _native.ints(grid)
    streams = [torch.cuda.current_stream(r) for r in range(G)]

    def launch(r):
        torch.cuda.set_device(r)
        _native.check(L.rbx_fused_harness(dims, len(grid), r, ptrs, n, 0, args.nblocks, 512,
                                          ctypes.c_void_p(streams[r].cuda_stream)))

    for r in range(G):
        launch(r)
    for r in range(G):
        torch.cuda.synchronize(r)
    if G == 2:
        # grid (2,): every element is x0 + x1 (one IEEE add, commutative): torch's add is the reference order
        want = torch.from_numpy(parts[0]) + torch.from_numpy(parts[1])
        ok = all(torch.equal(b.cpu(), want) for b in bufs)
    else:
        # grid (2,2): every region is a nested pair fold; fp32 rounding differs from float64 by < 1e-5
        want = sum(torch.from_numpy(p).double() for p in parts)
        got = [b.cpu() for b in bufs]
        ok = all(torch.equal(g, got[0]) for g in got) and bool(((got[0].double() - want).abs() < 1e-4).all())
    ts = []
    for _ in range(args.iters):
        ev = []
        for r in range(G):
            torch.cuda.set_device(r)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(streams[r])
            launch(r)
            e.record(streams[r])
            ev.append((s, e))
        for r in range(G):
            torch.cuda.synchronize(r)
        ts.append(max(s.elapsed_time(e) for s, e in ev) / 1e3)
    t = statistics.median(ts)
    S = 2 * (G - 1) / G * n * 4
    kern = "rbx_fused_kernel<float,2,1,2,1>" if G == 2 else "rbx_fused_kernel<float,4,2,4,1>"
    print(json.dumps({"harness": f"{kern}: rank r's share on cuda:r for r < {G}, concurrent, flag protocol off",
                      "grid": grid, ("bit_exact_vs_reference_order" if G == 2 else "consistent_and_close"): ok,
                      "elems": n, "nblocks": args.nblocks, "event_us": round(t * 1e6, 1),
                      "bus_bytes_per_direction": S, "busbw_gbs": round(S / t / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
