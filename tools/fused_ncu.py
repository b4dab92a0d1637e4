"""Profilable view of the product's FUSED kernel (single process, 2 GPUs).

ncu must never wrap the multi-rank run (replaying a kernel that waits on a
peer's flags would hang).  This harness launches the SAME rbx_fused_kernel the
per-rank path uses (rbx_fused_harness: the plan and arguments of rank r's share
of a FUSED allreduce, flag protocol off) from one process: rank 0's share on
cuda:0 and rank 1's share on cuda:1, each reading the other's buffer and
writing its result into both over NVLink -- the bidirectional traffic pattern
of a real N=2 call, minus the entry/exit handshakes.  Outside ncu the two
launches run concurrently and are timed; the result is checked bit-exact.

  python tools/fused_ncu.py [--elems 25600000] [--iters 20]
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
    args = ap.parse_args()
    import torch

    from paper_1708_02188_b200 import _native
    from paper_1708_02188_b200.runtime import Workload, generate_input

    L = _native.lib()
    _native.check(L.rbx_enable_peer_access(0, 1))
    _native.check(L.rbx_enable_peer_access(1, 0))
    n = args.elems
    wl = Workload(lengths=(n,), dtype="f32", seed=0)
    parts = [generate_input(wl, 0, r, n) for r in range(2)]
    bufs = [torch.from_numpy(parts[0]).to("cuda:0"), torch.from_numpy(parts[1]).to("cuda:1")]
    ptrs = (ctypes.c_void_p * 2)(bufs[0].data_ptr(), bufs[1].data_ptr())
    dims = _native.ints([2])
    streams = [torch.cuda.current_stream(0), torch.cuda.current_stream(1)]

    def launch(r):
        torch.cuda.set_device(r)
        _native.check(L.rbx_fused_harness(dims, 1, r, ptrs, n, 0, args.nblocks, 512,
                                          ctypes.c_void_p(streams[r].cuda_stream)))

    for r in (0, 1):
        launch(r)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    # grid (2,): every element is x0 + x1 (one IEEE add, commutative), so torch's add is the reference order
    want = torch.from_numpy(parts[0]) + torch.from_numpy(parts[1])
    ok = all(torch.equal(b.cpu(), want) for b in bufs)
    ts = []
    for _ in range(args.iters):
        ev = []
        for r in (0, 1):
            torch.cuda.set_device(r)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(streams[r])
            launch(r)
            e.record(streams[r])
            ev.append((s, e))
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        ts.append(max(s.elapsed_time(e) for s, e in ev) / 1e3)
    t = statistics.median(ts)
    S = n * 4
    print(json.dumps({"harness": "rbx_fused_kernel<float,2,1,1>: rank 0's share on cuda:0 and rank 1's on cuda:1, "
                                 "concurrent, flag protocol off",
                      "bit_exact_vs_reference_order": ok, "elems": n, "nblocks": args.nblocks,
                      "event_us": round(t * 1e6, 1), "bus_bytes_per_direction": S,
                      "busbw_gbs": round(S / t / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
