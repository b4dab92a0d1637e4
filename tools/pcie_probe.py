"""Host<->device PCIe ceiling for bench.py's e2e leg.

  python tools/pcie_probe.py                      (1 GPU)
  torchrun --nproc-per-node N tools/pcie_probe.py (N GPUs at once)

Per rank: pinned host buffers of --mb MB, timed with CUDA events, all ranks
released together (NCCL barrier), max over ranks.  Cases: H2D alone, D2H
alone, H2D + D2H at once on two streams, and the e2e pipeline shape (window k:
H2D -> D2H, k+1's H2D overlapping k's D2H) for several window counts.
Prints one JSON line per case on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import bind_host_to_gpu  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--mb", type=float, default=102.4)
    p.add_argument("--iters", type=int, default=8)
    p.add_argument("--no-bind", action="store_true")
    a = p.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cores = [] if a.no_bind else bind_host_to_gpu(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    nbytes = int(a.mb * 1e6) // 16 * 16
    n = nbytes // 4
    src = torch.randn(n).pin_memory()
    dst = torch.empty(n).pin_memory()
    dbuf = torch.empty(n, device=dev)
    dbuf2 = torch.empty(n, device=dev)
    main_s = torch.cuda.current_stream(dev)
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def timed(body):
        out = []
        for _ in range(a.iters + 2):
            sync_all()
            torch.cuda._sleep(50_000)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(main_s)
            s_in.wait_event(s)
            s_out.wait_event(s)
            body()
            for st in (s_in, s_out):
                ev = torch.cuda.Event()
                ev.record(st)
                main_s.wait_event(ev)
            e.record(main_s)
            torch.cuda.synchronize()
            out.append(s.elapsed_time(e))
        out = out[2:]
        t = torch.tensor([statistics.median(out)], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def h2d():
        with torch.cuda.stream(s_in):
            dbuf.copy_(src, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s_out):
            dst.copy_(dbuf2, non_blocking=True)

    def both():
        h2d()
        d2h()

    def pipe(chunks):
        bounds = [(n * k // chunks, n * (k + 1) // chunks) for k in range(chunks)]

        def body():
            for lo, hi in bounds:
                with torch.cuda.stream(s_in):
                    dbuf[lo:hi].copy_(src[lo:hi], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s_in)
                s_out.wait_event(ev)
                with torch.cuda.stream(s_out):
                    dst[lo:hi].copy_(dbuf[lo:hi], non_blocking=True)
        return body

    cases = [("h2d", h2d, nbytes, 0), ("d2h", d2h, 0, nbytes), ("h2d+d2h", both, nbytes, nbytes)]
    for c in (4, 8, 16, 32, 64, 128):
        cases.append((f"pipe{c}", pipe(c), nbytes, nbytes))
    for name, body, bi, bo in cases:
        ms = timed(body)
        if rank == 0:
            print(json.dumps({"case": name, "world": world, "bytes": nbytes, "ms": round(ms, 4),
                              "h2d_gbs": round(bi / ms / 1e6, 2), "d2h_gbs": round(bo / ms / 1e6, 2),
                              "bound_cores": len(cores)}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
