"""Tuning sweep for the multi-GPU kernel (run under torchrun, one process per GPU).

  torchrun --nproc-per-node N tools/tune_multi.py [--elems 25600000] [--dims 2x2x2]

Prints one line per (mode, nblocks, threads, size) with the max-over-ranks
busbw.  Diagnostic only; bench.py is the contract.
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--elems", default="25600000")
    ap.add_argument("--dims", default=None)
    ap.add_argument("--modes", default="fused,fused_pull,ring_dims")
    ap.add_argument("--ops", default="allreduce", help="allreduce,reduce_scatter,allgather")
    ap.add_argument("--nblocks", default="148,296")
    ap.add_argument("--threads", default="256,512")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--flush", type=int, default=1)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import RankContext

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    dims = tuple(int(x) for x in args.dims.split("x")) if args.dims else {2: (2,), 4: (2, 2), 8: (2, 2, 2)}[world]
    scratch = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    for nb in [int(x) for x in args.nblocks.split(",")]:
        for th in [int(x) for x in args.threads.split(",")]:
            ctx = RankContext(rank, Grid(dims), device=rank, nblocks=nb, threads=th, blocking=False)
            for n in [int(x) for x in args.elems.split(",")]:
                work = ctx.empty(n, "f32")
                work.normal_()
                for op in args.ops.split(","):
                    for mode in args.modes.split(","):
                        ts = []
                        for it in range(args.iters + 3):
                            if args.flush:
                                scratch.fill_(1.0)
                                scratch.sum()
                            torch.cuda._sleep(100_000)
                            ctx.barrier()
                            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                            s.record(stream)
                            ctx.collective(op, work, mode=mode)
                            e.record(stream)
                            torch.cuda.synchronize()
                            if it >= 3:
                                ts.append(s.elapsed_time(e))
                            work.mul_(0.125)
                        ctx.check()
                        t = torch.tensor(ts, device=dev)
                        dist.all_reduce(t, op=dist.ReduceOp.MAX)
                        med = t.median().item() / 1e3
                        # bus bytes: 2(N-1)/N S for allreduce, (N-1)/N S for either half alone
                        f = 2 if op == "allreduce" else 1
                        bw = f * (world - 1) / world * n * 4 / med / 1e9
                        if rank == 0:
                            print(f"op={op:14s} mode={mode:10s} nb={ctx.nblocks:4d}(req {nb:4d}) th={th:4d} n={n:10d} "
                                  f"t={med * 1e6:9.1f}us busbw={bw:7.1f} GB/s", flush=True)
            ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
