"""Does a rank process exit cleanly when it never closes its RankContext?
(diagnostic)  torchrun --nproc-per-node 2 tools/exit_probe.py [--close 0|1] [--graph 0|1]"""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--close", type=int, default=0)
    ap.add_argument("--graph", type=int, default=0)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import RankContext

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    gloo = dist.new_group(backend="gloo")
    ctx = RankContext(rank, Grid((world,)), group=gloo, device=rank, blocking=False)
    t = ctx.empty(1 << 20, "f32")
    t.fill_(1.0)
    ctx.collective("allreduce", t)
    if args.graph:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            ctx.collective("allreduce", t)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            ctx.collective("allreduce", t)
        g.replay()
    ctx.synchronize()
    if args.close:
        ctx.close()
    t0 = time.time()
    dist.destroy_process_group()
    print(f"rank {rank}: destroy_process_group took {time.time() - t0:.2f} s", flush=True)


if __name__ == "__main__":
    main()
