"""Direct launch vs CUDA-graph replay of one allreduce (diagnostic).
  torchrun --nproc-per-node N tools/graph_probe.py
Per iteration: L2 flush + device spin, device flag barrier, events around the
collective (direct) or around graph.replay(); per-iteration max over ranks."""

import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import RankContext

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    dims = {2: (2,), 4: (2, 2), 8: (2, 2, 2)}[world]
    ctx = RankContext(rank, Grid(dims), device=rank, blocking=False)
    n = int(os.environ.get("GRAPH_ELEMS", "25600000"))
    work = ctx.empty(n, "f32")
    work.fill_(1.0)
    scratch = torch.empty(64 << 20, device=dev)
    stream = torch.cuda.current_stream(dev)

    def measure(fn, iters=12):
        ev = []
        for _ in range(iters):
            scratch.fill_(1.0)
            torch.cuda._sleep(1_000_000)
            ctx.barrier()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            fn()
            e.record(stream)
            ev.append((s, e))
        torch.cuda.synchronize()
        ctx.check()
        t = torch.tensor([s.elapsed_time(e) * 1e3 for s, e in ev], device=dev)
        mine = t.tolist()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [round(x, 1) for x in t.tolist()], [round(x, 1) for x in mine]

    direct = measure(lambda: ctx.collective("allreduce", work))
    side = torch.cuda.Stream(dev)
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        ctx.collective("allreduce", work)
    stream.wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ctx.collective("allreduce", work)
    replay = measure(g.replay)
    direct2 = measure(lambda: ctx.collective("allreduce", work))
    every = [None] * world
    dist.all_gather_object(every, {"direct_mine": direct[1], "replay_mine": replay[1]})
    if rank == 0:
        print(json.dumps({"n": n, "world": world, "pdl": os.environ.get("RBX_PDL", "1"),
                          "direct_max_us": direct[0], "replay_max_us": replay[0], "direct_after_capture_max_us": direct2[0],
                          "median": {"direct": statistics.median(direct[0]), "replay": statistics.median(replay[0]),
                                     "direct_after": statistics.median(direct2[0])},
                          "per_rank": every}), flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
